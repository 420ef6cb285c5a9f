#!/bin/bash
bash tools/prof_kernel.sh h3z "k_hist3" 7 100 102 0 4 6
python - <<'PY' > gpurun_out/h3z_metrics.txt
import csv
rows=list(csv.reader(open("gpurun_out/h3z_raw.csv")))
hdr=rows[0]; data=rows[2:]
want=["gpu__time_duration.sum","dram__bytes_read.sum","lts__t_sectors_op_red.sum","lts__t_sectors_op_atom.sum","l1tex__t_requests_pipe_lsu_mem_global_op_red.sum","smsp__inst_executed.sum","l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum","smsp__inst_executed_op_ldgsts.sum","lts__t_sectors_srcunit_tex_op_read.sum"]
idx={w:[i for i,h in enumerate(hdr) if h==w] for w in want}
for r in data:
    print(" | ".join(f"{w.split('.')[0][-30:]}={r[idx[w][0]]}" for w in want if idx[w]))
PY
rm -f gpurun_out/h3z_raw.csv
