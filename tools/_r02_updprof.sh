#!/bin/bash
# fused update kernel (k_hist2<UPDROOT>): ncu --set full of tree 40's update launch, per-SASS and per-CUDA-line dumps
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name regex:"k_hist2" \
    --launch-skip 81 -c 1 -o /tmp/upd python tools/profile_fit.py --trees 42 --repeat 1 > gpurun_out/upd_fit.log 2>&1
python tools/ncu_summary.py /tmp/upd.ncu-rep gpurun_out/upd "tree 40 update launch of a 42-tree C3 fit (upd)"
ncu -i /tmp/upd.ncu-rep --page source --csv --print-source sass > gpurun_out/upd_sass.csv 2>/dev/null
ncu -i /tmp/upd.ncu-rep --page source --csv --print-source cuda > gpurun_out/upd_cuda.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/upd_sass.csv > gpurun_out/upd_stalls.txt 2>&1
python tools/ncu_exec_groups.py gpurun_out/upd_sass.csv 25 > gpurun_out/upd_exec.txt 2>&1
