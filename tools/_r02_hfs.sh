#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "sharded or multi_rank or variants" 2>&1 | tail -3 > gpurun_out/hfs_tests.log
rm -f gpurun_out/hfs_ab.txt
for E in "LLMP_HFIX=1" "LLMP_HFIX=0" "LLMP_HFIX=1"; do
  env $E timeout 600 python bench.py --nccl1 --steps 5 --warmup 3 --no-cv --no-c5 --no-rf --no-wg --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/hfs_b.json
  python - "$E" <<'PY' >> gpurun_out/hfs_ab.txt
import json,sys
d=json.load(open("gpurun_out/hfs_b.json"))
k=d["kernels"]
print(f"nccl1 {sys.argv[1]:14s} ms/step {d['ms_per_step']:.2f} value {d['value']/1e9:.2f} G  part {k['partition']['ms_avg']*1e3:.1f}  hist {k['hist_level']['ms_avg']*1e3:.1f}  split {k['split']['ms_avg']*1e3:.1f}  upd {k['update']['ms_avg']*1e3:.1f} us")
PY
done
