#!/bin/bash
# partition A/B: parity subset, then bench fit legs per variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "fit_parity or variants or sharded or multi_rank or ragged" 2>&1 | tail -5 > gpurun_out/part_tests.log
for v in 2 1 3; do
  LLMP_PART=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cv --no-c5 --no-rf --no-wg --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/part_b$v.json
  python - "$v" <<'PY' >> gpurun_out/part_ab.txt
import json,sys
d=json.load(open(f"gpurun_out/part_b{sys.argv[1]}.json"))
k=d["kernels"]
print(f"LLMP_PART={sys.argv[1]} ms/step {d['ms_per_step']:.2f} value {d['value']/1e9:.2f} G  part {k['partition']['ms_avg']*1e3:.1f} us  hist {k['hist_level']['ms_avg']*1e3:.1f} us  split {k['split']['ms_avg']*1e3:.1f} us  upd {k['update']['ms_avg']*1e3:.1f} us")
PY
done
