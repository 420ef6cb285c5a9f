#!/bin/bash
# A/B/C of an environment switch: parity subset, then the bench fit leg per setting (interleaved twice)
NAME=$1; A=$2; B=$3; C=$4; K=${5:-"fit_parity or variants"}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" 2>&1 | tail -3 > gpurun_out/${NAME}_tests.log
rm -f gpurun_out/${NAME}_ab.txt
for E in "$A" "$B" "$C" "$A" "$B" "$C"; do
  env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-cv --no-c5 --no-rf --no-wg --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/${NAME}_b.json
  python - "$E" "$NAME" <<'PY' >> gpurun_out/${NAME}_ab.txt
import json,sys
d=json.load(open(f"gpurun_out/{sys.argv[2]}_b.json"))
k=d["kernels"]
print(f"{sys.argv[1]:24s} ms/step {d['ms_per_step']:.2f} value {d['value']/1e9:.2f} G  part {k['partition']['ms_avg']*1e3:.1f} us  hist {k['hist_level']['ms_avg']*1e3:.1f} us  split {k['split']['ms_avg']*1e3:.1f} us  upd {k['update']['ms_avg']*1e3:.1f} us")
PY
done
