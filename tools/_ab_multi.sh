#!/bin/bash
# A/B of several environment settings on the bench fit leg (interleaved, 2 rounds), after a parity subset
#   bash tools/_ab_multi.sh NAME "PYTEST_K" "ENV_A" "ENV_B" ...   ("AB_ROOT=_abv/X": another build, tools/build_variant.sh)
NAME=$1; K=$2; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${NAME}_build.log 2>&1
if [ -n "$K" ]; then timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" 2>&1 | tail -3 > gpurun_out/${NAME}_tests.log; fi
rm -f gpurun_out/${NAME}_ab.txt
for R in 1 2; do
for E in "$@"; do
  B=bench.py
  case "$E" in AB_ROOT=*) AR=${E#AB_ROOT=}; cp bench.py $AR/; ln -sfn $(pwd)/profiles $AR/profiles; B=$AR/bench.py;; esac
  env $E timeout 600 python $B --steps 5 --warmup 3 --no-cv --no-c5 --no-rf --no-wg --no-cpu-baseline --no-e2e 2>gpurun_out/${NAME}_b.err | tail -1 > gpurun_out/${NAME}_b.json
  python - "$E" "$NAME" <<'PY' >> gpurun_out/${NAME}_ab.txt
import json,sys
try:
    d=json.load(open(f"gpurun_out/{sys.argv[2]}_b.json"))
    k=d["kernels"]
    print(f"{sys.argv[1]:24s} ms/step {d['ms_per_step']:.2f} value {d['value']/1e9:.2f} G  part {k['partition']['ms_avg']*1e3:.1f} us  hist {k['hist_level']['ms_avg']*1e3:.1f} us  split {k['split']['ms_avg']*1e3:.1f} us  upd {k['update']['ms_avg']*1e3:.1f} us")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
done
cat gpurun_out/${NAME}_ab.txt
