#!/bin/bash
# recommendation grid predictor: parity tests, then the bench's predict (C3 sweep) and C5 legs with
# the grid predictor (default) and the per-row walk (LLMP_PRED_GRID=0), interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pg_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "recommend or c5 or predict or toy or cv_parity_c1 or cv_hand" 2>&1 | tail -3 > gpurun_out/pg_tests.log
rm -f gpurun_out/pg_ab.txt
for R in 1 2; do for E in 1 0; do
  LLMP_PRED_GRID=$E timeout 900 python bench.py --steps 3 --no-cv --no-wg --no-rf --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/pg_b.json
  python - $E >> gpurun_out/pg_ab.txt <<'PY'
import json,sys
d=json.load(open("gpurun_out/pg_b.json"))
c=d.get("c5_sweep",{})
print(f"LLMP_PRED_GRID={sys.argv[1]}  step {d['ms_per_step']:.2f} ms  predict(C3 sweep) {d['predict']['value']/1e6:.1f} M rows/s ({d['predict']['ms_per_step']:.3f} ms)  C5 {c.get('value',0)/1e6:.1f} M rows/s (recommend {c.get('recommend_call_ms',0):.3f} ms)")
PY
done; done
cat gpurun_out/pg_tests.log gpurun_out/pg_ab.txt
