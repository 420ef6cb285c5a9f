set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fo_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "fit_parity or variants or sharded or c3_full or random_forest or importance or sequential or predict_and" > gpurun_out/fo_pytest.log 2>&1; tail -3 gpurun_out/fo_pytest.log
for v in "" "LLMP_FOLD=0"; do
  env $v timeout 900 python bench.py --no-wg --no-cv --no-c5 --no-rf --no-cpu-baseline --no-e2e > gpurun_out/fo_$(echo $v | tr '=' '_').json 2>/dev/null
  python -c "import json,sys; j=json.load(open('gpurun_out/fo_$(echo $v | tr '=' '_').json')); print('$v', j['value']/1e9, j['fit']['ms_per_step'], {k: (v['ms_avg'], v['launches']) for k, v in j['kernels'].items() if k in ('hist_level','split','partition','update')})"
done
