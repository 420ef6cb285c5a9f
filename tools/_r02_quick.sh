set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "fit_parity or variants or c3_full or random_forest or sequential or cv_parity_c1" > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
for i in 1 2; do timeout 900 python bench.py --no-wg --no-cv --no-c5 --no-rf --no-cpu-baseline --no-e2e > gpurun_out/q_bench$i.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/q_bench$i.json')); print(j['value']/1e9, j['fit']['ms_per_step'], {k: round(v['ms_avg']*1000,1) for k, v in j['kernels'].items() if k in ('hist_level','split','partition','update')})"; done
