set -x
TAG=${TAG:-h3c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h3_build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "histogram_parity or fit_parity or sharded or cv_parity_c1" > gpurun_out/h3_pytest.log 2>&1; tail -3 gpurun_out/h3_pytest.log
timeout 600 python bench.py --no-wg --no-cv --no-e2e --no-cpu-baseline > gpurun_out/h3_bench.json 2> gpurun_out/h3_bench.err; head -c 300 gpurun_out/h3_bench.json
bash tools/prof_kernel.sh $TAG "k_hist3" 7 10 12 0 2 4 5 6
