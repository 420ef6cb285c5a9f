set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/f_pytest.log 2>&1; tail -3 gpurun_out/f_pytest.log
timeout 900 python bench.py --no-wg --no-cv --no-c5 --no-rf --no-cpu-baseline > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; head -c 300 gpurun_out/f_bench.json
timeout 900 python bench.py --nccl1 --no-wg --no-cv --no-c5 --no-rf --no-cpu-baseline --no-e2e > gpurun_out/f_bench_nccl1.json 2> gpurun_out/f_bench_nccl1.err; head -c 300 gpurun_out/f_bench_nccl1.json; tail -5 gpurun_out/f_bench_nccl1.err
