set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -2 gpurun_out/f_smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/f_pytest.log 2>&1; tail -3 gpurun_out/f_pytest.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; head -c 300 gpurun_out/f_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; head -c 300 gpurun_out/f_ref.json
