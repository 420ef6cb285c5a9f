set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "c5_sweep or grid5" > gpurun_out/b_pytest.log 2>&1; tail -3 gpurun_out/b_pytest.log
timeout 900 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; head -c 300 gpurun_out/b_bench.json; tail -3 gpurun_out/b_bench.err
timeout 1200 python bench.py --strong --no-cv --no-wg --no-c5 --no-cpu-baseline --steps 2 > gpurun_out/b_strong.json 2> gpurun_out/b_strong.err; head -c 300 gpurun_out/b_strong.json; tail -3 gpurun_out/b_strong.err
