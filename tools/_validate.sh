set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/v_pytest.log 2>&1; tail -3 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; cat gpurun_out/v_bench.json | head -c 600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_ref.json 2> gpurun_out/v_ref.err; head -c 400 gpurun_out/v_ref.json
