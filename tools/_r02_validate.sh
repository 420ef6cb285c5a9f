set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "stress or multi_rank or cv_hand or smoke" > gpurun_out/v_pytest_new.log 2>&1; tail -5 gpurun_out/v_pytest_new.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/v_pytest.log 2>&1; tail -3 gpurun_out/v_pytest.log
timeout 600 python bench.py --no-wg > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; head -c 400 gpurun_out/v_bench.json
