set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -k "fit_parity or variants or sharded or c3_full or sequential_mode" > gpurun_out/u_pytest.log 2>&1; tail -3 gpurun_out/u_pytest.log
timeout 600 python bench.py --no-wg --no-cv --no-e2e --no-cpu-baseline --no-c5 > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err; head -c 200 gpurun_out/u_bench.json
LLMP_UPD=2 timeout 600 python bench.py --no-wg --no-cv --no-e2e --no-cpu-baseline --no-c5 > gpurun_out/u2_bench.json 2> gpurun_out/u2_bench.err; head -c 200 gpurun_out/u2_bench.json
