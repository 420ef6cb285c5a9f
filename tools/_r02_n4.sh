set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n4_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -k "wide_bins or bins_limits or cv or bin_parity or random_forest" > gpurun_out/n4_pytest.log 2>&1; tail -15 gpurun_out/n4_pytest.log
