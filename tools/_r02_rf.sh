set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rf_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -k "random_forest or fit_parity_c1 or importance or cv_parity_c1 or hand" > gpurun_out/rf_pytest.log 2>&1; tail -15 gpurun_out/rf_pytest.log
