set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "bin_parity or fit_parity_c1 or ragged or c3_full or predict_and_recommend or cv_hand" > gpurun_out/k_pytest.log 2>&1; tail -3 gpurun_out/k_pytest.log
python tools/profile_fit.py --trees 2 > gpurun_out/k_prof.json 2>&1; grep -A3 '"codes"' gpurun_out/k_prof.json
