timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "variants" > gpurun_out/ab_pytest.log 2>&1; tail -2 gpurun_out/ab_pytest.log
timeout 1500 python tools/ab_fit.py --trees 200 --reps 3 --rounds 3 -- "" "LLMP_HIST_SWAR=2" "AB_ROOT=$PWD/_ab_base" > gpurun_out/ab_fit.txt 2>&1; cat gpurun_out/ab_fit.txt
