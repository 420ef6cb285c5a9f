timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; tail -2 gpurun_out/ab_pytest.log
timeout 1500 python tools/ab_fit.py --trees 200 --reps 3 --rounds 3 -- "" "AB_ROOT=$PWD/_ab_base" > gpurun_out/ab_fit.txt 2>&1; cat gpurun_out/ab_fit.txt
