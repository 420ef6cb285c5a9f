set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cv_build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "cv" > gpurun_out/cv_pytest.log 2>&1; tail -15 gpurun_out/cv_pytest.log
timeout 600 python tools/time_cv.py > gpurun_out/cv_time.json 2> gpurun_out/cv_time.err; cat gpurun_out/cv_time.json; tail -3 gpurun_out/cv_time.err

bash tools/prof_cv_small.sh $TAG
