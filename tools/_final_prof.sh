# end-of-round evidence for HEAD: steady-state ncu --set full capture + the bench command's launch list
timeout 1500 bash tools/prof_late.sh r01n 100 102 > gpurun_out/r01n_prof.log 2>&1; tail -3 gpurun_out/r01n_prof.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01n_launches_ncu.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/r01n_bench_under_ncu.log 2>&1; wc -l gpurun_out/r01n_launches_ncu.csv
rm -f gpurun_out/*.csv.tmp
