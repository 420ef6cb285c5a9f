#!/bin/bash
# end-of-round validation of HEAD on one B200: build, smoke, GPU tests, bench (all legs), the
# reference arm, configs[3] at N=1, the sharded path, and the ncu evidence (launch list, steady-state
# --set full, DRAM bytes per row, NVTX-filtered capture)
TAG=${1:-r02z}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/${TAG}_gpu_tests.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 1500 python bench.py --strong --no-cv --no-wg --no-c5 --no-rf --no-cpu-baseline --steps 2 > gpurun_out/${TAG}_strong.json 2> gpurun_out/${TAG}_strong.err
timeout 900 python bench.py --nccl1 --no-cv --no-wg --no-c5 --no-rf --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_nccl1.json 2> gpurun_out/${TAG}_nccl1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches_ncu.csv \
  python bench.py --steps 2 --warmup 3 --no-cv --no-wg --no-c5 --no-rf --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
timeout 1200 python tools/prof_traffic.py ${TAG}t > gpurun_out/${TAG}_traffic.log 2>&1
timeout 1500 bash tools/prof_late.sh ${TAG}f 100 102 > gpurun_out/${TAG}_prof.log 2>&1
rm -f gpurun_out/${TAG}f_sass_*.csv
# NVTX ranges: capture only the partition launches inside "level 3" of plain-launch trees
timeout 600 ncu --nvtx --nvtx-include "llmpilot_fit/tree/level 3/" --metrics gpu__time_duration.sum \
  --clock-control none -c 8 --csv python tools/profile_fit.py --trees 2 --repeat 1 > gpurun_out/${TAG}_nvtx.csv 2>&1
timeout 600 ncu --nvtx --print-nvtx-rename kernel --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  python tools/profile_fit.py --trees 1 --repeat 1 > gpurun_out/${TAG}_nvtx_all.csv 2>&1
