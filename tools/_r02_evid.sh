#!/bin/bash
# degenerate-input parity, then the DRAM-bytes-per-row capture and a steady-state --set full capture of HEAD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "degenerate or save_load" 2>&1 | tail -3 > gpurun_out/evid_tests.log
timeout 1200 python tools/prof_traffic.py r02t > gpurun_out/r02t_traffic.log 2>&1
timeout 1500 bash tools/prof_late.sh r02f 100 102 > gpurun_out/r02f_prof.log 2>&1
rm -f gpurun_out/r02f_sass_*.csv
