set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/prof_c5.py > gpurun_out/c5g_time.json 2>&1; cat gpurun_out/c5g_time.json
ncu --set full --clock-control none --import-source on --kernel-name regex:"k_predict" -c 1 -o /tmp/c5p python tools/prof_c5.py --reps 1 > gpurun_out/c5g_ncu_run.log 2>&1
ncu -i /tmp/c5p.ncu-rep --page source --csv --print-source sass > gpurun_out/c5g_sass.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/c5g_sass.csv > gpurun_out/c5g_stalls.txt 2>&1
python tools/ncu_exec_groups.py gpurun_out/c5g_sass.csv 20 > gpurun_out/c5g_exec.txt 2>&1
ncu -i /tmp/c5p.ncu-rep --page details --csv > gpurun_out/c5g_details.csv 2>/dev/null
rm -f gpurun_out/c5g_sass.csv
