set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:"k_codes" -c 1 -o /tmp/kc python tools/profile_fit.py --trees 1 --repeat 1 > gpurun_out/kc_run.log 2>&1
ncu -i /tmp/kc.ncu-rep --page source --csv --print-source sass > gpurun_out/kc_sass.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/kc_sass.csv > gpurun_out/kc_stalls.txt 2>&1
python tools/ncu_exec_groups.py gpurun_out/kc_sass.csv 20 > gpurun_out/kc_exec.txt 2>&1
ncu -i /tmp/kc.ncu-rep --page details --csv > gpurun_out/kc_details.csv 2>/dev/null
rm -f gpurun_out/kc_sass.csv
