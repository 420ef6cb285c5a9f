#!/bin/bash
# compute-sanitizer runs of tools/sanitize_fit.py (graph mode: memcheck, synccheck; plain launches:
# racecheck, initcheck) -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for T in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize_fit.py > gpurun_out/sanitize_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$T.log
done
for T in racecheck initcheck; do
  SANITIZE_PLAIN=1 timeout 2400 compute-sanitizer --tool $T --error-exitcode 9 python tools/sanitize_fit.py > gpurun_out/sanitize_$T.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$T.log
done
tail -n 3 gpurun_out/sanitize_*.log
