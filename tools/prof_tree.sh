#!/bin/bash
# ncu --set full of tree 0 (target 0) of a C3 fit + SASS/stall source pages of one deep-level launch
# of each hot kernel.  Run on the GPU box:  bash tools/prof_tree.sh TAG [extra env...]
set -x
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p gpurun_out
REP=/tmp/$TAG.ncu-rep
rm -f $REP
ncu --set full --clock-control none --import-source on \
    --kernel-name regex:"k_pcount|k_pscatter|k_hist|k_split|k_part" -c ${NCU_COUNT:-31} -o /tmp/$TAG \
    python tools/profile_fit.py --trees 2 --repeat 1 > ${OUT}_fit.log 2>&1
python tools/ncu_summary.py $REP $OUT "tree 0 of target 0 ($TAG)"
for spec in "k_part:4" "k_hist:5" "k_hist:7" "k_hist:8" "k_split3:5" "${EXTRA_SASS}"; do
  [ -z "$spec" ] && continue
  k=${spec%%:*}; s=${spec##*:}
  ncu -i $REP --page source --csv --print-source sass --kernel-name "regex:$k" --launch-skip $s --launch-count 1 \
      > ${OUT}_sass_${k}_${s}.csv 2>/dev/null
  python tools/ncu_stalls.py ${OUT}_sass_${k}_${s}.csv > ${OUT}_stalls_${k}_${s}.txt 2>&1
done
ncu -i $REP --page details --csv > ${OUT}_details.csv 2>/dev/null
ls -la gpurun_out
