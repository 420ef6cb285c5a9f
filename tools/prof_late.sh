#!/bin/bash
# ncu --set full of the histogram kernels of a LATE tree (steady state) of a C3 fit, paired plain
# launches (timing mode): skips the launches of the first TREE trees (24 matching launches per
# depth-8 tree: root, 8 splits, 7 partitions, 7 levels, fused update).
# Run on the GPU box:  bash tools/prof_late.sh TAG [TREE] [TREES]
TAG=${1:-late}
TREE=${2:-100}
TREES=${3:-102}
OUT=gpurun_out/$TAG
mkdir -p gpurun_out
REP=/tmp/$TAG.ncu-rep
rm -f $REP
ncu --set full --clock-control none --import-source on --kernel-name regex:"k_hist|k_part|k_split" \
    --launch-skip $((TREE * 24)) -c 24 -o /tmp/$TAG \
    python tools/profile_fit.py --trees $TREES --repeat 1 > ${OUT}_fit.log 2>&1
python tools/ncu_summary.py $REP $OUT "tree $TREE of a $TREES-tree C3 fit, both targets paired ($TAG)"
# report-local launch indices: k_hist* = root (0), levels 1..7, fused update (8); k_part = levels 0..6
for spec in "k_hist:1" "k_hist:3" "k_hist:5" "k_hist:7" "k_hist:8" "k_part:2" "k_part:5" "k_split3:4"; do
  k=${spec%%:*}; i=${spec##*:}
  ncu -i $REP --page source --csv --print-source sass --kernel-name "regex:$k" --launch-skip $i --launch-count 1 \
      > ${OUT}_sass_${k}_$i.csv 2>/dev/null
  python tools/ncu_stalls.py ${OUT}_sass_${k}_$i.csv > ${OUT}_stalls_${k}_$i.txt 2>&1
done
