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
for k in 1 3 5 7; do
  ncu -i $REP --page source --csv --print-source sass --kernel-name "regex:k_hist<1>" --launch-skip $((k - 1)) \
      --launch-count 1 > ${OUT}_sass_level$k.csv 2>/dev/null
  python tools/ncu_stalls.py ${OUT}_sass_level$k.csv > ${OUT}_stalls_level$k.txt 2>&1
done
ncu -i $REP --page source --csv --print-source sass --kernel-name "regex:k_hist2<3>" --launch-count 1 \
    > ${OUT}_sass_update.csv 2>/dev/null
python tools/ncu_stalls.py ${OUT}_sass_update.csv > ${OUT}_stalls_update.txt 2>&1
