#!/bin/bash
# ncu --set full of one kernel (regex) over the launches of one late tree of a C3 fit (paired plain
# launches, tools/profile_fit.py), then the per-launch summary, stall and executed-instruction breakdowns.
#   bash tools/prof_kernel.sh TAG KREGEX PER_TREE [TREE] [TREES] [LAUNCHES...]
TAG=$1; KRE=$2; PER=$3; TREE=${4:-10}; TREES=${5:-12}; shift 5; LS=${@:-"0 2 4 6"}
OUT=gpurun_out/$TAG
mkdir -p gpurun_out
REP=/tmp/$TAG.ncu-rep
rm -f $REP
ncu --set full --clock-control none --import-source on --kernel-name regex:"$KRE" \
    --launch-skip $((TREE * PER)) -c $PER -o /tmp/$TAG \
    python tools/profile_fit.py --trees $TREES --repeat 1 > ${OUT}_fit.log 2>&1
python tools/ncu_summary.py $REP $OUT "tree $TREE of a $TREES-tree C3 fit, both targets paired ($TAG)"
for i in $LS; do
  ncu -i $REP --page source --csv --print-source sass --kernel-name "regex:$KRE" --launch-skip $i --launch-count 1 \
      > ${OUT}_sass_$i.csv 2>/dev/null
  python tools/ncu_stalls.py ${OUT}_sass_$i.csv > ${OUT}_stalls_$i.txt 2>&1
  python tools/ncu_exec_groups.py ${OUT}_sass_$i.csv > ${OUT}_exec_$i.txt 2>&1
  rm -f ${OUT}_sass_$i.csv
done
ncu -i $REP --page raw --csv > ${OUT}_raw.csv 2>/dev/null
