#!/bin/bash
# ncu --set full of the batched small-fit kernel (C2 leave-one-LLM-out, 50 trees depth 6)
TAG=${1:-sf}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/cv50.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2410_02425_b200 as lp, synth
d = synth.make("C2")
ctx = lp.Context(0, torch.cuda.current_stream())
lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [lp.hparams(n_trees=50, max_depth=6)], 100.0, 50.0, 200, d.cost)
PY
ncu --set full --clock-control none --import-source on --kernel-name regex:"k_fit_small" -c 1 -o /tmp/$TAG python /tmp/cv50.py > gpurun_out/${TAG}_run.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/${TAG}_sass.csv > gpurun_out/${TAG}_stalls.txt 2>&1
python tools/ncu_exec_groups.py gpurun_out/${TAG}_sass.csv 25 > gpurun_out/${TAG}_exec.txt 2>&1
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
rm -f gpurun_out/${TAG}_sass.csv
