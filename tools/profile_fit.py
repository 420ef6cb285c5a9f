"""Profiling driver: one C3-shaped fit (10M rows x 32 features, depth 8) with a few trees, then
per-kernel-class event timings.  Used under ncu (launch list / --set full) and on its own.

    python tools/profile_fit.py [--trees 3] [--llms 78125] [--s1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_02425_b200 as lp
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--trees", type=int, default=3)
ap.add_argument("--depth", type=int, default=8)
ap.add_argument("--llms", type=int, default=78125)
ap.add_argument("--s1", action="store_true", help="S1 control data (uniform random features)")
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
if a.s1:
    d = synth.make_s1(a.llms * 128)
else:
    d = synth.make_scaled(a.llms)
dev = torch.device("cuda", 0)
X, y = torch.from_numpy(d.X).to(dev), torch.from_numpy(d.y).to(dev)
li, pi = torch.from_numpy(d.llm_id).to(dev), torch.from_numpy(d.prof_id).to(dev)
w = None if d.w is None else torch.from_numpy(d.w).to(dev)
ctx = lp.Context(0, torch.cuda.current_stream())
hp = lp.hparams(n_trees=a.trees, max_depth=a.depth, use_eq4_weights=0 if a.s1 else 1)
for r in range(a.repeat):
    ctx.reset_stats()
    ctx.set_timing(r == a.repeat - 1)
    m = lp.fit(ctx, X, y, hp, d.users_col, li, pi, d.n_llm, d.n_prof, 100.0, 50.0, w=w)
    st = ctx.stats()
    m.free()
torch.cuda.synchronize()
out = {"rows": d.n, "trees": a.trees, "depth": a.depth, "data": "S1" if a.s1 else "S2/C3"}
for k, v in st["classes"].items():
    out[k] = {"launches": v["launches"], "ms": round(v["ms"], 3), "us_per_launch": round(1000 * v["ms"] / max(1, v["launches"]), 2),
              "units": v["rows"]}
print(json.dumps(out, indent=1))
