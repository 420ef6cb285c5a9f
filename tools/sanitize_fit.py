"""Small fit + predict + recommend + workload generator for compute-sanitizer runs (memcheck,
racecheck, synccheck, initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_fit.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_02425_b200 as lp  # noqa: E402
import synth  # noqa: E402

ctx = lp.Context(0, torch.cuda.current_stream())
if os.environ.get("SANITIZE_PLAIN"):   # plain launches instead of CUDA graphs (racecheck)
    ctx.set_timing(1)
d = synth.make("C1")
m = lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=3, max_depth=4), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof,
           100.0, 50.0)
p = m.predict(ctx, d.X)
lf = d.X[::32, :d.f_llm]
pf = np.stack([d.X[d.prof_id == g][0, d.f_llm:d.f_llm + d.f_prof] for g in range(d.n_prof)])
rec = lp.recommend(ctx, m, lf, pf, d.cost, d.user_levels, 100.0, 50.0, 200)
s1 = synth.make_s1(5000, seed=2)
m2 = lp.fit(ctx, s1.X, s1.y, lp.hparams(n_trees=2, max_depth=6, use_eq4_weights=0), s1.users_col, w=s1.w)
# a mid-size paper-shaped fit (76,800 rows > one 65,536-row chunk; many pieces per level): the level
# histogram's multi-segment pipeline, the partition's tile loop and the dual-ensemble update
c3s = synth.make_scaled(600)
m3 = lp.fit(ctx, c3s.X, c3s.y, lp.hparams(n_trees=2, max_depth=7), c3s.users_col, c3s.llm_id, c3s.prof_id,
            c3s.n_llm, c3s.n_prof, 100.0, 50.0)
g = lp.WorkloadGenerator(ctx, synth.make_traces(3000))
smp = g.sample(ctx, 100, seed=1)
torch.cuda.synchronize()
print("sanitize run ok", p.shape, len(rec), smp.shape)
