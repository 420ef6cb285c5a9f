"""C5 sweep (BASELINE configs[4]): the C2-shaped model (2 x 1000 trees, depth 6) and one
recommendation over 6,554 unseen LLMs x 10 profiles x 16 levels; per-kernel-class event timings.
    python tools/prof_c5.py [--reps 3]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.environ.get("AB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_02425_b200 as lp
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
d = synth.make("C2")
ctx = lp.Context(0, torch.cuda.current_stream())
m = lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=1000, max_depth=6), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
lf, pf, cost, levels = synth.sweep_tables(n_llm=6554, seed=1, profiles=synth.PROFILES_C2)
lfd, pfd = torch.from_numpy(lf).cuda(), torch.from_numpy(pf).cuda()
lp.recommend(ctx, m, lfd, pfd, cost, levels, 100.0, 50.0, 200, as_array=True)
torch.cuda.synchronize()
ctx.reset_stats()
ctx.set_timing(1)
t0 = time.perf_counter()
for _ in range(a.reps):
    lp.recommend(ctx, m, lfd, pfd, cost, levels, 100.0, 50.0, 200, as_array=True)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / a.reps
st = ctx.stats()
out = {"wall_ms_per_call": wall * 1e3}
for k, v in st["classes"].items():
    out[k] = {"launches": v["launches"], "ms_per_call": v["ms"] / a.reps}
print(json.dumps(out))
