"""Wall time of llmpilot_cv_leave_one_llm_out on C2 (BASELINE configs[1]): plain LOO (grid of one,
2 x 1000 trees, depth 6) and a 4-point grid (nested LOO, 2 x 30 x 29 x 4 inner fits).
    python tools/time_cv.py [--trees 1000] [--grid 4]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_02425_b200 as lp
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--trees", type=int, default=1000)
ap.add_argument("--grid", type=int, default=4)
ap.add_argument("--grid-trees", type=int, default=200)
a = ap.parse_args()
d = synth.make("C2")
ctx = lp.Context(0, torch.cuda.current_stream())
out = {}
g1 = [lp.hparams(n_trees=a.trees, max_depth=6)]
lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, g1, 100.0, 50.0, 200, d.cost)
t0 = time.perf_counter()
folds, S, O, SO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, g1, 100.0, 50.0, 200, d.cost)
out["loo_s"] = time.perf_counter() - t0
out["loo"] = {"S": S, "O": O, "SO": SO, "folds": len(folds)}
if a.grid > 1:
    gk = [dict(n_trees=a.grid_trees, max_depth=6, eta=0.3), dict(n_trees=a.grid_trees, max_depth=4, eta=0.3),
          dict(n_trees=a.grid_trees, max_depth=6, eta=0.1), dict(n_trees=a.grid_trees, max_depth=6, eta=0.3, subsample=0.8,
                                                                  colsample_bytree=0.8)][:a.grid]
    g = [lp.hparams(**k) for k in gk]
    t0 = time.perf_counter()
    folds, S, O, SO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, g, 100.0, 50.0, 200, d.cost)
    out["grid_s"] = time.perf_counter() - t0
    out["grid"] = {"points": len(g), "trees": a.grid_trees, "S": S, "O": O, "SO": SO,
                   "hp_chosen": [f["hp_index"] for f in folds]}
print(json.dumps(out))
