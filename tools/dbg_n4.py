import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, oracle, synth, paper_2410_02425_b200 as lp
d = synth.make("C1")
X = d.X.copy()
X[:, 1] = np.asarray(synth.u01(4, np.arange(len(X)), 77) * 1000.0, np.float32)
ctx = lp.Context(0, torch.cuda.current_stream())
for data, XX in (("wide", X), ("c1", d.X)):
    for k in [dict(n_trees=8, max_depth=4, max_bin=256, eta=0.5), dict(n_trees=8, max_depth=4, max_bin=1024, eta=0.3),
              dict(n_trees=8, max_depth=4, max_bin=1024, eta=0.5), dict(n_trees=1, max_depth=4, max_bin=1024, eta=0.5),
              dict(n_trees=2, max_depth=4, max_bin=1024, eta=0.5), dict(n_trees=8, max_depth=2, eta=0.5),
              dict(n_trees=8, max_depth=4, eta=0.5, monotone_users=0)]:
        of = oracle.cv(XX, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [oracle.hparams(**k)], 100., 50., 200, d.cost)
        gf = lp.cv(ctx, XX, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [lp.hparams(**k)], 100., 50., 200, d.cost)
        print(data, k, of == gf)
