"""Offline statistic behind the level histogram's four-row fast path: on a C3 slice (1M rows), the
fraction of four-row groups of each level's built-child row list (identity order) in which none of
the non-users features changes code.

    python tools/level_group_stats.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, oracle
d = synth.make_scaled(7812)
m = oracle.fit(d.X, d.y, oracle.hparams(n_trees=3, max_depth=8), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, 100., 50., n_trees_limit=3)
ct, nc = oracle.cuts(d.X)
codes = oracle.codes(d.X, ct, nc)
feat, thr = m.feat[0, 2], m.thr[0, 2]
n = d.n
node = np.zeros(n, np.int64)
uc = d.users_col
others = [f for f in range(d.X.shape[1]) if f != uc]
for lev in range(1, 8):
    f = feat[node]; t = thr[node]
    split = f >= 0
    go = np.where(split, np.where(d.X[np.arange(n), np.maximum(f, 0)] < t, 2 * node + 1, 2 * node + 2), -1)
    node = np.where(split, go, -1)
    # built child per parent: smaller count
    tot_rows = 0; clean = 0; groups = 0
    ids, cnts = np.unique(node[node >= 0], return_counts=True)
    cnt = dict(zip(ids.tolist(), cnts.tolist()))
    for k in ids.tolist():
        if k % 2 == 1:
            sib = k + 1
            built = k if cnt.get(k, 0) <= cnt.get(sib, 0) else sib
            rows = np.nonzero(node == built)[0]
            tot_rows += len(rows)
            c = codes[rows][:, others]
            ch = np.any(c[1:] != c[:-1], axis=1)   # change at transition i -> i+1
            g = len(rows) // 4
            if g:
                # group j covers rows 4j..4j+3: transitions 4j..4j+2
                trans = np.concatenate([ch, [False]])[:g * 4].reshape(g, 4)[:, :3]
                clean += int((~trans.any(axis=1)).sum()); groups += g
    print("level", lev, "built rows", tot_rows, "groups", groups, "clean frac %.2f" % (clean / max(groups, 1)))
