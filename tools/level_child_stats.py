"""Per-level statistics of the built children (rows, flagged rows per 32-row batch of the change-row
level histogram, distinct 8-row packed-pair sectors per row) on a C3 slice, from the oracle's fit.

    python tools/level_child_stats.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, oracle
t0=time.time()
d = synth.make_scaled(7812)
m = oracle.fit(d.X, d.y, oracle.hparams(n_trees=3, max_depth=8), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, 100., 50., n_trees_limit=3)
ct, nc = oracle.cuts(d.X)
codes = oracle.codes(d.X, ct, nc)
print("fit", time.time()-t0, file=sys.stderr)
uc = d.users_col
others = [f for f in range(d.X.shape[1]) if f != uc]
n = d.n
for tg in (0,1):
  feat, thr = m.feat[tg, 2], m.thr[tg, 2]
  node = np.zeros(n, np.int64)
  for lev in range(1, 8):
    f = feat[node]; t = thr[node]
    split = f >= 0
    go = np.where(split, np.where(d.X[np.arange(n), np.maximum(f, 0)] < t, 2 * node + 1, 2 * node + 2), -1)
    node = np.where(split, go, -1)
    ids, cnts = np.unique(node[node >= 0], return_counts=True)
    cnt = dict(zip(ids.tolist(), cnts.tolist()))
    tot=0; flagged=0; csec=set(); gsec=0; pieces=0; batches=0
    for k in ids.tolist():
        if k % 2 == 1:
            sib = k + 1
            built = k if cnt.get(k, 0) <= cnt.get(sib, 0) else sib
            rows = np.nonzero(node == built)[0]
            if len(rows)==0: continue
            pieces+=1
            tot += len(rows)
            c = codes[rows][:, others]
            ch = np.any(c[1:] != c[:-1], axis=1)
            flagged += int(ch.sum())+1
            gsec += len(np.unique(rows // 8))
            batches += (len(rows)+31)//32
    print(f"tg{tg} level {lev}: pieces {pieces} built rows {tot} ({tot/n:.3f} of n)  flagged/row {flagged/max(tot,1):.3f}  flagged/batch {32*flagged/max(tot,1):.2f}  pair sectors/row {gsec/max(tot,1):.3f}")
