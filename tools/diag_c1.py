import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2410_02425_b200 as lp, synth, oracle
d = synth.make("C1")
ctx = lp.Context(0, torch.cuda.current_stream())
kw = dict(n_trees=20, max_depth=4)
om, otp = oracle.fit(d.X, d.y, oracle.hparams(**kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, 100.0, 50.0, return_train_pred=True)
res = []
for rep in range(4):
    gm = lp.fit(ctx, torch.from_numpy(d.X).cuda(), torch.from_numpy(d.y).cuda(), lp.hparams(**kw), d.users_col,
                torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda(), d.n_llm, d.n_prof, 100.0, 50.0)
    e = gm.export()
    res.append(e)
    for tg in range(2):
        bad = [t for t in range(20) if not (np.array_equal(om.feat[tg, t], e['feat'][tg, t]) and np.array_equal(om.val[tg,t].view(np.uint32), e['val'][tg,t].view(np.uint32)))]
        print("rep", rep, "target", tg, "first bad trees", bad[:5])
    if rep:
        print(" same as rep0:", all(np.array_equal(res[0][k], e[k]) for k in ('feat','val')))
t = [t for t in range(20) if not np.array_equal(om.feat[0, t], res[0]['feat'][0, t]) or not np.array_equal(om.val[0,t].view(np.uint32), res[0]['val'][0,t].view(np.uint32))]
if t:
    t = t[0]
    print("oracle feat", om.feat[0, t]); print("gpu    feat", res[0]['feat'][0, t])
    print("oracle val", om.val[0, t]); print("gpu    val", res[0]['val'][0, t])
t = [t for t in range(20) if not np.array_equal(om.feat[1, t], res[0]['feat'][1, t]) or not np.array_equal(om.val[1,t].view(np.uint32), res[0]['val'][1,t].view(np.uint32))]
if t:
    t = t[0]
    print("T1 oracle feat", om.feat[1, t]); print("gpu    feat", res[0]['feat'][1, t])
    print("oracle val", om.val[1, t]); print("gpu    val", res[0]['val'][1, t])
