"""Subprocess helper for test_gpu_parity.test_kernel_variants: the kernel-variant switches
(LLMP_NOFUSE, LLMP_ROOT2, LLMP_SPLIT_CLUSTER, LLMP_NO_UROW, LLMP_HIST2, LLMP_PAIRED, LLMP_GRAPH_REPLAY,
LLMP_HIST_SWAR, LLMP_PRED_DC) are read once per process, so each variant is checked in
its own interpreter.  Fits paper-shaped (C1 with 12 features, C2) and random (S1, ragged) data through the
C-ABI in both execution modes (graph replay, instrumented plain launches) and compares with the oracle;
checks the histogram test hook (the variant's histogram kernel) against brute-force sums."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
import torch  # noqa: E402

import paper_2410_02425_b200 as lp  # noqa: E402

L1, L2 = 100.0, 50.0


def same(om, ge):
    ok = np.array_equal(om.base.view(np.uint32), ge["base"].view(np.uint32)) and np.array_equal(om.feat, ge["feat"])
    split = om.feat >= 0
    ok = ok and np.array_equal(om.bin[split], ge["bin"][split])
    ok = ok and np.array_equal(om.thr.view(np.uint32), ge["thr"].view(np.uint32))
    return ok and np.array_equal(om.val.view(np.uint32), ge["val"].view(np.uint32))


def main():
    ctx = lp.Context(0, torch.cuda.current_stream())
    rng = np.random.default_rng(3)
    codes = np.repeat(rng.integers(0, 256, (2000 // 7 + 1, 32)), 7, axis=0)[:2000].astype(np.uint8)
    codes[:, 5] = rng.integers(0, 16, 2000)
    qg = rng.integers(-(1 << 14), (1 << 14) + 1, 2000).astype(np.int32)
    qh = rng.integers(0, (1 << 14) + 1, 2000).astype(np.int32)
    Og, Oh = oracle.node_hist(codes, np.arange(2000), qg, qh)
    Gg, Gh = lp.debug_histogram(ctx, torch.from_numpy(codes).cuda(), torch.from_numpy(qg).cuda(),
                                torch.from_numpy(qh).cuda())
    if not (np.array_equal(Og, Gg) and np.array_equal(Oh, Gh)):
        print("MISMATCH histogram hook")
        return 1
    cases = [(synth.make("C1"), None, dict(n_trees=20, max_depth=4)),
             (synth.make("C2"), None, dict(n_trees=12, max_depth=7)),
             (synth.make_s1(70001, seed=5), "w", dict(n_trees=4, max_depth=8, use_eq4_weights=0)),
             (synth.make_s1(4097, seed=6), "w", dict(n_trees=3, max_depth=6, use_eq4_weights=0)),
             (synth.make_s1(30001, seed=7), "w", dict(n_trees=3, max_depth=10, use_eq4_weights=0,
                                                       min_child_weight=0.0))]
    for d, wk, kw in cases:
        w = d.w if wk else None
        om, otp = oracle.fit(d.X, d.y, oracle.hparams(**kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof,
                             L1, L2, w=w, return_train_pred=True)
        for every in (0, 1):
            ctx.set_timing(every)
            gm = lp.fit(ctx, d.X, d.y, lp.hparams(**kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2,
                        w=w)
            ctx.set_timing(0)
            if not same(om, gm.export()):
                print("MISMATCH model n=%d timing=%d" % (d.n, every))
                return 1
            if not np.array_equal(np.asarray(otp, np.float32).view(np.uint32),
                                  np.asarray(gm.train_pred(d.n), np.float32).view(np.uint32)):
                print("MISMATCH train_pred n=%d timing=%d" % (d.n, every))
                return 1
            if not np.array_equal(np.asarray(otp, np.float32).view(np.uint32),
                                  np.asarray(gm.predict(ctx, d.X), np.float32).view(np.uint32)):
                print("MISMATCH predict n=%d timing=%d" % (d.n, every))
                return 1
            gm.free()
    print("OK")
    return 0


if __name__ == "__main__":
    sys.exit(main())
