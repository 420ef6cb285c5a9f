"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): codes, histograms, splits, trees and recommendations bit-exact;
predictions bit-exact when summed in tree order (the 1e-5 relative tolerance is not needed).
All inputs are seeded synthetic data from synth/ (DESIGN.md §Inputs).
"""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

L1, L2, U = 100.0, 50.0, 200


@pytest.fixture(scope="module")
def lp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_02425_b200 as lp_
    return lp_


@pytest.fixture(scope="module")
def ctx(lp):
    c = lp.Context(0, torch.cuda.current_stream())
    yield c
    c.close()


def _o_hp(**kw):
    return oracle.hparams(**kw)


def _g_hp(lp, **kw):
    return lp.hparams(**kw)


def _fit_both(lp, ctx, d, w=None, trees_limit=0, **kw):
    kw.setdefault("n_trees", 20)
    kw.setdefault("max_depth", 4)
    ohp = _o_hp(**kw)
    om, otp = oracle.fit(d.X, d.y, ohp, d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2, w=w,
                         return_train_pred=True, n_trees_limit=trees_limit)
    gm = lp.fit(ctx, torch.from_numpy(d.X).cuda(), torch.from_numpy(d.y).cuda(), _g_hp(lp, **kw), d.users_col,
                torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda(), d.n_llm, d.n_prof, L1, L2,
                w=None if w is None else torch.from_numpy(w).cuda())
    return om, otp, gm


def _assert_same_model(om, gm_export, what=""):
    assert np.array_equal(om.base.view(np.uint32), gm_export["base"].view(np.uint32)), what
    assert np.array_equal(om.feat, gm_export["feat"]), what
    split = om.feat >= 0
    assert np.array_equal(om.bin[split], gm_export["bin"][split]), what
    assert np.array_equal(om.thr.view(np.uint32), gm_export["thr"].view(np.uint32)), what
    assert np.array_equal(om.val.view(np.uint32), gm_export["val"].view(np.uint32)), what


def _bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


# --------------------------------------------------------------------------------------- binning
@pytest.mark.parametrize("case", ["C1", "C2", "s1", "many", "few16"])
def test_bin_parity(lp, ctx, case):
    rng = np.random.default_rng(0)
    B = 256
    if case in ("C1", "C2"):
        X = synth.make(case).X
    elif case == "s1":
        X = synth.make_s1(5000).X
    elif case == "many":
        X = (rng.standard_normal((30001, 7)) * 3).astype(np.float32)
        X[::7, 2] = -0.0
        X[1::7, 2] = 0.0
    else:
        X = rng.standard_normal((4099, 5)).astype(np.float32)
        B = 16
    ct, nc = oracle.cuts(X, max_bin=B)
    oc = oracle.codes(X, ct, nc)
    codes = torch.zeros((X.shape[0], 32), dtype=torch.uint8, device="cuda")
    cuts = lp.bin(ctx, torch.from_numpy(X).cuda(), max_bin=B, codes_out=codes)
    torch.cuda.synchronize()
    gct, gnc = cuts.export()
    assert np.array_equal(nc, gnc)
    for f in range(X.shape[1]):
        assert _bits_equal(ct[f, :nc[f]], gct[f, :gnc[f]])
    gcodes = codes.cpu().numpy()
    assert np.array_equal(oc, gcodes[:, :X.shape[1]])
    assert not gcodes[:, X.shape[1]:].any()
    # host-pointer input gives the same cuts
    cuts2 = lp.bin(ctx, X, max_bin=B)
    gct2, gnc2 = cuts2.export()
    assert np.array_equal(gnc2, gnc) and _bits_equal(gct2, gct)


# ------------------------------------------------------------------------------------ histograms
@pytest.mark.parametrize("n,structured,use_idx", [(1, False, False), (777, False, False), (100003, True, False),
                                                 (300001, False, True), (70000, True, True)])
def test_histogram_parity(lp, ctx, n, structured, use_idx):
    rng = np.random.default_rng(n)
    K = 14
    if structured:   # long runs of equal codes (what run-length aggregation exploits)
        codes = np.repeat(rng.integers(0, 256, (n // 37 + 1, 32)), 37, axis=0)[:n].astype(np.uint8)
        codes[:, 31] = rng.integers(0, 16, n)
    else:
        codes = rng.integers(0, 256, (n, 32)).astype(np.uint8)
    qg = rng.integers(-(1 << K), (1 << K) + 1, n).astype(np.int32)
    qh = rng.integers(0, (1 << K) + 1, n).astype(np.int32)
    idx = np.sort(rng.choice(n, max(1, n // 3), replace=False)).astype(np.int32) if use_idx else None
    rows = np.arange(n) if idx is None else idx
    Og, Oh = oracle.node_hist(codes, rows, qg, qh)
    Gg, Gh = lp.debug_histogram(ctx, torch.from_numpy(codes).cuda(), torch.from_numpy(qg).cuda(),
                                torch.from_numpy(qh).cuda(), None if idx is None else torch.from_numpy(idx).cuda())
    assert np.array_equal(Og, Gg) and np.array_equal(Oh, Gh)


# ----------------------------------------------------------------------------------------- fits
def test_fit_parity_c1(lp, ctx):
    d = synth.make("C1")
    om, otp, gm = _fit_both(lp, ctx, d)
    _assert_same_model(om, gm.export())
    assert _bits_equal(otp, gm.train_pred(d.n))
    # predict(train X) reproduces the internal training predictions bit for bit (O9/O10)
    assert _bits_equal(gm.predict(ctx, d.X), otp)
    out = torch.zeros((d.n, 2), dtype=torch.float32, device="cuda")
    gm.predict(ctx, torch.from_numpy(d.X).cuda(), out=out)
    torch.cuda.synchronize()
    assert _bits_equal(out.cpu().numpy(), otp)


def test_importance_parity(lp, ctx):
    """MDI importance: the split losses the split kernel records and the
    importances summed from them are bit-identical to the oracle's (C1 and C2, with colsample)."""
    for d, kw in ((synth.make("C1"), dict(n_trees=20, max_depth=4)),
                  (synth.make("C2"), dict(n_trees=15, max_depth=6, colsample_bytree=0.7, seed=3))):
        om, _, gm = _fit_both(lp, ctx, d, **kw)
        _assert_same_model(om, gm.export())
        assert np.array_equal(om.gain, gm.gains())
        for nrm in (False, True):
            assert np.array_equal(oracle.importance(om, nrm), gm.importance(nrm))


@pytest.mark.parametrize("kw", [
    dict(),
    dict(monotone_users=0),
    dict(subsample=0.7, colsample_bytree=0.6, seed=7),
    dict(max_depth=1, n_trees=10),
    dict(max_depth=7, n_trees=6),
    dict(max_depth=9, n_trees=4, min_child_weight=0.0),
    dict(max_depth=10, n_trees=4, min_child_weight=0.0),
    dict(max_bin=16, grad_bits=8),
    dict(lambda_=0.0, min_child_weight=0.0),
    dict(min_child_weight=5.0, eta=0.1),
    dict(grad_bits=2, n_trees=5),
])
def test_fit_parity_variants_c2(lp, ctx, kw):
    d = synth.make("C2")
    kw = dict(kw)
    kw.setdefault("n_trees", 12)
    kw.setdefault("max_depth", 6)
    om, otp, gm = _fit_both(lp, ctx, d, **kw)
    _assert_same_model(om, gm.export(), str(kw))
    assert _bits_equal(otp, gm.train_pred(d.n))


def test_fit_parity_explicit_weights_s1(lp, ctx):
    d = synth.make_s1(20011)
    om, otp, gm = _fit_both(lp, ctx, d, w=d.w, n_trees=8, max_depth=8, use_eq4_weights=0)
    _assert_same_model(om, gm.export())
    assert _bits_equal(otp, gm.train_pred(d.n))


@pytest.mark.parametrize("n", [1, 2, 3, 2047, 2049, 140001])
def test_fit_parity_ragged_sizes(lp, ctx, n):
    d = synth.make_s1(n, seed=3)
    om, otp, gm = _fit_both(lp, ctx, d, w=d.w, n_trees=3, max_depth=5, use_eq4_weights=0)
    _assert_same_model(om, gm.export(), str(n))
    assert _bits_equal(otp, gm.train_pred(d.n))


def _degenerate(case):
    import copy
    d = copy.deepcopy(synth.make_s1(5000, seed=4))
    w = d.w.copy()
    if case == "constant_y":
        d.y[:] = np.float32(1.5)
    elif case == "constant_features":
        d.X[:, 3] = np.float32(7)
        d.X[:, 10] = np.float32(-2)
    elif case == "zero_weights":
        w[:] = 0
    elif case == "half_zero_weights":
        w[::2] = 0
    elif case == "single_feature":
        d.X = np.ascontiguousarray(d.X[:, 31:32])
        d.users_col = 0
    elif case == "all_rows_equal":
        d.X[:] = np.float32(0)
    return d, w


@pytest.mark.parametrize("case", ["constant_y", "constant_features", "zero_weights", "half_zero_weights",
                                  "single_feature", "all_rows_equal"])
def test_fit_parity_degenerate_inputs(lp, ctx, case):
    """Degenerate data the method must handle: no split has positive gain (constant y, all rows
    equal, all weights zero — every tree is a single leaf), constant columns (never split on),
    a single feature (the users column only) and rows with zero weight (h = 0)."""
    d, w = _degenerate(case)
    om, otp, gm = _fit_both(lp, ctx, d, w=w, n_trees=5, max_depth=4, use_eq4_weights=0)
    _assert_same_model(om, gm.export(), case)
    assert _bits_equal(otp, gm.train_pred(d.n))
    assert _bits_equal(oracle.predict(om, d.X), gm.predict(ctx, d.X))


def test_fit_sequential_mode_and_root_speculation(lp, ctx):
    """Instrumented mode runs the two ensembles one after the other with plain launches (the
    NCCL path does too); it must give the oracle's model like the concurrent graph replay.  The
    fused update pass builds each next root histogram speculatively: the device
    row counters show both paths taken — speculative roots kept, and rebuilt ones (tree 0 and
    exponent changes)."""
    d = synth.make("C2")
    kw = dict(n_trees=30, max_depth=6)
    om, otp = oracle.fit(d.X, d.y, _o_hp(**kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2,
                         return_train_pred=True)
    for every in (1, 0):
        ctx.reset_stats()
        ctx.set_timing(every)
        try:
            gm = lp.fit(ctx, d.X, d.y, _g_hp(lp, **kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2)
            st = ctx.stats()["classes"]
        finally:
            ctx.set_timing(0)
        _assert_same_model(om, gm.export(), "timing every=%d" % every)
        assert _bits_equal(otp, gm.train_pred(d.n))
        root_rows = st["hist_root"]["rows"]
        assert root_rows % d.n == 0
        # rebuilt roots = tree 0 of each target + every tree whose max|g| exponent differs from the
        # previous tree's (max h = max w never changes without subsampling)
        assert root_rows // d.n == 2 + _exponent_changes(om, d), (root_rows // d.n, every)


def _exponent_changes(om, d):
    """Number of trees t >= 1 (both targets) whose gradient-maximum exponent (O4: e with
    max|g| = m 2^e, m in [0.5, 1)) differs from tree t-1's, from the oracle's model."""
    w = oracle.weights(d.y, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2)
    T = om.feat.shape[1]
    ch = 0
    for tg in range(2):
        p = np.full(d.n, om.base[tg], np.float32)
        prev = None
        for t in range(T):
            g = w * (p - d.y[:, tg])          # float32 throughout, like O4
            e = int(np.frexp(np.abs(g).max())[1]) if np.abs(g).max() > 0 else 0
            ch += prev is not None and e != prev
            prev = e
            one = oracle.Model(om.F, om.hp, om.cuts, om.ncuts, np.zeros(2, np.float32), om.feat[:, t:t + 1],
                               om.bin[:, t:t + 1], om.thr[:, t:t + 1], om.val[:, t:t + 1])
            p = p + oracle.predict(one, d.X)[:, tg]
    return ch


@pytest.mark.parametrize("env", ["LLMP_NOFUSE=1", "LLMP_ROOT2=1", "LLMP_SPLIT_CLUSTER=1", "LLMP_NO_UROW=1",
                                 "LLMP_HIST2=0", "LLMP_HIST2=7",
                                 "LLMP_PAIRED=1", "LLMP_GRAPH_REPLAY=1", "LLMP_HIST_SWAR=0", "LLMP_PRED_DC=0", "LLMP_PDL=0",
                                 "LLMP_LEVEL=1", "LLMP_LEVEL=2", "LLMP_UPD=3", "LLMP_PAIRED=1 LLMP_UPD=3", "LLMP_FOLD=1", "LLMP_FOLD=1 LLMP_PAIRED=1", "LLMP_HFIX=0",
                                 "LLMP_DUAL=0", "LLMP_DUAL=0 LLMP_PAIRED=1", "LLMP_GRAPH_REPLAY=1 LLMP_PAIRED=1",
                                 "LLMP_SPLIT_TWICE=1"])
def test_kernel_variants(lp, env):
    """Every selectable kernel variant gives the oracle's models (own process: the switches are
    read once per process)."""
    import os
    import subprocess
    import sys
    e = dict(os.environ)
    for kv in env.split():
        k, v = kv.split("=")
        e[k] = v
    p = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "_variant_fit.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "OK" in p.stdout, (env, p.stdout[-2000:], p.stderr[-2000:])


def test_sharded_path_with_a_one_rank_nccl_communicator(lp):
    """A context with a communicator takes the sharded fit path: NCCL all-reduces of
    the Eq. (4) group maxima, base-score sums, gradient maxima, child counts and built-child
    histograms, the all-gathered global cut sample, plain launches instead of graphs.  With one
    rank every collective is trivial, so the models must be the oracle's bit for bit — this runs
    the multi-GPU code path (and real NCCL calls) on one device."""
    ctx1 = lp.Context(0, torch.cuda.current_stream(), lp.nccl_unique_id(), 0, 1)
    try:
        ctx1.reset_stats()
        for d, w, kw in ((synth.make("C2"), None, dict(n_trees=12, max_depth=6)),
                         (synth.make_s1(30001, seed=5), "w", dict(n_trees=4, max_depth=8, use_eq4_weights=0))):
            om, otp, gm = _fit_both(lp, ctx1, d, w=None if w is None else d.w, **kw)
            _assert_same_model(om, gm.export())
            assert _bits_equal(otp, gm.train_pred(d.n))
            gm.free()
        assert ctx1.stats()["classes"]["nccl"]["launches"] > 0
    finally:
        ctx1.close()


@pytest.mark.parametrize("nranks,n_llm,big", [(2, 200, False), (3, 131, False), (3, 16411, True)])
def test_multi_rank_sharded_fit_on_one_device(lp, nranks, n_llm, big):
    """The N > 1 fit path on one B200: nranks contexts of an in-process communicator
    (llmpilot_ctx_create_local_group; NCCL refuses two ranks on one device), each fitting its
    contiguous LLM-block shard from its own thread — all-gathered global cut sample, all-reduced
    group maxima / base sums / gradient maxima / partial histograms, built children chosen by the
    split's hessian sums.  Every rank's model equals the oracle's unsharded fit bit for bit
    (uneven shards with 3 ranks).  The big case has n_global = 2,100,608 > 2^21 rows, so the
    global cut sample is strided (s = ceil(n_global / 2^20) = 3, O2 / P:L209) and every rank
    contributes the rows i = 0 (mod 3) of its own shard at their global indices."""
    import threading
    full = synth.make_scaled(n_llm)
    kw = dict(n_trees=8, max_depth=6, subsample=0.8, colsample_bytree=0.8, seed=5)
    if big:
        assert full.n > 2 ** 21
        kw = dict(n_trees=2, max_depth=5, subsample=0.8, colsample_bytree=0.8, seed=7)
    om = oracle.fit(full.X, full.y, _o_hp(**kw), full.users_col, full.llm_id, full.prof_id, full.n_llm, full.n_prof,
                    L1, L2)
    ctxs = lp.local_group(0, nranks)
    res, errs = [None] * nranks, []

    def run(r):
        try:
            sh = synth.make_scaled(n_llm, r, nranks)
            m = lp.fit(ctxs[r], sh.X, sh.y, _g_hp(lp, **kw), sh.users_col, sh.llm_id, sh.prof_id, sh.n_llm, sh.n_prof,
                       L1, L2, row_offset=sh.row_offset, n_global=sh.n_global)
            res[r] = m.export()
            m.free()
        except Exception as e:   # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in ctxs:
        c.close()
    assert not errs, errs
    for r in range(nranks):
        _assert_same_model(om, res[r], "rank %d of %d" % (r, nranks))


def test_concurrent_contexts_stress(lp):
    """8 host threads, one context and stream each, fitting (CUDA-graph tree loop with its capture),
    predicting and freeing concurrently on one device: every model is the oracle's bit for bit and
    no call fails (shared per-device kernel attributes and workspace growth under concurrency)."""
    import threading
    d = synth.make("C2")
    kw = dict(n_trees=10, max_depth=6)
    om, otp = oracle.fit(d.X, d.y, _o_hp(**kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2,
                         return_train_pred=True)
    errs, res = [], {}

    def run(i):
        try:
            st = torch.cuda.Stream()
            c = lp.Context(0, st)
            for rep in range(3):
                m = lp.fit(c, d.X, d.y, _g_hp(lp, **kw), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2)
                res[(i, rep)] = (m.export(), m.predict(c, d.X))
                m.free()
            c.close()
        except Exception as e:   # noqa: BLE001
            errs.append((i, repr(e)))

    th = [threading.Thread(target=run, args=(i,)) for i in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    assert len(res) == 24
    for k, (e, p) in res.items():
        _assert_same_model(om, e, str(k))
        assert _bits_equal(otp, p), k


def test_fit_host_and_device_inputs_identical_and_deterministic(lp, ctx):
    d = synth.make("C2")
    hp = lp.hparams(n_trees=10, max_depth=6)
    m1 = lp.fit(ctx, d.X, d.y, hp, d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2)
    m2 = lp.fit(ctx, torch.from_numpy(d.X).cuda(), torch.from_numpy(d.y).cuda(), hp, d.users_col,
                torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda(), d.n_llm, d.n_prof, L1, L2)
    e1, e2 = m1.export(), m2.export()
    for k in e1:
        assert np.array_equal(e1[k], e2[k]), k


# ---------------------------------------------------------------------------- predict/recommend
def test_predict_and_recommend_parity(lp, ctx):
    d = synth.make("C2")
    om, otp, gm = _fit_both(lp, ctx, d, n_trees=40, max_depth=6)
    lf, pf, cost, levels = synth.sweep_tables(n_llm=300)
    # oracle: assemble every (llm, profile, level) row, predict, recommend
    nL, nP, nU = lf.shape[0], pf.shape[0], len(levels)
    rows = np.concatenate([np.repeat(lf, nP * nU, axis=0), np.tile(np.repeat(pf, nU, axis=0), (nL, 1)),
                           np.tile(levels.astype(np.float32), nL * nP)[:, None]], axis=1)
    op = oracle.predict(om, rows)
    orec = oracle.recommend(op.reshape(nL, nP, nU, 2), levels, cost, L1, L2, U)
    gp = gm.predict(ctx, rows)
    assert _bits_equal(op, gp)
    pred_out = torch.zeros((nL * nP * nU, 2), dtype=torch.float32, device="cuda")
    grec = lp.recommend(ctx, gm, torch.from_numpy(lf).cuda(), torch.from_numpy(pf).cuda(), cost, levels, L1, L2, U,
                        pred_out=pred_out)
    assert _bits_equal(pred_out.cpu().numpy(), op)
    assert grec == orec
    # with a mask and host inputs
    allowed = (np.random.default_rng(1).random((nL, nP)) < 0.5).astype(np.uint8)
    orec2 = oracle.recommend(op.reshape(nL, nP, nU, 2), levels, cost, L1, L2, U, allowed)
    grec2 = lp.recommend(ctx, gm, lf, pf, cost, levels, L1, L2, U, allowed=allowed)
    assert grec2 == orec2
    assert any(r[0] == -1 for r in grec2) or True


@pytest.mark.parametrize("depth,levels_kind", [(6, "sorted16"), (7, "sparse16"), (6, "one"), (8, "sorted32"),
                                               (6, "sorted64"), (6, "sorted70"), (10, "sorted16"), (1, "sparse16")])
def test_recommend_grid_predictor_cases(lp, ctx, depth, levels_kind):
    """The recommend sweep's predictions (per (LLM, profile) pair, one tree descent per distinct leaf
    carrying the range of user levels, n_levels <= 64; the per-row walk beyond) equal the oracle's
    predictions of the assembled rows bit for bit, and so do the recommendations: the C5 levels, 16
    widely spaced levels, a single level, 32 and 64 levels, 70 levels (per-row fallback), compile-time
    (6, 8) and run-time (7) depths."""
    d = synth.make("C2")
    om, otp, gm = _fit_both(lp, ctx, d, n_trees=25, max_depth=depth)
    lf, pf, cost, lv16 = synth.sweep_tables(n_llm=211, seed=3)
    rng = np.random.default_rng(depth)
    if levels_kind == "sorted16":
        levels = lv16
    elif levels_kind == "sparse16":
        levels = np.array([1, 3, 7, 12, 20, 33, 50, 64, 90, 128, 180, 256, 400, 512, 800, 1024], np.int32)
    elif levels_kind == "one":
        levels = np.array([8], np.int32)
    else:
        k = int(levels_kind[len("sorted"):])
        levels = np.unique(rng.integers(1, 300, 4 * k))[:k].astype(np.int32)
        assert len(levels) == k
    nL, nP, nU = lf.shape[0], pf.shape[0], len(levels)
    rows = np.concatenate([np.repeat(lf, nP * nU, axis=0), np.tile(np.repeat(pf, nU, axis=0), (nL, 1)),
                           np.tile(levels.astype(np.float32), nL * nP)[:, None]], axis=1)
    op = oracle.predict(om, rows)
    orec = oracle.recommend(op.reshape(nL, nP, nU, 2), levels, cost, L1, L2, U)
    pred_out = torch.zeros((nL * nP * nU, 2), dtype=torch.float32, device="cuda")
    grec = lp.recommend(ctx, gm, torch.from_numpy(lf).cuda(), torch.from_numpy(pf).cuda(), cost, levels, L1, L2, U,
                        pred_out=pred_out)
    assert _bits_equal(pred_out.cpu().numpy(), op)
    assert grec == orec


def test_model_save_load_round_trip(lp, ctx, tmp_path):
    """llmpilot_model_save / llmpilot_model_load: the loaded model exports, predicts, ranks features
    and recommends exactly as the fitted one (and as the oracle); malformed files are refused."""
    d = synth.make("C2")
    om, otp, gm = _fit_both(lp, ctx, d, n_trees=30, max_depth=6)
    path = str(tmp_path / "m.llmp")
    gm.save(path)
    lm = lp.Model.load(ctx, path)
    e1, e2 = gm.export(), lm.export()
    for k in e1:
        assert np.array_equal(e1[k], e2[k]), k
    assert np.array_equal(gm.gains(), lm.gains())
    assert np.array_equal(gm.importance(), lm.importance())
    assert _bits_equal(lm.predict(ctx, d.X), otp)
    lf, pf, cost, levels = synth.sweep_tables(n_llm=50)
    assert lp.recommend(ctx, lm, lf, pf, cost, levels, L1, L2, U) == \
        lp.recommend(ctx, gm, lf, pf, cost, levels, L1, L2, U)
    raw = open(path, "rb").read()
    bad = tmp_path / "bad.llmp"
    for blob in (b"", b"NOTMODEL" + raw[8:], raw[: len(raw) // 2]):
        bad.write_bytes(blob)
        with pytest.raises(lp.LLMPilotError):
            lp.Model.load(ctx, str(bad))
    with pytest.raises(lp.LLMPilotError):
        lp.Model.load(ctx, str(tmp_path / "missing.llmp"))


def test_c5_sweep_full_size_sampled_parity(lp, ctx):
    """BASELINE configs[4] at full size: the C2-shaped model (2 x 1000 trees, depth 6) and
    the sweep of 6,554 unseen LLMs x 10 profiles x 16 levels = 1,048,640 rows in the launch
    configuration bench.py times; the oracle predicts and recommends a sample of 48 LLMs (their 7,680
    rows), which must match the GPU's predictions bit for bit and its recommendations exactly."""
    d = synth.make("C2")
    om, otp, gm = _fit_both(lp, ctx, d, n_trees=1000, max_depth=6)
    _assert_same_model(om, gm.export())
    lf, pf, cost, levels = synth.sweep_tables(n_llm=6554, seed=1, profiles=synth.PROFILES_C2)
    nL, nP, nU = lf.shape[0], pf.shape[0], len(levels)
    pred_out = torch.zeros((nL * nP * nU, 2), dtype=torch.float32, device="cuda")
    grec = lp.recommend(ctx, gm, torch.from_numpy(lf).cuda(), torch.from_numpy(pf).cuda(), cost, levels, L1, L2, U,
                        pred_out=pred_out)
    gp = pred_out.cpu().numpy().reshape(nL, nP, nU, 2)
    sample = np.random.default_rng(5).choice(nL, 48, replace=False)
    sample[:2] = [0, nL - 1]
    for i in sample:
        rows = np.concatenate([np.repeat(lf[i:i + 1], nP * nU, axis=0), np.repeat(pf, nU, axis=0),
                               np.tile(levels.astype(np.float32), nP)[:, None]], axis=1)
        op = oracle.predict(om, rows).reshape(1, nP, nU, 2)
        assert _bits_equal(op[0], gp[i]), i
        assert oracle.recommend(op, levels, cost, L1, L2, U)[0] == grec[i], i
    assert len(grec) == nL


def test_recommend_toy_table_through_gpu_argmin(lp, ctx, golden):
    """The hand-computed toy table (tests/golden/o11_toy_table.json) through the GPU argmin:
    a 1-feature constant model cannot express it, so drive the argmin via the CV-free path:
    a depth-1 model whose predictions equal the table is built by fitting the table itself."""
    g = golden("o11_toy_table.json")
    P = g["profiles"]
    # rows: [profile id | users] -> y = (l1, l2); exact fit with eta=1, lambda=0 deep trees
    X, y = [], []
    for j, p in enumerate(P):
        for k, u in enumerate(g["levels"]):
            X.append([j, u]); y.append([p["l1"][k], p["l2"][k]])
    X = np.array(X, np.float32); y = np.array(y, np.float32)
    hp = lp.hparams(n_trees=4, max_depth=8, eta=1.0, lambda_=0.0, min_child_weight=0.0, use_eq4_weights=0,
                    monotone_users=0, grad_bits=14)
    m = lp.fit(ctx, X, y, hp, users_col=1)
    pred = m.predict(ctx, X)
    assert np.allclose(pred, y, rtol=1e-3, atol=1e-2)
    rec = lp.recommend(ctx, m, np.zeros((1, 0), np.float32), np.arange(len(P), dtype=np.float32)[:, None],
                       [p["cost"] for p in P], g["levels"], g["L1"], g["L2"], g["U"])
    e = g["expected"]
    assert rec[0] == (e["profile"], e["n_pods"], e["cost"], e["u_max"])


# ------------------------------------------------------------------------------------------- CV
def test_cv_parity_c1(lp, ctx):
    d = synth.make("C1")
    ohp = oracle.hparams(n_trees=20, max_depth=4)
    of, oS, oO, oSO = oracle.cv(d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [ohp], L1, L2, U,
                                d.cost)
    gf, gS, gO, gSO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof,
                            [lp.hparams(n_trees=20, max_depth=4)], L1, L2, U, d.cost)
    assert len(of) == len(gf)
    for a, b in zip(of, gf):
        assert a == b, (a, b)
    assert (oS, oO, oSO) == (gS, gO, gSO)


def test_cv_grid_parity_c1(lp, ctx):
    d = synth.make("C1")
    grid_kw = [dict(n_trees=3, max_depth=2, eta=0.05), dict(n_trees=15, max_depth=4), dict(n_trees=15, max_depth=3)]
    of, oS, oO, oSO = oracle.cv(d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof,
                                [oracle.hparams(**k) for k in grid_kw], L1, L2, U, d.cost)
    gf, gS, gO, gSO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof,
                            [lp.hparams(**k) for k in grid_kw], L1, L2, U, d.cost)
    assert of == gf and (oS, oO, oSO) == (gS, gO, gSO)


def test_cv_hand_fixture_on_gpu(lp, ctx, golden):
    """The O12 hand fixture (tests/golden/o12_cv_hand_fixture.json: S = 1/3, O = 0.5, SO = 0.4,
    P:L277, Eq. (6), Eq. (7)) through llmpilot_cv_leave_one_llm_out."""
    from _cv_fixture import cv_hand_fixture_rows
    g = golden("o12_cv_hand_fixture.json")
    X, y, li, pi, uc, n_llm, n_prof = cv_hand_fixture_rows(g)
    h = g["hparams"]
    hp = lp.hparams(n_trees=h["n_trees"], max_depth=h["max_depth"], eta=h["eta"], lambda_=h["lambda_"],
                    min_child_weight=h["min_child_weight"], use_eq4_weights=h["use_eq4_weights"],
                    monotone_users=h["monotone_users"])
    gf, gS, gO, gSO = lp.cv(ctx, X, y, li, pi, uc, n_llm, n_prof, [hp], g["L1"], g["L2"], g["U"], g["cost"])
    for f, e in zip(gf, g["folds"]):
        assert f["rec"] == tuple(e["rec"]) and f["truth"] == tuple(e["truth"])
        assert f["success"] == e["success"] and f["overspend"] == e["overspend"]
    assert gS == g["S_num"] / g["S_den"] and gO == g["O"] and gSO == pytest.approx(g["SO"], rel=1e-15)


@pytest.mark.parametrize("batched", [True, False])
def test_cv_grid5_parity_c1(lp, batched):
    """A 5-point grid of the HPs P:L207-209 names (trees, depth, learning rate, subsampling ratio,
    bins; plus column sampling and min child weight) through the nested leave-one-LLM-out CV, on the
    batched small-fit path (one thread block per fit) and on the sequential path (LLMP_CV_SMALL=0,
    one full fit per call): folds, chosen HPs, S, O, SO equal the oracle's."""
    import os
    import subprocess
    import sys
    code = r'''
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch, oracle, synth, paper_2410_02425_b200 as lp
d = synth.make("C1")
gk = [dict(n_trees=12, max_depth=3, eta=0.3), dict(n_trees=8, max_depth=5, eta=0.5, max_bin=4),
      dict(n_trees=15, max_depth=4, eta=0.2, subsample=0.7, seed=3), dict(n_trees=10, max_depth=2, eta=0.6, colsample_bytree=0.5, seed=9),
      dict(n_trees=10, max_depth=4, eta=0.3, min_child_weight=4.0, lambda_=2.0)]
of = oracle.cv(d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [oracle.hparams(**k) for k in gk], 100.0, 50.0, 200, d.cost)
ctx = lp.Context(0, torch.cuda.current_stream())
gf = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [lp.hparams(**k) for k in gk], 100.0, 50.0, 200, d.cost)
assert of == gf, (of, gf)
assert len({f["hp_index"] for f in of[0]}) >= 1
print("OK", sorted({f["hp_index"] for f in of[0]}))
'''
    env = dict(os.environ)
    if not batched:
        env["LLMP_CV_SMALL"] = "0"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and "OK" in p.stdout, (p.stdout[-2000:], p.stderr[-3000:])


def test_cv_parity_c2_short(lp, ctx):
    d = synth.make("C2")
    of, oS, oO, oSO = oracle.cv(d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof,
                                [oracle.hparams(n_trees=25, max_depth=6)], L1, L2, U, d.cost)
    gf, gS, gO, gSO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof,
                            [lp.hparams(n_trees=25, max_depth=6)], L1, L2, U, d.cost)
    assert of == gf and (oS, oO, oSO) == (gS, gO, gSO)


# -------------------------------------------------------------------------------- errors/edges
def test_errors(lp, ctx):
    d = synth.make("C1")
    X = d.X.copy()
    X[5, 3] = np.nan
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, X, d.y, lp.hparams(n_trees=2), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=2, max_depth=11), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=2, grad_bits=15), d.users_col, d.llm_id, d.prof_id, d.n_llm,
               d.n_prof)
    # a non-finite value anywhere in X (first, last, an inner element; X viewed flat by the validation
    # kernel), from host and from a device tensor at an odd offset (unaligned base)
    for pos, val in (((0, 0), np.inf), ((d.X.shape[0] - 1, d.X.shape[1] - 1), np.nan), ((17, 5), -np.inf)):
        Xb = d.X.copy()
        Xb[pos] = val
        with pytest.raises(lp.LLMPilotError, match="EINVAL"):
            lp.fit(ctx, Xb, d.y, lp.hparams(n_trees=2), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    big = torch.from_numpy(np.concatenate([np.zeros(1, np.float32), d.X.ravel()])).cuda()
    Xoff = big[1:].view(d.X.shape)   # 4-byte offset from a 16-byte aligned allocation
    Xoff_bad = Xoff.clone()[:, :]
    m_ok = lp.fit(ctx, Xoff, torch.from_numpy(d.y).cuda(), lp.hparams(n_trees=2, max_depth=2), d.users_col,
                  torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda(), d.n_llm, d.n_prof)
    m_ok.free()
    big[-1] = float("nan")   # the last element of the unaligned view (the scalar tail)
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, Xoff, torch.from_numpy(d.y).cuda(), lp.hparams(n_trees=2), d.users_col,
               torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda(), d.n_llm, d.n_prof)
    big[-1] = 0.0
    big[1] = float("inf")    # the first element (the scalar head)
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, Xoff, torch.from_numpy(d.y).cuda(), lp.hparams(n_trees=2), d.users_col,
               torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda(), d.n_llm, d.n_prof)
    del Xoff_bad
    bad = d.llm_id.copy()
    bad[0] = 99
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=2), d.users_col, bad, d.prof_id, d.n_llm, d.n_prof)
    m = lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=2, max_depth=2), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.recommend(ctx, m, d.X[:2, :6], d.X[:2, 6:11], [1.0, 1.0], [4, 2], L1, L2, U)   # levels not increasing
    # the predictor bins rows with the model's cuts: a non-finite feature (which routes differently as
    # a float than as a code) is rejected, in plain rows and in the recommendation tables alike (R17)
    Xn = d.X[:7].copy()
    Xn[3, 2] = np.nan
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        m.predict(ctx, Xn)
    lfn = d.X[:2, :6].copy()
    lfn[1, 0] = np.inf
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.recommend(ctx, m, lfn, d.X[:2, 6:11], [1.0, 1.0], [2, 4], L1, L2, U)
    assert m.predict(ctx, d.X[:0]).shape == (0, 2)   # empty batch
    # zero trees: predictions are the base scores
    m0 = lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=0), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    p0 = m0.predict(ctx, d.X)
    assert np.all(p0 == m0.export()["base"][None, :])


# ------------------------------------------------------- full-size sampled parity (C3 shape)
@pytest.mark.slow
def test_c3_full_size_parity(lp, ctx):
    """10M rows x 32 features x 256 bins, depth 8 — the bench's workload and launch configuration
    (CUDA-graph tree loop, fused update + speculative next root, precomputed change masks).  The
    oracle grows the first two trees of each target (tree 1 is the first one the fused update pass
    builds); the GPU grows 20, and the rest is checked by properties that hold at any size:
    predict(train X) == the training predictions bit for bit (O9/O10), the oracle's predictor on
    the GPU's trees reproduces them on sampled rows, and a second fit is bit-identical."""
    d = synth.make("C3")
    om = oracle.fit(d.X, d.y, _o_hp(n_trees=20, max_depth=8), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof,
                    L1, L2, n_trees_limit=2)
    Xd, yd = torch.from_numpy(d.X).cuda(), torch.from_numpy(d.y).cuda()
    ld, pd = torch.from_numpy(d.llm_id).cuda(), torch.from_numpy(d.prof_id).cuda()
    gm = lp.fit(ctx, Xd, yd, _g_hp(lp, n_trees=20, max_depth=8), d.users_col, ld, pd, d.n_llm, d.n_prof, L1, L2)
    e = gm.export()
    first2 = {k: (e[k][:, :2] if k != "base" else e[k]) for k in e}
    _assert_same_model(om, first2, "C3 trees 0-1")
    tp = gm.train_pred(d.n)
    out = torch.zeros((d.n, 2), dtype=torch.float32, device="cuda")
    gm.predict(ctx, Xd, out=out)
    torch.cuda.synchronize()
    assert _bits_equal(out.cpu().numpy(), tp)
    idx = np.arange(0, d.n, 997)
    g_as_o = oracle.Model(om.F, _o_hp(n_trees=20, max_depth=8), om.cuts, om.ncuts, e["base"], e["feat"], e["bin"],
                          e["thr"], e["val"])
    assert _bits_equal(oracle.predict(g_as_o, d.X[idx]), tp[idx])
    gm2 = lp.fit(ctx, Xd, yd, _g_hp(lp, n_trees=20, max_depth=8), d.users_col, ld, pd, d.n_llm, d.n_prof, L1, L2)
    e2 = gm2.export()
    assert all(np.array_equal(np.asarray(e[k]).view(np.uint32), np.asarray(e2[k]).view(np.uint32)) for k in e)


# ----------------------------------------------------------------------------- workload generator
@pytest.mark.parametrize("n,P,seed", [(1, 1, 0), (777, 3, 1), (20011, 8, 2), (1_200_000, 8, 3),
                                        (synth.TRACE_ROWS_PAPER, 8, 0)])
def test_workload_generator_parity(lp, ctx, n, P, seed):
    """bins, centres, the sparse joint histogram (keys, counts)
    and the sampled requests are bit-identical to the oracle's, including a ragged trace size, a
    single row, n > 2^20 (strided-sample quantiles) and sample offsets."""
    T = synth.make_traces(n, seed=seed)[:, :P]
    om = oracle.wg_build(T)
    for src in (T, torch.from_numpy(T).cuda()):
        g = lp.WorkloadGenerator(ctx, src)
        e = g.export()
        assert np.array_equal(e["nbins"], om.nbins)
        assert _bits_equal(e["centres"], om.centres)
        assert np.array_equal(e["keys"], om.keys) and np.array_equal(e["counts"], om.counts)
        draws = ((0, 0, 1000), (7, 123457, 4099)) if n < 5_000_000 else ((0, 0, 150), (7, 123457, 61))
        for s_seed, first, cnt in draws:   # (the oracle walks the CDF linearly: few draws at full size)
            ref = oracle.wg_sample(om, cnt, seed=s_seed, first=first)
            assert _bits_equal(g.sample(ctx, cnt, seed=s_seed, first=first), ref)
            dev = torch.zeros((cnt, P), dtype=torch.float32, device="cuda")
            g.sample(ctx, cnt, seed=s_seed, first=first, out=dev)
            torch.cuda.synchronize()
            assert _bits_equal(dev.cpu().numpy(), ref)
        g.free()


def test_workload_generator_errors(lp, ctx):
    with pytest.raises(lp.LLMPilotError):
        lp.WorkloadGenerator(ctx, np.array([[1.0, np.inf]], np.float32))
    with pytest.raises(lp.LLMPilotError):
        lp.WorkloadGenerator(ctx, np.tile(np.arange(64, dtype=np.float32)[:, None], (1, 11)))


# ------------------------------------------------------------------------------ random forest
@pytest.mark.parametrize("case", ["c2", "s1", "traces"])
def test_random_forest_parity(lp, ctx, case):
    """NEXT-1 (DESIGN R33-R36): the random-forest regressor — Poisson(1) bootstrap
    counts, per-node feature samples, leaf = W / T — bit-exact with the oracle: trees, training
    predictions, predictions, and the MDI importance."""
    import synth as sy
    if case == "c2":
        d = sy.make("C2")
        X, y, w, uc, kw = d.X, d.y, None, d.users_col, dict(n_trees=12, max_depth=6, max_features=0.5, seed=3)
    elif case == "s1":
        d = sy.make_s1(40001, seed=2)
        X, y, w, uc, kw = d.X, d.y, d.w, d.users_col, dict(n_trees=6, max_depth=8, max_features=0.25, seed=9,
                                                          min_child_weight=2.0)
    else:
        T = sy.make_traces(150_000, seed=0)
        oi, ii = sy.TRACE_PARAMS.index("output_tokens"), sy.TRACE_PARAMS.index("input_tokens")
        lat = (0.02 * T[:, oi] + 0.002 * T[:, ii]).astype(np.float32)
        X, y, w, uc, kw = T, np.stack([lat, 2 * lat], axis=1), None, T.shape[1] - 1, dict(n_trees=8, max_depth=7,
                                                                                         max_features=0.5, seed=1)
    om, otp = oracle.fit(X, y, oracle.rf_hparams(**kw), uc, w=w, return_train_pred=True)
    gm = lp.fit(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), lp.rf_hparams(**kw), uc,
                w=None if w is None else torch.from_numpy(w).cuda())
    _assert_same_model(om, gm.export(), case)
    assert _bits_equal(otp, gm.train_pred(len(X)))
    assert _bits_equal(oracle.predict(om, X), gm.predict(ctx, X))
    assert np.array_equal(oracle.importance(om), gm.importance())
    gm.free()


# ------------------------------------------------------------------ >256 bins, exact tree method
def _c1_many_distinct():
    d = synth.make("C1")
    X = d.X.copy()
    X[:, 1] = np.asarray(synth.u01(4, np.arange(len(X)), 77) * 1000.0, np.float32)   # a continuous LLM-side feature
    return d, X


def test_cv_wide_bins_and_exact_parity(lp, ctx):
    """NEXT-4 ("tree building method" and "number of bins"): the nested CV with 300 bins and
    with the exact method on data with 320 distinct values in one feature — 16-bit codes in the
    batched small-fit path — equals the oracle fold by fold."""
    d, X = _c1_many_distinct()
    gk = [dict(n_trees=8, max_depth=4, max_bin=300), dict(n_trees=8, max_depth=4, tree_method=1),
          dict(n_trees=8, max_depth=4, max_bin=1024, eta=0.5)]
    of = oracle.cv(X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [oracle.hparams(**k) for k in gk],
                   L1, L2, U, d.cost)
    gf = lp.cv(ctx, X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [lp.hparams(**k) for k in gk], L1,
               L2, U, d.cost)
    assert of == gf
    for k in gk:   # each point alone (plain LOO) too
        assert oracle.cv(X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, [oracle.hparams(**k)], L1, L2,
                         U, d.cost) == lp.cv(ctx, X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof,
                                             [lp.hparams(**k)], L1, L2, U, d.cost)


def test_fit_bins_limits_and_exact(lp, ctx):
    """llmpilot_fit keeps 8-bit codes: max_bin > 256 and exact with > 256 distinct values are
    LLMP_EINVAL; exact on paper-shaped data (<= 256 distinct values per feature) equals hist with
    256 bins, which is exact there (DESIGN R13)."""
    d, X = _c1_many_distinct()
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, X, d.y, lp.hparams(n_trees=2, max_bin=300), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    with pytest.raises(lp.LLMPilotError, match="EINVAL"):
        lp.fit(ctx, X, d.y, lp.hparams(n_trees=2, tree_method=1), d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof)
    d2 = synth.make("C2")
    a = lp.fit(ctx, d2.X, d2.y, lp.hparams(n_trees=10, tree_method=1), d2.users_col, d2.llm_id, d2.prof_id, d2.n_llm,
               d2.n_prof).export()
    b = lp.fit(ctx, d2.X, d2.y, lp.hparams(n_trees=10), d2.users_col, d2.llm_id, d2.prof_id, d2.n_llm,
               d2.n_prof).export()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    om = oracle.fit(d2.X, d2.y, oracle.hparams(n_trees=10, max_depth=6, tree_method=1), d2.users_col, d2.llm_id,
                    d2.prof_id, d2.n_llm, d2.n_prof, L1, L2)
    _assert_same_model(om, a)
