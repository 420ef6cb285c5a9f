"""Pins for the oracle's random-forest regressor ("a RF
regressor ... to predict the latency", "a RF regressor to predict the TTFT and ITL latencies"
and their MDI studies; readings R33-R36).  Each test checks the oracle against something
other than itself: the Poisson(1) law, a textbook library routine (sklearn's weighted CART, to which
one bootstrap tree reduces), replication semantics of integer bootstrap counts, and the per-node
feature sample re-derived from the counter-based generator."""
import math

import numpy as np
import pytest

import oracle

from test_oracle_pins import _leaf_ids, _same_partition


def test_poisson1_law_and_counter_based():
    """R34: counts follow Poisson(1) (chi-square over k = 0..5, >= 6 pooled; 200K draws) and are a
    pure function of (seed, tree, row)."""
    n = 200_000
    c = np.array([oracle.poisson1(7, 3, i) for i in range(n)])
    assert abs(c.mean() - 1.0) < 0.01 and abs(c.var() - 1.0) < 0.02
    pmf = [math.exp(-1) / math.factorial(k) for k in range(6)]
    exp = np.array(pmf + [1 - sum(pmf)]) * n
    obs = np.array([np.sum(c == k) for k in range(6)] + [np.sum(c >= 6)])
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert chi2 < 22.46   # chi-square, 6 dof, p = 0.001
    assert [oracle.poisson1(7, 3, i) for i in (0, 5, 99)] == [c[0], c[5], c[99]]
    assert any(oracle.poisson1(8, 3, i) != c[i] for i in range(50))        # the seed matters
    assert any(oracle.poisson1(7, 4, i) != c[i] for i in range(50))        # the tree matters


def _dyadic_data(seed, m=70, F=3):
    rng = np.random.default_rng(seed)
    a = (2 * rng.permutation(np.arange(1, 220))[:m] + 1) / 512.0
    y1 = np.concatenate([a, a / 2 + 0.25]).astype(np.float32)
    n = len(y1)
    X = rng.standard_normal((n, F)).astype(np.float32)
    y = np.stack([y1, y1], axis=1)
    w = rng.choice([0.5, 1.0], n).astype(np.float32)
    return X, y, w


@pytest.mark.parametrize("D", [1, 2, 4])
def test_rf_tree_is_weighted_cart_on_bootstrap_counts(D):
    """R33/R34/R36: one forest tree (max_features = 1) is weighted CART on w_i * c_i, c_i its
    Poisson(1) bootstrap counts — the same tree sklearn grows on the rows replicated c_i times — and
    its leaf value is the (c w)-weighted mean of y (dyadic data: exact).  A forest of T trees
    averages: prediction = sum_t (float)(W_t / T)."""
    from sklearn.tree import DecisionTreeRegressor
    X, y, w = _dyadic_data(3)
    n = len(X)
    T = 4
    hp = oracle.rf_hparams(n_trees=T, max_depth=D, seed=11)
    model, tp = oracle.fit(X, y, hp, users_col=2, w=w, return_train_pred=True)
    assert model.base[0] == 0.0 and model.base[1] == 0.0
    acc = np.zeros(n, np.float32)
    for t in range(T):
        c = np.array([oracle.poisson1(11, t, i) for i in range(n)], np.float64)
        sw = c * w
        sk = DecisionTreeRegressor(max_depth=D, random_state=0).fit(X[sw > 0], y[sw > 0, 0], sample_weight=sw[sw > 0])
        sub = oracle.Model(model.F, hp, model.cuts, model.ncuts, np.zeros(2, np.float32), model.feat[:, t:t + 1],
                           model.bin[:, t:t + 1], model.thr[:, t:t + 1], model.val[:, t:t + 1])
        keep = sw > 0
        assert _same_partition(_leaf_ids(sub, X[keep]), sk.apply(X[keep])), (D, t)
        # leaf values: the weighted mean / T
        pred_t = oracle.predict(sub, X[keep])[:, 0]
        np.testing.assert_allclose(pred_t * T, sk.predict(X[keep]), rtol=0, atol=1e-7)
        acc = acc + oracle.predict(sub, X)[:, 0]
    assert np.array_equal(acc.view(np.uint32), tp[:, 0].view(np.uint32))   # tree-order fp32 sum = training prediction
    assert np.array_equal(oracle.predict(model, X).view(np.uint32), tp.view(np.uint32))


def test_rf_without_bootstrap_trees_are_identical():
    """rf_bootstrap = 0, max_features = 1: every tree is the same CART on w, so the forest's
    prediction equals one tree's (T = 4, (float)(W/4) exact)."""
    from sklearn.tree import DecisionTreeRegressor
    X, y, w = _dyadic_data(5)
    hp = oracle.rf_hparams(n_trees=4, max_depth=3, bootstrap=0)
    model = oracle.fit(X, y, hp, users_col=2, w=w)
    for t in range(1, 4):
        assert np.array_equal(model.feat[:, t], model.feat[:, 0]) and np.array_equal(model.val[:, t], model.val[:, 0])
    sk = DecisionTreeRegressor(max_depth=3, random_state=0).fit(X, y[:, 0], sample_weight=w)
    np.testing.assert_allclose(oracle.predict(model, X)[:, 0], sk.predict(X), rtol=0, atol=1e-7)


def test_rf_node_feature_samples():
    """R35: each split node's feature belongs to the node's own sample of ceil(max_features F)
    features — re-derived here from rng4(seed, 2 target + 1, t, (k + 1) 32 + f) — and the samples
    differ between nodes (per-node, not per-tree, column sampling)."""
    rng = np.random.default_rng(2)
    n, F = 3000, 8
    X = rng.standard_normal((n, F)).astype(np.float32)
    y = np.stack([X @ rng.standard_normal(F) + 0.1 * rng.standard_normal(n)] * 2, axis=1).astype(np.float32)
    seed, mf, T, D = 21, 0.375, 3, 4
    model = oracle.fit(X, y, oracle.rf_hparams(n_trees=T, max_depth=D, max_features=mf, seed=seed), users_col=F - 1)
    mk = math.ceil(mf * F)
    samples = set()
    checked = 0
    for tg in range(2):
        for t in range(T):
            for k in range((1 << D) - 1):
                f = model.feat[tg, t, k]
                keys = [oracle.rng4(seed, 2 * tg + 1, t, (k + 1) * 32 + j) for j in range(F)]
                order = sorted(range(F), key=lambda j: (keys[j], j))
                samp = frozenset(order[:mk])
                samples.add(samp)
                if f >= 0:
                    assert f in samp, (tg, t, k)
                    checked += 1
    assert checked > 20 and len(samples) > 5


def test_rf_mdi_on_traces_favours_output_tokens():
    """the RF + MDI importance study on the traces ranks the number of output tokens first
    (synthetic traces whose latency model is driven by output then input tokens)."""
    import synth
    T = synth.make_traces(20000, seed=0)
    P = T.shape[1]
    oi = synth.TRACE_PARAMS.index("output_tokens")
    ii = synth.TRACE_PARAMS.index("input_tokens")
    lat = (0.02 * T[:, oi] + 0.002 * T[:, ii] + 0.05 * T[:, synth.TRACE_PARAMS.index("batch_size")]).astype(np.float32)
    y = np.stack([lat, lat], axis=1)
    model = oracle.fit(T, y, oracle.rf_hparams(n_trees=8, max_depth=6, max_features=0.5, seed=1), users_col=P - 1)
    imp = oracle.importance(model)[0]
    assert np.argmax(imp) == oi and imp[oi] > imp[ii]
    assert abs(imp.sum() - 1.0) < 1e-12
