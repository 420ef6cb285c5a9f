"""Oracle pins for the workload generator (§III-B),
checked against brute force and the paper's own statements, not against the oracle's formulas:

* P:L128 "64 bins (unless the cardinality of the parameter is lower, in which case ... as many bins
  as there are unique values)" and "approximately equal number of requests" per bin;
* P:L128 values replaced by the centres of their bins (a single-valued bin's centre is the value);
* P:L128-130 one joint bin per distinct combination of bin assignments, counts = requests in it;
* P:L132 a sample picks a joint bin with probability count / n and emits the bins' centres.
"""
import collections

import numpy as np
import pytest

import oracle
import synth


def _model_tuples(m):
    """decode every key into its per-parameter bin tuple (mixed radix, parameter 0 fastest)"""
    out = []
    for k in m.keys.tolist():
        t = []
        for nb in m.nbins.tolist():
            t.append(k % nb)
            k //= nb
        out.append(tuple(t))
    return out


def test_low_cardinality_one_bin_per_value_and_centre_is_the_value():
    rng = np.random.default_rng(1)
    vals = np.array([-3.5, -0.0, 0.0, 1.0, 2.25, 1e6], np.float32)    # -0 and +0 are one value
    T = np.stack([rng.choice(vals, 5000), rng.integers(0, 64, 5000)], axis=1).astype(np.float32)
    m = oracle.wg_build(T)
    assert m.nbins.tolist() == [5, 64]
    assert m.centres[0, :5].tolist() == [-3.5, 0.0, 1.0, 2.25, 1e6]
    assert m.centres[1, :64].tolist() == list(range(64))


def test_equal_frequency_bins_and_interval_centres():
    n = 6400
    x = np.random.default_rng(2).permutation(np.arange(n)).astype(np.float32) * 0.5   # distinct values
    m = oracle.wg_build(x[:, None])
    assert m.nbins[0] == 64
    tuples = _model_tuples(m)
    per_bin = collections.Counter()
    for t, c in zip(tuples, m.counts.tolist()):
        per_bin[t[0]] += c
    assert set(per_bin.values()) == {100}                 # exactly n / 64 requests in each bin
    # bin b holds the values 100 b .. 100 b + 99 (times 0.5): its centre is their midpoint
    assert np.array_equal(m.centres[0, :64], ((100 * np.arange(64) + 49.5) * 0.5).astype(np.float32))


def test_joint_histogram_is_bruteforce_count_of_bin_tuples():
    """Bins are contiguous value ranges that never split equal values; a row's bin tuple,
    re-derived by brute force from each column's sorted values and the model's per-bin counts,
    reproduces the model's joint counts exactly; each centre is the midpoint of its bin's
    smallest and largest member."""
    T = synth.make_traces(3000, seed=4)
    m = oracle.wg_build(T)
    assert (np.diff(m.keys.astype(np.float64)) > 0).all()          # ascending, distinct
    assert m.counts.sum() == len(T) and (m.counts > 0).all()
    tuples = _model_tuples(m)
    ranks = []
    for p in range(T.shape[1]):
        marg = collections.Counter()
        for t, c in zip(tuples, m.counts.tolist()):
            assert 0 <= t[p] < m.nbins[p]
            marg[t[p]] += c
        col = np.where(T[:, p] == 0, np.float32(0), T[:, p])
        srt = np.sort(col)
        edges = np.cumsum([marg[b] for b in range(m.nbins[p])])
        assert edges[-1] == len(col)
        for e in edges[:-1]:
            assert srt[e - 1] < srt[e]                              # no value split across bins
        starts = np.concatenate([[0], edges[:-1]])
        for b in range(m.nbins[p]):
            lo, hi = float(srt[starts[b]]), float(srt[edges[b] - 1])
            assert m.centres[p, b] == np.float32((lo + hi) * 0.5)
        upper = srt[edges - 1]                                     # largest member of each bin
        ranks.append(np.searchsorted(upper, col, side="left"))
    rows = collections.Counter(zip(*[r.tolist() for r in ranks]))
    assert rows == collections.Counter(dict(zip(tuples, m.counts.tolist())))


def test_sampling_is_inverse_cdf_over_joint_bins():
    T = synth.make_traces(2000, seed=5)
    m = oracle.wg_build(T)
    n = int(m.counts.sum())
    cum = np.cumsum(m.counts)
    tuples = _model_tuples(m)
    S = oracle.wg_sample(m, 500, seed=9, first=1000)
    for s in range(500):
        r = oracle.rng4(9, 0x5747, 1000 + s, 0)
        t = (r * n) >> 64                                       # exact integer arithmetic
        j = int(np.searchsorted(cum, t, side="right"))          # first cumulative count > t
        expect = [m.centres[p, tuples[j][p]] for p in range(m.P)]
        assert S[s].tolist() == expect
    # offsets: samples are indexed globally (shards draw disjoint, reproducible ranges)
    assert np.array_equal(oracle.wg_sample(m, 200, seed=9, first=1100), S[100:300])


def test_sampled_frequencies_follow_counts():
    """each joint bin is drawn with probability count / n (chi-square, fixed seed)."""
    rng = np.random.default_rng(6)
    a = rng.integers(0, 4, 4000)
    T = np.stack([a, 10 * a + rng.integers(0, 2, 4000)], axis=1).astype(np.float32)   # correlated
    m = oracle.wg_build(T)
    assert len(m.keys) == 8                                  # 4 x 2 combinations occur, not 4 x 8
    S = oracle.wg_sample(m, 200000, seed=3)
    # correlation preserved: the second parameter's bin always matches the first's
    assert np.array_equal(np.floor(S[:, 1] / 10), S[:, 0])
    obs = collections.Counter(map(tuple, S.tolist()))
    n = m.counts.sum()
    tuples = _model_tuples(m)
    chi2 = 0.0
    for t, c in zip(tuples, m.counts.tolist()):
        key = (float(m.centres[0, t[0]]), float(m.centres[1, t[1]]))
        e = 200000 * c / n
        chi2 += (obs[key] - e) ** 2 / e
    assert chi2 < 24.3        # 7 degrees of freedom, p = 0.001


def test_invalid_inputs():
    with pytest.raises(ValueError):
        oracle.wg_build(np.array([[1.0, np.nan]], np.float32))
    # key space above 2^63: 11 parameters x 64 bins = 2^66
    X = np.tile(np.arange(64, dtype=np.float32)[:, None], (1, 11))
    with pytest.raises(ValueError):
        oracle.wg_build(X)
