"""oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded CPU oracle of the LLM-Pilot hot path (arxiv 2410.02425), written
in C (``oracle/llmpilot_oracle.c``) from SURVEY.md §8(c) O1-O12 and PAPER.md.  This module is a
thin ctypes wrapper with numpy marshalling.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product package ``paper_2410_02425_b200`` never does,
and this module never imports the product package: the two share no code.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "llmpilot_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
MAX_F = 32
MAX_BIN = 1024   # bins per feature (16-bit codes, NEXT-4)

GCC_FLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-msse2", "-mfpmath=sse",
             "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, no FMA contraction).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "llmpilot_oracle.h"))):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Hparams(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("max_depth", C.c_int32), ("max_bin", C.c_int32),
                ("grad_bits", C.c_int32), ("eta", C.c_float), ("lambda_", C.c_float),
                ("min_child_weight", C.c_float), ("subsample", C.c_float),
                ("colsample_bytree", C.c_float), ("seed", C.c_uint64),
                ("use_eq4_weights", C.c_int32), ("monotone_users", C.c_int32),
                ("model", C.c_int32), ("max_features", C.c_float), ("rf_bootstrap", C.c_int32),
                ("tree_method", C.c_int32)]


def hparams(n_trees=20, max_depth=4, max_bin=256, grad_bits=14, eta=0.3, lambda_=1.0,
            min_child_weight=1.0, subsample=1.0, colsample_bytree=1.0, seed=0, use_eq4_weights=1,
            monotone_users=1, model=0, max_features=1.0, rf_bootstrap=1, tree_method=0) -> Hparams:
    """Defaults = XGBoost defaults with K = 14 gradient bits.
    model=1: random forest (DESIGN R33-R36)."""
    return Hparams(n_trees, max_depth, max_bin, grad_bits, eta, lambda_, min_child_weight,
                   subsample, colsample_bytree, seed, use_eq4_weights, monotone_users, model, max_features,
                   rf_bootstrap, tree_method)


def rf_hparams(n_trees=20, max_depth=8, max_bin=256, max_features=1.0, min_child_weight=0.0, seed=0,
               use_eq4_weights=0, bootstrap=1, grad_bits=14) -> Hparams:
    """Random-forest regressor: lambda 0, no monotone constraint, no row subsampling."""
    return hparams(n_trees=n_trees, max_depth=max_depth, max_bin=max_bin, grad_bits=grad_bits, eta=1.0, lambda_=0.0,
                   min_child_weight=min_child_weight, seed=seed, use_eq4_weights=use_eq4_weights, monotone_users=0,
                   model=1, max_features=max_features, rf_bootstrap=bootstrap)


def poisson1(seed, t, i) -> int:
    return lib().orc_poisson1(seed, t, i)


class Split(C.Structure):
    _fields_ = [("f", C.c_int32), ("b", C.c_int32), ("loss", C.c_double), ("wl", C.c_double),
                ("wr", C.c_double), ("GLq", C.c_int64), ("HLq", C.c_int64), ("GRq", C.c_int64),
                ("HRq", C.c_int64)]


class Rec(C.Structure):
    _fields_ = [("profile", C.c_int32), ("n_pods", C.c_int64), ("cost", C.c_double),
                ("u_max", C.c_int32)]


class Fold(C.Structure):
    _fields_ = [("llm", C.c_int32), ("hp_index", C.c_int32), ("rec", Rec), ("truth", Rec),
                ("success", C.c_int32), ("overspend", C.c_double), ("truth_feasible", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        L = _lib
        L.orc_rng4.restype = C.c_uint64
        L.orc_rng4.argtypes = [C.c_uint64] * 4
        L.orc_poisson1.restype = C.c_int32
        L.orc_poisson1.argtypes = [C.c_uint64, C.c_int32, C.c_int64]
        L.orc_weights.argtypes = [C.c_int64, P, P, P, C.c_int32, C.c_int32, C.c_float, C.c_float, P]
        L.orc_cuts.restype = C.c_int
        L.orc_cuts.argtypes = [P, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int32, P, P]
        L.orc_codes.argtypes = [P, C.c_int64, C.c_int32, P, P, P]
        L.orc_quantize.restype = C.c_int32
        L.orc_quantize.argtypes = [C.c_int64, P, C.c_int32, P]
        L.orc_calc_weight.restype = C.c_double
        L.orc_calc_weight.argtypes = [C.c_double] * 6
        L.orc_calc_gain.restype = C.c_double
        L.orc_calc_gain.argtypes = [C.c_double] * 4
        L.orc_node_hist.argtypes = [P, C.c_int32, P, C.c_int64, P, P, P, P]
        L.orc_best_split.restype = C.c_int
        L.orc_best_split.argtypes = [P, P, C.c_int32, P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, P]
        L.orc_fit.restype = C.c_int
        L.orc_fit.argtypes = [P, P, P, P, P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                              C.c_int64, C.c_int64, P, C.c_float, C.c_float, P, P, P, P, P, P, P, P,
                              C.c_int32]
        L.orc_fit_gain.restype = C.c_int
        L.orc_fit_gain.argtypes = L.orc_fit.argtypes[:22] + [P] + L.orc_fit.argtypes[22:]
        L.orc_importance.restype = None
        L.orc_importance.argtypes = [C.c_int32, C.c_int32, C.c_int32, P, P, C.c_int32, P]
        L.orc_wg_build.restype = C.c_int
        L.orc_wg_build.argtypes = [P, C.c_int64, C.c_int32, P, P, P, P, P]
        L.orc_wg_sample.restype = None
        L.orc_wg_sample.argtypes = [P, P, C.c_int64, C.c_int32, P, P, C.c_uint64, C.c_int64, C.c_int64, P]
        L.orc_predict.argtypes = [P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, P, P, P, P, P]
        L.orc_recommend.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, P, P, P, C.c_float, C.c_float,
                                    C.c_int64, P]
        L.orc_cv.restype = C.c_int
        L.orc_cv.argtypes = [P, P, P, P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P,
                             C.c_int32, C.c_float, C.c_float, C.c_int64, P, P, P, P, P, P]
        L.orc_wmape.restype = C.c_double
        L.orc_wmape.argtypes = [C.c_int64, P, P, P, C.c_int]
        L.orc_so_score.restype = C.c_double
        L.orc_so_score.argtypes = [C.c_double, C.c_double]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def rng4(seed, a, b, c) -> int:
    return int(lib().orc_rng4(seed, a, b, c))


def weights(y, llm_id, prof_id, n_llm, n_prof, L1, L2) -> np.ndarray:
    """O1 / Eq. (4)."""
    y = _c(y, np.float32); li = _c(llm_id, np.int32); pi = _c(prof_id, np.int32)
    w = np.empty(len(li), np.float32)
    lib().orc_weights(len(li), _p(y), _p(li), _p(pi), n_llm, n_prof, L1, L2, _p(w))
    return w


def cuts(X, max_bin=256, row_offset=0, n_global=None):
    """O2 cuts -> (cuts [F, MAX_BIN - 1] float32, ncuts [F] int32).  max_bin = 0: exact (every
    distinct value its own bin)."""
    X = _c(X, np.float32)
    n, F = X.shape
    ct = np.zeros((MAX_F, MAX_BIN - 1), np.float32)
    nc = np.zeros(MAX_F, np.int32)
    rc = lib().orc_cuts(_p(X), n, F, row_offset, n if n_global is None else n_global, max_bin, _p(ct), _p(nc))
    if rc:
        raise ValueError("orc_cuts: invalid input")
    return ct[:F].copy(), nc[:F].copy()


def codes(X, ct, nc) -> np.ndarray:
    X = _c(X, np.float32)
    n, F = X.shape
    ctf = np.zeros((MAX_F, MAX_BIN - 1), np.float32); ctf[:F, :ct.shape[1]] = ct
    ncf = np.zeros(MAX_F, np.int32); ncf[:F] = nc
    out = np.empty((n, F), np.uint16)
    lib().orc_codes(_p(X), n, F, _p(ctf), _p(ncf), _p(out))
    return out if out.size and out.max() > 255 else out.astype(np.uint8)


def quantize(v, K):
    v = _c(v, np.float32)
    q = np.empty(len(v), np.int32)
    e = lib().orc_quantize(len(v), _p(v), K, _p(q))
    return int(e), q


def calc_weight(G, H, lo, hi, lambda_, mcw) -> float:
    return lib().orc_calc_weight(G, H, lo, hi, lambda_, mcw)


def calc_gain(G, H, w, lambda_) -> float:
    return lib().orc_calc_gain(G, H, w, lambda_)


def node_hist(codes_, rows, qg, qh):
    codes_ = _c(codes_, np.uint16); rows = _c(rows, np.int64)
    qg = _c(qg, np.int32); qh = _c(qh, np.int32)
    F = codes_.shape[1]
    Hg = np.zeros((F, MAX_BIN), np.int64); Hh = np.zeros((F, MAX_BIN), np.int64)
    lib().orc_node_hist(_p(codes_), F, _p(rows), len(rows), _p(qg), _p(qh), _p(Hg), _p(Hh))
    if codes_.size == 0 or int(codes_.max()) < 256:   # 8-bit codes: the [F][256] layout of the GPU's hook
        return Hg[:, :256].copy(), Hh[:, :256].copy()
    return Hg, Hh


def best_split(Hg, Hh, nbins, users_col=-1, monotone_users=0, eg=0, eh=0, K=0, lo=-np.inf, hi=np.inf,
               lambda_=1.0, mcw=1.0, fmask=None):
    F = np.asarray(Hg).shape[0]
    if np.asarray(Hg).shape[1] < MAX_BIN:   # accept narrower hand-built histograms
        Hg = np.pad(np.asarray(Hg), ((0, 0), (0, MAX_BIN - np.asarray(Hg).shape[1])))
        Hh = np.pad(np.asarray(Hh), ((0, 0), (0, MAX_BIN - np.asarray(Hh).shape[1])))
    Hg = _c(Hg, np.int64); Hh = _c(Hh, np.int64)
    nb = _c(nbins, np.int32)
    fm = _c(np.ones(F) if fmask is None else fmask, np.uint8)
    s = Split()
    ok = lib().orc_best_split(_p(Hg), _p(Hh), F, _p(nb), _p(fm), users_col, monotone_users, eg, eh, K,
                              lo, hi, lambda_, mcw, C.byref(s))
    return (s if ok else None)


class Model:
    """Oracle ensemble: complete-binary trees [2][T][2^(D+1)-1]."""

    def __init__(self, F, hp, cuts_, ncuts, base, feat, bin_, thr, val, gain=None):
        self.F, self.hp = F, hp
        self.cuts, self.ncuts, self.base = cuts_, ncuts, base
        self.feat, self.bin, self.thr, self.val = feat, bin_, thr, val
        self.gain = gain   # [2][T][nodes] split losses (fp64), 0 at leaves / unused slots

    @property
    def n_trees(self):
        return self.feat.shape[1]


def fit(X, y, hp: Hparams, users_col, llm_id=None, prof_id=None, n_llm=1, n_prof=1, L1=100.0, L2=50.0,
        w=None, row_offset=0, n_global=None, n_trees_limit=0, return_train_pred=False):
    """O1-O9.  Returns Model (and the internal training predictions if asked)."""
    X = _c(X, np.float32); y = _c(y, np.float32)
    n, F = X.shape
    li = _c(np.zeros(n) if llm_id is None else llm_id, np.int32)
    pi = _c(np.zeros(n) if prof_id is None else prof_id, np.int32)
    wv = None if w is None else _c(w, np.float32)
    T, D = hp.n_trees, hp.max_depth
    nn = (1 << (D + 1)) - 1
    ct = np.zeros((MAX_F, MAX_BIN - 1), np.float32)
    nc = np.zeros(MAX_F, np.int32)
    base = np.zeros(2, np.float32)
    feat = np.full((2, T, nn), -2, np.int32)
    bin_ = np.zeros((2, T, nn), np.int32)
    thr = np.zeros((2, T, nn), np.float32)
    val = np.zeros((2, T, nn), np.float32)
    gain = np.zeros((2, T, nn), np.float64)
    tp = np.zeros((n, 2), np.float32)
    rc = lib().orc_fit_gain(_p(X), _p(y), None if wv is None else _p(wv), _p(li), _p(pi), n, F, users_col, n_llm,
                            n_prof, row_offset, n if n_global is None else n_global, C.byref(hp), L1, L2, _p(ct),
                            _p(nc), _p(base), _p(feat), _p(bin_), _p(thr), _p(val), _p(gain), _p(tp), n_trees_limit)
    if rc:
        raise ValueError("orc_fit: invalid input")
    if n_trees_limit and n_trees_limit < T:
        feat, bin_, thr, val, gain = (a[:, :n_trees_limit].copy() for a in (feat, bin_, thr, val, gain))
    m = Model(F, hp, ct[:F].copy(), nc[:F].copy(), base, feat, bin_, thr, val, gain)
    return (m, tp) if return_train_pred else m


def importance(model: Model, normalize=True) -> np.ndarray:
    """MDI feature importance: 2 x F, fp64."""
    feat = _c(model.feat, np.int32)
    T, nn = feat.shape[1], feat.shape[2]
    D = int(np.log2(nn + 1)) - 1
    out = np.zeros((2, model.F), np.float64)
    lib().orc_importance(T, D, model.F, _p(feat), _p(_c(model.gain, np.float64)), 1 if normalize else 0, _p(out))
    return out


WG_BINS = 64


class WorkloadModel:
    """Workload-generator model (§III-B): per-parameter bins and centres and the
    sparse joint histogram (ascending mixed-radix keys with their row counts)."""

    def __init__(self, nbins, centres, keys, counts):
        self.nbins, self.centres, self.keys, self.counts = nbins, centres, keys, counts

    @property
    def P(self):
        return len(self.nbins)


def wg_build(T) -> WorkloadModel:
    T = _c(T, np.float32)
    n, P = T.shape
    nb = np.zeros(P, np.int32)
    ce = np.zeros((P, WG_BINS), np.float32)
    keys = np.zeros(n, np.uint64)
    counts = np.zeros(n, np.int64)
    m = C.c_int64(0)
    if lib().orc_wg_build(_p(T), n, P, _p(nb), _p(ce), _p(keys), _p(counts), C.byref(m)):
        raise ValueError("orc_wg_build: invalid input")
    return WorkloadModel(nb, ce, keys[:m.value].copy(), counts[:m.value].copy())


def wg_sample(model: WorkloadModel, n_samples, seed=0, first=0) -> np.ndarray:
    """samples first .. first + n_samples - 1 of `seed`, n_samples x P."""
    out = np.zeros((n_samples, model.P), np.float32)
    lib().orc_wg_sample(_p(model.keys), _p(model.counts), len(model.keys), model.P, _p(model.nbins),
                        _p(model.centres), seed, first, n_samples, _p(out))
    return out


def predict(model: Model, X) -> np.ndarray:
    X = _c(X, np.float32)
    n, F = X.shape
    out = np.empty((n, 2), np.float32)
    T = model.feat.shape[1]
    D = model.hp.max_depth
    lib().orc_predict(_p(X), n, F, T, D, _p(model.base), _p(_c(model.feat, np.int32)),
                      _p(_c(model.thr, np.float32)), _p(_c(model.val, np.float32)), _p(out))
    return out


def recommend(pred, user_levels, cost, L1, L2, U, allowed=None):
    """O11 / Eq. (1)-(3).  pred: [n_llm, n_prof, n_levels, 2]."""
    pred = _c(pred, np.float32)
    n_llm, n_prof, n_lv, _ = pred.shape
    lv = _c(user_levels, np.int32); cs = _c(cost, np.float64)
    al = None if allowed is None else _c(allowed, np.uint8)
    out = (Rec * n_llm)()
    lib().orc_recommend(_p(pred), n_llm, n_prof, n_lv, _p(lv), _p(cs), None if al is None else _p(al), L1, L2, U,
                        out)
    return [(r.profile, r.n_pods, r.cost, r.u_max) for r in out]


def cv(X, y, llm_id, prof_id, users_col, n_llm, n_prof, grid, L1, L2, U, cost):
    """O12 nested leave-one-LLM-out CV.  Returns (folds, S, O, SO)."""
    X = _c(X, np.float32); y = _c(y, np.float32)
    li = _c(llm_id, np.int32); pi = _c(prof_id, np.int32)
    n, F = X.shape
    g = (Hparams * len(grid))(*grid)
    cs = _c(cost, np.float64)
    folds = (Fold * n_llm)()
    nf = C.c_int32(0)
    S, O, SO = C.c_double(), C.c_double(), C.c_double()
    rc = lib().orc_cv(_p(X), _p(y), _p(li), _p(pi), n, F, users_col, n_llm, n_prof, g, len(grid), L1, L2, U,
                      _p(cs), folds, C.byref(nf), C.byref(S), C.byref(O), C.byref(SO))
    if rc:
        raise ValueError("orc_cv: invalid input")
    out = []
    for f in folds[:nf.value]:
        out.append(dict(llm=f.llm, hp_index=f.hp_index,
                        rec=(f.rec.profile, f.rec.n_pods, f.rec.cost, f.rec.u_max),
                        truth=(f.truth.profile, f.truth.n_pods, f.truth.cost, f.truth.u_max),
                        success=f.success, overspend=f.overspend, truth_feasible=f.truth_feasible))
    return out, S.value, O.value, SO.value


def wmape(pred, y, w, target) -> float:
    pred = _c(pred, np.float32); y = _c(y, np.float32); w = _c(w, np.float32)
    return lib().orc_wmape(len(w), _p(pred), _p(y), _p(w), target)


def so_score(S, O) -> float:
    return lib().orc_so_score(S, O)
