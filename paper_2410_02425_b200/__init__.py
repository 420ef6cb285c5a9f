"""paper_2410_02425_b200 — B200-native LLM-Pilot hot path (arxiv 2410.02425).

Thin ctypes binding over the C-ABI in ``include/llmpilot.h`` (``libllmpilot.so``, built in-tree
by ``paper_2410_02425_b200.build``).  Argument marshalling only: every step of the path runs in
the library's sm_100a kernels.  Arrays may be torch tensors (CUDA or CPU) or numpy arrays (host);
host arrays are copied to the device inside the C call.  If the library is missing or cannot be
loaded this module raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libllmpilot.so")

LLMP_OK = 0
STATUS = {0: "LLMP_OK", 1: "LLMP_EINVAL", 2: "LLMP_ENOMEM", 3: "LLMP_ECUDA", 4: "LLMP_ENCCL", 5: "LLMP_EINTERNAL"}
N_KERNEL_CLASSES = 16


class LLMPilotError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class HParams(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("max_depth", C.c_int32), ("max_bin", C.c_int32),
                ("grad_bits", C.c_int32), ("eta", C.c_float), ("lambda_", C.c_float),
                ("min_child_weight", C.c_float), ("subsample", C.c_float),
                ("colsample_bytree", C.c_float), ("seed", C.c_uint64),
                ("use_eq4_weights", C.c_int32), ("monotone_users", C.c_int32),
                ("model", C.c_int32), ("max_features", C.c_float), ("rf_bootstrap", C.c_int32),
                ("tree_method", C.c_int32)]


class DatasetC(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("row_offset", C.c_int64), ("n_rows_global", C.c_int64),
                ("n_features", C.c_int32), ("users_col", C.c_int32), ("n_llm", C.c_int32),
                ("n_prof", C.c_int32), ("X", C.c_void_p), ("y", C.c_void_p), ("llm_id", C.c_void_p),
                ("profile_id", C.c_void_p), ("w", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("launches", C.c_uint64 * N_KERNEL_CLASSES), ("timed", C.c_uint64 * N_KERNEL_CLASSES),
                ("ms", C.c_double * N_KERNEL_CLASSES), ("rows", C.c_double * N_KERNEL_CLASSES),
                ("total_launches", C.c_uint64)]


class Rec(C.Structure):
    _fields_ = [("profile", C.c_int32), ("n_pods", C.c_int64), ("cost", C.c_double), ("u_max", C.c_int32)]


class CvFold(C.Structure):
    _fields_ = [("llm", C.c_int32), ("hp_index", C.c_int32), ("rec", Rec), ("truth", Rec),
                ("success", C.c_int32), ("overspend", C.c_double), ("truth_feasible", C.c_int32)]


class CvReport(C.Structure):
    _fields_ = [("S", C.c_double), ("O", C.c_double), ("SO", C.c_double), ("n_folds", C.c_int32),
                ("n_scored", C.c_int32), ("folds", C.POINTER(CvFold))]


_lib = None


def lib():
    """Load libllmpilot.so (raises if it is missing: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libllmpilot.so is not built (run `python -m paper_2410_02425_b200.build`)")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    L.llmpilot_last_error.restype = C.c_char_p
    L.llmpilot_version.restype = C.c_char_p
    L.llmpilot_kernel_class_name.restype = C.c_char_p
    L.llmpilot_kernel_class_name.argtypes = [C.c_int]
    for name, args in {
        "llmpilot_ctx_create": [C.c_int, P, P, C.c_int, C.c_int, C.POINTER(P)],
        "llmpilot_ctx_set_timing": [P, C.c_int],
        "llmpilot_ctx_stats": [P, C.POINTER(Stats)],
        "llmpilot_ctx_reset_stats": [P],
        "llmpilot_bin": [P, P, I64, I32, I32, P, C.POINTER(P), P],
        "llmpilot_cuts_export": [P, C.POINTER(I32), P, P],
        "llmpilot_fit": [P, C.POINTER(DatasetC), C.POINTER(HParams), F32, F32, C.POINTER(P)],
        "llmpilot_model_info": [P, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)],
        "llmpilot_model_export": [P, P, P, P, P, P],
        "llmpilot_model_train_pred": [P, P],
        "llmpilot_model_save": [P, C.c_char_p],
        "llmpilot_model_load": [P, C.c_char_p, C.POINTER(P)],
        "llmpilot_model_gains": [P, P],
        "llmpilot_model_importance": [P, I32, P],
        "llmpilot_predict": [P, P, P, I64, P],
        "llmpilot_recommend": [P, P, P, I32, I32, P, I32, I32, P, P, P, I32, F32, F32, I64, C.POINTER(Rec), P],
        "llmpilot_cv_leave_one_llm_out": [P, C.POINTER(DatasetC), C.POINTER(HParams), I32, F32, F32, I64, P,
                                          C.POINTER(C.POINTER(CvReport))],
        "llmpilot_debug_histogram": [P, P, I64, P, I64, P, P, P, P],
        "llmpilot_nccl_unique_id": [P],
        "llmpilot_ctx_create_local_group": [C.c_int, C.c_int, P],
        "llmpilot_wg_build": [P, P, I64, I32, C.POINTER(P)],
        "llmpilot_wg_info": [P, C.POINTER(I32), C.POINTER(I64), C.POINTER(I64)],
        "llmpilot_wg_export": [P, P, P, P, P],
        "llmpilot_wg_sample": [P, P, I64, C.c_uint64, I64, P],
    }.items():
        fn = getattr(L, name)
        fn.restype = C.c_int
        fn.argtypes = args
    L.llmpilot_ctx_destroy.argtypes = [P]
    L.llmpilot_cuts_free.argtypes = [P]
    L.llmpilot_model_free.argtypes = [P]
    L.llmpilot_wg_free.argtypes = [P]
    L.llmpilot_cv_report_free.argtypes = [C.POINTER(CvReport)]
    L.llmpilot_hparams_default.argtypes = [C.POINTER(HParams)]
    _lib = L
    return L


def _check(st):
    if st != LLMP_OK:
        raise LLMPilotError(st, lib().llmpilot_last_error().decode())


def version() -> str:
    return lib().llmpilot_version().decode()


def local_group(device: int, nranks: int) -> list:
    """llmpilot_ctx_create_local_group: nranks Contexts on one device sharing an in-process
    communicator (drive each from its own thread, same call sequence on every rank)."""
    hs = (C.c_void_p * nranks)()
    _check(lib().llmpilot_ctx_create_local_group(device, nranks, hs))
    return [Context._wrap(C.c_void_p(hs[r]), device, r, nranks) for r in range(nranks)]


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for Context(nccl_unique_id=..., rank, nranks)."""
    buf = C.create_string_buffer(128)
    _check(lib().llmpilot_nccl_unique_id(buf))
    return buf.raw


def kernel_class_names():
    return [lib().llmpilot_kernel_class_name(i).decode() for i in range(N_KERNEL_CLASSES)]


# ----------------------------------------------------------------------------------------------
# marshalling: (pointer, keep-alive) for torch tensors or numpy arrays
def _ptr(a, dtype):
    """Return (c_void_p, keepalive).  torch tensors pass their data_ptr (device or host);
    numpy arrays are made contiguous with the requested dtype."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            tdt = {np.float32: torch.float32, np.int32: torch.int32, np.uint8: torch.uint8,
                   np.float64: torch.float64, np.int64: torch.int64}[dtype]
            if a.dtype != tdt or not a.is_contiguous():
                a = a.to(tdt).contiguous()
            return C.c_void_p(a.data_ptr()), a
    except ImportError:
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data_as(C.c_void_p), arr


def _out_ptr(out, shape, what):
    """Pointer of a caller-supplied OUTPUT buffer: it must be C-contiguous float32 of exactly `shape`
    (the library writes through the pointer, so a converted copy would silently lose the result)."""
    if out is None:
        return None
    if tuple(out.shape) != tuple(shape):
        raise ValueError("%s must have shape %s, got %s" % (what, tuple(shape), tuple(out.shape)))
    try:
        import torch
        if isinstance(out, torch.Tensor):
            if out.dtype != torch.float32 or not out.is_contiguous():
                raise ValueError("%s must be a contiguous float32 tensor" % what)
            return C.c_void_p(out.data_ptr())
    except ImportError:
        pass
    if not isinstance(out, np.ndarray) or out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"] \
            or not out.flags["WRITEABLE"]:
        raise ValueError("%s must be a writeable C-contiguous float32 array" % what)
    return out.ctypes.data_as(C.c_void_p)


def _stream_handle(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Context:
    """llmpilot_ctx: a device, a CUDA stream, optionally an NCCL communicator."""

    def __init__(self, device: int = 0, stream=None, nccl_unique_id: Optional[bytes] = None, rank: int = 0,
                 nranks: int = 1):
        self._h = C.c_void_p()
        uid = None
        if nccl_unique_id is not None:
            uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
        _check(lib().llmpilot_ctx_create(device, _stream_handle(stream), uid, rank, nranks, C.byref(self._h)))
        self.device, self.rank, self.nranks = device, rank, nranks

    @classmethod
    def _wrap(cls, h, device, rank, nranks):
        c = cls.__new__(cls)
        c._h, c.device, c.rank, c.nranks = h, device, rank, nranks
        return c

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().llmpilot_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, every: int):
        """0: off (trees replay from CUDA graphs); k >= 1: CUDA-event-time every k-th launch of each
        kernel class (plain launches)."""
        _check(lib().llmpilot_ctx_set_timing(self._h, int(every)))

    def reset_stats(self):
        _check(lib().llmpilot_ctx_reset_stats(self._h))

    def stats(self) -> dict:
        s = Stats()
        _check(lib().llmpilot_ctx_stats(self._h, C.byref(s)))
        names = kernel_class_names()
        out = {"total_launches": int(s.total_launches), "classes": {}}
        for i, nm in enumerate(names):
            if s.launches[i] or s.rows[i]:
                timed = int(s.timed[i])
                avg = float(s.ms[i]) / timed if timed else 0.0
                out["classes"][nm] = {"launches": int(s.launches[i]), "timed": timed, "ms_timed": float(s.ms[i]),
                                      "ms_avg": avg, "ms": avg * int(s.launches[i]), "rows": float(s.rows[i])}
        return out


def hparams(n_trees=100, max_depth=6, max_bin=256, grad_bits=14, eta=0.3, lambda_=1.0, min_child_weight=1.0,
            subsample=1.0, colsample_bytree=1.0, seed=0, use_eq4_weights=1, monotone_users=1, model=0,
            max_features=1.0, rf_bootstrap=1, tree_method=0) -> HParams:
    return HParams(n_trees, max_depth, max_bin, grad_bits, eta, lambda_, min_child_weight, subsample,
                   colsample_bytree, seed, use_eq4_weights, monotone_users, model, max_features, rf_bootstrap,
                   tree_method)


def rf_hparams(n_trees=100, max_depth=8, max_bin=256, max_features=1.0, min_child_weight=0.0, seed=0,
               use_eq4_weights=0, bootstrap=1, grad_bits=14) -> HParams:
    """Random-forest regressor (DESIGN R33-R36): lambda 0, no monotone constraint."""
    return hparams(n_trees=n_trees, max_depth=max_depth, max_bin=max_bin, grad_bits=grad_bits, eta=1.0, lambda_=0.0,
                   min_child_weight=min_child_weight, seed=seed, use_eq4_weights=use_eq4_weights, monotone_users=0,
                   model=1, max_features=max_features, rf_bootstrap=bootstrap)


def _dataset(X, y, llm_id, prof_id, users_col, n_llm, n_prof, w=None, row_offset=0, n_global=None):
    n, F = int(X.shape[0]), int(X.shape[1])
    keep = []
    px, k = _ptr(X, np.float32); keep.append(k)
    py, k = _ptr(y, np.float32); keep.append(k)
    pl, k = _ptr(llm_id, np.int32); keep.append(k)
    pp, k = _ptr(prof_id, np.int32); keep.append(k)
    pw, k = _ptr(w, np.float32); keep.append(k)
    ds = DatasetC(n, row_offset, n if n_global is None else n_global, F, users_col, n_llm, n_prof, px, py, pl, pp, pw)
    return ds, keep


class Cuts:
    def __init__(self, h):
        self._h = h

    def export(self):
        F = C.c_int32()
        cuts = np.zeros((32, 255), np.float32)
        nc = np.zeros(32, np.int32)
        _check(lib().llmpilot_cuts_export(self._h, C.byref(F), cuts.ctypes.data_as(C.c_void_p),
                                          nc.ctypes.data_as(C.c_void_p)))
        return cuts[:F.value].copy(), nc[:F.value].copy()

    def __del__(self):
        try:
            if self._h:
                lib().llmpilot_cuts_free(self._h)
        except Exception:
            pass


def bin(ctx: Context, X, max_bin: int = 256, cuts: Optional[Cuts] = None, codes_out=None):
    """Quantile cuts + codes.  codes_out: a CUDA uint8 tensor of n x 32 (or None)."""
    n, F = int(X.shape[0]), int(X.shape[1])
    px, keep = _ptr(X, np.float32)
    h = C.c_void_p()
    pc = None if codes_out is None else C.c_void_p(codes_out.data_ptr())
    _check(lib().llmpilot_bin(ctx.handle, px, n, F, max_bin, cuts._h if cuts else None,
                              None if cuts else C.byref(h), pc))
    return cuts if cuts else Cuts(h)


class Model:
    """llmpilot_model: two ensembles (nTTFT, ITL)."""

    def __init__(self, h):
        self._h = h
        F, T, D, uc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().llmpilot_model_info(h, C.byref(F), C.byref(T), C.byref(D), C.byref(uc)))
        self.F, self.n_trees, self.max_depth, self.users_col = F.value, T.value, D.value, uc.value
        self.n_nodes = (1 << (self.max_depth + 1)) - 1

    def export(self) -> dict:
        shp = (2, self.n_trees, self.n_nodes)
        base = np.zeros(2, np.float32)
        feat = np.zeros(shp, np.int32); bin_ = np.zeros(shp, np.int32)
        thr = np.zeros(shp, np.float32); val = np.zeros(shp, np.float32)
        _check(lib().llmpilot_model_export(self._h, *(a.ctypes.data_as(C.c_void_p) for a in (base, feat, bin_, thr, val))))
        return dict(base=base, feat=feat, bin=bin_, thr=thr, val=val)

    def gains(self) -> np.ndarray:
        """llmpilot_model_gains: [2][n_trees][nodes] split losses (fp64)."""
        out = np.zeros((2, self.n_trees, self.n_nodes), np.float64)
        _check(lib().llmpilot_model_gains(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def importance(self, normalize: bool = True) -> np.ndarray:
        """llmpilot_model_importance: MDI feature importance, 2 x F (fp64)."""
        out = np.zeros((2, self.F), np.float64)
        _check(lib().llmpilot_model_importance(self._h, 1 if normalize else 0, out.ctypes.data_as(C.c_void_p)))
        return out

    def train_pred(self, n_rows: int) -> np.ndarray:
        out = np.zeros((n_rows, 2), np.float32)
        _check(lib().llmpilot_model_train_pred(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def predict(self, ctx: Context, X, out=None):
        """out: None (returns a host numpy array) or a tensor/array of n x 2 float32."""
        n = int(X.shape[0])
        if X.ndim != 2 or int(X.shape[1]) != self.F:
            raise ValueError("X must be n x %d (the model's feature count), got %s" % (self.F, tuple(X.shape)))
        px, keep = _ptr(X, np.float32)
        if out is None:
            out = np.zeros((n, 2), np.float32)
        po = _out_ptr(out, (n, 2), "out")
        _check(lib().llmpilot_predict(ctx.handle, self._h, px, n, po))
        return out

    def save(self, path: str):
        """llmpilot_model_save: persist the model (binary, see include/llmpilot.h)."""
        _check(lib().llmpilot_model_save(self._h, os.fsencode(path)))

    @staticmethod
    def load(ctx: "Context", path: str) -> "Model":
        """llmpilot_model_load: a model saved by Model.save, its tables on ctx's device."""
        h = C.c_void_p()
        _check(lib().llmpilot_model_load(ctx.handle, os.fsencode(path), C.byref(h)))
        return Model(h)

    def free(self):
        if self._h:
            lib().llmpilot_model_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def fit(ctx: Context, X, y, hp: HParams, users_col: int, llm_id=None, prof_id=None, n_llm: int = 1, n_prof: int = 1,
        L1: float = 100.0, L2: float = 50.0, w=None, row_offset: int = 0, n_global: Optional[int] = None) -> Model:
    """llmpilot_fit on arrays (torch CUDA tensors for HBM-resident inputs, or host arrays)."""
    n = int(X.shape[0])
    if llm_id is None:
        llm_id = np.zeros(n, np.int32)
    if prof_id is None:
        prof_id = np.zeros(n, np.int32)
    ds, keep = _dataset(X, y, llm_id, prof_id, users_col, n_llm, n_prof, w, row_offset, n_global)
    h = C.c_void_p()
    _check(lib().llmpilot_fit(ctx.handle, C.byref(ds), C.byref(hp), L1, L2, C.byref(h)))
    return Model(h)


class WorkloadGenerator:
    """llmpilot_wg: request model of the workload generator (§III-B)."""

    def __init__(self, ctx: Context, traces):
        n, P = int(traces.shape[0]), int(traces.shape[1])
        pt, keep = _ptr(traces, np.float32)
        h = C.c_void_p()
        _check(lib().llmpilot_wg_build(ctx.handle, pt, n, P, C.byref(h)))
        self._h = h
        Pc, nr, m = C.c_int32(), C.c_int64(), C.c_int64()
        _check(lib().llmpilot_wg_info(h, C.byref(Pc), C.byref(nr), C.byref(m)))
        self.P, self.n_rows, self.n_nonempty = Pc.value, nr.value, m.value

    def export(self) -> dict:
        nb = np.zeros(self.P, np.int32)
        ce = np.zeros((self.P, 64), np.float32)
        keys = np.zeros(self.n_nonempty, np.uint64)
        counts = np.zeros(self.n_nonempty, np.int64)
        _check(lib().llmpilot_wg_export(self._h, *(a.ctypes.data_as(C.c_void_p) for a in (nb, ce, keys, counts))))
        return dict(nbins=nb, centres=ce, keys=keys, counts=counts)

    def sample(self, ctx: Context, n_samples: int, seed: int = 0, first: int = 0, out=None):
        """out: None (returns a host numpy array) or a tensor/array of n_samples x P float32."""
        if out is None:
            out = np.zeros((n_samples, self.P), np.float32)
        po, keep = _ptr(out, np.float32)
        _check(lib().llmpilot_wg_sample(ctx.handle, self._h, n_samples, seed, first, po))
        if keep is not None and keep is not out and isinstance(out, np.ndarray):
            out[...] = keep
        return out

    def free(self):
        if self._h:
            lib().llmpilot_wg_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


REC_DTYPE = np.dtype({"names": ["profile", "n_pods", "cost", "u_max"], "formats": [np.int32, np.int64, np.float64,
                                                                                    np.int32],
                      "offsets": [Rec.profile.offset, Rec.n_pods.offset, Rec.cost.offset, Rec.u_max.offset],
                      "itemsize": C.sizeof(Rec)})


def recommend(ctx: Context, model: Model, llm_feats, prof_feats, cost, user_levels, L1: float, L2: float, U: int,
              allowed=None, pred_out=None, as_array: bool = False):
    """Eq. (1)-(3) for every row of llm_feats.  Returns a list of (profile, n_pods, cost, u_max), or
    with as_array=True a numpy structured array (REC_DTYPE) over the library's output records."""
    n_llm, F_llm = int(llm_feats.shape[0]), int(llm_feats.shape[1])
    n_prof, F_prof = int(prof_feats.shape[0]), int(prof_feats.shape[1])
    pl, k1 = _ptr(llm_feats, np.float32)
    pp, k2 = _ptr(prof_feats, np.float32)
    cs = np.ascontiguousarray(cost, np.float64)
    lv = np.ascontiguousarray(user_levels, np.int32)
    al = None if allowed is None else np.ascontiguousarray(allowed, np.uint8)
    po = _out_ptr(pred_out, (n_llm * n_prof * len(lv), 2), "pred_out")
    out = (Rec * max(n_llm, 1))()
    _check(lib().llmpilot_recommend(ctx.handle, model._h, pl, n_llm, F_llm, pp, n_prof, F_prof,
                                    cs.ctypes.data_as(C.c_void_p), None if al is None else al.ctypes.data_as(C.c_void_p),
                                    lv.ctypes.data_as(C.c_void_p), len(lv), L1, L2, U, out, po))
    if as_array:
        return np.frombuffer(out, dtype=REC_DTYPE, count=n_llm).copy()
    return [(r.profile, r.n_pods, r.cost, r.u_max) for r in out[:n_llm]]


def cv(ctx: Context, X, y, llm_id, prof_id, users_col: int, n_llm: int, n_prof: int, grid: Sequence[HParams],
       L1: float, L2: float, U: int, cost):
    """Nested leave-one-LLM-out CV.  Returns (folds, S, O, SO)."""
    ds, keep = _dataset(X, y, llm_id, prof_id, users_col, n_llm, n_prof)
    g = (HParams * len(grid))(*grid)
    cs = np.ascontiguousarray(cost, np.float64)
    rep = C.POINTER(CvReport)()
    _check(lib().llmpilot_cv_leave_one_llm_out(ctx.handle, C.byref(ds), g, len(grid), L1, L2, U,
                                               cs.ctypes.data_as(C.c_void_p), C.byref(rep)))
    r = rep.contents
    folds = []
    for i in range(r.n_folds):
        f = r.folds[i]
        folds.append(dict(llm=f.llm, hp_index=f.hp_index,
                          rec=(f.rec.profile, f.rec.n_pods, f.rec.cost, f.rec.u_max),
                          truth=(f.truth.profile, f.truth.n_pods, f.truth.cost, f.truth.u_max),
                          success=f.success, overspend=f.overspend, truth_feasible=f.truth_feasible))
    S, O, SO = r.S, r.O, r.SO
    lib().llmpilot_cv_report_free(rep)
    return folds, S, O, SO


def debug_histogram(ctx: Context, codes, qg, qh, idx=None):
    """int64 histograms [32][256] of (qg, qh) over codes (CUDA tensors) — the fit's kernel."""
    n = int(codes.shape[0])
    Hg = np.zeros((32, 256), np.int64)
    Hh = np.zeros((32, 256), np.int64)
    m = n if idx is None else int(idx.shape[0])
    _check(lib().llmpilot_debug_histogram(ctx.handle, C.c_void_p(codes.data_ptr()), n,
                                          None if idx is None else C.c_void_p(idx.data_ptr()), m,
                                          C.c_void_p(qg.data_ptr()), C.c_void_p(qh.data_ptr()),
                                          Hg.ctypes.data_as(C.c_void_p), Hh.ctypes.data_as(C.c_void_p)))
    return Hg, Hh
