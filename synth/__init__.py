"""synth — seeded synthetic inputs shaped like LLM-Pilot's characterization dataset.

This module generates INPUTS only: it holds none of the method's arithmetic (no weights, cuts,
gradients, trees or recommendations).  It is the one module that both the oracle side (tests,
bench cpu_baseline) and the CUDA side (tests, bench) consume, as the task's rules allow.

Shapes follow SURVEY.md §8(d) and BASELINE.json configs:
  C1 tiny     10 LLMs x 4 GPU types (x1) x 8 user levels {1..128} = 320 rows, 12 features
  C2 paper    30 LLMs x 10 profiles x 16 levels (memory-masked, Table III), 32 features
  C3 scaled   78,125 LLMs x 8 profiles x 16 levels = 10,000,000 rows, 32 features ("S2" structured)
  C4 sharded  781,250 LLMs x 8 x 16 = 100,000,000 rows (row shards of contiguous LLM blocks)
  C5 sweep    6,554 unseen LLMs (seed 1) x the 10 C2 profiles x 16 levels = 1,048,640 rows
  S1 control  x ~ U[0,1)^32, u = x_31, smooth target + noise, explicit weights

Every random quantity is a counter-based hash of (seed, entity, field) — splitmix64 — so any
row or LLM can be regenerated independently on any shard.  Feature semantics follow P:L189;
the GPU catalog holds spec-sheet-like constants (generator constants, not paper data); the
latency model follows the paper's qualitative description P:L253-259 (TTFT linear in users,
ITL flat until memory saturates, queueing jump on weak GPUs).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

# ------------------------------------------------------------------------------------------
# counter-based RNG (generator-private; the method's own RNG lives separately in each side)
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _sm64(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & _M64
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
    return z ^ (z >> np.uint64(31))


def _hash(seed: int, entity, field: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        e = np.asarray(entity, dtype=np.uint64)
        h = _sm64(np.full(e.shape, np.uint64(seed), np.uint64) ^ np.uint64(0x5157A11D))
        h = _sm64(h ^ e)
        return _sm64(h ^ np.uint64(field))


def u01(seed: int, entity, field: int) -> np.ndarray:
    """uniform [0,1) float64 from 53 hash bits"""
    return (_hash(seed, entity, field) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, entity, field: int) -> np.ndarray:
    """standard normal via Box-Muller on two counter streams"""
    a = u01(seed, entity, field)
    b = u01(seed, entity, field + 7919)
    return np.sqrt(-2.0 * np.log1p(-a)) * np.cos(2.0 * np.pi * b)


# ------------------------------------------------------------------------------------------
# GPU catalog (spec-sheet-like generator constants; P:L189 lists the feature kinds)
GPU_FIELDS = ("mem_gb", "bw_gbs", "arch", "tensor_cores", "rt_cores", "cuda_cores", "tmus", "rops", "sms",
              "fp16_tf", "bf16_tf", "fp32_tf", "fp64_tf", "int8_tops", "cc", "pcie_gen", "sxm", "nvlink")
GPU_CATALOG = {
    #        mem  bw    arch tc   rt  cuda   tmu  rop sm   fp16  bf16  fp32  fp64  int8  cc   pcie sxm nvl
    "H100": (80, 3350, 3, 528, 0, 16896, 528, 24, 132, 989., 989., 67.0, 34.0, 1979., 9.0, 5, 1, 1),
    "A100": (40, 1555, 2, 432, 0, 6912, 432, 160, 108, 312., 312., 19.5, 9.7, 624., 8.0, 4, 1, 1),
    "A10": (24, 600, 2, 288, 72, 9216, 288, 96, 72, 125., 125., 31.2, 0.98, 250., 8.6, 4, 0, 0),
    "T4": (16, 320, 1, 320, 40, 2560, 160, 64, 40, 65., 0., 8.1, 0.25, 130., 7.5, 3, 0, 0),
    "V100": (16, 900, 0, 640, 0, 5120, 320, 128, 80, 125., 0., 15.7, 7.8, 62., 7.0, 3, 1, 1),
}
# synthetic on-demand price per GPU-hour (the paper uses AWS tables, values not printed)
GPU_PRICE = {"H100": 12.29, "A100": 4.10, "A10": 1.21, "T4": 0.53, "V100": 3.06}

PROFILES_C1 = [("H100", 1), ("A100", 1), ("A10", 1), ("T4", 1)]
PROFILES_C2 = [("H100", 1), ("H100", 2), ("H100", 4), ("A100", 1), ("A100", 2), ("A100", 4), ("A10", 1),
               ("A10", 2), ("T4", 1), ("T4", 4)]
PROFILES_C3 = [("H100", 1), ("H100", 2), ("H100", 4), ("A100", 1), ("A100", 2), ("A100", 4), ("A10", 2),
               ("T4", 4)]
LEVELS_8 = [1, 2, 4, 8, 16, 32, 64, 128]
LEVELS_16 = [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256]

# LLM features, P:L189 (11): type, enc-dec, params, layers, positions, heads, flash, vocab,
# rel-attn max distance, rel-attn buckets, dtype.
LLM_FIELDS = ("type", "encdec", "params_b", "layers", "positions", "heads", "flash", "vocab", "rel_dist",
              "rel_buckets", "dtype")
LLM_FIELDS_C1 = ("type", "encdec", "params_b", "layers", "heads", "vocab")
GPU_FIELDS_C1 = ("n_gpus", "mem_gb", "bw_gbs", "fp16_tf", "sms")
# profile features: 20 = n_gpus + mem_total + the 18 catalog fields
PROFILE_FIELDS = ("n_gpus", "mem_total_gb") + GPU_FIELDS
_ENCDEC_TYPES = (0, 7, 5)   # t5, ul2, mt0 are encoder-decoder families
_VOCABS = np.array([32000, 32128, 50257, 250112], np.float64)
_POSITIONS = np.array([512, 1024, 2048, 4096, 8192], np.float64)


def llm_table(seed: int, ids: np.ndarray, params_lo: float, params_hi: float) -> dict:
    """Per-LLM features from counter hashes of (seed, llm id)."""
    ids = np.asarray(ids, np.int64)
    typ = np.floor(u01(seed, ids, 1) * 8).astype(np.int64)
    encdec = np.isin(typ, _ENCDEC_TYPES).astype(np.float64)
    lp = np.log(params_lo) + u01(seed, ids, 2) * (np.log(params_hi) - np.log(params_lo))
    params = np.exp(lp).astype(np.float32).astype(np.float64)     # continuous: fills all bins
    layers = np.round(20.0 * (params / 7.0) ** 0.33 + 4.0 * u01(seed, ids, 3))
    heads = np.round(layers * (0.8 + 0.4 * u01(seed, ids, 4)))
    positions = _POSITIONS[np.floor(u01(seed, ids, 5) * 5).astype(np.int64)]
    flash = np.where(encdec > 0, 0.0, (u01(seed, ids, 6) < 0.8).astype(np.float64))
    vocab = _VOCABS[np.floor(u01(seed, ids, 7) * 4).astype(np.int64)]
    rel_dist = np.where(encdec > 0, 128.0, 0.0)
    rel_buckets = np.where(encdec > 0, 32.0, 0.0)
    dtype = np.floor(u01(seed, ids, 8) * 2.2)                     # 0 fp16, 1 bf16, 2 fp32 (rare)
    return dict(type=typ.astype(np.float64), encdec=encdec, params_b=params, layers=layers, positions=positions,
                heads=heads, flash=flash, vocab=vocab, rel_dist=rel_dist, rel_buckets=rel_buckets, dtype=dtype)


def profile_table(profiles) -> dict:
    cols = {k: [] for k in PROFILE_FIELDS}
    for name, cnt in profiles:
        spec = dict(zip(GPU_FIELDS, GPU_CATALOG[name]))
        cols["n_gpus"].append(cnt)
        cols["mem_total_gb"].append(spec["mem_gb"] * cnt)
        for k in GPU_FIELDS:
            cols[k].append(spec[k])
    return {k: np.asarray(v, np.float64) for k, v in cols.items()}


def profile_cost(profiles) -> np.ndarray:
    return np.asarray([GPU_PRICE[nm] * cnt for nm, cnt in profiles], np.float64)


def latency_model(seed: int, llm: dict, prof: dict, li: np.ndarray, pi: np.ndarray, u: np.ndarray,
                  row_key: np.ndarray):
    """Truth latencies (nTTFT, ITL) in ms, shaped after P:L253-259.  Returns (y1, y2, feasible)."""
    params = llm["params_b"][li]
    n_gpu = prof["n_gpus"][pi]
    mem_total = prof["mem_total_gb"][pi]
    bw = prof["bw_gbs"][pi]
    tf = prof["fp16_tf"][pi]
    weights_gb = 2.0 * params                                    # fp16 serving
    kv_per_user = 0.04 * params * (1.0 + llm["encdec"][li])
    free_gb = 0.9 * mem_total - weights_gb
    feasible = free_gb >= kv_per_user                            # Table III "x" cells
    cap = np.maximum(free_gb / kv_per_user, 0.5)                 # users before memory saturation
    tp_eff = 1.0 + 0.15 * (n_gpu - 1)                            # tensor-parallel overhead
    # decode: memory-bandwidth bound, flat until saturation, then rising fast
    itl = 1000.0 * weights_gb / (bw * n_gpu) * tp_eff / 0.55 + 4.0
    itl = itl * (1.0 + 0.004 * u) * np.where(u > cap, 1.0 + 1.5 * (u - cap) / cap, 1.0)
    # prefill: compute bound, linear in users, queueing jump beyond saturation
    ttft0 = 120.0 * 2.0 * params * 1e9 / (tf * 1e12 * n_gpu * 0.4) * 1e3 * tp_eff
    nttft = ttft0 * (1.0 + u / 6.0) * np.where(u > cap, 2.0 + (u - cap) / cap, 1.0)
    noise1 = np.exp(0.05 * normal(seed, row_key, 101))
    noise2 = np.exp(0.05 * normal(seed, row_key, 102))
    return nttft * noise1, itl * noise2, feasible


@dataclasses.dataclass
class Dataset:
    X: np.ndarray            # n x F float32, row = [llm feats | profile feats | u]
    y: np.ndarray            # n x 2 float32 (nTTFT, ITL) in ms
    llm_id: np.ndarray       # int32
    prof_id: np.ndarray      # int32
    users_col: int
    n_llm: int
    n_prof: int
    f_llm: int
    f_prof: int
    profiles: list
    cost: np.ndarray         # per profile, float64
    user_levels: np.ndarray  # int32
    w: Optional[np.ndarray] = None   # explicit weights (S1 control only)
    name: str = ""

    @property
    def n(self):
        return self.X.shape[0]

    @property
    def F(self):
        return self.X.shape[1]


def _assemble(seed, llm_ids, profiles, levels, params_lo, params_hi, llm_fields, prof_fields, mask_infeasible,
              local_ids=True):
    llm = llm_table(seed, llm_ids, params_lo, params_hi)
    prof = profile_table(profiles)
    nL, nP, nU = len(llm_ids), len(profiles), len(levels)
    li = np.repeat(np.arange(nL), nP * nU)
    pi = np.tile(np.repeat(np.arange(nP), nU), nL)
    u = np.tile(np.asarray(levels, np.float64), nL * nP)
    gid = np.asarray(llm_ids, np.int64)[li]
    row_key = (gid * 1000 + pi) * 1000 + np.searchsorted(levels, u)
    y1, y2, feas = latency_model(seed, llm, prof, li, pi, u, row_key)
    # true latencies are non-decreasing in users: cumulative max within each group
    y1 = np.maximum.accumulate(y1.reshape(-1, nU), axis=1).reshape(-1)
    y2 = np.maximum.accumulate(y2.reshape(-1, nU), axis=1).reshape(-1)
    cols = [llm[k][li] for k in llm_fields] + [prof[k][pi] for k in prof_fields] + [u]
    X = np.stack(cols, axis=1).astype(np.float32)
    y = np.stack([y1, y2], axis=1).astype(np.float32)
    keep = feas if mask_infeasible else np.ones_like(feas)
    ids = li if local_ids else gid
    return (X[keep], y[keep], ids[keep].astype(np.int32), pi[keep].astype(np.int32), len(llm_fields),
            len(prof_fields))


def make(config: str, seed: int = 0, shard: int = 0, n_shards: int = 1) -> Dataset:
    """Build one of the named configs (see module docstring)."""
    c = config.upper()
    if c == "C1":
        prof, levels = PROFILES_C1, LEVELS_8
        X, y, li, pi, fl, fp = _assemble(seed, np.arange(10), prof, levels, 1.0, 6.0, LLM_FIELDS_C1,
                                         GPU_FIELDS_C1, False)
        n_llm = 10
    elif c == "C2":
        prof, levels = PROFILES_C2, LEVELS_16
        X, y, li, pi, fl, fp = _assemble(seed, np.arange(30), prof, levels, 1.0, 40.0, LLM_FIELDS, PROFILE_FIELDS,
                                         True)
        n_llm = 30
    elif c in ("C3", "C4"):
        n_total = 78125 if c == "C3" else 781250
        lo = shard * n_total // n_shards
        hi = (shard + 1) * n_total // n_shards
        prof, levels = PROFILES_C3, LEVELS_16
        X, y, li, pi, fl, fp = _assemble(seed, np.arange(lo, hi), prof, levels, 1.0, 16.0, LLM_FIELDS,
                                         PROFILE_FIELDS, False, local_ids=False)
        n_llm = n_total
    elif c == "C5":
        prof, levels = PROFILES_C2, LEVELS_16
        X, y, li, pi, fl, fp = _assemble(1 if seed == 0 else seed, np.arange(6554), prof, levels, 1.0, 40.0,
                                         LLM_FIELDS, PROFILE_FIELDS, False)
        n_llm = 6554
    else:
        raise ValueError("unknown config " + config)
    return Dataset(X=X, y=y, llm_id=li, prof_id=pi, users_col=X.shape[1] - 1, n_llm=n_llm, n_prof=len(prof),
                   f_llm=fl, f_prof=fp, profiles=list(prof), cost=profile_cost(prof),
                   user_levels=np.asarray(levels, np.int32), name=c)


def make_scaled(n_llm_total: int, shard: int = 0, n_shards: int = 1, seed: int = 0) -> Dataset:
    """C3/C4 family: n_llm_total LLMs x the 8 C3 profiles x 16 levels, rows in (LLM, profile, u)
    order, contiguous LLM-block shards (shard boundaries are multiples of 128 rows, so every
    Eq. (4) group stays on one rank).  C3 = make_scaled(78125); C4 = make_scaled(781250, r, p)."""
    lo = shard * n_llm_total // n_shards
    hi = (shard + 1) * n_llm_total // n_shards
    X, y, li, pi, fl, fp = _assemble(seed, np.arange(lo, hi), PROFILES_C3, LEVELS_16, 1.0, 16.0, LLM_FIELDS,
                                     PROFILE_FIELDS, False, local_ids=False)
    ds = Dataset(X=X, y=y, llm_id=li, prof_id=pi, users_col=X.shape[1] - 1, n_llm=n_llm_total,
                 n_prof=len(PROFILES_C3), f_llm=fl, f_prof=fp, profiles=list(PROFILES_C3),
                 cost=profile_cost(PROFILES_C3), user_levels=np.asarray(LEVELS_16, np.int32), name="scaled")
    ds.row_offset = lo * len(PROFILES_C3) * len(LEVELS_16)
    ds.n_global = n_llm_total * len(PROFILES_C3) * len(LEVELS_16)
    return ds


def make_s1(n: int, seed: int = 0, F: int = 32, row_offset: int = 0) -> Dataset:
    """S1 control (best case for atomics): uniform random features, SURVEY §8(d)."""
    rows = np.arange(row_offset, row_offset + n, dtype=np.int64)
    X = np.stack([u01(seed, rows, 200 + j) for j in range(F)], axis=1).astype(np.float32)
    u = X[:, F - 1].astype(np.float64)
    x0 = X[:, 0].astype(np.float64)
    x1 = X[:, 1].astype(np.float64)
    y1 = 10.0 * (1.0 + u) * (1.0 + 0.5 * np.sin(2 * np.pi * x0) * x1) + 0.1 * normal(seed, rows, 301)
    y2 = 5.0 + 3.0 * X[:, 2] + 2.0 * u + 0.1 * normal(seed, rows, 302)
    w = (1.0 - u01(seed, rows, 303)).astype(np.float32)          # (0, 1]
    y = np.stack([y1, y2], axis=1).astype(np.float32)
    return Dataset(X=X, y=y, llm_id=np.zeros(n, np.int32), prof_id=np.zeros(n, np.int32), users_col=F - 1,
                   n_llm=1, n_prof=1, f_llm=0, f_prof=F - 1, profiles=[], cost=np.ones(1), user_levels=np.arange(1),
                   w=w, name="S1")


def sweep_tables(n_llm: int = 6554, seed: int = 1, profiles=PROFILES_C2, levels=LEVELS_16, params_lo=1.0,
                 params_hi=40.0, first_id: int = 0):
    """C5 recommendation sweep inputs: unseen-LLM feature table, profile feature table, costs, levels.
    Rows [llm feats | profile feats | u] are assembled by the recommend call itself."""
    ids = np.arange(first_id, first_id + n_llm)
    llm = llm_table(seed, ids, params_lo, params_hi)
    prof = profile_table(profiles)
    lf = np.stack([llm[k] for k in LLM_FIELDS], axis=1).astype(np.float32)
    pf = np.stack([prof[k] for k in PROFILE_FIELDS], axis=1).astype(np.float32)
    return lf, pf, profile_cost(profiles), np.asarray(levels, np.int32)


# ------------------------------------------------------------------------------------------
# Synthetic inference-request traces for the workload generator (§III-A/B, Table II
# 17.3M requests; the parameters that matter are the numbers of input and output
# tokens, the batch size and the token-sampling parameters, strongly correlated).
TRACE_PARAMS = ("input_tokens", "output_tokens", "batch_size", "decoding", "temperature", "top_p", "top_k",
                "max_new_tokens")
TRACE_ROWS_PAPER = 17_300_000


def make_traces(n: int, seed: int = 0, first: int = 0) -> np.ndarray:
    """n x 8 float32 requests (rows first .. first + n - 1 of `seed`, so shards regenerate exactly):
    lognormal input tokens; output tokens correlated with the input; batch size growing with the
    input length; greedy (0) or sampling (1) decoding; sampling parameters only when sampling
    (temperature on a 0.05 grid, top_p, top_k from small menus); max_new_tokens the next power of
    two above the output length.  Integer-valued parameters are exact in float32."""
    r = np.arange(first, first + n, dtype=np.uint64)
    z1, z2 = normal(seed, r, 901), normal(seed, r, 902)
    inp = np.clip(np.rint(np.exp(5.5 + 1.1 * z1)), 1, 8192)
    out = np.clip(np.rint(np.exp(3.8 + 0.35 * np.log(inp) * 0.5 + 0.9 * (0.6 * z1 + 0.8 * z2))), 1, 4096)
    bs = np.clip(np.floor(1 + 16 * u01(seed, r, 903) * (1 + np.log2(inp) / 13)), 1, 32)
    samp = (u01(seed, r, 904) < 0.45).astype(np.float64)
    temp = np.where(samp > 0, np.rint((0.1 + 1.4 * u01(seed, r, 905) ** 2) * 20) / 20, 0.0)
    top_p = np.where(samp > 0, np.array([0.8, 0.9, 0.95, 1.0])[(u01(seed, r, 906) * 4).astype(np.int64)], 1.0)
    top_k = np.where(samp > 0, np.array([0.0, 10.0, 50.0, 100.0])[(u01(seed, r, 907) * 4).astype(np.int64)], 0.0)
    mnt = np.minimum(2.0 ** np.ceil(np.log2(out + 1)), 4096)
    return np.stack([inp, out, bs, samp, temp, top_p, top_k, mnt], axis=1).astype(np.float32)


def trace_latency(T: np.ndarray, seed: int = 0, first: int = 0) -> np.ndarray:
    """End-to-end latency (s) of each trace request, for the RF + MDI study of P:L120 (a regressor
    predicting the latency of individual requests from their parameters): prefill proportional to
    the input tokens, decode proportional to the output tokens times a per-token time that grows with
    the batch size and with sampling, lognormal noise (sigma 0.1).  The ordering the paper reports —
    output tokens, then input tokens, then batch size and the sampling parameters — follows from the
    magnitudes.  n x 2 float32 (latency, per-output-token latency)."""
    n = T.shape[0]
    r = np.arange(first, first + n, dtype=np.uint64)
    inp, out, bs, samp, temp = (T[:, k].astype(np.float64) for k in range(5))
    tpot = 0.012 * (1.0 + 0.04 * bs) * (1.0 + 0.15 * samp + 0.05 * temp)
    lat = (0.05 + 0.0008 * inp + out * tpot) * np.exp(0.1 * normal(seed, r, 910))
    return np.stack([lat, lat / np.maximum(out, 1.0)], axis=1).astype(np.float32)
