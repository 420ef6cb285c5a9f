#!/usr/bin/env python
"""bench.py — LLM-Pilot GPU-recommendation hot path on B200 (arxiv 2410.02425).

Metric (BASELINE.json): GBDT train row-iters/s (+ predict rows/s), 1/2/4/8 B200, % of HBM peak.

One STEP = one pass of the whole hot path over the resident synthetic batch:
  llmpilot_fit      Eq. (4) weights, quantile cuts, bin codes, 2 targets x 500 trees x depth 8
                    (root histogram, partitions, smaller-child histograms, split scans, updates)
  llmpilot_recommend  assemble [unseen-LLM | profile | users] rows, predict both targets,
                    Eq. (1)-(3) cheapest-feasible argmin per LLM.
Workload: C3 shape per GPU — 10,000,000 rows = 78,125 LLMs x 8 GPU profiles x 16 user levels,
32 features, 256 bins — weak-scaled over N ranks (C4 family: N x 78,125 LLMs, contiguous row
shards, NCCL histogram all-reduce per level).  value = row-iters (2 targets x global rows x trees
x steps) / max-over-ranks device time of the K timed steps.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun each rank drives one GPU; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0's stdout carries exactly one JSON line: NCCL logs (including the "NCCL version" line it
# prints at the WARN level) go to stderr
os.environ.setdefault("NCCL_DEBUG", "WARN")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

import numpy as np  # noqa: E402

L1, L2, U = 100.0, 50.0, 200
LLMS_PER_GPU = 78125                  # C3: 78,125 x 8 x 16 = 10,000,000 rows per GPU
SWEEP_LLMS_PER_GPU = 6554             # C5-sized unseen-LLM batch per GPU
METRIC = "GBDT train row-iters/s & predict rows/s, 1/2/4/8 B200, % HBM peak"
UNIT = "row-iters/s"

# algorithmic bytes per unit: unit = one row processed by that kernel
BYTES_PER_UNIT = {
    "hist_root": 48.0,    # 32 B code row + y, w, p (12 B) read + 4 B packed gradient pair written
    "partition": 9.0,     # row index read + 1 B split-feature code + row index written (the tile
                          # design reads the row index twice: 13 B moved, 9 B algorithmic)
    "hist_level": 40.0,   # 32 B code row + 4 B packed pair (both gathered by row index) + 4 B row index
    "update": 34.0,       # fused update of tree t + root histograms of trees t+1, BOTH ensembles in one
                          # pass (k_hist2<UPDROOT, DUAL>), per row and ensemble: (32 B code row + w) / 2
                          # + y, p read (8 B) + p and the packed pair written (8 B); 52 B with LLMP_DUAL=0
    "codes": 192.0,       # 128 B f32 row read + 32 B row-major + 32 B column-major codes written
}



def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--trees", type=int, default=500)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--llms-per-gpu", type=int, default=LLMS_PER_GPU)
    ap.add_argument("--sweep-llms", type=int, default=SWEEP_LLMS_PER_GPU)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-wg", action="store_true", help="skip the workload-generator leg")
    ap.add_argument("--no-cv", action="store_true", help="skip the paper-shaped C2 cross-validation legs")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 recommendation-sweep leg")
    ap.add_argument("--no-rf", action="store_true", help="skip the random-forest trace-importance leg")
    ap.add_argument("--strong", action="store_true",
                    help="BASELINE configs[3]: 100M rows (781,250 LLMs) in total, row-sharded over the N ranks "
                         "(strong scaling) instead of 10M rows per GPU")
    ap.add_argument("--strong-llms", type=int, default=781250)
    ap.add_argument("--nccl1", action="store_true",
                    help="N = 1 through a one-rank NCCL communicator: the sharded fit path on one GPU")
    ap.add_argument("--grid-trees", type=int, default=1000, help="trees of the cv_c2_grid leg's points")
    ap.add_argument("--wg-rows", type=int, default=17_300_000, help="trace rows of the workload-generator leg")
    ap.add_argument("--wg-samples", type=int, default=4_000_000, help="requests drawn per sampling step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=2_000_000, help="oracle sample rows (cpu_baseline)")
    ap.add_argument("--ref-rows", type=int, default=1_000_000, help="oracle sample rows per reference step")
    return ap.parse_args()


def bench_wg(lp, ctx, stream, dev, args):
    """Workload-generator leg: build (quantile bins, bin centres, sparse joint histogram) on an
    HBM-resident trace and sampling, device-timed (CUDA events on the context stream, best of 3
    after a warm-up); the oracle is timed on a bounded sample for context (rank 0, 1 core)."""
    import torch

    import synth
    T = synth.make_traces(args.wg_rows, seed=0)
    Td = torch.from_numpy(T).to(dev)
    out = torch.empty((args.wg_samples, T.shape[1]), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def timed(fn):
        best = None
        for r in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = fn()
            b.record(stream)
            torch.cuda.synchronize()
            if r:
                best = a.elapsed_time(b) if best is None else min(best, a.elapsed_time(b))
            if r < 3 and isinstance(res, lp.WorkloadGenerator):
                res.free()
        return best, res

    build_ms, g = timed(lambda: lp.WorkloadGenerator(ctx, Td))
    samp_ms, _ = timed(lambda: g.sample(ctx, args.wg_samples, seed=1, out=out))
    res = {"trace_rows": args.wg_rows, "parameters": list(synth.TRACE_PARAMS), "nonempty_bins": g.n_nonempty,
           "build": {"value": args.wg_rows / (build_ms / 1000.0), "unit": "rows/s", "ms": build_ms},
           "sample": {"value": args.wg_samples / (samp_ms / 1000.0), "unit": "requests/s", "ms": samp_ms,
                      "requests": args.wg_samples},
           "paper_context": "1000 requests in 22 ms on an unstated CPU, 46.5K non-empty of 10.7B bins over 17.3M "
                            "real requests (P:L245)"}
    g.free()
    if not args.no_cpu_baseline:
        import oracle
        n_o = min(args.wg_rows, 1_000_000)
        t0 = time.perf_counter()
        om = oracle.wg_build(T[:n_o])
        t1 = time.perf_counter()
        oracle.wg_sample(om, 1000, seed=1)
        t2 = time.perf_counter()
        res["cpu_baseline"] = {"kind": "oracle", "cores": 1, "build": {"value": n_o / (t1 - t0), "unit": "rows/s"},
                               "sample": {"value": 1000 / (t2 - t1), "unit": "requests/s"},
                               "sample_note": "build on the first %d trace rows, 1000 requests (linear CDF walk)" % n_o}
    return res


def bench_cv_c2(lp, ctx, args):
    """BASELINE.json configs[1]: C2 (30 LLMs x 10 profiles x 16 user levels, memory-masked), 1000
    trees depth 6, full nested leave-one-LLM-out CV (grid of one) + cheapest-feasible recommendation
    per held-out LLM; wall time of one llmpilot_cv_leave_one_llm_out call (it synchronises) after a
    warm-up call.  The oracle is timed on one fold's fit for context (rank 0, 1 core)."""
    import synth
    d = synth.make("C2")
    grid = [lp.hparams(n_trees=1000, max_depth=6)]
    lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, grid, L1, L2, U, d.cost)
    t0 = time.perf_counter()
    folds, S, O, SO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, grid, L1, L2, U,
                            d.cost)
    dt = time.perf_counter() - t0
    fit_rows = sum(int((d.llm_id != f["llm"]).sum()) for f in folds)   # each fold refits on the other LLMs' rows
    res = {"workload": "C2 paper-shaped: %d rows (%d LLMs x %d profiles x 16 user levels, memory-masked), 2 targets "
                       "x 1000 trees, depth 6, %d-fold leave-one-LLM-out CV + recommendation" % (d.n, d.n_llm, d.n_prof,
                                                                                              len(folds)),
           "seconds": dt, "folds": len(folds), "fits_per_s": len(folds) / dt,
           "row_iters_per_s": 2.0 * 1000 * fit_rows / dt, "S": S, "O": O, "SO": SO}
    if not args.no_cpu_baseline:
        import oracle
        keep = d.llm_id != folds[0]["llm"]
        t0 = time.perf_counter()
        oracle.fit(d.X[keep], d.y[keep], oracle.hparams(n_trees=1000, max_depth=6), d.users_col, d.llm_id[keep],
                   d.prof_id[keep], d.n_llm, d.n_prof, L1, L2)
        t1 = time.perf_counter()
        res["cpu_baseline"] = {"kind": "oracle", "cores": 1, "seconds_one_fold_fit": t1 - t0,
                               "row_iters_per_s": 2.0 * 1000 * int(keep.sum()) / (t1 - t0),
                               "sample": "the oracle's fit of the first fold (1000 trees x 2 targets)"}
    return res


def bench_cv_c2_grid(lp, ctx, args):
    """Nested leave-one-LLM-out CV with an HP grid on C2 (trees, depth, learning rate,
    subsampling; 4 points): 30 x 29 x 4 inner fits (wMAPE per point) + 30 refits + recommendations.
    Every fit of a stage runs in one launch (one thread block per fit and ensemble, fit_small.cu)."""
    import synth
    d = synth.make("C2")
    T = args.grid_trees
    gk = [dict(n_trees=T, max_depth=6, eta=0.3), dict(n_trees=T, max_depth=4, eta=0.3),
          dict(n_trees=T, max_depth=6, eta=0.1), dict(n_trees=T, max_depth=6, eta=0.3, subsample=0.8)]
    grid = [lp.hparams(**k) for k in gk]
    t0 = time.perf_counter()
    folds, S, O, SO = lp.cv(ctx, d.X, d.y, d.llm_id, d.prof_id, d.users_col, d.n_llm, d.n_prof, grid, L1, L2, U,
                            d.cost)
    dt = time.perf_counter() - t0
    n_llm = len(folds)
    inner = n_llm * (n_llm - 1) * len(grid)
    fits = inner + n_llm
    rows = sum(int((d.llm_id != f["llm"]).sum()) for f in folds)   # outer fits' rows
    inner_rows = sum(int(((d.llm_id != f["llm"]) & (d.llm_id != g["llm"])).sum()) for f in folds for g in folds
                     if g["llm"] != f["llm"]) * len(grid)
    return {"workload": "C2 nested leave-one-LLM-out CV, grid of %d (trees %d; depth 6/4; eta 0.3/0.1; subsample 1/0.8),"
                        " %d inner + %d outer fits x 2 targets" % (len(grid), T, inner, n_llm),
            "seconds": dt, "fits": fits, "fits_per_s": fits / dt,
            "row_iters_per_s": 2.0 * T * (rows + inner_rows) / dt,
            "hp_chosen": sorted({f["hp_index"] for f in folds}), "S": S, "O": O, "SO": SO}


def bench_c5(lp, ctx, stream, dev, args, rank, world):
    """BASELINE configs[4]: recommendation sweep of 6,554 unseen LLMs (seed 1) x the 10 C2 profiles x
    16 user levels = 1,048,640 candidate rows through the C2-shaped model (2 x 1000 trees, depth 6),
    Eq. (1)-(3) argmin per LLM; the LLMs are split over the ranks and the per-LLM results gathered.
    Device-timed (CUDA events), K steps after one warm-up."""
    import torch
    import torch.distributed as dist

    import synth
    d = synth.make("C2")
    m = lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=1000, max_depth=6), d.users_col, d.llm_id, d.prof_id, d.n_llm,
               d.n_prof, L1, L2)
    n_total = 6554
    lo, hi = rank * n_total // world, (rank + 1) * n_total // world
    lf, pf, cost, levels = synth.sweep_tables(n_llm=hi - lo, seed=1, profiles=synth.PROFILES_C2, first_id=lo)
    lfd, pfd = torch.from_numpy(lf).to(dev), torch.from_numpy(pf).to(dev)
    rows = (hi - lo) * pf.shape[0] * len(levels)
    gathered = torch.zeros((n_total, 4), dtype=torch.float64, device=dev)

    rec_ms = []

    def step(record=False):
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        recs = lp.recommend(ctx, m, lfd, pfd, cost, levels, L1, L2, U, as_array=True)
        if record:
            e1.record(stream)
            rec_ms.append((e0, e1))
        mine = torch.from_numpy(np.stack([recs["profile"].astype(np.float64), recs["n_pods"].astype(np.float64),
                                          recs["cost"], recs["u_max"].astype(np.float64)], axis=1)).to(dev)
        if world > 1:
            parts = [torch.zeros(((r + 1) * n_total // world - r * n_total // world, 4), dtype=torch.float64,
                                 device=dev) for r in range(world)]
            dist.all_gather(parts, mine)
            torch.cat(parts, out=gathered)
        else:
            gathered.copy_(mine)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        step(record=True)
    b.record(stream)
    torch.cuda.synchronize()
    call_ms = sum(x.elapsed_time(y) for x, y in rec_ms) / args.steps
    ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item() / args.steps
    m.free()
    total_rows = n_total * pf.shape[0] * len(levels)
    visits = total_rows * 2 * 1000 * 6
    return {"workload": "C5: %d unseen LLMs x %d profiles x %d user levels = %d rows, C2-shaped model (2 x 1000 trees,"
                        " depth 6), LLMs split over %d rank(s), per-LLM results all-gathered" %
                        (n_total, pf.shape[0], len(levels), total_rows, world),
            "value": total_rows / (ms / 1000.0), "unit": "rows/s", "ms_per_step": ms, "rows": total_rows,
            "rows_per_rank": rows, "row_node_visits_per_s": visits / (ms / 1000.0),
            "recommend_call_ms": call_ms,
            "row_node_visits_per_row": 2 * 1000 * 6,
            "note": "the predictor routes on bin codes through fixed-depth trees: SM-issue bound, not HBM "
                    "(DESIGN.md §6). With <= 64 user levels the grid predictor walks each tree once per "
                    "(LLM, profile) pair carrying the range of levels, so row_node_visits_per_s counts the "
                    "per-row definition's visits (2 x 1000 x 6 per row), not the walks executed"}


def bench_rf_traces(lp, ctx, stream, dev, args):
    """The paper's random-forest importance study (§III-A): an RF regressor predicting the
    latency of every request of a Table II-sized trace (17.3M requests x 8 parameters)
    from its parameters, then the MDI importance.  100 trees, depth 10, half the parameters per node,
    Poisson(1) bootstrap (DESIGN R33-R36); device-timed fit after one warm-up fit."""
    import torch

    import synth
    n = args.wg_rows
    T = synth.make_traces(n, seed=0)
    y = synth.trace_latency(T, seed=0)
    Td, yd = torch.from_numpy(T).to(dev), torch.from_numpy(y).to(dev)
    hp = lp.rf_hparams(n_trees=100, max_depth=10, max_features=0.5, seed=1)
    lp.fit(ctx, Td, yd, lp.rf_hparams(n_trees=2, max_depth=10, max_features=0.5, seed=1), T.shape[1] - 1).free()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    m = lp.fit(ctx, Td, yd, hp, T.shape[1] - 1)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    imp = m.importance()
    pred = m.predict(ctx, Td[: 1 << 20])
    yt = y[: 1 << 20, 0].astype(np.float64)
    r2 = 1.0 - float(((pred[:, 0] - yt) ** 2).sum() / ((yt - yt.mean()) ** 2).sum())
    m.free()
    order = [synth.TRACE_PARAMS[i] for i in np.argsort(-imp[0])]
    return {"workload": "RF regressor on %d synthetic trace requests x %d parameters, 2 targets (latency, latency "
                        "per output token) x 100 trees, depth 10, max_features 0.5, Poisson(1) bootstrap" %
                        (n, T.shape[1]),
            "value": 2.0 * 100 * n / (ms / 1000.0), "unit": "row-iters/s", "ms": ms,
            "r2_latency_train_first_1M": r2, "mdi_order_latency": order,
            "paper_context": "R^2 ~ 0.93 on the real traces; MDI: output tokens, then input tokens, batch size, "
                             "sampling parameters (P:L120)"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the profiled kernels (profiles/ncu_traffic.json, from ncu --set full)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


# ------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled every 100 ms by an in-process NVML thread.  NVML is
    initialised before the warm-up (no driver initialisation overlaps the timed region) and only
    the samples taken between begin() and end() — the timed region — are reported.  Falls back to
    an `nvidia-smi -lms` process started at open() when NVML is unavailable."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, cuda_index):
        self.cuda_index = cuda_index
        self.samples = []          # (monotonic time, sm MHz, max sm MHz, set of reasons)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.thread = self.proc = self.path = None

    def open(self):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(self.cuda_index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.cuda_index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.monotonic(), float(sm), float(mx),
                                             {k for k, b in bits.items() if r & b}))
                    except Exception:
                        pass
                    self._stop.wait(0.1)

            self.nvml = pynvml
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
            fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
            os.close(fd)
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.cuda_index), "--query-gpu=" + q,
                                              "--format=csv,noheader,nounits", "-lms", "200"],
                                             stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except OSError:
                self.proc = None
        return self

    def begin(self):
        self.t0 = time.monotonic()

    def end(self):
        self.t1 = time.monotonic()

    def window(self, t0, t1):
        """(median SM MHz, reasons, samples) of the NVML samples taken in [t0, t1]"""
        sel = [(a, r) for t, a, b, r in self.samples if t0 <= t <= t1]
        if not sel:
            return None
        return {"sm_mhz": statistics.median(a for a, r in sel), "reasons": sorted(set().union(*[r for a, r in sel])),
                "samples": len(sel)}

    def close(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm, mx, reasons = [], [], set()
        if self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=2)
            for t, a, b, r in self.samples:
                if self.t0 is not None and self.t0 <= t <= (self.t1 or t):
                    sm.append(a)
                    mx.append(b)
                    reasons |= r
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
            out["source"] = "nvml (in-process, 100 ms, timed region only)"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) < 9:
                        continue
                    try:
                        sm.append(float(parts[1]))
                        mx.append(float(parts[2]))
                    except ValueError:
                        continue
                    for nm, v in zip(self.REASONS, parts[5:9]):
                        if v.lower() == "active":
                            reasons.add(nm)
            os.unlink(self.path)
            out["source"] = "nvidia-smi -lms 200 (warm-up + timed region)"
        if sm:
            out.update({"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                        "samples": len(sm)})
        return out


# ---------------------------------------------------------------------------------- reference
def arm_config(args, world):
    """The workload both arms report: BASELINE.json configs[2] per GPU, weak-scaled (default), or
    configs[3] (--strong: 100M rows in total, row-sharded over the N ranks)."""
    sweep_rows = args.sweep_llms * 8 * 16
    if args.strong:
        rows_g = args.strong_llms * 8 * 16
        rows = rows_g // world
        desc = ("C4 row-sharded fit: %d rows in total = %d LLMs x 8 profiles x 16 user levels over %d GPU(s), 32 "
                "features, 256 bins, 2 targets x %d trees, depth %d; recommend sweep %d unseen LLMs/GPU"
                % (rows_g, args.strong_llms, world, args.trees, args.depth, args.sweep_llms))
    else:
        rows = args.llms_per_gpu * 8 * 16
        rows_g = rows * world
        desc = ("C3 per GPU (C4 family when N > 1): %d rows/GPU = %d LLMs x 8 profiles x 16 user levels, "
                "32 features, 256 bins, 2 targets x %d trees, depth %d; recommend sweep %d unseen LLMs/GPU"
                % (rows, args.llms_per_gpu, args.trees, args.depth, args.sweep_llms))
    return {"workload": desc, "rows_global": rows_g, "rows_per_gpu": rows, "features": 32, "bins": 256,
            "trees": args.trees, "depth": args.depth, "targets": 2, "sweep_rows_per_gpu": sweep_rows,
            "global_batch": rows_g, "parallelism": "row-sharded dp%d, NCCL int64 histogram all-reduce" % world,
            "l2": "inputs larger than L2 (codes %d MB + state per GPU), no flush" % (rows * 32 // 2 ** 20)}


def run_reference(args, rank, world):
    """The reference arm for this tier is the CPU oracle, as it stands, on a bounded sample."""
    if rank != 0:
        return 0
    import oracle
    import synth
    n_llm = max(1, args.ref_rows // 128)
    d = synth.make_scaled(n_llm)
    hp = oracle.hparams(n_trees=args.trees, max_depth=args.depth)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.fit(d.X, d.y, hp, d.users_col, d.llm_id, d.prof_id, d.n_llm, d.n_prof, L1, L2, n_trees_limit=1)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    row_iters = 2.0 * d.n * 1 * len(times)
    value = row_iters / total
    sample = ("oracle fit of the first tree of each target (depth %d, 256 bins) on the first %d rows "
              "(%d LLMs x 8 profiles x 16 levels) of the C3 workload, incl. its binning" % (args.depth, d.n, n_llm))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/i64",
        "data": "synthetic (seeded, synth/)",
        "config": dict(arm_config(args, world), sample=sample),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _gen_chunk(a):
    import synth
    n_total, shard, n_shards = a
    c = synth.make_scaled(n_total, shard, n_shards)
    return c.X, c.y, c.llm_id, c.prof_id, c.row_offset, c.n_global


def device_shard(n_llm_total, rank, world, dev, chunks=16):
    """Rank `rank`'s contiguous LLM-block shard of make_scaled(n_llm_total) built straight into HBM,
    chunk by chunk (the concatenation of make_scaled(n, rank*c + j, world*c) over j is exactly
    make_scaled(n, rank, world)), generated by a process pool to bound host memory and time."""
    import concurrent.futures as cf
    import types

    import torch
    lo, hi = rank * n_llm_total // world, (rank + 1) * n_llm_total // world
    rows_per_llm = 8 * 16
    n = (hi - lo) * rows_per_llm
    X = torch.empty((n, 32), dtype=torch.float32, device=dev)
    y = torch.empty((n, 2), dtype=torch.float32, device=dev)
    li = torch.empty(n, dtype=torch.int32, device=dev)
    pi = torch.empty(n, dtype=torch.int32, device=dev)
    jobs = [(n_llm_total, rank * chunks + j, world * chunks) for j in range(chunks)]
    off = 0
    row_offset = None
    workers = max(1, min(8, (os.cpu_count() or 2) - 1))
    with cf.ProcessPoolExecutor(workers) as ex:
        for Xc, yc, lc, pc, ro, ng in ex.map(_gen_chunk, jobs):
            m = Xc.shape[0]
            X[off:off + m].copy_(torch.from_numpy(Xc))
            y[off:off + m].copy_(torch.from_numpy(yc))
            li[off:off + m].copy_(torch.from_numpy(lc))
            pi[off:off + m].copy_(torch.from_numpy(pc))
            if row_offset is None:
                row_offset = ro
            off += m
            n_global = ng
    assert off == n
    import synth
    meta = types.SimpleNamespace(n=n, users_col=31, n_llm=n_llm_total, n_prof=len(synth.PROFILES_C3),
                                 row_offset=row_offset, n_global=n_global, X=None, y=None, llm_id=None, prof_id=None)
    return meta, X, y, li, pi


# ---------------------------------------------------------------------------------------- ours
def main():
    args = parse()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2410_02425_b200 as lp
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(lp.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().numpy().tobytes())
    elif args.nccl1:
        uid = lp.nccl_unique_id()

    # ---- synthetic inputs (seeded), resident in HBM before the timed region
    n_llm_total = args.strong_llms if args.strong else args.llms_per_gpu * world
    if args.strong:
        args.no_e2e = True   # (a 13 GB pinned host copy per rank is not what configs[3] measures)
        d, Xd, yd, ld, pd = device_shard(n_llm_total, rank, world, dev)
    else:
        d = synth.make_scaled(n_llm_total, rank, world)
    lf, pf, cost, levels = synth.sweep_tables(n_llm=args.sweep_llms, seed=1, profiles=synth.PROFILES_C3,
                                              params_lo=1.0, params_hi=16.0, first_id=rank * args.sweep_llms)
    stream = torch.cuda.current_stream()
    if not args.strong:
        Xd = torch.from_numpy(d.X).to(dev)
        yd = torch.from_numpy(d.y).to(dev)
        ld = torch.from_numpy(d.llm_id).to(dev)
        pd = torch.from_numpy(d.prof_id).to(dev)
    lfd = torch.from_numpy(lf).to(dev)
    pfd = torch.from_numpy(pf).to(dev)
    torch.cuda.synchronize()
    ctx = lp.Context(local_rank, stream, uid, rank, world)
    hp = lp.hparams(n_trees=args.trees, max_depth=args.depth, max_bin=256)
    n_global = d.n_global
    sweep_rows = lf.shape[0] * pf.shape[0] * len(levels)

    ev = []
    host = {"fit": 0.0, "recommend": 0.0, "free": 0.0}   # host wall time per phase (diagnostics)

    def step(X, y, li, pi, lfx, pfx, record=None, hacc=None):
        if record is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e2 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        h0 = time.perf_counter()
        m = lp.fit(ctx, X, y, hp, d.users_col, li, pi, d.n_llm, d.n_prof, L1, L2, row_offset=d.row_offset,
                   n_global=n_global)
        h1 = time.perf_counter()
        if record is not None:
            e1.record(stream)
        recs = lp.recommend(ctx, m, lfx, pfx, cost, levels, L1, L2, U, as_array=True)   # one structured copy, not a Python list
        h2 = time.perf_counter()
        if record is not None:
            e2.record(stream)
            record.append((e0, e1, e2))
        m.free()
        if hacc is not None:
            hacc["fit"] += h1 - h0
            hacc["recommend"] += h2 - h1
            hacc["free"] += time.perf_counter() - h2
        return recs

    clocks = ClockSampler(local_rank).open()   # before the warm-up: no NVML init in the timed region
    for _ in range(args.warmup):
        step(Xd, yd, ld, pd, lfd, pfd)
    torch.cuda.synchronize()

    # ---- timed region: K steps, device-resident inputs, CUDA events on the context stream
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.set_timing(0)            # production mode: each tree replays from a CUDA graph
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clocks.begin()
    t_start.record(stream)
    for _ in range(args.steps):
        step(Xd, yd, ld, pd, lfd, pfd, record=ev, hacc=host)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks.end()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    stats = ctx.stats()
    fit_ms = sum(a.elapsed_time(b) for a, b, c in ev)
    pred_ms = sum(b.elapsed_time(c) for a, b, c in ev)
    agg = torch.tensor([elapsed_ms, fit_ms, pred_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(agg, op=dist.ReduceOp.MAX)
    elapsed_ms, fit_ms, pred_ms = agg.tolist()

    row_iters = 2.0 * n_global * args.trees * args.steps
    value = row_iters / (elapsed_ms / 1000.0)
    predict_rows = float(sweep_rows) * world * args.steps

    # ---- per-kernel durations: one more step, instrumented (plain launches, every 8th launch of
    # each kernel class bracketed by CUDA events on the context stream)
    ctx.reset_stats()
    ctx.set_timing(8)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step(Xd, yd, ld, pd, lfd, pfd)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_step_ms = p0.elapsed_time(p1)
    pstats = ctx.stats()
    ctx.set_timing(0)

    # ---- per-kernel roofline from the live event timings
    peak, peak_src = measured_peaks()
    traffic = ncu_traffic()
    kernels = {}
    for name, c in pstats["classes"].items():
        if c["ms"] <= 0:
            continue
        k = {"launches": c["launches"], "timed_launches": c["timed"], "ms_total": round(c["ms"], 3),
             "ms_avg": c["ms_avg"], "share_of_step": c["ms"] / prof_step_ms}
        if name in BYTES_PER_UNIT and c["rows"] > 0:
            nbytes = BYTES_PER_UNIT[name] * c["rows"]
            gbs = nbytes / (c["ms"] / 1000.0) / 1e9
            k.update({"units": c["rows"], "bytes_per_unit": nbytes / c["rows"], "achieved_gbs": gbs,
                      "frac_hbm": gbs / peak})
        kernels[name] = k
    dom = max((n for n in kernels if n in BYTES_PER_UNIT and "achieved_gbs" in kernels[n]),
              key=lambda n: kernels[n]["ms_total"], default=None)
    roofline = None
    if dom:
        kd = kernels[dom]
        tr = traffic.get(dom)
        roofline = {"kernel": dom, "bound": "hbm", "achieved": kd["achieved_gbs"], "peak": peak, "unit": "GB/s",
                    "frac": kd["achieved_gbs"] / peak, "peak_source": peak_src,
                    "bytes_per_unit": kd["bytes_per_unit"], "units_per_launch": kd["units"] / kd["launches"],
                    "traffic": ((tr["dram_bytes_per_unit"] * kd["units"] / kd["launches"]) if tr and
                                "dram_bytes_per_unit" in tr else tr.get("dram_bytes_per_launch") if tr else None),
                    "traffic_note": ((tr.get("note") + "; scaled to this run's units_per_launch")
                                     if tr and "dram_bytes_per_unit" in tr else tr.get("note") if tr
                                     else "no ncu capture committed")}

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(d.X).pin_memory()
        yh = torch.from_numpy(d.y).pin_memory()
        lh = torch.from_numpy(d.llm_id).pin_memory()
        ph = torch.from_numpy(d.prof_id).pin_memory()
        lfh = torch.from_numpy(lf).pin_memory()
        pfh = torch.from_numpy(pf).pin_memory()
        step(Xh, yh, lh, ph, lfh, pfh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        host_e2e = {"fit": 0.0, "recommend": 0.0, "free": 0.0}
        te0 = time.monotonic()
        e0.record(stream)
        for _ in range(args.steps):
            step(Xh, yh, lh, ph, lfh, pfh, hacc=host_e2e)
        e1.record(stream)
        torch.cuda.synchronize()
        te1 = time.monotonic()
        e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        nn = (1 << (args.depth + 1)) - 1
        h2d = d.X.nbytes + d.y.nbytes + d.llm_id.nbytes + d.prof_id.nbytes + lf.nbytes + pf.nbytes
        d2h = 2 * args.trees * nn * 16 + 8 + lf.shape[0] * 24
        e2e = {"value": row_iters / (e2e_ms.item() / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms.item() / args.steps,
               "host_ms_per_step": {k: 1000.0 * v / args.steps for k, v in host_e2e.items()},
               "clocks": clocks.window(te0, te1)}

    clk = clocks.close()   # SM clocks of the timed region (the e2e leg's are in e2e["clocks"])

    # ---- workload generator: build the request model from a
    # Table II-sized synthetic trace (17.3M requests) resident in HBM, then draw requests;
    # N = 1 only (it does not shard), outside the fit's timed region
    wg = None
    if rank == 0 and world == 1 and not args.no_wg:
        wg = bench_wg(lp, ctx, stream, dev, args)
    rf = None
    if rank == 0 and world == 1 and not args.no_rf:
        rf = bench_rf_traces(lp, ctx, stream, dev, args)
    # ---- the paper-shaped config (BASELINE.json configs[1]): full leave-one-LLM-out CV of C2
    cv_c2 = cv_grid = None
    if rank == 0 and world == 1 and not args.no_cv:
        cv_c2 = bench_cv_c2(lp, ctx, args)
        cv_grid = bench_cv_c2_grid(lp, ctx, args)
    # ---- BASELINE configs[4]: the C5 recommendation sweep, LLMs split over the ranks
    c5 = None
    if not args.no_c5:
        c5 = bench_c5(lp, ctx, stream, dev, args, rank, world)

    # ---- CPU baseline: the oracle as it stands, rank 0, N = 1, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        nl = max(1, args.cpu_rows // 128)
        ds = synth.make_scaled(nl)
        ohp = oracle.hparams(n_trees=args.trees, max_depth=args.depth)
        t0 = time.perf_counter()
        oracle.fit(ds.X, ds.y, ohp, ds.users_col, ds.llm_id, ds.prof_id, ds.n_llm, ds.n_prof, L1, L2,
                   n_trees_limit=1)
        dt = time.perf_counter() - t0
        cpu = {"value": 2.0 * ds.n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": "first tree of each target (depth %d) on the first %d rows of this workload, single-threaded "
                         "C oracle incl. its binning; %.1f s" % (args.depth, ds.n, dt)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "u8/i64",
            "data": "synthetic (seeded counter-based generator, synth/; shapes of the paper's dataset)",
            "config": arm_config(args, world),
            "predict": {"value": predict_rows / (pred_ms / 1000.0), "unit": "rows/s", "rows_per_step": sweep_rows * world,
                        "ms_per_step": pred_ms / args.steps},
            "fit": {"value": row_iters / (fit_ms / 1000.0), "unit": UNIT, "ms_per_step": fit_ms / args.steps},
            "host_ms_per_step": {k: 1000.0 * v / args.steps for k, v in host.items()},
            "roofline": roofline,
            "kernels": kernels,
            "kernels_note": "per-kernel durations from one extra instrumented step (plain launches, every 8th "
                            "launch of each class CUDA-event-timed on the context stream, %.1f ms); the timed "
                            "steps replay each tree from a CUDA graph" % prof_step_ms,
            "gpu_launches": stats["total_launches"],
            "gpu_launches_per_step": stats["total_launches"] / args.steps,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "workload_generator": wg,
            "rf_traces": rf,
            "cv_c2": cv_c2,
            "cv_c2_grid": cv_grid,
            "c5_sweep": c5,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
