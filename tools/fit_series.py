"""Consecutive production fits of the bench workload in one process, each timed with CUDA events,
with NVML SM-clock / throttle-reason / power samples (10 ms) during each fit (variance check).
    python tools/fit_series.py [--fits 10] [--trees 500] [--timing]   (--timing: per-class times)"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import torch

import paper_2410_02425_b200 as lp
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--fits", type=int, default=10)
ap.add_argument("--trees", type=int, default=500)
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        try:
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)))
        except pynvml.NVMLError:
            pass
        time.sleep(0.01)


d = synth.make_scaled(78125)
dev = torch.device("cuda", 0)
X, y = torch.from_numpy(d.X).to(dev), torch.from_numpy(d.y).to(dev)
li, pi = torch.from_numpy(d.llm_id).to(dev), torch.from_numpy(d.prof_id).to(dev)
s = torch.cuda.current_stream()
ctx = lp.Context(0, s)
hp = lp.hparams(n_trees=a.trees, max_depth=8)
th = threading.Thread(target=sampler, daemon=True)
th.start()
for r in range(a.fits):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ctx.reset_stats()
    if a.timing:
        ctx.set_timing(1)
    k0 = len(samples)
    e0.record(s)
    m = lp.fit(ctx, X, y, hp, d.users_col, li, pi, d.n_llm, d.n_prof, 100.0, 50.0)
    e1.record(s)
    torch.cuda.synchronize()
    ctx.set_timing(0)
    sm = samples[k0:]
    m.free()
    clk = sorted(x[0] for x in sm) or [0]
    reasons = 0
    for x in sm:
        reasons |= x[1]
    pw = max((x[2] for x in sm), default=0)
    extra = ""
    if a.timing:
        st = ctx.stats()["classes"]
        extra = " ".join("%s=%.0f" % (k, v["ms"]) for k, v in st.items() if v["ms"] > 5)
    print("fit %2d  gpu %8.1f ms  sm clk min %4d med %4d  mem %d  reasons 0x%x  power max %.0f W  %s" % (
        r, e0.elapsed_time(e1), clk[0], clk[len(clk) // 2], sm[0][3] if sm else 0, reasons, pw, extra), flush=True)
stop.set()
