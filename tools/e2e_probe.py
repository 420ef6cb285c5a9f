"""Where does the host-input (e2e) fit spend its time?  Times, on the bench workload: a plain torch
pinned->device copy of the inputs, fit with device inputs, fit with pinned host inputs, and fit
with pinned host inputs under instrumentation (per-kernel-class times).

    python tools/e2e_probe.py [--trees 100]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_02425_b200 as lp  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--trees", type=int, default=100)
a = ap.parse_args()
d = synth.make_scaled(78125)
s = torch.cuda.current_stream()
ctx = lp.Context(0, s)
hp = lp.hparams(n_trees=a.trees, max_depth=8)
pin = {k: torch.from_numpy(getattr(d, k)).pin_memory() for k in ("X", "y", "llm_id", "prof_id")}
dev = {k: v.cuda() for k, v in pin.items()}
torch.cuda.synchronize()


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(1000 * (time.perf_counter() - t0))
    return min(out)


res = {}
res["torch_copy_ms"] = timed(lambda: [v.cuda(non_blocking=True) for v in pin.values()])


def fit(src):
    m = lp.fit(ctx, src["X"], src["y"], hp, d.users_col, src["llm_id"], src["prof_id"], d.n_llm, d.n_prof, 100.0, 50.0)
    m.free()


fit(dev)
res["fit_device_ms"] = timed(lambda: fit(dev))
res["fit_pinned_host_ms"] = timed(lambda: fit(pin))
ctx.reset_stats()
ctx.set_timing(1)
fit(pin)
st = ctx.stats()["classes"]
ctx.set_timing(0)
res["instrumented_pinned"] = {k: round(v["ms"], 2) for k, v in st.items()}
ctx.reset_stats()
ctx.set_timing(1)
fit(dev)
st = ctx.stats()["classes"]
ctx.set_timing(0)
res["instrumented_device"] = {k: round(v["ms"], 2) for k, v in st.items()}
print(json.dumps(res, indent=1))

# after instrumented fits: do production fits slow down?
res2 = {"fit_device_after_instrumented_ms": timed(lambda: fit(dev)),
        "fit_pinned_after_instrumented_ms": timed(lambda: fit(pin))}
ctx.reset_stats()
ctx.set_timing(8)
fit(dev)
ctx.set_timing(0)
res2["fit_device_after_timing8_ms"] = timed(lambda: fit(dev))
res2["fit_pinned_after_timing8_ms"] = timed(lambda: fit(pin))
print(json.dumps(res2, indent=1))
