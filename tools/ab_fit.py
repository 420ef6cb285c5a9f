"""A/B timing of the production fit path (CUDA-graph replay, no instrumentation) on the bench
workload: each variant runs in its own process (kernel-variant switches are read once per
process from the environment), variants interleaved, several rounds.

    python tools/ab_fit.py --trees 100 --rounds 3 -- "" "LLMP_NOFUSE=1"
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(trees, reps, llms):
    # AB_ROOT=<dir>: load the package (and its built library) from another tree, e.g. a copy of
    # the previous build, so two builds can be compared on the same box
    sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))
    import torch

    import paper_2410_02425_b200 as lp
    import synth
    d = synth.make_scaled(llms)
    dev = torch.device("cuda", 0)
    X, y = torch.from_numpy(d.X).to(dev), torch.from_numpy(d.y).to(dev)
    li, pi = torch.from_numpy(d.llm_id).to(dev), torch.from_numpy(d.prof_id).to(dev)
    s = torch.cuda.current_stream()
    ctx = lp.Context(0, s)
    hp = lp.hparams(n_trees=trees, max_depth=8)
    out = []
    for r in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        m = lp.fit(ctx, X, y, hp, d.users_col, li, pi, d.n_llm, d.n_prof, 100.0, 50.0)
        b.record(s)
        torch.cuda.synchronize()
        m.free()
        if r:
            out.append(a.elapsed_time(b))
    ctx.reset_stats()
    ctx.set_timing(1)
    m = lp.fit(ctx, X, y, hp, d.users_col, li, pi, d.n_llm, d.n_prof, 100.0, 50.0)
    st = ctx.stats()["classes"]
    # digest of the model (variants must agree bit for bit)
    import hashlib
    import numpy as np
    e = m.export()
    h = hashlib.sha1()
    for k in ("feat", "val", "thr", "base"):
        h.update(np.ascontiguousarray(np.asarray(e[k])).tobytes())
    m.free()
    print(json.dumps({"ms": out, "digest": h.hexdigest()[:12], "rows_hist_root": st.get("hist_root", {}).get("rows", 0),
                      "rows_hist_level": st.get("hist_level", {}).get("rows", 0)}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trees", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--llms", type=int, default=78125)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("variants", nargs="*", default=[""])
    a = ap.parse_args()
    if a.child:
        return child(a.trees, a.reps, a.llms)
    res = {v: [] for v in a.variants}
    extra = {}
    for _ in range(a.rounds):
        for v in a.variants:
            env = dict(os.environ)
            for kv in v.split():
                k, val = kv.split("=", 1)
                env[k] = val
            p = subprocess.run([sys.executable, __file__, "--child", "--trees", str(a.trees), "--reps", str(a.reps),
                                "--llms", str(a.llms)], env=env, capture_output=True, text=True)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print("variant %r failed:\n%s" % (v, p.stderr[-2000:]))
                continue
            j = json.loads(line[-1])
            res[v] += j["ms"]
            extra[v] = {k: j[k] for k in j if k != "ms"}
    for v, ms in res.items():
        if ms:
            ms = sorted(ms)
            print("%-28s min %8.2f  median %8.2f ms per fit (%d trees)  %s  all %s" % (
                repr(v), ms[0], ms[len(ms) // 2], a.trees, extra.get(v), " ".join("%.1f" % x for x in res[v])))


if __name__ == "__main__":
    main()
