"""A/B timing of the recommend sweep (the bench's predict leg: 6,554 unseen LLMs x 8 profiles x 16
user levels through 2 x 500 depth-8 trees), each variant in its own process (switches are read once).

    python tools/ab_predict.py -- "" "LLMP_PRED_R=8"
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    sys.path.insert(0, os.environ.get("AB_ROOT", ROOT))   # AB_ROOT: another build (tools/build_variant.sh)
    import torch

    import paper_2410_02425_b200 as lp
    import synth
    d = synth.make_scaled(7812)   # ~1M training rows: the model shape is what matters
    ctx = lp.Context(0, torch.cuda.current_stream())
    m = lp.fit(ctx, d.X, d.y, lp.hparams(n_trees=500, max_depth=8), d.users_col, d.llm_id, d.prof_id, d.n_llm,
               d.n_prof, 100.0, 50.0)
    lf, pf, cost, levels = synth.sweep_tables(n_llm=6554, seed=1, profiles=synth.PROFILES_C3, params_lo=1.0,
                                              params_hi=16.0)
    s = torch.cuda.current_stream()
    lfd, pfd = torch.from_numpy(lf).cuda(), torch.from_numpy(pf).cuda()
    out = []
    for r in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        lp.recommend(ctx, m, lfd, pfd, cost, levels, 100.0, 50.0, 200)
        b.record(s)
        torch.cuda.synchronize()
        if r:
            out.append(a.elapsed_time(b))
    rows = lf.shape[0] * pf.shape[0] * len(levels)
    print(json.dumps({"ms": out, "rows": rows}))


def main():
    if "--child" in sys.argv:
        return child()
    variants = sys.argv[sys.argv.index("--") + 1:] if "--" in sys.argv else [""]
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
        if not line:
            print("variant %r failed:\n%s" % (v, p.stderr[-1500:]))
            continue
        j = json.loads(line[-1])
        ms = sorted(j["ms"])
        print("%-20s min %7.3f ms  median %7.3f ms  -> %.1f M rows/s" % (repr(v), ms[0], ms[len(ms) // 2],
                                                                      j["rows"] / ms[0] / 1e3))


if __name__ == "__main__":
    main()
