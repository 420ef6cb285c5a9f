"""Group the SASS of one `ncu --page source --csv --print-source sass` dump by execution count:
each group is a straight-line region executed the same number of times (a loop body, a prologue),
with its share of all executed warp-instructions and of the stall samples.

    python tools/ncu_exec_groups.py SASS.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n_show = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
iex, iss, isrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
seen, data = set(), []
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[0] in seen:
        continue
    seen.add(r[0])
    data.append(r)


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


by = defaultdict(lambda: [0, 0.0, 0.0, []])
for r in data:
    e = f(r[iex])
    g = by[e]
    g[0] += 1
    g[1] += e
    g[2] += f(r[iss])
    g[3].append(r[isrc].strip())
tot = sum(v[1] for v in by.values())
tss = sum(v[2] for v in by.values()) or 1.0
print("warp-instructions executed %.0f, stall samples %.0f" % (tot, tss))
for e, (c, s, ss, src) in sorted(by.items(), key=lambda kv: -kv[1][1])[:n_show]:
    ops = defaultdict(int)
    for x in src:
        op = x.split()[1] if x.startswith("@") else x.split()[0]
        ops[op.split(".")[0]] += 1
    top = " ".join("%s:%d" % kv for kv in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    print("exec %10d  n_instr %4d  %5.1f%% of instr  %5.1f%% of stalls  | %s" % (e, c, 100 * s / tot, 100 * ss / tss, top))
