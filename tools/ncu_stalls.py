"""Stall-reason totals of an `ncu --page source --csv --print-source sass` dump, overall and for
the top source regions (instruction ranges with equal execution counts).

    python tools/ncu_stalls.py SASS.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
seen, d2 = set(), []
for r in data:
    if r[0] not in seen:
        seen.add(r[0])
        d2.append(r)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = defaultdict(float)
for r in d2:
    for c in cols:
        tot[c] += f(r[idx[c]])
s = sum(tot.values()) or 1
print("total samples", s)
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print("  %-24s %5.1f%%" % (c, 100 * v / s))
ie, isrc = h.index("Instructions Executed"), h.index("Source")
top = sorted(d2, key=lambda r: -sum(f(r[idx[c]]) for c in cols))[:25]
print("top instructions by stall samples:")
for r in sorted(top, key=lambda r: int(r[0], 16)):
    st = sorted(((f(r[idx[c]]), c) for c in cols), reverse=True)[:2]
    print("  %s %-44s %6.1f%%  %s" % (r[0][-5:], r[isrc][:44], 100 * sum(f(r[idx[c]]) for c in cols) / s,
                                     ", ".join("%s %.0f" % (c[6:], v) for v, c in st if v)))
