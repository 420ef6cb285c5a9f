"""Summarise an `ncu --page source --csv --print-source sass` dump: top SASS lines by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if r and r[0].startswith("0x")] if any(r and r[0].startswith("0x") for r in rows) else [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0] != "Address"]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[iss]) for r in data)
totx = sum(f(r[iex]) for r in data)
print("samples", tot, "warp-instructions", totx)
top = sorted(data, key=lambda r: -f(r[iss]))[:n]
for r in sorted(top, key=lambda r: int(r[ia], 16) if r[ia].startswith("0x") else 0):
    print(r[ia], "%5.1f%%" % (100 * f(r[iss]) / max(tot, 1)), "%10d" % f(r[iex]), r[isrc][:100])
