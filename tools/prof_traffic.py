"""DRAM bytes per processed row of each hot kernel class, averaged over whole trees: ncu collects
only dram__bytes_read/write.sum and gpu__time_duration.sum for every histogram / partition launch of
a 20-tree C3 fit (both targets paired, timing mode), and the fit's own row counters give the rows
each class processed.  Writes profiles/ncu_traffic.json (bench.py reports roofline.traffic from it).

    python tools/prof_traffic.py TAG          (on the GPU box; needs ncu)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import kclass  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "traffic"
out_csv = os.path.join(ROOT, "gpurun_out", tag + "_dram.csv")
cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--clock-control",
       "none", "--kernel-name", "regex:k_hist|k_part", "--csv", "--log-file", out_csv, sys.executable,
       os.path.join(ROOT, "tools", "profile_fit.py"), "--trees", "20", "--repeat", "1"]
p = subprocess.run(cmd, capture_output=True, text=True)
js = p.stdout[p.stdout.index("{"):p.stdout.rindex("}") + 1]
fit = json.loads(js)
rows = list(csv.reader(io.StringIO(open(out_csv).read()[open(out_csv).read().index('"ID"'):])))
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iu = hdr.index("Metric Unit")
agg = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
for r in rows[1:]:
    cls, _ = kclass(r[ik])
    a = agg.setdefault(cls, {"bytes": 0.0, "s": 0.0, "launches": 0})
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    if r[im].startswith("dram__bytes"):
        a["bytes"] += v
    else:
        a["s"] += v
        a["launches"] += 1
traffic = {}
for cls, a in agg.items():
    units = fit.get(cls, {}).get("units", 0)
    if not units or not a["launches"]:
        continue
    traffic[cls] = {"dram_bytes_per_unit": a["bytes"] / units, "dram_bytes_per_launch": a["bytes"] / a["launches"],
                    "units_profiled": units, "launches_profiled": a["launches"],
                    "note": "dram__bytes_read.sum + dram__bytes_write.sum over every %s launch of a 20-tree C3 fit "
                            "(ncu, cold-cache serialised replay) / the rows those launches processed (%s)" % (cls, tag)}
    print("%-12s %6d launches  %8.1f B/row  (%.0f rows)" % (cls, a["launches"], a["bytes"] / units, units))
json.dump(traffic, open(os.path.join(ROOT, "gpurun_out", "ncu_traffic_" + tag + ".json"), "w"), indent=1)
