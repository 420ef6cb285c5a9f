"""Summarise an `ncu --set full` capture of one tree (tools/profile_fit.py --trees 1) into
profiles/: a per-launch CSV, a per-kernel-class text summary, and profiles/ncu_traffic.json
(measured DRAM bytes per launch per kernel class, which bench.py reports as roofline.traffic).

    python tools/ncu_summary.py REP.ncu-rep OUT_PREFIX ["what was captured"] [kernel1,kernel2,...]

(the optional kernel list also dumps the SASS source page of each kernel's first launch; run it
on the GPU box next to the report and ship only the CSVs — reports exceed gpurun's copy limit)
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]
CLASS = {"k_hist<0>": "hist_root", "k_hist<1>": "hist_level", "k_hist<3>": "update", "k_hist_root2": "hist_root",
         "k_pcount": "partition", "k_pscan": "partition", "k_pscatter2": "partition", "k_split3": "split",
         "k_update": "update", "k_root_fix": "misc", "k_next_tree": "misc", "k_next_tree_cond": "misc",
         "k_part": "partition", "k_hist2<0>": "hist_root", "k_hist2<1>": "hist_level", "k_hist2<3>": "update"}


HIST_MODE = {"0": "hist_root", "1": "hist_level", "3": "update"}


def kclass(name):
    base = name.split("(")[0].replace("void ", "").replace("llmp::", "").strip()
    if base.startswith("k_hist<") or base.startswith("k_hist2<") or base.startswith("k_hist3<"):   # first template argument = the mode
        return HIST_MODE.get(base.split("<")[1].split(",")[0].split(">")[0].strip(), base), base
    return CLASS.get(base, base), base


def dump_sass(rep, prefix, recs, names):
    """Source (SASS) page of the first launch of each named kernel -> prefix_sass_<name>.csv"""
    for nm in names:
        idx = next((i for i, r in enumerate(recs) if r["kernel"] == nm), None)
        if idx is None:
            continue
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                              "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
        safe = nm.replace("<", "_").replace(">", "")
        with open("%s_sass_%s.csv" % (prefix, safe), "w") as f:
            f.write(out)


def main(rep, prefix, sass=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    data = rows[2:]
    idx = {m: hdr.index(m) for m in METRICS}
    ik = hdr.index("Kernel Name")
    recs = []
    for r in data:
        cls, base = kclass(r[ik])
        rec = {"kernel": base, "class": cls}
        for m in METRICS:
            try:
                rec[m] = float(r[idx[m]].replace(",", ""))
            except ValueError:
                rec[m] = None
        recs.append(rec)
    with open(prefix + "_ncu_launches.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["kernel", "class"] + METRICS)
        w.writeheader()
        w.writerows(recs)
    summarise(recs, prefix, os.path.basename(rep), sys.argv[3] if len(sys.argv) > 3 else "one tree of both ensembles")
    if sass:
        dump_sass(rep, prefix, recs, sass)


def summarise(recs, prefix, rep_name, what):
    """per-class totals -> PREFIX_ncu_summary.txt and ncu_traffic.json next to it"""
    agg = {}
    for r in recs:
        a = agg.setdefault(r["class"], {"launches": 0, "us": 0.0, "dram": 0.0, "inst": 0.0})
        a["launches"] += 1
        a["us"] += r["gpu__time_duration.sum"] or 0.0
        a["dram"] += ((r["dram__bytes_read.sum"] or 0) + (r["dram__bytes_write.sum"] or 0)) * 1e6  # Mbyte -> B
        a["inst"] += r["smsp__inst_executed.sum"] or 0.0
    lines = ["ncu --set full --clock-control none, %s (C3: 10M rows, depth 8); cold cache, serialised launches"
             % what, ""]
    traffic = {}
    for c, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        per = a["dram"] / a["launches"]
        lines.append("%-12s launches %3d  total %9.1f us  avg %8.1f us  DRAM %8.1f MB/launch  %6.2f TB/s  %7.1f M inst"
                     % (c, a["launches"], a["us"], a["us"] / a["launches"], per / 1e6,
                        a["dram"] / (a["us"] * 1e-6) / 1e12, a["inst"] / 1e6))
        traffic[c] = {"dram_bytes_per_launch": per, "avg_duration_us": a["us"] / a["launches"],
                      "launches_profiled": a["launches"],
                      "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch from %s" % rep_name}
    with open(prefix + "_ncu_summary.txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(os.path.dirname(prefix), "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


def from_csv(csv_path, prefix, what):
    """re-classify an existing PREFIX_ncu_launches.csv (e.g. after the class table changed)"""
    recs = []
    for r in csv.DictReader(open(csv_path)):
        cls, base = kclass(r["kernel"])
        rec = {"kernel": base, "class": cls}
        for m in METRICS:
            try:
                rec[m] = float(r[m])
            except (TypeError, ValueError):
                rec[m] = None
        recs.append(rec)
    summarise(recs, prefix, os.path.basename(csv_path).replace("_ncu_launches.csv", ".ncu-rep"), what)


if __name__ == "__main__":
    if sys.argv[1] == "--from-csv":
        from_csv(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "re-summarised launches")
    else:
        main(sys.argv[1], sys.argv[2], sys.argv[4].split(",") if len(sys.argv) > 4 else ())
