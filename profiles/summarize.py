"""Summarise ncu outputs: launch lists (per-kernel time share) and --set full captures.

usage: python profiles/summarize.py launches <launches.csv> [runs]
       python profiles/summarize.py full <report.ncu-rep>
"""
import collections
import csv
import subprocess
import sys


def launches(path, runs=1):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            nm = d["Kernel Name"].split("(")[0][:48]
            agg[nm][0] += 1
            agg[nm][1] += float(d["Metric Value"]) / 1e3  # us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':48s} {'launches':>8s} {'ms/run':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {v[0] / runs:8.1f} {v[1] / 1e3 / runs:9.3f} {100 * v[1] / tot:5.1f}%")
    print(f"{'total':48s} {'':8s} {tot / 1e3 / runs:9.3f}")


def full(path):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size"]
    idx = [hdr.index(w) for w in want if w in hdr]
    print(" | ".join(want))
    for r in rows[2:]:
        print(" | ".join((r[i].split("(")[0][:40] if j == 0 else r[i]) + ("" if j == 0 else " " + units[i])
                         for j, i in enumerate(idx)))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)
    else:
        full(sys.argv[2])
