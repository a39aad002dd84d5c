"""Per CUDA source line: instructions executed and stall samples, from an ncu report.
usage: python profiles/srclines.py <report.ncu-rep> <kernel-regex> [top] [launch-skip]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                               "-k", "regex:" + kern, "--launch-skip", skip, "--launch-count", "1"], text=True,
                              stderr=subprocess.DEVNULL)
rows = list(csv.reader(out.splitlines()))
agg, fname, hdr = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] and r[0] != "Line No" and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            ins = int(d["Instructions Executed"]); smp = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        agg.append((ins, smp, f"{fname}:{r[0]}", r[1].strip()[:90]))
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for ins, smp, loc, src in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{100 * ins / ti:5.1f}% ins {100 * smp / ts:5.1f}% stall  {loc:18s} {src}")
