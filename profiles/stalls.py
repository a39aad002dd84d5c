"""Top SASS lines by warp-stall samples for one kernel of an ncu report.
usage: python profiles/stalls.py <report.ncu-rep> <kernel-regex> [launch-skip] [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                               "--launch-skip", skip, "--launch-count", "1"], text=True,
                              stderr=subprocess.DEVNULL)
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Source" in r and "Address" in r)
start = rows.index(hdr) + 1
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[i_s]), r[0], r[i_src]) for r in rows[start:] if len(r) > i_s and r[i_s].isdigit()]
tot = sum(d[0] for d in data) or 1
print(rows[0][1][:100], "samples", tot)
for s, a, src in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {a[-5:]} {src.strip()[:100]}")
