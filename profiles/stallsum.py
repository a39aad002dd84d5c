"""Warp-stall reason totals and a few throughput counters of each kernel in an ncu report.
usage: python profiles/stallsum.py <report.ncu-rep>"""
import csv
import subprocess
import sys

out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], text=True,
                              stderr=subprocess.DEVNULL)
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:70], d["gpu__time_duration.sum"], "us")
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    print("  stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
    for k in ["smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
              "dram__bytes_write.sum", "lts__t_sectors.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__thread_inst_executed_per_inst_executed.ratio"]:
        if k in d:
            print(f"  {k} = {d[k]}")
