"""DRAM traffic per launch of the row-pass families (profiles/traffic.json, bench.py `traffic`).

Runs scripts/timeline.py under ncu (dram bytes + duration of every k_rowpass launch of the
fourth, profiled cc_run; the first three are warm-up) and averages per family over the
iterations of that run, the way bench.py averages the family's achieved bandwidth.

usage (GPU box): python scripts/traffic.py [--config c2] [--out profiles/traffic.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAM = {"true": "k_rowpass<A> +k_long1/2 (Alg.1 lines 8-16)",
       "false": "k_rowpass<B> +k_long1/2 (Alg.1 lines 17-25)"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "traffic.json"))
    ap.add_argument("--from-csv", default=None, help="recompute from a CSV an earlier run saved")
    args = ap.parse_args()
    if args.from_csv:
        return summarize(open(args.from_csv).read(), args)
    # launches of one cc_run: count them in a plain run first
    tl = os.path.join(ROOT, "gpurun_out", f"traffic_tl_{args.config}.json")
    subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "timeline.py"), "--config", args.config,
                           "--out", tl], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    per_run = sum(1 for o in json.load(open(tl))["ops"] if "k_rowpass" in o[2])  # both variants
    out = subprocess.check_output(
        ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
         "--clock-control", "none", "--csv", "-k", "regex:k_rowpass", "-s", str(3 * per_run), "-c", str(per_run),
         sys.executable, os.path.join(ROOT, "scripts", "timeline.py"), "--config", args.config, "--out", tl],
        text=True, stderr=subprocess.DEVNULL)
    with open(os.path.join(ROOT, "gpurun_out", f"traffic_{args.config}.csv"), "w") as f:
        f.write(out[out.index('"ID"'):])
    summarize(out, args)


def summarize(out, args):
    rows = [r for r in csv.reader(io.StringIO(out[out.index('"ID"'):]))]
    hdr = rows[0]
    acc = {}
    busy = set()  # launches that did the pass (the variant the device did not pick returns at once)
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            us = float(d["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                                             "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
            if us > 20.0:
                busy.add(d["ID"])
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum") or d["ID"] not in busy:
            continue
        kn = d["Kernel Name"]
        fam = FAM["true" if ("k_rowpass<true" in kn or "k_rowpass<1" in kn) else "false"]
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        key = (fam, d["ID"])
        acc[key] = acc.get(key, 0.0) + v
    res = {}
    for (fam, i), v in acc.items():
        res.setdefault(fam, []).append(v)
    data = json.load(open(args.out)) if os.path.exists(args.out) else {}
    data[f"{args.config}/csr"] = {f: sum(v) / len(v) for f, v in res.items()}
    data["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every k_rowpass launch "
                       "of one cc_run (scripts/traffic.py): mean per launch over the run's iterations")
    json.dump(data, open(args.out, "w"), indent=1)
    print(json.dumps(data[f"{args.config}/csr"]), {f: len(v) for f, v in res.items()})


if __name__ == "__main__":
    main()
