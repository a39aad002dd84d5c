"""DRAM traffic of one cc_run by kernel family (profiles/traffic.json, used by bench.py).

Runs scripts/timeline.py under ncu (dram bytes read + written and duration of every kernel of
the fourth cc_run; the first three are warm-up) and sums the bytes per kernel family (the
family names of include/cc.h cc_kernel_name), per cc_run.  The per-launch list is kept beside.

usage (GPU box): python scripts/traffic.py [--config c4] [--out profiles/traffic.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# kernel-name substring -> family (the names cc_kernel_name returns)
FAMILIES = [
    (("k_deg_part", "k_deg_order", "k_deg_count", "k_degree", "k_hub"),
     "degree count (k_deg_part, k_deg_order, k_deg_count)"),
    (("k_deg_hist", "k_hist_pairs"), "degree distribution (k_deg_hist, k_hist_pairs)"),
    (("k_bfs_level",), "k_bfs_level"),
    # k_u0 / k_pull0: iteration 0's pass A by pull (timed in the same family by the library)
    (("k_rowpass<true", "k_rowpass<1", "k_long1<true", "k_long2<true", "k_long1<1", "k_long2<1", "k_u0", "k_pull0"),
     "k_rowpass<A> +k_long1/2 (Alg.1 lines 8-16)"),
    (("k_rowpass<false", "k_rowpass<0", "k_long1<false", "k_long2<false", "k_long1<0", "k_long2<0"),
     "k_rowpass<B> +k_long1/2 (Alg.1 lines 17-25)"),
    (("k_pstat", "k_list_from_bits"), "k_pstat1/k_pstat2/k_list_from_bits (partition slot scans)"),
    (("k_rows", "k_fill", "k_bucket", "k_scatter", "k_place", "k_gscan"),
     "CSR build (k_rows, k_fill_*, k_bucket, k_scatter)"),
    (("k_compact", "k_collapse"), "k_compact (ordered exclusion of completed rows)"),
    (("k_onesweep", "k_hist<", "radix::k_hist"), "k_hist+k_onesweep (radix regroup)"),
]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TUNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def family(name):
    for keys, fam in FAMILIES:
        if any(k in name for k in keys):
            return fam
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--regroup", default="csr")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "traffic.json"))
    ap.add_argument("--from-csv", default=None, help="recompute from a CSV an earlier run saved")
    args = ap.parse_args()
    tag = args.config + ("" if args.mode == "auto" else "_" + args.mode)
    csv_path = os.path.join(ROOT, "gpurun_out", f"traffic_{tag}.csv")
    if args.from_csv:
        return summarize(open(args.from_csv).read(), args)
    tl = os.path.join(ROOT, "gpurun_out", f"traffic_tl_{tag}.json")
    tl_args = ["--config", args.config, "--mode", args.mode, "--out", tl]
    subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "timeline.py"), *tl_args],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    per_run = sum(1 for o in json.load(open(tl))["ops"] if not o[2].startswith(("Memset", "Memcpy")))
    out = subprocess.check_output(
        ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
         "--clock-control", "none", "--csv", "-s", str(3 * per_run), "-c", str(per_run),
         sys.executable, os.path.join(ROOT, "scripts", "timeline.py"), *tl_args],
        text=True, stderr=subprocess.DEVNULL)
    os.makedirs(os.path.dirname(csv_path), exist_ok=True)
    with open(csv_path, "w") as f:
        f.write(out[out.index('"ID"'):])
    summarize(out, args)


def summarize(out, args):
    rows = [r for r in csv.reader(io.StringIO(out[out.index('"ID"'):]))]
    hdr = rows[0]
    per = {}  # launch id -> [name, dram bytes, us]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        i = d["ID"]
        e = per.setdefault(i, [d["Kernel Name"], 0.0, 0.0])
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            e[1] += v * UNIT.get(d["Metric Unit"], 1.0)
        elif d["Metric Name"] == "gpu__time_duration.sum":
            e[2] += v * TUNIT.get(d["Metric Unit"], 1.0)
    fams = {}
    for name, by, us in per.values():
        f = family(name)
        fams[f] = fams.get(f, 0.0) + by
    data = json.load(open(args.out)) if os.path.exists(args.out) else {}
    data[f"{args.config}/{args.regroup}" + ("" if args.mode == "auto" else "/" + args.mode)] = fams
    data["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every kernel of one "
                       "cc_run after three warm-up runs (scripts/traffic.py): bytes per cc_run by kernel family")
    json.dump(data, open(args.out, "w"), indent=1)
    print(json.dumps(fams))
    print("launches", len(per), "ncu us total", round(sum(e[2] for e in per.values()), 1))


if __name__ == "__main__":
    main()
