"""Kernel timeline of one cc_run (CUPTI through torch.profiler): per-kernel start/duration and
the idle gaps between consecutive kernels on the device, to see where a step's time goes
beyond the kernels themselves (launch latency, host round trips, memsets).

usage: python scripts/timeline.py [--config c2] [--mode auto] [--out gpurun_out/timeline.json]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--op", default="run", choices=["run", "degrees"],
                    help="degrees: only the prediction-stage degree count (cc_degrees_u32)")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import graphgen
    import paper_1607_06156_b200 as cc
    g = graphgen.make(args.config, args.scale)
    dev = torch.device("cuda", 0)
    ctx = cc.CC(device=0)
    u64 = g.n == 0
    ctx.load(torch.from_numpy(g.edges.view(np.int64 if u64 else np.int32)).to(dev), g.n,
             ids="u64" if u64 else "u32")
    op = (lambda: ctx.run(args.mode)) if args.op == "run" else (lambda: ctx.degrees(g.n))
    for _ in range(3):
        op()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        op()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    rows = []
    for e in evs:
        rows.append((e.time_range.start, e.time_range.end, e.name[:60]))
    rows.sort()
    if not rows:  # no CUPTI records (e.g. under ncu, which owns the profiling interface)
        print("timeline: no kernel records")
        ctx.close()
        return
    t0, t1 = rows[0][0], rows[-1][1]
    busy = sum(b - a for a, b, _ in rows)
    gaps = [(rows[i + 1][0] - rows[i][1], rows[i][2], rows[i + 1][2]) for i in range(len(rows) - 1)]
    by = collections.defaultdict(lambda: [0, 0.0])
    for a, b, nm in rows:
        by[nm][0] += 1
        by[nm][1] += (b - a)
    out = {"config": args.config, "span_us": t1 - t0, "busy_us": busy, "n_ops": len(rows),
           "gap_us": sum(max(0, g[0]) for g in gaps),
           "by_kernel": sorted([[k, v[0], round(v[1], 1)] for k, v in by.items()], key=lambda x: -x[2]),
           "largest_gaps": sorted([[round(g[0], 1), g[1], g[2]] for g in gaps], key=lambda x: -x[0])[:25],
           "ops": [[round(a - t0, 1), round(b - a, 1), nm] for a, b, nm in rows]}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("span_us", "busy_us", "gap_us", "n_ops")}))
    for k in out["by_kernel"][:20]:
        print(k)
    for gp in out["largest_gaps"][:12]:
        print("gap", gp)
    ctx.close()


if __name__ == "__main__":
    main()
