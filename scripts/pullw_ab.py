"""A/B of iteration 0's pull windows (CC_PULLW, sv_rows.cu rowpass_a0_pull) in one process:
the graph is drawn and loaded once, then cc_run(mode) is timed per window size (wall clock
around the call, which returns after the device is idle; best and median of --reps runs).

usage: python scripts/pullw_ab.py [--config c4] [--mode sv] [--windows 0,24,23,25]
       [--envs 'CC_HOT_A=20;CC_HOT_B=5'] [--out f.json]   (other library knobs, same way)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--mode", default="sv")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--windows", default="0,24,23,25")
    ap.add_argument("--envs", default="", help="further settings, e.g. 'CC_HOT_A=20;CC_PULLW=24,CC_HOT_B=5'")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--out", default="gpurun_out/pullw_ab.json")
    args = ap.parse_args()
    import torch
    import graphgen
    import paper_1607_06156_b200 as cc
    g = graphgen.make(args.config, args.scale)
    dev = torch.device("cuda", 0)
    ctx = cc.CC(device=0)
    ctx.load(torch.from_numpy(g.edges.view(np.int32)).to(dev), g.n, ids="u32")
    res, ref = {}, None
    settings = args.windows.split(",") + (args.envs.split(";") if args.envs else [])
    touched = set()
    for si, w in enumerate(settings):
        for k in touched:  # every setting starts from the defaults
            os.environ.pop(k, None)
        kv = [x.split("=") for x in w.split(",")] if "=" in w else [["CC_PULLW", w]]
        for k, v in kv:
            os.environ[k] = v
            touched.add(k)
        ts = []
        for i in range(args.reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.run(args.mode)
            torch.cuda.synchronize()
            if i:
                ts.append((time.perf_counter() - t0) * 1e3)
        lab = ctx.labels()
        lab = lab if isinstance(lab, np.ndarray) else np.asarray(lab.cpu())
        if ref is None:
            ref = lab
        w = f"{si}:{w}"
        res[w] = {"best_ms": round(min(ts), 3), "median_ms": round(float(np.median(ts)), 3),
                  "labels_equal_first": bool(np.array_equal(lab, ref))}
        print(w, res[w], flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump({"config": args.config, "mode": args.mode, "n": int(g.n), "windows": res}, open(args.out, "w"), indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
