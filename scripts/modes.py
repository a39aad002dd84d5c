"""fig:dynamic / fig:dynamic_opp analog: every config in
the route the gate picks (auto) and in both hard-coded routes, one B200, edges resident.

    python scripts/modes.py [--configs c1,c2,c3,c4] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen  # noqa: E402
import paper_1607_06156_b200 as cc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-s", type=float, default=60.0, help="skip further reps past this")
    args = ap.parse_args()
    out = []
    for cfg in args.configs.split(","):
        g = graphgen.make(cfg)
        ctx = cc.CC(device=0)
        ctx.load(torch.from_numpy(g.edges.view(np.int32)).cuda(), g.n)
        row = {"config": cfg, "n": g.n, "m": g.m}
        for mode in ("auto", "sv", "bfs+sv"):
            t0 = time.time()
            rep = ctx.run(mode)  # warm-up
            if time.time() - t0 > args.max_s:
                row[mode] = {"ms": rep["ms_total"], "reps": 1, "route": "bfs+sv" if rep["ran_bfs"] else "sv"}
                continue
            ms = []
            for _ in range(args.reps):
                rep = ctx.run(mode)
                ms.append(rep["ms_total"])
            row[mode] = {"ms": float(np.median(ms)), "reps": args.reps,
                         "route": "bfs+sv" if rep["ran_bfs"] else "sv",
                         "sv_iterations": rep["sv_iterations"], "bfs_levels": rep["bfs_levels"]}
        row["opposite_over_auto"] = (row["bfs+sv" if row["auto"]["route"] == "sv" else "sv"]["ms"]
                                     / row["auto"]["ms"])
        ctx.close()
        print(json.dumps(row), flush=True)
        out.append(row)


if __name__ == "__main__":
    main()
