#!/usr/bin/env python
"""Benchmark: undirected edges/s to final component labels (BASELINE.json metric).

One step = one cc_run(mode=auto) -- the whole hot path of Alg. 2 (degree distribution,
gate, optional BFS peel + filter, edge-tuple SV to convergence) -- on the BASELINE.json
workload configs[1] (C2, de Bruijn-like, ~16.1 M vertices / ~16.9 M edges), with the edge
list already resident in HBM.  See DESIGN.md §6 for the byte models behind `roofline`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--mode auto]
  python bench.py --impl reference ...      # the CPU oracle, timed on the host cores

N > 1 (torchrun, one process per GPU): the same workload sharded over the ranks -- rank k
loads block k of the edge list, the library regroups arcs to vertex-block owners and combines
partition slots over NCCL (cc_comm over torch.distributed) -- strong scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "undirected edges/sec to final labels"
UNIT = "edges/s"
WORKLOADS = {
    "c1": "C1 forest-of-blocks: n=65,536, m=200,000, 4,096 blocks of 16 (BASELINE configs[0])",
    "c2": "C2 de Bruijn-like: 50,000 geometric(mean 320) paths + 5% bubbles + 0.5% joins, "
          "ids permuted (BASELINE configs[1])",
    "c3": "C3 road-like: 4096x4096 lattice, p=0.55, +1% diagonals, ids permuted (configs[2])",
    "c4": "C4 R-MAT scale 26, edge factor 16, a/b/c/d=.57/.19/.19/.05, ids permuted (configs[3])",
    "c5": "C5 R-MAT scale 28 U 10 M geometric(mean 64) paths, u64 ids (configs[4]) at --scale",
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


def make_graph(cfg, scale=1.0):
    import graphgen
    return graphgen.make(cfg, scale)


def default_scale(cfg, ws):
    """C5 (u64 ids, 4.9 G edges) needs 8 GPUs at full size, and every rank
    here draws the whole edge list on the host before taking its block (79 GB at full size):
    the default is 1/16 of it at any N; --scale 1 asks for the full config."""
    return 1.0 / 16 if cfg == "c5" else 1.0


def shard(edges, rank, ws):
    """Block distribution of the edge list over the ranks."""
    m = edges.shape[0]
    return np.ascontiguousarray(edges[m * rank // ws:m * (rank + 1) // ws])


def alg_bytes(rep, n, m):
    """SURVEY.md §8(d) byte model (u32 ids): B_SV = 8m + 8A_0 + sum_i B_i + 4n + 4n_p with
    B_i = 32 A_i + 48 A_{i+1} + 40 T_i; BFS route adds 32m + 20n."""
    its = rep["iters"]
    m_sv = rep["remainder_edges"] if rep["ran_bfs"] else m
    b = 8.0 * m_sv + 4.0 * n + 4.0 * rep["n_present"]
    for i, it in enumerate(its):
        a_i = it["active_in"]
        a_next = its[i + 1]["active_in"] if i + 1 < len(its) else 0
        b += 32.0 * a_i + 48.0 * a_next + 40.0 * it["temps"]
    if its:
        b += 8.0 * its[0]["active_in"]
    if rep["ran_bfs"]:
        b += 32.0 * m + 20.0 * n
    return b


def run_reference(args):
    """--impl reference: the CPU oracle (union-find, oracle/uf.c), as it stands."""
    ws, rk, _ = dist_info()
    if rk != 0:
        return 0
    import oracle
    scale = args.scale or default_scale(args.config, ws)
    g = make_graph(args.config, scale)
    oracle.build()
    run = (lambda: oracle.uf_labels_u64(g.edges)) if g.n == 0 else (lambda: oracle.uf_labels(g.n, g.edges))
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = time.perf_counter() - t0
    v = g.m * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64" if g.n == 0 else "u32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "scale": scale, "n": g.n, "m": g.m, "mode": "auto"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"whole {args.config} graph per step (union-find, 1 thread)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(g, budget_s=12.0):
    import oracle
    oracle.build()
    reps, t_used = 0, 0.0
    if g.n == 0:  # u64 ids: the oracle (sort-unique + union-find) on a bounded prefix
        e = g.edges[:min(g.m, 20_000_000)]
        t0 = time.perf_counter()
        oracle.uf_labels_u64(e)
        t_used = time.perf_counter() - t0
        return {"value": e.shape[0] / t_used, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"u64 union-find oracle (sort-unique + union-find) on the first "
                          f"{e.shape[0]} edge records of the workload, {t_used:.1f} s, single thread"}
    t0 = time.perf_counter()
    while reps < 20 and t_used < budget_s:
        oracle.uf_labels(g.n, g.edges)
        reps += 1
        t_used = time.perf_counter() - t0
    return {"value": g.m * reps / t_used, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"union-find oracle on the whole workload graph, {reps} repetition(s), "
                      f"{t_used:.1f} s, single thread"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="auto", choices=["auto", "sv", "bfs+sv"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--regroup", default="csr", choices=["csr", "csrbfs", "direct", "sort"],
                    help="SV bucket regroup engine (DESIGN.md §5.3)")
    ap.add_argument("--scale", type=float, default=None,
                    help="fraction of the config's size (default 1; c5 on one GPU: 1/16)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true",
                    help="time without the per-kernel CUDA events (no roofline breakdown)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1607_06156_b200 as cc

    ws, rk, lr = dist_info()
    # CC_DIST_BACKEND=gloo CC_SHARE_GPU=1 exercise the N > 1 code path on one GPU (correctness
    # only: ranks then share the device and exchange through host memory)
    backend = os.environ.get("CC_DIST_BACKEND", "nccl")
    if os.environ.get("CC_SHARE_GPU") == "1":
        lr = 0
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    stream = torch.cuda.current_stream(dev)

    scale = args.scale or default_scale(args.config, ws)
    g = make_graph(args.config, scale)
    n, m = g.n, g.m
    u64 = n == 0  # C5: u64 ids, relabelled on the device (Alg. 2 line 4)
    ids = "u64" if u64 else "u32"
    mine = shard(g.edges, rk, ws)
    flags = (0 if args.no_profile else cc.CC_FLAG_PROFILE) | cc.REGROUP_FLAGS[args.regroup]
    comm = cc.TorchComm(device=dev) if ws > 1 else None
    ctx = cc.CC(device=lr, stream=stream, flags=flags, comm=comm)
    d_edges = torch.from_numpy(mine.view(np.int64 if u64 else np.int32)).to(dev)
    ctx.load(d_edges, n, ids=ids)
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    for _ in range(max(3, args.warmup)):
        rep = ctx.run(args.mode)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = Clocks(lr)
    clocks.start()
    names = cc.kernel_families()
    fam = {i: [0.0, 0.0, 0] for i in range(len(names))}
    launches = 0

    def timed_steps(profiled):
        """K steps, L2 flushed before each (outside the step's events); returns total ms."""
        nonlocal launches, rep
        ctx.set_profiling(profiled)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        torch.cuda.synchronize()
        for k in range(args.steps):
            l2_flush.zero_()
            ev[k][0].record(stream)
            rep = ctx.run(args.mode)
            ev[k][1].record(stream)
            if profiled:
                for f in fam:
                    s = ctx.kernel_stats(f)
                    fam[f][0] += s["ms"]
                    fam[f][1] += s["bytes"]
                    fam[f][2] += s["launches"]
            else:
                launches += ctx.launches()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev)

    # the step time without per-kernel events (they cost ~4 % in host API calls), then the
    # same K steps with CUDA events around each kernel family for the roofline breakdown
    ms = timed_steps(False)
    ms_prof = timed_steps(not args.no_profile)
    ctx.set_profiling(False)
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    red_dev = dev if backend == "nccl" else "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = m * args.steps / (ms_max / 1e3)

    # ---------------- e2e: host buffers through the public API (H2D + run + D2H)
    e2e = None
    if not args.no_e2e:
        host = torch.from_numpy(mine.view(np.int64 if u64 else np.int32)).pin_memory()
        lo, hi = ctx.block_range()
        hout = torch.empty(hi - lo, dtype=torch.int32).pin_memory()
        hnp = host.numpy().view(np.uint64 if u64 else np.uint32)
        onp = hout.numpy().view(np.uint32)

        def e2e_step():
            ctx.load(hnp, n, ids=ids)
            ctx.run(args.mode)
            return ctx.labels_u64() if u64 else ctx.labels(onp)
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ke = max(1, min(args.steps, 5))
        e0.record(stream)
        for _ in range(ke):
            out_lab = e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": m * ke / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(mine.nbytes),
               "d2h_bytes_per_step": int((16 if u64 else 4) * (hi - lo)), "steps": ke}
        ok = None
        if rk == 0:
            orc = __import__("oracle")
            if not u64:
                ok = bool(np.array_equal(onp, orc.uf_labels(n, g.edges)[lo:hi]))
            elif ws == 1:  # (sorted distinct ids, labels) against the u64 oracle
                want = orc.uf_labels_u64(g.edges)
                ok = bool(np.array_equal(out_lab[0], want[0]) and np.array_equal(out_lab[1], want[1]))

    if rk == 0:
        peak, peak_src = peaks()
        # dominant kernel: the single-kernel family with the largest device time in the timed
        # region (family 1 is the whole-iteration aggregate, excluded)
        leaf = [i for i in fam if i != 1 and fam[i][0] > 0]
        dom = max(leaf, key=lambda i: fam[i][0]) if leaf else None
        kernels = {names[i]: {"ms_per_step": fam[i][0] / args.steps,
                              "alg_GBps": (fam[i][1] / (fam[i][0] / 1e3)) / 1e9 if fam[i][0] else None,
                              "launches_per_step": fam[i][2] / args.steps}
                   for i in fam if fam[i][0] > 0}
        if dom is not None:
            d_ms, d_bytes, d_launches = fam[dom]
            achieved = (d_bytes / (d_ms / 1e3)) / 1e9
        else:
            d_ms, d_bytes, d_launches, achieved = 0.0, 0.0, 0, None
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            tr = json.load(open(tp)).get(f"{args.config}/{args.regroup}", {})
            traffic = tr.get(names[dom]) if dom is not None else None
        path_bytes = alg_bytes(rep, n if not u64 else rep["n_present"], m)
        step_s = ms_max / 1e3 / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps,
            "ms_per_step_profiled": ms_prof / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64" if u64 else "u32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "scale": scale,
                       "n": n if not u64 else int(rep["n_present"]), "m": m, "mode": args.mode,
                       "regroup": args.regroup,
                       "route": "bfs+sv" if rep["ran_bfs"] else "sv",
                       "sv_iterations": rep["sv_iterations"],
                       "l2": "flushed between timed steps (256 MiB write, outside step events)",
                       "parallelism": (f"{ws} ranks: edge blocks, vertex-block owners, NCCL slot "
                                       "exchange" if ws > 1 else "1 GPU")},
            "roofline": {"bound": "hbm", "kernel": names[dom] if dom is not None else None,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": (d_bytes / d_launches) if d_launches else None,
                         "ms_per_launch": (d_ms / d_launches) if d_launches else None,
                         "share_of_step": (d_ms / ms_prof) if ms_prof else None,
                         "timing": "CUDA events around each launch on the library stream, in a "
                                   "second pass of the same K steps (ms_per_step_profiled)",
                         "launches_per_step": d_launches / args.steps},
            "kernels": kernels,
            "path_roofline": {"alg_bytes_per_step": path_bytes,
                              "frac": (path_bytes / (peak * 1e9)) / step_s,
                              "model": "SURVEY.md §8(d): 8m+8A0+sum(32A_i+48A_i+1+40T_i)+4n+4n_p"},
            "stages_ms": {k: rep[k] for k in ("ms_relabel", "ms_prediction", "ms_bfs", "ms_filter", "ms_sv",
                                              "ms_finalize")},
            "sv_iters": [{"A": it["active_in"], "P": it["partitions"], "ms": round(it["ms"], 4)}
                         for it in rep["iters"]],
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "e2e_labels_match_oracle": ok if e2e else None,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(g)
        print(json.dumps(line))
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
