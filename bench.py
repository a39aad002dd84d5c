#!/usr/bin/env python
"""Benchmark: undirected edges/s to final component labels (BASELINE.json metric).

One step = one cc_run(mode=auto) -- the whole hot path of Alg. 2 (degree distribution, power-law
gate, BFS peel + filter when the gate says scale-free, edge-tuple SV to convergence on the rest)
-- with the edge list already resident in HBM (profiling starts after the edges
are loaded).  The default workload is BASELINE.json configs[3] (C4: R-MAT scale 26, 1.07 G
edges), the largest config that fits one GPU (C5 needs several).  See
DESIGN.md §6 for the byte and access models behind `roofline`, `kernels` and `path_roofline`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--mode auto]
  python bench.py --impl reference ...      # the CPU oracle, timed on the host cores

N > 1 (torchrun, one process per GPU): the same workload sharded over the ranks -- rank k
loads block k of the edge list, the library regroups arcs to vertex-block owners and combines
partition slots over NCCL -- strong scaling.
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
    "c4": "C4 R-MAT scale 26, edge factor 16, a/b/c/d=.57/.19/.19/.05, ids permuted (BASELINE configs[3])",
    "c5": "C5 R-MAT scale 28 U 10 M geometric(mean 64) paths, u64 ids (configs[4]) at --scale",
}
# the CPU reference arm's bounded sample per step (edges): the first REF_SAMPLE[c] edge records
# of the config (C4's are i.i.d., so a prefix is a uniform sample), same id range
REF_SAMPLE = {"c4": 1 << 25}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def micro_peaks():
    """Measured request-rate ceilings on this B200 (scripts/micro/l2_peaks.cu, smem_atomics.cu;
    profiles/r02/micro_peaks.json): the denominators of the access-bound roofline fractions."""
    p = os.path.join(ROOT, "profiles", "r02", "micro_peaks.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                mem = round(int(ln.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "cpu_model": model,
            "ram_gib": mem}


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
    """C5 (u64 ids, 4.9 G edges, 79 GB of records) needs 8 GPUs at full size (SURVEY §8
    table): full size at N = 8 (each rank draws its own block, graphgen.make_block), 1/16 of
    it below; --scale overrides."""
    if cfg != "c5":
        return 1.0
    return 1.0 if ws >= 8 else 1.0 / 16


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


def oracle_threads():
    return 1  # oracle/uf.c is a single-threaded union-find


def run_reference(args):
    """--impl reference: the CPU oracle (union-find, oracle/uf.c) as it stands, on the host cores.
    Each step is a bounded sample of the workload (REF_SAMPLE: a prefix of the edge list with the
    same id range; the whole graph for the small configs), so the K + W steps take a few minutes."""
    ws, rk, _ = dist_info()
    if rk != 0:
        return 0
    import graphgen
    import oracle
    scale = args.scale or default_scale(args.config, ws)
    if args.config in REF_SAMPLE and scale == 1.0:
        g = graphgen.make_prefix(args.config, REF_SAMPLE[args.config])
        sample = (f"first {g.m:,} edge records of {args.config} (of {16 << 26:,}; i.i.d. R-MAT edges, "
                  f"n = {g.n:,}), union-find, 1 thread, per step")
    else:
        g = make_graph(args.config, scale)
        sample = f"whole {args.config} graph (scale {scale}) per step (union-find, 1 thread)"
    oracle.build()
    run = (lambda: oracle.uf_labels_u64(g.edges)) if g.n == 0 else (lambda: oracle.uf_labels(g.n, g.edges))
    for _ in range(max(3, args.warmup)):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = time.perf_counter() - t0
    v = g.m * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64" if g.n == 0 else "u32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "scale": scale, "n": g.n, "m_per_step": g.m,
                   "mode": "auto"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(g, budget_s=12.0):
    import oracle
    oracle.build()
    reps, t_used = 0, 0.0
    host = host_info()
    if g.n == 0:  # u64 ids: the oracle (sort-unique + union-find) on a bounded prefix
        e = g.edges[:min(g.m, 20_000_000)]
        t0 = time.perf_counter()
        oracle.uf_labels_u64(e)
        t_used = time.perf_counter() - t0
        return {"value": e.shape[0] / t_used, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
                "sample": f"u64 union-find oracle (sort-unique + union-find) on the first "
                          f"{e.shape[0]} edge records of the workload, {t_used:.1f} s, single thread",
                "host": host}
    t0 = time.perf_counter()
    while reps < 20 and t_used < budget_s:
        oracle.uf_labels(g.n, g.edges)
        reps += 1
        t_used = time.perf_counter() - t0
    return {"value": g.m * reps / t_used, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
            "sample": f"union-find oracle on the whole workload graph, {reps} repetition(s), "
                      f"{t_used:.1f} s, single thread", "host": host}


def traffic_for(config, regroup, mode="auto"):
    """ncu DRAM bytes per cc_run by kernel family (profiles/traffic.json, scripts/traffic.py)."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return {}, None
    d = json.load(open(tp))
    return d.get(f"{config}/{regroup}" + ("" if mode == "auto" else "/" + mode), {}), d.get("_source")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="auto", choices=["auto", "sv", "bfs+sv"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--regroup", default="csr", choices=["csr", "csrbfs", "direct", "sort"],
                    help="SV bucket regroup engine (DESIGN.md §5.2)")
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
    if ws > 1 and args.config == "c5":
        # each rank draws only its own block of records (graphgen.make_block): at full size
        # the whole C5 list is 79 GB of host memory
        import graphgen
        g = graphgen.make_block(args.config, scale, rk, ws)
        n, m = g.n, int(g.params["m_total"])
        mine = g.edges
    else:
        g = make_graph(args.config, scale)
        n, m = g.n, g.m
        mine = shard(g.edges, rk, ws)
    u64 = n == 0  # C5: u64 ids, relabelled on the device (Alg. 2 line 4)
    ids = "u64" if u64 else "u32"
    flags = (0 if args.no_profile else cc.CC_FLAG_PROFILE) | cc.REGROUP_FLAGS[args.regroup]
    # N > 1: the library owns an NCCL communicator (cfg.nccl_id, include/cc.h) and enqueues
    # every exchange on its stream; the process group only broadcasts the NCCL id.  gloo (one
    # shared GPU, correctness runs) goes through the cc_comm callbacks instead.
    comm = None
    if ws > 1:
        comm = cc.NcclGroup.from_process_group() if backend == "nccl" else cc.TorchComm(device=dev)
    ctx = cc.CC(device=lr, stream=stream, flags=flags, comm=comm)
    d_edges = torch.from_numpy(mine.view(np.int64 if u64 else np.int32)).to(dev)
    ctx.load(d_edges, n, ids=ids)
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    warmup = max(3, args.warmup)
    for _ in range(warmup):
        rep = ctx.run(args.mode)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = Clocks(lr)
    clocks.start()
    names = cc.kernel_families()
    fam = {i: {"ms": 0.0, "bytes": 0.0, "launches": 0, "ops": 0.0, "ops_unit": ""} for i in range(len(names))}
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
                    for key in ("ms", "bytes", "launches", "ops"):
                        fam[f][key] += s[key]
                    fam[f]["ops_unit"] = s["ops_unit"]
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
    e2e, ok = None, None
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
               "d2h_bytes_per_step": int((16 if u64 else 4) * (hi - lo)), "steps": ke,
               "path": "cc_load_edges(pinned host pairs) + cc_run + cc_labels (pinned host out)"}
        if rk == 0:
            orc = __import__("oracle")
            if not u64:
                ok = bool(np.array_equal(onp, orc.uf_labels(n, g.edges)[lo:hi]))
            elif ws == 1:  # (sorted distinct ids, labels) against the u64 oracle
                want = orc.uf_labels_u64(g.edges)
                ok = bool(np.array_equal(out_lab[0], want[0]) and np.array_equal(out_lab[1], want[1]))

    if rk == 0:
        peak, peak_src = peaks()
        mp = micro_peaks()
        traffic, traffic_src = traffic_for(args.config, args.regroup, args.mode)
        K = args.steps
        # dominant kernel: the single-kernel family with the largest device time in the timed
        # region (family 1 is the whole-iteration aggregate, excluded)
        leaf = [i for i in fam if i != 1 and fam[i]["ms"] > 0]
        dom = max(leaf, key=lambda i: fam[i]["ms"]) if leaf else None
        ops_peak = {"random 4-byte L2 reads (2 per edge of the level)": ("l2_random_read_Gops", "L2"),
                    "shared-memory atomics (2 per arc: bucket claim + count)": ("smem_atomic_Gops", "SMEM")}
        kernels = {}
        for i in fam:
            f = fam[i]
            if f["ms"] <= 0:
                continue
            row = {"ms_per_step": f["ms"] / K,
                   "alg_GBps": (f["bytes"] / (f["ms"] / 1e3)) / 1e9,
                   "hbm_frac": (f["bytes"] / (f["ms"] / 1e3)) / 1e9 / peak,
                   "launches_per_step": f["launches"] / K,
                   "share_of_step": f["ms"] / ms_prof if ms_prof else None}
            tr = traffic.get(names[i])
            if tr:
                row["dram_bytes_per_step_ncu"] = tr
                row["dram_GBps"] = tr / (f["ms"] / K / 1e3) / 1e9
                row["dram_frac"] = row["dram_GBps"] / peak
            if f["ops"] > 0:
                pk = ops_peak.get(f["ops_unit"])
                row["ops_unit"] = f["ops_unit"]
                row["Gops_per_s"] = f["ops"] / (f["ms"] / 1e3) / 1e9
                if pk and mp.get(pk[0]):
                    row["ops_peak_Gops"] = mp[pk[0]]
                    row["ops_frac"] = row["Gops_per_s"] / mp[pk[0]]
            kernels[names[i]] = row
        roof = {"bound": "hbm", "kernel": None}
        if dom is not None:
            f = fam[dom]
            achieved = (f["bytes"] / (f["ms"] / 1e3)) / 1e9
            kr = kernels[names[dom]]
            roof = {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak,
                    "traffic": (traffic.get(names[dom]) / (f["launches"] / K)) if traffic.get(names[dom]) else None,
                    "traffic_unit": "ncu dram bytes read+written per launch (profiles/traffic.json)",
                    "peak_source": peak_src,
                    "alg_bytes_per_launch": f["bytes"] / f["launches"] if f["launches"] else None,
                    "ms_per_launch": f["ms"] / f["launches"] if f["launches"] else None,
                    "share_of_step": f["ms"] / ms_prof if ms_prof else None,
                    "timing": "CUDA events around each launch on the library stream, in a second pass "
                              "of the same K steps (ms_per_step_profiled)",
                    "launches_per_step": f["launches"] / K}
            if "ops_frac" in kr:
                # what actually bounds it: the random-access request rate, against the measured
                # ceiling of the same access pattern on this GPU
                roof["access_bound"] = {"unit": kr["ops_unit"], "achieved_Gops": kr["Gops_per_s"],
                                        "peak_Gops": kr["ops_peak_Gops"], "frac": kr["ops_frac"],
                                        "peak_source": mp.get("source")}
            if "dram_GBps" in kr:
                roof["dram_GBps_live"] = kr["dram_GBps"]
                roof["dram_frac"] = kr["dram_frac"]
        # north star: DRAM bytes the SV iterations move (ncu, per run) over the
        # iterations' device time (family 1, CUDA events around each iteration)
        sv_dram = None
        if 1 in fam and fam[1]["ms"] > 0 and traffic:
            sv_fams = [k for k in traffic if k.startswith(("k_rowpass", "k_pstat", "k_compact"))]
            b = sum(traffic[k] for k in sv_fams)
            if b > 0:
                gbps = b / (fam[1]["ms"] / K / 1e3) / 1e9
                sv_dram = {"ncu_bytes_per_step": b, "ms_per_step": fam[1]["ms"] / K, "GBps": gbps,
                           "frac": gbps / peak, "families": sv_fams,
                           "target": "north star: >= 0.5 of HBM per SV iteration"}
        path_bytes = alg_bytes(rep, n if not u64 else rep["n_present"], m)
        step_s = ms_max / 1e3 / K
        dram_step = sum(v for k, v in traffic.items()) if traffic else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
            "warmup": warmup, "ms_per_step": ms_max / K,
            "ms_per_step_profiled": ms_prof / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64" if u64 else "u32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "scale": scale,
                       "n": n if not u64 else int(rep["n_present"]), "m": m, "mode": args.mode,
                       "regroup": args.regroup,
                       "route": "bfs+sv" if rep["ran_bfs"] else "sv",
                       "bfs_levels": rep["bfs_levels"], "remainder_edges": rep["remainder_edges"],
                       "sv_iterations": rep["sv_iterations"],
                       "l2": ("inputs larger than L2 (edge list %.1f GB) and a 256 MiB write between "
                              "timed steps, outside the step's events" % (mine.nbytes / 1e9)),
                       "parallelism": (f"{ws} ranks: edge blocks, vertex-block owners, library-owned "
                                       f"NCCL exchange ({backend})" if ws > 1 else "1 GPU")},
            "roofline": roof,
            "kernels": kernels,
            "path_roofline": {"alg_bytes_per_step": path_bytes,
                              "frac": (path_bytes / (peak * 1e9)) / step_s,
                              "model": "SURVEY.md §8(d): 8m+8A0+sum(32A_i+48A_i+1+40T_i)+4n+4n_p, BFS route "
                                       "+32m+20n; the bytes a sort-based regroup would move, not what this "
                                       "design moves: read as 'equivalent to that design at X of peak'"},
            "dram_path": ({"ncu_bytes_per_step": dram_step, "GBps": dram_step / step_s / 1e9,
                           "frac": dram_step / step_s / 1e9 / peak, "source": traffic_src}
                          if dram_step else None),
            "sv_iteration_dram": sv_dram,
            "stages_ms": {k: rep[k] for k in ("ms_relabel", "ms_prediction", "ms_bfs", "ms_filter", "ms_sv",
                                              "ms_finalize")},
            "sv_iters": [{"A": it["active_in"], "P": it["partitions"], "ms": round(it["ms"], 4)}
                         for it in rep["iters"]],
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "e2e_labels_match_oracle": ok,
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
