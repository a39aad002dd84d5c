"""Alg. 2, the hybrid driver.  TEST INFRASTRUCTURE.

  D <- Degree_Distribution(G)                       line 2  (oracle.degree)
  if K-S(D) < tau (paper) / gate G (default, C11):  line 3
      relabel (u64 input only)                      line 5  (oracle.relabel_u64)
      choose seed s; VI <- BFS(s)                   lines 7-8 (oracle.bfs)
      V <- V \\ VI; E <- E \\ {(u,v) | u in VI}      lines 10-11
  Parallel-SV(G(V,E))                               line 13 (oracle.sv)

mode: "auto" (the gate decides), "sv" (never BFS), "bfs+sv" (always BFS), matching the
fig:dynamic experiments and SPEC's force_mode.
"""
from __future__ import annotations

import numpy as np

from . import bfs as _bfs
from . import degree as _deg
from . import sv as _sv


def hybrid(n, edges, mode="auto", gate="ls", tau=_deg.KS_TAU, with_trace=True):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    deg, hist = _deg.degree_distribution(n, e)
    g = _deg.gate_ls(hist)
    ks = _deg.ks_powerlaw(hist)
    if mode == "auto":
        if gate == "ls":
            run_bfs = g["scale_free"]
        else:
            run_bfs = (ks["ks"] == ks["ks"]) and ks["ks"] < tau
    else:
        run_bfs = mode == "bfs+sv"
    report = dict(gate=g, ks=ks, ran_bfs=bool(run_bfs), max_degree=int(deg.max()) if n else 0)
    labels = np.arange(n, dtype=np.int64)
    rem = e
    if run_bfs and e.shape[0]:
        root = _bfs.bfs_root(deg)
        visited, levels = _bfs.bfs(n, e, root)
        ids = np.flatnonzero(visited)
        labels[ids] = ids.min()
        rem = _bfs.filter_edges(e, visited)
        report.update(bfs_root=root, bfs_visited=int(ids.shape[0]), bfs_levels=levels,
                      remainder_edges=int(rem.shape[0]))
    if with_trace:
        lab_sv, trace = _sv.sv_trace(n, rem)
        present = np.unique(rem)
        labels[present] = lab_sv[present]
        report["trace"] = trace
    else:
        from . import uf_labels
        lab_sv = uf_labels(n, rem.astype(np.uint32))
        present = np.unique(rem)
        labels[present] = lab_sv[present]
    return labels, report
