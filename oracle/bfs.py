"""BFS peel and filter of Alg. 2.  TEST INFRASTRUCTURE.

* root: "choose a seed s in V" -- reading R10: the vertex
  of maximum degree, ties to the smallest id.
* :func:`bfs` -- level-synchronous BFS from the root over the arc list (each undirected
  edge as two arcs), frontier by frontier; returns the visited set VI and
  the number of levels (the root's eccentricity).
* :func:`filter_edges` -- "V <- V \\ VI; E <- E \\ {(u,v) | u in VI}".
  With both arcs stored, an edge with one visited endpoint has both endpoints visited, so
  the remainder is the set of edges with an unvisited first endpoint.
* label of the visited component = min id in VI.
"""
from __future__ import annotations

import numpy as np


def bfs_root(deg):
    deg = np.asarray(deg)
    return int(np.argmax(deg))  # argmax returns the first (smallest id) maximum


def bfs(n, edges, root):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    order = np.argsort(src, kind="stable")
    src, dst = src[order], dst[order]
    off = np.searchsorted(src, np.arange(n + 1))
    visited = np.zeros(n, bool)
    visited[root] = True
    frontier = np.array([root], dtype=np.int64)
    levels = 0
    while True:
        # all arcs out of the frontier
        starts, ends = off[frontier], off[frontier + 1]
        lens = ends - starts
        if lens.sum() == 0:
            break
        idx = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + \
            np.arange(lens.sum())
        nb = np.unique(dst[idx])
        nb = nb[~visited[nb]]
        if nb.shape[0] == 0:
            break
        visited[nb] = True
        frontier = nb
        levels += 1
    return visited, levels


def filter_edges(edges, visited):
    e = np.asarray(edges).reshape(-1, 2)
    return e[~visited[e[:, 0].astype(np.int64)]]
