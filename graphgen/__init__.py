"""Seeded synthetic graph generators (inputs only; no connected-components arithmetic).

This is the single module shared by the oracle side (``oracle/``, ``tests/``) and the
CUDA side (``bench.py``, GPU tests).  It only draws edge lists; see ``gen.c`` for the
counter-based RNG and the Feistel id/edge-order bijections.

The five BASELINE.json configs (SURVEY.md §8(d) table "Synthetic inputs") are exposed
through :func:`make`, each with a ``scale`` knob so tests can draw smaller analogs of the
same structure.  Every graph is returned as an ``(m, 2)`` uint32 array of undirected
edge records (duplicates and self-loops kept) plus the id bound ``n``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgraphgen.so")
_lib = None

BASE_SEED = 1607061560


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        u64, u32, i32, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
        p32 = ctypes.c_void_p
        p64 = ctypes.POINTER(ctypes.c_uint64)
        lib.gg_rand.restype = u64
        lib.gg_rand.argtypes = [u64, u64, u64]
        lib.gg_perm_value.restype = u64
        lib.gg_perm_value.argtypes = [u64, u64, u64, u64]
        lib.gg_blocks.argtypes = [u64, u64, u64, u64, p32]
        lib.gg_er.argtypes = [u64, u64, u64, p32]
        lib.gg_paths.argtypes = [u64, u64, dbl, u64, u64, p64, p32]
        lib.gg_grid.argtypes = [u64, u64, u32, u64, p64, p32]
        lib.gg_rmat.argtypes = [u64, u32, u64, u32, u32, u32, i32, p32]
        lib.gg_union_u64.argtypes = [u64, p32, u64, u64, p32, u64, p32]
        lib.gg_mix64_value.restype = u64
        lib.gg_mix64_value.argtypes = [u64]
        lib.gg_c5_block.argtypes = [u64, u64, u32, u64, u32, u32, u32, p32, u64, u64, u64, p32]
        lib.gg_c5_block.restype = i32
        for f in (lib.gg_blocks, lib.gg_er, lib.gg_paths, lib.gg_grid, lib.gg_rmat, lib.gg_union_u64):
            f.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class Graph:
    name: str
    n: int              # id bound: ids are in [0, n) (0 for u64 ids: V = ids that appear)
    edges: np.ndarray   # (m, 2) uint32 (u64 for c5), undirected edge records
    params: dict

    @property
    def m(self) -> int:
        return int(self.edges.shape[0])


def blocks(seed: int, n: int, m: int, block: int) -> np.ndarray:
    out = np.empty((m, 2), dtype=np.uint32)
    rc = _L().gg_blocks(seed, n, m, block, _ptr(out))
    if rc:
        raise ValueError("n must be a multiple of block")
    return out


def er(seed: int, n: int, m: int) -> np.ndarray:
    out = np.empty((m, 2), dtype=np.uint32)
    _L().gg_er(seed, n, m, _ptr(out))
    return out


def paths(seed: int, n_paths: int, mean_len: float, bubble_ppm: int, join_ppm: int):
    counts = (ctypes.c_uint64 * 2)()
    _L().gg_paths(seed, n_paths, mean_len, bubble_ppm, join_ppm, counts, None)
    n, m = int(counts[0]), int(counts[1])
    out = np.empty((m, 2), dtype=np.uint32)
    _L().gg_paths(seed, n_paths, mean_len, bubble_ppm, join_ppm, counts, _ptr(out))
    return n, out


def grid(seed: int, side: int, keep_p: float, n_diag: int):
    keep32 = int(keep_p * 2**32)
    counts = (ctypes.c_uint64 * 2)()
    _L().gg_grid(seed, side, keep32, n_diag, counts, None)
    n, m = int(counts[0]), int(counts[1])
    out = np.empty((m, 2), dtype=np.uint32)
    _L().gg_grid(seed, side, keep32, n_diag, counts, _ptr(out))
    return n, out


def rmat(seed: int, scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19,
         permute_ids: bool = True, m: int | None = None) -> np.ndarray:
    """R-MAT edges 0 .. m-1 (default m = edge_factor << scale).  Edge e is a pure function of
    (seed, e) and the id permutation depends only on the scale, so a smaller m draws exactly
    the first m edges of the full list (a uniform sample: R-MAT edges are i.i.d.)."""
    m = (edge_factor << scale) if m is None else int(m)
    ta, tab, tabc = int(a * 2**32), int((a + b) * 2**32), int((a + b + c) * 2**32)
    out = np.empty((m, 2), dtype=np.uint32)
    _L().gg_rmat(seed, scale, m, ta, tab, tabc, int(permute_ids), _ptr(out))
    return out


def perm_value(n: int, seed: int, stream: int, x: int) -> int:
    return int(_L().gg_perm_value(n, seed, stream, x))


def union_u64(seed: int, a: np.ndarray, na: int, b: np.ndarray) -> np.ndarray:
    """Edges of a (indices < na) and b (indices offset by na) as u64 ids mix64(index), edge
    order scrambled (gen.c gg_union_u64)."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    out = np.empty((a.shape[0] + b.shape[0], 2), dtype=np.uint64)
    _L().gg_union_u64(seed, _ptr(a), a.shape[0], na, _ptr(b), b.shape[0], _ptr(out))
    return out


def mix64(k: int) -> int:
    return int(_L().gg_mix64_value(k))


def make(config: str, scale: float = 1.0, seed: int | None = None) -> Graph:
    """Draw one BASELINE.json config (``c1``..``c5``) at a fraction ``scale`` of its size.

    ``scale`` shrinks the vertex/edge counts while keeping the structure (block size,
    path length mix, keep probability, R-MAT parameters); scale=1 is the full config.
    """
    k = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}[config]
    s = BASE_SEED + k if seed is None else seed
    if config == "c1":
        # 65,536 vertices in 4,096 blocks of 16; 200,000 edges (BASELINE configs[0])
        n = max(16, int(65536 * scale) // 16 * 16)
        m = max(1, int(200000 * scale))
        return Graph("c1", n, blocks(s, n, m, 16), dict(block=16, scale=scale))
    if config == "c2":
        # 50,000 geometric(mean 320) paths, +5% bubbles, +0.5% joins (configs[1])
        npaths = max(1, int(50000 * scale))
        n, e = paths(s, npaths, 320.0, 50000, 5000)
        return Graph("c2", n, e, dict(n_paths=npaths, mean_len=320, scale=scale))
    if config == "c3":
        # 4096x4096 lattice, p=0.55, 1% diagonals of the lattice edge count (configs[2], C21)
        side = max(2, int(round(4096 * scale ** 0.5)))
        ndiag = (2 * side * (side - 1)) // 100
        n, e = grid(s, side, 0.55, ndiag)
        return Graph("c3", n, e, dict(side=side, scale=scale))
    if config == "c4":
        # R-MAT scale 26, edge factor 16, a/b/c/d = .57/.19/.19/.05 (configs[3])
        sc = max(4, 26 + int(round(np.log2(scale))) if scale != 1.0 else 26)
        e = rmat(s, sc, 16)
        return Graph("c4", 1 << sc, e, dict(rmat_scale=sc, scale=scale))
    if config == "c5":
        # R-MAT scale 28 (C4's parameters) U 10,000,000 geometric(mean 64) paths on fresh
        # indices 2^28 + j; u64 id = mix64(index); edge order scrambled (configs[4]).
        # Graph.n = 0: u64 ids, V = the ids that appear (C2).
        sc = max(4, 28 + int(round(np.log2(scale))) if scale != 1.0 else 28)
        a = rmat(s, sc, 16)
        npaths = max(1, int(10_000_000 * scale))
        _, b = paths(s + 100, npaths, 64.0, 0, 0)
        return Graph("c5", 0, union_u64(s, a, 1 << sc, b), dict(rmat_scale=sc, n_paths=npaths,
                                                                  scale=scale))
    raise KeyError(config)


def make_block(config: str, scale: float, rank: int, world: int) -> Graph:
    """Rank ``rank``'s block (PAPER.md:205 block distribution: records [m*rank/world,
    m*(rank+1)/world)) of ``make(config, scale)``, drawn without the other ranks' records.
    C5: the R-MAT part is drawn edge by edge inside the block (gen.c gg_c5_block); only the
    path part (~1/8 of the records) is drawn whole.  Other configs: drawn whole and sliced.
    ``Graph.params['m_total']`` is the whole list's length."""
    if config != "c5":
        g = make(config, scale)
        m = g.m
        e = np.ascontiguousarray(g.edges[m * rank // world:m * (rank + 1) // world])
        return Graph(config, g.n, e, dict(g.params, m_total=m, rank=rank, world=world))
    s = BASE_SEED + 5
    sc = max(4, 28 + int(round(np.log2(scale))) if scale != 1.0 else 28)
    npaths = max(1, int(10_000_000 * scale))
    _, b = paths(s + 100, npaths, 64.0, 0, 0)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    ma = 16 << sc
    m = ma + b.shape[0]
    i0, i1 = m * rank // world, m * (rank + 1) // world
    out = np.empty((i1 - i0, 2), dtype=np.uint64)
    a, ab, abc = int(0.57 * 2**32), int((0.57 + 0.19) * 2**32), int((0.57 + 0.19 + 0.19) * 2**32)
    _L().gg_c5_block(s, s, sc, ma, a, ab, abc, _ptr(b), b.shape[0], i0, i1, _ptr(out))
    return Graph("c5", 0, out, dict(rmat_scale=sc, n_paths=npaths, scale=scale, m_total=m, rank=rank,
                                    world=world))


def make_prefix(config: str, m_prefix: int) -> Graph:
    """The first ``m_prefix`` edge records of a full-size R-MAT config (c4), same id range:
    the bounded sample the CPU reference arm of bench.py times per step."""
    if config != "c4":
        raise KeyError("prefix samples are drawn for the R-MAT config c4 only")
    s = BASE_SEED + 4
    return Graph("c4", 1 << 26, rmat(s, 26, 16, m=m_prefix), dict(rmat_scale=26, m_prefix=m_prefix))


def rmat_scale_graph(scale: int, seed: int | None = None) -> Graph:
    s = BASE_SEED + 4 if seed is None else seed
    return Graph("c4", 1 << scale, rmat(s, scale, 16), dict(rmat_scale=scale))
