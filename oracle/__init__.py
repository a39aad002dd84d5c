"""CPU oracle for the adaptive connected-components hot path (arXiv 1607.06156).

TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import, call, link or execute anything under ``oracle/``.  The oracle shares
no code with the CUDA path (``paper_1607_06156_b200/``); neither imports the other.
Inputs come only from ``graphgen`` (which holds none of the method's arithmetic).

Contents (each function cites the passage it follows):

* :func:`uf_labels` / :func:`uf_labels_u64` -- union-find labels, the plain definition
  label(v) = min id of v's component.  Plain C.
* :mod:`oracle.sv`      -- Alg. 1 transcribed step by step with the
  completed-partition exclusion of §3.1.4; per-iteration trace.
* :mod:`oracle.degree`  -- degree distribution (Alg. 2 line 2),
  the least-squares power-law gate G and the Clauset/K-S statistic.
* :mod:`oracle.bfs`     -- BFS peel + filter of Alg. 2.
* :mod:`oracle.hybrid`  -- Alg. 2 driver.
* :func:`relabel_u64`   -- order-preserving dense relabel.

Parity status per function is listed in DESIGN.md §4 ("Oracle and pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_uf.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the plain-C union-find (building the checker is not using it)."""
    src = os.path.join(_HERE, "uf.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _SO, src])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.oracle_uf_labels_u32.restype = ctypes.c_int64
        lib.oracle_uf_labels_u32.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                             ctypes.c_void_p]
        lib.oracle_uf_labels_u64.restype = ctypes.c_int64
        lib.oracle_uf_labels_u64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                             ctypes.c_void_p]
        _lib = lib
    return _lib


def uf_labels(n: int, edges: np.ndarray) -> np.ndarray:
    """label[v] = min vertex id connected to v, for ids in [0, n) (SURVEY.md §8(c) C2:
    ids touched by no edge are singleton components labelled by themselves)."""
    e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
    lab = np.empty(n, dtype=np.uint32)
    rc = _L().oracle_uf_labels_u32(n, e.ctypes.data, e.shape[0], lab.ctypes.data)
    if rc < 0:
        raise ValueError("edge id out of range [0, n)")
    return lab


def uf_labels_u64(edges: np.ndarray):
    """u64 mode: V = ids that appear in the edge list.  Returns
    (sorted distinct ids, label of each) with label = min id of the component."""
    e = np.ascontiguousarray(edges, dtype=np.uint64).reshape(-1, 2)
    ids = np.empty(2 * e.shape[0], dtype=np.uint64)
    lab = np.empty(2 * e.shape[0], dtype=np.uint64)
    nv = _L().oracle_uf_labels_u64(e.ctypes.data, e.shape[0], ids.ctypes.data, lab.ctypes.data)
    if nv < 0:
        raise ValueError("too many distinct ids")
    return ids[:nv].copy(), lab[:nv].copy()


def relabel_u64(edges: np.ndarray):
    """Alg. 2 line 4 relabel to [0,|V|): 'after the first sort, we perform a
    parallel prefix (scan) operation to label the source vertices with a unique id'
    (PAPER.md:277).  Dense id = rank of the original id among the sorted distinct ids
    (order preserving).  Returns (dense edges uint32, sorted distinct ids)."""
    e = np.asarray(edges, dtype=np.uint64).reshape(-1, 2)
    ids = np.unique(e)
    dense = np.searchsorted(ids, e).astype(np.uint32)
    return dense, ids


def components_from_labels(labels: np.ndarray) -> int:
    return int(np.count_nonzero(labels == np.arange(labels.shape[0], dtype=labels.dtype)))


def component_size_histogram(labels: np.ndarray) -> dict:
    """{component size: number of components of that size} from min-id labels (the
    north-star invariant 'component-size histogram'; a component = the ids sharing a label,
    PAPER.md:28)."""
    lab = np.asarray(labels, dtype=np.int64)
    if lab.shape[0] == 0:
        return {}
    _, sizes = np.unique(lab, return_counts=True)
    s, c = np.unique(sizes, return_counts=True)
    return {int(a): int(b) for a, b in zip(s, c)}
