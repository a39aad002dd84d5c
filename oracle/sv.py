"""Alg. 1 of arXiv 1607.06156 ("Connected components labeling"),
transcribed step by step, with the completed-partition exclusion of §3.1.4
(sec:distSVOpt1).  TEST INFRASTRUCTURE (see oracle/__init__.py).

Notation follows Fig. 1a (tab:symbols): a tuple is <p, q, r>
(partition, candidate, vertex); A_i the tuple array; P_i the distinct partitions;
PB_i(p) / VB_i(u) the partition / vertex buckets; C_i(p) the candidates of p;
M_i(u) the partitions in VB_i(u).

Two transcriptions of the same algorithm:

* :func:`sv_literal` -- pure Python on lists of tuples, for tiny graphs; the loop
  body reads line by line against Alg. 1.
* :func:`sv_trace`   -- the same steps with numpy arrays (``argsort`` as the sort,
  ``minimum.reduceat`` as the bucket scan) for larger graphs.

Both return (labels, trace); ``trace`` is a list of per-iteration dicts with the
counters of SURVEY.md §8(c) "Trace oracle":
  A        non-temporary tuples entering the iteration
  P        |P_i| = distinct p among them at the first partition pass (before relabel)
  T        temporary tuples appended (one per surviving partition bucket, C5)
  completed partitions whose tuples are all "potentially completed"
  changed  #{p in P_i : p_min(p) != p} at the first partition pass
  changed2 the same count over the distinct p of the second partition pass

Readings: vertex tuples <x,_,x> only for ids touched by an edge (C2);
completed partitions leave immediately after the first partition pass (C4,
``exclusion="early"``), or after the iteration (``"end"``, the paper's timing), or
never (``"none"``, the fig:loadbal 'Naive' variant, looping on the converged flag of
P:142-163).  ``exclusion="stable"`` implements the UNSAFE reading 'drop partitions
with p_min = p' (C3) and exists only so tests can show it is wrong.
"""
from __future__ import annotations

import numpy as np

INF = np.iinfo(np.int64).max


# --------------------------------------------------------------------------------------
# literal pure-Python transcription (tiny graphs)
# --------------------------------------------------------------------------------------
def sv_literal(n, edges, exclusion="early", max_iter=None):
    edges = [(int(a), int(b)) for a, b in edges]
    present = sorted({x for e in edges for x in e})
    # Alg.1 lines 1-3: A_0 = [<x,_,x> for x in V] + [<x,_,y>, <y,_,x> for {x,y} in E]
    # tuple = [p, q, r, is_vertex_tuple, is_tmp]
    A = [[x, None, x, True, False] for x in present]
    for x, y in edges:
        A.append([x, None, y, False, False])
        A.append([y, None, x, False, False])
    labels = list(range(n))
    trace = []
    it = 0
    if max_iter is None:
        max_iter = 4 * (max(n, 2).bit_length() + 8)
    converged = False
    while A and not converged:
        it += 1
        if it > max_iter:
            raise RuntimeError("no convergence")
        converged = True                                   # line 6 (alg:loopFirstLine)
        rec = dict(A=len(A))
        # line 8 (alg:sort1): sort A_i by third element; lines 9-13: vertex buckets
        A.sort(key=lambda t: t[2])
        pc = {}
        for u in {t[2] for t in A}:
            M_u = [t[0] for t in A if t[2] == u]           # M_i(u)
            u_min = min(M_u)
            for t in A:
                if t[2] == u:
                    t[1] = u_min                           # <p, u_min, r>
            pc[u] = len(set(M_u)) == 1                     # 'potentially completed'
        # line 14 (alg:sort2): sort by first element; lines 15-21: partition buckets
        A.sort(key=lambda t: t[0])
        P_i = sorted({t[0] for t in A})
        rec["P"] = len(P_i)
        p_min_of, completed = {}, set()
        changed = 0
        for p in P_i:
            PB = [t for t in A if t[0] == p]
            p_min = min(t[1] for t in PB)                  # p_min = min C_i(p)
            if p != p_min:                                 # line 17 (alg:convergence)
                converged = False
                changed += 1
            p_min_of[p] = p_min
            if all(pc[t[2]] for t in PB):                  # completed
                completed.add(p)
        rec["changed"] = changed
        rec["completed"] = len(completed)
        if exclusion == "stable":
            dropset = {p for p in P_i if p_min_of[p] == p}
        elif exclusion == "early":
            dropset = completed
        else:
            dropset = set()
        if dropset:
            for t in A:
                if t[0] in dropset and t[3]:
                    labels[t[2]] = t[0]
            A = [t for t in A if t[0] not in dropset]
        for t in A:                                        # line 20: p <- p_min
            t[0] = p_min_of[t[0]]
        # line 22 (alg:appendTuples): one temporary tuple per partition bucket
        temps = [p_min_of[p] for p in P_i if p not in dropset]
        for pm in temps:
            A.append([pm, None, pm, False, True])
        rec["T"] = len(temps)
        # line 24 (alg:sort3): redo lines 8-13
        A.sort(key=lambda t: t[2])
        for u in {t[2] for t in A}:
            u_min = min(t[0] for t in A if t[2] == u)
            for t in A:
                if t[2] == u:
                    t[1] = u_min
        # line 25 (alg:sort4): redo lines 14-21
        A.sort(key=lambda t: t[0])
        changed2 = 0
        new_p = {}
        for p in sorted({t[0] for t in A}):
            p_min = min(t[1] for t in A if t[0] == p)
            if p != p_min:
                converged = False
                changed2 += 1
            new_p[p] = p_min
        for t in A:
            t[0] = new_p[t[0]]
        rec["changed2"] = changed2
        # lines 26-28: erase the temporary tuples
        A = [t for t in A if not t[4]]
        if exclusion == "end":
            for t in A:
                if t[0] in completed and t[3]:
                    labels[t[2]] = t[0]
            A = [t for t in A if t[0] not in completed]
        trace.append(rec)
        if exclusion in ("early", "end", "stable"):
            converged = len(A) == 0
    # project the label of u from any tuple <c,_,u>
    for t in A:
        labels[t[2]] = t[0]
    return np.asarray(labels, dtype=np.int64), trace


# --------------------------------------------------------------------------------------
# numpy transcription (same steps; sort = argsort, bucket scan = reduceat)
# --------------------------------------------------------------------------------------
def _buckets(key):
    """Sort by key (line 8 / line 14) and return (order, starts, bucket_of_sorted)."""
    order = np.argsort(key, kind="stable")
    ks = key[order]
    head = np.empty(ks.shape[0], dtype=bool)
    if ks.shape[0]:
        head[0] = True
        head[1:] = ks[1:] != ks[:-1]
    starts = np.flatnonzero(head)
    bucket = np.cumsum(head) - 1
    return order, starts, bucket


def sv_trace(n, edges, exclusion="early", max_iter=None, present=None, doubling=True):
    """``doubling=False`` skips lines 22-28 (no temporaries, no pointer jumping) -- the
    plain iteration of lines 6-21 that the paper says needs O(n) iterations."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if present is None:
        present = np.unique(e)
    x = np.asarray(present, dtype=np.int64)
    # A_0 (Alg.1 lines 1-3)
    p = np.concatenate([x, e[:, 0], e[:, 1]])
    r = np.concatenate([x, e[:, 1], e[:, 0]])
    vt = np.concatenate([np.ones(x.shape[0], bool), np.zeros(2 * e.shape[0], bool)])
    labels = np.arange(n, dtype=np.int64)
    trace = []
    if max_iter is None:
        max_iter = 4 * (max(n, 2).bit_length() + 8) if doubling else 2 * n + 8
    it = 0
    converged = False
    while p.shape[0] and not converged:
        it += 1
        if it > max_iter:
            raise RuntimeError("no convergence")
        rec = dict(A=int(p.shape[0]))
        # --- lines 8-13: sort by r; u_min = min M_i(u); q <- u_min; PC iff |M_i(u)| = 1
        o, st, b = _buckets(r)
        ps = p[o]
        umin = np.minimum.reduceat(ps, st)
        umax = np.maximum.reduceat(ps, st)
        q = np.empty_like(p)
        q[o] = umin[b]
        pc = np.empty(p.shape[0], bool)
        pc[o] = (umin == umax)[b]
        # --- lines 14-21: sort by p; p_min = min C_i(p); completed iff all tuples PC
        o, st, b = _buckets(p)
        pkeys = p[o][st]
        pkeys_pass2 = pkeys
        pmin = np.minimum.reduceat(q[o], st)
        comp = np.logical_and.reduceat(pc[o], st)
        rec["P"] = int(st.shape[0])
        rec["changed"] = int(np.count_nonzero(pmin != pkeys))
        rec["completed"] = int(np.count_nonzero(comp))
        if exclusion == "stable":
            drop_b = pmin == pkeys
        elif exclusion == "early":
            drop_b = comp
        else:
            drop_b = np.zeros_like(comp)
        drop = np.empty(p.shape[0], bool)
        drop[o] = drop_b[b]
        newp = np.empty_like(p)
        newp[o] = pmin[b]
        # labels of vertices in dropped partitions (P:197 projection)
        sel = drop & vt
        labels[r[sel]] = p[sel]
        keep = ~drop
        p, r, vt = newp[keep], r[keep], vt[keep]
        if not doubling:
            rec["T"] = 0
            rec["changed2"] = 0
            trace.append(rec)
            converged = (rec["changed"] == 0) if exclusion == "none" else p.shape[0] == 0
            continue
        # --- line 22: temporaries <p_min,_,p_min>_tmp, one per surviving bucket (C5)
        tmp_ids = pmin[~drop_b]
        rec["T"] = int(tmp_ids.shape[0])
        na = p.shape[0]
        p2 = np.concatenate([p, tmp_ids])
        r2 = np.concatenate([r, tmp_ids])
        # --- line 24: redo lines 8-13 on A_i with temporaries
        o, st, b = _buckets(r2)
        umin = np.minimum.reduceat(p2[o], st)
        q2 = np.empty_like(p2)
        q2[o] = umin[b]
        # --- line 25: redo lines 14-21
        o, st, b = _buckets(p2)
        pkeys = p2[o][st]
        pmin2 = np.minimum.reduceat(q2[o], st)
        rec["changed2"] = int(np.count_nonzero(pmin2 != pkeys))
        newp2 = np.empty_like(p2)
        newp2[o] = pmin2[b]
        # --- lines 26-28: erase temporaries
        p = newp2[:na]
        if exclusion == "end":
            # partitions completed at the first partition pass leave after the
            # iteration ('swapped to the end'); a completed partition is
            # stable and isolated, so passes 3-4 leave its id unchanged
            cmask = np.isin(p, pkeys_pass2[comp])
            sel = cmask & vt
            labels[r[sel]] = p[sel]
            p, r, vt = p[~cmask], r[~cmask], vt[~cmask]
        trace.append(rec)
        if exclusion == "none":
            converged = rec["changed"] == 0 and rec["changed2"] == 0
        else:
            converged = p.shape[0] == 0
    labels[r] = p  # P:197 projection for whatever remains (exclusion="none")
    return labels, trace
