"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Labels are integer results and must be bit-identical to the union-find oracle; the SV
per-iteration counters are order-independent functions of the input and
must equal the Alg. 1 transcription exactly; the gate's floating-point outputs are compared
to the oracle's FP64 within 1e-9 relative (same formula, same precision, different
summation order), and the route decision must be identical.
"""
import itertools
import json
import os

import numpy as np
import pytest

import graphgen
import oracle
from oracle import bfs as obfs
from oracle import degree as odeg
from oracle import sv as osv

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", params=["csr", "csrbfs", "sort", "direct"])
def cc(request):
    """All regroup engines: r-stationary CSR (default), the same with the
    full-CSR prediction and direction-optimising BFS (CC_FLAG_BFS_CSR), the paper's radix
    regroups, and fully direct-addressed buckets; same sets, same counters."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    if request.param == "csrbfs":
        flags = ccmod.CC_FLAG_TRACE | ccmod.CC_FLAG_BFS_CSR
    else:
        flags = ccmod.CC_FLAG_TRACE | ccmod.REGROUP_FLAGS[request.param]
    ctx = ccmod.CC(device=0, flags=flags)
    yield ctx
    ctx.close()


def run(cc, n, edges, mode="auto"):
    e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
    cc.load(e, n)
    rep = cc.run(mode)
    lab = cc.labels().astype(np.int64)
    assert rep["components"] == np.unique(lab).shape[0]  # isolated ids included
    return lab, rep


def trace_of(rep):
    return [dict(A=it["active_in"], P=it["partitions"], T=it["temps"], completed=it["completed"],
                 changed=it["changed"], changed2=it["changed2"]) for it in rep["iters"]]


def norm(tr):
    return [{k: int(r[k]) for k in ("A", "P", "T", "completed", "changed", "changed2")} for r in tr]


# ------------------------------------------------------------------ hand cases + tiny
def test_hand_cases(cc):
    h = json.load(open(os.path.join(ROOT, "tests", "golden", "hand_cases.json")))
    for c in h["cases"]:
        for mode in ("auto", "sv", "bfs+sv"):
            lab, _ = run(cc, c["n"], c["edges"], mode)
            assert lab.tolist() == c["labels"], (c["name"], mode)


def test_fig1b_trace(cc):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "fig1b.json")))
    lab, rep = run(cc, g["n"], g["edges"], "sv")
    assert lab.tolist() == g["labels"]
    assert norm(trace_of(rep)) == g["trace"]


def test_exhaustive_tiny(cc):
    for n in (1, 2, 3, 4):
        pairs = list(itertools.combinations_with_replacement(range(n), 2))
        for mask in range(1 << len(pairs)):
            edges = [pairs[i] for i in range(len(pairs)) if mask >> i & 1]
            want, tr = osv.sv_trace(n, edges)
            lab, rep = run(cc, n, edges, "sv")
            assert np.array_equal(lab, want), edges
            assert norm(trace_of(rep)) == norm(tr), edges


@pytest.mark.parametrize("seed", range(12))
def test_random_small_trace(cc, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 3000))
    m = int(rng.integers(0, 3 * n))
    e = graphgen.er(seed, n, m)
    want, tr = osv.sv_trace(n, e)
    lab, rep = run(cc, n, e, "sv")
    assert np.array_equal(lab, want)
    assert norm(trace_of(rep)) == norm(tr)


def test_regression_trees(cc):
    """SURVEY.md C3 counterexamples to 'drop stable partitions': must label all 0."""
    t1 = [(19, 12), (21, 10), (24, 5), (24, 14), (17, 18), (16, 1), (11, 23), (11, 9), (6, 3),
          (15, 4), (22, 5), (8, 23), (12, 20), (10, 19), (9, 2), (3, 4), (17, 0), (21, 22),
          (15, 18), (7, 13), (6, 7), (13, 16), (1, 14), (20, 8)]
    t2 = [(9, 13), (5, 19), (12, 3), (17, 10), (13, 7), (19, 10), (6, 7), (12, 18), (16, 14),
          (3, 6), (1, 14), (8, 15), (16, 18), (11, 9), (4, 0), (8, 2), (11, 2), (4, 17), (15, 5)]
    for n, t in ((25, t1), (20, t2)):
        lab, _ = run(cc, n, t, "sv")
        assert np.all(lab == 0)


# ------------------------------------------------------------------ edge cases
def test_empty_and_isolated(cc):
    lab, rep = run(cc, 10, np.zeros((0, 2), np.uint32))
    assert lab.tolist() == list(range(10))
    assert rep["sv_iterations"] == 0
    lab, _ = run(cc, 1, [(0, 0)])
    assert lab.tolist() == [0]


def test_range_error(cc):
    import paper_1607_06156_b200 as ccmod
    with pytest.raises(ccmod.CCError) as ei:
        cc.load(np.array([[0, 5]], np.uint32), 5)
    assert ei.value.status == ccmod.CC_ERR_RANGE


@pytest.mark.parametrize("m", [4095, 4096, 4097, 8191, 2 * 4096 * 16 + 3, 100003])
def test_ragged_tiles(cc, m):
    """Tuple counts straddling radix tiles (4096), segment chunks (2048) and pass tiles."""
    n = max(64, m // 3)
    e = graphgen.er(m, n, m)
    want, tr = osv.sv_trace(n, e)
    lab, rep = run(cc, n, e, "sv")
    assert np.array_equal(lab, want)
    assert norm(trace_of(rep)) == norm(tr)


def test_long_path_and_star(cc):
    """Giant buckets spanning many tiles (star hub) and deep pointer jumping (path)."""
    n = 200000
    perm = np.random.default_rng(3).permutation(n).astype(np.uint32)
    path = np.stack([perm[:-1], perm[1:]], 1)
    lab, rep = run(cc, n, path, "sv")
    assert np.all(lab == 0)
    assert rep["sv_iterations"] <= 2 * 18 + 2
    star = np.stack([np.full(n - 1, 7, np.uint32), np.delete(np.arange(n, dtype=np.uint32), 7)], 1)
    for mode in ("sv", "bfs+sv"):
        lab, _ = run(cc, n, star, mode)
        assert np.all(lab == 0)


@pytest.mark.parametrize("seed", [0, 1])
def test_row_lengths_straddle_tiles(cc, seed):
    """Vertex buckets (rows) whose lengths straddle the row-pass tile (2048 tuples) and the
    extension limit (256) land at every offset of a tile edge: short crossing rows are
    finished by the tile holding their head, long ones by the fix-up.  Stars of those sizes,
    joined by random leaf-leaf edges so several iterations run."""
    rng = np.random.default_rng(77 + seed)
    sizes = [1, 2, 3, 7, 31, 32, 33, 254, 255, 256, 257, 258, 1000, 2046, 2047, 2048, 2049,
             2302, 2303, 2304, 2305, 4095, 4096, 4097, 6000]
    sizes = sizes * 3 + list(rng.integers(1, 400, size=200))
    n = int(sum(sizes) + len(sizes) + 1000)
    perm = rng.permutation(n).astype(np.uint32)
    edges, nxt = [], 0
    for s in rng.permutation(np.array(sizes)):
        c = perm[nxt]
        leaves = perm[nxt + 1:nxt + 1 + int(s) - 1]  # row length = degree + 1 = s
        edges.append(np.stack([np.full(leaves.shape[0], c, np.uint32), leaves], 1))
        nxt += int(s)
    used = perm[:nxt]
    joins = rng.choice(used, size=(len(sizes) // 2, 2)).astype(np.uint32)
    e = np.concatenate(edges + [joins]).astype(np.uint32)
    want, tr = osv.sv_trace(n, e)
    lab, rep = run(cc, n, e, "sv")
    assert np.array_equal(lab, want)
    assert norm(trace_of(rep)) == norm(tr)


@pytest.mark.parametrize("graph", ["straddle0", "straddle1", "er", "c1", "path", "rmat12"])
def test_row_collapse_forced(graph, monkeypatch):
    """Row collapse after every iteration from the first, at any size
    (CC_COLLAPSE_FORCE=1): rows straddling collapse tiles (2048) and row-pass tiles, long rows
    (never collapsed), every tile edge.  Labels and every counter of every iteration (A_i =
    live + folded tuples) equal the Alg. 1 transcription, and equal a run with
    CC_FLAG_NO_COLLAPSE."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    rng = np.random.default_rng(5)
    if graph.startswith("straddle"):
        seed = int(graph[-1])
        r2 = np.random.default_rng(91 + seed)
        sizes = [1, 2, 3, 31, 33, 255, 256, 257, 258, 1000, 2046, 2047, 2048, 2049, 2050, 4097] * 3
        sizes += list(r2.integers(1, 300, size=300))
        n = int(sum(sizes) + 500)
        perm = r2.permutation(n).astype(np.uint32)
        parts, nxt = [], 0
        for s_ in r2.permutation(np.array(sizes)):
            parts.append(np.stack([np.full(int(s_) - 1, perm[nxt], np.uint32), perm[nxt + 1:nxt + int(s_)]], 1))
            nxt += int(s_)
        joins = r2.choice(perm[:nxt], size=(len(sizes) // 3, 2)).astype(np.uint32)
        e = np.concatenate(parts + [joins]).astype(np.uint32)
    elif graph == "er":
        n = 30000
        e = graphgen.er(17, n, 24000)
    elif graph == "c1":
        g = graphgen.make("c1")
        n, e = g.n, g.edges
    elif graph == "path":
        n = 100000
        perm = rng.permutation(n).astype(np.uint32)
        e = np.stack([perm[:-1], perm[1:]], 1)
    else:
        g = graphgen.rmat_scale_graph(12)
        n, e = g.n, g.edges
    want, tr = osv.sv_trace(n, e)
    ctx = ccmod.CC(device=0, flags=ccmod.CC_FLAG_TRACE)
    ref = ccmod.CC(device=0, flags=ccmod.CC_FLAG_TRACE | ccmod.CC_FLAG_NO_COLLAPSE)
    try:
        monkeypatch.setenv("CC_COLLAPSE_FORCE", "1")
        for mode in ("sv", "auto"):
            lab, rep = run(ctx, n, e, mode)
            assert np.array_equal(lab, oracle.uf_labels(n, e).astype(np.int64)), mode
            if mode == "sv":
                assert np.array_equal(lab, want)
                assert norm(trace_of(rep)) == norm(tr)
        monkeypatch.delenv("CC_COLLAPSE_FORCE")
        lab2, rep2 = run(ref, n, e, "sv")
        assert np.array_equal(lab2, want)
        assert norm(trace_of(rep2)) == norm(tr)
    finally:
        ctx.close()
        ref.close()


@pytest.mark.parametrize("graph", ["stars", "rmat14", "c1", "c2s"])
def test_pass_a0_pull_vs_push(graph, monkeypatch):
    """Iteration 0's pass A by pull (PA[p] = min over row p's values x of
    u_min(x)) against the push form (CC_PULL0=0) and the oracle: labels and every counter of
    every iteration, on hubs longer than one long-row segment (stars of 300 / 1024 / 1025 /
    5000 leaves with cross links), an R-MAT in mode sv, C1 and a C2 sample."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    if graph == "stars":
        rng = np.random.default_rng(3)
        n, parts, nxt = 20000, [], 0
        perm = rng.permutation(n).astype(np.uint32)
        for k in (300, 1024, 1025, 5000, 2, 1):
            parts.append(np.stack([np.full(k, perm[nxt], np.uint32), perm[nxt + 1:nxt + 1 + k]], 1))
            nxt += k + 1
        parts.append(rng.choice(perm[:nxt], size=(400, 2)).astype(np.uint32))
        e = np.concatenate(parts).astype(np.uint32)
    elif graph == "rmat14":
        g = graphgen.rmat_scale_graph(14)
        n, e = g.n, g.edges
    elif graph == "c1":
        g = graphgen.make("c1")
        n, e = g.n, g.edges
    else:
        g = graphgen.make("c2", 0.02)
        n, e = g.n, g.edges
    want = oracle.uf_labels(n, e).astype(np.int64)
    _, tr = osv.sv_trace(n, e)
    got = {}
    # "w": the pull by id windows of U (CC_PULLW = log2 of the window's ids; 2^9 and 2^11 ids
    # give these graphs 8 to 128 windows, the default 2^24 gives them none)
    # (windows are for the long rows' warps; CC_PULLW_SHORT=1 also windows the short rows' pull)
    for env, win, short in (("1", None, "0"), ("0", None, "0"), ("1", "9", "0"), ("1", "11", "1")):
        monkeypatch.setenv("CC_PULL0", env)
        monkeypatch.setenv("CC_PULLW_SHORT", short)
        if win is None:
            monkeypatch.delenv("CC_PULLW", raising=False)
        else:
            monkeypatch.setenv("CC_PULLW", win)
            env = "w" + win
        ctx = ccmod.CC(device=0, flags=ccmod.CC_FLAG_TRACE)
        try:
            lab, rep = run(ctx, n, e, "sv")
        finally:
            ctx.close()
        assert np.array_equal(lab, want), env
        got[env] = norm(trace_of(rep))
        assert got[env] == norm(tr), env


@pytest.mark.parametrize("exclusion", ["end", "none"])
def test_exclusion_variants_trace(exclusion):
    """The paper's exclusion timings (SURVEY C4, sec:distSVOpt1 P:220-225) and the
    fig:loadbal 'Naive' variant with no exclusion: labels and every per-iteration counter
    equal the Alg. 1 transcription run with the same choice."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    ctx = ccmod.CC(device=0, flags=ccmod.CC_FLAG_TRACE | ccmod.EXCLUSION_FLAGS[exclusion])
    try:
        graphs = [graphgen.er(s, 3000, 2500 + 700 * s) for s in range(4)]
        graphs.append(graphgen.make("c1", 1.0).edges)
        graphs.append(graphgen.make("c3", 0.01).edges)
        for e in graphs:
            n = int(e.max()) + 1 if e.size else 1
            want, tr = osv.sv_trace(n, e, exclusion=exclusion)
            lab, rep = run(ctx, n, e, "sv")
            assert np.array_equal(lab, want)
            assert norm(trace_of(rep)) == norm(tr)
            for it in rep["iters"]:
                assert it["active_min"] == it["active_max"] == it["active_in"]
        with pytest.raises(ccmod.CCError):  # variants are a csr-engine feature
            bad = ccmod.CC(device=0, flags=ccmod.EXCLUSION_FLAGS[exclusion] | ccmod.CC_FLAG_REGROUP_SORT)
            try:
                run(bad, 4, [(0, 1)], "sv")
            finally:
                bad.close()
    finally:
        ctx.close()


# ------------------------------------------------------------------ configs (BASELINE.json)
@pytest.mark.parametrize("cfg,scale", [("c1", 1.0), ("c2", 0.02), ("c3", 0.02)])
def test_config_trace_parity(cc, cfg, scale):
    g = graphgen.make(cfg, scale)
    want, tr = osv.sv_trace(g.n, g.edges)
    lab, rep = run(cc, g.n, g.edges, "sv")
    assert np.array_equal(lab, want)
    assert norm(trace_of(rep)) == norm(tr)


def _golden_trace(cfg):
    """Full-size SV trace written by tests/golden/make_traces.py (oracle.sv.sv_trace only)."""
    p = os.path.join(ROOT, "tests", "golden", f"trace_{cfg}.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    g = graphgen.make(cfg)
    assert (d["n"], d["m"]) == (g.n, g.m), "golden trace was written for another graph"
    return d["trace"]


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_config_full_labels(cc, cfg):
    """Full BASELINE.json sizes, the launch configuration bench.py times (mode=auto), plus
    the two hard-coded routes of fig:dynamic: labels bit-exact in every mode, the
    mode=sv trace equal to the oracle's full-size golden trace counter by counter, and the
    forced BFS (root, visited set size, levels, remainder) equal to oracle.bfs."""
    g = graphgen.make(cfg)
    want = oracle.uf_labels(g.n, g.edges).astype(np.int64)
    golden = _golden_trace(cfg)
    assert golden is not None or cfg != "c1"
    deg, _ = odeg.degree_distribution(g.n, g.edges)
    root = obfs.bfs_root(deg)
    vis, levels = obfs.bfs(g.n, g.edges, root)
    for mode in ("auto", "sv", "bfs+sv"):
        lab, rep = run(cc, g.n, g.edges, mode)
        assert np.array_equal(lab, want), mode
        assert oracle.component_size_histogram(lab) == oracle.component_size_histogram(want)
        if mode == "auto":
            assert rep["ran_bfs"] == 0  # bounded-degree configs: the gate says SV
        if mode == "sv" and golden is not None:
            assert norm(trace_of(rep)) == norm(golden), mode
        if mode == "bfs+sv":
            assert rep["ran_bfs"] == 1
            assert rep["bfs_root"] == root
            assert rep["bfs_visited"] == int(vis.sum())
            assert rep["bfs_levels"] == levels
            assert rep["remainder_edges"] == int(obfs.filter_edges(g.edges, vis).shape[0])
        # trace invariants at any size (C5): T = P - completed; A non-increasing
        its = rep["iters"]
        for i, it in enumerate(its):
            assert it["temps"] == it["partitions"] - it["completed"]
            if i:
                assert it["active_in"] <= its[i - 1]["active_in"]
        assert not its or its[-1]["changed"] == 0


@pytest.mark.parametrize("graph", ["c1", "c2s", "rmat14", "rmat18"])
@pytest.mark.parametrize("tau", [0.05, 0.2, 1.0])
def test_gate_ks_decision(graph, tau):
    """CC_FLAG_GATE_KS: the route is the paper's K-S < tau decision,
    identical to the oracle's (oracle.hybrid with gate='ks'); labels bit-exact."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    if graph == "c1":
        g = graphgen.make("c1")
    elif graph == "c2s":
        g = graphgen.make("c2", 0.05)
    else:
        g = graphgen.rmat_scale_graph(int(graph[4:]))
    _, hist = odeg.degree_distribution(g.n, g.edges)
    ks = odeg.ks_powerlaw(hist)
    if ks["ks"] == ks["ks"]:
        assert abs(ks["ks"] - tau) > 1e-6, "tau too close to the statistic for a stable decision"
    want_bfs = bool(ks["ks"] == ks["ks"] and ks["ks"] < tau)
    ctx = ccmod.CC(device=0, flags=ccmod.CC_FLAG_GATE_KS, tau=tau)
    try:
        lab, rep = run(ctx, g.n, g.edges, "auto")
    finally:
        ctx.close()
    assert bool(rep["ran_bfs"]) == want_bfs
    assert np.array_equal(lab, oracle.uf_labels(g.n, g.edges).astype(np.int64))
    if graph == "rmat18" and tau == 0.05:
        assert not want_bfs  # K-S does not call the synthetic R-MAT a power law


def test_rmat_bfs_route(cc):
    g = graphgen.rmat_scale_graph(18)
    want = oracle.uf_labels(g.n, g.edges).astype(np.int64)
    deg, hist = odeg.degree_distribution(g.n, g.edges)
    root = obfs.bfs_root(deg)
    vis, levels = obfs.bfs(g.n, g.edges, root)
    for mode in ("auto", "bfs+sv", "sv"):
        lab, rep = run(cc, g.n, g.edges, mode)
        assert np.array_equal(lab, want), mode
        if mode != "sv":
            assert rep["ran_bfs"] == 1
            assert rep["bfs_root"] == root
            assert rep["bfs_visited"] == int(vis.sum())
            assert rep["bfs_levels"] == levels
            rem = obfs.filter_edges(g.edges, vis)
            assert rep["remainder_edges"] == rem.shape[0]
            # SV trace on the remainder equals the oracle's
            _, tr = osv.sv_trace(g.n, rem)
            assert norm(trace_of(rep)) == norm(tr)


def _peel_graph(seed, n, hub, small):
    """A star-like giant component on `hub` random ids (the BFS peel) plus `small` small
    components (paths, cycles, trees with a duplicate edge and a self-loop) on other ids spread
    over [0, n), ids 0 and n-1 included: the remainder touches a small fraction of the ids."""
    rng = np.random.default_rng(seed)
    ids = rng.permutation(n)
    root, H = ids[1], ids[2:2 + hub]
    e = [np.stack([np.full(hub, root), H], 1), np.stack([H, rng.choice(H, hub)], 1)]
    rest = np.concatenate([[0, n - 1], ids[2 + hub:]])
    pos = 0
    for k in range(small):
        sz = 2 + (k % 7)
        vs = rest[pos:pos + sz]
        pos += sz
        kind = k % 4
        if kind == 0:  # path
            e.append(np.stack([vs[:-1], vs[1:]], 1))
        elif kind == 1:  # cycle
            e.append(np.stack([vs, np.roll(vs, 1)], 1))
        elif kind == 2:  # random tree + duplicate edge + self-loop
            par = [vs[rng.integers(0, i)] for i in range(1, sz)]
            t = np.stack([vs[1:], par], 1)
            e.append(np.concatenate([t, t[:1], [[vs[0], vs[0]]]]))
        else:  # star
            e.append(np.stack([np.full(sz - 1, vs[-1]), vs[:-1]], 1))
    edges = np.concatenate(e).astype(np.uint32)
    return edges[rng.permutation(edges.shape[0])]


@pytest.mark.parametrize("seed,n,hub,small", [(0, 1 << 16, 4000, 200), (1, 1 << 20, 60000, 3000),
                                              (2, (1 << 22) + 37, 200000, 9000)])
def test_renumbered_remainder(cc, request, seed, n, hub, small):
    """BFS route with a small remainder: the SV runs on the remainder's endpoints renumbered
    densely in id order.  Labels, the SV trace (Alg. 1 counters, which the
    monotone renumbering must not change) and n' equal the oracle's, and equal the ablation
    that keeps the original id range (CC_FLAG_NO_RENUMBER)."""
    import paper_1607_06156_b200 as ccmod
    edges = _peel_graph(seed, n, hub, small)
    want = oracle.uf_labels(n, edges).astype(np.int64)
    deg, _ = odeg.degree_distribution(n, edges)
    vis, _ = obfs.bfs(n, edges, obfs.bfs_root(deg))
    rem = obfs.filter_edges(edges, vis)
    _, tr = osv.sv_trace(n, rem)
    lab, rep = run(cc, n, edges, "bfs+sv")
    assert np.array_equal(lab, want)
    assert rep["remainder_edges"] == rem.shape[0]
    assert norm(trace_of(rep)) == norm(tr)
    # the edge-streaming BFS route renumbers (csrbfs peels on its CSR rows and keeps n)
    assert rep["sv_ids"] in (n, np.unique(rem).shape[0])
    if request.node.callspec.params["cc"] != "csrbfs":
        assert rep["sv_ids"] == np.unique(rem).shape[0]
    ab = ccmod.CC(device=0, flags=ccmod.CC_FLAG_TRACE | ccmod.CC_FLAG_NO_RENUMBER)
    try:
        lab2, rep2 = run(ab, n, edges, "bfs+sv")
    finally:
        ab.close()
    assert np.array_equal(lab2, want)
    assert rep2["sv_ids"] == n
    assert norm(trace_of(rep2)) == norm(tr)


# ------------------------------------------------------------------ prediction / gate
@pytest.mark.parametrize("graph", ["c1", "c2s", "rmat14", "rmat18"])
def test_gate_parity(cc, graph):
    if graph == "c1":
        g = graphgen.make("c1")
    elif graph == "c2s":
        g = graphgen.make("c2", 0.05)
    else:
        g = graphgen.rmat_scale_graph(int(graph[4:]))
    _, hist = odeg.degree_distribution(g.n, g.edges)
    gl = odeg.gate_ls(hist)
    ks = odeg.ks_powerlaw(hist)
    lab, rep = run(cc, g.n, g.edges, "auto")
    assert rep["max_degree"] == gl["dmax"]
    assert rep["n_present"] == int(hist.sum())
    assert rep["ran_bfs"] == int(gl["scale_free"])
    if np.isnan(gl["alpha"]):
        assert np.isnan(rep["ls_alpha"])
    else:
        assert rep["ls_alpha"] == pytest.approx(gl["alpha"], rel=1e-9)
        assert rep["ls_r2"] == pytest.approx(gl["r2"], rel=1e-9)
    if np.isnan(ks["ks"]):
        assert np.isnan(rep["ks_stat"])
    else:
        assert rep["ks_xmin"] == ks["xmin"]
        assert rep["ks_alpha"] == pytest.approx(ks["alpha"], rel=1e-9)
        assert rep["ks_stat"] == pytest.approx(ks["ks"], rel=1e-7, abs=1e-9)


def test_device_input_and_output(cc):
    import torch
    g = graphgen.make("c1", 0.5)
    want = oracle.uf_labels(g.n, g.edges)
    t = torch.from_numpy(g.edges.view(np.int32)).cuda()
    cc.load(t, g.n)
    cc.run("auto")
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    cc.labels(out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)


def test_config_c4_full(cc, request):
    """C4 (R-MAT scale 26, 1.07 B edges) at full size through the BFS route: labels
    bit-identical to union-find; the peeled component is exactly the root's component."""
    if "[csr]" not in request.node.name:
        pytest.skip("full-size C4 runs once, with the default engine")
    g = graphgen.make("c4")
    want = oracle.uf_labels(g.n, g.edges)
    cc.load(g.edges, g.n)
    rep = cc.run("auto")
    lab = cc.labels()
    assert rep["ran_bfs"] == 1
    assert np.array_equal(lab, want)
    root = rep["bfs_root"]
    assert rep["bfs_visited"] == int(np.count_nonzero(want == want[root]))
    assert rep["max_degree"] == int(np.bincount(g.edges.reshape(-1), minlength=g.n).max())
    # the hard-coded SV route (fig:dynamic 'never BFS') on 2.18 G tuples, whose
    # 67 M-slot partition arrays exceed L2: labels bit-identical, trace invariants
    rep = cc.run("sv")
    assert rep["ran_bfs"] == 0
    assert np.array_equal(cc.labels(), want)
    assert oracle.component_size_histogram(cc.labels()) == oracle.component_size_histogram(want)
    its = rep["iters"]
    assert its[0]["active_in"] == 2 * g.m + int(np.count_nonzero(np.bincount(g.edges.reshape(-1), minlength=g.n)))
    for i, it in enumerate(its):
        assert it["temps"] == it["partitions"] - it["completed"]
        if i:
            assert it["active_in"] <= its[i - 1]["active_in"]


def test_degree_counts_large_id_range(cc, request):
    """n = 2^25 (> the 2^24-id L2 window: the degree count streams the edges once per
    window); the degree statistics and gate equal the oracle's (numpy bincount of the arc
    sources) and the labels the union-find's."""
    if "[csr]" not in request.node.name:
        pytest.skip("prediction is shared by the engines: once")
    e = graphgen.rmat(graphgen.BASE_SEED + 25, 25, 2)
    e = np.concatenate([e, np.array([[7, 7], [7, 7], [2**25 - 1, 3]], np.uint32)])
    n = 1 << 25
    deg, hist = odeg.degree_distribution(n, e)
    gl = odeg.gate_ls(hist)
    lab, rep = run(cc, n, e, "auto")
    assert rep["max_degree"] == int(deg.max())
    assert rep["n_present"] == int(np.count_nonzero(deg))
    assert rep["ls_alpha"] == pytest.approx(gl["alpha"], rel=1e-9)
    assert rep["ls_r2"] == pytest.approx(gl["r2"], rel=1e-9)
    assert rep["ran_bfs"] == int(gl["scale_free"])
    assert np.array_equal(lab, oracle.uf_labels(n, e).astype(np.int64))


# ------------------------------------------------------------------ u64 ids (relabel)
def _u64_graph(seed, nv, m):
    rng = np.random.default_rng(seed)
    table = np.unique(rng.integers(0, 2**64 - 1, size=nv, dtype=np.uint64, endpoint=True))
    table = np.concatenate([table, np.array([0, 2**64 - 1], dtype=np.uint64)])
    idx = rng.integers(0, table.shape[0], size=(m, 2))
    return table[idx]


@pytest.mark.parametrize("seed,nv,m", [(1, 50, 40), (2, 3000, 5000), (3, 200000, 300000)])
def test_u64_ids(cc, seed, nv, m):
    """u64 ids are relabelled in id order (Alg. 2 line 4): labels are the min original id
    of each component, bit-identical to the oracle; the SV trace runs on the dense ids."""
    e = _u64_graph(seed, nv, m)
    ids_o, lab_o = oracle.uf_labels_u64(e)
    cc.load(e, 0, ids="u64")
    rep = cc.run("sv")
    ids, lab = cc.labels_u64()
    assert np.array_equal(ids, ids_o)
    assert np.array_equal(lab, lab_o)
    dense, uniq = oracle.relabel_u64(e)
    _, tr = osv.sv_trace(uniq.shape[0], dense)
    assert norm(trace_of(rep)) == norm(tr)
    rep = cc.run("auto")
    ids, lab = cc.labels_u64()
    assert np.array_equal(lab, lab_o)


@pytest.mark.parametrize("kind", ["matching", "path", "star_dups"])
def test_u64_relabel_table_sizes(cc, request, kind):
    """The hash relabel starts with a table for ~m/2 distinct ids and redoes
    the insertion at full size on a long probe run: a perfect matching (every id distinct,
    2m of them) and a long path (m + 1 distinct) force the retry; a star with repeated edges
    stays in the small table.  Labels equal the u64 oracle's either way."""
    if "[csr-" not in request.node.name:
        pytest.skip("relabel is engine-independent")
    rng = np.random.default_rng(17)
    if kind == "matching":
        ids = np.unique(rng.integers(0, 2**64 - 1, size=400_000, dtype=np.uint64, endpoint=True))
        ids = rng.permutation(ids)[: (ids.shape[0] // 2) * 2]
        e = ids.reshape(-1, 2)
    elif kind == "path":
        ids = rng.permutation(np.unique(rng.integers(0, 2**63, size=300_000, dtype=np.uint64)))
        e = np.stack([ids[:-1], ids[1:]], 1)
        e = e[rng.permutation(e.shape[0])]
    else:
        leaves = rng.integers(1, 2**40, size=5000, dtype=np.uint64)
        e = np.stack([np.full(200_000, 2**64 - 1, np.uint64), leaves[rng.integers(0, 5000, 200_000)]], 1)
    ids_o, lab_o = oracle.uf_labels_u64(e)
    cc.load(e, 0, ids="u64")
    rep = cc.run("auto")
    ids, lab = cc.labels_u64()
    assert np.array_equal(ids, ids_o)
    assert np.array_equal(lab, lab_o)
    assert rep["n_present"] == ids_o.shape[0]


@pytest.mark.parametrize("scale", [1 / 4096, 1 / 256])
def test_config_c5_scaled(cc, request, scale):
    """C5 structure (R-MAT U geometric paths, u64 ids = mix64 of dense indices, scrambled
    edge order) at reduced scale on one GPU: the full config needs 8 GPUs.
    u64 relabel -> gate (BFS route) -> BFS peel -> SV on the path remainder; labels
    bit-identical to the u64 union-find oracle."""
    if "[csr" not in request.node.name and scale < 1 / 1024:
        pytest.skip("one small case for the other engines")
    g = graphgen.make("c5", scale)
    ids_o, lab_o = oracle.uf_labels_u64(g.edges)
    cc.load(g.edges, 0, ids="u64")
    rep = cc.run("auto")
    ids, lab = cc.labels_u64()
    assert np.array_equal(ids, ids_o)
    assert np.array_equal(lab, lab_o)
    assert rep["ran_bfs"] == 1
    assert rep["n_present"] == ids_o.shape[0]


def _mix64_ref(x):
    """Independent transcription of the 64-bit integer mix named by PAPER.md:320 (test side)."""
    M = (1 << 64) - 1
    k = int(x)
    k = ((~k) + (k << 21)) & M
    k ^= k >> 24
    k = (k + (k << 3) + (k << 8)) & M
    k ^= k >> 14
    k = (k + (k << 2) + (k << 4)) & M
    k ^= k >> 28
    k = (k + (k << 31)) & M
    return k


@pytest.mark.parametrize("seed,nv,m", [(4, 40, 60), (5, 20000, 30000)])
def test_permute_ids(seed, nv, m):
    """CC_FLAG_PERMUTE_IDS: SV runs on the ids ordered by their 64-bit mix, the
    labels come back as each component's minimum ORIGINAL id (C1); the trace equals the
    transcription run on the permuted dense ids."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    e = _u64_graph(seed, nv, m)
    ids_o, lab_o = oracle.uf_labels_u64(e)
    dense, uniq = oracle.relabel_u64(e)
    mixed = np.array([_mix64_ref(x) for x in uniq], dtype=np.uint64)
    pi = np.empty(uniq.shape[0], dtype=np.int64)
    pi[np.argsort(mixed, kind="stable")] = np.arange(uniq.shape[0])
    _, tr = osv.sv_trace(uniq.shape[0], pi[dense])
    ctx = ccmod.CC(device=0, flags=ccmod.CC_FLAG_TRACE | ccmod.CC_FLAG_PERMUTE_IDS)
    try:
        ctx.load(e, 0, ids="u64")
        for mode in ("sv", "auto"):
            rep = ctx.run(mode)
            ids, lab = ctx.labels_u64()
            assert np.array_equal(ids, ids_o)
            assert np.array_equal(lab, lab_o), mode
            if mode == "sv":
                assert norm(trace_of(rep)) == norm(tr)
    finally:
        ctx.close()


def test_bfs_eccentricity():
    """BFS depth from seeds (the paper's approximate diameter) equals the
    oracle's level count; on an ordered path the depth from an end is the path length."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    ctx = ccmod.CC(device=0)
    try:
        for g in (graphgen.make("c3", 0.01), graphgen.rmat_scale_graph(14), graphgen.make("c2", 0.01)):
            rng = np.random.default_rng(3)
            seeds = rng.integers(0, g.n, size=6).astype(np.uint64)
            ctx.load(g.edges, g.n)
            got = ctx.eccentricity(seeds)
            wants = []
            for s, lev in zip(seeds, got):
                _, want = obfs.bfs(g.n, g.edges, int(s))
                assert int(lev) == want
                wants.append(want)
            # the approximate diameter over the same seeds (taken in the library)
            assert ccmod.cc_approx_diameter(ctx.ctx, seeds) == max(wants)
        path = np.stack([np.arange(999), np.arange(1, 1000)], 1).astype(np.uint32)
        ctx.load(path, 1000)
        assert ctx.eccentricity(np.array([0, 500, 999], np.uint64)).tolist() == [999, 500, 999]
        assert ccmod.cc_approx_diameter(ctx.ctx, np.array([3, 500], np.uint64)) == 996
        assert ccmod.cc_approx_diameter(ctx.ctx, np.zeros(0, np.uint64)) == 0
        assert 500 <= ccmod.approx_diameter(ctx.ctx, 1000, runs=20, seed=1) <= 999
    finally:
        ctx.close()


def test_u64_mode_errors(cc):
    import paper_1607_06156_b200 as ccmod
    e = _u64_graph(9, 10, 5)
    cc.load(e, 0, ids="u64")
    cc.run("auto")
    with pytest.raises(ccmod.CCError):
        cc.labels()  # u32 labels of a u64 graph
    with pytest.raises(ccmod.CCError):
        cc.load(e, 7, ids="u64")  # n_vertices must be 0


@pytest.mark.parametrize("n,bits", [(1, 64), (4097, 64), (100003, 40), (300000, 17)])
def test_radix_sort_pairs(n, bits):
    """The onesweep regroup primitive through the ABI: stable sort by the low `bits` bits,
    payload carried (checked against numpy's stable argsort)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    rng = np.random.default_rng(n)
    k = rng.integers(0, 2**63, size=n, dtype=np.int64) * 2 + rng.integers(0, 2, size=n)
    if bits < 64:  # the ABI sorts keys < 2^key_bits
        k = (k.view(np.uint64) & np.uint64((1 << bits) - 1)).view(np.int64)
    key = k.view(np.uint64)
    order = np.argsort(key, kind="stable")
    dk = torch.from_numpy(k).cuda()
    dv = torch.arange(n, dtype=torch.int32, device="cuda")
    ccmod.cc_radix_sort_pairs(dk, dv, torch.empty_like(dk), torch.empty_like(dv), bits)
    assert np.array_equal(dv.cpu().numpy(), order.astype(np.int32))
    assert np.array_equal(dk.cpu().numpy(), k[order])
