"""Pins for the CPU oracle (runs without a GPU).

Each oracle function is checked against something other than itself: brute-force DFS on
every tiny graph, hand-derived values from the paper's worked example (tests/golden/),
closed forms, invariants, and library routines on special cases.
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

import graphgen
import oracle
from oracle import bfs as obfs
from oracle import degree as odeg
from oracle import hybrid as ohyb
from oracle import sv as osv


# ------------------------------------------------------------------ independent checkers
def dfs_min_labels(n, edges):
    """Brute force: explicit DFS per vertex, label = min id reached."""
    adj = [[] for _ in range(n)]
    for a, b in edges:
        adj[a].append(b)
        adj[b].append(a)
    lab = [None] * n
    for s in range(n):
        if lab[s] is not None:
            continue
        stack, comp, seen = [s], [], {s}
        while stack:
            x = stack.pop()
            comp.append(x)
            for y in adj[x]:
                if y not in seen:
                    seen.add(y)
                    stack.append(y)
        mn = min(comp)
        for x in comp:
            lab[x] = mn
    return np.array(lab, dtype=np.int64)


def scipy_min_labels(n, edges):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    g = sp.coo_matrix((np.ones(e.shape[0]), (e[:, 0], e[:, 1])), shape=(n, n))
    nc, comp = connected_components(g, directed=False)
    mins = np.full(nc, n, dtype=np.int64)
    np.minimum.at(mins, comp, np.arange(n))
    return mins[comp], nc


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ union-find labels
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_uf_exhaustive_tiny(n):
    pairs = list(itertools.combinations(range(n), 2))
    for mask in range(1 << len(pairs)):
        edges = [pairs[i] for i in range(len(pairs)) if mask >> i & 1]
        want = dfs_min_labels(n, edges)
        got = oracle.uf_labels(n, np.array(edges, dtype=np.uint32).reshape(-1, 2))
        assert np.array_equal(got, want), edges


def test_uf_hand_cases(golden_dir):
    for c in load(golden_dir, "hand_cases.json")["cases"]:
        got = oracle.uf_labels(c["n"], np.array(c["edges"], dtype=np.uint32).reshape(-1, 2))
        assert got.tolist() == c["labels"], c["name"]


def test_uf_fig1b(golden_dir):
    g = load(golden_dir, "fig1b.json")
    got = oracle.uf_labels(g["n"], np.array(g["edges"], dtype=np.uint32))
    assert got.tolist() == g["labels"]


@pytest.mark.parametrize("seed", range(6))
def test_uf_vs_scipy_and_invariants(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    m = int(rng.integers(0, 2 * n))
    e = graphgen.er(seed, n, m)
    lab = oracle.uf_labels(n, e).astype(np.int64)
    want, nc = scipy_min_labels(n, e)
    assert np.array_equal(lab, want)
    # invariants: equal across every edge, label <= v, idempotent, #components
    if m:
        assert np.all(lab[e[:, 0]] == lab[e[:, 1]])
    assert np.all(lab <= np.arange(n))
    assert np.array_equal(lab[lab], lab)
    assert oracle.components_from_labels(lab) == nc


@pytest.mark.parametrize("seed", range(4))
def test_uf_component_size_histogram_vs_scipy(seed):
    """Component-size histogram (north-star invariant) against scipy's component sizes."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(100, 5000))
    e = graphgen.er(seed + 11, n, int(rng.integers(0, n)))
    h = oracle.component_size_histogram(oracle.uf_labels(n, e))
    g = sp.coo_matrix((np.ones(e.shape[0]), (e[:, 0].astype(np.int64), e[:, 1].astype(np.int64))),
                      shape=(n, n))
    _, comp = connected_components(g, directed=False)
    s, c = np.unique(np.bincount(comp), return_counts=True)
    assert h == {int(a): int(b) for a, b in zip(s, c)}
    assert sum(k * v for k, v in h.items()) == n


def test_uf_component_size_histogram_closed_form():
    """Closed forms: disjoint cliques of sizes 1..12 (each size three times), paths of
    lengths 1..40 and a star, ids scrambled by a random permutation; the histogram is known
    by construction, independent of any labelling."""
    rng = np.random.default_rng(7)
    sizes, edges, base = [], [], 0
    for k in list(range(1, 13)) * 3:
        edges += [(base + a, base + b) for a, b in itertools.combinations(range(k), 2)]
        sizes.append(k)
        base += k
    for k in range(1, 41):
        edges += [(base + i, base + i + 1) for i in range(k - 1)]
        sizes.append(k)
        base += k
    edges += [(base, base + i) for i in range(1, 500)]
    sizes.append(500)
    base += 500
    perm = rng.permutation(base)
    e = perm[np.array(edges, dtype=np.int64)].astype(np.uint32)
    e = e[rng.permutation(e.shape[0])]
    want = {}
    for k in sizes:
        want[k] = want.get(k, 0) + 1
    assert oracle.component_size_histogram(oracle.uf_labels(base, e)) == want


def test_uf_rejects_out_of_range():
    with pytest.raises(ValueError):
        oracle.uf_labels(3, np.array([[0, 3]], dtype=np.uint32))


def test_uf_u64_matches_relabel():
    rng = np.random.default_rng(5)
    ids = rng.integers(0, 2**63, size=400, dtype=np.uint64)
    e = ids[rng.integers(0, 400, size=(600, 2))]
    ids_out, lab = oracle.uf_labels_u64(e)
    dense, uniq = oracle.relabel_u64(e)
    assert np.array_equal(ids_out, uniq)
    lab_dense = oracle.uf_labels(uniq.shape[0], dense)
    assert np.array_equal(lab, uniq[lab_dense])
    # order preserving and bijective
    assert np.all(np.diff(uniq.astype(np.float64)) > 0)
    assert np.array_equal(uniq[dense], e)


# ------------------------------------------------------------------ Alg. 1 transcription
def test_sv_fig1b_trace(golden_dir):
    g = load(golden_dir, "fig1b.json")
    for fn in (osv.sv_literal, osv.sv_trace):
        lab, tr = fn(g["n"], g["edges"])
        assert lab.tolist() == g["labels"]
        assert tr == g["trace"]


def test_sv_path4_trace(golden_dir):
    g = load(golden_dir, "path4.json")
    for fn in (osv.sv_literal, osv.sv_trace):
        lab, tr = fn(g["n"], g["edges"])
        assert lab.tolist() == g["labels"]
        assert tr == g["trace"]


def test_sv_fig1b_sets(golden_dir):
    """VB_0(u), P_0, PB_0(u), N_0(v1) of Fig. 1b from the initial tuple array."""
    g = load(golden_dir, "fig1b.json")
    u, v1 = 5, 2
    e = g["edges"]
    x = sorted({a for ed in e for a in ed})
    A0 = [(a, a) for a in x] + [(a, b) for a, b in e] + [(b, a) for a, b in e]  # (p, r)
    assert sorted(p for p, r in A0 if r == u) == g["VB0_u_partitions"]
    assert sorted({p for p, r in A0}) == g["P0"]
    assert sorted(r for p, r in A0 if p == u) == g["PB0_u_vertices"]
    V_v1 = {r for p, r in A0 if p == v1}
    N = sorted({p for p, r in A0 if r in V_v1})
    assert N == g["N0_v1"]


def test_sv_hand_traces(golden_dir):
    h = load(golden_dir, "hand_cases.json")
    cases = {c["name"]: c for c in h["cases"]}
    for t in h["trace_cases"]:
        c = cases[t["name"]]
        lab, tr = osv.sv_trace(c["n"], c["edges"])
        assert lab.tolist() == c["labels"]
        assert len(tr) == t["iterations"]
        for k, v in t["trace0"].items():
            assert tr[0][k] == v


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_sv_exhaustive_tiny(n):
    pairs = list(itertools.combinations_with_replacement(range(n), 2))
    for mask in range(1 << min(len(pairs), 10)):
        edges = [pairs[i] for i in range(len(pairs)) if mask >> i & 1]
        want = dfs_min_labels(n, edges)
        l1, t1 = osv.sv_literal(n, edges)
        l2, t2 = osv.sv_trace(n, edges)
        assert np.array_equal(l1, want) and np.array_equal(l2, want), edges
        assert t1 == t2


@pytest.mark.parametrize("seed", range(40))
def test_sv_random_vs_dfs_and_variants(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 40))
    m = int(rng.integers(0, 2 * n))
    e = rng.integers(0, n, size=(m, 2))
    want = dfs_min_labels(n, e.tolist())
    lab, tr = osv.sv_trace(n, e)
    assert np.array_equal(lab, want)
    lab_l, tr_l = osv.sv_literal(n, e.tolist())
    assert np.array_equal(lab_l, want) and tr_l == tr
    # C4: early / end-of-iteration / no exclusion give identical labels and iteration counts
    for ex in ("end", "none"):
        l2, t2 = osv.sv_trace(n, e, exclusion=ex)
        assert np.array_equal(l2, want)
        assert len(t2) == len(tr)
    # trace invariants: T = P - completed (C5, early exclusion); A non-increasing;
    # A_{i+1} = A_i minus tuples of completed partitions; last iteration completes all
    for i, r in enumerate(tr):
        assert r["T"] == r["P"] - r["completed"]
        if i:
            assert r["A"] <= tr[i - 1]["A"]
        assert r["changed"] <= r["P"]
    assert tr == [] or tr[-1]["changed"] == 0 and tr[-1]["P"] == tr[-1]["completed"]
    if n >= 2:
        assert len(tr) <= 2 * int(np.ceil(np.log2(n))) + 2  # logarithmic


def test_sv_temp_count_equals_partitions_without_exclusion():
    """'the global count of the temporary tuples equals |P_i| in each iteration'."""
    e = graphgen.er(7, 300, 260)
    _, tr = osv.sv_trace(300, e, exclusion="none")
    for r in tr:
        assert r["T"] == r["P"]


def test_sv_doubling_is_logarithmic():
    """without pointer doubling O(n) iterations, with it logarithmic."""
    for n in (64, 256):
        e = [(i, i + 1) for i in range(n - 1)]
        with_d = len(osv.sv_trace(n, e)[1])
        without = len(osv.sv_trace(n, e, doubling=False)[1])
        assert with_d <= int(np.log2(n)) + 1
        assert without >= n // 2
        lab, _ = osv.sv_trace(n, e, doubling=False)
        assert np.all(lab == 0)


def test_sv_stable_dropping_is_wrong():
    """dropping merely-stable partitions (p_min = p) breaks labels; the
    paper drops *completed* partitions.  Two tree counterexamples."""
    t1 = [(19, 12), (21, 10), (24, 5), (24, 14), (17, 18), (16, 1), (11, 23), (11, 9), (6, 3),
          (15, 4), (22, 5), (8, 23), (12, 20), (10, 19), (9, 2), (3, 4), (17, 0), (21, 22),
          (15, 18), (7, 13), (6, 7), (13, 16), (1, 14), (20, 8)]
    t2 = [(9, 13), (5, 19), (12, 3), (17, 10), (13, 7), (19, 10), (6, 7), (12, 18), (16, 14),
          (3, 6), (1, 14), (8, 15), (16, 18), (11, 9), (4, 0), (8, 2), (11, 2), (4, 17), (15, 5)]
    for n, t in ((25, t1), (20, t2)):
        assert np.all(dfs_min_labels(n, t) == 0)
        good, _ = osv.sv_trace(n, t)
        assert np.all(good == 0)
        bad, _ = osv.sv_trace(n, t, exclusion="stable")
        assert not np.all(bad == 0)


def test_sv_config_analogs_match_uf():
    for cfg, sc in (("c1", 0.05), ("c2", 0.002), ("c3", 0.002)):
        g = graphgen.make(cfg, sc)
        lab, tr = osv.sv_trace(g.n, g.edges)
        assert np.array_equal(lab, oracle.uf_labels(g.n, g.edges))
        assert all(r["T"] == r["P"] - r["completed"] for r in tr)


# ------------------------------------------------------------------ degree distribution
def test_degree_hand_cases(golden_dir):
    for c in load(golden_dir, "degree_cases.json")["cases"]:
        _, h = odeg.degree_distribution(c["n"], np.array(c["edges"]).reshape(-1, 2))
        got = {str(d): int(h[d]) for d in np.flatnonzero(h)}
        assert got == c["hist"], c["name"]


@pytest.mark.parametrize("seed", range(4))
def test_degree_sums_and_bincount(seed):
    g = graphgen.make("c1", 0.1, seed=seed)
    deg, h = odeg.degree_distribution(g.n, g.edges)
    e = g.edges.astype(np.int64)
    # independent count: two bincounts (a self-loop adds to both)
    want = np.bincount(e[:, 0], minlength=g.n) + np.bincount(e[:, 1], minlength=g.n)
    assert np.array_equal(deg, want)
    n_present = np.unique(e).shape[0]
    assert h.sum() == n_present                              # sum D[d] = n_p
    assert int((np.arange(h.shape[0]) * h).sum()) == 2 * g.m  # sum d D[d] = 2m (handshake)


# ------------------------------------------------------------------ gate G (closed form)
@pytest.mark.parametrize("alpha", [1.5, 2.0, 2.5, 3.0])
@pytest.mark.parametrize("dtop", [1000, 10000])
def test_gate_exact_power_law(alpha, dtop):
    d = np.arange(1, dtop + 1, dtype=np.float64)
    h = np.zeros(dtop + 1, dtype=np.int64)
    h[1:] = np.floor(1e12 * d ** (-alpha)).astype(np.int64)
    g = odeg.gate_ls(h)
    assert abs(g["alpha"] - alpha) < 0.02
    assert g["r2"] > 0.999
    assert g["scale_free"] == (alpha < 3.5)


def test_gate_log_bin_edges():
    assert odeg.log_bin_edges(100) == [1, 2, 3, 6, 10, 15, 25, 39, 63, 100, 101]
    assert odeg.log_bin_edges(7) == [1, 2, 3, 6, 8]


def test_gate_constant_degree_is_not_scale_free():
    h = np.zeros(8, dtype=np.int64)
    h[7] = 1000
    assert not odeg.gate_ls(h)["scale_free"]
    h = np.zeros(300, dtype=np.int64)
    h[4] = 10**6
    h[299] = 1
    assert not odeg.gate_ls(h)["scale_free"]  # < 3 non-empty bins


def test_gate_routes_config_analogs():
    """SURVEY.md C11 expected routes: C1-C3 -> SV, R-MAT -> BFS."""
    for cfg, sc in (("c1", 1.0), ("c2", 0.02), ("c3", 0.02)):
        g = graphgen.make(cfg, sc)
        _, h = odeg.degree_distribution(g.n, g.edges)
        assert not odeg.gate_ls(h)["scale_free"], cfg
    g = graphgen.rmat_scale_graph(16)
    _, h = odeg.degree_distribution(g.n, g.edges)
    r = odeg.gate_ls(h)
    assert r["scale_free"] and r["r2"] > 0.8 and 1.5 < r["alpha"] < 2.2


# ------------------------------------------------------------------ K-S statistic
def test_hurwitz_zeta_vs_direct_sum():
    from scipy.special import zeta
    for s, q in ((2.5, 1.0), (1.7, 3.0), (3.1, 10.0)):
        k = np.arange(0, 200000, dtype=np.float64)
        direct = np.sum((k + q) ** (-s))
        tail = (200000 + q) ** (1 - s) / (s - 1)  # integral tail
        assert abs(zeta(s, q) - (direct + tail)) < 1e-6 * zeta(s, q)


def test_ks_recovers_power_law():
    """SPEC.md:460 style: discrete power-law samples, alpha = 2.5, x_min = 1, by inverse
    CDF over the exact pmf; the fit recovers alpha and a small K-S distance."""
    from scipy.special import zeta
    rng = np.random.default_rng(11)
    alpha = 2.5
    dmax = 10**6
    k = np.arange(1, dmax + 1, dtype=np.float64)
    cdf = np.cumsum(k ** (-alpha)) / zeta(alpha, 1.0)
    u = rng.random(100000)
    x = np.searchsorted(cdf, u) + 1
    x = x[x <= dmax]
    h = np.bincount(x)
    r = odeg.ks_powerlaw(h)
    assert 2.4 <= r["alpha"] <= 2.6
    assert r["ks"] < 0.05


def test_ks_no_admissible_xmin():
    h = np.zeros(8, dtype=np.int64)
    h[2:8] = 5
    assert np.isnan(odeg.ks_powerlaw(h)["ks"])


# ------------------------------------------------------------------ BFS + filter + hybrid
def bfs_ecc_pure(n, edges, root):
    adj = [[] for _ in range(n)]
    for a, b in edges:
        adj[a].append(b)
        adj[b].append(a)
    dist = {root: 0}
    q = [root]
    for x in q:
        for y in adj[x]:
            if y not in dist:
                dist[y] = dist[x] + 1
                q.append(y)
    return set(dist), max(dist.values())


@pytest.mark.parametrize("seed", range(5))
def test_bfs_component_and_levels(seed):
    rng = np.random.default_rng(seed)
    n = 200
    e = rng.integers(0, n, size=(150, 2))
    deg, _ = odeg.degree_distribution(n, e)
    root = obfs.bfs_root(deg)
    assert deg[root] == deg.max() and np.all(deg[:root] < deg[root])
    vis, lev = obfs.bfs(n, e, root)
    want_set, want_ecc = bfs_ecc_pure(n, e.tolist(), root)
    assert set(np.flatnonzero(vis).tolist()) == want_set
    assert lev == want_ecc
    rem = obfs.filter_edges(e, vis)
    # no edge has exactly one visited endpoint
    assert not np.any(vis[e[:, 0]] ^ vis[e[:, 1]])
    assert np.all(~vis[rem[:, 0]]) and np.all(~vis[rem[:, 1]])


@pytest.mark.parametrize("mode", ["auto", "sv", "bfs+sv"])
def test_hybrid_mode_invariance(mode):
    for g in (graphgen.make("c1", 0.05), graphgen.rmat_scale_graph(12)):
        lab, rep = ohyb.hybrid(g.n, g.edges, mode=mode)
        assert np.array_equal(lab, oracle.uf_labels(g.n, g.edges))
        if mode == "bfs+sv":
            assert rep["ran_bfs"]


# ------------------------------------------------------------------ generators (host logic)
def test_generators_deterministic_and_sized():
    a = graphgen.make("c1")
    b = graphgen.make("c1")
    assert np.array_equal(a.edges, b.edges)
    assert a.n == 65536 and a.m == 200000 and a.edges.max() < a.n
    c3 = graphgen.make("c3", 1 / 256)
    assert c3.n == 256 * 256
    g = graphgen.rmat_scale_graph(10)
    assert g.m == 16 * 1024 and g.edges.max() < 1024
    # the id permutation is a bijection
    n = 1000
    vals = {graphgen.perm_value(n, 1, 2, x) for x in range(n)}
    assert vals == set(range(n))


def test_c5_generator_is_a_relabelled_union():
    """graphgen C5 (inputs only): the u64 ids are a bijective mix of the dense indices of an
    R-MAT part and a path part on disjoint index ranges; edge order is scrambled, not the
    multiset (checked against the two parts drawn separately)."""
    import graphgen
    g = graphgen.make("c5", 1 / 4096)
    sc, npaths = g.params["rmat_scale"], g.params["n_paths"]
    a = graphgen.rmat(graphgen.BASE_SEED + 5, sc, 16)
    _, b = graphgen.paths(graphgen.BASE_SEED + 5 + 100, npaths, 64.0, 0, 0)
    idx = np.concatenate([a.astype(np.uint64), b.astype(np.uint64) + np.uint64(1 << sc)])
    mixed = np.vectorize(graphgen.mix64, otypes=[np.uint64])(idx)
    assert g.edges.shape == mixed.shape
    assert np.array_equal(np.sort(g.edges.reshape(-1)), np.sort(mixed.reshape(-1)))
    sample = np.arange(20000, dtype=np.uint64)
    assert len({graphgen.mix64(int(x)) for x in sample}) == sample.shape[0]


def test_graphgen_c5_blocks_concatenate():
    """Per-rank C5 generation (graphgen.make_block, bench.py at N > 1) draws exactly the rows
    of the whole list that the block distribution gives each rank."""
    g = graphgen.make("c5", 1 / 4096)
    for world in (2, 3, 8):
        parts = [graphgen.make_block("c5", 1 / 4096, r, world) for r in range(world)]
        assert all(p.params["m_total"] == g.m for p in parts)
        assert np.array_equal(np.concatenate([p.edges for p in parts]), g.edges)
