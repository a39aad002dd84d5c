"""GPU parity of the speculative root level (graph.cu k_deg_sample).

The BFS root is the max-degree vertex, smallest id on ties (Alg. 2 line 7, PAPER.md:262;
SURVEY.md C13).  On edge lists of >= 2^26 records the degree pass guesses it from the counts
of a prefix of the list and runs the guess's BFS level while it streams the rest; cc_run keeps
that level only if the guess is the exact root, and otherwise runs level 1 as usual.  The
CC_SPEC_MIN_EDGES / CC_SPEC_SAMPLE_EDGES hooks make small graphs take that path, so a kept
guess, a discarded guess and the prefix split of the degree count are all compared with the
oracle: labels bit-exact; degrees element by element; the degree distribution bin by bin;
root, visited count, levels and remainder exactly.
"""
import os

import numpy as np
import pytest

import graphgen
import oracle
from oracle import bfs as obfs
from oracle import degree as odeg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ccm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    return ccmod


@pytest.fixture
def spec_env():
    keys = ("CC_SPEC_MIN_EDGES", "CC_SPEC_SAMPLE_EDGES", "CC_DEG_ALGO")
    old = {k: os.environ.get(k) for k in keys}

    def set_(sample, min_edges=1):
        os.environ["CC_SPEC_MIN_EDGES"] = str(min_edges)
        os.environ["CC_SPEC_SAMPLE_EDGES"] = str(sample)
        os.environ["CC_DEG_ALGO"] = "radix"  # the speculation rides on the bucketed count
    yield set_
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def check(ccm, n, e, mode, want_spec):
    e = np.ascontiguousarray(e, dtype=np.uint32).reshape(-1, 2)
    want = oracle.uf_labels(n, e).astype(np.int64)
    deg, hist = odeg.degree_distribution(n, e)
    root = obfs.bfs_root(deg)
    vis, levels = obfs.bfs(n, e, root)
    ctx = ccm.CC(device=0, flags=ccm.CC_FLAG_TRACE)  # TRACE: the distribution in every mode
    try:
        ctx.load(e, n)
        rep = ctx.run(mode)
        assert np.array_equal(ctx.labels().astype(np.int64), want)
        assert rep["ran_bfs"] == 1
        assert rep["bfs_spec_root"] == int(want_spec)
        assert rep["bfs_root"] == root
        assert rep["bfs_visited"] == int(vis.sum())
        assert rep["bfs_levels"] == levels
        assert rep["remainder_edges"] == obfs.filter_edges(e, vis).shape[0]
        assert rep["max_degree"] == int(deg.max())
        d, c = ctx.degree_histogram()
        nz = np.flatnonzero(hist)
        assert np.array_equal(d, nz.astype(np.uint64))
        assert np.array_equal(c, hist[nz].astype(np.uint64))
        # the same dispatch through cc_degrees_u32: every degree, prefix split included
        assert np.array_equal(ctx.degrees(n).astype(np.int64), deg)
    finally:
        ctx.close()


def test_spec_kept_rmat(ccm, spec_env):
    g = graphgen.rmat_scale_graph(18)
    spec_env(1 << 16)
    for mode in ("auto", "bfs+sv"):
        check(ccm, g.n, g.edges, mode, True)


def test_spec_not_in_sv_mode(ccm, spec_env):
    g = graphgen.rmat_scale_graph(16)
    spec_env(1 << 12)
    ctx = ccm.CC(device=0)
    try:
        ctx.load(g.edges, g.n)
        rep = ctx.run("sv")
        assert rep["ran_bfs"] == 0 and rep["bfs_spec_root"] == 0
        assert np.array_equal(ctx.labels().astype(np.int64), oracle.uf_labels(g.n, g.edges))
    finally:
        ctx.close()


def test_spec_discarded(ccm, spec_env):
    """The prefix's heaviest id (a star of 12,000 edges) is not the graph's (a star of
    20,000 edges after the prefix): the guess is discarded, level 1 runs from the true root."""
    rng = np.random.default_rng(3)
    n = 1 << 20
    P = 1 << 14
    a, b = 1000, 77
    pre = np.concatenate([np.stack([np.full(12000, a, np.uint32), rng.integers(0, n, 12000, dtype=np.uint32)], 1),
                          rng.integers(0, n, size=(P - 12000, 2), dtype=np.uint32)])
    rest = np.concatenate([np.stack([rng.integers(0, n, 20000, dtype=np.uint32), np.full(20000, b, np.uint32)], 1),
                           rng.integers(0, n, size=(300_001, 2), dtype=np.uint32)])
    rng.shuffle(pre)
    rng.shuffle(rest)
    e = np.concatenate([pre, rest])
    spec_env(P)
    check(ccm, n, e, "bfs+sv", False)


def test_spec_tie_and_odd(ccm, spec_env):
    """Two ids tie for the maximum degree (the smaller is the root, C13) and the prefix sees
    the larger one more often; odd edge count and odd sample size (rounded down to even)."""
    rng = np.random.default_rng(4)
    n = 1 << 20
    lo_id, hi_id = 4242, 90001
    s_hi = np.stack([np.full(5000, hi_id, np.uint32), rng.integers(0, n, 5000, dtype=np.uint32)], 1)
    s_lo = np.stack([rng.integers(0, n, 5000, dtype=np.uint32), np.full(5000, lo_id, np.uint32)], 1)
    noise = rng.integers(0, n, size=(200_400, 2), dtype=np.uint32)
    noise = noise[~np.isin(noise, [lo_id, hi_id]).any(1)][:200_001]
    # hi_id's star first: the prefix guess is hi_id, the root is lo_id
    e = np.concatenate([s_hi, noise[:1001], s_lo, noise[1001:]])
    deg, _ = odeg.degree_distribution(n, e)
    assert deg[lo_id] == deg[hi_id] == deg.max()
    spec_env(6001)
    check(ccm, n, e, "bfs+sv", False)
    # the smaller id first: kept
    e = np.concatenate([s_lo, noise[:1001], s_hi, noise[1001:]])
    check(ccm, n, e, "bfs+sv", True)


def test_spec_self_loop_root(ccm, spec_env):
    """The root's only edges are self-loops (degree 2 each, C9): its level finds nothing and
    the BFS stops at level 0."""
    rng = np.random.default_rng(6)
    n = 1 << 20
    loops = np.full((3000, 2), 31337, np.uint32)
    noise = rng.integers(0, n, size=(100_000, 2), dtype=np.uint32)
    e = np.concatenate([loops, noise])
    spec_env(4096)
    check(ccm, n, e, "bfs+sv", True)


def test_spec_super_windows(ccm, spec_env):
    """n > 2^26: the degree pass runs once per 2^26-id super-window and only the first pass
    carries the guess's level; the root sits in the second window."""
    rng = np.random.default_rng(8)
    n = (1 << 27) + 3
    root = (1 << 26) + 12345
    star = np.stack([np.full(40000, root, np.uint32), rng.integers(0, n, 40000, dtype=np.uint32)], 1)
    noise = rng.integers(0, n, size=(2_000_000, 2), dtype=np.uint32)
    e = np.concatenate([star[:20000], noise, star[20000:]])
    rng.shuffle(e)
    spec_env(1 << 18)
    check(ccm, n, e, "bfs+sv", True)
