"""GPU parity of the degree count and degree distribution (Alg. 2 line 2).

Through the C ABI: ``cc_degrees_u32`` (deg(v) for every id, the prediction stage's kernels) must
equal the oracle's sort-by-source run lengths (``oracle.degree.degree_distribution``) element by
element, and ``cc_degree_histogram`` (the gate's input after ``cc_run``) must equal the oracle's
D[d] bin by bin.  Both degree kernels are covered: the bucketed shared-memory count (default for
n >= 2^20) and the L2-window increments (``CC_DEG_ALGO`` forces one), on graphs that exercise
the bucketed count's fallbacks (a staging row overflowing within a round, a bucket region
overflowing its 2x-mean capacity), odd edge counts, self-loops, and ids in several buckets and
super-windows.
"""
import os

import numpy as np
import pytest

import graphgen
from oracle import degree as odeg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ccm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1607_06156_b200 as ccmod
    return ccmod


@pytest.fixture(params=["radix", "window"])
def algo(request):
    old = os.environ.get("CC_DEG_ALGO")
    os.environ["CC_DEG_ALGO"] = request.param
    yield request.param
    if old is None:
        os.environ.pop("CC_DEG_ALGO", None)
    else:
        os.environ["CC_DEG_ALGO"] = old


def _graphs():
    rng = np.random.default_rng(11)
    out = {}
    g = graphgen.make("c1")
    out["c1"] = (g.n, g.edges)
    g = graphgen.make("c2", 0.05)
    out["c2_5pct"] = (g.n, g.edges)
    g = graphgen.rmat_scale_graph(18)
    out["rmat18"] = (g.n, g.edges)
    # star on 2^20 ids: one bucket receives half of all endpoints (staging-row and region
    # overflow fall back to direct increments); odd m; self-loops count 2 (C9)
    n = 1 << 20
    leaves = rng.integers(0, n, size=300_001, dtype=np.uint32)
    e = np.stack([np.full_like(leaves, 12345), leaves], 1)
    e = np.concatenate([e, np.array([[7, 7], [n - 1, n - 1]], np.uint32)])
    out["star_2p20"] = (n, e)
    # every endpoint in the first bucket of a 2^21-id range: the other buckets are empty
    e = rng.integers(0, 1 << 15, size=(200_003, 2), dtype=np.uint32)
    out["one_bucket"] = (1 << 21, e)
    # ids in the last, ragged bucket of a non-power-of-two id range
    n = (1 << 20) + 777
    e = rng.integers(n - 5000, n, size=(50_001, 2), dtype=np.uint32)
    e = np.concatenate([e, rng.integers(0, n, size=(100_000, 2), dtype=np.uint32)])
    out["ragged_tail"] = (n, e)
    # one edge
    out["one_edge"] = ((1 << 20), np.array([[5, 1 << 19]], np.uint32))
    return out


GRAPHS = _graphs()


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_degrees_equal_oracle(ccm, algo, name):
    n, e = GRAPHS[name]
    want, hist = odeg.degree_distribution(n, e)
    ctx = ccm.CC(device=0)
    try:
        ctx.load(e, n)
        got = ctx.degrees(n)
        assert np.array_equal(got.astype(np.int64), want), name
        rep = ctx.run("auto")
        d, c = ctx.degree_histogram()
        nz = np.flatnonzero(hist)
        assert np.array_equal(d, nz.astype(np.uint64)), name
        assert np.array_equal(c, hist[nz].astype(np.uint64)), name
        assert rep["max_degree"] == int(want.max())
        assert rep["n_present"] == int(np.count_nonzero(want))
    finally:
        ctx.close()


def test_degrees_super_windows(ccm, algo):
    """n = 2^27 + 3: two bucketed super-windows of 2^26 ids plus a ragged third (or eight
    L2 windows); hubs near both window edges."""
    n = (1 << 27) + 3
    rng = np.random.default_rng(5)
    e = rng.integers(0, n, size=(3_000_000, 2), dtype=np.uint32)
    hubs = np.array([0, (1 << 26) - 1, 1 << 26, n - 1], np.uint32)
    e = np.concatenate([e, np.stack([np.repeat(hubs, 20000), rng.integers(0, n, 80000, dtype=np.uint32)], 1)])
    want = np.bincount(e.reshape(-1).astype(np.int64), minlength=n)
    ctx = ccm.CC(device=0)
    try:
        ctx.load(e, n)
        got = ctx.degrees(n)
        assert np.array_equal(got.astype(np.int64), want)
    finally:
        ctx.close()


def test_degree_histogram_c2_c3_full(ccm):
    """Full C2 and C3 (bench sizes): the gate's distribution bin by bin."""
    for cfg in ("c2", "c3"):
        g = graphgen.make(cfg)
        _, hist = odeg.degree_distribution(g.n, g.edges)
        ctx = ccm.CC(device=0)
        try:
            ctx.load(g.edges, g.n)
            ctx.run("auto")
            d, c = ctx.degree_histogram()
            nz = np.flatnonzero(hist)
            assert np.array_equal(d, nz.astype(np.uint64)), cfg
            assert np.array_equal(c, hist[nz].astype(np.uint64)), cfg
        finally:
            ctx.close()


def test_degree_histogram_needs_a_run(ccm):
    ctx = ccm.CC(device=0)
    try:
        ctx.load(np.array([[0, 1]], np.uint32), 4)
        with pytest.raises(ccm.CCError):
            ctx.degree_histogram()
        ctx.run("sv")  # mode=sv without CC_FLAG_TRACE builds no distribution
        with pytest.raises(ccm.CCError):
            ctx.degree_histogram()
        ctx.run("auto")
        d, c = ctx.degree_histogram()
        assert d.tolist() == [1] and c.tolist() == [2]
    finally:
        ctx.close()
