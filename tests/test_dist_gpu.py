"""Multi-GPU path (world_size > 1) on one B200: 2-4 ranks run as processes
that share cuda:0 and exchange through gloo (host copies) -- no kernel waits on another rank,
so sharing the device is safe.  Each rank loads its block of the edge list; the concatenated
label blocks must equal the union-find oracle bit for bit, and the SV counters (computed
from the rank-combined partition slots) must equal the Alg. 1 transcription, i.e. be
independent of the number of ranks (SURVEY.md §8(c) 'multi-GPU' pin)."""
import numpy as np
import pytest

import graphgen
import oracle
from oracle import sv as osv
from dist_util import run_ranks

pytestmark = pytest.mark.gpu


def _rank_run(rank, world, n, edges, modes, flags):
    import torch
    import paper_1607_06156_b200 as cc
    torch.cuda.set_device(0)
    comm = cc.TorchComm(device=torch.device("cuda", 0))
    ctx = cc.CC(device=0, flags=cc.CC_FLAG_TRACE | flags, comm=comm)
    m = edges.shape[0]
    a, b = m * rank // world, m * (rank + 1) // world  # block distribution
    ctx.load(np.ascontiguousarray(edges[a:b]), n)
    out = {}
    for mode in modes:
        rep = ctx.run(mode)
        lo, hi = ctx.block_range()
        out[mode] = (lo, hi, ctx.labels().copy(), rep)
    ctx.close()
    return out


def _check(res, n, edges, modes, trace=True):
    want = oracle.uf_labels(n, edges)
    for mode in modes:
        lab = np.zeros(n, dtype=np.uint32)
        covered = 0
        for r in res:
            lo, hi, l, rep = r[mode]
            lab[lo:hi] = l
            covered += hi - lo
        assert covered == n
        assert np.array_equal(lab, want), mode
        reps = [r[mode][3] for r in res]
        assert all(rep["components"] == np.unique(want).shape[0] for rep in reps)
        assert len({rep["sv_iterations"] for rep in reps}) == 1
        assert all(rep["m_edges"] == edges.shape[0] for rep in reps)
        for it in reps[0]["iters"]:  # per-rank load (fig:loadbal): min <= mean <= max
            w = len(res)
            assert it["active_min"] * w <= it["active_in"] <= it["active_max"] * w
        if trace and mode == "sv":
            _, tr = osv.sv_trace(n, edges)
            got = [dict(A=it["active_in"], P=it["partitions"], T=it["temps"],
                        completed=it["completed"], changed=it["changed"], changed2=it["changed2"])
                   for it in reps[0]["iters"]]
            assert [{k: int(v) for k, v in d.items()} for d in got] == \
                [{k: int(d[k]) for k in ("A", "P", "T", "completed", "changed", "changed2")} for d in tr]
    return want


@pytest.mark.parametrize("world", [2, 3, 8])
def test_dist_c1(world):
    g = graphgen.make("c1", 0.5)
    modes = ("sv", "auto", "bfs+sv")
    _check(run_ranks(_rank_run, world, g.n, g.edges, modes, 0), g.n, g.edges, modes)


def test_dist_rmat_bfs_route():
    g = graphgen.rmat_scale_graph(14)
    modes = ("auto", "sv")
    res = run_ranks(_rank_run, 2, g.n, g.edges, modes, 0)
    want = _check(res, g.n, g.edges, modes)
    from oracle import bfs as obfs
    from oracle import degree as odeg
    deg, _ = odeg.degree_distribution(g.n, g.edges)
    root = obfs.bfs_root(deg)
    vis, levels = obfs.bfs(g.n, g.edges, root)
    for r in res:
        rep = r["auto"][3]
        assert rep["ran_bfs"] == 1
        assert rep["bfs_root"] == root
        assert rep["bfs_visited"] == int(vis.sum())
        assert rep["bfs_levels"] == levels
        assert rep["remainder_edges"] == obfs.filter_edges(g.edges, vis).shape[0]
        assert rep["n_present"] == int(np.count_nonzero(deg))
        assert rep["max_degree"] == int(deg.max())


def test_dist_edge_cases():
    # a path and a star whose rows cross rank blocks and tile edges; an isolated tail of ids
    n = 70000
    perm = np.random.default_rng(5).permutation(n - 100).astype(np.uint32)
    path = np.stack([perm[:-1], perm[1:]], 1)
    star = np.stack([np.full(3000, 11, np.uint32), np.arange(20000, 23000, dtype=np.uint32)], 1)
    e = np.concatenate([path[:40000], star, path[40000:], [[5, 5], [5, 5]]]).astype(np.uint32)
    _check(run_ranks(_rank_run, 2, n, e, ("sv", "bfs+sv"), 0), n, e, ("sv", "bfs+sv"))
    # fewer edges than ranks: some ranks load nothing
    e2 = np.array([[0, 1], [2, 3]], np.uint32)
    _check(run_ranks(_rank_run, 3, 40, e2, ("sv", "auto"), 0), 40, e2, ("sv", "auto"))


def test_dist_degree_tail():
    """A degree >= 2^20 (beyond the dense histogram bins) on a rank: the tail lists of all
    ranks are gathered for the gate (cc_dist.cu); route, max degree and labels as on one GPU."""
    leaves = (1 << 20) + 5
    n = leaves + 100
    rng = np.random.default_rng(3)
    star = np.stack([np.full(leaves, 7, np.uint32), np.arange(100, 100 + leaves, dtype=np.uint32)], 1)
    other = rng.integers(0, 100, size=(300, 2)).astype(np.uint32)
    e = np.concatenate([star, other])[rng.permutation(leaves + 300)]
    res = run_ranks(_rank_run, 2, n, e, ("auto",), 0)
    _check(res, n, e, ("auto",), trace=False)
    deg = np.bincount(e.ravel(), minlength=n) + np.bincount(e[e[:, 0] == e[:, 1], 0], minlength=n)
    for r in res:
        assert r["auto"][3]["max_degree"] == int(deg.max())


def test_dist_exclusion_variants():
    """fig:loadbal variants on 2 ranks: same trace as the transcription with that choice."""
    import paper_1607_06156_b200 as cc
    g = graphgen.make("c1", 0.25)
    for excl in ("none", "end"):
        res = run_ranks(_rank_run, 2, g.n, g.edges, ("sv",), cc.EXCLUSION_FLAGS[excl])
        want, tr = osv.sv_trace(g.n, g.edges, exclusion=excl)
        lab = np.zeros(g.n, dtype=np.uint32)
        for r in res:
            lo, hi, l, rep = r["sv"]
            lab[lo:hi] = l
        assert np.array_equal(lab, want)
        got = [(it["active_in"], it["partitions"], it["temps"], it["completed"], it["changed"],
                it["changed2"]) for it in res[0]["sv"][3]["iters"]]
        assert got == [(d["A"], d["P"], d["T"], d["completed"], d["changed"], d["changed2"]) for d in tr]


def test_dist_matches_single_gpu_c2_sample():
    g = graphgen.make("c2", 0.05)
    _check(run_ranks(_rank_run, 2, g.n, g.edges, ("auto",), 0), g.n, g.edges, ("auto",), trace=False)


# ------------------------------------------------------------------ u64 ids over ranks
def _u64_graph(seed, nv, m):
    rng = np.random.default_rng(seed)
    table = np.unique(rng.integers(0, 2**64 - 1, size=nv, dtype=np.uint64, endpoint=True))
    table = np.concatenate([table, np.array([0, 2**64 - 1], dtype=np.uint64)])
    idx = rng.integers(0, table.shape[0], size=(m, 2))
    return table[idx]


def _rank_run_u64(rank, world, edges, modes):
    import torch
    import paper_1607_06156_b200 as cc
    torch.cuda.set_device(0)
    comm = cc.TorchComm(device=torch.device("cuda", 0))
    ctx = cc.CC(device=0, flags=cc.CC_FLAG_TRACE, comm=comm)
    m = edges.shape[0]
    a, b = m * rank // world, m * (rank + 1) // world
    ctx.load(np.ascontiguousarray(edges[a:b]), 0, ids="u64")
    out = {}
    for mode in modes:
        rep = ctx.run(mode)
        ids, lab = ctx.labels_u64()
        out[mode] = (ctx.block_range(), ids.copy(), lab.copy(), rep)
    ctx.close()
    return out


def _check_u64(res, edges, modes, trace=True):
    """Distributed relabel (SURVEY §8(e) 'distributed sort-unique + rank map'): the ranks'
    blocks concatenate to the sorted distinct ids with the u64 union-find labels, and the SV
    counters equal the transcription on the order-preserving dense relabel."""
    ids_o, lab_o = oracle.uf_labels_u64(edges)
    for mode in modes:
        ids = np.concatenate([r[mode][1] for r in res])
        lab = np.concatenate([r[mode][2] for r in res])
        assert np.array_equal(ids, ids_o), mode
        assert np.array_equal(lab, lab_o), mode
        lo_hi = [r[mode][0] for r in res]
        assert lo_hi[0][0] == 0 and lo_hi[-1][1] == ids_o.shape[0]
        assert all(lo_hi[i][1] == lo_hi[i + 1][0] for i in range(len(lo_hi) - 1))
        reps = [r[mode][3] for r in res]
        assert all(rep["components"] == np.unique(lab_o).shape[0] for rep in reps)
        assert all(rep["m_edges"] == edges.shape[0] for rep in reps)
        if trace and mode == "sv":
            dense, uniq = oracle.relabel_u64(edges)
            _, tr = osv.sv_trace(uniq.shape[0], dense)
            got = [(it["active_in"], it["partitions"], it["temps"], it["completed"], it["changed"],
                    it["changed2"]) for it in reps[0]["iters"]]
            assert got == [(d["A"], d["P"], d["T"], d["completed"], d["changed"], d["changed2"]) for d in tr]


@pytest.mark.parametrize("world,seed,nv,m", [(2, 1, 50, 40), (3, 2, 3000, 5000), (2, 3, 200000, 300000),
                                             (4, 4, 60000, 50000)])
def test_dist_u64(world, seed, nv, m):
    e = _u64_graph(seed, nv, m)
    modes = ("sv", "auto")
    _check_u64(run_ranks(_rank_run_u64, world, e, modes), e, modes)


def test_dist_u64_c5_scaled():
    """C5 (R-MAT U paths, u64 ids, edges sharded over ranks) at 1/4096 scale on 2 ranks:
    distributed relabel -> gate (BFS route) -> BFS peel -> SV on the path remainder."""
    g = graphgen.make("c5", 1 / 4096)
    res = run_ranks(_rank_run_u64, 2, g.edges, ("auto",))
    _check_u64(res, g.edges, ("auto",), trace=False)
    assert all(r["auto"][3]["ran_bfs"] == 1 for r in res)


def test_dist_u64_edge_cases():
    # fewer edges than ranks; the same ids on every rank; extreme ids; skewed shares (one
    # rank's ids all above the others')
    e1 = np.array([[2**64 - 1, 0]], np.uint64)
    _check_u64(run_ranks(_rank_run_u64, 3, e1, ("sv", "auto")), e1, ("sv", "auto"))
    e2 = np.tile(np.array([[7, 9], [9, 11], [2**63, 7]], np.uint64), (6, 1))
    _check_u64(run_ranks(_rank_run_u64, 3, e2, ("sv",)), e2, ("sv",))
    lo = np.arange(0, 4000, dtype=np.uint64).reshape(-1, 2)
    hi = (np.arange(0, 4000, dtype=np.uint64) + np.uint64(2**40)).reshape(-1, 2)
    e3 = np.concatenate([lo, hi, [[5, 2**40 + 7]]]).astype(np.uint64)
    _check_u64(run_ranks(_rank_run_u64, 2, e3, ("sv", "bfs+sv")), e3, ("sv", "bfs+sv"))


def _nccl_world1(rank, world):
    """The NCCL forms of the TorchComm collectives (all_gather_into_tensor, uneven
    all_to_all_single, typed all_reduce) on device buffers, on a 1-rank NCCL group."""
    import ctypes
    import os
    import torch
    import torch.distributed as dist
    import paper_1607_06156_b200 as cc
    dev = torch.device("cuda", 0)
    g = dist.new_group([0], backend="nccl")
    comm = cc.TorchComm(group=g, device=dev)
    assert not comm.host_copy
    s = comm.struct
    a = torch.tensor([5, 0x7FFFFFFF, -3], dtype=torch.int32, device=dev)
    assert s.allreduce(None, a.data_ptr(), 3, cc.CC_DT_I32, cc.CC_OP_MIN, None) == 0
    b = torch.tensor([1, 2], dtype=torch.int64, device=dev)
    assert s.allreduce(None, b.data_ptr(), 2, cc.CC_DT_I64, cc.CC_OP_SUM, None) == 0
    src = torch.arange(12, dtype=torch.uint8, device=dev)
    dst = torch.zeros(12, dtype=torch.uint8, device=dev)
    assert s.allgather(None, src.data_ptr(), dst.data_ptr(), 12, None) == 0
    sb = (ctypes.c_uint64 * 1)(8)
    rb = (ctypes.c_uint64 * 1)(8)
    x = torch.arange(8, dtype=torch.uint8, device=dev) + 100
    y = torch.zeros(8, dtype=torch.uint8, device=dev)
    assert s.alltoallv(None, x.data_ptr(), sb, y.data_ptr(), rb, None) == 0
    return a.tolist(), b.tolist(), dst.tolist(), y.tolist()


def test_torchcomm_nccl_world1():
    res = run_ranks(_nccl_world1, 1)[0]
    assert res[0] == [5, 0x7FFFFFFF, -3]
    assert res[1] == [1, 2]
    assert res[2] == list(range(12))
    assert res[3] == [100 + i for i in range(8)]


# ------------------------------------------------------------------ library-owned NCCL
def _nccl_own_world1(rank, world, cases):
    """cfg.nccl_id at world 1: the sharded driver (owner regroup, prediction reductions,
    bottom-up BFS, slot exchanges, u64 distributed relabel) on a 1-rank NCCL communicator
    created by the library, every collective an NCCL call on the library stream."""
    import torch
    import paper_1607_06156_b200 as cc
    torch.cuda.set_device(0)
    grp = cc.NcclGroup.single()
    ctx = cc.CC(device=0, flags=cc.CC_FLAG_TRACE, comm=grp)
    out = []
    try:
        for kind, n, e, modes in cases:
            if kind == "u32":
                ctx.load(e, n)
                for mode in modes:
                    rep = ctx.run(mode)
                    out.append((kind, mode, ctx.labels().copy(), rep))
            else:
                ctx.load(e, 0, ids="u64")
                for mode in modes:
                    rep = ctx.run(mode)
                    out.append((kind, mode, ctx.labels_u64(), rep))
    finally:
        ctx.close()
    return out


def test_nccl_owned_world1():
    g1 = graphgen.make("c1", 0.5)
    g2 = graphgen.rmat_scale_graph(14)
    rng = np.random.default_rng(9)
    ids = rng.integers(0, 2**63, size=3000, dtype=np.uint64)
    e64 = ids[rng.integers(0, 3000, size=(5000, 2))]
    cases = [("u32", g1.n, g1.edges, ("sv", "bfs+sv")), ("u32", g2.n, g2.edges, ("auto", "sv")),
             ("u64", 0, e64, ("sv",))]
    res = run_ranks(_nccl_own_world1, 1, cases)[0]
    k = 0
    for kind, n, e, modes in cases:
        for mode in modes:
            _, mode_got, lab, rep = res[k]
            k += 1
            assert mode_got == mode
            if kind == "u32":
                assert np.array_equal(lab, oracle.uf_labels(n, e)), mode
                if mode == "sv":
                    _, tr = osv.sv_trace(n, e)
                    got = [dict(A=it["active_in"], P=it["partitions"], T=it["temps"],
                                completed=it["completed"], changed=it["changed"], changed2=it["changed2"])
                           for it in rep["iters"]]
                    assert [{a: int(b) for a, b in d.items()} for d in got] == \
                        [{a: int(d[a]) for a in ("A", "P", "T", "completed", "changed", "changed2")} for d in tr]
                if mode == "auto":
                    assert rep["ran_bfs"] == 1
            else:
                want = oracle.uf_labels_u64(e)
                assert np.array_equal(lab[0], want[0]) and np.array_equal(lab[1], want[1])


# ------------------------------------------------------------------ failure agreement
def _rank_fail(rank, world, n, edges, limit_rank, limit):
    import torch
    import paper_1607_06156_b200 as cc
    torch.cuda.set_device(0)
    comm = cc.TorchComm(device=torch.device("cuda", 0))
    ctx = cc.CC(device=0, comm=comm, alloc_limit=limit if rank == limit_rank else None)
    m = edges.shape[0]
    a, b = m * rank // world, m * (rank + 1) // world
    try:
        ctx.load(np.ascontiguousarray(edges[a:b]), n)
        ctx.run("sv")
        return ("ok", None)
    except cc.CCError as e:
        return ("err", e.status)
    finally:
        ctx.close()


def test_dist_failure_agreement():
    """A local failure on one rank (an allocation the allocator refuses) is agreed on by every
    rank before the next collective: all ranks raise (the failing rank NOMEM, the others
    COMM), none is left blocked in a collective (collective error paths)."""
    import paper_1607_06156_b200 as cc
    g = graphgen.make("c1", 0.5)
    res = run_ranks(_rank_fail, 2, g.n, g.edges, 1, 1 << 16, timeout=120)
    assert res[1] == ("err", cc.CC_ERR_NOMEM)
    assert res[0] == ("err", cc.CC_ERR_COMM)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_dist_edge_partitioned_bfs(world):
    """The BFS route over ranks (cc_dist.cu): degrees counted per rank and summed, each rank
    streams its own edges with a replicated state (bfs_stream: level found bitmaps OR-ed, every
    rank marks the others' finds visited, local compaction), only the remainder is regrouped.
    Root, visited count, levels, remainder size and the remainder's SV trace equal the oracle's."""
    from oracle import bfs as obfs
    from oracle import degree as odeg
    g = graphgen.rmat_scale_graph(16)
    modes = ("auto", "bfs+sv")
    res = run_ranks(_rank_run, world, g.n, g.edges, modes, 0)
    _check(res, g.n, g.edges, modes, trace=False)
    deg, _ = odeg.degree_distribution(g.n, g.edges)
    root = obfs.bfs_root(deg)
    vis, levels = obfs.bfs(g.n, g.edges, root)
    rem = obfs.filter_edges(g.edges, vis)
    _, tr = osv.sv_trace(g.n, rem)
    want_tr = [tuple(int(d[k]) for k in ("A", "P", "T", "completed", "changed", "changed2")) for d in tr]
    for mode in modes:
        for r in res:
            rep = r[mode][3]
            assert rep["ran_bfs"] == 1
            assert rep["bfs_root"] == root
            assert rep["bfs_visited"] == int(vis.sum())
            assert rep["bfs_levels"] == levels
            assert rep["remainder_edges"] == rem.shape[0]
            assert rep["max_degree"] == int(deg.max())
            assert rep["n_present"] == int(np.count_nonzero(deg))
            got = [(it["active_in"], it["partitions"], it["temps"], it["completed"], it["changed"],
                    it["changed2"]) for it in rep["iters"]]
            assert got == want_tr


def _skewed_graph(seed, n):
    """A long random tree on the low quarter of the ids (many SV iterations, rows owned by
    rank 0) and triangles/pairs on the rest (complete within two iterations): with exclusion
    the higher ranks run out of live tuples (fig:loadbal)."""
    rng = np.random.default_rng(seed)
    k = n // 4
    order = rng.permutation(k)
    tree = np.stack([order[1:], order[rng.integers(0, np.arange(1, k))]], 1)
    rest = np.arange(k, n - (n - k) % 3).reshape(-1, 3)
    tri = np.concatenate([rest[:, [0, 1]], rest[:, [1, 2]], rest[::2][:, [2, 0]]])
    e = np.concatenate([tree, tri]).astype(np.uint32)
    return e[rng.permutation(e.shape[0])]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("graph", ["skewed", "c1"])
def test_dist_balanced(world, graph):
    """The paper's 'balanced' variant (CC_FLAG_BALANCE): live rows redistributed
    evenly over the ranks.  Labels and every Alg. 1 counter equal the oracle's (rows moving
    between ranks change no set); after the first iteration the per-rank loads stay within a
    sixteenth of the mean plus one row, where without it they drift apart."""
    import paper_1607_06156_b200 as cc
    if graph == "skewed":
        n = 1 << 17
        edges = _skewed_graph(7, n)
    else:
        g = graphgen.make("c1", 0.5)
        n, edges = g.n, g.edges
    maxrow = int(np.bincount(edges.reshape(-1).astype(np.int64), minlength=n).max()) + 1
    res_b = run_ranks(_rank_run, world, n, edges, ("sv",), cc.CC_FLAG_BALANCE)
    _check(res_b, n, edges, ("sv",))
    res_u = run_ranks(_rank_run, world, n, edges, ("sv",), 0)
    _check(res_u, n, edges, ("sv",))

    def spread(res):
        its = res[0]["sv"][3]["iters"]
        return [(it["active_max"] * world - it["active_in"], it["active_in"]) for it in its[1:]]
    for excess, a in spread(res_b):
        assert excess <= world * (a // (16 * world) + maxrow + 1), (excess, a)
    if graph == "skewed":
        assert any(excess > world * (a // (16 * world) + maxrow + 1) for excess, a in spread(res_u))


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("dense", [False, True])
def test_dist_exchange_modes(world, dense):
    """Both slot exchanges of the sharded SV: owner-computes (default; SURVEY NEXT-1 -- foreign
    slot partials to their owner, statistics per owner block, p_min / PB replied to the
    senders, temporaries routed to their rows' owner) and the dense all-reduce ablation
    (CC_FLAG_DENSE_EXCHANGE).  Labels and every Alg. 1 counter equal the oracle's."""
    import paper_1607_06156_b200 as cc
    flags = cc.CC_FLAG_DENSE_EXCHANGE if dense else 0
    g = graphgen.make("c1", 0.5)
    modes = ("sv", "auto")
    _check(run_ranks(_rank_run, world, g.n, g.edges, modes, flags), g.n, g.edges, modes)
    s = graphgen.make("c2", 0.01)
    _check(run_ranks(_rank_run, world, s.n, s.edges, ("sv",), flags), s.n, s.edges, ("sv",))
    r = graphgen.rmat_scale_graph(12)
    _check(run_ranks(_rank_run, world, r.n, r.edges, ("sv", "bfs+sv"), flags), r.n, r.edges, ("sv", "bfs+sv"))
