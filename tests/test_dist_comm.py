"""world_size 2 (gloo, CPU): the cc_comm collectives the binding hands to the C library
(include/cc.h) move exactly the bytes the ABI promises.  Host buffers stand in for device
buffers (TorchComm(device=None)); the callbacks are called through their C function pointers,
as libcc.so calls them."""
import ctypes

import numpy as np
import pytest

from dist_util import run_ranks


def _collectives(rank, world):
    import paper_1607_06156_b200 as cc
    comm = cc.TorchComm(device=None)
    s = comm.struct
    out = {}
    # allreduce: min over ranks of u32 slots after the library's sign flip -> i32 MIN
    a = np.array([5 + rank, 0xFFFFFFFF, 7 - rank, 3], dtype=np.uint32) ^ np.uint32(0x80000000)
    assert s.allreduce(None, a.ctypes.data, a.size, cc.CC_DT_I32, cc.CC_OP_MIN, None) == 0
    out["min"] = (a ^ np.uint32(0x80000000)).tolist()
    b = np.array([rank + 1, 10 * rank], dtype=np.int64)
    assert s.allreduce(None, b.ctypes.data, b.size, cc.CC_DT_I64, cc.CC_OP_SUM, None) == 0
    out["sum"] = b.tolist()
    c = np.array([rank, 255 - rank, 9], dtype=np.uint8)
    assert s.allreduce(None, c.ctypes.data, c.size, cc.CC_DT_U8, cc.CC_OP_MAX, None) == 0
    out["max"] = c.tolist()
    # allgather, rank-major
    g = np.full(3, 100 + rank, dtype=np.uint32)
    r = np.zeros(3 * world, dtype=np.uint32)
    assert s.allgather(None, g.ctypes.data, r.ctypes.data, g.nbytes, None) == 0
    out["gather"] = r.tolist()
    # alltoallv with uneven (and empty) blocks: rank k sends k+j+... bytes to rank j
    send_counts = [(rank + j) % 3 for j in range(world)]  # u32 elements to rank j
    send = np.concatenate([np.full(cnt, 1000 * rank + j, dtype=np.uint32)
                           for j, cnt in enumerate(send_counts)])
    recv_counts = [(k + rank) % 3 for k in range(world)]
    recv = np.zeros(sum(recv_counts), dtype=np.uint32)
    sb = (ctypes.c_uint64 * world)(*[4 * x for x in send_counts])
    rb = (ctypes.c_uint64 * world)(*[4 * x for x in recv_counts])
    assert s.alltoallv(None, send.ctypes.data if send.size else None, sb,
                       recv.ctypes.data if recv.size else None, rb, None) == 0
    out["a2a"] = recv.tolist()
    return out


def test_collectives_world2():
    res = run_ranks(_collectives, 2)
    for rank, r in enumerate(res):
        assert r["min"] == [5, 0xFFFFFFFF, 6, 3]
        assert r["sum"] == [3, 10]
        assert r["max"] == [1, 255, 9]
        assert r["gather"] == [100, 100, 100, 101, 101, 101]
        want = []
        for k in range(2):
            want += [1000 * k + rank] * ((k + rank) % 3)
        assert r["a2a"] == want


def _errors(rank, world):
    import paper_1607_06156_b200 as cc
    comm = cc.TorchComm(device=None)
    # a failing collective reports nonzero (the library turns it into CC_ERR_COMM)
    bad = comm.struct.allreduce(None, None, 4, 99, cc.CC_OP_SUM, None)
    return bad


def test_collective_failure_is_reported():
    assert run_ranks(_errors, 2) == [1, 1]
