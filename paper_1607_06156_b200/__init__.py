"""Thin Python binding of libcc.so (include/cc.h): argument marshalling only.

Every step of the connected-components path runs in the sm_100a kernels of ``csrc/``;
this module only converts arguments, supplies PyTorch's stream and caching allocator to
the library, and converts the report.  There is no CPU fallback: if ``libcc.so`` is
missing, importing the binding raises.

Names follow the C ABI: :func:`cc_init`, :func:`cc_load_edges`, :func:`cc_run`,
:func:`cc_labels_u32`, :func:`cc_destroy`, plus the convenience class :class:`CC`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcc.so")

CC_OK, CC_ERR_INVALID, CC_ERR_RANGE, CC_ERR_NOMEM, CC_ERR_CUDA, CC_ERR_COMM, CC_ERR_STATE, \
    CC_ERR_NOCONV = range(8)
MODES = {"auto": 0, "sv": 1, "bfs+sv": 2}
CC_U32, CC_U64 = 0, 1
CC_FLAG_TRACE = 0x1
CC_FLAG_GATE_KS = 0x2
CC_FLAG_NO_EARLY_EXCLUDE = 0x4
CC_FLAG_REGROUP_SORT = 0x8
CC_FLAG_REGROUP_DIRECT = 0x20
REGROUP_FLAGS = {"csr": 0, "sort": 0x8, "direct": 0x20, "csrbfs": 0x40}
CC_FLAG_PROFILE = 0x10
CC_FLAG_BFS_CSR = 0x40
CC_FLAG_NO_EXCLUDE = 0x80
CC_FLAG_PERMUTE_IDS = 0x100
CC_FLAG_NO_COLLAPSE = 0x200
CC_FLAG_NO_RENUMBER = 0x400
CC_FLAG_BALANCE = 0x800
CC_FLAG_DENSE_EXCHANGE = 0x1000
EXCLUSION_FLAGS = {"early": 0, "end": CC_FLAG_NO_EARLY_EXCLUDE, "none": CC_FLAG_NO_EXCLUDE}

ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                ctypes.c_int, ctypes.c_int, ctypes.c_void_p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_uint64, ctypes.c_void_p)
ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p,
                                ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p)
CC_DT_I32, CC_DT_I64, CC_DT_U8 = 0, 1, 2
CC_OP_SUM, CC_OP_MIN, CC_OP_MAX = 0, 1, 2


class cc_comm(ctypes.Structure):
    _fields_ = [("user", ctypes.c_void_p), ("allreduce", ALLREDUCE_FN), ("allgather", ALLGATHER_FN),
                ("alltoallv", ALLTOALLV_FN)]


class cc_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world_size", ctypes.c_int), ("comm", ctypes.POINTER(cc_comm)),
                ("alloc", ALLOC_FN), ("free", FREE_FN),
                ("alloc_user", ctypes.c_void_p), ("tau", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("flags", ctypes.c_uint32),
                ("nccl_id", ctypes.c_void_p)]


class cc_iter_stat(ctypes.Structure):
    _fields_ = [("active_in", ctypes.c_uint64), ("partitions", ctypes.c_uint64),
                ("temps", ctypes.c_uint64), ("completed", ctypes.c_uint64),
                ("changed", ctypes.c_uint64), ("changed2", ctypes.c_uint64),
                ("active_min", ctypes.c_uint64), ("active_max", ctypes.c_uint64),
                ("ms", ctypes.c_double)]


class cc_report(ctypes.Structure):
    _fields_ = [("ran_bfs", ctypes.c_int), ("ls_alpha", ctypes.c_double), ("ls_r2", ctypes.c_double),
                ("ks_stat", ctypes.c_double), ("ks_alpha", ctypes.c_double),
                ("ks_xmin", ctypes.c_uint32), ("max_degree", ctypes.c_uint64),
                ("n_present", ctypes.c_uint64), ("m_edges", ctypes.c_uint64),
                ("components", ctypes.c_uint64), ("bfs_root", ctypes.c_uint64),
                ("bfs_visited", ctypes.c_uint64), ("bfs_levels", ctypes.c_uint64),
                ("remainder_edges", ctypes.c_uint64), ("sv_iterations", ctypes.c_uint32),
                ("ms_total", ctypes.c_double), ("ms_prediction", ctypes.c_double),
                ("ms_relabel", ctypes.c_double), ("ms_bfs", ctypes.c_double),
                ("ms_filter", ctypes.c_double), ("ms_sv", ctypes.c_double),
                ("ms_finalize", ctypes.c_double), ("iters", ctypes.POINTER(cc_iter_stat)),
                ("n_iters", ctypes.c_uint32),
                ("bfs_spec_root", ctypes.c_int), ("sv_ids", ctypes.c_uint64)]


EXPORTS = ["cc_version", "cc_get_unique_id", "cc_init", "cc_load_edges", "cc_run", "cc_labels_u32", "cc_labels_u64",
           "cc_labels_device", "cc_block_range", "cc_bfs_eccentricity", "cc_approx_diameter", "cc_radix_sort_pairs",
           "cc_degree_histogram", "cc_degrees_u32",
           "cc_set_profiling", "cc_last_launch_count",
           "cc_kernel_stats", "cc_kernel_ops",
           "cc_kernel_name", "cc_destroy", "cc_status_string", "cc_last_error"]


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libcc.so not built ({path}); run __graft_entry__.build() -- "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.cc_version.restype = ctypes.c_char_p
    lib.cc_status_string.restype = ctypes.c_char_p
    lib.cc_status_string.argtypes = [ctypes.c_int]
    lib.cc_last_error.restype = ctypes.c_char_p
    lib.cc_last_error.argtypes = [P]
    lib.cc_init.argtypes = [ctypes.POINTER(cc_config), ctypes.POINTER(P)]
    lib.cc_get_unique_id.argtypes = [P, P, ctypes.c_size_t]
    lib.cc_load_edges.argtypes = [P, ctypes.c_int, P, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
    lib.cc_run.argtypes = [P, ctypes.c_int, ctypes.POINTER(cc_report)]
    lib.cc_labels_u32.argtypes = [P, P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    lib.cc_labels_u64.argtypes = [P, P, P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    lib.cc_labels_device.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_uint64)]
    lib.cc_block_range.argtypes = [P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    lib.cc_degree_histogram.argtypes = [P, P, P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
    lib.cc_degrees_u32.argtypes = [P, P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    lib.cc_bfs_eccentricity.argtypes = [P, P, ctypes.c_uint32, P]
    lib.cc_approx_diameter.argtypes = [P, P, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64)]
    lib.cc_radix_sort_pairs.argtypes = [P, P, P, P, ctypes.c_uint64, ctypes.c_int, P]
    lib.cc_radix_sort_pairs.restype = ctypes.c_int
    lib.cc_set_profiling.argtypes = [P, ctypes.c_int]
    lib.cc_set_profiling.restype = ctypes.c_int
    lib.cc_last_launch_count.restype = ctypes.c_uint64
    lib.cc_last_launch_count.argtypes = [P]
    lib.cc_kernel_stats.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]
    lib.cc_kernel_ops.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_char_p)]
    lib.cc_kernel_ops.restype = ctypes.c_int
    lib.cc_destroy.argtypes = [P]
    lib.cc_kernel_name.restype = ctypes.c_char_p
    lib.cc_kernel_name.argtypes = [ctypes.c_int]
    for f in ("cc_init", "cc_load_edges", "cc_run", "cc_labels_u32", "cc_labels_u64",
              "cc_labels_device", "cc_block_range", "cc_bfs_eccentricity", "cc_approx_diameter",
              "cc_kernel_stats", "cc_destroy", "cc_degree_histogram", "cc_degrees_u32"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


class CCError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{lib().cc_status_string(status).decode()}: {msg}")
        self.status = status


def _check(ctx, status):
    if status != CC_OK:
        msg = lib().cc_last_error(ctx).decode() if ctx else ""
        raise CCError(status, msg)


# ------------------------------------------------------------------ collectives (cc_comm)
class _CudaBuf:
    """A raw device pointer seen by torch.as_tensor (no copy)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr or 0), False), "version": 3}


class TorchComm:
    """The cc_comm collectives (include/cc.h) over torch.distributed: NCCL over NVLink for
    device buffers, or gloo, which the binding feeds through host copies.  With
    ``device=None`` the buffers are host memory (used by the CPU tests).  Argument marshalling
    only: every element the library exchanges is produced and consumed by its kernels."""

    _DT = {CC_DT_I32: "int32", CC_DT_I64: "int64", CC_DT_U8: "uint8"}
    _SZ = {CC_DT_I32: 4, CC_DT_I64: 8, CC_DT_U8: 1}

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        self.host_copy = dist.get_backend(group) != "nccl"
        self._fns = (ALLREDUCE_FN(self._allreduce), ALLGATHER_FN(self._allgather),
                     ALLTOALLV_FN(self._alltoallv))
        self.struct = cc_comm(None, *self._fns)

    def _bytes(self, ptr, nbytes):
        import torch
        if nbytes == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.device or "cpu")
        if self.device is None:
            arr = np.ctypeslib.as_array((ctypes.c_uint8 * int(nbytes)).from_address(int(ptr)))
            return torch.from_numpy(arr)
        return torch.as_tensor(_CudaBuf(ptr, nbytes), device=self.device)

    def _run(self, fn, *tensors):
        """Run collective ``fn`` on ``tensors`` (device or host), results written back."""
        import torch
        if self.device is not None and self.host_copy:
            host = [t.cpu() for t in tensors]
            fn(*host)
            for t, h in zip(tensors, host):
                t.copy_(h)
        else:
            fn(*tensors)
        if self.device is not None:
            torch.cuda.synchronize(self.device)

    def _allreduce(self, user, buf, count, dtype, op, stream):
        try:
            import torch
            t = self._bytes(buf, count * self._SZ[dtype]).view(getattr(torch, self._DT[dtype]))
            rop = {CC_OP_SUM: self.dist.ReduceOp.SUM, CC_OP_MIN: self.dist.ReduceOp.MIN,
                   CC_OP_MAX: self.dist.ReduceOp.MAX}[op]
            self._run(lambda x: self.dist.all_reduce(x, op=rop, group=self.group), t)
            return 0
        except Exception as e:  # reported to the library as CC_ERR_COMM
            print(f"cc comm allreduce failed: {e!r}")
            return 1

    def _allgather(self, user, send, recv, nbytes, stream):
        try:
            src = self._bytes(send, nbytes)
            dst = self._bytes(recv, nbytes * self.world)

            def fn(s, d):
                if self.host_copy:
                    self.dist.all_gather(list(d.chunk(self.world)), s, group=self.group)
                else:
                    self.dist.all_gather_into_tensor(d, s, group=self.group)
            self._run(fn, src, dst)
            return 0
        except Exception as e:
            print(f"cc comm allgather failed: {e!r}")
            return 1

    def _alltoallv(self, user, send, send_bytes, recv, recv_bytes, stream):
        try:
            sb = [int(send_bytes[k]) for k in range(self.world)]
            rb = [int(recv_bytes[k]) for k in range(self.world)]
            src = self._bytes(send, sum(sb))
            dst = self._bytes(recv, sum(rb))
            self._run(lambda s, d: self.dist.all_to_all_single(d, s, rb, sb, group=self.group), src, dst)
            return 0
        except Exception as e:
            print(f"cc comm alltoallv failed: {e!r}")
            return 1


class NcclGroup:
    """Library-owned NCCL communicator (include/cc.h cfg.nccl_id): rank 0 draws the 128-byte
    id with cc_get_unique_id and torch.distributed broadcasts it (the only use of the process
    group); cc_init then builds the communicator and every exchange is an NCCL call on the
    library's stream.  ``NcclGroup.single()`` is a 1-rank communicator (the sharded driver on
    one GPU, for tests)."""

    def __init__(self, rank, world, uid: bytes):
        if len(uid) != CC_UNIQUE_ID_BYTES:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.rank, self.world, self.uid = rank, world, bytes(uid)
        self._buf = ctypes.create_string_buffer(self.uid, CC_UNIQUE_ID_BYTES)

    @classmethod
    def from_process_group(cls, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cc_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        return cls(rank, world, obj[0])

    @classmethod
    def single(cls):
        return cls(0, 1, cc_get_unique_id())


CC_UNIQUE_ID_BYTES = 128


def cc_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(CC_UNIQUE_ID_BYTES)
    why = ctypes.create_string_buffer(512)
    st = lib().cc_get_unique_id(buf, why, 512)
    if st != CC_OK:
        raise CCError(st, why.value.decode(errors="replace"))
    return buf.raw


# ------------------------------------------------------------------ C-ABI-named wrappers
def cc_init(device=0, stream=None, flags=0, tau=0.05, torch_alloc=True, comm=None, alloc_limit=None):
    """Create a context.  ``stream``: a torch.cuda.Stream or raw cudaStream_t int (default:
    torch's current stream).  ``torch_alloc``: route device allocations through PyTorch's
    caching allocator.  ``comm``: a :class:`NcclGroup` (library-owned NCCL) or a
    :class:`TorchComm` (callbacks) for a multi-GPU context; rank and world size are taken
    from it.  ``alloc_limit`` (tests): allocations above this many bytes fail (NOMEM)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    cfg = cc_config()
    cfg.device = device
    cfg.stream = sptr
    cfg.rank = comm.rank if comm else 0
    cfg.world_size = comm.world if comm else 1
    if isinstance(comm, NcclGroup):
        cfg.nccl_id = ctypes.cast(comm._buf, ctypes.c_void_p)
    elif comm:
        cfg.comm = ctypes.pointer(comm.struct)
    cfg.tau = tau
    cfg.flags = flags
    keep = [comm]
    if torch_alloc:
        dev = device

        def _alloc(nbytes, st, user):
            if alloc_limit is not None and nbytes > alloc_limit:
                return None
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st or 0)
            except Exception:  # OOM -> NULL -> CC_ERR_NOMEM
                return None

        def _free(ptr, nbytes, st, user):
            torch.cuda.caching_allocator_delete(ptr)

        a, f = ALLOC_FN(_alloc), FREE_FN(_free)
        cfg.alloc, cfg.free = a, f
        keep += [a, f]
    h = ctypes.c_void_p()
    _check(None, lib().cc_init(ctypes.byref(cfg), ctypes.byref(h)))
    return h, keep


def cc_load_edges(ctx, pairs, n_vertices, ids="u32"):
    """pairs: (m,2) array of ids -- numpy (host; converted to uint32 / uint64) or a torch CUDA
    tensor (device; 4-byte elements for ids='u32', 8-byte for 'u64', passed as is)."""
    if ids not in ("u32", "u64"):
        raise ValueError(f"ids must be 'u32' or 'u64', not {ids!r}")
    w = CC_U32 if ids == "u32" else CC_U64
    if hasattr(pairs, "is_cuda") and pairs.is_cuda:
        if pairs.dim() != 2 or pairs.shape[1] != 2:
            raise ValueError(f"device edge tensor must have shape (m, 2), not {tuple(pairs.shape)}")
        want = 4 if w == CC_U32 else 8
        if pairs.element_size() != want or pairs.is_floating_point():
            raise ValueError(f"ids={ids!r} needs {want}-byte integer elements, got {pairs.dtype}")
        t = pairs.contiguous()
        m = t.shape[0]
        _check(ctx, lib().cc_load_edges(ctx, w, ctypes.c_void_p(t.data_ptr()), m, n_vertices, 1))
        return m
    a = np.ascontiguousarray(pairs, dtype=np.uint32 if w == CC_U32 else np.uint64).reshape(-1, 2)
    m = a.shape[0]
    _check(ctx, lib().cc_load_edges(ctx, w, a.ctypes.data_as(ctypes.c_void_p), m, n_vertices, 0))
    return m


def _report(r: cc_report) -> dict:
    d = {k: getattr(r, k) for k, _ in cc_report._fields_ if k != "iters"}
    d["iters"] = [{k: getattr(r.iters[i], k) for k, _ in cc_iter_stat._fields_}
                  for i in range(r.n_iters)]
    return d


def cc_run(ctx, mode="auto") -> dict:
    r = cc_report()
    _check(ctx, lib().cc_run(ctx, MODES[mode], ctypes.byref(r)))
    return _report(r)


def cc_labels_u32(ctx, out=None):
    """Labels into a new numpy array (host) or into ``out`` (numpy or torch CUDA uint32/int32)."""
    cnt = ctypes.c_uint64()
    lib().cc_labels_u32(ctx, None, 0, ctypes.byref(cnt), 0)  # query n (returns INVALID)
    n = cnt.value
    if out is None:
        out = np.empty(n, dtype=np.uint32)
    if hasattr(out, "is_cuda") and out.is_cuda:
        if out.element_size() != 4 or out.is_floating_point() or not out.is_contiguous():
            raise ValueError(f"label output must be a contiguous 4-byte integer tensor, got {out.dtype}")
        _check(ctx, lib().cc_labels_u32(ctx, ctypes.c_void_p(out.data_ptr()), out.numel(),
                                        ctypes.byref(cnt), 1))
    else:
        if out.dtype.itemsize != 4 or out.dtype.kind not in "iu" or not out.flags.c_contiguous:
            raise ValueError(f"label output must be a contiguous 4-byte integer array, got {out.dtype}")
        _check(ctx, lib().cc_labels_u32(ctx, out.ctypes.data_as(ctypes.c_void_p), out.shape[0],
                                        ctypes.byref(cnt), 0))
    return out


def cc_labels_u64(ctx):
    """u64 mode: (sorted distinct ids, label of each) as numpy uint64 arrays."""
    cnt = ctypes.c_uint64()
    lib().cc_labels_u64(ctx, None, None, 0, ctypes.byref(cnt), 0)  # query count
    n = cnt.value
    ids = np.empty(n, dtype=np.uint64)
    lab = np.empty(n, dtype=np.uint64)
    _check(ctx, lib().cc_labels_u64(ctx, ids.ctypes.data_as(ctypes.c_void_p),
                                    lab.ctypes.data_as(ctypes.c_void_p), n, ctypes.byref(cnt), 0))
    return ids, lab


def cc_degree_histogram(ctx):
    """The degree distribution the gate consumed in the last cc_run: (degrees, counts) numpy
    uint64 arrays of the non-empty bins, ascending."""
    cnt = ctypes.c_uint64()
    lib().cc_degree_histogram(ctx, None, None, 0, ctypes.byref(cnt))  # query the bin count
    nb = cnt.value
    d = np.zeros(nb, dtype=np.uint64)
    c = np.zeros(nb, dtype=np.uint64)
    _check(ctx, lib().cc_degree_histogram(ctx, d.ctypes.data_as(ctypes.c_void_p),
                                          c.ctypes.data_as(ctypes.c_void_p), nb, ctypes.byref(cnt)))
    return d, c


def cc_degrees_u32(ctx, n):
    """deg(v) for v in [0, n) as a numpy uint32 array (the prediction-stage count)."""
    out = np.empty(n, dtype=np.uint32)
    cnt = ctypes.c_uint64()
    _check(ctx, lib().cc_degrees_u32(ctx, out.ctypes.data_as(ctypes.c_void_p), n, ctypes.byref(cnt), 0))
    return out


def cc_block_range(ctx):
    """(lo, hi): the vertex block whose labels cc_labels_u32 returns on this rank."""
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _check(ctx, lib().cc_block_range(ctx, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def cc_bfs_eccentricity(ctx, seeds):
    """BFS eccentricity of each seed (numpy uint64 array)."""
    s = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.zeros(s.shape[0], dtype=np.uint64)
    _check(ctx, lib().cc_bfs_eccentricity(ctx, s.ctypes.data_as(ctypes.c_void_p), s.shape[0],
                                          out.ctypes.data_as(ctypes.c_void_p)))
    return out


def approx_diameter(ctx, n, runs=100, seed=0, present=None):
    """The paper's approximate diameter: max BFS depth over ``runs`` random
    seed vertices (drawn among ``present`` ids if given)."""
    rng = np.random.default_rng(seed)
    pool = np.arange(n) if present is None else np.flatnonzero(present)
    seeds = rng.choice(pool, size=min(runs, pool.shape[0]), replace=False)
    return cc_approx_diameter(ctx, seeds)


def cc_approx_diameter(ctx, seeds):
    """Maximum BFS eccentricity over the given seeds, taken in the library."""
    s = np.ascontiguousarray(seeds, dtype=np.uint64)
    d = ctypes.c_uint64()
    _check(ctx, lib().cc_approx_diameter(ctx, s.ctypes.data_as(ctypes.c_void_p), s.shape[0], ctypes.byref(d)))
    return int(d.value)


def cc_radix_sort_pairs(keys, vals, tmp_keys, tmp_vals, key_bits=64, stream=None):
    """Sort torch CUDA tensors keys (int64/uint64, n) with payload vals (int32/uint32, n) in
    place by the low ``key_bits`` bits (stable LSD onesweep); tmp_*: scratch of the same shape."""
    import torch
    st = stream if stream is not None else torch.cuda.current_stream(keys.device)
    sptr = st.cuda_stream if hasattr(st, "cuda_stream") else int(st)
    _check(None, lib().cc_radix_sort_pairs(ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(vals.data_ptr()),
                                           ctypes.c_void_p(tmp_keys.data_ptr()),
                                           ctypes.c_void_p(tmp_vals.data_ptr()), keys.numel(), key_bits,
                                           ctypes.c_void_p(sptr)))


def cc_kernel_stats(ctx, which):
    ms, by, ln = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    _check(ctx, lib().cc_kernel_stats(ctx, which, ctypes.byref(ms), ctypes.byref(by), ctypes.byref(ln)))
    ops, unit = ctypes.c_double(), ctypes.c_char_p()
    _check(ctx, lib().cc_kernel_ops(ctx, which, ctypes.byref(ops), ctypes.byref(unit)))
    return dict(ms=ms.value, bytes=by.value, launches=ln.value, ops=ops.value,
                ops_unit=(unit.value or b"").decode())


def kernel_families():
    out, i = [], 0
    while True:
        nm = lib().cc_kernel_name(i)
        if nm is None:
            return out
        out.append(nm.decode())
        i += 1


def cc_destroy(ctx):
    _check(None, lib().cc_destroy(ctx))


class CC:
    """Convenience wrapper: ``CC().load(edges, n).run('auto')`` then ``.labels()``."""

    def __init__(self, device=0, stream=None, flags=0, tau=0.05, torch_alloc=True, comm=None,
                 alloc_limit=None):
        self.ctx, self._keep = cc_init(device, stream, flags, tau, torch_alloc, comm, alloc_limit)

    def load(self, pairs, n_vertices, ids="u32"):
        cc_load_edges(self.ctx, pairs, n_vertices, ids)
        return self

    def run(self, mode="auto"):
        return cc_run(self.ctx, mode)

    def labels(self, out=None):
        return cc_labels_u32(self.ctx, out)

    def eccentricity(self, seeds):
        return cc_bfs_eccentricity(self.ctx, seeds)

    def block_range(self):
        return cc_block_range(self.ctx)

    def degree_histogram(self):
        return cc_degree_histogram(self.ctx)

    def degrees(self, n):
        return cc_degrees_u32(self.ctx, n)

    def labels_u64(self):
        return cc_labels_u64(self.ctx)

    def set_profiling(self, on):
        _check(self.ctx, lib().cc_set_profiling(self.ctx, 1 if on else 0))

    def launches(self):
        return int(lib().cc_last_launch_count(self.ctx))

    def kernel_stats(self, which):
        return cc_kernel_stats(self.ctx, which)

    def close(self):
        if self.ctx:
            cc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
