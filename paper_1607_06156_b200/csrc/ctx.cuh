// ctx.cuh -- the library context (opaque cc_ctx of include/cc.h) and host helpers shared by
// the single-GPU driver (cc_api.cu) and the multi-GPU driver (cc_dist.cu).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "../../include/cc.h"
#include "csr.cuh"
#include "graph.cuh"
#include "nccl_comm.h"
#include "radix.cuh"
#include "relabel.cuh"
#include "scan.cuh"
#include "sv.cuh"

using namespace cc;

struct cc_ctx {
  cc_config cfg{};
  cudaStream_t st = nullptr;
  void* nccl = nullptr;  // library-owned ncclComm_t (cfg.nccl_id), else the cfg.comm callbacks
  bool dist = false;     // sharded driver: world_size > 1, or a 1-rank NCCL communicator
  std::string err;
  // graph
  bool loaded = false, ran = false;
  cc_idw idw = CC_U32;
  uint64_t n = 0, m = 0;
  uint64_t m_total = 0;  // edges over all ranks
  int kbits = 0;
  uint2* d_edges = nullptr;
  uint2* d_rem = nullptr;
  uint2* d_rem2 = nullptr;
  uint64_t* d_ids64 = nullptr;  // u64 mode: loaded endpoints (2m)
  uint64_t* d_uids = nullptr;   // u64 mode: sorted distinct ids (rank -> id)
  uint64_t* d_htab = nullptr;   // u64 mode: relabel hash table (first-attempt size, grown on overflow)
  uint64_t htab_slots = 0;
  uint64_t* d_mix = nullptr;    // CC_FLAG_PERMUTE_IDS: mixed ids / their sorted copy
  uint32_t* d_pi = nullptr;     // CC_FLAG_PERMUTE_IDS: original rank -> permuted rank
  uint64_t n_alloc = 0;         // id bound the n-sized buffers were sized for
  // u64 ids, world_size > 1 (relabel_dist.cu): this rank's share of the sorted distinct ids
  // (dense ids [gbase[rank], gbase[rank + 1])), and every rank's share boundaries
  uint64_t* d_gids = nullptr;
  uint64_t gids_cap = 0;
  std::vector<uint64_t> gbase;
  uint64_t* d_xid = nullptr;    // exchange scratch: received ids / label requests
  uint64_t xid_cap = 0;
  uint32_t* d_xu32 = nullptr;   // exchange scratch: dense ids of the received ids
  uint64_t xu32_cap = 0;
  uint64_t* d_out64 = nullptr;  // staging of the u64 label output (ids, labels)
  uint64_t out64_cap = 0;
  uint32_t* d_label = nullptr;
  uint32_t* d_deg = nullptr;
  uint32_t* d_hist = nullptr;
  uint2* d_hpairs = nullptr;    // non-empty histogram bins (degree, count) for the host gate
  uint32_t* d_tail = nullptr;
  uint32_t* d_bm[3] = {nullptr, nullptr, nullptr};  // visited, frontier, next
  uint32_t* d_sbm[3] = {nullptr, nullptr, nullptr}; // direct SV: notpc, ncp, head
  uint64_t* d_w[2] = {nullptr, nullptr};
  uint32_t* d_q[2] = {nullptr, nullptr};
  uint64_t cap = 0;
  uint32_t* d_segA = nullptr;
  uint32_t* d_segB = nullptr;
  uint32_t* d_plist[2] = {nullptr, nullptr};  // csr engine: partition-id supersets L_i (slot scans)
  uint64_t* d_plcnt = nullptr;                // their lengths
  uint32_t* d_nx = nullptr;                   // bitmap of the next L (values of PB)
  uint32_t* d_hw = nullptr;                   // csr engine: tuples folded into each row (collapse)
  uint64_t* d_umin = nullptr;  // csr engine: tagged partial row minima / maxima
  uint64_t* d_umax = nullptr;
  csr::LongSeg* d_lsegs = nullptr;  // csr engine: segments of rows longer than csr::LONG
  uint64_t* d_nlsegs = nullptr;
  uint32_t row_tag = 0;
  // multi-GPU (cc_dist.cu): owned vertex block [lo, hi), block size blk (multiple of 32)
  uint64_t blk = 0, lo = 0, hi = 0;
  uint2* d_send = nullptr;       // arcs grouped by owner rank
  uint2* d_recv = nullptr;       // arcs received from all ranks (r in [lo, hi))
  uint64_t recv_cap = 0;
  uint32_t* d_gath = nullptr;    // allgather scratch (world_size x bitmap words)
  uint64_t gath_cap = 0;
  uint64_t* d_cnt = nullptr;     // per-owner arc counts (world_size^2 after the gather)
  uint2* d_xsend = nullptr;      // sparse slot exchange: my touched entries / everyone's
  uint2* d_xrecv = nullptr;
  uint64_t* d_bal = nullptr;     // balanced variant: split points and the gathered send counts
  // owner-computes slot exchange (NEXT-1): entries sent (kept for the reply and the clears)
  struct OcSide {
    uint2* send = nullptr;
    uint64_t nsend = 0, nrecv = 0;
    std::vector<uint64_t> sc, rc;  // entries per destination / per source rank
  } ocA, ocB, ocT;
  uint2* d_ocrecv = nullptr;     // entries received for this rank's slot block
  uint32_t* d_ocval[2] = {nullptr, nullptr};  // reply values (sent / received)
  uint64_t* d_occnt = nullptr;   // counts [world], cursors [world], gathered counts [world^2]
  uint64_t oc_cap = 0;           // entries each buffer holds
  uint64_t xsend_cap = 0, xrecv_cap = 0;
  uint32_t* d_garc = nullptr;  // CSR vertex-group scratch: arcs per group (<= 2048 groups)
  uint64_t* d_gcur = nullptr;  // group cursors [0, 2048), long-row count at [2048]
  uint64_t* d_agree = nullptr; // comm_agree word (cudaMalloc at cc_init, outside `allocs`)
  uint64_t* d_ctr = nullptr;   // sv counters
  uint64_t* d_gctr = nullptr;  // graph counters
  uint64_t* h_ctr = nullptr;   // pinned mirrors
  uint64_t* h_ctr2 = nullptr;  // pinned: the two alternating SV counter blocks (look-ahead)
  uint64_t* h_gctr = nullptr;
  uint32_t* h_hist = nullptr;  // pinned histogram staging
  uint32_t* h_word = nullptr;
  radix::Workspace rws;
  scan::State ss;
  std::vector<std::pair<void*, size_t>> allocs;
  // report
  std::vector<std::pair<uint64_t, uint64_t>> dhist;  // gate input of the last cc_run: (degree, count)
  bool dhist_valid = false;
  std::vector<cc_iter_stat> iters;
  cc_report rep{};
  uint64_t launches = 0;
  // profiling (CC_FLAG_TRACE): per-family events
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<cudaEvent_t> it_ev;  // SV iteration start events
  struct KStat {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    double bytes = 0, ms = 0, ops = 0;
    uint64_t launches = 0;
  } kst[16];
};

// ------------------------------------------------------------------------------ helpers
static inline cc_status fail(cc_ctx* c, cc_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}
#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, e_ == cudaErrorMemoryAllocation ? CC_ERR_NOMEM : CC_ERR_CUDA,        \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define CKL()                                                                             \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, CC_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)
#define TRY(x)                        \
  do {                                \
    cc_status s_ = (x);               \
    if (s_ != CC_OK) return s_;       \
  } while (0)

static inline cc_status dalloc(cc_ctx* c, void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  if (c->cfg.alloc) {
    *p = c->cfg.alloc(bytes, (void*)c->st, c->cfg.alloc_user);
    if (!*p) return fail(c, CC_ERR_NOMEM, "allocator hook returned NULL for %zu bytes", bytes);
  } else {
    cudaError_t e = cudaMallocAsync(p, bytes, c->st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, CC_ERR_NOMEM, "cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
  }
  c->allocs.push_back({*p, bytes});
  return CC_OK;
}
template <typename T>
static inline cc_status dalloc_t(cc_ctx* c, T** p, size_t count) {
  return dalloc(c, reinterpret_cast<void**>(p), count * sizeof(T));
}
static inline void dfree_all(cc_ctx* c) {
  for (auto& a : c->allocs) {
    if (c->cfg.free) c->cfg.free(a.first, a.second, (void*)c->st, c->cfg.alloc_user);
    else cudaFreeAsync(a.first, c->st);
  }
  c->allocs.clear();
  c->d_edges = c->d_rem = c->d_rem2 = nullptr;
  c->d_ids64 = c->d_uids = c->d_mix = c->d_htab = nullptr;
  c->d_gids = c->d_xid = c->d_out64 = nullptr;
  c->d_xu32 = nullptr;
  c->gids_cap = c->xid_cap = c->xu32_cap = c->out64_cap = 0;
  c->gbase.clear();
  c->d_pi = nullptr;
  c->d_label = c->d_deg = c->d_hist = c->d_tail = c->d_segA = c->d_segB = nullptr;
  c->d_hpairs = nullptr;
  c->d_plist[0] = c->d_plist[1] = c->d_nx = nullptr;
  c->d_plcnt = nullptr;
  c->d_umin = c->d_umax = c->d_nlsegs = nullptr;
  c->d_garc = nullptr;
  c->d_gcur = nullptr;
  c->d_send = c->d_recv = nullptr;
  c->d_gath = nullptr;
  c->d_cnt = nullptr;
  c->d_xsend = c->d_xrecv = nullptr;
  c->d_bal = nullptr;
  c->ocA.send = c->ocB.send = c->ocT.send = nullptr;
  c->d_ocrecv = nullptr;
  c->d_ocval[0] = c->d_ocval[1] = nullptr;
  c->d_occnt = nullptr;
  c->oc_cap = 0;
  c->xsend_cap = c->xrecv_cap = 0;
  c->recv_cap = c->gath_cap = 0;
  c->d_lsegs = nullptr;
  c->row_tag = 0;
  c->d_bm[0] = c->d_bm[1] = c->d_bm[2] = nullptr;
  c->d_sbm[0] = c->d_sbm[1] = c->d_sbm[2] = nullptr;
  c->d_w[0] = c->d_w[1] = nullptr;
  c->d_q[0] = c->d_q[1] = nullptr;
  c->d_ctr = c->d_gctr = nullptr;
  c->rws = radix::Workspace();
  c->ss = scan::State();
  c->cap = 0;
}

static inline cudaEvent_t ev_get(cc_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}
static inline float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}
static inline bool profiling(const cc_ctx* c) { return (c->cfg.flags & CC_FLAG_PROFILE) != 0; }

// kernel families timed under CC_FLAG_PROFILE (cc_kernel_stats / cc_kernel_name)
enum KFam { KF_RADIX = 0, KF_SVITER, KF_BFS, KF_ROWA, KF_ROWB, KF_SLOTS, KF_CSR, KF_PREDICT,
            KF_COMPACT, KF_HIST, KF_N };
static const char* const kKfNames[KF_N] = {
    "k_hist+k_onesweep (radix regroup)", "SV iteration (all bucket passes)", "k_bfs_level",
    "k_rowpass<A> +k_long1/2 (Alg.1 lines 8-16)", "k_rowpass<B> +k_long1/2 (Alg.1 lines 17-25)",
    "k_pstat1/k_pstat2/k_list_from_bits (partition slot scans)",
    "CSR build (k_rows, k_fill_*, k_bucket, k_scatter)",
    "degree count (k_deg_part, k_deg_order, k_deg_count)",
    "k_compact (ordered exclusion of completed rows)",
    "degree distribution (k_deg_hist, k_hist_pairs)"};
// unit of the per-family `ops` count (cc_kernel_ops): the random accesses that bound the family
static const char* const kKfOps[KF_N] = {
    "", "", "random 4-byte L2 reads (2 per edge of the level)", "", "", "", "",
    "shared-memory atomics (2 per arc: bucket claim + count)", "", ""};

// NVTX ranges (header-only nvtx3; a no-op pointer call unless a tool such as Nsight Systems is
// attached): cc_load_edges / cc_run, the stages of a run, every SV iteration and every kernel
// family below, so a timeline reads in the paper's terms.  Ranges nest per host thread.
struct NvtxRange {
  explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
// consecutive stages of one call: next() closes the open stage and opens the named one
struct NvtxStages {
  bool open = false;
  void next(const char* s) {
    if (open) nvtxRangePop();
    nvtxRangePushA(s);
    open = true;
  }
  void close() {
    if (open) nvtxRangePop();
    open = false;
  }
  ~NvtxStages() { close(); }
};

struct Prof {
  cc_ctx* c;
  int f;
  cudaEvent_t a = nullptr;
  Prof(cc_ctx* c_, int f_) : c(c_), f(f_) {
    nvtxRangePushA(kKfNames[f]);
    if (profiling(c)) { a = ev_get(c); cudaEventRecord(a, c->st); }
  }
  ~Prof() { nvtxRangePop(); }
  Prof(const Prof&) = delete;
  Prof& operator=(const Prof&) = delete;
  void end(double bytes, uint64_t nl, double ops = 0) {
    if (!profiling(c)) return;
    cudaEvent_t b = ev_get(c);
    cudaEventRecord(b, c->st);
    c->kst[f].ev.push_back({a, b});
    c->kst[f].bytes += bytes;
    c->kst[f].launches += nl;
    c->kst[f].ops += ops;
  }
};

static inline int bits_for(uint64_t n) {
  int b = 0;
  while (b < 63 && (1ull << b) < n) b++;
  return b;
}

// ------------------------------------------------------------------------------ ABI

struct Timer {
  cc_ctx* c;
  cudaEvent_t a;
  explicit Timer(cc_ctx* c_) : c(c_), a(ev_get(c_)) { cudaEventRecord(a, c->st); }
  std::pair<cudaEvent_t, cudaEvent_t> stop() {
    cudaEvent_t b = ev_get(c);
    cudaEventRecord(b, c->st);
    return {a, b};
  }
};

static inline cc_status sync_read(cc_ctx* c) {
  CK(cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(uint64_t) * sv::C_NUM, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(c->h_gctr, c->d_gctr, sizeof(uint64_t) * graph::G_NUM, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

// radix sort wrapper with optional per-call timing
static inline void seg_begin(cc_ctx* c, cudaEvent_t* a) {
  if (profiling(c)) { *a = ev_get(c); cudaEventRecord(*a, c->st); }
}
static inline void seg_end(cc_ctx* c, cudaEvent_t a, double bytes, int nl, int fam = KF_SVITER) {
  if (profiling(c)) {
    cudaEvent_t b = ev_get(c);
    cudaEventRecord(b, c->st);
    c->kst[fam].ev.push_back({a, b});
    c->kst[fam].bytes += bytes;
    c->kst[fam].launches += nl;
  }
}

static inline cc_status scan_epoch_guard(cc_ctx* c) {
  if (((c->ss.epoch + 4) & scan::EPOCH_MASK) < 4) {
    CK(cudaMemsetAsync(c->ss.flags, 0, sizeof(uint64_t) * c->ss.max_tiles, c->st));
    c->ss.epoch += 8;
  }
  return CC_OK;
}

// scan look-back flags for the tuple capacity and the id range (grown, never shrunk)
static inline cc_status ensure_scan_tiles(cc_ctx* c) {
  const uint64_t need = (c->cap + c->n) / 2048 + 4;
  if (c->ss.flags && c->ss.max_tiles >= need) return CC_OK;
  c->ss.max_tiles = need;
  TRY(dalloc_t(c, &c->ss.flags, need));
  CK(cudaMemsetAsync(c->ss.flags, 0, sizeof(uint64_t) * need, c->st));
  return CC_OK;
}
// (re)allocate the tuple / sort buffers (d_w, d_q: `tuples` entries each) with the scan and
// radix look-back state that scales with them; contents are not preserved
static inline cc_status ensure_tuple_cap(cc_ctx* c, uint64_t tuples) {
  if (tuples + 64 <= c->cap) return CC_OK;
  const uint64_t cap = (tuples + 64 + 1023) & ~1023ull;
  for (int i = 0; i < 2; i++) {
    TRY(dalloc_t(c, &c->d_w[i], cap));
    TRY(dalloc_t(c, &c->d_q[i], cap));
  }
  c->cap = cap;
  TRY(dalloc_t(c, &c->d_lsegs, csr::long_seg_cap(cap)));
  const uint64_t rt = cap / radix::TILE_MIN + 2;
  if (rt > c->rws.max_tiles) {
    c->rws.max_tiles = rt;
    TRY(dalloc_t(c, &c->rws.lookback, rt * radix::RADIX));
    CK(cudaMemsetAsync(c->rws.lookback, 0, sizeof(uint64_t) * rt * radix::RADIX, c->st));
  }
  return ensure_scan_tiles(c);
}

// ------------------------------------------------------------------------------ collectives
// Library-owned NCCL (cfg.nccl_id): enqueued on the library stream, ordered by the device,
// no host synchronisation.  Caller callbacks (cfg.comm): synchronise the stream, call, map a
// nonzero return to CC_ERR_COMM.  No-ops on one GPU.
static inline bool multi_gpu(const cc_ctx* c) { return c->dist; }
static inline cc_status comm_allreduce(cc_ctx* c, void* buf, uint64_t count, int dt, int op) {
  if (!multi_gpu(c)) return CC_OK;
  if (c->nccl) {
    std::string e;
    if (nccl::allreduce(c->nccl, buf, count, dt, op, c->st, &e))
      return fail(c, CC_ERR_COMM, "allreduce(count=%llu): %s", (unsigned long long)count, e.c_str());
    return CC_OK;
  }
  CK(cudaStreamSynchronize(c->st));
  if (c->cfg.comm->allreduce(c->cfg.comm->user, buf, count, dt, op, (void*)c->st) != 0)
    return fail(c, CC_ERR_COMM, "allreduce(count=%llu, dtype=%d, op=%d) failed",
                (unsigned long long)count, dt, op);
  return CC_OK;
}
static inline cc_status comm_allgather(cc_ctx* c, const void* send, void* recv, uint64_t bytes) {
  if (!multi_gpu(c)) return CC_OK;
  if (c->nccl) {
    std::string e;
    if (nccl::allgather(c->nccl, send, recv, bytes, c->st, &e))
      return fail(c, CC_ERR_COMM, "allgather(%llu bytes): %s", (unsigned long long)bytes, e.c_str());
    return CC_OK;
  }
  CK(cudaStreamSynchronize(c->st));
  if (c->cfg.comm->allgather(c->cfg.comm->user, send, recv, bytes, (void*)c->st) != 0)
    return fail(c, CC_ERR_COMM, "allgather(%llu bytes) failed", (unsigned long long)bytes);
  return CC_OK;
}
static inline cc_status comm_alltoallv(cc_ctx* c, const void* send, const uint64_t* sb, void* recv,
                                       const uint64_t* rb) {
  if (!multi_gpu(c)) return CC_OK;
  if (c->nccl) {
    std::string e;
    if (nccl::alltoallv(c->nccl, c->cfg.world_size, send, sb, recv, rb, c->st, &e))
      return fail(c, CC_ERR_COMM, "alltoallv: %s", e.c_str());
    return CC_OK;
  }
  CK(cudaStreamSynchronize(c->st));
  if (c->cfg.comm->alltoallv(c->cfg.comm->user, send, sb, recv, rb, (void*)c->st) != 0)
    return fail(c, CC_ERR_COMM, "alltoallv failed");
  return CC_OK;
}
// Failure agreement: every rank contributes its local status (MAX over ranks), so a rank
// that fails locally (allocation, capacity, input checks) never leaves the others blocked in
// the next collective -- all ranks return a failure together (CC_ERR_COMM on the ranks that
// were fine, naming the failing status).  Costs one 8-byte all-reduce and a stream sync.
static inline cc_status comm_agree(cc_ctx* c, cc_status mine) {
  if (!multi_gpu(c)) return mine;
  uint64_t* w = c->d_agree;
  uint64_t v = (uint64_t)mine;
  CK(cudaMemcpyAsync(w, &v, sizeof(uint64_t), cudaMemcpyHostToDevice, c->st));
  TRY(comm_allreduce(c, w, 1, CC_DT_I64, CC_OP_MAX));
  CK(cudaMemcpyAsync(&v, w, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (v == (uint64_t)CC_OK) return CC_OK;
  if (mine != CC_OK) return mine;  // this rank's own error text is already in c->err
  return fail(c, CC_ERR_COMM, "another rank failed with status %llu", (unsigned long long)v);
}
// min over ranks of u32 slots (INF = 0xFFFFFFFF): flip the sign bit so that the signed order of
// the exchanged int32 equals the unsigned order, reduce, flip back
static inline cc_status comm_min_u32(cc_ctx* c, uint32_t* a, uint64_t count) {
  if (!multi_gpu(c)) return CC_OK;
  if (c->nccl) return comm_allreduce(c, a, count, nccl::DT_U32, CC_OP_MIN);  // NCCL has u32 MIN
  csr::flip_sign(a, count, c->st);
  TRY(comm_allreduce(c, a, count, CC_DT_I32, CC_OP_MIN));
  csr::flip_sign(a, count, c->st);
  c->launches += 2;
  return CC_OK;
}
// OR over ranks of a bitmap (NCCL has no bitwise reduction): gather every rank's words, fold
static inline cc_status comm_or_bits(cc_ctx* c, uint32_t* bm, uint64_t words) {
  if (!multi_gpu(c)) return CC_OK;
  const uint64_t need = words * (uint64_t)c->cfg.world_size;
  if (!c->d_gath || c->gath_cap < need) {
    cc_status s = dalloc_t(c, &c->d_gath, need);
    if (s == CC_OK) c->gath_cap = need;
    TRY(comm_agree(c, s));
  }
  TRY(comm_allgather(c, bm, c->d_gath, words * sizeof(uint32_t)));
  csr::or_parts(c->d_gath, words, c->cfg.world_size, bm, c->st);
  c->launches += 1;
  return CC_OK;
}

// Sparse form of the slot exchange for late iterations (few partitions): every rank
// all-gathers its touched (slot, value | NCP bit) entries, padded to the largest list, and
// min-applies everyone's entries to its own copy -- the same result as comm_min_u32 (and
// comm_or_bits for NCP) with volume proportional to the touched partitions.
static inline cc_status comm_sparse_slots(cc_ctx* c, uint32_t* S, uint32_t* BM, uint64_t count) {
  if (!multi_gpu(c)) return CC_OK;
  const uint64_t world = (uint64_t)c->cfg.world_size;
  if (!c->d_xsend || c->xsend_cap < count + 1) {
    cc_status s = dalloc_t(c, &c->d_xsend, count + 1);
    if (s == CC_OK) c->xsend_cap = count + 1;
    TRY(comm_agree(c, s));
  }
  uint64_t* cnt = c->d_gcur + 2052;  // [2052]: my entries, [2053]: max over ranks
  csr::extract_slots(S, BM, count, c->d_xsend, cnt, c->st);
  CK(cudaMemcpyAsync(cnt + 1, cnt, sizeof(uint64_t), cudaMemcpyDeviceToDevice, c->st));
  TRY(comm_allreduce(c, cnt + 1, 1, CC_DT_I64, CC_OP_MAX));
  uint64_t cm[2] = {0, 0};
  CK(cudaMemcpyAsync(cm, cnt, sizeof(cm), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const uint64_t mine = cm[0], pad = cm[1];
  if (pad == 0) return CC_OK;
  if (pad > mine)  // padding entries (slot ~0) up to the common length
    CK(cudaMemsetAsync(c->d_xsend + mine, 0xFF, sizeof(uint2) * (pad - mine), c->st));
  if (!c->d_xrecv || c->xrecv_cap < world * pad + 1) {
    cc_status s = dalloc_t(c, &c->d_xrecv, world * pad + 1);
    if (s == CC_OK) c->xrecv_cap = world * pad + 1;
    TRY(comm_agree(c, s));
  }
  TRY(comm_allgather(c, c->d_xsend, c->d_xrecv, pad * sizeof(uint2)));
  csr::apply_slots(c->d_xrecv, world * pad, S, BM, c->st);
  c->launches += 2;
  return CC_OK;
}

// ------------------------------------------------------------ owner-computes exchange (NEXT-1)
// rank k owns the partition slots [lo, hi) (the same block as its rows).
// After a row pass every rank holds partials for the slots its tuples touched; oc_push sends
// those outside its block to their owner as (slot, value | flag) entries (one all-to-all-v,
// entry counts exchanged first) and the owner min-combines them (and ORs the flag bitmap);
// the owner computes the block's statistics, and oc_reply sends the final value of every
// received slot back to the rank that sent it, in the order sent.  Volume per rank: the
// distinct slots its tuples touch, not n.
static inline cc_status oc_ensure(cc_ctx* c) {
  const uint64_t world = (uint64_t)c->cfg.world_size;
  const uint64_t need = std::max<uint64_t>(c->n, world * c->blk) + 1;
  if (c->oc_cap >= need) return CC_OK;
  cc_status s = CC_OK;
  for (auto* p : {&c->ocA.send, &c->ocB.send, &c->ocT.send, &c->d_ocrecv})
    if (s == CC_OK) s = dalloc_t(c, p, need);
  for (int i = 0; i < 2 && s == CC_OK; i++) s = dalloc_t(c, &c->d_ocval[i], need);
  if (s == CC_OK && !c->d_occnt) s = dalloc_t(c, &c->d_occnt, 2 * world + world * world);
  TRY(comm_agree(c, s));
  c->oc_cap = need;
  return CC_OK;
}
static inline cc_status oc_push(cc_ctx* c, uint32_t* S, uint32_t* BM, cc_ctx::OcSide& side) {
  const int world = c->cfg.world_size, rank = c->cfg.rank;
  uint64_t* cnt = c->d_occnt;
  CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * world, c->st));
  csr::oc_count(S, BM, c->n, c->lo, c->hi, c->blk, world, cnt, c->st);
  side.sc.assign(world, 0);
  CK(cudaMemcpyAsync(side.sc.data(), cnt, sizeof(uint64_t) * world, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  std::vector<uint64_t> cur(world);
  uint64_t o = 0;
  for (int k = 0; k < world; k++) { cur[k] = o; o += side.sc[k]; }
  side.nsend = o;
  CK(cudaMemcpyAsync(cnt + world, cur.data(), sizeof(uint64_t) * world, cudaMemcpyHostToDevice, c->st));
  csr::oc_scatter(S, BM, c->n, c->lo, c->hi, c->blk, cnt + world, side.send, c->st);
  c->launches += 2;
  // every rank's counts -> the counts this rank receives
  CK(cudaMemcpyAsync(cnt, side.sc.data(), sizeof(uint64_t) * world, cudaMemcpyHostToDevice, c->st));
  TRY(comm_allgather(c, cnt, cnt + 2 * world, sizeof(uint64_t) * world));
  std::vector<uint64_t> mat((size_t)world * world);
  CK(cudaMemcpyAsync(mat.data(), cnt + 2 * world, sizeof(uint64_t) * world * world, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  side.rc.assign(world, 0);
  side.nrecv = 0;
  for (int k = 0; k < world; k++) {
    side.rc[k] = mat[(size_t)k * world + rank];
    side.nrecv += side.rc[k];
  }
  if (side.nrecv > c->oc_cap || side.nsend > c->oc_cap)
    return fail(c, CC_ERR_INVALID, "internal: owner exchange of %llu / %llu entries", (unsigned long long)side.nsend,
                (unsigned long long)side.nrecv);
  std::vector<uint64_t> sb(world), rb(world);
  for (int k = 0; k < world; k++) { sb[k] = sizeof(uint2) * side.sc[k]; rb[k] = sizeof(uint2) * side.rc[k]; }
  TRY(comm_alltoallv(c, side.send, sb.data(), c->d_ocrecv, rb.data()));
  csr::oc_apply(c->d_ocrecv, side.nrecv, S, BM, c->st);
  c->launches += 1;
  return CC_OK;
}
static inline cc_status oc_reply(cc_ctx* c, uint32_t* S, const cc_ctx::OcSide& side) {
  const int world = c->cfg.world_size;
  csr::oc_gather(c->d_ocrecv, side.nrecv, S, c->d_ocval[1], c->st);
  std::vector<uint64_t> sb(world), rb(world);
  for (int k = 0; k < world; k++) { sb[k] = sizeof(uint32_t) * side.rc[k]; rb[k] = sizeof(uint32_t) * side.sc[k]; }
  TRY(comm_alltoallv(c, c->d_ocval[1], sb.data(), c->d_ocval[0], rb.data()));
  csr::oc_put(side.send, side.nsend, c->d_ocval[0], S, c->st);
  c->launches += 2;
  return CC_OK;
}

// u64 relabel through the hash table (relabel::run_hash), growing the table to the full size
// only if the first, small attempt overflowed (no 2m-sized table at load)
static inline cc_status relabel_hash(cc_ctx* c, uint64_t k, uint64_t* total) {
  uint32_t* vals[2] = {c->d_q[0], c->d_q[1]};
  uint64_t* scratch = c->d_gctr + graph::G_NUM + 1540;
  int r = relabel::run_hash(c->d_ids64, k, c->d_htab, c->htab_slots, false, c->d_w, vals, c->rws,
                            reinterpret_cast<uint32_t*>(c->d_edges), c->d_uids, total, scratch, c->st, &c->launches);
  if (r == 1) {
    const uint64_t need = relabel::hash_slots(k) + 1;
    TRY(dalloc_t(c, &c->d_htab, need));
    c->htab_slots = need;
    r = relabel::run_hash(c->d_ids64, k, c->d_htab, c->htab_slots, true, c->d_w, vals, c->rws,
                          reinterpret_cast<uint32_t*>(c->d_edges), c->d_uids, total, scratch, c->st, &c->launches);
  }
  if (r) return fail(c, CC_ERR_INVALID, "internal: relabel hash table");
  return CC_OK;
}

// Prediction stage on the host (cc_api.cu): gate fit and route from the device statistics.
cc_status predict_gate(cc_ctx* c, cc_mode mode, bool want_hist, bool* run_bfs, uint64_t* root);

// Alg. 1 iterations of the r-stationary engine on a built tuple array (cc_api.cu); with
// world_size > 1 the partition slots are combined across ranks after each row pass.
cc_status sv_iterate(cc_ctx* c, uint64_t A, uint64_t len, uint64_t A_local);

// Edge-streaming BFS peel over this rank's edges (cc_api.cu; replicated state, found bitmaps
// OR-ed over ranks): remainder edges out, visited bitmap in d_bm[0], labels of VI written.
cc_status bfs_stream(cc_ctx* c, uint64_t root, bool spec_ok, const uint2** rem, uint64_t* m_rem,
                     cudaEvent_t* e_bfs);

// cc_run for world_size > 1 (cc_dist.cu).
cc_status run_dist(cc_ctx* c, cc_mode mode);

// 'Balanced' variant (cc_dist.cu; CC_FLAG_BALANCE): even redistribution of the live rows
// (R, P of `len` tuples) over the ranks into (Rdst, Pdst); loads[2k] = rank k's live tuples,
// loads[2k + 1] = its tuple capacity.  Collective; *moved = false if the plan was skipped.
cc_status rebalance_rows(cc_ctx* c, const uint32_t* Rsrc, const uint32_t* Psrc, uint32_t* Rdst,
                         uint32_t* Pdst, uint64_t len, const std::vector<uint64_t>& loads,
                         uint64_t* new_len, bool* moved);

// n-sized buffers and the owned vertex block for id range n (cc_api.cu).
cc_status alloc_vertex_buffers(cc_ctx* c, uint64_t n);

// u64 ids with world_size > 1 (relabel_dist.cu): the distributed relabel of Alg. 2 line 4
// (dense ids in id order over all ranks, edges rewritten as u32, n-sized buffers allocated),
// and the collective label output of a rank's block as (original id, original label) pairs.
cc_status dist_relabel(cc_ctx* c);
cc_status dist_labels_u64(cc_ctx* c, uint64_t* ids, uint64_t* labels, int out_on_device);
