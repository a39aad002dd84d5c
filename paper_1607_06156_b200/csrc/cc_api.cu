// cc_api.cu -- the C ABI (include/cc.h) and the Alg. 2 driver.
//
// cc_run(mode):
//   prediction : degrees + degree distribution on device, gate on host   (Alg. 2 lines 2-3)
//   BFS route  : edge-streaming bitmap BFS from the max-degree root, label the visited
//                component with its min id, filter its edges            (lines 7-11)
//   SV         : Alg. 1 on the remaining edges, four regroups per iteration with
//                completed-partition exclusion
// All compute runs in the kernels of radix.cu / sv.cu / graph.cu; the host only sequences
// launches and reads small counters (one sync per SV iteration, one per BFS level).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cc.h"
#include "gate.h"
#include "graph.cuh"
#include "radix.cuh"
#include "sv.cuh"
#include "csr.cuh"
#include "relabel.cuh"
#include "ctx.cuh"
#include "bfs.cuh"

using namespace cc;

#define CC_VERSION_STR "cc-b200 0.1.0 (sm_100a)"

extern "C" {

const char* cc_version(void) { return CC_VERSION_STR; }

const char* cc_status_string(cc_status s) {
  switch (s) {
    case CC_OK: return "CC_OK";
    case CC_ERR_INVALID: return "CC_ERR_INVALID";
    case CC_ERR_RANGE: return "CC_ERR_RANGE";
    case CC_ERR_NOMEM: return "CC_ERR_NOMEM";
    case CC_ERR_CUDA: return "CC_ERR_CUDA";
    case CC_ERR_COMM: return "CC_ERR_COMM";
    case CC_ERR_STATE: return "CC_ERR_STATE";
    case CC_ERR_NOCONV: return "CC_ERR_NOCONV";
  }
  return "CC_ERR_UNKNOWN";
}

const char* cc_last_error(const cc_ctx* c) { return c ? c->err.c_str() : "null context"; }

uint64_t cc_last_launch_count(const cc_ctx* c) { return c ? c->launches : 0; }

cc_status cc_set_profiling(cc_ctx* c, int on) {
  if (!c) return CC_ERR_INVALID;
  if (on) c->cfg.flags |= CC_FLAG_PROFILE;
  else c->cfg.flags &= ~CC_FLAG_PROFILE;
  return CC_OK;
}

cc_status cc_get_unique_id(void* out128, char* why, size_t why_len) {
  if (!out128) return CC_ERR_INVALID;
  std::string e;
  if (nccl::unique_id(out128, &e)) {
    if (why && why_len) std::snprintf(why, why_len, "%s", e.c_str());
    return CC_ERR_COMM;
  }
  return CC_OK;
}

cc_status cc_init(const cc_config* cfg, cc_ctx** out) {
  if (!cfg || !out) return CC_ERR_INVALID;
  *out = nullptr;
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size) return CC_ERR_INVALID;
  if (cfg->world_size > 1 && !cfg->nccl_id &&
      (!cfg->comm || !cfg->comm->allreduce || !cfg->comm->allgather || !cfg->comm->alltoallv))
    return CC_ERR_INVALID;  // multi-GPU contexts need NCCL or the caller's collectives
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    return CC_ERR_CUDA;
  }
  if (cfg->device < 0 || cfg->device >= ndev) return CC_ERR_INVALID;
  if (cudaSetDevice(cfg->device) != cudaSuccess) return CC_ERR_CUDA;
  cc_ctx* c = new cc_ctx();
  c->cfg = *cfg;
  if (c->cfg.tau <= 0) c->cfg.tau = 0.05;
  if (cfg->nccl_id) {
    std::string e;
    if (nccl::init(&c->nccl, cfg->nccl_id, cfg->world_size, cfg->rank, cfg->device, &e)) {
      std::fprintf(stderr, "cc_init: %s\n", e.c_str());
      delete c;
      return CC_ERR_COMM;
    }
  }
  c->dist = cfg->world_size > 1 || c->nccl != nullptr;
  c->st = (cudaStream_t)cfg->stream;
  if (cudaMallocHost(&c->h_ctr, sizeof(uint64_t) * (sv::C_NUM + graph::G_NUM + 8)) != cudaSuccess ||
      cudaMallocHost(&c->h_ctr2, sizeof(uint64_t) * 2 * sv::C_NUM) != cudaSuccess ||
      cudaMallocHost(&c->h_hist, sizeof(uint32_t) * (graph::HIST_DENSE + graph::TAIL_CAP)) !=
          cudaSuccess) {
    if (c->h_ctr) cudaFreeHost(c->h_ctr);
    if (c->h_ctr2) cudaFreeHost(c->h_ctr2);
    if (c->h_hist) cudaFreeHost(c->h_hist);
    if (c->nccl) nccl::destroy(c->nccl);
    delete c;
    return CC_ERR_NOMEM;
  }
  c->h_gctr = c->h_ctr + sv::C_NUM;
  c->h_word = reinterpret_cast<uint32_t*>(c->h_gctr + graph::G_NUM);
  if (cudaMalloc(&c->d_agree, 2 * sizeof(uint64_t)) != cudaSuccess) {
    cudaGetLastError();
    cudaFreeHost(c->h_ctr);
    cudaFreeHost(c->h_ctr2);
    cudaFreeHost(c->h_hist);
    if (c->nccl) nccl::destroy(c->nccl);
    delete c;
    return CC_ERR_NOMEM;
  }
  *out = c;
  return CC_OK;
}

cc_status cc_destroy(cc_ctx* c) {
  if (!c) return CC_ERR_INVALID;
  cudaSetDevice(c->cfg.device);
  dfree_all(c);
  cudaStreamSynchronize(c->st);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->h_ctr) cudaFreeHost(c->h_ctr);
  if (c->h_ctr2) cudaFreeHost(c->h_ctr2);
  if (c->h_hist) cudaFreeHost(c->h_hist);
  if (c->d_agree) cudaFree(c->d_agree);
  if (c->nccl) nccl::destroy(c->nccl);
  delete c;
  return CC_OK;
}

}  // extern "C"

// n-sized buffers (labels, degrees, bitmaps, partition slots) and the owned vertex block:
// at load time, or after the distributed u64 relabel once the global id count is known
cc_status alloc_vertex_buffers(cc_ctx* c, uint64_t n) {
  const uint64_t world = (uint64_t)c->cfg.world_size;
  const uint64_t nw = (n + 31) / 32 + 1;
  c->n = n;
  c->n_alloc = n;
  c->kbits = bits_for(n);
  TRY(dalloc_t(c, &c->d_label, n + 1));
  TRY(dalloc_t(c, &c->d_deg, n + 1));
  // owned vertex block (multi-GPU): blk = 32 * ceil(n / (32 * world))
  c->blk = std::max<uint64_t>(32, (n + 32 * world - 1) / (32 * world) * 32);
  c->lo = std::min<uint64_t>(n, c->blk * (uint64_t)c->cfg.rank);
  c->hi = world > 1 ? std::min<uint64_t>(n, c->lo + c->blk) : n;
  if (world == 1) c->lo = 0;
  const uint64_t bmw = std::max<uint64_t>(2 * nw, world * c->blk / 32) + 2;
  for (int i = 0; i < 3; i++) TRY(dalloc_t(c, &c->d_bm[i], bmw));  // 2-bit BFS state fits
  for (int i = 0; i < 3; i++) TRY(dalloc_t(c, &c->d_sbm[i], nw + 2));
  TRY(dalloc_t(c, &c->d_segA, n + 64));  // padded: the slot scans read 4 slots per thread
  TRY(dalloc_t(c, &c->d_segB, n + 64));
  TRY(dalloc_t(c, &c->d_umin, n + 1));
  TRY(dalloc_t(c, &c->d_umax, n + 1));
  TRY(dalloc_t(c, &c->d_plist[0], n + 1));
  TRY(dalloc_t(c, &c->d_plist[1], n + 1));
  TRY(dalloc_t(c, &c->d_plcnt, 2));
  TRY(dalloc_t(c, &c->d_nx, nw + 2));
  TRY(dalloc_t(c, &c->d_hw, n + 1));
  CK(cudaMemsetAsync(c->d_umin, 0xFF, sizeof(uint64_t) * (n + 1), c->st));
  CK(cudaMemsetAsync(c->d_umax, 0, sizeof(uint64_t) * (n + 1), c->st));
  return ensure_scan_tiles(c);
}

// Device buffers of a load (local: a rank's own m); the caller agrees on the outcome over
// the ranks, so a rank that cannot allocate never leaves the others in a collective.
static cc_status load_buffers(cc_ctx* c, cc_idw w, uint64_t m, uint64_t n, bool dist64) {
  if (2 * m + 2 * n >= (1ull << 32))
    return fail(c, CC_ERR_INVALID, "tuple count 2m+2n exceeds 2^32 on one GPU");
  CK(cudaSetDevice(c->cfg.device));
  dfree_all(c);
  c->loaded = c->ran = false;
  c->idw = w;
  c->n = n;
  c->n_alloc = 0;
  c->m = m;
  c->kbits = bits_for(n);
  c->cap = (2 * m + 2 * n + 64 + 1023) & ~1023ull;  // keeps P = R + cap 16-byte aligned
  const uint64_t world = (uint64_t)c->cfg.world_size;
  TRY(dalloc_t(c, &c->d_edges, m + 1));
  TRY(dalloc_t(c, &c->d_hist, graph::HIST_DENSE));
  TRY(dalloc_t(c, &c->d_hpairs, graph::HIST_DENSE));
  TRY(dalloc_t(c, &c->d_tail, graph::TAIL_CAP));
  for (int i = 0; i < 2; i++) {
    TRY(dalloc_t(c, &c->d_w[i], c->cap));
    TRY(dalloc_t(c, &c->d_q[i], c->cap));
  }
  TRY(dalloc_t(c, &c->d_lsegs, csr::long_seg_cap(c->cap)));
  TRY(dalloc_t(c, &c->d_nlsegs, 2));
  if (multi_gpu(c)) {
    TRY(dalloc_t(c, &c->d_send, 2 * m + 1));
    TRY(dalloc_t(c, &c->d_cnt, 2 * world + world * world));
  }
  TRY(dalloc_t(c, &c->d_ctr, 2 * sv::C_NUM));  // two alternating blocks (SV look-ahead)
  TRY(dalloc_t(c, &c->d_gctr, graph::G_NUM + 512 + 1024 + 8));  // + relabel scratch
  TRY(dalloc_t(c, &c->d_garc, 2048 + 8));
  TRY(dalloc_t(c, &c->d_gcur, 2048 + 8));
  if (w == CC_U64) {
    TRY(dalloc_t(c, &c->d_ids64, 2 * m + 1));
    TRY(dalloc_t(c, &c->d_uids, 2 * m + 1));
    c->htab_slots = 0;
    if (relabel::hash_slots(2 * m)) {
      c->htab_slots = relabel::hash_first_slots(2 * m) + 1;
      TRY(dalloc_t(c, &c->d_htab, c->htab_slots));
    }
    if (c->cfg.flags & CC_FLAG_PERMUTE_IDS) {
      TRY(dalloc_t(c, &c->d_mix, n + 1));
      TRY(dalloc_t(c, &c->d_pi, n + 1));
    }
  }
  c->rws.max_tiles = c->cap / radix::TILE_MIN + 2;
  TRY(dalloc_t(c, &c->rws.ghist, radix::MAX_PASSES * radix::RADIX));
  TRY(dalloc_t(c, &c->rws.lookback, c->rws.max_tiles * radix::RADIX));
  TRY(dalloc_t(c, &c->rws.tile_ctr, radix::MAX_PASSES));
  TRY(dalloc_t(c, &c->ss.ticket, 4));
  CK(cudaMemsetAsync(c->rws.lookback, 0, sizeof(uint64_t) * c->rws.max_tiles * radix::RADIX, c->st));
  if (!dist64) TRY(alloc_vertex_buffers(c, n));
  else TRY(ensure_scan_tiles(c));
  return CC_OK;
}

extern "C" {

cc_status cc_load_edges(cc_ctx* c, cc_idw w, const void* pairs, uint64_t m, uint64_t n, int on_dev) {
  NvtxRange nv_load("cc_load_edges");
  if (!c) return CC_ERR_INVALID;
  if (m && !pairs) return fail(c, CC_ERR_INVALID, "pairs is NULL");
  if (w != CC_U32 && w != CC_U64) return fail(c, CC_ERR_INVALID, "bad id width %d", (int)w);
  // u64 ids over several ranks: the global id count is known only after the distributed
  // relabel in cc_run, which then allocates the n-sized buffers (relabel_dist.cu)
  const bool dist64 = w == CC_U64 && multi_gpu(c);
  if (dist64 && (c->cfg.flags & CC_FLAG_PERMUTE_IDS))
    return fail(c, CC_ERR_INVALID, "CC_FLAG_PERMUTE_IDS is single-GPU in this build");
  if (w == CC_U64) {
    if (n != 0) return fail(c, CC_ERR_INVALID, "u64 ids: n_vertices must be 0");
    n = std::min<uint64_t>(2 * m, 1ull << 30);  // bound on distinct ids (checked in cc_run)
  }
  if (n > (1ull << 30)) return fail(c, CC_ERR_INVALID, "n_vertices %llu > 2^30", (unsigned long long)n);
  TRY(comm_agree(c, load_buffers(c, w, m, n, dist64)));
  if (w == CC_U64) {
    if (m)
      CK(cudaMemcpyAsync(c->d_ids64, pairs, 2 * m * sizeof(uint64_t),
                         on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
    c->m_total = m;
    if (dist64) {  // every rank learns the global edge count
      CK(cudaMemcpyAsync(c->d_gctr + graph::G_REMAIN, &c->m_total, sizeof(uint64_t), cudaMemcpyHostToDevice,
                         c->st));
      TRY(comm_allreduce(c, c->d_gctr + graph::G_REMAIN, 1, CC_DT_I64, CC_OP_SUM));
      CK(cudaMemcpyAsync(&c->m_total, c->d_gctr + graph::G_REMAIN, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                         c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    c->loaded = true;
    return CC_OK;
  }
  if (m)
    CK(cudaMemcpyAsync(c->d_edges, pairs, m * sizeof(uint2),
                       on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
  // validate ids < n on device
  CK(cudaMemsetAsync(c->d_gctr, 0, sizeof(uint64_t) * graph::G_NUM, c->st));
  graph::launch_validate(c->d_edges, m, n, c->d_gctr, c->st);
  CKL();
  CK(cudaMemcpyAsync(c->h_gctr, c->d_gctr, sizeof(uint64_t) * graph::G_NUM, cudaMemcpyDeviceToHost, c->st));
  // every rank learns whether any rank's ids were out of range, and the global edge count
  TRY(comm_allreduce(c, c->d_gctr + graph::G_ERR, 1, CC_DT_I64, CC_OP_MAX));
  c->m_total = m;
  if (multi_gpu(c)) {
    CK(cudaMemcpyAsync(c->d_gctr + graph::G_REMAIN, &c->m_total, sizeof(uint64_t), cudaMemcpyHostToDevice,
                       c->st));
    TRY(comm_allreduce(c, c->d_gctr + graph::G_REMAIN, 1, CC_DT_I64, CC_OP_SUM));
  }
  CK(cudaMemcpyAsync(c->h_gctr, c->d_gctr, sizeof(uint64_t) * graph::G_NUM, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (multi_gpu(c)) c->m_total = c->h_gctr[graph::G_REMAIN];
  if (c->h_gctr[graph::G_ERR]) return fail(c, CC_ERR_RANGE, "edge endpoint >= n_vertices");
  c->loaded = true;
  return CC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------ stages
static int do_sort(cc_ctx* c, int cur, uint64_t n, bool pairs) {
  Prof pr(c, KF_RADIX);
  int r = radix::sort_pairs(c->rws, c->d_w, c->d_q, cur, n, c->kbits, pairs, c->st, &c->launches);
  const int P = radix::num_passes(c->kbits);
  // algorithmic bytes: the histogram reads the key word once, each pass reads and writes
  // the element once (8 B word + 4 B payload for the by-p regroups)
  pr.end((double)n * (8.0 + P * 2.0 * (pairs ? 12.0 : 8.0)), (uint64_t)(P + 1));
  return r;
}

// Alg. 1 with direct-addressed buckets (sv_direct.cu): same passes, no tuple movement
// except the compaction of the partition passes.
static cc_status run_sv_direct(cc_ctx* c, uint64_t A, int cur) {
  const uint64_t n = c->n;
  const uint64_t nw = (n + 31) / 32;
  uint32_t *umin = c->d_segA, *pmin = c->d_segB;
  uint32_t *notpc = c->d_sbm[0], *ncp = c->d_sbm[1], *head = c->d_sbm[2];
  const uint32_t max_iter = 2 * (uint32_t)c->kbits + 8;
  uint64_t chg2_prev = 0;
  for (uint32_t it = 0;; it++) {
    if (it >= max_iter) return fail(c, CC_ERR_NOCONV, "SV did not converge in %u iterations", max_iter);
    cudaEvent_t ev_it = ev_get(c);
    CK(cudaEventRecord(ev_it, c->st));
    cudaEvent_t a = nullptr;
    seg_begin(c, &a);
    // ---- lines 8-13: u_min per vertex bucket, 'potentially completed'
    CK(cudaMemsetAsync(umin, 0xFF, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(notpc, 0, sizeof(uint32_t) * nw, c->st));
    sv::launch_direct_vmin(c->d_w[cur], A, umin, c->st);
    sv::launch_direct_vpc(c->d_w[cur], A, umin, notpc, c->st);
    // ---- lines 14-22: p_min per partition bucket, completion, exclusion, temporaries
    CK(cudaMemsetAsync(pmin, 0xFF, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(ncp, 0, sizeof(uint32_t) * nw, c->st));
    CK(cudaMemsetAsync(head, 0, sizeof(uint32_t) * nw, c->st));
    CK(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint64_t) * (sv::C_TEMPS + 1), c->st));
    sv::launch_direct_pmin(true, c->d_w[cur], A, umin, notpc, pmin, ncp, c->st);
    sv::launch_direct_papply(true, c->d_w[cur], A, pmin, ncp, head, c->d_w[cur ^ 1], c->d_label,
                             c->d_ctr, c->st);
    c->launches += 4;
    cur ^= 1;
    CKL();
    TRY(sync_read(c));
    const uint64_t out = c->h_ctr[sv::C_OUT];
    const uint64_t T = c->h_ctr[sv::C_TEMPS];
    const uint64_t A1 = out - T;
    cc_iter_stat s{};
    s.active_in = A;
    s.active_min = s.active_max = A;
    s.partitions = c->h_ctr[sv::C_PARTITIONS];
    s.completed = c->h_ctr[sv::C_COMPLETED];
    s.changed = c->h_ctr[sv::C_CHANGED];
    s.temps = T;
    if (!c->iters.empty()) {
      c->iters.back().changed2 = c->h_ctr[sv::C_CHANGED2] - chg2_prev;
      chg2_prev = c->h_ctr[sv::C_CHANGED2];
    }
    c->iters.push_back(s);
    c->it_ev.push_back(ev_it);
    if (out == 0) {
      seg_end(c, a, (double)A * 32, 4);
      break;
    }
    // ---- line 24 (redo 8-13 with temporaries) and line 25 (redo 14-21), lines 26-28
    CK(cudaMemsetAsync(umin, 0xFF, sizeof(uint32_t) * n, c->st));
    sv::launch_direct_vmin(c->d_w[cur], out, umin, c->st);
    CK(cudaMemsetAsync(pmin, 0xFF, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(head, 0, sizeof(uint32_t) * nw, c->st));
    CK(cudaMemsetAsync(c->d_ctr + sv::C_OUT, 0, sizeof(uint64_t), c->st));
    sv::launch_direct_pmin(false, c->d_w[cur], out, umin, nullptr, pmin, nullptr, c->st);
    sv::launch_direct_papply(false, c->d_w[cur], out, pmin, nullptr, head, c->d_w[cur ^ 1],
                             c->d_label, c->d_ctr, c->st);
    c->launches += 3;
    cur ^= 1;
    CKL();
    // algorithmic bytes of the streamed tuple words (8 B per read / write)
    seg_end(c, a, (double)A * 32 + (double)out * (8 + 24) + (double)A1 * 8, 7);
    A = A1;
    if (A == 0) break;
  }
  TRY(sync_read(c));
  if (!c->iters.empty()) c->iters.back().changed2 = c->h_ctr[sv::C_CHANGED2] - chg2_prev;
  return CC_OK;
}

// Alg. 1, r-stationary engine (sv_csr.cu): one counting regroup by r (CSR build), then
// per iteration: vertex pass, partition pass, partition statistics + temporaries,
// ordered exclusion of completed partitions; second vertex/partition pass in place.
static cc_status run_sv_csr(cc_ctx* c, const uint2* edges, uint64_t m_sv, const uint32_t* vis) {
  const uint64_t n = c->n;
  uint32_t* R[2] = {reinterpret_cast<uint32_t*>(c->d_w[0]), reinterpret_cast<uint32_t*>(c->d_w[1])};
  uint32_t* P[2] = {R[0] + c->cap, R[1] + c->cap};
  uint32_t *off = c->d_q[0], *cur = c->d_q[1];
  CK(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint64_t) * sv::C_NUM, c->st));
  cudaEvent_t a = nullptr;
  seg_begin(c, &a);
  TRY(scan_epoch_guard(c));
  const int gshift = csr::group_shift(n, 2 * m_sv + n);
  uint32_t* garc = c->d_garc;
  uint64_t* gcur = c->d_gcur;
  uint64_t* nlong = gcur + 2048;
  csr::build(edges, m_sv, c->d_deg, vis, n, off, cur, garc, gshift, c->ss, c->d_ctr, c->st);
  c->launches += 1;
  CKL();
  TRY(sync_read(c));
  uint64_t A = c->h_ctr[sv::C_VT_OUT];  // live tuples (A_i)
  if (A == 0) return CC_OK;
  if (A > c->cap) return fail(c, CC_ERR_INVALID, "tuple count %llu exceeds capacity", (unsigned long long)A);
  // scratch: the bucketed arc list lives in the second tuple buffer (free until the first
  // compaction), the long-row list in the PMIN slots (free until the first partition pass)
  csr::fill(edges, m_sv, off, cur, n, A, R[0], P[0], garc, gshift, gcur,
            reinterpret_cast<uint2*>(c->d_w[1]), c->d_segB, nlong, c->st);
  c->launches += 5;
  CKL();
  seg_end(c, a, 4.0 * n + 8.0 * m_sv + 8.0 * A + 4.0 * n, 6, KF_CSR);
  return sv_iterate(c, A, A, A);
}

// Alg. 1 iterations on the tuple array in buffer 0 (R, P), `len` entries of which A (summed
// over ranks) are live.  Multi-GPU: rows are owned (r in this rank's block), partitions are
// global, so after each row pass the partition slots are combined across ranks (min of the
// minima, OR of the NCP bitmap) and every rank derives identical statistics and temporaries.
cc_status sv_iterate(cc_ctx* c, uint64_t A, uint64_t len, uint64_t A_local) {
  const uint64_t n = c->n;
  const uint64_t nw = (n + 31) / 32;
  const bool multi = multi_gpu(c);
  uint32_t* R[2] = {reinterpret_cast<uint32_t*>(c->d_w[0]), reinterpret_cast<uint32_t*>(c->d_w[1])};
  uint32_t* P[2] = {R[0] + c->cap, R[1] + c->cap};
  int cb = 0;  // buffer holding the tuple array
  const uint32_t max_iter = 2 * (uint32_t)c->kbits + 8;
  // slot arrays: PA (pass A minima), PB (pass B minima), NCP / TB bitmaps.  The slot scans
  // clear what the next pass needs, so these are the only full clears of the run.
  uint32_t *PA = c->d_segA, *PB = c->d_segB, *NCP = c->d_sbm[1], *TB = c->d_sbm[2];
  // P is double-buffered across passes: the P half of the current tuple buffer and the
  // (free after the CSR build) offsets array
  uint32_t *Pc = P[0], *Palt = c->d_q[0];
  // rows longer than csr::LONG exist only if some degree reaches LONG
  const bool have_long = c->rep.max_degree + 1 > csr::LONG;
  if (have_long) csr::longlist(R[0], P[0], len, c->d_deg, c->d_lsegs, c->d_nlsegs, c->st);
  const uint64_t n4 = (n + 3) / 4 * 4;
  const uint64_t nwp = nw + 2;
  CK(cudaMemsetAsync(PA, 0xFF, sizeof(uint32_t) * n4, c->st));
  CK(cudaMemsetAsync(PB, 0xFF, sizeof(uint32_t) * n4, c->st));
  CK(cudaMemsetAsync(NCP, 0, sizeof(uint32_t) * nwp, c->st));
  CK(cudaMemsetAsync(TB, 0, sizeof(uint32_t) * nwp, c->st));
  // slot scans after iteration 0 visit only the partition list L_i (lcur: L[lb] holds L_i;
  // lprev: L[lb ^ 1] holds L_i-1)
  uint32_t* NX = c->d_nx;
  uint32_t* L[2] = {c->d_plist[0], c->d_plist[1]};
  uint64_t* LC = c->d_plcnt;
  int lb = 0;
  bool lcur = false, lprev = false, lexact = false;
  CK(cudaMemsetAsync(NX, 0, sizeof(uint32_t) * nwp, c->st));
  // exclusion of completed partitions (fig:loadbal variants)
  const bool excl = !(c->cfg.flags & CC_FLAG_NO_EXCLUDE);
  const bool temps_all = !excl || (c->cfg.flags & CC_FLAG_NO_EARLY_EXCLUDE);
  // pstat2 marks P_i+1 exactly (and PA is preset) unless completed partitions keep their
  // temporaries while their tuples leave (CC_FLAG_NO_EARLY_EXCLUDE)
  const bool exact_next = !(excl && temps_all);
  // Look-ahead (one GPU, with exclusion): iteration i+1 is enqueued before the host reads
  // iteration i's counters, so the host round trip overlaps device work.  Its row passes pick
  // the hot variant, or nothing at all once iteration i left no live tuple, from those
  // counters on the device; counters alternate between two blocks.  Compaction (rare) is a
  // synchronisation point.  Several ranks, or no exclusion, run step by step.
  const bool ahead = !multi && excl;
  // iteration 0's pass A by pull (csr::rowpass_a0_pull; one GPU: the pull reads the u_min of
  // rows other ranks own).  The CSR offsets are still in d_q[0] then.  CC_PULL0=0: the push
  // (C2 5.61 -> 5.53 ms, C3 6.03 -> 5.92 ms, C4 mode sv 225 -> 205 ms with the pull)
  const char* p0 = getenv("CC_PULL0");
  const bool pull0 = !multi && !(p0 && p0[0] == '0');
  // several ranks: the owner-computes slot exchange (NEXT-1, ctx.cuh oc_push / oc_reply) unless
  // the dense all-reduce is asked for (CC_FLAG_DENSE_EXCHANGE), or completed partitions keep
  // temporaries, or rows leave their owner (balanced variant: TB(r) must reach the row holder)
  const bool oc = multi && excl && !temps_all && !(c->cfg.flags & (CC_FLAG_DENSE_EXCHANGE | CC_FLAG_BALANCE));
  if (oc) TRY(oc_ensure(c));
  const uint64_t nwl = c->lo / 32, nwh = (c->hi + 31) / 32;  // own words of the slot bitmaps
  uint64_t* CTR[2] = {c->d_ctr, c->d_ctr + sv::C_NUM};
  cudaEvent_t ev_read[2] = {ev_get(c), ev_get(c)};
  // hot thresholds measured on C2 (iterations with 490 k / 112 k / 16 k previous partitions):
  // pass A gains from the block tables below 1/512 partitions per live tuple, pass B below 1/128.
  // Iteration 0 has no previous counters: its pass B selects on the distinct slots it will
  // update (the p_min targets k_pstat1 counted, C_TDIST) -- on power-law graphs most
  // partitions join a few hubs' minima at once (C4 mode sv: 11 k targets for 2.2 G tuples,
  // cold pass B 223 ms serialised on those slots)
  // CC_HOT_SEL=1: select on the slot targets of this iteration instead (|P_i| for pass A, the
  // distinct p_min targets for pass B; csr.cuh rowpass), thresholds $CC_HOT_A / $CC_HOT_B
  const char* hs = getenv("CC_HOT_SEL");
  const bool hot_cur = hs && hs[0] == '1';
  const char* ha = getenv("CC_HOT_A");
  const char* hb = getenv("CC_HOT_B");
  const int HOT_A = ha ? atoi(ha) : 9, HOT_B = hb ? atoi(hb) : 7;
  uint32_t next_enq = 0;
  // Row collapse (one GPU, paper exclusion): once partitions are large, most rows are PC and
  // stay PC; collapse() folds each to its head tuple, so later passes stream ~one tuple per
  // vertex.  hidden = folded tuples of the rows still live (A_i = live tuples + hidden).
  const bool can_collapse = !multi && excl && !temps_all && !(c->cfg.flags & CC_FLAG_NO_COLLAPSE);
  bool collapse_ok = can_collapse, hw_ready = false, pending_collapse = false;
  uint64_t hidden = 0;
  uint32_t last_collapse = 0;
  // CC_COLLAPSE_FORCE=1 (tests): collapse after every iteration from the first, at any size
  const char* cf = getenv("CC_COLLAPSE_FORCE");
  const bool collapse_force = cf && cf[0] == '1';
  const uint64_t COLLAPSE_MIN_LEN = collapse_force ? 0 : (1ull << 16);
  auto enqueue = [&](uint32_t it) -> cc_status {
    NvtxRange nv_it("SV iteration (Alg. 1 lines 8-25)");
    cudaEvent_t ev_it = ev_get(c);
    CK(cudaEventRecord(ev_it, c->st));
    c->it_ev.push_back(ev_it);
    cudaEvent_t a = nullptr;
    seg_begin(c, &a);
    uint64_t* ctr = CTR[it & 1];
    const uint64_t* prevctr = it ? CTR[(it - 1) & 1] : nullptr;
    // the last known partition count (byte models; the sparse exchange of several ranks, which
    // run step by step so it is the previous iteration's)
    const uint64_t prevp = c->iters.empty() ? n : c->iters.back().partitions;
    uint32_t* Rc = R[cb];
    CK(cudaMemsetAsync(ctr, 0, sizeof(uint64_t) * (sv::C_SURVIVORS + 1), c->st));
    // ---- lines 8-16 (+ line 25 relabel of the previous iteration)
    { Prof k(c, KF_ROWA);
      if (it == 0 && pull0)
        csr::rowpass_a0_pull(c->d_q[0], Pc, n, PB, PA, NCP, c->d_umin, c->d_umax, ++c->row_tag, c->d_lsegs,
                             c->d_nlsegs, have_long, c->st);
      else
        csr::rowpass(true, Rc, Pc, it ? Palt : nullptr, len, it ? PB : nullptr, nullptr, nullptr, PA,
                     NCP, c->d_label, c->d_umin, c->d_umax, ++c->row_tag, c->d_lsegs, c->d_nlsegs,
                     have_long, false, ctr, c->st, true, /*preset=*/lexact, prevctr, HOT_A, nullptr,
                     hot_cur && lcur ? LC + lb : nullptr, 0);
      k.end(8.0 * len + (it ? 4.0 * len : 0.0), 1 + (have_long ? 2 : 0)); }
    if (it) std::swap(Pc, Palt);
    if (oc) {
      // ---- owner-computes (NEXT-1): the relabel read PB; clear the other owners' replies,
      // send the partials of foreign slots to their owners, statistics of the own block
      if (it) csr::oc_put(c->ocB.send, c->ocB.nsend, nullptr, PB, c->st);
      TRY(oc_push(c, PA, NCP, c->ocA));
      { Prof k(c, KF_SLOTS);
        csr::pstat1_block(PA, NCP, c->lo, c->hi, TB, PB, ctr, c->st);
        k.end(8.0 * (double)(c->hi - c->lo), 1); }
      CK(cudaMemsetAsync(NCP, 0, sizeof(uint32_t) * nwp, c->st));
      TRY(comm_allreduce(c, ctr + sv::C_PARTITIONS, 4, CC_DT_I64, CC_OP_SUM));
      // p_min (with the completed flag) back to the ranks holding those partitions; the
      // temporaries' targets to the owners of their rows
      TRY(oc_reply(c, PA, c->ocA));
      TRY(oc_push(c, nullptr, TB, c->ocT));
      if (nwl) CK(cudaMemsetAsync(TB, 0, sizeof(uint32_t) * nwl, c->st));
      if (nwp > nwh) CK(cudaMemsetAsync(TB + nwh, 0, sizeof(uint32_t) * (nwp - nwh), c->st));
    }
    // sparse exchange once few partitions remain: the entries all ranks touched (at most
    // |P_i-1| per rank) cost less than the dense n-slot reduction
    const bool sparse = multi && !oc && it > 0 && prevp * (uint64_t)c->cfg.world_size * 2 < n4;
    if (multi && !oc) {  // partition minima and 'not completed' flags over all ranks
      if (sparse) {
        TRY(comm_sparse_slots(c, PA, NCP, n4));
      } else {
        TRY(comm_min_u32(c, PA, n4));
        TRY(comm_or_bits(c, NCP, nwp));
      }
    }
    // ---- line 22 bookkeeping: |P_i|, completed, changed, temporaries
    if (!oc) {
      Prof k(c, KF_SLOTS);
      if (lcur) csr::pstat1(PA, NCP, n, TB, PB, ctr, c->st, temps_all, excl, L[lb], LC + lb,
                            lprev ? L[lb ^ 1] : nullptr, lprev ? LC + (lb ^ 1) : nullptr);
      else csr::pstat1(PA, NCP, n, TB, PB, ctr, c->st, temps_all, excl);
      k.end(lcur ? 12.0 * (double)prevp : 8.0 * n4, 1);
    }
    // ---- lines 17-21 (exclusion, p <- p_min), line 24 (+ temporaries), line 25 minima
    { Prof k(c, KF_ROWB);
      csr::rowpass(false, Rc, Pc, Palt, len, PA, NCP, TB, PB, nullptr, c->d_label, c->d_umin,
                   c->d_umax, ++c->row_tag, c->d_lsegs, c->d_nlsegs, have_long, false, ctr, c->st,
                   excl, /*B: write q = p too (owner exchange)*/ oc, prevctr, HOT_B, hw_ready ? c->d_hw : nullptr,
                   hot_cur || it == 0 ? ctr : nullptr, hot_cur ? 1 : 2);
      k.end(12.0 * len, 1 + (have_long ? 2 : 0)); }
    std::swap(Pc, Palt);
    // live tuples: this rank's (compaction) and the global count (convergence)
    if (multi) {
      CK(cudaMemcpyAsync(ctr + sv::C_SURVIVORS, ctr + sv::C_OUT, sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                         c->st));
      if (oc) {
        // the partials of foreign slots to their owners; the pass read PA: clear the replies
        TRY(oc_push(c, PB, nullptr, c->ocB));
        csr::oc_put(c->ocA.send, c->ocA.nsend, nullptr, PA, c->st);
      } else if (sparse) {
        TRY(comm_sparse_slots(c, PB, nullptr, n4));
      } else {
        TRY(comm_min_u32(c, PB, n4));
      }
      TRY(comm_allreduce(c, ctr + sv::C_OUT, 1, CC_DT_I64, CC_OP_SUM));
    }
    if (oc) {
      { Prof k(c, KF_SLOTS);
        csr::pstat2_block(PB, c->lo, c->hi, PA, TB, ctr, c->st);
        k.end(8.0 * (double)(c->hi - c->lo), 1); }
      CK(cudaMemsetAsync(TB, 0, sizeof(uint32_t) * nwp, c->st));
      TRY(comm_allreduce(c, ctr + sv::C_CHANGED2, 1, CC_DT_I64, CC_OP_SUM));
      TRY(oc_reply(c, PB, c->ocB));  // the next relabel's p -> PB[p]
    } else {
      Prof k(c, KF_SLOTS);
      csr::pstat2(PB, n, PA, TB, ctr, c->st, NX, lcur ? L[lb] : nullptr, lcur ? LC + lb : nullptr);
      csr::list_from_bits(NX, n, L[lb ^ 1], LC + (lb ^ 1), NCP, TB, exact_next ? PA : nullptr, c->st);
      k.end(lcur ? 12.0 * (double)prevp + n / 4.0 : 8.0 * n4 + n / 4.0, 2);
    }
    lexact = exact_next && !oc;
    lprev = lcur;
    lcur = true;
    lb ^= 1;
    c->launches += 6 + (have_long ? 4 : 0) + (it && ahead ? 2 : 0);
    CKL();
    CK(cudaMemcpyAsync(c->h_ctr2 + (it & 1) * sv::C_NUM, ctr, sizeof(uint64_t) * sv::C_NUM,
                       cudaMemcpyDeviceToHost, c->st));
    CK(cudaEventRecord(ev_read[it & 1], c->st));
    seg_end(c, a, 20.0 * len + 16.0 * n4, 8);
    next_enq = it + 1;
    return CC_OK;
  };
  // byte-model bookkeeping of the last enqueued iteration, undone if it turns out to be a
  // look-ahead that had nothing to do (its kernels returned at once)
  struct Snap { size_t nev; double bytes; uint64_t launches; } snap[KF_N];
  auto take_snap = [&]() {
    for (int f = 0; f < KF_N; f++) snap[f] = {c->kst[f].ev.size(), c->kst[f].bytes, c->kst[f].launches};
  };
  // 'balanced' variant (several ranks with exclusion, CC_FLAG_BALANCE): after an
  // iteration whose most loaded rank holds > 1/16 above the mean, the live rows are
  // redistributed evenly (rebalance_rows, cc_dist.cu); rows then live off their owner, so the
  // long-row list takes the global degrees and the labels are min-combined at the end
  const bool balance = multi && excl && (c->cfg.flags & CC_FLAG_BALANCE);
  bool deg_global = false, rebalanced = false;
  std::vector<uint64_t> loads;
  auto gather_loads = [&](uint64_t mine) -> cc_status {
    const int world = c->cfg.world_size;
    if (!c->d_bal) TRY(comm_agree(c, dalloc_t(c, &c->d_bal, (uint64_t)(world + 1) + (uint64_t)world * (world + 1))));
    const uint64_t v[2] = {mine, c->cap};
    CK(cudaMemcpyAsync(c->d_bal, v, sizeof(v), cudaMemcpyHostToDevice, c->st));
    TRY(comm_allgather(c, c->d_bal, c->d_bal + 2, sizeof(v)));
    loads.resize(2 * (size_t)world);
    CK(cudaMemcpyAsync(loads.data(), c->d_bal + 2, sizeof(uint64_t) * 2 * world, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return CC_OK;
  };
  uint64_t local_in = A_local;
  bool pending_compact = false;
  TRY(enqueue(0));
  for (uint32_t it = 0;; it++) {
    if (ahead && !pending_compact && next_enq == it + 1 && it + 1 < max_iter) {
      take_snap();
      TRY(enqueue(it + 1));
    }
    CK(cudaEventSynchronize(ev_read[it & 1]));
    const uint64_t* h = c->h_ctr2 + (it & 1) * sv::C_NUM;
    const uint64_t A1 = h[sv::C_OUT];
    const uint64_t len_live = multi ? h[sv::C_SURVIVORS] : A1;
    if (hw_ready) {
      if (h[sv::C_HIDDEN_DEAD] > hidden)
        return fail(c, CC_ERR_INVALID, "internal: collapsed-row count underflow");
      hidden -= h[sv::C_HIDDEN_DEAD];
    }
    // A_i+1: this iteration's survivors (counted before any collapse below folds them) plus
    // the tuples folded by earlier collapses into rows still live
    const uint64_t A_next = A1 + hidden;
    cc_iter_stat s{};
    s.active_in = A;
    s.partitions = h[sv::C_PARTITIONS];
    s.completed = h[sv::C_COMPLETED];
    s.changed = h[sv::C_CHANGED];
    s.temps = h[sv::C_TEMPS];
    s.changed2 = h[sv::C_CHANGED2];
    s.active_min = s.active_max = local_in;
    if (multi && (c->cfg.flags & CC_FLAG_TRACE)) {  // per-rank load (fig:loadbal): min / max over ranks
      uint64_t* mm = c->d_gcur + 2050;
      const uint64_t v2[2] = {local_in, local_in};
      CK(cudaMemcpyAsync(mm, v2, sizeof(v2), cudaMemcpyHostToDevice, c->st));
      TRY(comm_allreduce(c, mm, 1, CC_DT_I64, CC_OP_MIN));
      TRY(comm_allreduce(c, mm + 1, 1, CC_DT_I64, CC_OP_MAX));
      uint64_t r2[2];
      CK(cudaMemcpyAsync(r2, mm, sizeof(r2), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      s.active_min = r2[0];
      s.active_max = r2[1];
    }
    local_in = multi ? len_live : A1 + hidden;
    c->iters.push_back(s);
    if (!excl) {
      // 'Naive': nothing leaves; the partition passes decide convergence
      if (s.changed == 0 && s.changed2 == 0) {
        csr::final_labels(R[cb], Pc, len, c->d_label, c->st);
        c->launches += 1;
        break;
      }
    } else if (A1 == 0) {
      if (hidden) return fail(c, CC_ERR_INVALID, "internal: collapsed rows left at convergence");
      if (next_enq == it + 2)  // a look-ahead iteration is in flight: it returns at once
        for (int f = 0; f < KF_N; f++) {
          c->kst[f].ev.resize(snap[f].nev);
          c->kst[f].bytes = snap[f].bytes;
          c->kst[f].launches = snap[f].launches;
        }
      break;
    }
    if (it + 1 >= max_iter) return fail(c, CC_ERR_NOCONV, "SV did not converge in %u iterations", max_iter);
    // dead rows of completed partitions are squeezed out once they are a third of the array
    // (the paper's 'swapped to the end of the local array', sec:distSVOpt1); with the next
    // iteration already in flight, after it (its counts are exact then)
    // collapse once an average partition spans many tuples (then almost every row is PC),
    // at most every other iteration, and not again after one that folded little
    const bool want_collapse =
        collapse_force ? can_collapse && len_live > 0
                       : collapse_ok && it >= 1 && it >= last_collapse + 2 && len_live >= COLLAPSE_MIN_LEN &&
                             s.partitions * 16 < len_live;
    bool rebalance = false;
    if (balance) {
      TRY(gather_loads(len_live));
      uint64_t tot = 0, mx = 0;
      for (int k = 0; k < c->cfg.world_size; k++) {
        tot += loads[2 * k];
        mx = std::max(mx, loads[2 * k]);
      }
      const uint64_t mean = (tot + c->cfg.world_size - 1) / c->cfg.world_size;
      rebalance = tot > 0 && mx * 16 > mean * 17;
    }
    const bool want = 3 * (len - len_live) > len || want_collapse || (rebalance && len > len_live);
    if (pending_compact || (want && next_enq == it + 1)) {
      const bool do_collapse = pending_collapse || want_collapse;
      pending_compact = pending_collapse = false;
      TRY(scan_epoch_guard(c));
      if (do_collapse) {
        if (!hw_ready) {
          CK(cudaMemsetAsync(c->d_hw, 0, sizeof(uint32_t) * n, c->st));
          hw_ready = true;
        }
        uint64_t* hc = c->d_gcur + 2054;  // [2054]: folded tuples, [2055]: output length
        CK(cudaMemsetAsync(hc, 0, sizeof(uint64_t), c->st));
        { Prof k(c, KF_COMPACT);
          csr::collapse(R[cb], Pc, len, R[cb ^ 1], P[cb ^ 1], c->d_hw, hc, hc + 1, c->ss, c->st);
          k.end(8.0 * len + 8.0 * len_live, 1); }
        uint64_t hv[2] = {0, 0};
        CK(cudaMemcpyAsync(hv, hc, sizeof(hv), cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        hidden += hv[0];
        if (hv[1] + hv[0] != len_live)
          return fail(c, CC_ERR_INVALID, "internal: collapse kept %llu + folded %llu of %llu live tuples",
                      (unsigned long long)hv[1], (unsigned long long)hv[0], (unsigned long long)len_live);
        collapse_ok = hv[0] * 8 >= len_live;  // folded >= 1/8: worth trying again later
        last_collapse = it;
        len = hv[1];
      } else {
        { Prof k(c, KF_COMPACT); csr::compact(R[cb], Pc, len, R[cb ^ 1], P[cb ^ 1], c->ss, c->st);
          k.end(8.0 * len + 8.0 * len_live, 1); }
        len = len_live;
      }
      c->launches += 1;
      cb ^= 1;
      Pc = P[cb];
      Palt = c->d_q[0];
      if (have_long) csr::longlist(R[cb], Pc, len, c->d_deg, c->d_lsegs, c->d_nlsegs, c->st);
    } else if (want) {
      pending_compact = true;
      pending_collapse = want_collapse;
    }
    if (rebalance) {  // the live rows are now R[cb], Pc[0, len)
      uint32_t* Pdst = P[cb ^ 1];
      uint64_t nl = 0;
      bool moved = false;
      TRY(rebalance_rows(c, R[cb], Pc, R[cb ^ 1], Pdst, len, loads, &nl, &moved));
      if (moved) {
        if (!deg_global) {  // rows off their owner: the long-row list needs every degree
          TRY(comm_allreduce(c, c->d_deg, n, CC_DT_I32, CC_OP_SUM));
          deg_global = true;
        }
        rebalanced = true;
        cb ^= 1;
        Pc = P[cb];
        Palt = c->d_q[0];
        len = nl;
        local_in = nl;
        if (have_long) csr::longlist(R[cb], Pc, len, c->d_deg, c->d_lsegs, c->d_nlsegs, c->st);
      }
    }
    A = A_next;
    if (next_enq == it + 1) TRY(enqueue(it + 1));
  }
  // a vertex whose row moved was labelled on the rank that held it; every other rank holds
  // its own id or the (replicated) BFS label there, both >= the true label
  if (rebalanced) TRY(comm_min_u32(c, c->d_label, n));
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

// Alg. 1 on (edges, m_sv); vertices present iff deg > 0 and not BFS-visited.
static cc_status run_sv(cc_ctx* c, const uint2* edges, uint64_t m_sv, const uint32_t* vis) {
  const uint64_t n = c->n;
  if (!(c->cfg.flags & (CC_FLAG_REGROUP_SORT | CC_FLAG_REGROUP_DIRECT)))
    return run_sv_csr(c, edges, m_sv, vis);
  CK(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint64_t) * sv::C_NUM, c->st));
  sv::launch_init_tuples(edges, m_sv, c->d_deg, vis, n, c->d_w[0], c->d_ctr, c->st, &c->launches);
  CKL();
  TRY(sync_read(c));
  uint64_t A = 2 * m_sv + c->h_ctr[sv::C_VT_OUT];
  if (A == 0) return CC_OK;
  if (c->cfg.flags & CC_FLAG_REGROUP_DIRECT) return run_sv_direct(c, A, 0);
  const uint32_t max_iter = 2 * (uint32_t)c->kbits + 8;
  int cur = do_sort(c, 0, A, false);  // line 8: sort by r
  CKL();
  uint64_t chg2_prev = 0;
  for (uint32_t it = 0;; it++) {
    if (it >= max_iter) return fail(c, CC_ERR_NOCONV, "SV did not converge in %u iterations", max_iter);
    cudaEvent_t ev_it = ev_get(c);
    CK(cudaEventRecord(ev_it, c->st));
    cudaEvent_t a = nullptr;
    // ---- lines 9-13: vertex buckets, q <- u_min, PC
    seg_begin(c, &a);
    CK(cudaMemsetAsync(c->d_segA, 0xFF, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(c->d_segB, 0, sizeof(uint32_t) * n, c->st));
    sv::launch_seg_reduce(sv::SEG_VMINMAX, c->d_w[cur], nullptr, A, c->d_segA, c->d_segB, c->st);
    sv::launch_vertex_apply(true, c->d_w[cur], A, c->d_segA, c->d_segB, c->d_w[cur ^ 1],
                            c->d_q[cur ^ 1], c->st);
    seg_end(c, a, (double)A * (8 + 8 + 12), 2);
    c->launches += 2;
    cur ^= 1;
    CKL();
    // ---- line 14: sort by p;  lines 15-22: partition buckets, exclusion, temps
    cur = do_sort(c, cur, A, true);
    seg_begin(c, &a);
    CK(cudaMemsetAsync(c->d_segA, 0xFF, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(c->d_segB, 0, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint64_t) * (sv::C_TEMPS + 1), c->st));
    sv::launch_seg_reduce(sv::SEG_PMIN_NC, c->d_w[cur], c->d_q[cur], A, c->d_segA, c->d_segB, c->st);
    sv::launch_partition_apply(true, true, c->d_w[cur], c->d_q[cur], A, c->d_segA, c->d_segB,
                               c->d_w[cur ^ 1], c->d_label, c->d_ctr, c->st);
    c->launches += 2;
    cur ^= 1;
    CKL();
    TRY(sync_read(c));
    const uint64_t out = c->h_ctr[sv::C_OUT];
    const uint64_t T = c->h_ctr[sv::C_TEMPS];
    const uint64_t A1 = out - T;
    seg_end(c, a, (double)A * (12 + 12) + (double)out * 8, 2);
    cc_iter_stat s{};
    s.active_in = A;
    s.active_min = s.active_max = A;
    s.partitions = c->h_ctr[sv::C_PARTITIONS];
    s.completed = c->h_ctr[sv::C_COMPLETED];
    s.changed = c->h_ctr[sv::C_CHANGED];
    s.temps = T;
    if (!c->iters.empty()) {
      c->iters.back().changed2 = c->h_ctr[sv::C_CHANGED2] - chg2_prev;
      chg2_prev = c->h_ctr[sv::C_CHANGED2];
    }
    c->iters.push_back(s);
    c->it_ev.push_back(ev_it);
    if (out == 0) break;
    // ---- line 24: redo lines 8-13 with the temporaries
    cur = do_sort(c, cur, out, false);
    seg_begin(c, &a);
    CK(cudaMemsetAsync(c->d_segA, 0xFF, sizeof(uint32_t) * n, c->st));
    sv::launch_seg_reduce(sv::SEG_VMIN, c->d_w[cur], nullptr, out, c->d_segA, nullptr, c->st);
    sv::launch_vertex_apply(false, c->d_w[cur], out, c->d_segA, nullptr, c->d_w[cur ^ 1],
                            c->d_q[cur ^ 1], c->st);
    seg_end(c, a, (double)out * (8 + 8 + 12), 2);
    c->launches += 2;
    cur ^= 1;
    // ---- line 25: redo lines 14-21;  lines 26-28: erase temporaries
    cur = do_sort(c, cur, out, true);
    seg_begin(c, &a);
    CK(cudaMemsetAsync(c->d_segA, 0xFF, sizeof(uint32_t) * n, c->st));
    CK(cudaMemsetAsync(c->d_ctr + sv::C_OUT, 0, sizeof(uint64_t), c->st));
    sv::launch_seg_reduce(sv::SEG_PMIN, c->d_w[cur], c->d_q[cur], out, c->d_segA, nullptr, c->st);
    sv::launch_partition_apply(false, true, c->d_w[cur], c->d_q[cur], out, c->d_segA, nullptr,
                               c->d_w[cur ^ 1], c->d_label, c->d_ctr, c->st);
    seg_end(c, a, (double)out * (12 + 12) + (double)A1 * 8, 2);
    c->launches += 2;
    cur ^= 1;
    CKL();
    A = A1;
    if (A == 0) break;
    cur = do_sort(c, cur, A, false);  // next iteration's line 8
    CKL();
  }
  // changed2 of the last iteration
  TRY(sync_read(c));
  if (!c->iters.empty()) c->iters.back().changed2 = c->h_ctr[sv::C_CHANGED2] - chg2_prev;
  return CC_OK;
}

// Alg. 2 lines 2-3 on the host: read the degree statistics and histogram the prediction
// kernels left in d_gctr / d_hist / d_tail (summed over ranks when world_size > 1), fit the
// gate, decide the route.
cc_status predict_gate(cc_ctx* c, cc_mode mode, bool want_hist, bool* run_bfs_out, uint64_t* root) {
  cc_report& R = c->rep;
  // one host round trip in the common case: the non-empty bins are compacted before it (every
  // dense bin is scanned: bins past d_max are empty), and the counters, the pair count and the
  // first FAST pairs come back together into pinned memory; more pairs, or a tail list, take
  // a second round trip (it was three, through pageable memory: C4 spent ~0.14 ms here)
  constexpr uint64_t FAST = 8192;
  uint64_t* npairs = c->d_gctr + graph::G_NUM + 1544 - 1;
  uint64_t* h_np = c->h_gctr + graph::G_NUM + 4;  // pinned
  uint2* h_pairs = reinterpret_cast<uint2*>(c->h_hist);  // pinned, HIST_DENSE / 2 pairs
  if (want_hist) {
    graph::launch_hist_pairs(c->d_hist, graph::HIST_DENSE, c->d_hpairs, npairs, c->st);
    c->launches += 1;
    CK(cudaMemcpyAsync(h_np, npairs, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(h_pairs, c->d_hpairs, sizeof(uint2) * FAST, cudaMemcpyDeviceToHost, c->st));
  }
  TRY(sync_read(c));
  c->dhist.clear();
  c->dhist_valid = want_hist;  // an all-isolated graph has the empty distribution
  R.n_present = c->h_gctr[graph::G_NPRESENT];
  const uint64_t maxkey = c->h_gctr[graph::G_MAXKEY];
  R.max_degree = maxkey >> 32;
  *root = maxkey ? (uint64_t)(0xFFFFFFFFu - (uint32_t)maxkey) : 0;
  bool run_bfs = (mode == CC_MODE_BFS_SV);
  R.ls_alpha = R.ls_r2 = R.ks_stat = R.ks_alpha = NAN;
  if (want_hist && R.max_degree > 0) {
    const uint64_t tail_n = std::min<uint64_t>(c->h_gctr[graph::G_TAIL], graph::TAIL_CAP);
    const uint64_t np = *h_np;
    if (np > graph::HIST_DENSE / 2) return fail(c, CC_ERR_INVALID, "internal: %llu degree bins", (unsigned long long)np);
    const bool more = np > FAST;
    if (more)
      CK(cudaMemcpyAsync(h_pairs + FAST, c->d_hpairs + FAST, sizeof(uint2) * (np - FAST), cudaMemcpyDeviceToHost,
                         c->st));
    if (tail_n)
      CK(cudaMemcpyAsync(c->h_hist + graph::HIST_DENSE, c->d_tail, sizeof(uint32_t) * tail_n,
                         cudaMemcpyDeviceToHost, c->st));
    if (more || tail_n) CK(cudaStreamSynchronize(c->st));
    std::vector<uint2> pairs(h_pairs, h_pairs + np);
    std::sort(pairs.begin(), pairs.end(), [](const uint2& a, const uint2& b) { return a.x < b.x; });
    gate::Hist h;
    for (const uint2& pr : pairs) h.push_back({pr.x, pr.y});
    if (tail_n) {
      std::vector<uint32_t> t(c->h_hist + graph::HIST_DENSE, c->h_hist + graph::HIST_DENSE + tail_n);
      std::sort(t.begin(), t.end());
      for (size_t i = 0; i < t.size();) {
        size_t j = i;
        while (j < t.size() && t[j] == t[i]) j++;
        h.push_back({t[i], (uint64_t)(j - i)});
        i = j;
      }
    }
    c->dhist = h;
    c->dhist_valid = true;
    gate::LsFit g = gate::fit_ls(h);
    R.ls_alpha = g.alpha;
    R.ls_r2 = g.r2;
    const bool need_ks = (c->cfg.flags & CC_FLAG_GATE_KS) || (c->cfg.flags & CC_FLAG_TRACE);
    bool ks_ok = false;
    if (need_ks) {
      gate::KsFit k = gate::fit_ks(h);
      if (k.valid) {
        R.ks_stat = k.ks; R.ks_alpha = k.alpha; R.ks_xmin = k.xmin; ks_ok = true;
      }
    }
    if (mode == CC_MODE_AUTO)
      run_bfs = (c->cfg.flags & CC_FLAG_GATE_KS) ? (ks_ok && R.ks_stat < c->cfg.tau) : g.scale_free;
  }
  if (R.max_degree == 0) run_bfs = false;
  *run_bfs_out = run_bfs;
  return CC_OK;
}

// Edge-streaming BFS peel (Alg. 2 lines 7-11) from `root`
// over this rank's edge list c->d_edges.  With world_size > 1 the 2-bit state is replicated
// and each level's found bitmap is OR-ed over ranks before it is counted, so every rank takes
// the same levels; the edge lists stay where they were loaded.  spec_ok: level 1 already ran
// inside the degree pass (graph.cu k_deg_sample).  Out: the remainder E \ {(u,v) | u in VI}
// of this rank's edges (*rem, *m_rem), the visited bitmap in c->d_bm[0], labels of VI written,
// rep.bfs_visited / bfs_levels set; *e_bfs recorded after the labels.
cc_status bfs_stream(cc_ctx* c, uint64_t root, bool spec_ok, const uint2** rem, uint64_t* m_rem,
                     cudaEvent_t* e_bfs) {
  cc_report& R = c->rep;
  const uint64_t n = c->n, m = c->m;
  const uint64_t nw = (n + 31) / 32;
  uint32_t *V = c->d_bm[0], *S = c->d_bm[1], *X = c->d_bm[2];
  if (!c->d_rem) TRY(comm_agree(c, dalloc_t(c, &c->d_rem, m + 1)));
  if (!c->d_rem2) TRY(comm_agree(c, dalloc_t(c, &c->d_rem2, m + 1)));
  uint2* bufs[2] = {c->d_rem, c->d_rem2};
  if (!spec_ok) {
    CK(cudaMemsetAsync(S, 0, sizeof(uint32_t) * 2 * nw, c->st));
    c->h_word[0] = 1u << (2 * (root & 15));
    CK(cudaMemcpyAsync(S + root / 16, c->h_word, 4, cudaMemcpyHostToDevice, c->st));
  }
  if (!spec_ok) CK(cudaMemsetAsync(X, 0, sizeof(uint32_t) * nw, c->st));  // then cleared per level
  const uint2* cur = c->d_edges;
  uint64_t mcur = m;
  int nb = 0;  // next scratch buffer
  bool last_compacted = false;
  uint64_t visited = 1, levels = 0, front_arcs = 0;
  bool spec_pending = spec_ok;
  while (true) {
    const bool root_level = levels == 0;
    bool compact = false;
    if (!spec_pending) {
      // compact (keep only edges that can still matter) once most present vertices are
      // visited, or when the frontier's arcs are a fifth of the current edge list: every edge
      // at the frontier leaves, so the next level reads that much less (a local decision:
      // each rank compacts its own list)
      compact = !root_level && (2 * visited > R.n_present || 5 * front_arcs >= 2 * mcur);
      CK(cudaMemsetAsync(c->d_gctr + graph::G_REMAIN, 0, sizeof(uint64_t), c->st));
      Prof k(c, KF_BFS);
      graph::launch_bfs_level(root_level, compact, cur, mcur, (uint32_t)root, S, X, bufs[nb], c->d_gctr, c->st);
      c->launches += 1;
      k.end(8.0 * (double)mcur + (compact ? 8.0 * (double)mcur / 8 : 0.0) + (double)n / 4, 1,
            root_level ? 0.0 : 2.0 * (double)mcur);
    }
    spec_pending = false;
    // the level's found ids (OR over ranks: every rank's edges found some) and their arcs
    TRY(comm_or_bits(c, X, nw));
    CK(cudaMemsetAsync(c->d_gctr + graph::G_NEWVIS, 0, sizeof(uint64_t), c->st));
    CK(cudaMemsetAsync(c->d_gctr + graph::G_FARCS, 0, sizeof(uint64_t), c->st));
    // counts, S advanced (frontier <- X, visited |= X; a no-op past the last level), X cleared
    graph::launch_farcs_advance(X, S, n, c->d_deg, c->d_gctr + graph::G_NEWVIS, c->d_gctr + graph::G_FARCS, c->st);
    c->launches += 1;
    CKL();
    TRY(sync_read(c));
    last_compacted = compact;
    if (compact) {
      cur = bufs[nb];
      mcur = c->h_gctr[graph::G_REMAIN];
      nb ^= 1;
    }
    const uint64_t nv = c->h_gctr[graph::G_NEWVIS];
    if (nv == 0) break;
    visited += nv;
    front_arcs = c->h_gctr[graph::G_FARCS];
    levels++;
  }
  R.bfs_visited = visited;
  R.bfs_levels = levels;
  graph::launch_vis_bits(S, n, V, c->st);
  graph::launch_min_visited(V, n, c->d_gctr, c->st);
  graph::launch_bfs_labels(V, n, c->d_label, c->d_gctr, c->st);
  c->launches += 3;
  *e_bfs = ev_get(c);
  CK(cudaEventRecord(*e_bfs, c->st));
  if (last_compacted) {
    // a level that discovers nothing leaves no edge with exactly one visited endpoint:
    // its survivors are exactly E \ {(u,v) | u in VI}
    *m_rem = mcur;
    *rem = cur;
  } else {
    CK(cudaMemsetAsync(c->d_gctr + graph::G_REMAIN, 0, sizeof(uint64_t), c->st));
    graph::launch_filter(cur, mcur, S, bufs[nb], c->d_gctr, c->st);
    c->launches += 1;
    CKL();
    TRY(sync_read(c));
    *m_rem = c->h_gctr[graph::G_REMAIN];
    *rem = bufs[nb];
  }
  return CC_OK;
}

// SV on the BFS remainder with its endpoints renumbered densely in id order (graph.cu,
// "remainder renumbering").  Alg. 1 compares ids only, so the run on
// [0, n') has the same sets and counters; the labels go back through inv.  Scratch: the
// 2-bit BFS state (free after the peel) holds the bitmap and word prefixes, the other
// remainder buffer the renumbered edges, inv, degrees and labels.
static bool renumber_fits(const cc_ctx* c, const uint2* edges, uint64_t m_sv) {
  if (c->cfg.flags & CC_FLAG_NO_RENUMBER) return false;
  if (multi_gpu(c) || !c->d_rem || !c->d_rem2 || (edges != c->d_rem && edges != c->d_rem2)) return false;
  if (m_sv == 0 || m_sv * 8 > c->n) return false;  // worth it once n' <= 2 m_sv is a fraction of n
  const uint64_t nw = (c->n + 31) / 32;
  // 8 m_sv bytes of edges + 3 x 4 (2 m_sv) bytes (inv, sdeg, labels) + the tile sums
  return 32 * m_sv + 4 * graph::sub_bsum_words(nw) <= 8 * c->m;
}
static cc_status run_sv(cc_ctx* c, const uint2* edges, uint64_t m_sv, const uint32_t* vis);
static cc_status run_sv_renumbered(cc_ctx* c, const uint2* edges, uint64_t m_sv) {
  const uint64_t n = c->n, nw = (n + 31) / 32;
  uint32_t* bm = c->d_bm[1];  // 2 nw words (the BFS state)
  uint32_t* wpre = bm + nw;
  uint2* se = edges == c->d_rem ? c->d_rem2 : c->d_rem;
  uint32_t* inv = reinterpret_cast<uint32_t*>(se + m_sv);
  uint32_t* sdeg = inv + 2 * m_sv;
  uint32_t* slab = sdeg + 2 * m_sv;
  uint32_t* bsum = slab + 2 * m_sv;
  uint64_t* subn = c->d_gctr + graph::G_SUBN;
  CK(cudaMemsetAsync(bm, 0, sizeof(uint32_t) * nw, c->st));
  graph::launch_sub_mark(edges, m_sv, bm, c->st);
  graph::launch_sub_rank(bm, nw, bsum, wpre, subn, c->st);
  graph::launch_sub_edges(edges, m_sv, bm, wpre, c->d_deg, se, inv, sdeg, c->st);
  c->launches += 4;
  CKL();
  TRY(sync_read(c));
  const uint64_t ns = c->h_gctr[graph::G_SUBN];
  if (ns == 0 || ns > 2 * m_sv) return fail(c, CC_ERR_INVALID, "internal: renumbered %llu ids for %llu edges",
                                            (unsigned long long)ns, (unsigned long long)m_sv);
  c->rep.sv_ids = ns;
  sv::launch_init_labels(slab, ns, c->st);
  c->launches += 1;
  // the SV sees n' ids, their degrees and their labels
  const uint64_t n_save = c->n;
  uint32_t *deg_save = c->d_deg, *lab_save = c->d_label;
  c->n = ns;
  c->d_deg = sdeg;
  c->d_label = slab;
  const cc_status s = run_sv(c, se, m_sv, nullptr);
  c->n = n_save;
  c->d_deg = deg_save;
  c->d_label = lab_save;
  TRY(s);
  graph::launch_sub_labels(inv, slab, ns, c->d_label, c->st);
  c->launches += 1;
  CKL();
  return CC_OK;
}

// CSR rows of the whole graph from the bucketed arcs (csr::bucket_degrees already ran with
// the same gsf): offsets in c->d_q[0], tuples in buffer 0.  *A = tuple count.
static cc_status build_full_rows(cc_ctx* c, int gsf, uint64_t* A_out) {
  const uint64_t n = c->n, m = c->m;
  uint2* bucketed = reinterpret_cast<uint2*>(c->d_w[1]);
  uint32_t* R0 = reinterpret_cast<uint32_t*>(c->d_w[0]);
  uint32_t* P0 = R0 + c->cap;
  cudaEvent_t a = nullptr;
  seg_begin(c, &a);
  CK(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint64_t) * sv::C_NUM, c->st));
  TRY(scan_epoch_guard(c));
  csr::build(nullptr, m, c->d_deg, nullptr, n, c->d_q[0], c->d_q[1], c->d_garc, gsf, c->ss, c->d_ctr,
             c->st, /*count_groups=*/false);
  CKL();
  TRY(sync_read(c));
  const uint64_t A = c->h_ctr[sv::C_VT_OUT];
  if (A > c->cap) return fail(c, CC_ERR_INVALID, "tuple count exceeds capacity");
  csr::fill_from_buckets(c->d_q[0], c->d_q[1], n, A, R0, P0, bucketed, 2 * m, c->d_segB, c->d_gcur + 2048,
                         c->st);
  c->launches += 4;
  CKL();
  seg_end(c, a, 8.0 * n + 24.0 * m + 4.0 * (double)A, 4, KF_CSR);
  *A_out = A;
  return CC_OK;
}

// Direction-optimising BFS from `root` over the full CSR rows (c->d_q[0] offsets, P of tuple
// buffer 0, degrees in c->d_deg); visited bitmap in c->d_bm[0].  *levels = eccentricity of root.
static cc_status bfs_csr(cc_ctx* c, uint64_t root, uint64_t m, uint64_t* visited_out, uint64_t* levels_out) {
  const uint64_t n = c->n;
  const uint64_t nw = (n + 31) / 32;
  uint32_t* P0 = reinterpret_cast<uint32_t*>(c->d_w[0]) + c->cap;
  uint32_t *V = c->d_bm[0], *F = c->d_bm[1], *X = c->d_bm[2];
  uint32_t *list = c->d_segA, *next = c->d_segB;
  CK(cudaMemsetAsync(V, 0, sizeof(uint32_t) * nw, c->st));
  CK(cudaMemsetAsync(F, 0, sizeof(uint32_t) * nw, c->st));
  c->h_word[0] = 1u << (root & 31);
  c->h_word[1] = (uint32_t)root;
  CK(cudaMemcpyAsync(V + root / 32, c->h_word, 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(F + root / 32, c->h_word, 4, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(list, c->h_word + 1, 4, cudaMemcpyHostToDevice, c->st));
  uint32_t droot = 0;
  CK(cudaMemcpyAsync(&droot, c->d_deg + root, 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  uint64_t nf = 1, mf = droot, mu = 2 * m - droot;
  uint64_t visited = 1, levels = 0;
  uint64_t* bctr = c->d_gctr + graph::G_NEWVIS;  // [G_NEWVIS, G_REMAIN]: next count, its arcs
  static_assert(graph::G_REMAIN == graph::G_NEWVIS + 1, "level counters are adjacent");
  while (true) {
    CK(cudaMemsetAsync(X, 0, sizeof(uint32_t) * nw, c->st));
    CK(cudaMemsetAsync(bctr, 0, 2 * sizeof(uint64_t), c->st));
    const bool bottom_up = mf * 14 > mu;  // Beamer's direction rule on arc counts
    Prof k(c, KF_BFS);
    bfs::level(bottom_up, c->d_q[0], P0, c->d_deg, n, list, nf, F, V, X, next, bctr, c->st);
    k.end(bottom_up ? 8.0 * n + 4.0 * (double)mu : 8.0 * nf + 4.0 * (double)mf, 1);
    c->launches += 1;
    CKL();
    TRY(sync_read(c));
    const uint64_t nv = c->h_gctr[graph::G_NEWVIS];
    if (nv == 0) break;
    visited += nv;
    levels++;
    mf = c->h_gctr[graph::G_REMAIN];
    mu = mu > mf ? mu - mf : 0;
    nf = nv;
    std::swap(F, X);
    std::swap(list, next);
  }
  *visited_out = visited;
  *levels_out = levels;
  return CC_OK;
}

extern "C" cc_status cc_run(cc_ctx* c, cc_mode mode, cc_report* out) {
  if (!c) return CC_ERR_INVALID;
  if (!c->loaded) return fail(c, CC_ERR_STATE, "cc_run before cc_load_edges");
  if (mode != CC_MODE_AUTO && mode != CC_MODE_SV && mode != CC_MODE_BFS_SV)
    return fail(c, CC_ERR_INVALID, "bad mode %d", (int)mode);
  if ((c->cfg.flags & (CC_FLAG_NO_EXCLUDE | CC_FLAG_NO_EARLY_EXCLUDE)) &&
      (c->cfg.flags & (CC_FLAG_REGROUP_SORT | CC_FLAG_REGROUP_DIRECT)))
    return fail(c, CC_ERR_INVALID, "exclusion variants are implemented by the csr engine");
  CK(cudaSetDevice(c->cfg.device));
  c->ran = false;
  c->iters.clear();
  c->launches = 0;
  c->ev_used = 0;
  c->it_ev.clear();
  for (auto& k : c->kst) k = cc_ctx::KStat();
  cc_report& R = c->rep;
  R = cc_report{};
  const uint64_t m = c->m;
  R.m_edges = c->m_total;
  if (multi_gpu(c)) {
    double ms_rel = 0;
    if (c->idw == CC_U64) {  // Alg. 2 line 4 over all ranks (relabel_dist.cu)
      cudaEvent_t r0 = ev_get(c), r1 = ev_get(c);
      CK(cudaEventRecord(r0, c->st));
      TRY(dist_relabel(c));
      CK(cudaEventRecord(r1, c->st));
      CK(cudaEventSynchronize(r1));
      ms_rel = ev_ms(r0, r1);
    }
    if (c->n == 0) {  // no ids on any rank (u64 mode): nothing to label
      R.components = 0;
      R.ms_relabel = R.ms_total = ms_rel;
      c->ran = true;
      if (out) *out = R;
      return CC_OK;
    }
    TRY(run_dist(c, mode));
    R.ms_relabel = ms_rel;
    R.ms_total += ms_rel;
    R.iters = c->iters.data();
    R.n_iters = (uint32_t)c->iters.size();
    for (size_t i = 0; i < c->it_ev.size() && i < c->iters.size(); i++)
      c->iters[i].ms = i + 1 < c->it_ev.size() ? ev_ms(c->it_ev[i], c->it_ev[i + 1]) : 0.0;
    if (profiling(c))
      for (auto& k : c->kst)
        for (auto& p : k.ev) k.ms += ev_ms(p.first, p.second);
    c->ran = true;
    if (out) *out = R;
    return CC_OK;
  }

  cudaEvent_t e0 = ev_get(c), e_rel, e_pred, e_bfs, e_filter, e_sv, e_end;
  CK(cudaEventRecord(e0, c->st));
  NvtxRange nv_run("cc_run");
  NvtxStages nv;  // the stages of cc_report.ms_*
  nv.next("relabel (Alg. 2 line 4)");
  // ------------------------------------------------ relabel (Alg. 2 line 4; u64 ids only)
  // ids are made dense first: every later stage addresses buckets by id (R18)
  if (c->idw == CC_U64) {
    TRY(scan_epoch_guard(c));
    uint64_t* total = c->d_gctr + graph::G_NUM + 1537;
    uint32_t* vals[2] = {c->d_q[0], c->d_q[1]};
    if (c->d_htab)
      TRY(relabel_hash(c, 2 * m, total));
    else
      relabel::run(c->d_ids64, 2 * m, c->d_w, vals, c->rws, c->ss, reinterpret_cast<uint32_t*>(c->d_edges),
                   c->d_uids, total, c->st, &c->launches);
    CKL();
    CK(cudaMemcpyAsync(c->h_word, total, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    uint64_t nd = m ? *reinterpret_cast<uint64_t*>(c->h_word) : 0;
    if (nd > (1ull << 30)) return fail(c, CC_ERR_INVALID, "%llu distinct ids > 2^30", (unsigned long long)nd);
    c->n = nd;
    c->hi = nd;
    c->kbits = bits_for(nd);
    if (c->cfg.flags & CC_FLAG_PERMUTE_IDS) {
      // SV runs on ids permuted by the 64-bit mix; pi[v] = rank of mix(id_v)
      relabel::mix(c->d_uids, nd, c->d_mix, c->st);
      relabel::run(c->d_mix, nd, c->d_w, vals, c->rws, c->ss, c->d_pi, c->d_mix, total, c->st,
                   &c->launches);
      relabel::apply(reinterpret_cast<uint32_t*>(c->d_edges), 2 * m, c->d_pi, c->st);
      c->launches += 2;
      CKL();
    }
  }
  const uint64_t n = c->n;
  e_rel = ev_get(c);
  CK(cudaEventRecord(e_rel, c->st));
  nv.next("prediction (Alg. 2 lines 2-3)");
  // ------------------------------------------------ prediction (Alg. 2 lines 2-3)
  // csr engine, n <= 2^26: the arcs are bucketed by vertex group (the CSR build needs this
  // pass anyway) and degrees are counted per group in shared memory; otherwise counting
  // increments in L2 windows.
  // CC_FLAG_BFS_CSR: build the full CSR during prediction (degrees counted per bucketed vertex
  // group in shared memory) and peel with the direction-optimising BFS on it.  Off by default:
  // on C4 the 2.2 G-tuple CSR build costs more than the edge-streaming BFS saves.
  const bool csr_engine = !(c->cfg.flags & (CC_FLAG_REGROUP_SORT | CC_FLAG_REGROUP_DIRECT));
  const int gsf = (csr_engine && (c->cfg.flags & CC_FLAG_BFS_CSR)) ? csr::group_shift_full(n) : -1;
  uint2* bucketed = reinterpret_cast<uint2*>(c->d_w[1]);  // 2m arcs fit: cap >= 2m + 2n
  CK(cudaMemsetAsync(c->d_gctr, 0, sizeof(uint64_t) * graph::G_NUM, c->st));
  CK(cudaMemsetAsync(c->d_gctr + graph::G_MINVIS, 0xFF, sizeof(uint64_t), c->st));
  // speculative root level (graph.cu k_deg_sample): on large lists the degree pass also runs
  // the BFS level of a root guessed from a prefix; kept below if the guess is the root
  bool spec_ran = false;
  const bool spec_want = gsf < 0 && mode != CC_MODE_SV && m >= graph::spec_min_edges();
  graph::SpecLevel spec{c->d_bm[1], c->d_bm[2], c->d_gctr};
  if (spec_want) {
    const uint64_t nw = (n + 31) / 32;
    CK(cudaMemsetAsync(spec.S, 0, sizeof(uint32_t) * 2 * nw, c->st));
    CK(cudaMemsetAsync(spec.next, 0, sizeof(uint32_t) * nw, c->st));
  }
  {
    Prof k(c, KF_PREDICT);
    if (gsf >= 0) {
      csr::bucket_degrees(c->d_edges, m, n, gsf, c->d_garc, c->d_gcur, bucketed, c->d_deg, c->st);
      k.end(8.0 * m + 8.0 * m + 16.0 * m + 16.0 * m + 4.0 * n, 4);
    } else {
      CK(cudaMemsetAsync(c->d_deg, 0, sizeof(uint32_t) * n, c->st));
      // scratch: tuple buffer 1 (8 cap >= 16m + 16n bytes) is free until the SV / CSR stages
      const int ret = graph::launch_degree(c->d_edges, m, n, c->d_deg, c->st, c->d_tail,
                                           c->d_gctr + graph::G_NUM + 64, c->d_w[1],
                                           sizeof(uint64_t) * c->cap, c->d_garc,
                                           spec_want ? &spec : nullptr);
      const int algo = ret & 1;
      spec_ran = (ret & 2) != 0;
      if (spec_ran) c->launches += 3;
      // bucketed: edges read, u16 entries written and read, deg read + written; 2 shared
      // atomics per arc.  L2 windows: the edge list once per 2^24-id window, 1 L2 add per arc
      const double nwin = (double)((n + (1ull << 24) - 1) >> 24);
      if (algo == 1) k.end(8.0 * m + 4.0 * m + 4.0 * m + 8.0 * n, 3, 4.0 * m);
      else k.end(8.0 * m * (nwin > 0 ? nwin : 1) + 4.0 * n, 1, 0.0);
    }
  }
  const bool want_hist = (mode == CC_MODE_AUTO) || (c->cfg.flags & CC_FLAG_TRACE);
  if (want_hist) CK(cudaMemsetAsync(c->d_hist, 0, sizeof(uint32_t) * graph::HIST_DENSE, c->st));
  {
    Prof k(c, KF_HIST);
    graph::launch_deg_hist(c->d_deg, n, c->d_hist, c->d_tail, c->d_gctr, c->st);
    k.end(4.0 * n, 1);
  }
  c->launches += 3;
  CKL();
  bool run_bfs = false;
  uint64_t root = 0;
  TRY(predict_gate(c, mode, want_hist, &run_bfs, &root));
  // every id starts as its own label; on the BFS route k_bfs_labels writes them with L_bfs
  if (!run_bfs) {
    sv::launch_init_labels(c->d_label, n, c->st);
    c->launches += 1;
  }
  e_pred = ev_get(c);
  CK(cudaEventRecord(e_pred, c->st));
  nv.next(run_bfs ? "BFS peel + filter (Alg. 2 lines 7-11)" : "SV (Alg. 1)");

  // ------------------------------------------------ full CSR rows (csr engine, both routes)
  uint64_t A_full = 0;
  if (gsf >= 0) TRY(build_full_rows(c, gsf, &A_full));

  // ------------------------------------------------ BFS peel + filter (lines 7-11)
  const uint2* sv_edges = c->d_edges;
  uint64_t m_sv = m;
  const uint32_t* vis = nullptr;
  e_bfs = e_filter = e_pred;
  if (run_bfs && gsf >= 0) {
    // direction-optimising BFS over the CSR rows (bfs.cu)
    R.ran_bfs = 1;
    R.bfs_root = root;
    uint64_t visited = 0, levels = 0;
    TRY(bfs_csr(c, root, m, &visited, &levels));
    uint32_t* V = c->d_bm[0];
    R.bfs_visited = visited;
    R.bfs_levels = levels;
    graph::launch_min_visited(V, n, c->d_gctr, c->st);
    graph::launch_bfs_labels(V, n, c->d_label, c->d_gctr, c->st);
    c->launches += 2;
    e_bfs = ev_get(c);
    CK(cudaEventRecord(e_bfs, c->st));
    if (!c->d_rem) TRY(dalloc_t(c, &c->d_rem, m + 1));
    CK(cudaMemsetAsync(c->d_gctr + graph::G_REMAIN, 0, sizeof(uint64_t), c->st));
    bfs::filter(c->d_edges, m, V, c->d_rem, c->d_gctr + graph::G_REMAIN, c->st);
    c->launches += 1;
    CKL();
    TRY(sync_read(c));
    m_sv = c->h_gctr[graph::G_REMAIN];
    sv_edges = c->d_rem;
    R.remainder_edges = m_sv;
    vis = V;
    e_filter = ev_get(c);
    CK(cudaEventRecord(e_filter, c->st));
  } else if (run_bfs) {
    R.ran_bfs = 1;
    R.bfs_root = root;
    // the speculative level is the root's level iff the guess is the root (same id: the
    // claims are then exactly those level 1 makes)
    const uint64_t guess = c->h_gctr[graph::G_GUESS];
    const bool spec_ok = spec_ran && guess && (uint64_t)(0xFFFFFFFFu - (uint32_t)guess) == root;
    R.bfs_spec_root = spec_ok ? 1 : 0;
    TRY(bfs_stream(c, root, spec_ok, &sv_edges, &m_sv, &e_bfs));
    R.remainder_edges = m_sv;
    vis = c->d_bm[0];
    e_filter = ev_get(c);
    CK(cudaEventRecord(e_filter, c->st));
  }

  // ------------------------------------------------ SV (line 13)
  if (run_bfs) nv.next("SV on the remainder (Alg. 2 line 13)");
  if (gsf >= 0 && !run_bfs) {
    c->rep.sv_ids = n;
    if (A_full) TRY(sv_iterate(c, A_full, A_full, A_full));  // the rows built above
  } else if (run_bfs && renumber_fits(c, sv_edges, m_sv)) {
    TRY(run_sv_renumbered(c, sv_edges, m_sv));
  } else {
    c->rep.sv_ids = n;
    TRY(run_sv(c, sv_edges, m_sv, vis));
  }
  if (c->idw == CC_U64 && (c->cfg.flags & CC_FLAG_PERMUTE_IDS)) {
    // labels back to the minimum original id of each component (C1)
    relabel::canonicalize(c->d_pi, c->d_label, n, c->d_segA, c->d_segB, c->st);
    CK(cudaMemcpyAsync(c->d_label, c->d_segB, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, c->st));
    c->launches += 2;
    CKL();
  }
  R.sv_iterations = (uint32_t)c->iters.size();
  e_sv = ev_get(c);
  CK(cudaEventRecord(e_sv, c->st));
  nv.next("finalise");
  // components, isolated ids included (each has exactly one root: its minimum id)
  uint64_t* roots = c->d_gctr + graph::G_TAIL;
  CK(cudaMemsetAsync(roots, 0, sizeof(uint64_t), c->st));
  graph::launch_count_roots(c->d_label, 0, n, roots, c->st);
  c->launches += 1;
  CK(cudaMemcpyAsync(&R.components, roots, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  e_end = ev_get(c);
  CK(cudaEventRecord(e_end, c->st));
  CK(cudaStreamSynchronize(c->st));

  // ------------------------------------------------ report
  R.ms_total = ev_ms(e0, e_end);
  R.ms_relabel = ev_ms(e0, e_rel);
  R.ms_prediction = ev_ms(e_rel, e_pred);
  R.ms_bfs = run_bfs ? ev_ms(e_pred, e_bfs) : 0;
  R.ms_filter = run_bfs ? ev_ms(e_bfs, e_filter) : 0;
  R.ms_sv = ev_ms(e_filter, e_sv);
  R.ms_finalize = ev_ms(e_sv, e_end);
  for (size_t i = 0; i < c->it_ev.size() && i < c->iters.size(); i++)
    c->iters[i].ms = ev_ms(c->it_ev[i], i + 1 < c->it_ev.size() ? c->it_ev[i + 1] : e_sv);
  if (profiling(c))
    for (auto& k : c->kst)
      for (auto& p : k.ev) k.ms += ev_ms(p.first, p.second);
  R.iters = c->iters.data();
  R.n_iters = (uint32_t)c->iters.size();
  c->ran = true;
  if (out) *out = R;
  return CC_OK;
}

extern "C" cc_status cc_labels_u32(cc_ctx* c, uint32_t* out, uint64_t cap, uint64_t* count,
                                   int out_on_device) {
  if (!c) return CC_ERR_INVALID;
  if (!c->ran) return fail(c, CC_ERR_STATE, "cc_labels before cc_run");
  if (c->idw != CC_U32) return fail(c, CC_ERR_STATE, "u64 graph loaded: use cc_labels_u64");
  const uint64_t cnt = c->hi - c->lo;  // this rank's block ([0, n) on one GPU)
  if (count) *count = cnt;
  if (!out || cap < cnt) return fail(c, CC_ERR_INVALID, "output buffer too small");
  CK(cudaSetDevice(c->cfg.device));
  if (cnt)
    CK(cudaMemcpyAsync(out, c->d_label + c->lo, sizeof(uint32_t) * cnt,
                       out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

extern "C" cc_status cc_labels_u64(cc_ctx* c, uint64_t* ids, uint64_t* labels, uint64_t cap,
                                   uint64_t* count, int out_on_device) {
  if (!c) return CC_ERR_INVALID;
  if (!c->ran) return fail(c, CC_ERR_STATE, "cc_labels before cc_run");
  if (c->idw != CC_U64) return fail(c, CC_ERR_STATE, "u32 graph loaded: use cc_labels_u32");
  if (multi_gpu(c)) {  // this rank's block of the dense ids; collective
    const uint64_t cnt = c->hi - c->lo;
    if (count) *count = cnt;
    if (!ids || !labels || cap < cnt) return fail(c, CC_ERR_INVALID, "output buffers too small");
    CK(cudaSetDevice(c->cfg.device));
    return dist_labels_u64(c, ids, labels, out_on_device);
  }
  if (count) *count = c->n;
  if (!ids || !labels || cap < c->n) return fail(c, CC_ERR_INVALID, "output buffers too small");
  CK(cudaSetDevice(c->cfg.device));
  if (c->n) {
    uint64_t* tmp = c->d_w[0];  // SV state is finished; reuse as label staging
    relabel::labels(c->d_uids, c->d_label, c->n, tmp, c->st);
    CKL();
    const cudaMemcpyKind k = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpyAsync(ids, c->d_uids, sizeof(uint64_t) * c->n, k, c->st));
    CK(cudaMemcpyAsync(labels, tmp, sizeof(uint64_t) * c->n, k, c->st));
  }
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

extern "C" cc_status cc_degree_histogram(cc_ctx* c, uint64_t* degrees, uint64_t* counts, uint64_t cap,
                                         uint64_t* count) {
  if (!c) return CC_ERR_INVALID;
  if (!c->ran || !c->dhist_valid)
    return fail(c, CC_ERR_STATE, "no degree distribution: cc_run(AUTO) or CC_FLAG_TRACE first");
  const uint64_t nb = c->dhist.size();
  if (count) *count = nb;
  if (!degrees || !counts || cap < nb) return fail(c, CC_ERR_INVALID, "output buffers too small");
  for (uint64_t i = 0; i < nb; i++) {
    degrees[i] = c->dhist[i].first;
    counts[i] = c->dhist[i].second;
  }
  return CC_OK;
}

extern "C" cc_status cc_degrees_u32(cc_ctx* c, uint32_t* out, uint64_t cap, uint64_t* count,
                                    int out_on_device) {
  if (!c) return CC_ERR_INVALID;
  if (!c->loaded) return fail(c, CC_ERR_STATE, "cc_degrees_u32 before cc_load_edges");
  if (c->idw != CC_U32 || multi_gpu(c))
    return fail(c, CC_ERR_INVALID, "cc_degrees_u32: u32 ids on one GPU only");
  const uint64_t n = c->n, m = c->m;
  if (count) *count = n;
  if (!out || cap < n) return fail(c, CC_ERR_INVALID, "output buffer too small");
  CK(cudaSetDevice(c->cfg.device));
  // the prediction stage's count (Alg. 2 line 2), same kernels and dispatch as cc_run in
  // CC_MODE_AUTO (the speculative root level included on large lists: its prefix is counted
  // by k_deg_sample)
  CK(cudaMemsetAsync(c->d_deg, 0, sizeof(uint32_t) * n, c->st));
  const bool spec_want = m >= graph::spec_min_edges();
  graph::SpecLevel spec{c->d_bm[1], c->d_bm[2], c->d_gctr};
  if (spec_want) {
    const uint64_t nw = (n + 31) / 32;
    CK(cudaMemsetAsync(c->d_gctr, 0, sizeof(uint64_t) * graph::G_NUM, c->st));
    CK(cudaMemsetAsync(spec.S, 0, sizeof(uint32_t) * 2 * nw, c->st));
    CK(cudaMemsetAsync(spec.next, 0, sizeof(uint32_t) * nw, c->st));
  }
  graph::launch_degree(c->d_edges, m, n, c->d_deg, c->st, c->d_tail, c->d_gctr + graph::G_NUM + 64,
                       c->d_w[1], sizeof(uint64_t) * c->cap, c->d_garc, spec_want ? &spec : nullptr);
  CKL();
  c->ran = false;  // tuple buffer 1 was scratch: labels need a new cc_run
  if (n)
    CK(cudaMemcpyAsync(out, c->d_deg, sizeof(uint32_t) * n,
                       out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

extern "C" cc_status cc_block_range(const cc_ctx* c, uint64_t* lo, uint64_t* hi) {
  if (!c || !lo || !hi) return CC_ERR_INVALID;
  if (!c->loaded) return CC_ERR_STATE;
  *lo = c->lo;
  *hi = c->hi;
  return CC_OK;
}

extern "C" cc_status cc_labels_device(cc_ctx* c, const uint32_t** labels, uint64_t* count) {
  if (!c || !labels) return CC_ERR_INVALID;
  if (!c->ran) return fail(c, CC_ERR_STATE, "cc_labels_device before cc_run");
  *labels = c->d_label;
  if (count) *count = c->n;
  return CC_OK;
}

extern "C" cc_status cc_kernel_stats(const cc_ctx* c, int which, double* ms, double* bytes,
                                     uint64_t* launches) {
  if (!c || which < 0 || which >= KF_N) return CC_ERR_INVALID;
  if (ms) *ms = c->kst[which].ms;
  if (bytes) *bytes = c->kst[which].bytes;
  if (launches) *launches = c->kst[which].launches;
  return CC_OK;
}

extern "C" cc_status cc_kernel_ops(const cc_ctx* c, int which, double* ops, const char** unit) {
  if (!c || which < 0 || which >= KF_N) return CC_ERR_INVALID;
  if (ops) *ops = c->kst[which].ops;
  if (unit) *unit = kKfOps[which];
  return CC_OK;
}

extern "C" const char* cc_kernel_name(int which) {
  return (which >= 0 && which < KF_N) ? kKfNames[which] : nullptr;
}

// Eccentricity of each seed in its component (BFS depth), the paper's approximate diameter
// being the maximum over random seeds.  u32 graphs on one GPU
// with n <= 2^26: builds the full CSR rows and runs the direction-optimising BFS per seed.
extern "C" cc_status cc_bfs_eccentricity(cc_ctx* c, const uint64_t* seeds, uint32_t count, uint64_t* ecc) {
  if (!c || (count && (!seeds || !ecc))) return CC_ERR_INVALID;
  if (!c->loaded) return fail(c, CC_ERR_STATE, "cc_bfs_eccentricity before cc_load_edges");
  if (c->idw != CC_U32 || multi_gpu(c)) return fail(c, CC_ERR_STATE, "u32 ids on one GPU only");
  const int gsf = csr::group_shift_full(c->n);
  if (gsf < 0) return fail(c, CC_ERR_INVALID, "n > 2^26 is not supported here");
  for (uint32_t i = 0; i < count; i++)
    if (seeds[i] >= c->n) return fail(c, CC_ERR_RANGE, "seed %llu >= n", (unsigned long long)seeds[i]);
  CK(cudaSetDevice(c->cfg.device));
  c->ran = false;  // the SV buffers are reused
  const uint64_t n = c->n, m = c->m;
  csr::bucket_degrees(c->d_edges, m, n, gsf, c->d_garc, c->d_gcur, reinterpret_cast<uint2*>(c->d_w[1]),
                      c->d_deg, c->st);
  uint64_t A = 0;
  TRY(build_full_rows(c, gsf, &A));
  for (uint32_t i = 0; i < count; i++) {
    uint64_t vis = 0, lev = 0;
    TRY(bfs_csr(c, seeds[i], m, &vis, &lev));
    ecc[i] = lev;
  }
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

extern "C" cc_status cc_approx_diameter(cc_ctx* c, const uint64_t* seeds, uint32_t count, uint64_t* diameter) {
  if (!c || !diameter || (count && !seeds)) return CC_ERR_INVALID;
  std::vector<uint64_t> ecc(count);
  *diameter = 0;
  TRY(cc_bfs_eccentricity(c, seeds, count, ecc.data()));
  for (uint32_t i = 0; i < count; i++) *diameter = std::max(*diameter, ecc[i]);
  return CC_OK;
}

extern "C" cc_status cc_radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t* tmp_keys,
                                         uint32_t* tmp_vals, uint64_t n, int key_bits, void* stream) {
  if (key_bits < 1 || key_bits > 64 || (n && (!keys || !vals || !tmp_keys || !tmp_vals)))
    return CC_ERR_INVALID;
  if (n < 2) return CC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  radix::Workspace ws;
  ws.max_tiles = n / radix::TILE_MIN + 2;
  if (cudaMallocAsync(&ws.ghist, sizeof(uint64_t) * radix::MAX_PASSES * radix::RADIX, st) != cudaSuccess ||
      cudaMallocAsync(&ws.lookback, sizeof(uint64_t) * ws.max_tiles * radix::RADIX, st) != cudaSuccess ||
      cudaMallocAsync(&ws.tile_ctr, sizeof(uint32_t) * radix::MAX_PASSES, st) != cudaSuccess) {
    cudaGetLastError();
    if (ws.ghist) cudaFreeAsync(ws.ghist, st);
    if (ws.lookback) cudaFreeAsync(ws.lookback, st);
    return CC_ERR_NOMEM;
  }
  cudaMemsetAsync(ws.lookback, 0, sizeof(uint64_t) * ws.max_tiles * radix::RADIX, st);
  uint64_t* k[2] = {keys, tmp_keys};
  uint32_t* v[2] = {vals, tmp_vals};
  uint64_t launches = 0;
  const int cur = radix::sort_pairs(ws, k, v, 0, n, key_bits, true, st, &launches, 0);
  if (cur == 1) {
    cudaMemcpyAsync(keys, tmp_keys, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(vals, tmp_vals, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st);
  }
  cudaFreeAsync(ws.ghist, st);
  cudaFreeAsync(ws.lookback, st);
  cudaFreeAsync(ws.tile_ctr, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? CC_OK : CC_ERR_CUDA;
}
