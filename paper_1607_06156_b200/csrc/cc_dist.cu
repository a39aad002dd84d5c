// cc_dist.cu -- the multi-GPU driver of cc_run (world_size > 1): SURVEY.md §8(e).
//
// One process per GPU; rank k loads its block of the edge list and owns the
// vertex block [lo, hi) = [k*blk, (k+1)*blk) (blk a multiple of 32).
//   prediction  (modes auto, bfs+sv) each rank counts the degrees of its own edges with the
//               single-GPU kernels; the counts are summed over ranks, so every rank holds all
//               degrees, builds the same distribution and fits the same gate (Alg. 2 lines 2-3)
//   BFS peel    edge-partitioned (bfs_stream, cc_api.cu): every rank streams its own edges
//               with a replicated 2-bit vertex state and compacts its own list; the found
//               bitmaps are OR-ed after each level (Alg. 2 lines 7-11).  No edge moves.
//   regroup     the remaining arcs go to the owner of their third element r: Alg. 1's regroup
//               by r as one all-to-all, and since r never changes
//                no tuple moves again.  Mode sv: all arcs, the degrees (and the
//               distribution under CC_FLAG_TRACE) from the received arcs
//   SV          sv_iterate(): rows are local, partition slots are combined over ranks after
//               each row pass (min of minima, OR of NCP), statistics are identical on all ranks
// The exchange goes through the library's NCCL communicator (cfg.nccl_id) or the caller's
// cc_comm callbacks (gloo in the tests).
#include <algorithm>
#include <cmath>
#include <vector>

#include "ctx.cuh"

namespace cc {
namespace dist {

constexpr int DB = 256;
constexpr int MAXW = 256;        // ranks supported by the shared-memory owner histograms
constexpr uint32_t TAILX = 8192; // degrees >= HIST_DENSE per rank that the gate exchange carries


// arcs per owner rank of this rank's edges: {x,y} gives <x,_,y> to owner(y), <y,_,x> to owner(x)
__global__ void k_owner_count(const uint2* __restrict__ e, uint64_t m, uint32_t blk, int world,
                              unsigned long long* cnt) {
  __shared__ unsigned long long s[MAXW];
  for (int i = threadIdx.x; i < world; i += DB) s[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)DB + threadIdx.x; i < m; i += (uint64_t)gridDim.x * DB) {
    const uint2 xy = e[i];
    atomicAdd(&s[xy.y / blk], 1ull);
    atomicAdd(&s[xy.x / blk], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < world; i += DB)
    if (s[i]) atomicAdd(&cnt[i], s[i]);
}

// arcs (r, p) into per-owner runs of `out`; cursor[k] = next free slot of owner k's run.
constexpr int SITEMS = 4;
__global__ void __launch_bounds__(DB) k_owner_scatter(const uint2* __restrict__ e, uint64_t m,
                                                      uint32_t blk, int world,
                                                      unsigned long long* cursor,
                                                      uint2* __restrict__ out) {
  __shared__ uint32_t s_cnt[MAXW];
  __shared__ unsigned long long s_base[MAXW];
  for (int i = threadIdx.x; i < world; i += DB) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t e0 = blockIdx.x * (uint64_t)DB * SITEMS + threadIdx.x;
  uint2 arc[2 * SITEMS];
  uint32_t slot[2 * SITEMS];
  uint2 ld[SITEMS];  // all loads in flight before the first (ordering) shared atomic
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * DB;
    ld[k] = i < m ? e[i] : make_uint2(0, 0);
  }
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * DB;
    if (i < m) {
      const uint2 xy = ld[k];
      arc[2 * k] = make_uint2(xy.y, xy.x);      // <x,_,y>: r = y, p = x
      arc[2 * k + 1] = make_uint2(xy.x, xy.y);  // <y,_,x>: r = x, p = y
      slot[2 * k] = atomicAdd(&s_cnt[xy.y / blk], 1u);
      slot[2 * k + 1] = atomicAdd(&s_cnt[xy.x / blk], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < world; i += DB)
    s_base[i] = s_cnt[i] ? atomicAdd(&cursor[i], (unsigned long long)s_cnt[i]) : 0ull;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * DB;
    if (i < m) {
      out[s_base[arc[2 * k].x / blk] + slot[2 * k]] = arc[2 * k];
      out[s_base[arc[2 * k + 1].x / blk] + slot[2 * k + 1]] = arc[2 * k + 1];
    }
  }
}

// deg(r) = arcs with third element r (all of them arrive at r's owner; a self-loop gives 2)
__global__ void k_arc_degree(const uint2* __restrict__ arcs, uint64_t na, uint32_t* deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)DB + threadIdx.x; i < na; i += (uint64_t)gridDim.x * DB)
    atomicAdd(&deg[arcs[i].x], 1u);
}

static unsigned gsz(uint64_t work, unsigned cap) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + DB - 1) / DB, cap));
}

// 'Balanced' variant: split points of this rank's rows for an even
// redistribution.  R (flag-masked) is nondecreasing over the concatenation of all ranks'
// arrays (rank k's rows come before rank k+1's), so the tuple at global position g belongs to
// rank g / q, and a row goes whole to the rank of its head: split[t] is the first row head at
// or after global position t*q.
__global__ void k_bal_splits(const uint32_t* __restrict__ R, uint64_t len, uint64_t before, uint64_t q,
                             int world, unsigned long long* split) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > world) return;
  uint64_t s;
  if (t == 0) s = 0;
  else if (t == world) s = len;
  else {
    const uint64_t g = (uint64_t)t * q;
    if (g <= before) s = 0;
    else if (g - before >= len) s = len;
    else {
      uint64_t j = g - before;
      const uint32_t v = R[j] & ~csr::R_LONG;
      if ((R[j - 1] & ~csr::R_LONG) != v) s = j;
      else {  // first index past the row holding j
        uint64_t lo = j, hi = len;
        while (lo < hi) {
          const uint64_t mid = lo + (hi - lo) / 2;
          if ((R[mid] & ~csr::R_LONG) > v) hi = mid;
          else lo = mid + 1;
        }
        s = lo;
      }
    }
  }
  split[t] = s;
}

}  // namespace dist
}  // namespace cc

using namespace cc::dist;

// Degrees >= HIST_DENSE (mode sv, distribution from the owned blocks): every rank's short
// tail list is all-gathered and merged, so every rank fits the gate on the same distribution.
static cc_status gather_tails(cc_ctx* c) {
  const int world = c->cfg.world_size;
  const uint64_t mytail = c->h_gctr[graph::G_TAIL];
  cc_status s = CC_OK;
  if (mytail > TAILX) s = fail(c, CC_ERR_INVALID, "more than %u degrees >= 2^20 on one rank", TAILX);
  // scratch: everyone's lists [0, world (TAILX + 1)), then my own (count, entries)
  const uint64_t need = (uint64_t)(world + 1) * (TAILX + 1);
  if (s == CC_OK && (!c->d_gath || c->gath_cap < need)) {
    s = dalloc_t(c, &c->d_gath, need);
    if (s == CC_OK) c->gath_cap = need;
  }
  TRY(comm_agree(c, s));
  uint32_t* gathered = c->d_gath;
  uint32_t* stage = c->d_gath + (uint64_t)world * (TAILX + 1);
  uint32_t nt32 = (uint32_t)mytail;
  CK(cudaMemcpyAsync(stage, &nt32, sizeof(uint32_t), cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(stage + 1, c->d_tail, sizeof(uint32_t) * TAILX, cudaMemcpyDeviceToDevice, c->st));
  TRY(comm_allgather(c, stage, gathered, sizeof(uint32_t) * (TAILX + 1)));
  std::vector<uint32_t> h((size_t)world * (TAILX + 1)), merged;
  CK(cudaMemcpyAsync(h.data(), gathered, sizeof(uint32_t) * h.size(), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (int k = 0; k < world; k++) {
    const uint32_t* b = h.data() + (size_t)k * (TAILX + 1);
    merged.insert(merged.end(), b + 1, b + 1 + b[0]);
  }
  CK(cudaMemcpyAsync(c->d_tail, merged.data(), sizeof(uint32_t) * merged.size(), cudaMemcpyHostToDevice,
                     c->st));
  const uint64_t tn = merged.size();
  CK(cudaMemcpyAsync(c->d_gctr + graph::G_TAIL, &tn, sizeof(uint64_t), cudaMemcpyHostToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}

cc_status run_dist(cc_ctx* c, cc_mode mode) {
  cc_report& R = c->rep;
  const int world = c->cfg.world_size, rank = c->cfg.rank;
  const uint64_t n = c->n, m = c->m;
  const uint64_t blk = c->blk, lo = c->lo, hi = c->hi;
  if (world > MAXW) return fail(c, CC_ERR_INVALID, "world_size %d > %d", world, MAXW);
  cudaEvent_t e0 = ev_get(c), e_pred, e_bfs, e_filter, e_sv;
  CK(cudaEventRecord(e0, c->st));
  CK(cudaMemsetAsync(c->d_gctr, 0, sizeof(uint64_t) * graph::G_NUM, c->st));
  CK(cudaMemsetAsync(c->d_gctr + graph::G_MINVIS, 0xFF, sizeof(uint64_t), c->st));
  sv::launch_init_labels(c->d_label, n, c->st);
  c->launches += 1;

  // ------------------------------------------------ prediction on the rank's own edges
  // (Alg. 2 lines 2-3; modes auto and bfs+sv): every rank counts the degrees its edges give
  // (the single-GPU kernels) and the counts are summed over ranks, so every rank holds all
  // degrees and fits the same gate; no edge has moved yet.
  bool run_bfs = false, deg_known = false;
  uint64_t root = 0;
  const uint2* sv_edges = c->d_edges;
  uint64_t m_sv = m;
  const uint32_t* vis = nullptr;
  e_pred = e_bfs = e_filter = e0;
  if (mode != CC_MODE_SV) {
    CK(cudaMemsetAsync(c->d_deg, 0, sizeof(uint32_t) * (n + 1), c->st));
    {
      Prof k(c, KF_PREDICT);
      const int algo = graph::launch_degree(c->d_edges, m, n, c->d_deg, c->st, c->d_tail,
                                            c->d_gctr + graph::G_NUM + 64, c->d_w[1], sizeof(uint64_t) * c->cap,
                                            c->d_garc) & 1;
      k.end(algo ? 16.0 * m + 8.0 * n : 8.0 * m + 4.0 * n, algo ? 3 : 1, algo ? 4.0 * m : 0.0);
    }
    // sum over ranks (u32 sums as int32: the same bits)
    TRY(comm_allreduce(c, c->d_deg, n, CC_DT_I32, CC_OP_SUM));
    const bool want_hist = (mode == CC_MODE_AUTO) || (c->cfg.flags & CC_FLAG_TRACE);
    if (want_hist) CK(cudaMemsetAsync(c->d_hist, 0, sizeof(uint32_t) * graph::HIST_DENSE, c->st));
    graph::launch_deg_hist(c->d_deg, n, c->d_hist, c->d_tail, c->d_gctr, c->st);
    c->launches += 2;
    CKL();
    TRY(predict_gate(c, mode, want_hist, &run_bfs, &root));
    deg_known = true;
    e_pred = ev_get(c);
    CK(cudaEventRecord(e_pred, c->st));
    // ---------------------------------------------- BFS peel + filter (lines 7-11)
    // edge-partitioned: each rank streams its own edges with a replicated vertex state; the
    // found bitmaps are OR-ed after each level (bfs_stream), and each rank filters its own
    // list, so only the remainder is ever exchanged
    e_bfs = e_filter = e_pred;
    if (run_bfs) {
      R.ran_bfs = 1;
      R.bfs_root = root;
      TRY(bfs_stream(c, root, false, &sv_edges, &m_sv, &e_bfs));
      vis = c->d_bm[0];
      uint64_t* tmp = c->d_ctr + sv::C_ERR;
      CK(cudaMemcpyAsync(tmp, &m_sv, sizeof(uint64_t), cudaMemcpyHostToDevice, c->st));
      TRY(comm_allreduce(c, tmp, 1, CC_DT_I64, CC_OP_SUM));
      uint64_t rem_all = 0;
      CK(cudaMemcpyAsync(&rem_all, tmp, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      R.remainder_edges = rem_all;
      e_filter = ev_get(c);
      CK(cudaEventRecord(e_filter, c->st));
    }
  }

  // ------------------------------------------------ regroup by r: (remaining) arcs to their owners
  uint64_t* cnt = c->d_cnt;  // [0, world): my arcs per owner; [world, 2 world): cursors;
                             // [2 world, 2 world + world^2): everyone's counts (gathered)
  CK(cudaMemsetAsync(cnt, 0, sizeof(uint64_t) * world, c->st));
  auto* ucnt = reinterpret_cast<unsigned long long*>(cnt);
  if (m_sv) k_owner_count<<<gsz(m_sv, 148 * 4), DB, 0, c->st>>>(sv_edges, m_sv, (uint32_t)blk, world, ucnt);
  CKL();
  std::vector<uint64_t> mine(world), allc((size_t)world * world), sb(world), rb(world);
  CK(cudaMemcpyAsync(mine.data(), cnt, sizeof(uint64_t) * world, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  {
    std::vector<uint64_t> cur(world);
    uint64_t acc = 0;
    for (int k = 0; k < world; k++) { cur[k] = acc; acc += mine[k]; }
    CK(cudaMemcpyAsync(cnt + world, cur.data(), sizeof(uint64_t) * world, cudaMemcpyHostToDevice, c->st));
  }
  if (m_sv)  // d_send holds 2m + 1 arcs (cc_load_edges), m_sv <= m
    k_owner_scatter<<<(unsigned)((m_sv + DB * SITEMS - 1) / (DB * SITEMS)), DB, 0, c->st>>>(
        sv_edges, m_sv, (uint32_t)blk, world, ucnt + world, c->d_send);
  CKL();
  TRY(comm_allgather(c, cnt, cnt + 2 * world, sizeof(uint64_t) * world));
  CK(cudaMemcpyAsync(allc.data(), cnt + 2 * world, sizeof(uint64_t) * world * world,
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  uint64_t na = 0;
  for (int k = 0; k < world; k++) {
    sb[k] = mine[k] * sizeof(uint2);
    rb[k] = allc[(size_t)k * world + rank] * sizeof(uint2);
    na += allc[(size_t)k * world + rank];
  }
  {
    // the owned rows' tuples (received arcs + one vertex tuple per owned id) are indexed by
    // 32-bit CSR offsets (csr::build): a skewed rank must not wrap them.  Every local failure
    // before the next collective is agreed on by all ranks (comm_agree).
    cc_status s = CC_OK;
    if (na + (hi - lo) + 64 >= (1ull << 32))
      s = fail(c, CC_ERR_INVALID, "rank %d owns %llu arcs + %llu ids: more than 2^32 tuples", rank,
               (unsigned long long)na, (unsigned long long)(hi - lo));
    if (s == CC_OK && (!c->d_recv || c->recv_cap < na + 1)) {
      s = dalloc_t(c, &c->d_recv, na + 1);
      if (s == CC_OK) c->recv_cap = na + 1;
    }
    TRY(comm_agree(c, s));
  }
  TRY(comm_alltoallv(c, c->d_send, sb.data(), c->d_recv, rb.data()));
  TRY(comm_agree(c, ensure_tuple_cap(c, na + (hi - lo))));
  c->launches += 2;

  if (!deg_known) {
    // ---------------------------------------------- prediction from the received arcs (mode sv:
    // the distribution only under CC_FLAG_TRACE)
    CK(cudaMemsetAsync(c->d_deg, 0, sizeof(uint32_t) * (n + 1), c->st));
    if (na) k_arc_degree<<<gsz(na, 148 * 16), DB, 0, c->st>>>(c->d_recv, na, c->d_deg);
    const bool want_hist = (mode == CC_MODE_AUTO) || (c->cfg.flags & CC_FLAG_TRACE);
    CK(cudaMemsetAsync(c->d_hist, 0, sizeof(uint32_t) * graph::HIST_DENSE, c->st));
    if (hi > lo) graph::launch_deg_hist(c->d_deg + lo, hi - lo, c->d_hist, c->d_tail, c->d_gctr, c->st, lo);
    c->launches += 2;
    CKL();
    TRY(comm_allreduce(c, c->d_gctr + graph::G_MAXKEY, 1, CC_DT_I64, CC_OP_MAX));
    TRY(comm_allreduce(c, c->d_gctr + graph::G_NPRESENT, 1, CC_DT_I64, CC_OP_SUM));
    TRY(sync_read(c));
    const uint64_t dmax = c->h_gctr[graph::G_MAXKEY] >> 32;
    if (want_hist && dmax > 0) {
      const uint64_t dense_n = std::min<uint64_t>(dmax + 1, graph::HIST_DENSE);
      TRY(comm_allreduce(c, c->d_hist, dense_n, CC_DT_I32, CC_OP_SUM));
      // degrees beyond the dense bins: gather every rank's short tail list
      if (dmax >= graph::HIST_DENSE) TRY(gather_tails(c));
    }
    bool rb_unused = false;
    uint64_t root_unused = 0;
    TRY(predict_gate(c, mode, want_hist, &rb_unused, &root_unused));
    e_pred = e_bfs = e_filter = ev_get(c);
    CK(cudaEventRecord(e_pred, c->st));
  } else {
    // rows exist for owned ids only: the other ranks' degrees leave the CSR count
    if (lo) CK(cudaMemsetAsync(c->d_deg, 0, sizeof(uint32_t) * lo, c->st));
    if (n > hi) CK(cudaMemsetAsync(c->d_deg + hi, 0, sizeof(uint32_t) * (n - hi), c->st));
  }

  // ------------------------------------------------ owned CSR rows from the received arcs
  // (remainder route: visited ids get no vertex tuple; an unvisited id's arcs all stayed, so
  // its full degree is its remainder degree)
  uint32_t* Rt = reinterpret_cast<uint32_t*>(c->d_w[0]);
  uint32_t* Pt = Rt + c->cap;
  uint32_t *off = c->d_q[0], *cur = c->d_q[1];
  CK(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint64_t) * sv::C_NUM, c->st));
  TRY(scan_epoch_guard(c));
  const int gshift = csr::group_shift(n, na + (hi - lo));
  uint32_t* garc = c->d_garc;
  uint64_t* gcur = c->d_gcur;
  uint64_t* nlong = gcur + 2048;
  csr::build(nullptr, na, c->d_deg, vis, n, off, cur, garc, gshift, c->ss, c->d_ctr, c->st);
  CKL();
  TRY(sync_read(c));
  const uint64_t len = c->h_ctr[sv::C_VT_OUT];  // tuples of owned rows
  TRY(comm_agree(c, len > c->cap ? fail(c, CC_ERR_INVALID, "tuple count exceeds capacity") : CC_OK));
  csr::fill(c->d_recv, na, off, cur, n, len, Rt, Pt, garc, gshift, gcur,
            reinterpret_cast<uint2*>(c->d_w[1]), c->d_segB, nlong, c->st, /*directed=*/true);
  c->launches += 6;
  CKL();

  // ------------------------------------------------ SV on the owned rows (Alg. 2 line 13)
  const uint64_t A_local = len;
  uint64_t* tmp = c->d_ctr + sv::C_ERR;
  CK(cudaMemcpyAsync(tmp, &A_local, sizeof(uint64_t), cudaMemcpyHostToDevice, c->st));
  TRY(comm_allreduce(c, tmp, 1, CC_DT_I64, CC_OP_SUM));
  uint64_t A = 0;
  CK(cudaMemcpyAsync(&A, tmp, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  R.sv_ids = n;
  if (A) TRY(sv_iterate(c, A, len, A_local));
  R.sv_iterations = (uint32_t)c->iters.size();
  // components: roots of the owned block, summed over ranks
  uint64_t* roots = c->d_ctr + sv::C_ERR;
  CK(cudaMemsetAsync(roots, 0, sizeof(uint64_t), c->st));
  graph::launch_count_roots(c->d_label, lo, hi, roots, c->st);
  TRY(comm_allreduce(c, roots, 1, CC_DT_I64, CC_OP_SUM));
  CK(cudaMemcpyAsync(&R.components, roots, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  e_sv = ev_get(c);
  CK(cudaEventRecord(e_sv, c->st));
  CK(cudaStreamSynchronize(c->st));
  R.ms_total = ev_ms(e0, e_sv);
  R.ms_prediction = ev_ms(e0, e_pred);
  R.ms_bfs = run_bfs ? ev_ms(e_pred, e_bfs) : 0;
  R.ms_filter = run_bfs ? ev_ms(e_bfs, e_filter) : 0;
  R.ms_sv = ev_ms(e_filter, e_sv);
  return CC_OK;
}

// 'Balanced' variant (sec:distSVOpt2; CC_FLAG_BALANCE): the live rows of all
// ranks are redistributed evenly, whole rows, in global order (R nondecreasing over the ranks'
// concatenation), by one all-to-all-v of R and one of P.  Rows may leave their owner: the
// slots are combined over ranks anyway, the long-row list needs the global degrees
// (sv_iterate sums them first) and the labels are min-combined at the end.  Collective; the
// plan is computed identically on every rank from the gathered loads and split vectors, and a
// plan that would overflow some rank's tuple capacity is skipped (*moved = false).
cc_status rebalance_rows(cc_ctx* c, const uint32_t* Rsrc, const uint32_t* Psrc, uint32_t* Rdst,
                         uint32_t* Pdst, uint64_t len, const std::vector<uint64_t>& loads,
                         uint64_t* new_len, bool* moved) {
  const int world = c->cfg.world_size, rank = c->cfg.rank;
  *moved = false;
  uint64_t total = 0, before = 0;
  for (int k = 0; k < world; k++) {
    total += loads[2 * k];
    if (k < rank) before += loads[2 * k];
  }
  const uint64_t q = (total + world - 1) / world;
  if (!c->d_bal) {
    cc_status s = dalloc_t(c, &c->d_bal, (uint64_t)(world + 1) + (uint64_t)world * (world + 1));
    TRY(comm_agree(c, s));
  }
  uint64_t* split = c->d_bal;                // world + 1
  uint64_t* all = c->d_bal + world + 1;      // world x world send counts (tuples)
  k_bal_splits<<<(world + 128) / 128, 128, 0, c->st>>>(Rsrc, len, before, q, world,
                                                        reinterpret_cast<unsigned long long*>(split));
  c->launches += 1;
  CKL();
  std::vector<uint64_t> sp(world + 1), cnt(world), mat((size_t)world * world);
  CK(cudaMemcpyAsync(sp.data(), split, sizeof(uint64_t) * (world + 1), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (int t = 0; t < world; t++) cnt[t] = sp[t + 1] - sp[t];
  CK(cudaMemcpyAsync(split, cnt.data(), sizeof(uint64_t) * world, cudaMemcpyHostToDevice, c->st));
  TRY(comm_allgather(c, split, all, sizeof(uint64_t) * world));
  CK(cudaMemcpyAsync(mat.data(), all, sizeof(uint64_t) * world * world, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  // mat[j * world + k]: tuples rank j sends to rank k
  for (int k = 0; k < world; k++) {
    uint64_t in = 0;
    for (int j = 0; j < world; j++) in += mat[(size_t)j * world + k];
    if (in + 64 > loads[2 * k + 1]) return CC_OK;  // would overflow rank k: skip (all ranks agree)
  }
  std::vector<uint64_t> sb(world), rb(world);
  uint64_t nl = 0;
  for (int k = 0; k < world; k++) {
    sb[k] = sizeof(uint32_t) * mat[(size_t)rank * world + k];
    rb[k] = sizeof(uint32_t) * mat[(size_t)k * world + rank];
    nl += mat[(size_t)k * world + rank];
  }
  TRY(comm_alltoallv(c, Rsrc, sb.data(), Rdst, rb.data()));
  TRY(comm_alltoallv(c, Psrc, sb.data(), Pdst, rb.data()));
  *new_len = nl;
  *moved = true;
  return CC_OK;
}
