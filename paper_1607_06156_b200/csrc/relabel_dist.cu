// relabel_dist.cu -- u64 ids over several ranks (world_size > 1): the distributed form of
// Alg. 2 line 4 (sort the edge list, then "a parallel prefix (scan)
// operation to label the source vertices with a unique id in [0, V-1]") and the label
// output of a rank's vertex block in original ids (SURVEY.md §8(e) "u64 relabel =
// distributed sort-unique + rank map (two exchanges)").
//
//   1. local sort-unique of the rank's 2m endpoints (relabel::run_hash: hash dedupe, then a
//      radix sort of the distinct ids only): sorted distinct ids U and, per endpoint, its
//      index in U;
//   2. splitters: every rank contributes S regular samples of U weighted by |U|; the
//      all-gathered samples give world-1 splitters (sample sort);
//   3. U is cut at the splitters (binary search) and the runs go to their range owners by
//      one all-to-all-v; each owner sort-uniques what it received: its share G of the
//      globally distinct ids, in id order, disjoint from and ordered after lower ranks';
//   4. the share sizes are all-gathered: dense id of G[i] = (sizes of lower ranks) + i, so
//      dense order = id order over all ranks (the min label is preserved);
//   5. the dense ids go back along the reverse all-to-all-v, arriving in U order, and every
//      endpoint is rewritten as the dense id of its U entry (u32 edges).
// The rest of cc_run is the u32 multi-GPU path (cc_dist.cu) on id range n = sum of shares.
// Labels (cc_labels_u64): the block's original ids are slices of the shares (one
// all-to-all-v), and each label is translated by a request/reply exchange to the rank whose
// share holds it (labels sorted by value so each destination gets one run).
#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "relabel.cuh"

namespace cc {
namespace rdist {

constexpr int B = 256;
constexpr uint32_t S = 256;  // samples per rank

static unsigned grid(uint64_t work, unsigned cap) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + B - 1) / B, cap));
}

// S regular samples of the sorted array a[0..n)
__global__ void k_samples(const uint64_t* __restrict__ a, uint64_t n, uint64_t* __restrict__ out) {
  for (uint32_t j = threadIdx.x; j < S; j += B) out[j] = n ? a[(uint64_t)j * n / S] : ~0ull;
}
// pos[j] = first index i of the sorted a[0..n) with a[i] >= key[j]
__global__ void k_lower_bounds(const uint64_t* __restrict__ a, uint64_t n, const uint64_t* __restrict__ key,
                               uint32_t nk, uint64_t* __restrict__ pos) {
  const uint32_t j = blockIdx.x * B + threadIdx.x;
  if (j >= nk) return;
  uint64_t lo = 0, hi = n;
  const uint64_t x = key[j];
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  pos[j] = lo;
}
__global__ void k_add(uint32_t* a, uint64_t n, uint32_t base) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B) a[i] += base;
}
// label requests answered in place: dense id -> original id of this rank's share
__global__ void k_answer(uint64_t* x, uint64_t n, const uint64_t* __restrict__ gids, uint64_t base) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B)
    x[i] = gids[x[i] - base];
}
__global__ void k_label_keys(const uint32_t* __restrict__ label, uint64_t n, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B) {
    keys[i] = label[i];
    vals[i] = (uint32_t)i;
  }
}
__global__ void k_scatter(const uint64_t* __restrict__ x, const uint32_t* __restrict__ vals, uint64_t n,
                          uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B)
    out[vals[i]] = x[i];
}

}  // namespace rdist
}  // namespace cc

using namespace cc::rdist;

// grow-once scratch; the outcome is agreed on by all ranks (comm_agree), since every call
// site is followed by a collective that a rank which failed here would never enter
template <typename T>
static cc_status grow(cc_ctx* c, T** p, uint64_t* cap, uint64_t need) {
  cc_status s = CC_OK;
  if (!*p || *cap < need) {
    s = dalloc_t(c, p, need);
    if (s == CC_OK) *cap = need;
  }
  return comm_agree(c, s);
}

// counts[j] of this rank -> everyone's; returns what each rank sends to this one
static cc_status exchange_counts(cc_ctx* c, const std::vector<uint64_t>& mine, std::vector<uint64_t>* from) {
  const int world = c->cfg.world_size, rank = c->cfg.rank;
  uint64_t* cnt = c->d_cnt;
  CK(cudaMemcpyAsync(cnt, mine.data(), sizeof(uint64_t) * world, cudaMemcpyHostToDevice, c->st));
  TRY(comm_allgather(c, cnt, cnt + 2 * world, sizeof(uint64_t) * world));
  std::vector<uint64_t> all((size_t)world * world);
  CK(cudaMemcpyAsync(all.data(), cnt + 2 * world, sizeof(uint64_t) * world * world, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  from->assign(world, 0);
  for (int j = 0; j < world; j++) (*from)[j] = all[(size_t)j * world + rank];
  return CC_OK;
}

// run lengths of the sorted keys a[0..n) cut at split[0..world-1) (lower bounds)
static cc_status cut_runs(cc_ctx* c, const uint64_t* a, uint64_t n, const std::vector<uint64_t>& split,
                          uint64_t* scratch, std::vector<uint64_t>* runs) {
  const int world = c->cfg.world_size;
  std::vector<uint64_t> pos(world + 1, 0);
  pos[world] = n;
  if (world > 1) {
    CK(cudaMemcpyAsync(scratch, split.data(), sizeof(uint64_t) * (world - 1), cudaMemcpyHostToDevice, c->st));
    k_lower_bounds<<<grid(world - 1, 1024), B, 0, c->st>>>(a, n, scratch, (uint32_t)(world - 1),
                                                            scratch + world);
    c->launches += 1;
    CKL();
    CK(cudaMemcpyAsync(pos.data() + 1, scratch + world, sizeof(uint64_t) * (world - 1), cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  runs->assign(world, 0);
  for (int j = 0; j < world; j++) (*runs)[j] = pos[j + 1] - pos[j];
  return CC_OK;
}

static std::vector<uint64_t> bytes_of(const std::vector<uint64_t>& cnt, uint64_t w) {
  std::vector<uint64_t> b(cnt.size());
  for (size_t i = 0; i < cnt.size(); i++) b[i] = cnt[i] * w;
  return b;
}

cc_status dist_relabel(cc_ctx* c) {
  const int world = c->cfg.world_size, rank = c->cfg.rank;
  const uint64_t k = 2 * c->m;  // this rank's endpoints
  uint64_t* total = c->d_gctr + graph::G_NUM + 1537;
  uint32_t* vals[2] = {c->d_q[0], c->d_q[1]};
  // samples, splitters and bounds live in the (not yet used) label staging buffer
  TRY(grow(c, &c->d_out64, &c->out64_cap, (uint64_t)(S + 1) * (world + 1) + 2 * world + 8));
  uint64_t* small = c->d_out64;

  // 1. local sort-unique: U = c->d_uids[0..u), endpoint -> index in U in the u32 edge array
  TRY(scan_epoch_guard(c));
  CK(cudaMemsetAsync(total, 0, sizeof(uint64_t), c->st));
  if (c->d_htab)
    TRY(comm_agree(c, relabel_hash(c, k, total)));  // a rank may grow its table (local failure)
  else
    relabel::run(c->d_ids64, k, c->d_w, vals, c->rws, c->ss, reinterpret_cast<uint32_t*>(c->d_edges), c->d_uids,
                 total, c->st, &c->launches);
  CKL();
  uint64_t u = 0;
  CK(cudaMemcpyAsync(&u, total, sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));

  // 2. splitters from S regular samples per rank, each weighing |U| / S ids
  uint64_t* mysmp = small;                  // [u, S samples]
  uint64_t* allsmp = small + (S + 1);       // world x (S + 1)
  uint64_t* scratch = allsmp + (uint64_t)(S + 1) * world;
  CK(cudaMemcpyAsync(mysmp, &u, sizeof(uint64_t), cudaMemcpyHostToDevice, c->st));
  k_samples<<<1, B, 0, c->st>>>(c->d_uids, u, mysmp + 1);
  c->launches += 1;
  CKL();
  TRY(comm_allgather(c, mysmp, allsmp, sizeof(uint64_t) * (S + 1)));
  std::vector<uint64_t> hs((size_t)(S + 1) * world);
  CK(cudaMemcpyAsync(hs.data(), allsmp, sizeof(uint64_t) * hs.size(), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  std::vector<std::pair<uint64_t, double>> smp;
  double wsum = 0;
  for (int r = 0; r < world; r++) {
    const uint64_t ur = hs[(size_t)r * (S + 1)];
    if (!ur) continue;
    for (uint32_t j = 0; j < S; j++) smp.push_back({hs[(size_t)r * (S + 1) + 1 + j], (double)ur / S});
    wsum += (double)ur;
  }
  std::sort(smp.begin(), smp.end());
  std::vector<uint64_t> split(world > 1 ? world - 1 : 0, ~0ull);
  {
    double acc = 0;
    size_t i = 0;
    for (int d = 1; d < world; d++) {
      const double target = wsum * d / world;
      while (i < smp.size() && acc + smp[i].second <= target) acc += smp[i++].second;
      split[d - 1] = i < smp.size() ? smp[i].first : ~0ull;
    }
  }

  // 3. runs of U to their range owners; the owner sort-uniques what it receives
  std::vector<uint64_t> sendc, recvc;
  TRY(cut_runs(c, c->d_uids, u, split, scratch, &sendc));
  TRY(exchange_counts(c, sendc, &recvc));
  uint64_t r = 0;
  for (int j = 0; j < world; j++) r += recvc[j];
  TRY(grow(c, &c->d_xid, &c->xid_cap, r + 1));
  TRY(comm_alltoallv(c, c->d_uids, bytes_of(sendc, 8).data(), c->d_xid, bytes_of(recvc, 8).data()));
  TRY(ensure_tuple_cap(c, std::max(r, k)));
  vals[0] = c->d_q[0];
  vals[1] = c->d_q[1];
  TRY(grow(c, &c->d_xu32, &c->xu32_cap, r + 1));
  TRY(grow(c, &c->d_gids, &c->gids_cap, r + 1));
  TRY(scan_epoch_guard(c));
  CK(cudaMemsetAsync(total, 0, sizeof(uint64_t), c->st));
  relabel::run(c->d_xid, r, c->d_w, vals, c->rws, c->ss, c->d_xu32, c->d_gids, total, c->st, &c->launches);
  CKL();

  // 4. share sizes -> dense id bases (dense order = id order over all ranks)
  TRY(comm_allgather(c, total, c->d_cnt + 2 * world, sizeof(uint64_t)));
  std::vector<uint64_t> g(world);
  CK(cudaMemcpyAsync(g.data(), c->d_cnt + 2 * world, sizeof(uint64_t) * world, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->gbase.assign(world + 1, 0);
  for (int j = 0; j < world; j++) c->gbase[j + 1] = c->gbase[j] + g[j];
  const uint64_t n = c->gbase[world];
  if (n > (1ull << 30)) return fail(c, CC_ERR_INVALID, "%llu distinct ids > 2^30", (unsigned long long)n);

  // 5. dense ids back along the reverse exchange (arriving in U order); edges rewritten
  if (r) k_add<<<grid(r, 148 * 8), B, 0, c->st>>>(c->d_xu32, r, (uint32_t)c->gbase[rank]);
  TRY(comm_alltoallv(c, c->d_xu32, bytes_of(recvc, 4).data(), c->d_q[0], bytes_of(sendc, 4).data()));
  relabel::apply(reinterpret_cast<uint32_t*>(c->d_edges), k, c->d_q[0], c->st);
  c->launches += 2;
  CKL();
  if (!c->d_label || c->n_alloc < n) TRY(alloc_vertex_buffers(c, n));
  else {
    c->n = n;
    c->kbits = bits_for(n);
  }
  return CC_OK;
}

cc_status dist_labels_u64(cc_ctx* c, uint64_t* ids, uint64_t* labels, int out_on_device) {
  const int world = c->cfg.world_size, rank = c->cfg.rank;
  const uint64_t n = c->n, lo = c->lo, hi = c->hi, cnt = hi - lo, blk = c->blk;
  TRY(grow(c, &c->d_out64, &c->out64_cap, std::max<uint64_t>(2 * cnt, 2 * world) + 2 * world + 8));
  uint64_t* oid = c->d_out64;
  uint64_t* olab = c->d_out64 + cnt;
  uint64_t* scratch = c->d_out64 + 2 * cnt;

  // original ids of the block: the overlaps of the shares with the blocks, in rank order
  std::vector<uint64_t> sendc(world), recvc(world);
  auto overlap = [](uint64_t a0, uint64_t a1, uint64_t b0, uint64_t b1) {
    const uint64_t x = std::max(a0, b0), y = std::min(a1, b1);
    return y > x ? y - x : 0;
  };
  for (int j = 0; j < world; j++) {
    const uint64_t l = std::min<uint64_t>(n, blk * j), h = std::min<uint64_t>(n, l + blk);
    sendc[j] = overlap(c->gbase[rank], c->gbase[rank + 1], l, h);
    recvc[j] = overlap(c->gbase[j], c->gbase[j + 1], lo, hi);
  }
  TRY(comm_alltoallv(c, c->d_gids, bytes_of(sendc, 8).data(), oid, bytes_of(recvc, 8).data()));

  // labels: requests sorted by dense label, one run per share owner, answered in place
  uint32_t* vals[2] = {c->d_q[0], c->d_q[1]};
  int cur = 0;
  if (cnt) {
    k_label_keys<<<grid(cnt, 148 * 8), B, 0, c->st>>>(c->d_label + lo, cnt, c->d_w[0], vals[0]);
    c->launches += 1;
    CKL();
    cur = radix::sort_pairs(c->rws, c->d_w, vals, 0, cnt, std::max(1, bits_for(n)), true, c->st, &c->launches, 0);
  }
  std::vector<uint64_t> cuts(c->gbase.begin() + 1, c->gbase.begin() + world);
  std::vector<uint64_t> reqc, ansc;
  TRY(cut_runs(c, c->d_w[cur], cnt, cuts, scratch, &reqc));
  TRY(exchange_counts(c, reqc, &ansc));
  uint64_t na = 0;
  for (int j = 0; j < world; j++) na += ansc[j];
  TRY(grow(c, &c->d_xid, &c->xid_cap, na + 1));
  TRY(comm_alltoallv(c, c->d_w[cur], bytes_of(reqc, 8).data(), c->d_xid, bytes_of(ansc, 8).data()));
  if (na) k_answer<<<grid(na, 148 * 8), B, 0, c->st>>>(c->d_xid, na, c->d_gids, c->gbase[rank]);
  TRY(comm_alltoallv(c, c->d_xid, bytes_of(ansc, 8).data(), c->d_w[1 - cur], bytes_of(reqc, 8).data()));
  if (cnt) k_scatter<<<grid(cnt, 148 * 8), B, 0, c->st>>>(c->d_w[1 - cur], vals[cur], cnt, olab);
  c->launches += 2;
  CKL();
  const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (cnt) {
    CK(cudaMemcpyAsync(ids, oid, sizeof(uint64_t) * cnt, kind, c->st));
    CK(cudaMemcpyAsync(labels, olab, sizeof(uint64_t) * cnt, kind, c->st));
  }
  CK(cudaStreamSynchronize(c->st));
  return CC_OK;
}
