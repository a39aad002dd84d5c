// sv_csr.cu -- r-stationary edge-tuple SV (the default engine).
//
// Alg. 1 regroups A_i by the third element r (line 8) and by the first element p
// (line 14) in every pass.  r never changes ("The third
// element r ... is not changed throughout the algorithm") and the exclusion of completed
// partitions removes whole vertex buckets, so one stable regroup by r at the start keeps
// every later vertex bucket VB_i(u) contiguous: the tuple array is stored in CSR order
// (row u = VB(u) = <x,_,u> for x in N[u]) and is only ever compacted in order.  That
// one-time regroup is a counting sort on the degrees the prediction stage already
// computed (SURVEY.md §8(a) a4 "CSR build").  Partition buckets PB_i(p) are addressed
// directly: the minimum over PB_i(p) lives in slot p of an n-sized array kept in L2.
// The temporaries <p_min,_,p_min>_tmp of line 22 are a bitmap over vertices: all a temp
// does is add its own id p_min to VB(p_min) in pass 3 and its candidate to PB(p_min) in
// pass 4 (fig:doubling), which the pass kernels fold in from the bitmap.
// Every set and every counter of Alg. 1 is unchanged (tests/test_gpu_parity.py).
//
// Arrays (SoA, u32): R[i] = r (sorted), P[i] = p.  Slots: U[u] (u_min), NP (bitmap:
// |M(u)| > 1), PMIN[p] (p_min), NCP (bitmap: PB(p) has a tuple that is not potentially
// completed), TB (bitmap: temporary tuple targets).
#include <algorithm>

#include "csr.cuh"
#include "sv.cuh"

namespace cc {
namespace csr {

constexpr int B = 256;
constexpr uint32_t DEAD = 0xFFFFFFFFu;  // P of a tuple whose partition completed

CC_DEVI void min_slot(uint32_t* a, uint32_t i, uint32_t v) {
  if (v < *(volatile uint32_t*)&a[i]) atomicMin(&a[i], v);
}
CC_DEVI bool tbit(const uint32_t* bm, uint32_t i) { return (__ldg(&bm[i >> 5]) >> (i & 31)) & 1u; }
CC_DEVI bool tbit_v(const uint32_t* bm, uint32_t i) {
  return (*(volatile const uint32_t*)&bm[i >> 5] >> (i & 31)) & 1u;
}
CC_DEVI void set_bit(uint32_t* bm, uint32_t i) {
  const uint32_t m = 1u << (i & 31);
  if (!(*(volatile uint32_t*)&bm[i >> 5] & m)) atomicOr(&bm[i >> 5], m);
}

static unsigned grid(uint64_t work, unsigned per_block, unsigned cap) {
  uint64_t g = (work + per_block - 1) / per_block;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, cap));
}

// ===================================================================== CSR build (a4)
// cnt[v] = |VB_0(v)| = deg(v) + 1 for present v (the vertex tuple <v,_,v> + one tuple per
// arc into v), 0 otherwise.  Exclusive scan -> off[v]; cur[v] = off[v] + 1 is the next
// free slot for arcs.  Tile = B*8 vertices, single pass with decoupled look-back.
constexpr int SITEMS = 16;  // vertices per thread of k_rows (tiles of 4096: half the look-back chain of 8)
__global__ void __launch_bounds__(B) k_rows(const uint32_t* __restrict__ deg,
                                            const uint32_t* __restrict__ vis, uint64_t n,
                                            uint32_t* __restrict__ off, uint32_t* __restrict__ cur,
                                            uint64_t* flags, uint32_t* ticket, uint32_t epoch,
                                            unsigned long long* total, uint32_t* garc,
                                            int gshift, int count_groups) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_pref;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t v0 = tile * (B * SITEMS) + (uint64_t)threadIdx.x * SITEMS;
  uint32_t c[SITEMS];
  uint32_t sum = 0;
  const bool full = v0 + SITEMS <= n;  // 16-byte loads; the vertices' bits in one bitmap word
  if (full) {
#pragma unroll
    for (int q = 0; q < SITEMS / 4; q++) {
      const uint4 a = reinterpret_cast<const uint4*>(deg + v0)[q];
      c[4 * q] = a.x; c[4 * q + 1] = a.y; c[4 * q + 2] = a.z; c[4 * q + 3] = a.w;
    }
  }
  const uint32_t vb = vis ? (vis[v0 >> 5] >> (v0 & 31)) : 0u;
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    const uint64_t v = v0 + k;
    uint32_t x = full ? c[k] : (v < n ? deg[v] : 0u);
    if ((vb >> k) & 1u) x = 0;
    if (x) x += 1;
    c[k] = x;
    sum += x;
  }
  uint32_t tot;
  const uint32_t excl = block_excl_scan<B>(sum, s_scan, &tot);
  const uint64_t pref = scan::tile_prefix(flags, tile, tot, epoch, &s_pref);
  // arcs of this tile (tuples minus vertex tuples) for the CSR bucket pass; a tile of
  // B*SITEMS = 2^12 vertices lies inside one group of 2^gshift vertices (gshift >= 12)
  if (count_groups) {
    uint32_t nv = 0;
#pragma unroll
    for (int k = 0; k < SITEMS; k++) nv += (c[k] != 0);
    nv = warp_sum(nv);
    if ((threadIdx.x & 31) == 0 && nv) atomicSub(&garc[(tile * (B * SITEMS)) >> gshift], nv);
    if (threadIdx.x == 0 && tot) atomicAdd(&garc[(tile * (B * SITEMS)) >> gshift], tot);
  }
  uint32_t run = (uint32_t)pref + excl;
  uint32_t o[SITEMS];
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    o[k] = run;
    run += c[k];
  }
  if (full) {
#pragma unroll
    for (int q = 0; q < SITEMS / 4; q++) {
      reinterpret_cast<uint4*>(off + v0)[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      reinterpret_cast<uint4*>(cur + v0)[q] =
          make_uint4(o[4 * q] + 1, o[4 * q + 1] + 1, o[4 * q + 2] + 1, o[4 * q + 3] + 1);
    }
  } else {
#pragma unroll
    for (int k = 0; k < SITEMS; k++)
      if (v0 + k < n) {
        off[v0 + k] = o[k];
        cur[v0 + k] = o[k] + 1;
      }
  }
  if (n > 0 && v0 <= n - 1 && n - 1 < v0 + SITEMS) {  // owner of the last vertex
    off[n] = run;
    *total = run;
  }
}

// R and the vertex tuple <v,_,v> of each row: thread per vertex; rows longer than
// LONG_ROW (hubs) are appended to a list and filled by whole blocks.  R of rows longer than
// csr::LONG carries the R_LONG flag (sv_rows.cu: those rows go to the long-row kernels).
constexpr uint32_t LONG_ROW = 64;
static_assert(LONG_ROW <= LONG, "rows filled by threads are never long");
__global__ void __launch_bounds__(B) k_fill_rows(const uint32_t* __restrict__ off, uint64_t n,
                                                 uint32_t* __restrict__ R, uint32_t* __restrict__ P,
                                                 uint32_t* longlist, unsigned long long* nlong) {
  for (uint64_t v = blockIdx.x * (uint64_t)B + threadIdx.x; v < n; v += (uint64_t)gridDim.x * B) {
    const uint32_t a = off[v], b = off[v + 1];
    if (a == b) continue;
    P[a] = (uint32_t)v;
    if (b - a <= LONG_ROW) {
      for (uint32_t i = a; i < b; i++) R[i] = (uint32_t)v;
    } else {
      longlist[atomicAdd(nlong, 1ull)] = (uint32_t)v;
    }
  }
}
__global__ void __launch_bounds__(B) k_fill_long(const uint32_t* __restrict__ off,
                                                 const uint32_t* __restrict__ longlist,
                                                 const unsigned long long* nlong,
                                                 uint32_t* __restrict__ R) {
  const uint64_t cnt = *nlong;
  for (uint64_t j = blockIdx.x; j < cnt; j += gridDim.x) {
    const uint32_t v = longlist[j];
    const uint32_t a = off[v], b = off[v + 1];
    const uint32_t rv = v | (b - a > LONG ? R_LONG : 0u);  // long rows: row passes skip them
    for (uint32_t i = a + threadIdx.x; i < b; i += B) R[i] = rv;
  }
}

// Group cursor slot: with few groups (G <= 64, the large graphs) each cursor gets its own
// 256-byte line, so the per-block cursor atomics (C4 mode sv: 524 k blocks x 64 groups)
// spread over L2 slices instead of queueing on the two lines 64 packed counters share
__host__ __device__ inline uint32_t gslot(int g, int G) {
  return G <= 64 ? (uint32_t)g * 32u : G <= 256 ? (uint32_t)g * 8u : (uint32_t)g;
}
// Group start offsets of the bucketed arc list (exclusive scan of per-group arc counts).
__global__ void k_gscan(const uint32_t* __restrict__ garc, int G, unsigned long long* gcur) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  uint64_t carry = 0;
  for (int base = 0; base < G; base += B) {
    const int g = base + threadIdx.x;
    const uint32_t x = g < G ? garc[g] : 0u;
    uint32_t tot;
    const uint32_t e = block_excl_scan<B>(x, s_scan, &tot);
    if (g < G) gcur[gslot(g, G)] = carry + e;
    carry += tot;
  }
}

// CSR bucket pass: every arc (r = target, p = source) of Alg. 1 line 3 goes to the group
// of r (2^gshift consecutive vertices), written as (r,p) pairs; each block reserves one
// contiguous run per group, so the writes stay coalesced and the second pass below scatters
// inside one small window of P at a time (L2-resident, no partial-sector DRAM writes).
constexpr int BITEMS = 8;
constexpr int MAXG = 2048;
// DIRECTED: the input is already arcs (r, p) (multi-GPU: arcs received by their owner),
// one tuple each; otherwise undirected edges, two tuples each.
template <bool DIRECTED>
__global__ void __launch_bounds__(B, 4) k_bucket(const uint2* __restrict__ e, uint64_t m, int gshift,
                                              int G, unsigned long long* gcur,
                                              uint2* __restrict__ out) {
  constexpr int PER = DIRECTED ? 1 : 2;
  __shared__ uint32_t s_cnt[MAXG];
  __shared__ unsigned long long s_base[MAXG];
  for (int g = threadIdx.x; g < G; g += B) s_cnt[g] = 0;
  __syncthreads();
  const uint64_t e0 = (blockIdx.x * (uint64_t)B * BITEMS) + threadIdx.x;
  uint2 arc[PER * BITEMS];
  uint32_t slot[PER * BITEMS];
  // every load in flight before the first shared atomic: the atomics order memory, so loads
  // interleaved with them were issued one at a time (C4 mode sv: IPC 0.21, 32 ms)
  uint2 ld[BITEMS];
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    ld[k] = i < m ? e[i] : make_uint2(0, 0);
  }
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    if (i < m) {
      const uint2 xy = ld[k];
      if (DIRECTED) {
        arc[k] = xy;
        slot[k] = atomicAdd(&s_cnt[xy.x >> gshift], 1u);
      } else {
        arc[PER * k] = make_uint2(xy.y, xy.x);      // <x,_,y>: r = y, p = x
        arc[PER * k + PER - 1] = make_uint2(xy.x, xy.y);  // <y,_,x>: r = x, p = y
        slot[PER * k] = atomicAdd(&s_cnt[xy.y >> gshift], 1u);
        slot[PER * k + PER - 1] = atomicAdd(&s_cnt[xy.x >> gshift], 1u);
      }
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += B)
    s_base[g] = s_cnt[g] ? atomicAdd(&gcur[gslot(g, G)], (unsigned long long)s_cnt[g]) : 0ull;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    if (i < m) {
#pragma unroll
      for (int t = 0; t < PER; t++)
        out[s_base[arc[PER * k + t].x >> gshift] + slot[PER * k + t]] = arc[PER * k + t];
    }
  }
}

// The same pass with the block's arcs staged in shared memory in group order, for G <= 256
// groups (the large graphs): each group's run then leaves as consecutive 8-byte stores.
// Scattered from registers, a warp's 32 stores went to ~27 different sectors (each lane to
// another group's run), and on C4 in mode sv the pass was bound by 1.8 G partial-sector
// writes into L2 (32 ms for 26 GB of DRAM traffic).
constexpr int GST = 256;
template <bool DIRECTED>
__global__ void __launch_bounds__(B) k_bucket_st(const uint2* __restrict__ e, uint64_t m, int gshift, int G,
                                                 unsigned long long* gcur, uint2* __restrict__ out) {
  constexpr int PER = DIRECTED ? 1 : 2;
  static_assert(B == GST, "one thread per group counter in the scan");
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint32_t s_cnt[GST], s_off[GST];
  __shared__ unsigned long long s_base[GST];
  __shared__ uint2 s_arc[B * BITEMS * PER];
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t e0 = (blockIdx.x * (uint64_t)B * BITEMS) + threadIdx.x;
  uint2 ld[BITEMS];
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    ld[k] = i < m ? e[i] : make_uint2(0, 0);
  }
  uint2 arc[PER * BITEMS];
  uint32_t slot[PER * BITEMS];
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    if (i < m) {
      const uint2 xy = ld[k];
      if (DIRECTED) {
        arc[k] = xy;
        slot[k] = atomicAdd(&s_cnt[xy.x >> gshift], 1u);
      } else {
        arc[PER * k] = make_uint2(xy.y, xy.x);            // <x,_,y>: r = y, p = x
        arc[PER * k + PER - 1] = make_uint2(xy.x, xy.y);  // <y,_,x>: r = x, p = y
        slot[PER * k] = atomicAdd(&s_cnt[xy.y >> gshift], 1u);
        slot[PER * k + PER - 1] = atomicAdd(&s_cnt[xy.x >> gshift], 1u);
      }
    }
  }
  __syncthreads();
  const uint32_t c = threadIdx.x < (uint32_t)G ? s_cnt[threadIdx.x] : 0u;
  uint32_t tot;
  s_off[threadIdx.x] = block_excl_scan<B>(c, s_scan, &tot);
  if (c) s_base[threadIdx.x] = atomicAdd(&gcur[gslot(threadIdx.x, G)], (unsigned long long)c);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    if (i < m) {
#pragma unroll
      for (int t = 0; t < PER; t++) {
        const uint2 a = arc[PER * k + t];
        s_arc[s_off[a.x >> gshift] + slot[PER * k + t]] = a;
      }
    }
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < tot; q += B) {
    const uint2 a = s_arc[q];
    const uint32_t g = a.x >> gshift;
    out[s_base[g] + (q - s_off[g])] = a;
  }
}
template <bool DIRECTED>
static void launch_bucket(const uint2* edges, uint64_t m, int gshift, int G, unsigned long long* gc, uint2* out,
                          cudaStream_t st) {
  if (!m) return;
  const unsigned gb = (unsigned)((m + B * BITEMS - 1) / (B * BITEMS));
  if (G <= GST) k_bucket_st<DIRECTED><<<gb, B, 0, st>>>(edges, m, gshift, G, gc, out);
  else k_bucket<DIRECTED><<<gb, B, 0, st>>>(edges, m, gshift, G, gc, out);
}

// ---- degrees without global atomics (prediction of the csr engine, n <= 2^26)
// Alg. 2 line 2 counts arcs per source (sort + run lengths in the paper).  Here the
// arcs are first bucketed by the vertex group of r (the CSR bucket pass above, which the
// build needs anyway); a group is 2^gshift <= 2^15 vertices, so one block counts its arcs
// in shared memory.
__global__ void __launch_bounds__(B) k_group_hist(const uint2* __restrict__ e, uint64_t m, int gshift,
                                                  int G, uint32_t* garc) {
  __shared__ uint32_t s[MAXG];
  for (int g = threadIdx.x; g < G; g += B) s[g] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < m; i += (uint64_t)gridDim.x * B) {
    const uint2 xy = e[i];
    atomicAdd(&s[xy.x >> gshift], 1u);
    atomicAdd(&s[xy.y >> gshift], 1u);
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += B)
    if (s[g]) atomicAdd(&garc[g], s[g]);
}
__global__ void __launch_bounds__(1024) k_group_degree(const uint2* __restrict__ arcs,
                                                       const unsigned long long* __restrict__ gend,
                                                       int gshift, uint64_t n, uint32_t* deg) {
  extern __shared__ uint32_t s_deg[];
  const uint64_t g = blockIdx.x, base = g << gshift;
  const uint32_t cnt = (uint32_t)min((uint64_t)1 << gshift, n - base);
  for (uint32_t v = threadIdx.x; v < cnt; v += blockDim.x) s_deg[v] = 0;
  __syncthreads();
  const uint64_t a = g ? gend[gslot((int)g - 1, (int)gridDim.x)] : 0, b = gend[gslot((int)g, (int)gridDim.x)];
  const uint32_t lt = lanemask_lt();
  for (uint64_t i0 = a; i0 < b; i0 += blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const uint32_t v = i < b ? (uint32_t)(arcs[i].x - base) : 0xFFFFFFFFu;
    // hubs: lanes holding the same vertex add once (__match_any_sync)
    const uint32_t peers = __match_any_sync(0xffffffffu, v);
    if (v != 0xFFFFFFFFu && (peers & lt) == 0) atomicAdd(&s_deg[v], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (uint32_t v = threadIdx.x; v < cnt; v += blockDim.x) deg[base + v] = s_deg[v];
}

// ---- row placement without global cursor atomics (default path).  The arcs bucketed by
// group (k_bucket) are re-bucketed by subgroup of 2^SUBG ids into a P-aligned scratch array
// (subgroup s's arcs land in [off[v0], ...), inside the P range its rows will occupy), then
// one block per subgroup places its arcs with shared-memory row cursors and writes R and the
// vertex tuples of its rows: every global write stays inside the subgroup's own P window.
// 2^11 ids: smaller subgroups (2^7, so that a C4 subgroup's 4 k tuples would stage in
// k_place) spread a k_bucket2 tile over more subgroups than its counters hold, and the
// pass fell back to global cursor atomics (C4 in mode sv: k_bucket2 12 -> 115 ms).
constexpr int SUBG = 11;
constexpr int MAXS2 = 512;
__global__ void k_sub_init(const uint32_t* __restrict__ off, uint64_t ns, uint32_t* __restrict__ scur) {
  for (uint64_t s = blockIdx.x * (uint64_t)B + threadIdx.x; s < ns; s += (uint64_t)gridDim.x * B)
    scur[s] = off[s << SUBG];
}
__global__ void __launch_bounds__(B) k_bucket2(const uint2* __restrict__ in, uint64_t na,
                                               uint32_t* scur, uint2* __restrict__ out) {
  __shared__ uint32_t s_cnt[MAXS2];
  __shared__ uint32_t s_base[MAXS2];
  __shared__ uint32_t s_off[MAXS2];
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint2 s_arc[B * BITEMS];
  __shared__ uint32_t s_lo, s_hi;
  if (threadIdx.x == 0) {
    s_lo = 0xFFFFFFFFu;
    s_hi = 0;
  }
  for (int i = threadIdx.x; i < MAXS2; i += B) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t e0 = blockIdx.x * (uint64_t)B * BITEMS + threadIdx.x;
  uint2 arc[BITEMS];
  uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    arc[k] = i < na ? in[i] : make_uint2(0xFFFFFFFFu, 0);
    if (i < na) {
      lo = min(lo, arc[k].x >> SUBG);
      hi = max(hi, arc[k].x >> SUBG);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_lo, lo);
    atomicMax(&s_hi, hi);
  }
  __syncthreads();
  const uint32_t slo = s_lo;
  const bool local = s_hi - slo < (uint32_t)MAXS2;  // the tile's subgroups fit the counters
  uint32_t slot[BITEMS];
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    if (arc[k].x == 0xFFFFFFFFu) continue;
    const uint32_t sg = arc[k].x >> SUBG;
    slot[k] = local ? atomicAdd(&s_cnt[sg - slo], 1u) : atomicAdd(&scur[sg], 1u);
  }
  if (local && s_hi - slo < 128) {
    // few subgroups in the tile (>= 16 arcs per subgroup on average): staged in subgroup
    // order, then written as runs (scattered from registers, a warp's 32 stores touched ~31
    // sectors); with more subgroups the runs are too short to pay for the staging
    __syncthreads();
    static_assert(MAXS2 == 2 * B, "two counters per thread in the scan");
    const uint32_t c0 = s_cnt[2 * threadIdx.x], c1 = s_cnt[2 * threadIdx.x + 1];
    uint32_t tot;
    const uint32_t o = block_excl_scan<B>(c0 + c1, s_scan, &tot);
    s_off[2 * threadIdx.x] = o;
    s_off[2 * threadIdx.x + 1] = o + c0;
    if (c0) s_base[2 * threadIdx.x] = atomicAdd(&scur[slo + 2 * threadIdx.x], c0);
    if (c1) s_base[2 * threadIdx.x + 1] = atomicAdd(&scur[slo + 2 * threadIdx.x + 1], c1);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BITEMS; k++)
      if (arc[k].x != 0xFFFFFFFFu) s_arc[s_off[(arc[k].x >> SUBG) - slo] + slot[k]] = arc[k];
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < tot; q += B) {
      const uint2 a = s_arc[q];
      const uint32_t l = (a.x >> SUBG) - slo;
      out[s_base[l] + (q - s_off[l])] = a;
    }
    return;
  }
  if (local) {
    __syncthreads();
    for (int l = threadIdx.x; l < MAXS2; l += B)
      s_base[l] = s_cnt[l] ? atomicAdd(&scur[slo + l], s_cnt[l]) : 0u;
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    if (arc[k].x == 0xFFFFFFFFu) continue;
    const uint32_t pos = local ? s_base[(arc[k].x >> SUBG) - slo] + slot[k] : slot[k];
    out[pos] = arc[k];
  }
}
constexpr int PLACE_LONG_CAP = 64;
constexpr int PLACE_CAP = 7168;  // tuples of a subgroup assembled in shared memory
constexpr size_t PLACE_SMEM = sizeof(uint32_t) * (2 * ((1 << SUBG) + 1) + 2 * PLACE_CAP);
__global__ void __launch_bounds__(B) k_place(const uint32_t* __restrict__ off, uint64_t n,
                                             const uint32_t* __restrict__ scur_end,
                                             const uint2* __restrict__ arcs, uint32_t* __restrict__ R,
                                             uint32_t* __restrict__ P) {
  extern __shared__ uint32_t smem[];
  uint32_t* s_off = smem;                          // row starts relative to the subgroup
  uint32_t* s_cur = s_off + (1 << SUBG) + 1;       // next free slot of each row
  uint32_t* s_p = s_cur + (1 << SUBG) + 1;         // the subgroup's P, assembled
  uint32_t* s_r = s_p + PLACE_CAP;                 // and its R
  __shared__ uint32_t s_long[PLACE_LONG_CAP];
  __shared__ uint32_t s_nlong;
  const uint64_t s = blockIdx.x, v0 = s << SUBG;
  const uint32_t cnt = (uint32_t)min((uint64_t)1 << SUBG, n - v0);
  const uint32_t base0 = off[v0], T = off[v0 + cnt] - base0;
  if (T == 0) return;  // no rows here (e.g. the small remainder after a BFS peel)
  const bool staged = T <= (uint32_t)PLACE_CAP;  // else rows are written in place
  if (threadIdx.x == 0) s_nlong = 0;
  for (uint32_t l = threadIdx.x; l <= cnt; l += B) s_off[l] = off[v0 + l] - base0;
  __syncthreads();
  // rows: vertex tuple <v,_,v> first, R over the row; cursors after it
  for (uint32_t l = threadIdx.x; l < cnt; l += B) {
    const uint32_t a = s_off[l], b = s_off[l + 1];
    s_cur[l] = a + 1;
    if (a == b) continue;
    const uint32_t v = (uint32_t)(v0 + l);
    if (staged) {
      s_p[a] = v;
      for (uint32_t i = a; i < b; i++) s_r[i] = v;  // staged rows are short (T <= PLACE_CAP)
      if (b - a > LONG)
        for (uint32_t i = a; i < b; i++) s_r[i] = v | R_LONG;
    } else {
      P[base0 + a] = v;
      if (b - a <= LONG_ROW) {
        // R of short rows: written below by a warp per row (coalesced runs)
      } else {
        const uint32_t j = atomicAdd(&s_nlong, 1u);
        if (j < PLACE_LONG_CAP) {
          s_long[j] = l;
        } else {
          const uint32_t rv = v | (b - a > LONG ? R_LONG : 0u);
          for (uint32_t i = a; i < b; i++) R[base0 + i] = rv;
        }
      }
    }
  }
  __syncthreads();
  if (!staged) {  // R of the short rows, a warp per row: one store request per 32 tuples
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t l = threadIdx.x >> 5; l < cnt; l += B / 32) {
      const uint32_t a = s_off[l], b = s_off[l + 1];
      if (b - a > LONG_ROW) continue;
      for (uint32_t i = a + lane; i < b; i += 32) R[base0 + i] = (uint32_t)(v0 + l);
    }
  }
  // arcs of the subgroup: shared-memory row cursors
  const uint32_t a1 = scur_end[s];
  constexpr int PI = 8;  // arcs per thread in flight
  for (uint32_t i0 = base0; i0 < a1; i0 += B * PI) {
    uint2 rp[PI];
#pragma unroll
    for (int k = 0; k < PI; k++) {
      const uint32_t i = i0 + k * B + threadIdx.x;
      rp[k] = i < a1 ? arcs[i] : make_uint2(0xFFFFFFFFu, 0);
    }
#pragma unroll
    for (int k = 0; k < PI; k++) {
      if (rp[k].x == 0xFFFFFFFFu) continue;
      // shared-memory cursor: native atomics, same-row lanes serialise only among themselves
      const uint32_t slot = atomicAdd(&s_cur[rp[k].x - v0], 1u);
      if (staged) s_p[slot] = rp[k].y;
      else P[base0 + slot] = rp[k].y;
    }
  }
  if (staged) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T; i += B) {  // contiguous runs out
      P[base0 + i] = s_p[i];
      R[base0 + i] = s_r[i];
    }
  } else {
    const uint32_t nl = min(s_nlong, (uint32_t)PLACE_LONG_CAP);
    for (uint32_t j = 0; j < nl; j++) {
      const uint32_t l = s_long[j];
      const uint32_t a = s_off[l], b = s_off[l + 1];
      const uint32_t rv = (uint32_t)(v0 + l) | (b - a > LONG ? R_LONG : 0u);  // long rows skipped by row passes
      for (uint32_t i = a + threadIdx.x; i < b; i += B) R[base0 + i] = rv;
    }
  }
}

// Second pass: place each arc tuple in its row (cursor per vertex).
// SITEMS arcs per thread per step: their cursor atomics are independent and in flight
// together (the returned slot is needed before the store, so one arc at a time would expose
// the full L2 atomic round trip per arc).
constexpr int XITEMS = 8;
__global__ void __launch_bounds__(B) k_scatter(const uint2* __restrict__ arcs, uint64_t na,
                                               uint32_t* cur, uint32_t* __restrict__ P) {
  const uint64_t stride = (uint64_t)gridDim.x * B * XITEMS;
  for (uint64_t i0 = blockIdx.x * (uint64_t)B * XITEMS + threadIdx.x; i0 < na; i0 += stride) {
    uint2 rp[XITEMS];
    uint32_t slot[XITEMS];
#pragma unroll
    for (int k = 0; k < XITEMS; k++) {
      const uint64_t i = i0 + (uint64_t)k * B;
      rp[k] = i < na ? arcs[i] : make_uint2(0xFFFFFFFFu, 0);
    }
#pragma unroll
    for (int k = 0; k < XITEMS; k++)
      if (rp[k].x != 0xFFFFFFFFu) slot[k] = atomicAdd(&cur[rp[k].x], 1u);
#pragma unroll
    for (int k = 0; k < XITEMS; k++)
      if (rp[k].x != 0xFFFFFFFFu) P[slot[k]] = rp[k].y;
  }
}

// ===================================================================== compaction
// Ordered stream compaction of the live tuples (P != DEAD): tile prefix by decoupled
// look-back keeps R sorted.  Run when dead rows exceed a fraction of the array.
constexpr int CITEMS = 8;
constexpr int CTILE = B * CITEMS;
__global__ void __launch_bounds__(B) k_compact(const uint32_t* __restrict__ R,
                                               const uint32_t* __restrict__ P, uint64_t A,
                                               uint32_t* __restrict__ R2, uint32_t* __restrict__ P2,
                                               uint64_t* flags, uint32_t* ticket, uint32_t epoch) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_pref;
  __shared__ uint32_t s_r[CTILE], s_p[CTILE];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t i0 = tile * CTILE + (uint64_t)threadIdx.x * CITEMS;
  uint32_t r[CITEMS], p[CITEMS];
#pragma unroll
  for (int k = 0; k < CITEMS; k++) {
    r[k] = (i0 + k < A) ? R[i0 + k] : 0u;
    p[k] = (i0 + k < A) ? P[i0 + k] : DEAD;
  }
  uint32_t cnt = 0;
#pragma unroll
  for (int k = 0; k < CITEMS; k++) cnt += (p[k] != DEAD);
  uint32_t tot;
  const uint32_t excl = block_excl_scan<B>(cnt, s_scan, &tot);
  const uint64_t pref = scan::tile_prefix(flags, tile, tot, epoch, &s_pref);
  uint32_t o = excl;
#pragma unroll
  for (int k = 0; k < CITEMS; k++)
    if (p[k] != DEAD) { s_r[o] = r[k]; s_p[o] = p[k]; o++; }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tot; i += B) {
    R2[pref + i] = s_r[i];
    P2[pref + i] = s_p[i];
  }
}

// ===================================================================== row collapse
// Ordered compaction that also folds every collapsible row to its head tuple (csr.cuh
// collapse()).  A row is collapsible when it lies inside this tile (it neither continues from
// the previous tile nor into the next), is not a long row (k_long1/k_long2 own those, and
// their segment list is built from the degrees) and all its p are equal (PC).  Dead rows
// (completed partitions) leave whole, as in k_compact.
__global__ void __launch_bounds__(B) k_collapse(const uint32_t* __restrict__ R,
                                                const uint32_t* __restrict__ P, uint64_t A,
                                                uint32_t* __restrict__ R2, uint32_t* __restrict__ P2,
                                                uint32_t* __restrict__ HW, unsigned long long* hidden,
                                                unsigned long long* out_len, uint64_t ntiles,
                                                uint64_t* flags, uint32_t* ticket, uint32_t epoch) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_pref;
  __shared__ __align__(16) uint32_t s_r[CTILE];
  __shared__ __align__(16) uint32_t s_p[CTILE];
  __shared__ __align__(16) uint32_t s_bad[CTILE];  // per row head (local index)
  __shared__ __align__(16) uint32_t s_cnt[CTILE];
  __shared__ uint32_t s_wmax[B / 32];
  __shared__ unsigned long long s_hid;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(ticket, 1u);
    s_hid = 0;
  }
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t t0 = tile * CTILE;
  const uint32_t x0 = threadIdx.x * CITEMS;
  const uint32_t rbefore = t0 > 0 ? R[t0 - 1] : 0xFFFFFFFFu;           // uniform loads
  const uint32_t rafter = t0 + CTILE < A ? R[t0 + CTILE] : 0xFFFFFFFFu;
  uint32_t r[CITEMS], p[CITEMS];
  static_assert(CITEMS == 8, "two 16-byte vectors per thread");
  if (t0 + x0 + CITEMS <= A) {  // arrays are 16-byte aligned at tile offsets (CTILE * 4 bytes)
    const uint4 a = ldg_stream(reinterpret_cast<const uint4*>(R + t0 + x0));
    const uint4 b = ldg_stream(reinterpret_cast<const uint4*>(R + t0 + x0) + 1);
    const uint4 c = ldg_stream(reinterpret_cast<const uint4*>(P + t0 + x0));
    const uint4 d = ldg_stream(reinterpret_cast<const uint4*>(P + t0 + x0) + 1);
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    p[0] = c.x; p[1] = c.y; p[2] = c.z; p[3] = c.w; p[4] = d.x; p[5] = d.y; p[6] = d.z; p[7] = d.w;
  } else {
#pragma unroll
    for (int k = 0; k < CITEMS; k++) {
      const uint64_t i = t0 + x0 + k;
      r[k] = i < A ? R[i] : 0xFFFFFFFEu;  // past the end: a key no row has
      p[k] = i < A ? P[i] : DEAD;
    }
  }
  reinterpret_cast<uint4*>(s_r + x0)[0] = make_uint4(r[0], r[1], r[2], r[3]);
  reinterpret_cast<uint4*>(s_r + x0)[1] = make_uint4(r[4], r[5], r[6], r[7]);
  reinterpret_cast<uint4*>(s_p + x0)[0] = make_uint4(p[0], p[1], p[2], p[3]);
  reinterpret_cast<uint4*>(s_p + x0)[1] = make_uint4(p[4], p[5], p[6], p[7]);
  reinterpret_cast<uint4*>(s_bad + x0)[0] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(s_bad + x0)[1] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(s_cnt + x0)[0] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(s_cnt + x0)[1] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // head position (+1) of the row holding each item: block-wide inclusive max scan of the
  // heads (0 = the row started in the previous tile)
  uint32_t hh[CITEMS];
  uint32_t run = 0;
#pragma unroll
  for (int k = 0; k < CITEMS; k++) {
    const uint32_t x = x0 + k;
    const uint32_t rp = x ? s_r[x - 1] : rbefore;
    if (rp != r[k]) run = x + 1;
    hh[k] = run;
  }
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t v = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = max(v, y);
    }
    if (lane == 31) s_wmax[wid] = v;
    __syncthreads();
    uint32_t carry = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) carry = 0;
    for (int w = 0; w < wid; w++) carry = max(carry, s_wmax[w]);
#pragma unroll
    for (int k = 0; k < CITEMS; k++) {
      if (hh[k]) break;  // items before the thread's first head take the carry
      hh[k] = carry;
    }
  }
  // a row is not collapsible if it is long, has two different p, or reaches the next tile
#pragma unroll
  for (int k = 0; k < CITEMS; k++) {
    const uint32_t x = x0 + k;
    if (!hh[k] || p[k] == DEAD) continue;
    const uint32_t h = hh[k] - 1;
    bool bad = (r[k] & R_LONG) != 0;
    if (x != h && s_p[x - 1] != p[k]) bad = true;
    if (x == CTILE - 1 && rafter == r[k]) bad = true;
    if (bad) s_bad[h] = 1;
  }
  __syncthreads();
  uint32_t keep = 0, cnt = 0;
#pragma unroll
  for (int k = 0; k < CITEMS; k++) {
    const uint32_t x = x0 + k;
    bool kp = p[k] != DEAD;
    if (kp && hh[k] && x != hh[k] - 1 && !s_bad[hh[k] - 1]) {
      kp = false;
      atomicAdd(&s_cnt[hh[k] - 1], 1u);
    }
    keep |= (uint32_t)kp << k;
    cnt += kp;
  }
  __syncthreads();
  // heads of collapsed rows record the folded tuples (a row lies in one tile: plain add)
  unsigned long long hid = 0;
#pragma unroll
  for (int k = 0; k < CITEMS; k++) {
    const uint32_t x = x0 + k;
    if (hh[k] == x + 1 && s_cnt[x]) {
      atomicAdd(&HW[r[k]], s_cnt[x]);  // result unused: a fire-and-forget reduction, no dependent load
      hid += s_cnt[x];
    }
  }
  hid = warp_sum(hid);
  if ((threadIdx.x & 31) == 0 && hid) atomicAdd(&s_hid, hid);
  uint32_t tot;
  const uint32_t excl = block_excl_scan<B>(cnt, s_scan, &tot);
  const uint64_t pref = scan::tile_prefix(flags, tile, tot, epoch, &s_pref);
  uint32_t o = excl;
#pragma unroll
  for (int k = 0; k < CITEMS; k++)
    if ((keep >> k) & 1u) { s_r[o] = r[k]; s_p[o] = p[k]; o++; }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tot; i += B) {
    R2[pref + i] = s_r[i];
    P2[pref + i] = s_p[i];
  }
  if (threadIdx.x == 0) {
    if (s_hid) atomicAdd(hidden, s_hid);
    if (tile == ntiles - 1) *out_len = pref + tot;
  }
}

// ===================================================================== launchers
int group_shift(uint64_t n, uint64_t tuples) {
  int kb = 0;
  while ((1ull << kb) < n) kb++;
  int lg = 0;  // log2 G: about 256 k tuples per group (up to 256 groups, below)
  while (lg < 10 && (tuples >> (18 + lg)) > 0) lg++;
  int gs = kb - lg;
  // at most 256 groups while a group can stay within 2^18 ids: k_bucket gives every group one
  // run per 2048-edge tile (16 arcs at 256 groups, staged in shared memory: k_bucket_st;
  // with 1024 groups those runs were 4 arcs, one sector), and 2^18 ids are 128 subgroups, so
  // a k_bucket2 tile's subgroups fit its local counters and its runs are long enough to stage
  const int gs_min = std::min(18, kb - 8);
  if (gs < gs_min) gs = gs_min;
  return gs < 12 ? 12 : gs;  // a k_rows tile (2^12 vertices) lies inside one group
}

int group_shift_full(uint64_t n) {
  int kb = 0;
  while ((1ull << kb) < n) kb++;
  if (kb > 26) return -1;  // more than MAXG groups of 2^15 ids: use graph::launch_degree
  return kb - 11 < 12 ? 12 : kb - 11;
}

void build(const uint2* edges, uint64_t m, const uint32_t* deg, const uint32_t* vis, uint64_t n,
           uint32_t* off, uint32_t* cur, uint32_t* garc, int gshift, scan::State& ss, uint64_t* ctr,
           cudaStream_t st, bool count_groups) {
  // ctr[C_VT_OUT] receives A_0
  if (!n) return;
  const int G = (int)(((n - 1) >> gshift) + 1);
  cudaMemsetAsync(ss.ticket, 0, sizeof(uint32_t), st);
  if (count_groups) cudaMemsetAsync(garc, 0, sizeof(uint32_t) * G, st);
  const uint64_t tiles = (n + B * SITEMS - 1) / (B * SITEMS);
  k_rows<<<(unsigned)tiles, B, 0, st>>>(deg, vis, n, off, cur, ss.flags, ss.ticket, ++ss.epoch,
                                         reinterpret_cast<unsigned long long*>(ctr + sv::C_VT_OUT),
                                         garc, gshift, count_groups ? 1 : 0);
}

void bucket_degrees(const uint2* edges, uint64_t m, uint64_t n, int gshift, uint32_t* garc,
                    uint64_t* gcur, uint2* tmp, uint32_t* deg, cudaStream_t st) {
  if (!n) return;
  const int G = (int)(((n - 1) >> gshift) + 1);
  auto* gc = reinterpret_cast<unsigned long long*>(gcur);
  cudaMemsetAsync(garc, 0, sizeof(uint32_t) * G, st);
  if (m) k_group_hist<<<grid(m, B, 148 * 4), B, 0, st>>>(edges, m, gshift, G, garc);
  k_gscan<<<1, B, 0, st>>>(garc, G, gc);
  launch_bucket<false>(edges, m, gshift, G, gc, tmp, st);
  // k_bucket advanced every group cursor to its group's end
  const int smem = (int)(sizeof(uint32_t) << gshift);
  static int attr_set = 0;
  if (!attr_set) {
    cudaFuncSetAttribute(k_group_degree, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << 15);
    attr_set = 1;
  }
  k_group_degree<<<G, 1024, smem, st>>>(tmp, gc, gshift, n, deg);
}

void fill_from_buckets(const uint32_t* off, uint32_t* cur, uint64_t n, uint64_t A, uint32_t* R,
                       uint32_t* P, const uint2* tmp, uint64_t na, uint32_t* longlist, uint64_t* nlong,
                       cudaStream_t st) {
  if (!A) return;
  auto* nl = reinterpret_cast<unsigned long long*>(nlong);
  cudaMemsetAsync(nlong, 0, sizeof(uint64_t), st);
  k_fill_rows<<<grid(n, B, 148 * 8), B, 0, st>>>(off, n, R, P, longlist, nl);
  k_fill_long<<<148 * 2, B, 0, st>>>(off, longlist, nl, R);
  if (na) k_scatter<<<grid((na + XITEMS - 1) / XITEMS, B, 148 * 8), B, 0, st>>>(tmp, na, cur, P);
}
void fill(const uint2* edges, uint64_t m, const uint32_t* off, uint32_t* cur, uint64_t n, uint64_t A,
          uint32_t* R, uint32_t* P, const uint32_t* garc, int gshift, uint64_t* gcur, uint2* tmp,
          uint32_t* longlist, uint64_t* nlong, cudaStream_t st, bool directed) {
  if (!A) return;
  const int G = (int)(((n - 1) >> gshift) + 1);
  if (m && P > R && (uint64_t)(P - R) * 2 >= (directed ? 2 * m : 4 * m) && gshift >= SUBG) {
    // default: the group buckets go into R's buffer (R and P are the two halves of one
    // 8-byte-per-tuple allocation, free until placement), the P-aligned subgroup buckets
    // into tmp, then k_place writes R and P
    auto* gc = reinterpret_cast<unsigned long long*>(gcur);
    uint2* tmp1 = reinterpret_cast<uint2*>(R);
    k_gscan<<<1, B, 0, st>>>(garc, G, gc);
    if (directed) launch_bucket<true>(edges, m, gshift, G, gc, tmp1, st);
    else launch_bucket<false>(edges, m, gshift, G, gc, tmp1, st);
    const uint64_t na = directed ? m : 2 * m;
    const uint64_t ns = ((n - 1) >> SUBG) + 1;
    uint32_t* scur = longlist;  // n-sized scratch, ns entries used
    k_sub_init<<<grid(ns, B, 148 * 4), B, 0, st>>>(off, ns, scur);
    k_bucket2<<<(unsigned)((na + B * BITEMS - 1) / (B * BITEMS)), B, 0, st>>>(tmp1, na, scur, tmp);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLACE_SMEM);
      attr = true;
    }
    k_place<<<(unsigned)ns, B, PLACE_SMEM, st>>>(off, n, scur, tmp, R, P);
    return;
  }
  auto* nl = reinterpret_cast<unsigned long long*>(nlong);
  cudaMemsetAsync(nlong, 0, sizeof(uint64_t), st);
  k_fill_rows<<<grid(n, B, 148 * 8), B, 0, st>>>(off, n, R, P, longlist, nl);
  k_fill_long<<<148 * 2, B, 0, st>>>(off, longlist, nl, R);
  if (!m) return;
  auto* gc = reinterpret_cast<unsigned long long*>(gcur);
  k_gscan<<<1, B, 0, st>>>(garc, G, gc);
  if (directed) launch_bucket<true>(edges, m, gshift, G, gc, tmp, st);
  else launch_bucket<false>(edges, m, gshift, G, gc, tmp, st);
  const uint64_t na = directed ? m : 2 * m;
  k_scatter<<<grid((na + XITEMS - 1) / XITEMS, B, 148 * 8), B, 0, st>>>(tmp, na, cur, P);
}
void collapse(const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* R2, uint32_t* P2, uint32_t* HW,
              uint64_t* hidden, uint64_t* out_len, scan::State& ss, cudaStream_t st) {
  cudaMemsetAsync(out_len, 0, sizeof(uint64_t), st);
  if (!A) return;
  cudaMemsetAsync(ss.ticket, 0, sizeof(uint32_t), st);
  const uint64_t tiles = (A + CTILE - 1) / CTILE;
  k_collapse<<<(unsigned)tiles, B, 0, st>>>(R, P, A, R2, P2, HW, reinterpret_cast<unsigned long long*>(hidden),
                                            reinterpret_cast<unsigned long long*>(out_len), tiles, ss.flags,
                                            ss.ticket, ++ss.epoch);
}
void compact(const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* R2, uint32_t* P2,
             scan::State& ss, cudaStream_t st) {
  if (!A) return;
  cudaMemsetAsync(ss.ticket, 0, sizeof(uint32_t), st);
  const uint64_t tiles = (A + CTILE - 1) / CTILE;
  k_compact<<<(unsigned)tiles, B, 0, st>>>(R, P, A, R2, P2, ss.flags, ss.ticket, ++ss.epoch);
}

}  // namespace csr
}  // namespace cc
