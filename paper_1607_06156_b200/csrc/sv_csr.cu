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
constexpr uint32_t INF = 0xFFFFFFFFu;

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
constexpr int SITEMS = 8;
__global__ void __launch_bounds__(B) k_rows(const uint32_t* __restrict__ deg,
                                            const uint32_t* __restrict__ vis, uint64_t n,
                                            uint32_t* __restrict__ off, uint32_t* __restrict__ cur,
                                            uint64_t* flags, uint32_t* ticket, uint32_t epoch,
                                            unsigned long long* total, uint32_t* garc,
                                            int gshift) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_pref;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t v0 = tile * (B * SITEMS) + (uint64_t)threadIdx.x * SITEMS;
  uint32_t c[SITEMS];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    const uint64_t v = v0 + k;
    uint32_t x = 0;
    if (v < n) {
      x = deg[v];
      if (x && vis && ((vis[v >> 5] >> (v & 31)) & 1u)) x = 0;
      if (x) x += 1;
    }
    c[k] = x;
    sum += x;
  }
  uint32_t tot;
  const uint32_t excl = block_excl_scan<B>(sum, s_scan, &tot);
  const uint64_t pref = scan::tile_prefix(flags, tile, tot, epoch, &s_pref);
  // arcs of this tile (tuples minus vertex tuples) for the CSR bucket pass; a tile of
  // B*SITEMS = 2^11 vertices lies inside one group of 2^gshift vertices (gshift >= 11)
  {
    uint32_t nv = 0;
#pragma unroll
    for (int k = 0; k < SITEMS; k++) nv += (c[k] != 0);
    nv = warp_sum(nv);
    if ((threadIdx.x & 31) == 0 && nv) atomicSub(&garc[(tile * (B * SITEMS)) >> gshift], nv);
    if (threadIdx.x == 0 && tot) atomicAdd(&garc[(tile * (B * SITEMS)) >> gshift], tot);
  }
  uint32_t run = (uint32_t)pref + excl;
#pragma unroll
  for (int k = 0; k < SITEMS; k++) {
    const uint64_t v = v0 + k;
    if (v < n) {
      off[v] = run;
      cur[v] = run + 1;
    }
    run += c[k];
  }
  if (n > 0 && v0 <= n - 1 && n - 1 < v0 + SITEMS) {  // owner of the last vertex
    off[n] = run;
    *total = run;
  }
}

// R and the vertex tuple <v,_,v> of each row: thread per vertex; rows longer than
// LONG_ROW (hubs) are appended to a list and filled by whole blocks.
constexpr uint32_t LONG_ROW = 64;
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
    for (uint32_t i = a + threadIdx.x; i < b; i += B) R[i] = v;
  }
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
    if (g < G) gcur[g] = carry + e;
    carry += tot;
  }
}

// CSR bucket pass: every arc (r = target, p = source) of Alg. 1 line 3 goes to the group
// of r (2^gshift consecutive vertices), written as (r,p) pairs; each block reserves one
// contiguous run per group, so the writes stay coalesced and the second pass below scatters
// inside one small window of P at a time (L2-resident, no partial-sector DRAM writes).
constexpr int BITEMS = 8;
constexpr int MAXG = 1024;
__global__ void __launch_bounds__(B) k_bucket(const uint2* __restrict__ e, uint64_t m, int gshift,
                                              int G, unsigned long long* gcur,
                                              uint2* __restrict__ out) {
  __shared__ uint32_t s_cnt[MAXG];
  __shared__ unsigned long long s_base[MAXG];
  for (int g = threadIdx.x; g < G; g += B) s_cnt[g] = 0;
  __syncthreads();
  const uint64_t e0 = (blockIdx.x * (uint64_t)B * BITEMS) + threadIdx.x;
  uint2 arc[2 * BITEMS];
  uint32_t slot[2 * BITEMS];
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    if (i < m) {
      const uint2 xy = e[i];
      arc[2 * k] = make_uint2(xy.y, xy.x);      // <x,_,y>: r = y, p = x
      arc[2 * k + 1] = make_uint2(xy.x, xy.y);  // <y,_,x>: r = x, p = y
      slot[2 * k] = atomicAdd(&s_cnt[xy.y >> gshift], 1u);
      slot[2 * k + 1] = atomicAdd(&s_cnt[xy.x >> gshift], 1u);
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += B)
    s_base[g] = s_cnt[g] ? atomicAdd(&gcur[g], (unsigned long long)s_cnt[g]) : 0ull;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < BITEMS; k++) {
    const uint64_t i = e0 + (uint64_t)k * B;
    if (i < m) {
      out[s_base[arc[2 * k].x >> gshift] + slot[2 * k]] = arc[2 * k];
      out[s_base[arc[2 * k + 1].x >> gshift] + slot[2 * k + 1]] = arc[2 * k + 1];
    }
  }
}

// Second pass: place each arc tuple in its row (cursor per vertex).
__global__ void __launch_bounds__(B) k_scatter(const uint2* __restrict__ arcs, uint64_t na,
                                               uint32_t* cur, uint32_t* __restrict__ P) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < na; i += (uint64_t)gridDim.x * B) {
    const uint2 rp = arcs[i];
    P[atomicAdd(&cur[rp.x], 1u)] = rp.y;
  }
}

// ===================================================================== vertex passes
// Lines 9-13 (WITH_PC) / line 24: per vertex bucket VB(u) (a run of equal R), u_min = min p
// and, for PC, whether max p != min p (|M(u)| > 1).  A warp streams its chunk
// in 128-tuple windows (one 16-byte load of R and of P per lane, next window prefetched),
// stages the window in shared memory, and every run head walks its run inside the window;
// the run touching the window end is carried into the next window, so a bucket costs one
// atomic per 128-tuple window it spans at most.  Tuples of completed partitions are dead
// (P = DEAD, whole rows) and are skipped.
constexpr uint32_t DEAD = 0xFFFFFFFFu;
constexpr int VWIN = 128;
constexpr int VWINS = 16;  // windows per warp chunk
constexpr int VCHUNK = VWIN * VWINS;
CC_DEVI void load_window(const uint32_t* R, const uint32_t* P, uint64_t A, uint64_t base, int lane,
                         uint4& r4, uint4& p4) {
  const uint64_t i = base + 4 * (uint64_t)lane;
  if (i + 3 < A) {
    r4 = ldg_stream(reinterpret_cast<const uint4*>(R + i));
    p4 = ldg_stream(reinterpret_cast<const uint4*>(P + i));
  } else {
    r4 = make_uint4(INF, INF, INF, INF);
    p4 = make_uint4(DEAD, DEAD, DEAD, DEAD);
    if (i < A) { r4.x = R[i]; p4.x = P[i]; }
    if (i + 1 < A) { r4.y = R[i + 1]; p4.y = P[i + 1]; }
    if (i + 2 < A) { r4.z = R[i + 2]; p4.z = P[i + 2]; }
  }
}
template <bool WITH_PC>
__global__ void __launch_bounds__(B) k_vpass(const uint32_t* __restrict__ R,
                                             const uint32_t* __restrict__ P, uint64_t A,
                                             uint32_t* __restrict__ U, uint32_t* __restrict__ NP) {
  __shared__ __align__(16) uint32_t s_k[B / 32][VWIN];
  __shared__ __align__(16) uint32_t s_v[B / 32][VWIN];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t warp = (blockIdx.x * (uint64_t)B + threadIdx.x) >> 5;
  const uint64_t cbase = warp * VCHUNK;
  if (cbase >= A) return;
  uint32_t* sk = s_k[wid];
  uint32_t* sv = s_v[wid];
  auto emit = [&](uint32_t key, uint32_t mn, uint32_t mx) {
    atomicMin(&U[key], mn);
    if (WITH_PC && mn != mx) atomicOr(&NP[key >> 5], 1u << (key & 31));
  };
  uint32_t ckey = INF, cmin = INF, cmax = 0;  // carry (warp-uniform)
  uint4 r4, p4, nr4, np4;
  load_window(R, P, A, cbase, lane, r4, p4);
  for (int w = 0; w < VWINS; w++) {
    const uint64_t base = cbase + (uint64_t)w * VWIN;
    if (base >= A) break;
    if (w + 1 < VWINS && base + VWIN < A) load_window(R, P, A, base + VWIN, lane, nr4, np4);
    // dead tuples (completed partitions) and padding get key INF
    uint4 k4 = make_uint4(p4.x == DEAD ? INF : r4.x, p4.y == DEAD ? INF : r4.y,
                          p4.z == DEAD ? INF : r4.z, p4.w == DEAD ? INF : r4.w);
    reinterpret_cast<uint4*>(sk)[lane] = k4;
    reinterpret_cast<uint4*>(sv)[lane] = p4;
    __syncwarp();
    // the previous carry ends here unless window element 0 continues its run
    if (lane == 0 && ckey != INF && sk[0] != ckey) emit(ckey, cmin, cmax);
    bool tail = false;
    uint32_t tk = INF, tmn = INF, tmx = 0;
#pragma unroll
    for (int s2 = 0; s2 < 4; s2++) {
      const int e = lane + 32 * s2;
      const uint32_t k = sk[e];
      if (k == INF || (e > 0 && sk[e - 1] == k)) continue;  // not a run head
      uint32_t mn = sv[e], mx = mn;
      int j = e + 1;
      while (j < VWIN && sk[j] == k) {
        const uint32_t v = sv[j];
        mn = min(mn, v);
        mx = max(mx, v);
        j++;
      }
      if (e == 0 && k == ckey) { mn = min(mn, cmin); mx = max(mx, cmax); }
      if (j == VWIN) { tail = true; tk = k; tmn = mn; tmx = mx; }
      else emit(k, mn, mx);
    }
    const uint32_t tb = __ballot_sync(0xffffffffu, tail);
    if (tb) {
      const int src = __ffs(tb) - 1;
      ckey = __shfl_sync(0xffffffffu, tk, src);
      cmin = __shfl_sync(0xffffffffu, tmn, src);
      cmax = __shfl_sync(0xffffffffu, tmx, src);
    } else {
      ckey = INF; cmin = INF; cmax = 0;
    }
    __syncwarp();
    r4 = nr4;
    p4 = np4;
  }
  if (lane == 0 && ckey != INF) emit(ckey, cmin, cmax);
}

// ===================================================================== partition passes
// Line 15 (FIRST) / line 25: p_min = min over PB(p) of q = u_min(r) -> PMIN[p]; FIRST also
// marks PB(p) 'not completed' when a tuple's vertex is not potentially completed.
// Second pass: q includes the temporary <r,_,r> in VB(r) when TB(r).
// Each block keeps a small direct-mapped cache of slot values it has seen (key and value in
// one 64-bit word): slots only decrease, so q >= a cached value needs no global traffic.
// That keeps a partition shared by millions of tuples (the giant component late in the
// run) from serialising one L2 slice, while distinct partitions go straight to the atomic.
constexpr int PCACHE = 1024;
template <bool FIRST>
__global__ void __launch_bounds__(B) k_ppass(const uint32_t* __restrict__ R,
                                             const uint32_t* __restrict__ P, uint64_t A,
                                             const uint32_t* __restrict__ U,
                                             const uint32_t* __restrict__ NP,
                                             const uint32_t* __restrict__ TB, uint32_t* PMIN,
                                             uint32_t* NCP) {
  __shared__ unsigned long long s_pc[PCACHE];
  __shared__ uint32_t s_nc[PCACHE];
  for (int i = threadIdx.x; i < PCACHE; i += B) {
    s_pc[i] = ~0ull;
    s_nc[i] = INF;
  }
  __syncthreads();
  const uint64_t nq = (A + 3) >> 2;
  for (uint64_t t = blockIdx.x * (uint64_t)B + threadIdx.x; t < nq; t += (uint64_t)gridDim.x * B) {
    uint32_t r[4], p[4];
    if (4 * t + 3 < A) {
      const uint4 a = ldg_stream(reinterpret_cast<const uint4*>(R) + t);
      const uint4 b = ldg_stream(reinterpret_cast<const uint4*>(P) + t);
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
      p[0] = b.x; p[1] = b.y; p[2] = b.z; p[3] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        r[j] = (4 * t + j < A) ? R[4 * t + j] : 0u;
        p[j] = (4 * t + j < A) ? P[4 * t + j] : DEAD;
      }
    }
    uint32_t q[4];
    bool np[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      q[j] = INF;
      np[j] = false;
      if (p[j] != DEAD) {
        q[j] = __ldg(&U[r[j]]);
        if (!FIRST && tbit(TB, r[j])) q[j] = min(q[j], r[j]);
        if (FIRST) np[j] = tbit(NP, r[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (p[j] == DEAD) continue;
      const uint32_t h = (p[j] ^ (p[j] >> 10)) & (PCACHE - 1);
      const unsigned long long e = *(volatile unsigned long long*)&s_pc[h];
      if ((uint32_t)(e >> 32) == p[j] && q[j] >= (uint32_t)e) continue;
      const uint32_t old = atomicMin(&PMIN[p[j]], q[j]);
      s_pc[h] = ((unsigned long long)p[j] << 32) | min(old, q[j]);
    }
    if (FIRST) {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (!np[j]) continue;
        const uint32_t h = (p[j] ^ (p[j] >> 10)) & (PCACHE - 1);
        if (*(volatile uint32_t*)&s_nc[h] == p[j]) continue;
        atomicOr(&NCP[p[j] >> 5], 1u << (p[j] & 31));
        s_nc[h] = p[j];
      }
    }
  }
}

// Temporaries of line 22 in pass 4: <u,_,u>_tmp in PB(u) with q = u_min'(u) = min(U[u], u).
__global__ void k_temps(const uint32_t* __restrict__ TB, uint64_t n, const uint32_t* __restrict__ U,
                        uint32_t* PMIN) {
  const uint64_t nw = (n + 31) / 32;
  for (uint64_t w = blockIdx.x * (uint64_t)B + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * B) {
    uint32_t bits = TB[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint32_t u = (uint32_t)(w * 32 + b);
      min_slot(PMIN, u, min(__ldg(&U[u]), u));
    }
  }
}

// Partition statistics over the slots (P_i, completed, changed, T_i; or changed2) and the
// temporary-tuple bitmap (one temp <p_min,_,p_min> per surviving partition, line 22).
template <bool FIRST>
__global__ void __launch_bounds__(B) k_pscan(const uint32_t* __restrict__ PMIN,
                                             const uint32_t* __restrict__ NCP, uint64_t n,
                                             uint32_t* TB, unsigned long long* ctr) {
  uint32_t np = 0, nc = 0, ch = 0, nt = 0;
  for (uint64_t p = blockIdx.x * (uint64_t)B + threadIdx.x; p < n; p += (uint64_t)gridDim.x * B) {
    const uint32_t pm = PMIN[p];
    if (pm == INF) continue;
    ch += (pm != (uint32_t)p);
    if (FIRST) {
      np++;
      const bool comp = !tbit(NCP, (uint32_t)p) && pm == (uint32_t)p;
      nc += comp;
      if (!comp) {
        nt++;
        set_bit(TB, pm);
      }
    }
  }
  np = warp_sum(np); nc = warp_sum(nc); ch = warp_sum(ch); nt = warp_sum(nt);
  if ((threadIdx.x & 31) == 0) {
    if (FIRST) {
      if (np) atomicAdd(&ctr[sv::C_PARTITIONS], (unsigned long long)np);
      if (nc) atomicAdd(&ctr[sv::C_COMPLETED], (unsigned long long)nc);
      if (ch) atomicAdd(&ctr[sv::C_CHANGED], (unsigned long long)ch);
      if (nt) atomicAdd(&ctr[sv::C_TEMPS], (unsigned long long)nt);
    } else if (ch) {
      atomicAdd(&ctr[sv::C_CHANGED2], (unsigned long long)ch);
    }
  }
}

// Lines 17-21 + sec:distSVOpt1: tuples of completed partitions leave (their vertex takes
// label p), survivors get p <- p_min.  Leaving is done in place (P = DEAD,
// whole rows, R order untouched); k_compact squeezes dead rows out when they pile up.
__global__ void __launch_bounds__(B) k_papply1(const uint32_t* __restrict__ R, uint32_t* P,
                                               uint64_t A, const uint32_t* __restrict__ PMIN,
                                               const uint32_t* __restrict__ NCP,
                                               uint32_t* __restrict__ label,
                                               unsigned long long* ctr) {
  uint32_t live = 0;
  const uint64_t nq = (A + 3) >> 2;
  for (uint64_t t = blockIdx.x * (uint64_t)B + threadIdx.x; t < nq; t += (uint64_t)gridDim.x * B) {
    uint32_t p[4];
    const bool full = 4 * t + 3 < A;
    if (full) {
      const uint4 b = reinterpret_cast<const uint4*>(P)[t];
      p[0] = b.x; p[1] = b.y; p[2] = b.z; p[3] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) p[j] = (4 * t + j < A) ? P[4 * t + j] : DEAD;
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      o[j] = DEAD;
      if (p[j] == DEAD) continue;
      const uint32_t pm = __ldg(&PMIN[p[j]]);
      if (pm == p[j] && !tbit(NCP, p[j])) {
        label[R[4 * t + j]] = p[j];  // completed: every tuple of VB(r) is in p
      } else {
        o[j] = pm;
        live++;
      }
    }
    if (full) reinterpret_cast<uint4*>(P)[t] = make_uint4(o[0], o[1], o[2], o[3]);
    else
      for (int j = 0; j < 4; j++)
        if (4 * t + j < A) P[4 * t + j] = o[j];
  }
  live = warp_sum(live);
  if ((threadIdx.x & 31) == 0 && live) atomicAdd(&ctr[sv::C_OUT], (unsigned long long)live);
}

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

// Line 25 update: p <- p_min of the second partition pass, in place (temporaries are
// bitmap entries, so nothing is erased and the array stays in R order).
__global__ void __launch_bounds__(B) k_papply2(uint32_t* __restrict__ P, uint64_t A,
                                               const uint32_t* __restrict__ PMIN) {
  const uint64_t nq = (A + 3) >> 2;
  for (uint64_t t = blockIdx.x * (uint64_t)B + threadIdx.x; t < nq; t += (uint64_t)gridDim.x * B) {
    if (4 * t + 3 < A) {
      uint4 b = reinterpret_cast<const uint4*>(P)[t];
      if (b.x != DEAD) b.x = __ldg(&PMIN[b.x]);
      if (b.y != DEAD) b.y = __ldg(&PMIN[b.y]);
      if (b.z != DEAD) b.z = __ldg(&PMIN[b.z]);
      if (b.w != DEAD) b.w = __ldg(&PMIN[b.w]);
      reinterpret_cast<uint4*>(P)[t] = b;
    } else {
      for (uint64_t i = 4 * t; i < A; i++)
        if (P[i] != DEAD) P[i] = __ldg(&PMIN[P[i]]);
    }
  }
}

// ===================================================================== launchers
int group_shift(uint64_t n, uint64_t tuples) {
  int kb = 0;
  while ((1ull << kb) < n) kb++;
  int lg = 0;  // log2 G: about 2M tuples per group
  while (lg < 10 && (tuples >> (21 + lg)) > 0) lg++;
  int gs = kb - lg;
  return gs < 11 ? 11 : gs;
}

void build(const uint2* edges, uint64_t m, const uint32_t* deg, const uint32_t* vis, uint64_t n,
           uint32_t* off, uint32_t* cur, uint32_t* garc, int gshift, scan::State& ss, uint64_t* ctr,
           cudaStream_t st) {
  // ctr[C_VT_OUT] receives A_0
  if (!n) return;
  const int G = (int)(((n - 1) >> gshift) + 1);
  cudaMemsetAsync(ss.ticket, 0, sizeof(uint32_t), st);
  cudaMemsetAsync(garc, 0, sizeof(uint32_t) * G, st);
  const uint64_t tiles = (n + B * SITEMS - 1) / (B * SITEMS);
  k_rows<<<(unsigned)tiles, B, 0, st>>>(deg, vis, n, off, cur, ss.flags, ss.ticket, ++ss.epoch,
                                         reinterpret_cast<unsigned long long*>(ctr + sv::C_VT_OUT),
                                         garc, gshift);
}
void fill(const uint2* edges, uint64_t m, const uint32_t* off, uint32_t* cur, uint64_t n, uint64_t A,
          uint32_t* R, uint32_t* P, const uint32_t* garc, int gshift, uint64_t* gcur, uint2* tmp,
          uint32_t* longlist, uint64_t* nlong, cudaStream_t st) {
  if (!A) return;
  const int G = (int)(((n - 1) >> gshift) + 1);
  auto* nl = reinterpret_cast<unsigned long long*>(nlong);
  cudaMemsetAsync(nlong, 0, sizeof(uint64_t), st);
  k_fill_rows<<<grid(n, B, 148 * 8), B, 0, st>>>(off, n, R, P, longlist, nl);
  k_fill_long<<<148 * 2, B, 0, st>>>(off, longlist, nl, R);
  if (!m) return;
  auto* gc = reinterpret_cast<unsigned long long*>(gcur);
  k_gscan<<<1, B, 0, st>>>(garc, G, gc);
  k_bucket<<<(unsigned)((m + B * BITEMS - 1) / (B * BITEMS)), B, 0, st>>>(edges, m, gshift, G, gc, tmp);
  k_scatter<<<grid(2 * m, B, 148 * 16), B, 0, st>>>(tmp, 2 * m, cur, P);
}
void vpass(bool with_pc, const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* U, uint32_t* NP,
           cudaStream_t st) {
  if (!A) return;
  const uint64_t warps = (A + VCHUNK - 1) / VCHUNK;  // one warp per VCHUNK tuples
  const unsigned g = (unsigned)((warps * 32 + B - 1) / B);
  if (with_pc) k_vpass<true><<<g, B, 0, st>>>(R, P, A, U, NP);
  else k_vpass<false><<<g, B, 0, st>>>(R, P, A, U, NP);
}
void ppass(bool first, const uint32_t* R, const uint32_t* P, uint64_t A, const uint32_t* U,
           const uint32_t* NP, const uint32_t* TB, uint32_t* PMIN, uint32_t* NCP, cudaStream_t st) {
  if (!A) return;
  const unsigned g = grid((A + 3) / 4, B, 148 * 8);
  if (first) k_ppass<true><<<g, B, 0, st>>>(R, P, A, U, NP, TB, PMIN, NCP);
  else k_ppass<false><<<g, B, 0, st>>>(R, P, A, U, NP, TB, PMIN, NCP);
}
void temps(const uint32_t* TB, uint64_t n, const uint32_t* U, uint32_t* PMIN, cudaStream_t st) {
  if (n) k_temps<<<grid((n + 31) / 32, B, 148 * 4), B, 0, st>>>(TB, n, U, PMIN);
}
void pscan(bool first, const uint32_t* PMIN, const uint32_t* NCP, uint64_t n, uint32_t* TB,
           uint64_t* ctr, cudaStream_t st) {
  if (!n) return;
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  if (first) k_pscan<true><<<grid(n, B, 148 * 8), B, 0, st>>>(PMIN, NCP, n, TB, c);
  else k_pscan<false><<<grid(n, B, 148 * 8), B, 0, st>>>(PMIN, NCP, n, TB, c);
}
void papply1(const uint32_t* R, uint32_t* P, uint64_t A, const uint32_t* PMIN, const uint32_t* NCP,
             uint32_t* label, uint64_t* ctr, cudaStream_t st) {
  if (A)
    k_papply1<<<grid((A + 3) / 4, B, 148 * 8), B, 0, st>>>(R, P, A, PMIN, NCP, label,
                                                           reinterpret_cast<unsigned long long*>(ctr));
}
void compact(const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* R2, uint32_t* P2,
             scan::State& ss, cudaStream_t st) {
  if (!A) return;
  cudaMemsetAsync(ss.ticket, 0, sizeof(uint32_t), st);
  const uint64_t tiles = (A + CTILE - 1) / CTILE;
  k_compact<<<(unsigned)tiles, B, 0, st>>>(R, P, A, R2, P2, ss.flags, ss.ticket, ++ss.epoch);
}
void papply2(uint32_t* P, uint64_t A, const uint32_t* PMIN, cudaStream_t st) {
  if (A) k_papply2<<<grid((A + 3) / 4, B, 148 * 8), B, 0, st>>>(P, A, PMIN);
}

}  // namespace csr
}  // namespace cc
