// sv_direct.cu -- the SV bucket passes with direct-addressed buckets (B200 variant).
//
// Alg. 1 sorts A_i by r (line 8) and by p (line 14) only so that each bucket VB_i(u) /
// PB_i(p) is contiguous when its minimum is taken ("enables easy and
// cache efficient processing of each vertex bucket").  Ids here are dense in [0, n) (the
// relabel of Alg. 2 line 4), so a bucket can instead be addressed directly:
// its minimum lives in slot [u] / [p] of an n-sized array that stays resident in the
// 126 MB L2, and no tuple is ever moved except by the compaction that drops completed
// partitions.  Every set and counter of Alg. 1 is unchanged.
//
// Contention control: values only decrease (min) or only gain bits (or), so a plain read
// of the slot first skips every update that cannot change it; a bucket with 10^6 tuples
// (a hub vertex, the giant partition) then costs ~log(size) atomics, not 10^6.
#include <algorithm>

#include "sv.cuh"

namespace cc {
namespace sv {

constexpr int DBLOCK = 256;

CC_DEVI void min_slot(uint32_t* a, uint32_t i, uint32_t v) {
  if (v < *(volatile uint32_t*)&a[i]) atomicMin(&a[i], v);
}
CC_DEVI bool test_bit(const uint32_t* bm, uint32_t i) { return (bm[i >> 5] >> (i & 31)) & 1u; }
CC_DEVI void set_bit(uint32_t* bm, uint32_t i) {
  const uint32_t m = 1u << (i & 31);
  if (!(*(volatile uint32_t*)&bm[i >> 5] & m)) atomicOr(&bm[i >> 5], m);
}
// returns true for exactly one caller per bit (the bucket 'head')
CC_DEVI bool claim_bit(uint32_t* bm, uint32_t i) {
  const uint32_t m = 1u << (i & 31);
  if (*(volatile uint32_t*)&bm[i >> 5] & m) return false;
  return !(atomicOr(&bm[i >> 5], m) & m);
}

// Each thread handles two by-r words per step (one 16-byte load).
#define DIRECT_LOOP(...)                                                                \
  const uint64_t npair = (n + 1) >> 1;                                                   \
  for (uint64_t t = blockIdx.x * (uint64_t)DBLOCK + threadIdx.x; t < npair;              \
       t += (uint64_t)gridDim.x * DBLOCK) {                                              \
    uint32_t lo[2], hi[2];                                                               \
    int cnt;                                                                             \
    if (2 * t + 1 < n) {                                                                 \
      uint4 x = ldg_stream(reinterpret_cast<const uint4*>(w) + t);                       \
      lo[0] = x.x; hi[0] = x.y; lo[1] = x.z; hi[1] = x.w; cnt = 2;                       \
    } else {                                                                             \
      uint64_t x = w[2 * t];                                                             \
      lo[0] = lo32(x); hi[0] = hi32(x); cnt = 1;                                         \
    }                                                                                    \
    _Pragma("unroll") for (int j = 0; j < 2; j++) {                                      \
      if (j < cnt) { __VA_ARGS__ }                                                              \
    }                                                                                    \
  }

// vertex pass (lines 9-11 / line 24): umin[r] = min p over VB(u)
__global__ void __launch_bounds__(DBLOCK) k_d_vmin(const uint64_t* __restrict__ w, uint64_t n,
                                                   uint32_t* umin) {
  DIRECT_LOOP({
    const uint32_t r = hi[j], p = lo[j] & ID_MASK;
    min_slot(umin, r, p);
  })
}

// potentially completed: |M(u)| = 1 iff every tuple of VB(u) has p = u_min;
// record the complement bit notpc[r].
__global__ void __launch_bounds__(DBLOCK) k_d_vpc(const uint64_t* __restrict__ w, uint64_t n,
                                                  const uint32_t* __restrict__ umin,
                                                  uint32_t* notpc) {
  DIRECT_LOOP({
    const uint32_t r = hi[j], p = lo[j] & ID_MASK;
    if (p != __ldg(&umin[r])) set_bit(notpc, r);
  })
}

// partition pass (lines 15-16 / line 25): pmin[p] = min q over PB(p), q = umin[r];
// FIRST also ORs 'not potentially completed' into ncp[p] (completion).
template <bool FIRST>
__global__ void __launch_bounds__(DBLOCK) k_d_pmin(const uint64_t* __restrict__ w, uint64_t n,
                                                   const uint32_t* __restrict__ umin,
                                                   const uint32_t* __restrict__ notpc,
                                                   uint32_t* pmin, uint32_t* ncp) {
  DIRECT_LOOP({
    const uint32_t r = hi[j], p = lo[j] & ID_MASK;
    min_slot(pmin, p, __ldg(&umin[r]));
    if (FIRST && test_bit(notpc, r)) set_bit(ncp, p);
  })
}

// partition update + compaction.  FIRST: lines 17-22 with the exclusion of completed
// partitions; !FIRST: line 25's update and lines 26-28 (erase temporaries).  The bucket
// head (one tuple per partition, elected by claim_bit) does the per-partition work.
template <bool FIRST>
__global__ void __launch_bounds__(DBLOCK) k_d_papply(const uint64_t* __restrict__ w, uint64_t n,
                                                     const uint32_t* __restrict__ pmin,
                                                     const uint32_t* __restrict__ ncp,
                                                     uint32_t* headbm, uint64_t* __restrict__ wout,
                                                     uint32_t* __restrict__ label,
                                                     unsigned long long* ctr) {
  __shared__ uint32_t s_scan[DBLOCK / 32 + 1];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_stat[4];
  if (threadIdx.x < 4) s_stat[threadIdx.x] = 0;
  uint32_t st_part = 0, st_comp = 0, st_chg = 0, st_tmp = 0;
  const uint64_t npair = (n + 1) >> 1;
  const uint64_t stride = (uint64_t)gridDim.x * DBLOCK;
  // uniform trip count so every thread reaches the block scans
  const uint64_t iters = (npair + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; it++) {
    const uint64_t t = it * stride + blockIdx.x * (uint64_t)DBLOCK + threadIdx.x;
    uint64_t outw[4];
    uint32_t nout = 0;
    if (t < npair) {
      uint32_t lo[2], hi[2];
      int cnt;
      if (2 * t + 1 < n) {
        uint4 x = ldg_stream(reinterpret_cast<const uint4*>(w) + t);
        lo[0] = x.x; hi[0] = x.y; lo[1] = x.z; hi[1] = x.w; cnt = 2;
      } else {
        uint64_t x = w[2 * t];
        lo[0] = lo32(x); hi[0] = hi32(x); cnt = 1;
      }
#pragma unroll
      for (int j = 0; j < 2; j++) {
        if (j >= cnt) break;
        const uint32_t r = hi[j], l = lo[j], p = l & ID_MASK;
        const uint32_t pm = __ldg(&pmin[p]);
        if (FIRST) {
          const bool comp = !test_bit(ncp, p);
          if (claim_bit(headbm, p)) {
            st_part++;
            st_comp += comp;
            st_chg += (pm != p);
            if (!comp) {
              outw[nout++] = mk(pm, pm | F_TMP);
              st_tmp++;
            }
          }
          if (comp) {
            if (l & F_VT) label[r] = p;
          } else {
            outw[nout++] = mk(r, pm | (l & F_VT));
          }
        } else {
          if (claim_bit(headbm, p)) st_chg += (pm != p);
          if (!(l & F_TMP)) outw[nout++] = mk(r, pm | (l & F_VT));
        }
      }
    }
    uint32_t tot;
    const uint32_t off = block_excl_scan<DBLOCK>(nout, s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(&ctr[C_OUT], (unsigned long long)tot) : 0ull;
    __syncthreads();
    uint64_t* dst = wout + s_base + off;
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (j < (int)nout) dst[j] = outw[j];
    __syncthreads();
  }
  uint32_t a = warp_sum(st_part), b = warp_sum(st_comp), c = warp_sum(st_chg), d = warp_sum(st_tmp);
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(&s_stat[0], a);
    if (b) atomicAdd(&s_stat[1], b);
    if (c) atomicAdd(&s_stat[2], c);
    if (d) atomicAdd(&s_stat[3], d);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (FIRST) {
      if (s_stat[0]) atomicAdd(&ctr[C_PARTITIONS], (unsigned long long)s_stat[0]);
      if (s_stat[1]) atomicAdd(&ctr[C_COMPLETED], (unsigned long long)s_stat[1]);
      if (s_stat[2]) atomicAdd(&ctr[C_CHANGED], (unsigned long long)s_stat[2]);
      if (s_stat[3]) atomicAdd(&ctr[C_TEMPS], (unsigned long long)s_stat[3]);
    } else if (s_stat[2]) {
      atomicAdd(&ctr[C_CHANGED2], (unsigned long long)s_stat[2]);
    }
  }
}

static unsigned dgrid(uint64_t n) {
  uint64_t g = ((n + 1) / 2 + DBLOCK - 1) / DBLOCK;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148 * 8));
}

void launch_direct_vmin(const uint64_t* w, uint64_t n, uint32_t* umin, cudaStream_t st) {
  if (n) k_d_vmin<<<dgrid(n), DBLOCK, 0, st>>>(w, n, umin);
}
void launch_direct_vpc(const uint64_t* w, uint64_t n, const uint32_t* umin, uint32_t* notpc,
                       cudaStream_t st) {
  if (n) k_d_vpc<<<dgrid(n), DBLOCK, 0, st>>>(w, n, umin, notpc);
}
void launch_direct_pmin(bool first, const uint64_t* w, uint64_t n, const uint32_t* umin,
                        const uint32_t* notpc, uint32_t* pmin, uint32_t* ncp, cudaStream_t st) {
  if (!n) return;
  if (first) k_d_pmin<true><<<dgrid(n), DBLOCK, 0, st>>>(w, n, umin, notpc, pmin, ncp);
  else k_d_pmin<false><<<dgrid(n), DBLOCK, 0, st>>>(w, n, umin, notpc, pmin, ncp);
}
void launch_direct_papply(bool first, const uint64_t* w, uint64_t n, const uint32_t* pmin,
                          const uint32_t* ncp, uint32_t* headbm, uint64_t* wout, uint32_t* label,
                          uint64_t* ctr, cudaStream_t st) {
  if (!n) return;
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  if (first)
    k_d_papply<true><<<dgrid(n), DBLOCK, 0, st>>>(w, n, pmin, ncp, headbm, wout, label, c);
  else
    k_d_papply<false><<<dgrid(n), DBLOCK, 0, st>>>(w, n, pmin, ncp, headbm, wout, label, c);
}

}  // namespace sv
}  // namespace cc
