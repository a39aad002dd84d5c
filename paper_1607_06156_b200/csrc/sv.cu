// sv.cu -- tuple init, bucket reductions and the two bucket-update passes of Alg. 1.
//
// One SV iteration is, per regroup:
//   sort (radix.cu)  ->  k_seg_reduce (bucket minima into dense per-key slots)
//                    ->  k_vertex_apply / k_partition_apply (update + compaction)
// Bucket reductions follow the paper's "bucket updates": after the sort
// the tuples of a bucket are contiguous; buckets that span warps/blocks are combined
// through per-key slots (the GPU analogue of the two exclusive scans across processes).
#include "sv.cuh"

#include <algorithm>

namespace cc {
namespace sv {

constexpr int BLOCK = 256;

// ------------------------------------------------------------------------------ init
__global__ void k_init_labels(uint32_t* __restrict__ label, uint64_t n) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    label[v] = (uint32_t)v;
}

// Alg. 1 line 3: <x,_,y> and <y,_,x> per undirected edge {x,y}.  As by-r words:
// tuple <p=x, r=y> -> (y<<32 | x).
__global__ void k_init_arcs(const uint2* __restrict__ edges, uint64_t m, uint4* __restrict__ w) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint2 xy = edges[e];
    // word0 = (y<<32)|x , word1 = (x<<32)|y
    w[e] = make_uint4(xy.x, xy.y, xy.y, xy.x);
  }
}

// Alg. 1 line 2: <x,_,x> for every x in V that an edge touches, optionally
// excluding BFS-visited ids.  Appended at w[base + ...] through a block-aggregated cursor.
__global__ void k_init_vtuples(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ vis,
                               uint64_t n, uint64_t* __restrict__ w, uint64_t base,
                               unsigned long long* cursor) {
  __shared__ uint32_t s_scan[BLOCK / 32 + 1];
  __shared__ unsigned long long s_base;
  for (uint64_t v0 = blockIdx.x * (uint64_t)BLOCK; v0 < n; v0 += (uint64_t)gridDim.x * BLOCK) {
    uint64_t v = v0 + threadIdx.x;
    uint32_t pres = 0;
    if (v < n) {
      pres = deg[v] > 0;
      if (vis && ((vis[v >> 5] >> (v & 31)) & 1u)) pres = 0;
    }
    uint32_t tot;
    uint32_t off = block_excl_scan<BLOCK>(pres, s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(cursor, (unsigned long long)tot) : 0ull;
    __syncthreads();
    if (pres) w[base + s_base + off] = mk((uint32_t)v, (uint32_t)v | F_VT);
    __syncthreads();
  }
}

void launch_init_labels(uint32_t* label, uint64_t n, cudaStream_t st) {
  if (!n) return;
  int g = (int)std::min<uint64_t>((n + BLOCK - 1) / BLOCK, 148 * 16);
  k_init_labels<<<g, BLOCK, 0, st>>>(label, n);
}

void launch_init_tuples(const uint2* edges, uint64_t m, const uint32_t* deg,
                        const uint32_t* visited_bm, uint64_t n, uint64_t* w, uint64_t* ctr,
                        cudaStream_t st, uint64_t* launches) {
  if (m) {
    int g = (int)std::min<uint64_t>((m + BLOCK - 1) / BLOCK, 148 * 16);
    k_init_arcs<<<g, BLOCK, 0, st>>>(edges, m, reinterpret_cast<uint4*>(w));
    *launches += 1;
  }
  if (n) {
    int g = (int)std::min<uint64_t>((n + BLOCK - 1) / BLOCK, 148 * 8);
    k_init_vtuples<<<g, BLOCK, 0, st>>>(deg, visited_bm, n, w, 2 * m,
                                        reinterpret_cast<unsigned long long*>(ctr + C_VT_OUT));
    *launches += 1;
  }
}

// ---------------------------------------------------------------- bucket reductions
// Each warp reduces a contiguous chunk of SEG_CHUNK tuples in steps of 32.  Equal keys are
// contiguous (sorted input), so a segmented suffix-reduction over shuffles gives each run's
// value at its head lane; the run touching lane 31 is carried into the next step, so a
// bucket spanning the whole chunk costs one atomic per chunk, not per step.
constexpr int SEG_STEPS = 64;
constexpr int SEG_CHUNK = 32 * SEG_STEPS;
constexpr uint32_t SENT = 0xFFFFFFFFu;

template <int MODE>
CC_DEVI void seg_emit(uint32_t key, uint32_t v, uint32_t v2, uint32_t* segA, uint32_t* segB) {
  atomicMin(&segA[key], v);
  if (MODE == SEG_VMINMAX) atomicMax(&segB[key], v2);
  if (MODE == SEG_PMIN_NC && v2) segB[key] = 1u;  // benign race: every writer stores 1
}

template <int MODE>
__global__ void __launch_bounds__(BLOCK) k_seg_reduce(const uint64_t* __restrict__ w,
                                                      const uint32_t* __restrict__ q, uint64_t n,
                                                      uint32_t* __restrict__ segA,
                                                      uint32_t* __restrict__ segB) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)BLOCK + threadIdx.x) >> 5;
  const uint64_t cbase = warp * SEG_CHUNK;
  if (cbase >= n) return;
  uint32_t ckey = SENT, cv = SENT, cv2 = 0;
  for (int k = 0; k < SEG_STEPS; k++) {
    const uint64_t i = cbase + (uint64_t)k * 32 + lane;
    uint32_t key = SENT, v = SENT, v2 = 0;
    if (i < n) {
      uint64_t word = w[i];
      key = hi32(word);
      if (MODE == SEG_VMINMAX || MODE == SEG_VMIN) {
        v = lo32(word) & ID_MASK;
        v2 = v;
      } else {
        uint32_t qq = q[i];
        v = qq & ID_MASK;
        v2 = (qq & F_PC) ? 0u : 1u;  // "not potentially completed"
      }
    }
    if (__all_sync(0xffffffffu, key == SENT)) break;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t ko = __shfl_down_sync(0xffffffffu, key, o);
      uint32_t vo = __shfl_down_sync(0xffffffffu, v, o);
      uint32_t v2o = __shfl_down_sync(0xffffffffu, v2, o);
      if (lane + o < 32 && ko == key) {
        v = min(v, vo);
        v2 = (MODE == SEG_VMINMAX) ? max(v2, v2o) : (v2 | v2o);
      }
    }
    const uint32_t kprev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = (lane == 0) || (kprev != key);
    const uint32_t hmask = __ballot_sync(0xffffffffu, head);
    const int last = 31 - __clz(hmask);
    const uint32_t key0 = __shfl_sync(0xffffffffu, key, 0);
    uint32_t v0 = __shfl_sync(0xffffffffu, v, 0);
    uint32_t v20 = __shfl_sync(0xffffffffu, v2, 0);
    const uint32_t keyL = __shfl_sync(0xffffffffu, key, last);
    const uint32_t vL = __shfl_sync(0xffffffffu, v, last);
    const uint32_t v2L = __shfl_sync(0xffffffffu, v2, last);
    if (key0 == ckey) {
      v0 = min(v0, cv);
      v20 = (MODE == SEG_VMINMAX) ? max(v20, cv2) : (v20 | cv2);
    } else if (lane == 0 && ckey != SENT) {
      seg_emit<MODE>(ckey, cv, cv2, segA, segB);
    }
    if (last == 0) {
      ckey = key0; cv = v0; cv2 = v20;
    } else {
      if (lane == 0 && key0 != SENT) seg_emit<MODE>(key0, v0, v20, segA, segB);
      if (head && lane != 0 && lane != last && key != SENT) seg_emit<MODE>(key, v, v2, segA, segB);
      ckey = keyL; cv = vL; cv2 = v2L;
    }
  }
  if (lane == 0 && ckey != SENT) seg_emit<MODE>(ckey, cv, cv2, segA, segB);
}

void launch_seg_reduce(int mode, const uint64_t* w, const uint32_t* q, uint64_t n, uint32_t* segA,
                       uint32_t* segB, cudaStream_t st) {
  if (!n) return;
  uint64_t warps = (n + SEG_CHUNK - 1) / SEG_CHUNK;
  unsigned g = (unsigned)((warps * 32 + BLOCK - 1) / BLOCK);
  switch (mode) {
    case SEG_VMINMAX: k_seg_reduce<SEG_VMINMAX><<<g, BLOCK, 0, st>>>(w, q, n, segA, segB); break;
    case SEG_VMIN: k_seg_reduce<SEG_VMIN><<<g, BLOCK, 0, st>>>(w, q, n, segA, segB); break;
    case SEG_PMIN_NC: k_seg_reduce<SEG_PMIN_NC><<<g, BLOCK, 0, st>>>(w, q, n, segA, segB); break;
    default: k_seg_reduce<SEG_PMIN><<<g, BLOCK, 0, st>>>(w, q, n, segA, segB); break;
  }
}

// ------------------------------------------------------------------ vertex pass update
// Alg. 1 lines 10-12 (and line 24): q <- u_min for every tuple of VB(u); with_pc marks
// 'potentially completed' iff |M_i(u)| = 1, i.e. min p = max p over VB(u).
// Converts by-r words (r | p,flags) into by-p words (p | r,flags) + q word.
template <bool WITH_PC>
__global__ void __launch_bounds__(BLOCK) k_vertex_apply(const uint4* __restrict__ win, uint64_t n,
                                                        const uint32_t* __restrict__ segA,
                                                        const uint32_t* __restrict__ segB,
                                                        uint4* __restrict__ wout,
                                                        uint2* __restrict__ qout) {
  const uint64_t npair = n >> 1;
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i <= npair;
       i += (uint64_t)gridDim.x * BLOCK) {
    if (i < npair) {
      uint4 x = ldg_stream(&win[i]);  // two words: (x.x lo, x.y hi), (x.z lo, x.w hi)
      uint32_t r0 = x.y, r1 = x.w;
      uint32_t u0 = __ldg(&segA[r0]), u1 = __ldg(&segA[r1]);
      uint32_t pc0 = 0, pc1 = 0;
      if (WITH_PC) {
        pc0 = (u0 == __ldg(&segB[r0])) ? F_PC : 0u;
        pc1 = (u1 == __ldg(&segB[r1])) ? F_PC : 0u;
      }
      // by-p word: hi = p, lo = r | flags
      wout[i] = make_uint4(r0 | (x.x & FLAGS), x.x & ID_MASK, r1 | (x.z & FLAGS), x.z & ID_MASK);
      qout[i] = make_uint2(u0 | pc0, u1 | pc1);
    } else if (n & 1) {
      const uint64_t* w1 = reinterpret_cast<const uint64_t*>(win);
      uint64_t word = w1[n - 1];
      uint32_t r = hi32(word), lo = lo32(word);
      uint32_t u = segA[r];
      uint32_t pc = (WITH_PC && u == segB[r]) ? F_PC : 0u;
      reinterpret_cast<uint64_t*>(wout)[n - 1] = mk(lo & ID_MASK, r | (lo & FLAGS));
      reinterpret_cast<uint32_t*>(qout)[n - 1] = u | pc;
    }
  }
}

void launch_vertex_apply(bool with_pc, const uint64_t* win, uint64_t n, const uint32_t* segA,
                         const uint32_t* segB, uint64_t* wout, uint32_t* qout, cudaStream_t st) {
  if (!n) return;
  uint64_t work = (n >> 1) + 1;
  unsigned g = (unsigned)std::min<uint64_t>((work + BLOCK - 1) / BLOCK, 148 * 16);
  if (with_pc)
    k_vertex_apply<true><<<g, BLOCK, 0, st>>>(reinterpret_cast<const uint4*>(win), n, segA, segB,
                                              reinterpret_cast<uint4*>(wout),
                                              reinterpret_cast<uint2*>(qout));
  else
    k_vertex_apply<false><<<g, BLOCK, 0, st>>>(reinterpret_cast<const uint4*>(win), n, segA, segB,
                                               reinterpret_cast<uint4*>(wout),
                                               reinterpret_cast<uint2*>(qout));
}

// --------------------------------------------------------------- partition pass update
// FIRST (Alg. 1 lines 14-22 + sec:distSVOpt1): per PB(p): p_min = min C_i(p); counters at
// the bucket head; completed partitions (all tuples PC) write the labels of
// their vertex tuples and are dropped (stream compaction, C4 early exclusion); survivors
// get p <- p_min; each surviving bucket appends <p_min,_,p_min>_tmp (line 22).
// !FIRST (line 25 + lines 26-28): p <- p_min for every tuple, temporaries erased.
// Output: by-r words (r | p_min, VT) compacted through one atomic per block.
constexpr int PITEMS = 8;
constexpr int PTILE = BLOCK * PITEMS;

template <bool FIRST>
__global__ void __launch_bounds__(BLOCK) k_partition_apply(
    const uint64_t* __restrict__ win, const uint32_t* __restrict__ qin, uint64_t n,
    const uint32_t* __restrict__ segA, const uint32_t* __restrict__ segB,
    uint64_t* __restrict__ wout, uint32_t* __restrict__ label, unsigned long long* ctr) {
  __shared__ uint32_t s_scan[BLOCK / 32 + 1];
  __shared__ unsigned long long s_base;
  __shared__ uint32_t s_stat[4];
  if (threadIdx.x < 4) s_stat[threadIdx.x] = 0;
  const uint64_t t0 = (blockIdx.x * (uint64_t)PTILE) + (uint64_t)threadIdx.x * PITEMS;
  uint64_t outw[2 * PITEMS];
  uint32_t nout = 0;
  uint32_t st_part = 0, st_comp = 0, st_chg = 0, st_tmp = 0;
  uint32_t prevkey = (t0 > 0 && t0 <= n) ? hi32(win[t0 - 1]) : SENT;
#pragma unroll
  for (int j = 0; j < PITEMS; j++) {
    const uint64_t i = t0 + j;
    if (i < n) {
      const uint64_t word = win[i];
      const uint32_t p = hi32(word), lo = lo32(word);
      const uint32_t r = lo & ID_MASK;
      const bool head = (i == 0) || (p != prevkey);
      prevkey = p;
      const uint32_t pmin = segA[p];
      if (FIRST) {
        const bool comp = segB[p] == 0u;
        if (head) {
          st_part++;
          st_comp += comp;
          st_chg += (pmin != p);
          if (!comp) {
            outw[nout++] = mk(pmin, pmin | F_TMP);
            st_tmp++;
          }
        }
        if (comp) {
          if (lo & F_VT) label[r] = p;
        } else {
          outw[nout++] = mk(r, pmin | (lo & F_VT));
        }
      } else {
        if (head) st_chg += (pmin != p);
        if (!(lo & F_TMP)) outw[nout++] = mk(r, pmin | (lo & F_VT));
      }
    }
  }
  __syncthreads();  // s_stat init visible
  // counters
  if (FIRST) {
    uint32_t a = warp_sum(st_part), b = warp_sum(st_comp), c = warp_sum(st_chg),
             d = warp_sum(st_tmp);
    if ((threadIdx.x & 31) == 0) {
      if (a) atomicAdd(&s_stat[0], a);
      if (b) atomicAdd(&s_stat[1], b);
      if (c) atomicAdd(&s_stat[2], c);
      if (d) atomicAdd(&s_stat[3], d);
    }
  } else {
    uint32_t c = warp_sum(st_chg);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_stat[2], c);
  }
  uint32_t tot;
  uint32_t off = block_excl_scan<BLOCK>(nout, s_scan, &tot);
  if (threadIdx.x == 0) {
    s_base = tot ? atomicAdd(&ctr[C_OUT], (unsigned long long)tot) : 0ull;
    if (FIRST) {
      if (s_stat[0]) atomicAdd(&ctr[C_PARTITIONS], (unsigned long long)s_stat[0]);
      if (s_stat[1]) atomicAdd(&ctr[C_COMPLETED], (unsigned long long)s_stat[1]);
      if (s_stat[2]) atomicAdd(&ctr[C_CHANGED], (unsigned long long)s_stat[2]);
      if (s_stat[3]) atomicAdd(&ctr[C_TEMPS], (unsigned long long)s_stat[3]);
    } else if (s_stat[2]) {
      atomicAdd(&ctr[C_CHANGED2], (unsigned long long)s_stat[2]);
    }
  }
  __syncthreads();
  uint64_t* dst = wout + s_base + off;
#pragma unroll
  for (int j = 0; j < 2 * PITEMS; j++)
    if (j < (int)nout) dst[j] = outw[j];
}

void launch_partition_apply(bool first, bool sorted, const uint64_t* win, const uint32_t* qin,
                            uint64_t n, const uint32_t* segA, const uint32_t* segB,
                            uint64_t* wout, uint32_t* label, uint64_t* ctr, cudaStream_t st) {
  (void)sorted;
  if (!n) return;
  unsigned g = (unsigned)((n + PTILE - 1) / PTILE);
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  if (first)
    k_partition_apply<true><<<g, BLOCK, 0, st>>>(win, qin, n, segA, segB, wout, label, c);
  else
    k_partition_apply<false><<<g, BLOCK, 0, st>>>(win, qin, n, segA, segB, wout, label, c);
}

}  // namespace sv
}  // namespace cc
