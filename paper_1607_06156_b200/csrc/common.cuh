// common.cuh -- shared device helpers for libcc (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CC_DEVI __device__ __forceinline__

namespace cc {

// Tuple word layout (SURVEY.md §8(a) "Per-iteration SV layout detail").
// Ids are < 2^30.  The 64-bit word carries the sort key in its high 32 bits and the other
// id plus flags in the low 32 bits:
//   by-r word : hi = r (vertex),    lo = p | VT<<31 | TMP<<30
//   by-p word : hi = p (partition), lo = r | VT<<31 | TMP<<30,  q word = q | PC<<31
constexpr uint32_t ID_MASK = 0x3FFFFFFFu;
constexpr uint32_t F_VT = 0x80000000u;   // vertex tuple <x,_,x>
constexpr uint32_t F_TMP = 0x40000000u;  // temporary tuple <p_min,_,p_min>_tmp
constexpr uint32_t F_PC = 0x80000000u;   // potentially completed, |M(u)| = 1
constexpr uint32_t FLAGS = F_VT | F_TMP;

CC_DEVI uint32_t hi32(uint64_t w) { return (uint32_t)(w >> 32); }
CC_DEVI uint32_t lo32(uint64_t w) { return (uint32_t)w; }
CC_DEVI uint64_t mk(uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | lo; }

CC_DEVI uint32_t lane_id() { return threadIdx.x & 31; }
CC_DEVI uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

CC_DEVI uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
CC_DEVI void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// streaming (evict-first) 128-bit loads for read-once tuple streams
CC_DEVI uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 256-bit streaming load (sm_100: LDG.E.256): two uint4 from 32 bytes (p 32-byte aligned)
CC_DEVI void ldg_stream_v8(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.cs.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
// 256-bit store (sm_100: STG.E.256): 32 bytes, one full sector per request (p 32-byte aligned)
CC_DEVI void st_v8(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

template <typename T>
CC_DEVI T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide exclusive scan of one u32 per thread; returns exclusive prefix, *total set.
template <int BLOCK>
CC_DEVI uint32_t block_excl_scan(uint32_t v, uint32_t* smem /*>= BLOCK/32+1*/, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = (lane < BLOCK / 32) ? smem[lane] : 0;
    uint32_t t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < BLOCK / 32) smem[lane] = t - s;
    if (lane == BLOCK / 32 - 1) smem[BLOCK / 32] = t;
  }
  __syncthreads();
  uint32_t r = smem[wid] + x - v;
  *total = smem[BLOCK / 32];
  __syncthreads();
  return r;
}

}  // namespace cc
