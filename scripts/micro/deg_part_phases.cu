// Microbenchmark: the phases of the bucketed degree count's partition pass (graph.cu
// k_deg_part) in isolation, on 2^31 uniform random u32 ids < 2^26 (8.6 GB, C4's endpoint count):
//   V0 stream    : 16-byte streaming loads only (the edge list read)
//   V1 +insert   : + one shared atomicAdd and one u16 store per id into 2048 rings of 32
//   V2 +flush    : + the per-round write-out scan (rings >= 16 entries), no global stores
//   V3 +write    : + the 32-byte group stores to per-bucket regions (the full kernel)
// One block of 1024 threads per SM, 16 ids per thread per round.  Best of 3, CUDA events.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint4 ldcs(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__global__ void k_fill(uint32_t* ids, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ULL + 12345;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33;
    ids[i] = (uint32_t)x & ((1u << 26) - 1);
  }
}
template <int V>
__global__ void __launch_bounds__(1024, 1) k_part(const uint4* __restrict__ e, uint32_t rounds, uint16_t* reg,
                                                  uint32_t C, uint32_t* cur, uint32_t* out, uint32_t S) {
  // S sub-regions per bucket (block k uses sub-region k % S, capacity C / S)
  extern __shared__ __align__(16) uint32_t dsm[];
  uint32_t* s_w = dsm;
  uint16_t* s_row = reinterpret_cast<uint16_t*>(dsm + 2048);
  for (int b = threadIdx.x; b < 2048; b += 1024) s_w[b] = 0;
  uint32_t opos[2] = {0, 0};
  const uint32_t sub = blockIdx.x % S, Cs = (C / S) & ~15u;
  if (V == 8) { opos[0] = atomicAdd(&cur[threadIdx.x], 16u); opos[1] = atomicAdd(&cur[threadIdx.x + 1024], 16u); }
  else if (V >= 3) { opos[0] = atomicAdd(&cur[threadIdx.x * S + sub], 16u); opos[1] = atomicAdd(&cur[(threadIdx.x + 1024) * S + sub], 16u); }
  __syncthreads();
  uint32_t acc = 0;
  for (uint32_t r = blockIdx.x; r < rounds; r += gridDim.x) {
    const uint4* p = e + (uint64_t)r * 4096 + threadIdx.x;
    uint4 x[4];
#pragma unroll
    for (int j = 0; j < 4; j++) x[j] = ldcs(p + j * 1024);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint32_t v[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
      if (V == 0) { acc += v[0] ^ v[1] ^ v[2] ^ v[3]; continue; }
      uint32_t old[4];
#pragma unroll
      for (int h = 0; h < 4; h++) old[h] = atomicAdd(&s_w[v[h] >> 15], 1u);
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const uint32_t b = v[h] >> 15, w = old[h] & 0xFFFFu;
        if (w - (old[h] >> 16) < 32) s_row[b * 32 + ((w & 31u) ^ ((b << 2) & 24u))] = (uint16_t)(v[h] & 0x7FFF);
        else acc++;
      }
    }
    if (V >= 1) {
      __syncthreads();
      if (V == 1) {
        for (int b = threadIdx.x; b < 2048; b += 1024) { uint32_t wd = s_w[b]; uint32_t w = wd & 0xFFFF, f = wd >> 16;
          if (w - f >= 16) { f += 16; if (w - f > 32) w = f + 16; uint32_t base = f & ~31u; s_w[b] = ((f - base) << 16) | (w - base); } }
      } else {
#pragma unroll
        for (int i = 0; i < 2; i++) {
          const uint32_t b = threadIdx.x + i * 1024;
          const uint32_t wd = s_w[b];
          uint32_t w = wd & 0xFFFFu, f = wd >> 16;
          if (w - f < 16) continue;
          if (w - f > 32) w = f + 32;
          const uint32_t c0 = f & 16u;
          const uint4* row = reinterpret_cast<const uint4*>(s_row + b * 32);
          const uint4 r0 = row[((c0 & 31u) ^ ((b << 2) & 24u)) >> 3], r1 = row[(((c0 + 8) & 31u) ^ ((b << 2) & 24u)) >> 3];
          f += 16;
          const uint32_t base = f & ~31u;
          s_w[b] = ((f - base) << 16) | (w - base);
          if (V == 2) { acc += r0.x ^ r1.w; continue; }
          if (V == 6) {  // same stores, sequential coalesced addresses
            uint4* d = reinterpret_cast<uint4*>(reg + (((uint64_t)r * 2048 + i * 1024 + threadIdx.x) * 16) % ((uint64_t)2048 * C));
            d[0] = r0; d[1] = r1;
          } else if (V == 7) {  // scattered over 2048 streams, but every stream wraps in a 16 K-entry window
            uint4* d = reinterpret_cast<uint4*>(reg + (uint64_t)b * 16384 + (opos[i] & 16383u));
            d[0] = r0; d[1] = r1;
          } else if (V == 8) {  // shared stream per bucket, epoch-interleaved: chunk Q=S entries of every bucket per epoch
            const uint32_t Q = S;
            uint4* d = reinterpret_cast<uint4*>(reg + ((uint64_t)(opos[i] / Q) * 2048 + b) * Q + (opos[i] % Q));
            if (opos[i] < C) { d[0] = r0; d[1] = r1; }
          } else if (V != 5 && opos[i] < Cs) { uint4* d = reinterpret_cast<uint4*>(reg + (uint64_t)(b * S + sub) * Cs + opos[i]); d[0] = r0; d[1] = r1; }
          if (V == 5) acc += r0.x ^ r1.w;
          if (V == 4 || V == 6 || V == 7) opos[i] += 16;  // private positions, no atomic
          else if (V == 8) opos[i] = atomicAdd(&cur[b], 16u);
          else opos[i] = atomicAdd(&cur[b * S + sub], 16u);
        }
      }
      __syncthreads();
    }
  }
  if (acc == 0x9999999u) out[0] = acc;
}
int main() {
  const uint64_t nid = 1ull << 31;  // 8 GB of ids
  uint32_t *ids, *cur, *out;
  uint16_t* reg;
  const uint32_t C = (uint32_t)(4 * (nid / 2048));
  cudaMalloc(&ids, nid * 4); cudaMalloc(&cur, 2048 * 4 * 148); cudaMalloc(&out, 64);
  cudaMalloc(&reg, (uint64_t)2048 * C * 2);
  k_fill<<<148 * 16, 256>>>(ids, nid);
  const int smem = 2048 * 4 + 2048 * 64;
  cudaFuncSetAttribute(k_part<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const uint32_t rounds = (uint32_t)(nid / 16384);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](int v, uint32_t S = 1) {
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
      cudaMemset(cur, 0, 2048 * 4 * 148);
      cudaEventRecord(a);
      if (v == 0) k_part<0><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 1) k_part<1><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 2) k_part<2><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 3) k_part<3><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 4) k_part<4><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 5) k_part<5><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 6) k_part<6><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 7) k_part<7><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      if (v == 8) k_part<8><<<148, 1024, smem>>>((const uint4*)ids, rounds, reg, C, cur, out, S);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    return best;
  };
  printf("{\"ids\": %llu, \"V0_stream_ms\": %.3f, \"V1_insert_ms\": %.3f, \"V2_flushscan_ms\": %.3f, \"V3_write_ms\": {",
         (unsigned long long)nid, run(0), run(1), run(2));
  for (uint32_t S : {1u, 2u, 4u, 8u, 16u, 37u, 148u}) printf("%s\"S%u\": %.3f", S == 1 ? "" : ", ", S, run(3, S));
  printf("}, \"V4_write_noatomic_S148\": %.3f, \"V5_atomic_nowrite_S1\": %.3f, \"V6_seqwrite\": %.3f, \"V7_scatter_64MB\": %.3f}\n",
         run(4, 148), run(5, 1), run(6, 1), run(7, 1));
  for (uint32_t Q : {64u, 256u, 1024u, 4096u, 16384u}) printf("V8_epoch_Q%u: %.3f\n", Q, run(8, Q));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
