#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return (uint32_t)x;
}
template <int MODE>
__global__ void k(uint32_t mask, uint64_t trips, uint64_t seed, uint32_t* out) {
  __shared__ uint32_t s[8192];
  __shared__ uint16_t b[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (uint64_t kk = 0; kk < trips; kk++) {
    uint32_t h[8], r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) h[j] = hash32(seed + (t * trips + kk) * 8 + j) & mask;
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 8; j++) atomicAdd(&s[h[j]], 1u);
    } else if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = atomicAdd(&s[h[j]], 1u);
#pragma unroll
      for (int j = 0; j < 8; j++) acc += r[j];
    } else if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = atomicAdd(&s[h[j]], 1u);
#pragma unroll
      for (int j = 0; j < 8; j++) b[(h[j] * 4 + (r[j] & 3)) & 8191] = (uint16_t)h[j];
    } else if (MODE == 3) {
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = atomicInc(&s[h[j]], 0xFFFFFFFFu);
#pragma unroll
      for (int j = 0; j < 8; j++) acc += r[j];
    } else if (MODE == 4) {  // warp match-any aggregated
#pragma unroll
      for (int j = 0; j < 8; j++) {
        uint32_t peers = __match_any_sync(0xffffffffu, h[j]);
        int leader = __ffs(peers) - 1;
        uint32_t lt = peers & ((1u << (threadIdx.x & 31)) - 1);
        uint32_t base = 0;
        if ((threadIdx.x & 31) == leader) base = atomicAdd(&s[h[j]], __popc(peers));
        base = __shfl_sync(peers, base, leader);
        acc += base + __popc(lt);
      }
    }
  }
  __syncthreads();
  if (s[threadIdx.x] == 0x12345678u || acc == 0x12345u) out[0] = b[threadIdx.x];
}
template <class F> float best(F f) { cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float bst = 1e30;
  for (int r = 0; r < 5; r++) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < bst) bst = ms; } return bst; }
int main() {
  uint32_t* out; cudaMalloc(&out, 64);
  const int blocks = 148 * 4, threads = 512; const uint64_t trips = 256;
  const double nops = (double)blocks * threads * trips * 8;
  for (uint32_t mask : {2047u, 8191u}) {
    printf("mask %u: noret %.0f  ret %.0f  ret+sts16 %.0f  inc %.0f  match %.0f G/s\n", mask,
      nops / best([&]{ k<0><<<blocks, threads>>>(mask, trips, 1, out); }) / 1e6,
      nops / best([&]{ k<1><<<blocks, threads>>>(mask, trips, 1, out); }) / 1e6,
      nops / best([&]{ k<2><<<blocks, threads>>>(mask, trips, 1, out); }) / 1e6,
      nops / best([&]{ k<3><<<blocks, threads>>>(mask, trips, 1, out); }) / 1e6,
      nops / best([&]{ k<4><<<blocks, threads>>>(mask, trips, 1, out); }) / 1e6);
  }
  return cudaDeviceSynchronize() != cudaSuccess;
}
