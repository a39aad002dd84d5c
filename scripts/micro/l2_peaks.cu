// Microbenchmark: the measured ceilings of random 4-byte L2 requests on this B200, the
// denominators of the "l2" roofline fractions bench.py reports for the kernels whose bound is
// the L2 request rate rather than HBM bandwidth (the degree count of Alg. 2 line 2 and the BFS
// levels: DESIGN.md §5.1, §5.3).
//
//   red_hash   : red.global.add.u32 at hashed (uniform random) slots of a T-slot table,
//                indices computed in registers (no memory stream): the pure reduction rate
//   red_stream : the same increments, the slot ids read from a streamed u32 array (the shape
//                of k_degree: one id stream, one increment per id)
//   ld_hash    : random 4-byte gathers (ld.global) from a T-slot table, summed in registers
//   atoms_hash : shared-memory atomicAdd at hashed slots of a 8 K-slot table (reference)
// T = 2^16 .. 2^26 slots (256 KB .. 256 MB; L2 = 126 MB).  Best of 5, CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_peaks l2_peaks.cu && ./l2_peaks
// Output: one JSON object (ops per second per kernel and table size).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return (uint32_t)x;
}

constexpr int OPS = 16;  // ops per thread per loop trip

__global__ void k_red_hash(uint32_t* __restrict__ tab, uint32_t mask, uint64_t trips, uint64_t seed) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (uint64_t k = 0; k < trips; k++) {
#pragma unroll
    for (int j = 0; j < OPS; j++) {
      const uint32_t h = hash32(seed + (t * trips + k) * OPS + j) & mask;
      asm volatile("red.global.add.u32 [%0], 1;" ::"l"(tab + h) : "memory");
    }
  }
}

__global__ void k_red_stream(const uint4* __restrict__ ids, uint64_t n4, uint32_t* __restrict__ tab) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(ids + i));
    asm volatile("red.global.add.u32 [%0], 1;" ::"l"(tab + v.x) : "memory");
    asm volatile("red.global.add.u32 [%0], 1;" ::"l"(tab + v.y) : "memory");
    asm volatile("red.global.add.u32 [%0], 1;" ::"l"(tab + v.z) : "memory");
    asm volatile("red.global.add.u32 [%0], 1;" ::"l"(tab + v.w) : "memory");
  }
}

__global__ void k_ld_hash(const uint32_t* __restrict__ tab, uint32_t mask, uint64_t trips, uint64_t seed,
                          uint32_t* out) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (uint64_t k = 0; k < trips; k++) {
#pragma unroll
    for (int j = 0; j < OPS; j++) acc += tab[hash32(seed + (t * trips + k) * OPS + j) & mask];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_atoms_hash(uint32_t mask, uint64_t trips, uint64_t seed, uint32_t* out) {
  __shared__ uint32_t s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (uint64_t k = 0; k < trips; k++) {
#pragma unroll
    for (int j = 0; j < OPS; j++) atomicAdd(&s[hash32(seed + (t * trips + k) * OPS + j) & 8191u], 1u);
  }
  __syncthreads();
  if (s[threadIdx.x] == 0x12345678u) out[0] = 1;
}

__global__ void k_fill_ids(uint32_t* ids, uint64_t n, uint32_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    ids[i] = hash32(i * 0x9E3779B97F4A7C15ULL + 7) & mask;
}

template <class F>
static float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const int threads = 256, blocks = sms * 8;
  const uint64_t nthreads = (uint64_t)threads * blocks;
  const uint64_t trips = 64;                      // 16 ops x 64 trips per thread
  const double nops = (double)nthreads * trips * OPS;
  uint32_t *tab, *out, *ids;
  const uint64_t nid = 1ull << 29;  // 2 GB id stream (> L2)
  cudaMalloc(&tab, sizeof(uint32_t) << 26);
  cudaMalloc(&out, 64);
  cudaMalloc(&ids, sizeof(uint32_t) * nid);
  cudaMemset(tab, 0, sizeof(uint32_t) << 26);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"ops_per_launch\": %.0f, \"results\": [\n", p.name,
         sms, p.l2CacheSize, nops);
  bool first = true;
  for (int lg = 16; lg <= 26; lg += 2) {
    const uint32_t mask = (1u << lg) - 1;
    const float t_red = best_ms([&] { k_red_hash<<<blocks, threads>>>(tab, mask, trips, 1234); });
    const float t_ld = best_ms([&] { k_ld_hash<<<blocks, threads>>>(tab, mask, trips, 99, out); });
    k_fill_ids<<<sms * 16, 256>>>(ids, nid, mask);
    const float t_rs = best_ms([&] { k_red_stream<<<sms * 16, 256>>>((const uint4*)ids, nid / 4, tab); });
    printf("%s  {\"table_log2\": %d, \"table_MB\": %.1f, \"red_hash_Gops\": %.1f, \"ld_hash_Gops\": %.1f, "
           "\"red_stream_Gops\": %.1f}",
           first ? "" : ",\n", lg, (4.0 * (1u << lg)) / 1e6, nops / t_red / 1e6, nops / t_ld / 1e6,
           (double)nid / t_rs / 1e6);
    first = false;
  }
  const float t_s = best_ms([&] { k_atoms_hash<<<blocks, threads>>>(8191u, trips, 5, out); });
  // the k_degree shape with the 2^24-slot table marked persisting in L2 (access policy window)
  int maxp = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  float t_pers = 0;
  {
    const uint32_t mask = (1u << 24) - 1;
    k_fill_ids<<<sms * 16, 256>>>(ids, nid, mask);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp);
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = tab;
    a.accessPolicyWindow.num_bytes = sizeof(uint32_t) << 24;
    a.accessPolicyWindow.hitRatio = 1.0f;
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
    t_pers = best_ms([&] { k_red_stream<<<sms * 16, 256, 0, st>>>((const uint4*)ids, nid / 4, tab); });
    cudaStreamSynchronize(st);
  }
  printf("\n], \"atoms_hash_8K_Gops\": %.1f, \"max_persisting_l2_bytes\": %d, "
         "\"red_stream_2p24_persisting_Gops\": %.1f}\n", nops / t_s / 1e6, maxp, (double)nid / t_pers / 1e6);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "cuda error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
