// Microbenchmark: cost of one same-address atomicAdd "ticket" per block (decoupled look-back
// tile ordering), vs blocks that do nothing.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ticket(unsigned* ctr, unsigned* out) {
  __shared__ unsigned s;
  if (threadIdx.x == 0) s = atomicAdd(ctr, 1u);
  __syncthreads();
  if (threadIdx.x == 0 && s == 0xFFFFFFFFu) out[0] = s;
}
__global__ void k_empty(unsigned* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0xFFFFFFFFu) out[0] = 1;
}
int main() {
  unsigned *ctr, *out;
  cudaMalloc(&ctr, 4); cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {8192, 32768, 131072}) {
    float t1 = 0, t2 = 0;
    for (int rep = 0; rep < 3; rep++) {
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(a); k_ticket<<<blocks, 256>>>(ctr, out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&t1, a, b);
      cudaEventRecord(a); k_empty<<<blocks, 256>>>(out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&t2, a, b);
    }
    printf("blocks %d: ticket %.1f us, empty %.1f us\n", blocks, t1 * 1e3, t2 * 1e3);
  }
  return 0;
}
