// bfs.cu -- direction-optimising BFS peel on the CSR rows (Alg. 2 lines 7-8).
//
// The giant component is peeled by one BFS from the max-degree root (C13).  The rows built
// for SV double as the adjacency: row u = [off[u], off[u+1]) holds the vertex tuple first,
// then one tuple <x,_,u> per arc, whose p = x is a neighbour of u.  Each level
// runs top-down or bottom-up (Beamer's rule on arc counts): top-down expands the frontier
// list and claims unvisited neighbours; bottom-up scans the rows of unvisited vertices and
// stops at the first neighbour in the frontier bitmap, which on small-world graphs touches a
// small fraction of the arcs.  Both directions emit the next frontier as a bitmap and a list
// and accumulate its arc count.  The paper's CombBLAS 2-D BFS is replaced.
#include <algorithm>

#include "bfs.cuh"

namespace cc {
namespace bfs {

constexpr int B = 256;

CC_DEVI bool bit(const uint32_t* bm, uint32_t v) { return (bm[v >> 5] >> (v & 31)) & 1u; }

// append v to the next frontier (warp-aggregated cursor) and count its arcs
CC_DEVI void emit(bool take, uint32_t v, uint32_t dv, uint32_t* next, unsigned long long* ctr) {
  const uint32_t mask = __ballot_sync(0xffffffffu, take);
  if (!mask) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  uint32_t arcs = take ? dv : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) arcs += __shfl_xor_sync(0xffffffffu, arcs, o);
  if (lane == leader) {
    base = atomicAdd(&ctr[C_NEXT], (unsigned long long)__popc(mask));
    atomicAdd(&ctr[C_NEXT_ARCS], (unsigned long long)arcs);
  }
  base = __shfl_sync(0xffffffffu, base, leader);
  if (take) next[base + __popc(mask & ((1u << lane) - 1u))] = v;
}

// claim x (unvisited -> visited, frontier bit) ; true if this thread won it
CC_DEVI bool claim(uint32_t* V, uint32_t* X, uint32_t x) {
  const uint32_t b = 1u << (x & 31);
  if (V[x >> 5] & b) return false;
  if (atomicOr(&V[x >> 5], b) & b) return false;
  atomicOr(&X[x >> 5], b);
  return true;
}

// top-down, one (large) frontier vertex: the whole grid walks its row
__global__ void k_td_one(const uint32_t* __restrict__ off, const uint32_t* __restrict__ P,
                         const uint32_t* __restrict__ deg, const uint32_t* __restrict__ list,
                         uint32_t* V, uint32_t* X, uint32_t* next, unsigned long long* ctr) {
  const uint32_t u = list[0];
  const uint32_t a = off[u] + 1, b = off[u + 1];
  const uint64_t stride = (uint64_t)gridDim.x * B;
  for (uint64_t i0 = a + blockIdx.x * (uint64_t)B; i0 < b; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    bool take = false;
    uint32_t x = 0;
    if (i < b) {
      x = P[i];
      take = claim(V, X, x);
    }
    emit(take, x, take ? deg[x] : 0u, next, ctr);
  }
}

// top-down: a warp per frontier vertex, lanes over its arcs
__global__ void k_td(const uint32_t* __restrict__ off, const uint32_t* __restrict__ P,
                     const uint32_t* __restrict__ deg, const uint32_t* __restrict__ list, uint64_t nf,
                     uint32_t* V, uint32_t* X, uint32_t* next, unsigned long long* ctr) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * B) >> 5;
  for (uint64_t f = (blockIdx.x * (uint64_t)B + threadIdx.x) >> 5; f < nf; f += warps) {
    const uint32_t u = list[f];
    const uint32_t a = off[u] + 1, b = off[u + 1];
    for (uint32_t i0 = a; i0 < b; i0 += 32) {
      const uint32_t i = i0 + lane;
      bool take = false;
      uint32_t x = 0;
      if (i < b) {
        x = P[i];
        take = claim(V, X, x);
      }
      emit(take, x, take ? deg[x] : 0u, next, ctr);
    }
  }
}

// bottom-up: a thread per unvisited present vertex; stop at the first frontier neighbour
__global__ void k_bu(const uint32_t* __restrict__ off, const uint32_t* __restrict__ P,
                     const uint32_t* __restrict__ deg, uint64_t n, const uint32_t* __restrict__ F,
                     uint32_t* V, uint32_t* X, uint32_t* next, unsigned long long* ctr) {
  const uint64_t stride = (uint64_t)gridDim.x * B;
  for (uint64_t u0 = blockIdx.x * (uint64_t)B; u0 < n; u0 += stride) {
    const uint64_t u = u0 + threadIdx.x;
    bool take = false;
    uint32_t du = 0;
    if (u < n && !bit(V, (uint32_t)u)) {
      du = deg[u];
      if (du) {
        const uint32_t a = off[u] + 1, b = off[u + 1];
        for (uint32_t i = a; i < b; i++)
          if (bit(F, P[i])) { take = true; break; }
      }
    }
    if (take) {  // u is only ever written by this thread, other bits of the word by others
      atomicOr(&V[u >> 5], 1u << (u & 31));
      atomicOr(&X[u >> 5], 1u << (u & 31));
    }
    emit(take, (uint32_t)u, du, next, ctr);
  }
}

// Filter (Alg. 2 lines 10-11): E <- E \ {(u,v) | u in VI}; both arcs of an edge are
// represented by it, so keeping edges with an unvisited first endpoint is exact (C15).
__global__ void __launch_bounds__(B) k_filter_v(const uint2* __restrict__ e, uint64_t m,
                                                const uint32_t* __restrict__ V,
                                                uint2* __restrict__ out, unsigned long long* cnt) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ unsigned long long s_base;
  for (uint64_t b0 = blockIdx.x * (uint64_t)B * 4; b0 < m; b0 += (uint64_t)gridDim.x * B * 4) {
    uint2 x[4];
    uint32_t keep = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint64_t i = b0 + (uint64_t)j * B + threadIdx.x;
      x[j] = i < m ? e[i] : make_uint2(0, 0);
      if (i < m && !bit(V, x[j].x)) keep |= 1u << j;
    }
    uint32_t tot;
    const uint32_t o = block_excl_scan<B>(__popc(keep), s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(cnt, (unsigned long long)tot) : 0ull;
    __syncthreads();
    uint2* dst = out + s_base + o;
#pragma unroll
    for (int j = 0; j < 4; j++)
      if ((keep >> j) & 1u) *dst++ = x[j];
    __syncthreads();
  }
}

static unsigned gsz(uint64_t work, unsigned cap) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + B - 1) / B, cap));
}

void level(bool bottom_up, const uint32_t* off, const uint32_t* P, const uint32_t* deg, uint64_t n,
           const uint32_t* list, uint64_t nf, const uint32_t* F, uint32_t* V, uint32_t* X, uint32_t* next,
           uint64_t* ctr, cudaStream_t st) {
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  if (bottom_up) {
    k_bu<<<gsz(n, 148 * 16), B, 0, st>>>(off, P, deg, n, F, V, X, next, c);
  } else if (nf == 1) {
    k_td_one<<<148 * 8, B, 0, st>>>(off, P, deg, list, V, X, next, c);
  } else if (nf) {
    k_td<<<gsz(nf * 32, 148 * 16), B, 0, st>>>(off, P, deg, list, nf, V, X, next, c);
  }
}

void filter(const uint2* edges, uint64_t m, const uint32_t* V, uint2* out, uint64_t* cnt,
            cudaStream_t st) {
  if (m)
    k_filter_v<<<gsz(m / 4 + 1, 148 * 8), B, 0, st>>>(edges, m, V, out,
                                                       reinterpret_cast<unsigned long long*>(cnt));
}

}  // namespace bfs
}  // namespace cc
