// graph.cu -- degree distribution (Alg. 2 line 2), BFS peel (lines 7-8) and filter
// (lines 10-11) kernels.  PAPER.md:249-279.
#include "graph.cuh"

#include <algorithm>

namespace cc {
namespace graph {

constexpr int BLOCK = 256;

static unsigned grid_for(uint64_t work, unsigned cap) {
  uint64_t g = (work + BLOCK - 1) / BLOCK;
  if (g < 1) g = 1;
  return (unsigned)std::min<uint64_t>(g, cap);
}

// ---------------------------------------------------------------- input validation
__global__ void k_validate(const uint2* __restrict__ e, uint64_t m, uint64_t n,
                           unsigned long long* gctr) {
  bool bad = false;
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * BLOCK) {
    uint2 x = e[i];
    bad |= (x.x >= n) | (x.y >= n);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&gctr[G_ERR], 1ull);
}
void launch_validate(const uint2* edges, uint64_t m, uint64_t n, uint64_t* gctr, cudaStream_t st) {
  if (!m) return;
  k_validate<<<grid_for(m, 148 * 8), BLOCK, 0, st>>>(edges, m, n,
                                                       reinterpret_cast<unsigned long long*>(gctr));
}

// ---------------------------------------------------------------- degrees
// Degree of v = number of arcs with source v, each undirected edge being the two arcs
// (u,v),(v,u); a self-loop adds 2.  Ids are dense, so a
// counting increment replaces the paper's sort by source.
__global__ void k_degree(const uint2* __restrict__ e, uint64_t m, uint32_t* __restrict__ deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * BLOCK) {
    uint2 x = e[i];
    atomicAdd(&deg[x.x], 1u);
    atomicAdd(&deg[x.y], 1u);
  }
}
void launch_degree(const uint2* edges, uint64_t m, uint32_t* deg, cudaStream_t st) {
  if (!m) return;
  k_degree<<<grid_for(m, 148 * 16), BLOCK, 0, st>>>(edges, m, deg);
}

// Degree distribution D[d] = #{v : deg(v) = d}, d >= 1 (C10), plus n_present and the
// (max degree, smallest argmax) key used for the BFS root (C13).  Shared-memory bins for
// small degrees (where all the mass is), global bins up to 2^20, a tail list beyond.
constexpr int SBINS = 2048;
__global__ void __launch_bounds__(BLOCK) k_deg_hist(const uint32_t* __restrict__ deg, uint64_t n,
                                                    uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ tail,
                                                    unsigned long long* gctr) {
  __shared__ uint32_t sh[SBINS];
  for (int i = threadIdx.x; i < SBINS; i += BLOCK) sh[i] = 0;
  __syncthreads();
  uint32_t npres = 0;
  unsigned long long best = 0;
  const uint32_t lt = lanemask_lt();
  for (uint64_t base = blockIdx.x * (uint64_t)BLOCK; base < n; base += (uint64_t)gridDim.x * BLOCK) {
    uint64_t v = base + threadIdx.x;
    uint32_t d = v < n ? deg[v] : 0u;
    if (d) {
      npres++;
      unsigned long long key = ((unsigned long long)d << 32) | (0xFFFFFFFFu - (uint32_t)v);
      best = key > best ? key : best;
    }
    uint32_t bin = (d && d < SBINS) ? d : (SBINS + (threadIdx.x & 31));
    uint32_t peers = __match_any_sync(0xffffffffu, bin);
    if (bin < SBINS && (peers & lt) == 0) atomicAdd(&sh[bin], (uint32_t)__popc(peers));
    if (d >= SBINS) {
      if (d < HIST_DENSE) atomicAdd(&hist[d], 1u);
      else {
        unsigned long long pos = atomicAdd(&gctr[G_TAIL], 1ull);
        if (pos < TAIL_CAP) tail[pos] = d;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SBINS; i += BLOCK)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  npres = warp_sum(npres);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
  }
  if ((threadIdx.x & 31) == 0) {
    if (npres) atomicAdd(&gctr[G_NPRESENT], (unsigned long long)npres);
    if (best) atomicMax(&gctr[G_MAXKEY], best);
  }
}
void launch_deg_hist(const uint32_t* deg, uint64_t n, uint32_t* hist, uint32_t* tail,
                     uint64_t* gctr, cudaStream_t st) {
  if (!n) return;
  k_deg_hist<<<grid_for(n, 148 * 4), BLOCK, 0, st>>>(deg, n, hist, tail,
                                                       reinterpret_cast<unsigned long long*>(gctr));
}

// ---------------------------------------------------------------- BFS peel
// One level of a level-synchronous BFS from the root (Alg. 2 lines 7-8)
// over the edge list, with n-bit frontier / visited / next bitmaps (L2 resident for the
// configs here).  Every live edge is streamed once per level; an endpoint in the
// frontier claims its unvisited neighbour with atomicOr on the visited bitmap, so each
// vertex enters `next` exactly once.  (edge-streaming bitmap BFS.)
CC_DEVI bool bit(const uint32_t* bm, uint32_t v) { return (__ldg(&bm[v >> 5]) >> (v & 31)) & 1u; }
CC_DEVI bool claim(uint32_t* visited, uint32_t* next, uint32_t v) {
  uint32_t mask = 1u << (v & 31);
  if (visited[v >> 5] & mask) return false;  // cheap pre-check (relaxed read)
  uint32_t old = atomicOr(&visited[v >> 5], mask);
  if (old & mask) return false;
  atomicOr(&next[v >> 5], mask);
  return true;
}
__global__ void __launch_bounds__(BLOCK) k_bfs_level(const uint4* __restrict__ e2, uint64_t m,
                                                     const uint32_t* __restrict__ frontier,
                                                     uint32_t* visited, uint32_t* next,
                                                     unsigned long long* gctr) {
  uint32_t found = 0;
  const uint64_t npair = m >> 1;
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i <= npair;
       i += (uint64_t)gridDim.x * BLOCK) {
    uint32_t a[2], b[2];
    int cnt = 0;
    if (i < npair) {
      uint4 x = ldg_stream(&e2[i]);
      a[0] = x.x; b[0] = x.y; a[1] = x.z; b[1] = x.w; cnt = 2;
    } else if (m & 1) {
      uint2 x = reinterpret_cast<const uint2*>(e2)[m - 1];
      a[0] = x.x; b[0] = x.y; cnt = 1;
    }
    for (int j = 0; j < cnt; j++) {
      if (bit(frontier, a[j])) found += claim(visited, next, b[j]);
      if (bit(frontier, b[j])) found += claim(visited, next, a[j]);
    }
  }
  found = warp_sum(found);
  if ((threadIdx.x & 31) == 0 && found) atomicAdd(&gctr[G_NEWVIS], (unsigned long long)found);
}
void launch_bfs_level(const uint2* edges, uint64_t m, const uint32_t* frontier, uint32_t* visited,
                      uint32_t* next, uint64_t* gctr, cudaStream_t st) {
  if (!m) return;
  k_bfs_level<<<grid_for((m >> 1) + 1, 148 * 16), BLOCK, 0, st>>>(
      reinterpret_cast<const uint4*>(edges), m, frontier, visited, next,
      reinterpret_cast<unsigned long long*>(gctr));
}

// Filter (Alg. 2 lines 10-11): E <- E \ {(u,v) | u in VI}.  Both arcs of
// an edge are stored, so keeping edges with an unvisited first endpoint removes both
// directions (C15).  Block-aggregated compaction.
__global__ void __launch_bounds__(BLOCK) k_filter(const uint2* __restrict__ e, uint64_t m,
                                                  const uint32_t* __restrict__ visited,
                                                  uint2* __restrict__ out,
                                                  unsigned long long* gctr) {
  __shared__ uint32_t s_scan[BLOCK / 32 + 1];
  __shared__ unsigned long long s_base;
  for (uint64_t b0 = blockIdx.x * (uint64_t)BLOCK; b0 < m; b0 += (uint64_t)gridDim.x * BLOCK) {
    uint64_t i = b0 + threadIdx.x;
    uint2 x = make_uint2(0, 0);
    uint32_t keep = 0;
    if (i < m) {
      x = e[i];
      keep = !bit(visited, x.x);
    }
    uint32_t tot;
    uint32_t off = block_excl_scan<BLOCK>(keep, s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(&gctr[G_REMAIN], (unsigned long long)tot) : 0ull;
    __syncthreads();
    if (keep) out[s_base + off] = x;
    __syncthreads();
  }
}
void launch_filter(const uint2* edges, uint64_t m, const uint32_t* visited, uint2* out,
                   uint64_t* gctr, cudaStream_t st) {
  if (!m) return;
  k_filter<<<grid_for(m, 148 * 8), BLOCK, 0, st>>>(edges, m, visited, out,
                                                     reinterpret_cast<unsigned long long*>(gctr));
}

// L_bfs = min id in VI: first set bit of the visited bitmap.
__global__ void k_min_visited(const uint32_t* __restrict__ vis, uint64_t nwords,
                              unsigned long long* gctr) {
  for (uint64_t w = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; w < nwords;
       w += (uint64_t)gridDim.x * BLOCK) {
    uint32_t x = vis[w];
    if (x) {
      atomicMin(&gctr[G_MINVIS], (unsigned long long)(w * 32 + (__ffs(x) - 1)));
      return;
    }
  }
}
void launch_min_visited(const uint32_t* visited, uint64_t n, uint64_t* gctr, cudaStream_t st) {
  uint64_t nw = (n + 31) / 32;
  if (!nw) return;
  k_min_visited<<<grid_for(nw, 148 * 4), BLOCK, 0, st>>>(visited, nw,
                                                           reinterpret_cast<unsigned long long*>(gctr));
}

__global__ void k_bfs_labels(const uint32_t* __restrict__ vis, uint64_t n,
                             uint32_t* __restrict__ label, const unsigned long long* gctr) {
  const uint32_t L = (uint32_t)gctr[G_MINVIS];
  for (uint64_t v = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * BLOCK)
    if (bit(vis, (uint32_t)v)) label[v] = L;
}
void launch_bfs_labels(const uint32_t* visited, uint64_t n, uint32_t* label, uint64_t* gctr,
                       cudaStream_t st) {
  if (!n) return;
  k_bfs_labels<<<grid_for(n, 148 * 16), BLOCK, 0, st>>>(
      visited, n, label, reinterpret_cast<const unsigned long long*>(gctr));
}

}  // namespace graph
}  // namespace cc
