// bfs.cuh -- direction-optimising BFS on the CSR rows (bfs.cu).
#pragma once
#include "common.cuh"

namespace cc {
namespace bfs {

// counters of one level (u64, caller-zeroed)
enum Ctr : int { C_NEXT = 0, C_NEXT_ARCS = 1, C_NUM = 2 };

// One level from the frontier (list[0, nf) and bitmap F): newly visited vertices are set in V
// and X, appended to `next`; ctr[C_NEXT] = their number, ctr[C_NEXT_ARCS] = their arcs.
// bottom_up: scan the rows of unvisited vertices (F read); else expand the list (top-down).
void level(bool bottom_up, const uint32_t* off, const uint32_t* P, const uint32_t* deg, uint64_t n,
           const uint32_t* list, uint64_t nf, const uint32_t* F, uint32_t* V, uint32_t* X, uint32_t* next,
           uint64_t* ctr, cudaStream_t st);
// Edges whose first endpoint is not in V (Alg. 2 line 10); *cnt += kept (caller-zeroed).
void filter(const uint2* edges, uint64_t m, const uint32_t* V, uint2* out, uint64_t* cnt,
            cudaStream_t st);

}  // namespace bfs
}  // namespace cc
