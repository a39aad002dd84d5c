// csr.cuh -- launchers of the r-stationary SV engine (sv_csr.cu).
#pragma once
#include "scan.cuh"

namespace cc {
namespace csr {

// CSR build (counting regroup by r): off[v] / cur[v] from degrees; ctr[C_VT_OUT] = A_0.
int group_shift(uint64_t n, uint64_t tuples);
void build(const uint2* edges, uint64_t m, const uint32_t* deg, const uint32_t* vis, uint64_t n,
           uint32_t* off, uint32_t* cur, uint32_t* garc, int gshift, scan::State& ss, uint64_t* ctr,
           cudaStream_t st);
// R fill, vertex tuples, and the two-level arc scatter (bucket by vertex group, then rows).
// tmp: 2m uint2 scratch; longlist: n uint32 scratch; garc/gcur: 1024 entries.
void fill(const uint2* edges, uint64_t m, const uint32_t* off, uint32_t* cur, uint64_t n, uint64_t A,
          uint32_t* R, uint32_t* P, const uint32_t* garc, int gshift, uint64_t* gcur, uint2* tmp,
          uint32_t* longlist, uint64_t* nlong, cudaStream_t st);
void vpass(bool with_pc, const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* U, uint32_t* NP,
           cudaStream_t st);
void ppass(bool first, const uint32_t* R, const uint32_t* P, uint64_t A, const uint32_t* U,
           const uint32_t* NP, const uint32_t* TB, uint32_t* PMIN, uint32_t* NCP, cudaStream_t st);
void temps(const uint32_t* TB, uint64_t n, const uint32_t* U, uint32_t* PMIN, cudaStream_t st);
void pscan(bool first, const uint32_t* PMIN, const uint32_t* NCP, uint64_t n, uint32_t* TB,
           uint64_t* ctr, cudaStream_t st);
// in place: completed partitions' tuples become DEAD, survivors p <- p_min; ctr[C_OUT] += live
void papply1(const uint32_t* R, uint32_t* P, uint64_t A, const uint32_t* PMIN, const uint32_t* NCP,
             uint32_t* label, uint64_t* ctr, cudaStream_t st);
// ordered compaction of live tuples (R order kept); output count = live count
void compact(const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* R2, uint32_t* P2,
             scan::State& ss, cudaStream_t st);
void papply2(uint32_t* P, uint64_t A, const uint32_t* PMIN, cudaStream_t st);

}  // namespace csr
}  // namespace cc
