// sv.cuh -- kernels of the edge-tuple Shiloach-Vishkin iteration (Alg. 1)
#pragma once
#include "common.cuh"

namespace cc {
namespace sv {

// counters (u64) written by the partition passes; index into Ctx::d_ctr
enum Ctr : int {
  C_OUT = 0,        // output cursor of the compaction (survivors + temps)
  C_PARTITIONS,     // |P_i|
  C_COMPLETED,      // completed partitions
  C_CHANGED,        // p_min != p at pass 2
  C_TEMPS,          // temporaries emitted
  C_CHANGED2,       // p_min != p at pass 4
  C_HIDDEN_DEAD,    // csr engine: collapsed tuples of the rows that left in pass B (row collapse)
  C_TDIST,          // csr engine, iteration 0: distinct temporary targets p_min (set TB bits)
  C_SURVIVORS,      // non-temporary tuples kept
  C_VT_OUT,         // vertex-tuple cursor (init)
  C_ERR,            // error flags (range)
  C_NUM
};

enum SegMode : int { SEG_VMINMAX = 0, SEG_VMIN = 1, SEG_PMIN_NC = 2, SEG_PMIN = 3 };

void launch_init_labels(uint32_t* label, uint64_t n, cudaStream_t st);
// A_0 (Alg.1 lines 1-3): arcs at [0,2m), vertex tuples appended after.
void launch_init_tuples(const uint2* edges, uint64_t m, const uint32_t* deg,
                        const uint32_t* visited_bm, uint64_t n, uint64_t* w, uint64_t* ctr,
                        cudaStream_t st, uint64_t* launches);
void launch_seg_reduce(int mode, const uint64_t* w, const uint32_t* q, uint64_t n, uint32_t* segA,
                       uint32_t* segB, cudaStream_t st);
void launch_vertex_apply(bool with_pc, const uint64_t* win, uint64_t n, const uint32_t* segA,
                         const uint32_t* segB, uint64_t* wout, uint32_t* qout, cudaStream_t st);
void launch_partition_apply(bool first, bool sorted, const uint64_t* win, const uint32_t* qin,
                            uint64_t n, const uint32_t* segA, const uint32_t* segB,
                            uint64_t* wout, uint32_t* label, uint64_t* ctr, cudaStream_t st);

// direct-addressed bucket passes (sv_direct.cu)
void launch_direct_vmin(const uint64_t* w, uint64_t n, uint32_t* umin, cudaStream_t st);
void launch_direct_vpc(const uint64_t* w, uint64_t n, const uint32_t* umin, uint32_t* notpc,
                       cudaStream_t st);
void launch_direct_pmin(bool first, const uint64_t* w, uint64_t n, const uint32_t* umin,
                        const uint32_t* notpc, uint32_t* pmin, uint32_t* ncp, cudaStream_t st);
void launch_direct_papply(bool first, const uint64_t* w, uint64_t n, const uint32_t* pmin,
                          const uint32_t* ncp, uint32_t* headbm, uint64_t* wout, uint32_t* label,
                          uint64_t* ctr, cudaStream_t st);

}  // namespace sv
}  // namespace cc
