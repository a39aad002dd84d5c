// graph.cuh -- prediction (degree distribution), BFS peel and filter kernels (Alg. 2).
#pragma once
#include "common.cuh"

namespace cc {
namespace graph {

constexpr uint32_t HIST_DENSE = 1u << 20;  // dense histogram bins [0, 2^20); larger -> tail list
constexpr uint32_t TAIL_CAP = 1u << 20;

// counters (u64) in the graph-stage counter block
enum GCtr : int {
  G_NPRESENT = 0,  // ids with degree >= 1
  G_MAXKEY,        // max over (deg<<32 | ~v): max degree, ties -> smallest id
  G_TAIL,          // number of degrees >= HIST_DENSE (tail list length)
  G_NEWVIS,        // BFS: newly visited in the current level
  G_REMAIN,        // filter output cursor
  G_MINVIS,        // min visited id
  G_ERR,           // input validation flags
  G_FARCS,         // BFS: arcs (full-graph degrees) of the vertices found in the current level
  G_GUESS,         // speculative root: max over a prefix of (count<<32 | ~v)
  G_SUBN,          // remainder renumbering: n' (distinct endpoints of the remainder)
  G_NUM
};

// speculative root level (graph.cu, k_deg_sample): on lists of >= SPEC_MIN_EDGES edges the
// degree pass guesses the root from a prefix of SPEC_SAMPLE_EDGES edges and runs the guess's
// level on the side.  S (2-bit state) and next are zeroed by the caller; the guess key lands
// in gctr[G_GUESS], the ids found in the next bitmap.
constexpr uint64_t SPEC_MIN_EDGES = 1ull << 26;
constexpr uint64_t SPEC_SAMPLE_EDGES = 1ull << 21;
uint64_t spec_min_edges();  // SPEC_MIN_EDGES, or $CC_SPEC_MIN_EDGES (test hook)
struct SpecLevel {
  uint32_t* S;
  uint32_t* next;
  uint64_t* gctr;
};
void launch_validate(const uint2* edges, uint64_t m, uint64_t n, uint64_t* gctr, cudaStream_t st);
// deg[v] += arcs with source v (deg zeroed by the caller).  hub_scratch (>= 2048 u32) and
// hub_count (40 device u64): per-block shared-memory counting of high-degree ids (NULL: off)
// radix_scratch (>= degree_radix_scratch(m, n) bytes) and radix_cursor (2048 u32): the
// bucketed shared-memory count (graph.cu), used when n >= 2^20 (CC_DEG_ALGO=radix|window
// forces one); otherwise, or when the scratch is too small, L2 increments in id windows.
// returns bit 0: the bucketed count ran (else L2-window increments); bit 1: the speculative
// root level ran (spec != nullptr, bucketed count, m >= SPEC_MIN_EDGES)
int launch_degree(const uint2* edges, uint64_t m, uint64_t n, uint32_t* deg, cudaStream_t st,
                  uint32_t* hub_scratch = nullptr, uint64_t* hub_count = nullptr,
                  void* radix_scratch = nullptr, uint64_t radix_bytes = 0,
                  uint32_t* radix_cursor = nullptr, const SpecLevel* spec = nullptr);
uint64_t degree_radix_scratch(uint64_t m, uint64_t n);
// deg[0, n) are the degrees of ids base .. base+n-1 (base > 0: a rank's vertex block)
// the non-empty bins of hist[1, nb) as (degree, count) pairs into out, *cnt of them (unordered)
void launch_hist_pairs(const uint32_t* hist, uint64_t nb, uint2* out, uint64_t* cnt, cudaStream_t st);
void launch_deg_hist(const uint32_t* deg, uint64_t n, uint32_t* hist, uint32_t* tail,
                     uint64_t* gctr, cudaStream_t st, uint64_t base = 0);
// edge-streaming BFS level over 2-bit vertex state S (16 ids per word: bit0 visited, bit1
// frontier): the ids found are set in `next` (and visited in S); with `compact`, the edges
// that can still matter (an endpoint unvisited after the level) are appended to `out` (count
// in gctr[G_REMAIN]).  The level's counts come from launch_farcs on `next` afterwards.
void launch_bfs_level(bool root_level, bool compact, const uint2* edges, uint64_t m, uint32_t root,
                      uint32_t* S, uint32_t* next, uint2* out, uint64_t* gctr, cudaStream_t st);
// *found += |next|, *farcs += sum of deg[v] over the ids set in next
void launch_farcs(const uint32_t* next, uint64_t n, const uint32_t* deg, uint64_t* found, uint64_t* farcs,
                  cudaStream_t st);
void launch_bfs_advance(uint32_t* S, const uint32_t* next, uint64_t n, cudaStream_t st);
// both of the above in one pass, and next cleared (S: 2n bits, 16-byte aligned words)
void launch_farcs_advance(uint32_t* next, uint32_t* S, uint64_t n, const uint32_t* deg, uint64_t* found,
                          uint64_t* farcs, cudaStream_t st);
void launch_filter(const uint2* edges, uint64_t m, const uint32_t* S, uint2* out,
                   uint64_t* gctr, cudaStream_t st);
void launch_vis_bits(const uint32_t* S, uint64_t n, uint32_t* vis, cudaStream_t st);
void launch_bfs_labels(const uint32_t* visited, uint64_t n, uint32_t* label, uint64_t* gctr,
                       cudaStream_t st);
void launch_min_visited(const uint32_t* visited, uint64_t n, uint64_t* gctr, cudaStream_t st);

// Remainder renumbering: the edges left after the BFS peel touch few ids, so
// the SV runs on their endpoints renumbered densely in id order, [0, n').  The map is monotone,
// and Alg. 1 only compares ids, so its sets and counters are those of the original ids.
// bm (nw words, caller-zeroed): the endpoints' bits
void launch_sub_mark(const uint2* edges, uint64_t m, uint32_t* bm, cudaStream_t st);
// wpre[w] = set bits of bm before word w; *total = n' (bsum: sub_bsum_words(nw) scratch words)
uint64_t sub_bsum_words(uint64_t nw);
void launch_sub_rank(const uint32_t* bm, uint64_t nw, uint32_t* bsum, uint32_t* wpre, uint64_t* total,
                     cudaStream_t st);
// out[i] = (rank(u), rank(v)); inv[rank(x)] = x; sdeg[rank(x)] = deg[x]
void launch_sub_edges(const uint2* edges, uint64_t m, const uint32_t* bm, const uint32_t* wpre,
                      const uint32_t* deg, uint2* out, uint32_t* inv, uint32_t* sdeg, cudaStream_t st);
// label[inv[i]] = inv[slabel[i]] for i < ns
void launch_sub_labels(const uint32_t* inv, const uint32_t* slabel, uint64_t ns, uint32_t* label,
                       cudaStream_t st);

// *cnt += #{v in [lo, hi) : label[v] = v} (caller-zeroed)
void launch_count_roots(const uint32_t* label, uint64_t lo, uint64_t hi, uint64_t* cnt, cudaStream_t st);

}  // namespace graph
}  // namespace cc
