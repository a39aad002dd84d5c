// radix.cuh -- onesweep LSD radix sort of packed tuple words (sm_100a).
//
// The regroup steps of Alg. 1 ("sort A_i by third element" line 8 / "by first element"
// line 14; "the bulk step of the algorithm is the sorting of tuples",
// PAPER.md:207) are stable LSD radix sorts on the key held in the high 32 bits of a
// 64-bit tuple word, using only the ceil(log2 n) key bits.
//
// Design:
//  * one histogram kernel reads the keys once and counts every digit of every pass (per-
//    thread run-length counting into shared memory, robust to skewed digits); a pass whose
//    digit is the same for every key is the identity and is skipped;
//  * one scatter kernel per 8-bit digit: tiles of 3072 elements (12 per thread, 3 blocks
//    per SM) are ranked in shared memory with warp multi-split (__match_any_sync peers +
//    popc), the per-tile digit counts are published and combined across tiles by decoupled
//    look-back (tiles take tickets from an atomic counter so every predecessor is resident
//    or done; eight predecessors are read per round trip), and the tile is staged in shared
//    memory in digit order so global stores are coalesced runs;
//  * look-back entries carry (flag, epoch, count) in one 64-bit word, so they never need
//    clearing between passes.
#pragma once
#include "common.cuh"

namespace cc {
namespace radix {

constexpr int RADIX_BITS = 8;
constexpr int RADIX = 1 << RADIX_BITS;
constexpr int BLOCK = 256;  // == RADIX: thread d owns digit d in the per-tile phases
constexpr int WARPS = BLOCK / 32;
constexpr int ITEMS = 12;                 // items per thread of a scatter pass
constexpr int PASS_MINB = 3;              // resident blocks per SM (80 registers)
constexpr int TILE = BLOCK * ITEMS;       // 3072 elements
constexpr int TILE_MIN = TILE;            // look-back sizing
constexpr int MAX_PASSES = 8;        // up to 64-bit keys (u64 relabel)

constexpr uint64_t LB_AGG = 1ull << 62;
constexpr uint64_t LB_INC = 2ull << 62;
constexpr uint64_t LB_FLAGS = 3ull << 62;
constexpr int LB_EPOCH_SHIFT = 40;
constexpr uint64_t LB_EPOCH_MASK = (1ull << 22) - 1;
constexpr uint64_t LB_VAL_MASK = (1ull << 40) - 1;

struct Workspace {
  uint64_t* ghist = nullptr;      // MAX_PASSES * RADIX
  uint64_t* lookback = nullptr;   // max_tiles * RADIX
  uint32_t* tile_ctr = nullptr;   // MAX_PASSES
  uint64_t max_tiles = 0;
  uint32_t epoch = 0;
};

// Sort `n` elements by bits [base_bit, base_bit+kbits) of the 64-bit words k[cur] (with u32
// payload v[cur] when has_val).  Tuple words keep their key in the high half (base_bit 32);
// u64 ids use the whole word (base_bit 0, kbits 64).  Ping-pongs between buffer 0 and 1;
// returns the index holding the result.
int sort_pairs(Workspace& ws, uint64_t* k[2], uint32_t* v[2], int cur, uint64_t n, int kbits,
               bool has_val, cudaStream_t st, uint64_t* launches, int base_bit = 32);

size_t smem_bytes(bool has_val, int items = ITEMS);
int num_passes(int kbits);

}  // namespace radix
}  // namespace cc
