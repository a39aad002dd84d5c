// scan.cuh -- single-pass tile prefix (decoupled look-back) for ordered compaction/scans.
//
// Tiles take tickets from an atomic counter (so every predecessor is resident or done),
// publish their aggregate, and warp 0 resolves the exclusive prefix by examining 32
// predecessors per step in parallel.  Entries pack (flag, epoch, value) into 64 bits so the
// flag array never needs clearing between launches.
#pragma once
#include "common.cuh"

namespace cc {
namespace scan {

constexpr uint64_t F_AGG = 1ull << 62;
constexpr uint64_t F_INC = 2ull << 62;
constexpr uint64_t F_MASK = 3ull << 62;
constexpr int EPOCH_SHIFT = 40;
constexpr uint64_t EPOCH_MASK = (1ull << 22) - 1;
constexpr uint64_t VAL_MASK = (1ull << 40) - 1;

struct State {
  uint64_t* flags = nullptr;  // one entry per tile
  uint32_t* ticket = nullptr;
  uint64_t max_tiles = 0;
  uint32_t epoch = 0;
};

// Called by all threads of the block (contains __syncthreads).  `agg` is the tile's total,
// valid in thread 0.  Returns the exclusive prefix of this tile in every thread.
CC_DEVI uint64_t tile_prefix(uint64_t* flags, uint64_t tile, uint64_t agg, uint32_t epoch,
                             uint64_t* s_out) {
  const uint64_t ep = ((uint64_t)(epoch & EPOCH_MASK)) << EPOCH_SHIFT;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0) st_relaxed_u64(&flags[tile], (tile == 0 ? F_INC : F_AGG) | ep | agg);
    uint64_t excl = 0;
    if (tile > 0) {
      int64_t base = (int64_t)tile - 1;
      while (true) {
        const int64_t j = base - lane;
        uint64_t e;
        if (j >= 0) {
          do {
            e = ld_relaxed_u64(&flags[j]);
          } while ((e & F_MASK) == 0 || ((e >> EPOCH_SHIFT) & EPOCH_MASK) != (epoch & EPOCH_MASK));
        } else {
          e = F_INC;  // virtual predecessor with value 0
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (e & F_MASK) == F_INC);
        uint64_t v = e & VAL_MASK;
        if (inc) {
          const int first = __ffs(inc) - 1;
          if (lane > first) v = 0;
#pragma unroll
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          excl += v;
          break;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        base -= 32;
      }
      if (lane == 0) st_relaxed_u64(&flags[tile], F_INC | ep | (excl + agg));
    }
    if (lane == 0) *s_out = excl;
  }
  __syncthreads();
  return *s_out;
}

}  // namespace scan
}  // namespace cc
