// radix.cu -- onesweep LSD radix sort kernels (see radix.cuh for the design notes).
#include "radix.cuh"

#include <algorithm>

namespace cc {
namespace radix {

int num_passes(int kbits) { return kbits <= 0 ? 0 : (kbits + RADIX_BITS - 1) / RADIX_BITS; }

// ---------------------------------------------------------------------------------------
// Histogram of every pass digit in one read of the keys.  Warp-aggregated (match_any)
// shared-memory counting, so a key distribution dominated by one bucket (the giant
// partition of late SV iterations) does not serialise on one shared-memory bank.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(BLOCK) k_hist(const uint64_t* __restrict__ keys, uint64_t n,
                                                int passes, int base_bit,
                                                uint64_t* __restrict__ ghist) {
  __shared__ uint32_t sh[MAX_PASSES][RADIX];
  for (int i = threadIdx.x; i < MAX_PASSES * RADIX; i += BLOCK) (&sh[0][0])[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
  const uint32_t lt = lanemask_lt();
  for (uint64_t base = (uint64_t)blockIdx.x * BLOCK; base < n; base += stride) {
    uint64_t i = base + threadIdx.x;
    bool valid = i < n;
    const uint64_t key = valid ? keys[i] : 0ull;
    for (int p = 0; p < passes; p++) {
      uint32_t d = valid ? (uint32_t)((key >> (base_bit + p * RADIX_BITS)) & (RADIX - 1))
                         : (RADIX + lane_id());
      uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (valid && (peers & lt) == 0) atomicAdd(&sh[p][d], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RADIX; i += BLOCK) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd((unsigned long long*)&ghist[i], (unsigned long long)c);
  }
}

// ---------------------------------------------------------------------------------------
// One scatter pass (digit at key bits [shift, shift+8)).
// ---------------------------------------------------------------------------------------
template <bool HAS_VAL>
__global__ void __launch_bounds__(BLOCK, 2) k_onesweep(const uint64_t* __restrict__ kin,
                                                    const uint32_t* __restrict__ vin,
                                                    uint64_t* __restrict__ kout,
                                                    uint32_t* __restrict__ vout, uint64_t n,
                                                    int shift, const uint64_t* __restrict__ ghist,
                                                    uint64_t* lookback, uint32_t* tile_ctr,
                                                    uint32_t epoch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(smem_raw);                        // TILE
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + TILE * sizeof(uint64_t));  // TILE
  __shared__ uint32_t s_wcnt[WARPS][RADIX];
  __shared__ uint32_t s_dstart[RADIX];
  __shared__ uint32_t s_bstart[RADIX];
  __shared__ uint64_t s_gbase[RADIX];
  __shared__ uint32_t s_scan[WARPS + 1];
  __shared__ uint32_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < WARPS * RADIX; i += BLOCK) (&s_wcnt[0][0])[i] = 0;
  // bucket starts of this pass: exclusive scan of the global digit histogram
  uint32_t tot;
  uint32_t hb = (uint32_t)ghist[tid];
  s_bstart[tid] = block_excl_scan<BLOCK>(hb, s_scan, &tot);  // (contains __syncthreads)
  const uint64_t tile = s_tile;
  const uint64_t tbase = tile * TILE;
  const uint32_t lt = lanemask_lt();

  // ---- load + warp multi-split rank: warp w owns [tbase + w*WARP_ITEMS, +WARP_ITEMS)
  uint64_t key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t rank[ITEMS];
  const uint64_t wbase = tbase + (uint64_t)wid * WARP_ITEMS + lane;
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    uint64_t i = wbase + (uint64_t)k * 32;
    key[k] = (i < n) ? kin[i] : ~0ull;
    if (HAS_VAL) val[k] = (i < n) ? vin[i] : 0u;
  }
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    uint64_t i = wbase + (uint64_t)k * 32;
    bool valid = i < n;
    uint32_t d = valid ? ((uint32_t)(key[k] >> shift) & (RADIX - 1)) : (RADIX + lane);
    uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = 0;
    if (valid) before = s_wcnt[wid][d];
    __syncwarp();
    rank[k] = before + __popc(peers & lt);
    if (valid && (peers & lt) == 0) s_wcnt[wid][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // ---- per-digit: exclusive prefix over warps, tile total
  const int d = tid;
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < WARPS; w++) {
    uint32_t c = s_wcnt[w][d];
    s_wcnt[w][d] = run;
    run += c;
  }
  const uint32_t tcount = run;
  // publish aggregate (or inclusive prefix for tile 0) as early as possible
  const uint64_t ep = ((uint64_t)(epoch & LB_EPOCH_MASK)) << LB_EPOCH_SHIFT;
  if (tile == 0) st_relaxed_u64(&lookback[d], LB_INC | ep | tcount);
  else st_relaxed_u64(&lookback[tile * RADIX + d], LB_AGG | ep | tcount);
  uint32_t ttot;
  s_dstart[d] = block_excl_scan<BLOCK>(tcount, s_scan, &ttot);

  // ---- decoupled look-back for digit d
  uint64_t excl = 0;
  if (tile > 0) {
    int64_t j = (int64_t)tile - 1;
    while (true) {
      uint64_t e = ld_relaxed_u64(&lookback[(uint64_t)j * RADIX + d]);
      if ((e & LB_FLAGS) == 0 || ((e >> LB_EPOCH_SHIFT) & LB_EPOCH_MASK) != (epoch & LB_EPOCH_MASK))
        continue;  // predecessor not published yet: spin
      excl += e & LB_VAL_MASK;
      if ((e & LB_FLAGS) == LB_INC) break;
      j--;
    }
    st_relaxed_u64(&lookback[tile * RADIX + d], LB_INC | ep | (excl + tcount));
  }
  s_gbase[d] = (uint64_t)s_bstart[d] + excl - s_dstart[d];
  __syncthreads();

  // ---- stage in digit order
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    uint64_t i = wbase + (uint64_t)k * 32;
    if (i < n) {
      uint32_t dg = (uint32_t)(key[k] >> shift) & (RADIX - 1);
      uint32_t lp = s_dstart[dg] + s_wcnt[wid][dg] + rank[k];
      s_keys[lp] = key[k];
      if (HAS_VAL) s_vals[lp] = val[k];
    }
  }
  __syncthreads();

  // ---- coalesced scatter of digit runs
  const uint32_t tn = (n - tbase < (uint64_t)TILE) ? (uint32_t)(n - tbase) : (uint32_t)TILE;
  for (uint32_t i = tid; i < tn; i += BLOCK) {
    uint64_t kk = s_keys[i];
    uint32_t dg = (uint32_t)(kk >> shift) & (RADIX - 1);
    uint64_t pos = s_gbase[dg] + i;
    kout[pos] = kk;
    if (HAS_VAL) vout[pos] = s_vals[i];
  }
}

size_t smem_bytes(bool has_val) {
  return TILE * sizeof(uint64_t) + (has_val ? TILE * sizeof(uint32_t) : 0);
}

int sort_pairs(Workspace& ws, uint64_t* k[2], uint32_t* v[2], int cur, uint64_t n, int kbits,
               bool has_val, cudaStream_t st, uint64_t* launches, int base_bit) {
  const int passes = num_passes(kbits);
  if (n <= 1 || passes == 0) return cur;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_bytes(true));
    cudaFuncSetAttribute(k_onesweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_bytes(false));
    attr_set = true;
  }
  cudaMemsetAsync(ws.ghist, 0, sizeof(uint64_t) * MAX_PASSES * RADIX, st);
  cudaMemsetAsync(ws.tile_ctr, 0, sizeof(uint32_t) * MAX_PASSES, st);
  const uint64_t tiles = (n + TILE - 1) / TILE;
  int hblocks = (int)std::min<uint64_t>((n + BLOCK - 1) / BLOCK, 148 * 8);
  k_hist<<<hblocks, BLOCK, 0, st>>>(k[cur], n, passes, base_bit, ws.ghist);
  *launches += 1;
  for (int p = 0; p < passes; p++) {
    uint32_t epoch = ++ws.epoch;
    if ((epoch & LB_EPOCH_MASK) == 0) {  // epoch wrapped: clear stale entries once
      cudaMemsetAsync(ws.lookback, 0, sizeof(uint64_t) * ws.max_tiles * RADIX, st);
      epoch = ++ws.epoch;
    }
    if (has_val)
      k_onesweep<true><<<(unsigned)tiles, BLOCK, smem_bytes(true), st>>>(
          k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], n, base_bit + p * RADIX_BITS, ws.ghist + p * RADIX,
          ws.lookback, ws.tile_ctr + p, epoch);
    else
      k_onesweep<false><<<(unsigned)tiles, BLOCK, smem_bytes(false), st>>>(
          k[cur], nullptr, k[cur ^ 1], nullptr, n, base_bit + p * RADIX_BITS, ws.ghist + p * RADIX,
          ws.lookback, ws.tile_ctr + p, epoch);
    *launches += 1;
    cur ^= 1;
  }
  return cur;
}

}  // namespace radix
}  // namespace cc
