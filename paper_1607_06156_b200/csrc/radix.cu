// radix.cu -- onesweep LSD radix sort kernels (see radix.cuh for the design notes).
#include "radix.cuh"

#include <algorithm>

namespace cc {
namespace radix {

int num_passes(int kbits) { return kbits <= 0 ? 0 : (kbits + RADIX_BITS - 1) / RADIX_BITS; }

// ---------------------------------------------------------------------------------------
// Histogram of every pass digit in one read of the keys.  Each thread keeps, per pass, the
// digit it saw last and a run count, and adds a run to the shared-memory bin only when the
// digit changes: random digits cost one shared atomic per key and pass, while a skewed
// distribution (the giant partition of late SV iterations, constant high bytes of u64
// ids) collapses into a few long runs instead of serialising 32 lanes on one bank.
// ---------------------------------------------------------------------------------------
constexpr int HIST_UNROLL = 4;

__global__ void __launch_bounds__(BLOCK) k_hist(const uint64_t* __restrict__ keys, uint64_t n,
                                                int passes, int base_bit,
                                                uint64_t* __restrict__ ghist) {
  __shared__ uint32_t sh[MAX_PASSES][RADIX];
  for (int i = threadIdx.x; i < MAX_PASSES * RADIX; i += BLOCK) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t cur[MAX_PASSES], cnt[MAX_PASSES];
#pragma unroll
  for (int p = 0; p < MAX_PASSES; p++) cur[p] = 0, cnt[p] = 0;
  const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
  for (uint64_t i0 = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; i0 < n; i0 += stride * HIST_UNROLL) {
    uint64_t key[HIST_UNROLL];
#pragma unroll
    for (int u = 0; u < HIST_UNROLL; u++) {
      const uint64_t i = i0 + u * stride;
      key[u] = i < n ? __ldg(&keys[i]) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < HIST_UNROLL; u++) {
      if (i0 + u * stride >= n) break;
#pragma unroll
      for (int p = 0; p < MAX_PASSES; p++) {
        if (p >= passes) break;
        const uint32_t d = (uint32_t)(key[u] >> (base_bit + p * RADIX_BITS)) & (RADIX - 1);
        if (d != cur[p]) {
          if (cnt[p]) atomicAdd(&sh[p][cur[p]], cnt[p]);
          cur[p] = d;
          cnt[p] = 0;
        }
        cnt[p]++;
      }
    }
  }
#pragma unroll
  for (int p = 0; p < MAX_PASSES; p++)
    if (cnt[p]) atomicAdd(&sh[p][cur[p]], cnt[p]);
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RADIX; i += BLOCK) {
    uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd((unsigned long long*)&ghist[i], (unsigned long long)c);
  }
}

// ---------------------------------------------------------------------------------------
// One scatter pass (digit at key bits [shift, shift+8)).
// ---------------------------------------------------------------------------------------
template <bool HAS_VAL, int ITEMS, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep(const uint64_t* __restrict__ kin,
                                                    const uint32_t* __restrict__ vin,
                                                    uint64_t* __restrict__ kout,
                                                    uint32_t* __restrict__ vout, uint64_t n,
                                                    int shift, const uint64_t* __restrict__ ghist,
                                                    uint64_t* lookback, uint32_t* tile_ctr,
                                                    uint32_t epoch) {
  constexpr int WARP_ITEMS = 32 * ITEMS;
  constexpr int TILE = BLOCK * ITEMS;
  constexpr int LB_WIN = 8;  // look-back entries read per round trip
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(smem_raw);                        // TILE
  uint32_t* s_vals = reinterpret_cast<uint32_t*>(smem_raw + TILE * sizeof(uint64_t));  // TILE
  __shared__ uint32_t s_wcnt[WARPS][RADIX];
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
  const uint32_t dstart = block_excl_scan<BLOCK>(tcount, s_scan, &ttot);

  // ---- decoupled look-back for digit d
  uint64_t excl = 0;
  if (tile > 0) {
    // LB_WIN predecessors are read per round trip (independent loads), then consumed in
    // order up to the first inclusive prefix; an unpublished entry ends the round and is
    // re-read.  Tile 0 always publishes an inclusive prefix, so the walk stops at j >= 0.
    int64_t j = (int64_t)tile - 1;
    const uint64_t want = epoch & LB_EPOCH_MASK;
    bool done = false;
    while (!done) {
      uint64_t e[LB_WIN];
#pragma unroll
      for (int u = 0; u < LB_WIN; u++)
        e[u] = j - u >= 0 ? ld_relaxed_u64(&lookback[(uint64_t)(j - u) * RADIX + d]) : 0ull;
      int used = 0;
#pragma unroll
      for (int u = 0; u < LB_WIN; u++) {
        if ((e[u] & LB_FLAGS) == 0 || ((e[u] >> LB_EPOCH_SHIFT) & LB_EPOCH_MASK) != want) break;
        excl += e[u] & LB_VAL_MASK;
        used = u + 1;
        if ((e[u] & LB_FLAGS) == LB_INC) {
          done = true;
          break;
        }
      }
      j -= used;
      if (!used) {  // the nearest predecessor has not published: wait on that one entry only
        uint64_t e0;
        do {
          e0 = ld_relaxed_u64(&lookback[(uint64_t)j * RADIX + d]);
          if ((e0 & LB_FLAGS) == 0) __nanosleep(32);
        } while ((e0 & LB_FLAGS) == 0 || ((e0 >> LB_EPOCH_SHIFT) & LB_EPOCH_MASK) != want);
      }
    }
    st_relaxed_u64(&lookback[tile * RADIX + d], LB_INC | ep | (excl + tcount));
  }
  s_gbase[d] = (uint64_t)s_bstart[d] + excl - dstart;
#pragma unroll
  for (int w = 0; w < WARPS; w++) s_wcnt[w][d] += dstart;
  __syncthreads();

  // ---- stage in digit order
#pragma unroll
  for (int k = 0; k < ITEMS; k++) {
    uint64_t i = wbase + (uint64_t)k * 32;
    if (i < n) {
      uint32_t dg = (uint32_t)(key[k] >> shift) & (RADIX - 1);
      uint32_t lp = s_wcnt[wid][dg] + rank[k];
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

size_t smem_bytes(bool has_val, int items) {
  return (size_t)BLOCK * items * (sizeof(uint64_t) + (has_val ? sizeof(uint32_t) : 0));
}

template <bool HAS_VAL>
static void launch_pass(uint64_t n, const uint64_t* kin, const uint32_t* vin, uint64_t* kout,
                        uint32_t* vout, int shift, const uint64_t* gh, Workspace& ws,
                        uint32_t* tctr, uint32_t epoch, cudaStream_t st) {
  auto* kern = k_onesweep<HAS_VAL, ITEMS, PASS_MINB>;
  static bool attr = (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem_bytes(HAS_VAL, ITEMS)),
                      true);
  (void)attr;
  const unsigned tiles = (unsigned)((n + TILE - 1) / TILE);
  kern<<<tiles, BLOCK, smem_bytes(HAS_VAL, ITEMS), st>>>(kin, vin, kout, vout, n, shift, gh,
                                                          ws.lookback, tctr, epoch);
}

int sort_pairs(Workspace& ws, uint64_t* k[2], uint32_t* v[2], int cur, uint64_t n, int kbits,
               bool has_val, cudaStream_t st, uint64_t* launches, int base_bit) {
  const int passes = num_passes(kbits);
  if (n <= 1 || passes == 0) return cur;
  cudaMemsetAsync(ws.ghist, 0, sizeof(uint64_t) * MAX_PASSES * RADIX, st);
  cudaMemsetAsync(ws.tile_ctr, 0, sizeof(uint32_t) * MAX_PASSES, st);
  const uint64_t hthreads = (n + HIST_UNROLL - 1) / HIST_UNROLL;
  int hblocks = (int)std::min<uint64_t>((hthreads + BLOCK - 1) / BLOCK, 148 * 8);
  k_hist<<<hblocks, BLOCK, 0, st>>>(k[cur], n, passes, base_bit, ws.ghist);
  *launches += 1;
  // A pass whose digit is the same for every key is the identity permutation: skip it.
  uint64_t hh[MAX_PASSES * RADIX];
  bool trivial[MAX_PASSES] = {};
  {
    cudaMemcpyAsync(hh, ws.ghist, sizeof(uint64_t) * passes * RADIX, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) == cudaSuccess)
      for (int p = 0; p < passes; p++)
        for (int d = 0; d < RADIX; d++)
          if (hh[p * RADIX + d]) {
            trivial[p] = hh[p * RADIX + d] == n;
            break;
          }
  }
  for (int p = 0; p < passes; p++) {
    if (trivial[p]) continue;
    uint32_t epoch = ++ws.epoch;
    if ((epoch & LB_EPOCH_MASK) == 0) {  // epoch wrapped: clear stale entries once
      cudaMemsetAsync(ws.lookback, 0, sizeof(uint64_t) * ws.max_tiles * RADIX, st);
      epoch = ++ws.epoch;
    }
    const int shift = base_bit + p * RADIX_BITS;
    const uint64_t* gh = ws.ghist + p * RADIX;
    uint32_t* tctr = ws.tile_ctr + p;
    if (has_val)
      launch_pass<true>(n, k[cur], v[cur], k[cur ^ 1], v[cur ^ 1], shift, gh, ws, tctr, epoch, st);
    else
      launch_pass<false>(n, k[cur], nullptr, k[cur ^ 1], nullptr, shift, gh, ws, tctr, epoch, st);
    *launches += 1;
    cur ^= 1;
  }
  return cur;
}

}  // namespace radix
}  // namespace cc
