// relabel.cu -- u64 ids -> dense u32 ids (Alg. 2 line 4).
//
// "This process requires sorting the edge list ... After the first sort, we perform a
// parallel prefix (scan) operation to label the source vertices with a unique id in
// [0, V-1]".  Here all 2m endpoints are sorted once (64-bit onesweep radix
// sort, payload = endpoint position), a scan over 'first of its value' flags gives each
// endpoint its rank among the distinct ids, and the rank is scattered back to the
// endpoint's position.  Rank order = id order, so the minimum dense id of
// a component maps back to its minimum original id.
#include <algorithm>

#include "relabel.cuh"
#include "scan.cuh"

namespace cc {
namespace relabel {

constexpr int B = 256;
constexpr int ITEMS = 8;
constexpr int TILE = B * ITEMS;

__global__ void k_init(const uint64_t* __restrict__ ids, uint64_t k, uint64_t* __restrict__ keys,
                       uint32_t* __restrict__ vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < k; i += (uint64_t)gridDim.x * B) {
    keys[i] = ids[i];
    vals[i] = (uint32_t)i;
  }
}

// rank[i] = #distinct values among keys[0..i] - 1; dense[vals[i]] = rank; uids[rank] = key.
__global__ void __launch_bounds__(B) k_rank(const uint64_t* __restrict__ keys,
                                            const uint32_t* __restrict__ vals, uint64_t k,
                                            uint32_t* __restrict__ dense, uint64_t* __restrict__ uids,
                                            uint64_t* flags, uint32_t* ticket, uint32_t epoch,
                                            unsigned long long* total) {
  __shared__ uint32_t s_scan[B / 32 + 1];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_pref;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t i0 = tile * TILE + (uint64_t)threadIdx.x * ITEMS;
  uint64_t key[ITEMS];
  uint32_t head = 0, nh = 0;
  uint64_t prev = (i0 > 0 && i0 <= k) ? keys[i0 - 1] : 0;
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const uint64_t i = i0 + j;
    if (i < k) {
      key[j] = keys[i];
      const bool h = (i == 0) || key[j] != prev;
      head |= (uint32_t)h << j;
      nh += h;
      prev = key[j];
    }
  }
  uint32_t tot;
  const uint32_t excl = block_excl_scan<B>(nh, s_scan, &tot);
  const uint64_t pref = scan::tile_prefix(flags, tile, tot, epoch, &s_pref);
  uint64_t r = pref + excl;  // heads before this thread's first item
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const uint64_t i = i0 + j;
    if (i < k) {
      if (head >> j & 1u) {
        uids[r] = key[j];
        r++;
      }
      dense[vals[i]] = (uint32_t)(r - 1);
    }
  }
  if (i0 < k && i0 + ITEMS >= k) *total = r;  // owner of the last element
}

// labels of the distinct ids: out[i] = uids[label[i]]
__global__ void k_labels(const uint64_t* __restrict__ uids, const uint32_t* __restrict__ label,
                         uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B)
    out[i] = uids[label[i]];
}

static unsigned grid(uint64_t work, unsigned cap) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + B - 1) / B, cap));
}

cc_status_t run(const uint64_t* ids, uint64_t k, uint64_t* keys[2], uint32_t* vals[2],
                radix::Workspace& rws, scan::State& ss, uint32_t* dense, uint64_t* uids,
                uint64_t* total, cudaStream_t st, uint64_t* launches) {
  if (!k) return 0;
  k_init<<<grid(k, 148 * 16), B, 0, st>>>(ids, k, keys[0], vals[0]);
  *launches += 1;
  const int cur = radix::sort_pairs(rws, keys, vals, 0, k, 64, true, st, launches, 0);
  cudaMemsetAsync(ss.ticket, 0, sizeof(uint32_t), st);
  const uint64_t tiles = (k + TILE - 1) / TILE;
  k_rank<<<(unsigned)tiles, B, 0, st>>>(keys[cur], vals[cur], k, dense, uids, ss.flags, ss.ticket,
                                         ++ss.epoch, reinterpret_cast<unsigned long long*>(total));
  *launches += 1;
  return 0;
}

// ---- id permutation ("permuting the vertex ids using Robert Jenkins' 64 bit mix
// invertible hash function").  The 64-bit integer mix below (shift-add/xor rounds, each a
// bijection of 64-bit words) is that family's 7-step variant; SV then runs in the order of
// the mixed ids and the labels are mapped back to the minimum original id (C1).
CC_DEVI uint64_t mix64(uint64_t k) {
  k = (~k) + (k << 21);
  k = k ^ (k >> 24);
  k = (k + (k << 3)) + (k << 8);
  k = k ^ (k >> 14);
  k = (k + (k << 2)) + (k << 4);
  k = k ^ (k >> 28);
  k = k + (k << 31);
  return k;
}
__global__ void k_mix(const uint64_t* __restrict__ uids, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B)
    out[i] = mix64(uids[i]);
}
__global__ void k_apply(uint32_t* __restrict__ e, uint64_t k, const uint32_t* __restrict__ pi) {
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < k; i += (uint64_t)gridDim.x * B)
    e[i] = pi[e[i]];
}
// mino[c] = min original rank v of the vertices whose permuted label is c
__global__ void k_canon1(const uint32_t* __restrict__ pi, const uint32_t* __restrict__ label, uint64_t n,
                         uint32_t* mino) {
  for (uint64_t v = blockIdx.x * (uint64_t)B + threadIdx.x; v < n; v += (uint64_t)gridDim.x * B)
    atomicMin(&mino[label[pi[v]]], (uint32_t)v);
}
__global__ void k_canon2(const uint32_t* __restrict__ pi, const uint32_t* __restrict__ label, uint64_t n,
                         const uint32_t* __restrict__ mino, uint32_t* __restrict__ out) {
  for (uint64_t v = blockIdx.x * (uint64_t)B + threadIdx.x; v < n; v += (uint64_t)gridDim.x * B)
    out[v] = mino[label[pi[v]]];
}

void mix(const uint64_t* uids, uint64_t n, uint64_t* out, cudaStream_t st) {
  if (n) k_mix<<<grid(n, 148 * 16), B, 0, st>>>(uids, n, out);
}
void apply(uint32_t* e, uint64_t k, const uint32_t* pi, cudaStream_t st) {
  if (k) k_apply<<<grid(k, 148 * 16), B, 0, st>>>(e, k, pi);
}
void canonicalize(const uint32_t* pi, const uint32_t* label, uint64_t n, uint32_t* mino, uint32_t* out,
                  cudaStream_t st) {
  if (!n) return;
  cudaMemsetAsync(mino, 0xFF, sizeof(uint32_t) * n, st);
  k_canon1<<<grid(n, 148 * 16), B, 0, st>>>(pi, label, n, mino);
  k_canon2<<<grid(n, 148 * 16), B, 0, st>>>(pi, label, n, mino, out);
}

void labels(const uint64_t* uids, const uint32_t* label, uint64_t n, uint64_t* out, cudaStream_t st) {
  if (n) k_labels<<<grid(n, 148 * 16), B, 0, st>>>(uids, label, n, out);
}

}  // namespace relabel
}  // namespace cc
