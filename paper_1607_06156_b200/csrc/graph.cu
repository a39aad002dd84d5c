// graph.cu -- degree distribution (Alg. 2 line 2), BFS peel (lines 7-8) and filter
// (lines 10-11) kernels.  PAPER.md:249-279.
#include "graph.cuh"

#include <algorithm>
#include <cstdlib>

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
// counting increment replaces the paper's sort by source.  When the
// counter array is larger than a window that stays L2-resident (2^24 ids = 64 MB), the
// edge list is streamed once per window and only endpoints inside it are counted, so the
// random increments never reach DRAM.
constexpr uint64_t DEG_WINDOW = 1ull << 24;
// Hub vertices: on skewed graphs (R-MAT: the top id has ~0.1 % of all arc endpoints) every
// increment of one hub serialises on one L2 address.  A 1/HUB_SAMPLE prefix of the (randomly
// ordered) edge list is counted first, straight into deg; ids whose sample count reaches
// HUB_MIN are hubs and are counted per block in a shared-memory table for the rest of the
// list (one global add per hub per block at the end).  Exact either way: every endpoint is
// counted once, in deg or in a block's table.
constexpr uint64_t HUB_SAMPLE = 64;
constexpr uint32_t HUB_MIN = 64;      // sampled count: degree ~ 4096 and up
constexpr int HUB_CAP = 2048;         // hubs kept (more are counted globally)
constexpr int HUB_TAB = 4096;         // shared-memory table slots (power of two)
CC_DEVI uint32_t hub_hash(uint32_t v) { return (v * 2654435761u) >> 20; }  // 12 bits
template <bool HUBS>
__global__ void k_degree(const uint4* __restrict__ e2, uint64_t m, uint32_t* __restrict__ deg,
                         uint32_t lo, uint32_t hi, const uint32_t* __restrict__ hubs,
                         const unsigned long long* nhubs) {
  __shared__ uint32_t s_key[HUBS ? HUB_TAB : 1], s_cnt[HUBS ? HUB_TAB : 1];
  if (HUBS) {
    for (int i = threadIdx.x; i < HUB_TAB; i += BLOCK) {
      s_key[i] = 0xFFFFFFFFu;
      s_cnt[i] = 0;
    }
    __syncthreads();
    const uint32_t nh = (uint32_t)min(*nhubs, (unsigned long long)HUB_CAP);
    for (uint32_t i = threadIdx.x; i < nh; i += BLOCK) {  // linear probing, keys fixed
      const uint32_t v = hubs[i];
      if (v < lo || v >= hi) continue;
      uint32_t h = hub_hash(v) & (HUB_TAB - 1);
      while (atomicCAS(&s_key[h], 0xFFFFFFFFu, v) != 0xFFFFFFFFu) h = (h + 1) & (HUB_TAB - 1);
    }
    __syncthreads();
  }
  const uint64_t npair = m >> 1;
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i <= npair;
       i += (uint64_t)gridDim.x * BLOCK) {
    uint32_t v[4];
    int cnt = 0;
    if (i < npair) {
      const uint4 x = ldg_stream(&e2[i]);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; cnt = 4;
    } else if (m & 1) {
      const uint2 x = reinterpret_cast<const uint2*>(e2)[m - 1];
      v[0] = x.x; v[1] = x.y; cnt = 2;
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j >= cnt || v[j] < lo || v[j] >= hi) continue;
      if (HUBS) {
        uint32_t h = hub_hash(v[j]) & (HUB_TAB - 1), k;
        while ((k = s_key[h]) != v[j] && k != 0xFFFFFFFFu) h = (h + 1) & (HUB_TAB - 1);
        if (k == v[j]) {
          atomicAdd(&s_cnt[h], 1u);
          continue;
        }
      }
      atomicAdd(&deg[v[j]], 1u);
    }
  }
  if (HUBS) {
    __syncthreads();
    for (int i = threadIdx.x; i < HUB_TAB; i += BLOCK)
      if (s_cnt[i]) atomicAdd(&deg[s_key[i]], s_cnt[i]);
  }
}
bool launch_degree_radix(const uint2* edges, uint64_t m, uint64_t n, uint32_t* deg, void* scratch,
                         uint64_t scratch_bytes, uint32_t* cursor, cudaStream_t st, const SpecLevel* spec,
                         bool* spec_ran);
// histogram of floor(log2(sample count)) over ids with count >= HUB_MIN (picks the threshold
// that keeps the hubs within HUB_CAP: the largest ones)
__global__ void k_hub_hist(const uint32_t* __restrict__ deg, uint64_t n, unsigned long long* bins) {
  __shared__ uint32_t s[32];
  if (threadIdx.x < 32) s[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t v = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; v < n; v += (uint64_t)gridDim.x * BLOCK) {
    const uint32_t d = deg[v];
    if (d >= HUB_MIN) atomicAdd(&s[31 - __clz(d)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32 && s[threadIdx.x]) atomicAdd(&bins[threadIdx.x], (unsigned long long)s[threadIdx.x]);
}
// ids with sample count >= t -> hubs[0 .. *nhubs)
__global__ void k_hubs(const uint32_t* __restrict__ deg, uint64_t n, uint32_t t, uint32_t* hubs,
                       unsigned long long* nhubs) {
  for (uint64_t v = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; v < n; v += (uint64_t)gridDim.x * BLOCK)
    if (deg[v] >= t) {
      const unsigned long long j = atomicAdd(nhubs, 1ull);
      if (j < HUB_CAP) hubs[j] = (uint32_t)v;
    }
}
int launch_degree(const uint2* edges, uint64_t m, uint64_t n, uint32_t* deg, cudaStream_t st,
                  uint32_t* hub_scratch, uint64_t* hub_count, void* radix_scratch,
                  uint64_t radix_bytes, uint32_t* radix_cursor, const SpecLevel* spec) {
  // hub_count[0]: hub count; hub_count[8 .. 40): log2 histogram of the sample counts
  if (!m) return 0;
  {
    // bucketed shared-memory count (default for n >= 2^20); CC_DEG_ALGO=radix|window forces one
    const char* e = getenv("CC_DEG_ALGO");
    const bool force_radix = e && e[0] == 'r', force_window = e && e[0] == 'w';
    bool spec_ran = false;
    if (radix_scratch && !force_window && (force_radix || n >= (1ull << 20)) &&
        launch_degree_radix(edges, m, n, deg, radix_scratch, radix_bytes, radix_cursor, st, spec, &spec_ran))
      return 1 | (spec_ran ? 2 : 0);
  }
  static uint64_t window = 0;
  if (!window) {  // CC_DEG_WINDOW_LOG2: experiment hook for the counter window
    const char* e = getenv("CC_DEG_WINDOW_LOG2");
    window = e ? (1ull << atoi(e)) : DEG_WINDOW;
  }
  auto* nh = reinterpret_cast<unsigned long long*>(hub_count);
  // the hub table pays only on large edge lists (its sample must see the hubs)
  const bool hubs = hub_scratch && m >= (1ull << 27);
  uint64_t m0 = 0;
  if (hubs) {
    m0 = (m / HUB_SAMPLE) & ~1ull;  // even: the rest starts on a 16-byte boundary
    k_degree<false><<<grid_for((m0 >> 1) + 1, 148 * 16), BLOCK, 0, st>>>(
        reinterpret_cast<const uint4*>(edges), m0, deg, 0u, 0xFFFFFFFFu, nullptr, nullptr);
    cudaMemsetAsync(hub_count, 0, sizeof(uint64_t) * 40, st);
    k_hub_hist<<<grid_for(n, 148 * 8), BLOCK, 0, st>>>(deg, n, nh + 8);
    uint64_t bins[32];
    cudaMemcpyAsync(bins, hub_count + 8, sizeof(bins), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    uint32_t t = 0xFFFFFFFFu;  // smallest power of two whose ids fit the table
    uint64_t above = 0;
    for (int b = 31; b >= 0; b--) {
      if (above + bins[b] > (uint64_t)HUB_CAP) break;
      above += bins[b];
      if (bins[b]) t = 1u << b;
    }
    if (above) k_hubs<<<grid_for(n, 148 * 8), BLOCK, 0, st>>>(deg, n, t, hub_scratch, nh);
  }
  for (uint64_t lo = 0; lo < n; lo += window) {
    const uint64_t hi = std::min<uint64_t>(n, lo + window);
    const uint64_t mr = m - m0;
    if (hubs)
      k_degree<true><<<grid_for((mr >> 1) + 1, 148 * 8), BLOCK, 0, st>>>(
          reinterpret_cast<const uint4*>(edges + m0), mr, deg, (uint32_t)lo, (uint32_t)hi, hub_scratch, nh);
    else
      k_degree<false><<<grid_for((mr >> 1) + 1, 148 * 16), BLOCK, 0, st>>>(
          reinterpret_cast<const uint4*>(edges + m0), mr, deg, (uint32_t)lo, (uint32_t)hi, nullptr, nullptr);
  }
  return 0;
}

// ---------------------------------------------------------------- BFS state helpers
// 2-bit vertex state of the BFS peel (see k_bfs_level): bit 0 visited, bit 1 frontier
CC_DEVI uint32_t st2(const uint32_t* S, uint32_t v) { return (S[v >> 4] >> (2 * (v & 15))) & 3u; }
// claim v (unvisited when its state was read) for the next frontier: the visited bit and the
// next bit, both fire-and-forget reductions (idempotent: concurrent claims of one id are
// harmless).  A level's found ids and their degree sum are counted afterwards from `next`
// (k_farcs), so no thread waits on an atomic's result inside the level.
CC_DEVI void mark2(uint32_t* S, uint32_t* next, uint32_t v) {
  atomicOr(&S[v >> 4], 1u << (2 * (v & 15)));
  atomicOr(&next[v >> 5], 1u << (v & 31));
}

// ---------------------------------------------------------------- speculative root level
// The BFS root is the max-degree vertex, smallest id on ties (Alg. 2 line 7, PAPER.md:262;
// SURVEY.md C13), so it is known only once every degree is; its level (frontier = {root})
// would be one more stream over the edge list.  On large lists the root is guessed from the
// counts of a prefix of the (randomly ordered) list -- counted straight into deg, so the
// degree count stays exact -- and the bucketed degree pass claims the guess's neighbours
// while it streams the rest (k_deg_part, SpecRoot).  cc_run keeps the claims only if the
// guess equals the exact root; otherwise the state is cleared and level 1 runs as usual.
// best key = max over the prefix of (count << 32 | ~v): largest count, smallest id
__global__ void __launch_bounds__(BLOCK) k_deg_sample(const uint4* __restrict__ e2, uint64_t npair,
                                                      uint32_t* __restrict__ deg,
                                                      unsigned long long* best) {
  unsigned long long key = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < npair; i += (uint64_t)gridDim.x * BLOCK) {
    const uint4 q = ldg_stream(e2 + i);
    const uint32_t v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const uint32_t c = atomicAdd(&deg[v[h]], 1u) + 1u;
      const unsigned long long k = ((unsigned long long)c << 32) | (0xFFFFFFFFu - v[h]);
      key = k > key ? k : key;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, key, o);
    key = x > key ? x : key;
  }
  if ((threadIdx.x & 31) == 0 && key) atomicMax(best, key);
}
template <bool ROOT, bool COMPACT>
__global__ void __launch_bounds__(BLOCK) k_bfs_level(const uint2* __restrict__ e, uint64_t m, uint32_t root,
                                                     const unsigned long long* root_key, uint32_t* S,
                                                     uint32_t* next, uint2* __restrict__ out,
                                                     unsigned long long* gctr);
// the guess is visited (its level's frontier is itself)
__global__ void k_spec_root(const unsigned long long* best, uint32_t* S) {
  const unsigned long long k = *best;
  if (k) {
    const uint32_t r = 0xFFFFFFFFu - (uint32_t)k;
    atomicOr(&S[r >> 4], 1u << (2 * (r & 15)));
  }
}
// a level's found ids (*found += |next|) and their arcs (*farcs += sum of deg over next)
__global__ void __launch_bounds__(BLOCK) k_farcs(const uint32_t* __restrict__ next, uint64_t nw,
                                                 const uint32_t* __restrict__ deg,
                                                 unsigned long long* found, unsigned long long* farcs) {
  unsigned long long s = 0;
  uint32_t c = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * BLOCK) {
    uint32_t x = next[w];
    c += __popc(x);
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      s += __ldg(&deg[w * 32 + b]);
    }
  }
  s = warp_sum(s);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) {
    atomicAdd(found, (unsigned long long)c);
    atomicAdd(farcs, s);
  }
}

// ---------------------------------------------------------------- degrees, bucketed
// The same count with shared-memory counters instead of L2 increments.  A random 4-byte
// increment costs one L2 request whichever way it is issued (the L2-resident ceiling measured
// by scripts/micro/l2_peaks.cu is ~195 G/s on this B200), while a shared-memory atomicAdd at a
// random slot runs at ~1.45 T/s (scripts/micro/smem_atomics.cu).  So the endpoints are first
// bucketed by id >> 15 (<= 2048 buckets of 2^15 ids: the counters of one bucket fill 128 KB of
// shared memory), then each bucket is counted by one block in shared memory:
//   k_deg_part  : one block per SM streams its share of the edge list (two register sets in
//                 turn keep the next round's 16-byte loads in flight); every endpoint claims a
//                 slot in its bucket's 32-entry shared-memory ring (one shared atomic); after
//                 each round of 8192 endpoints every ring holding >= 16 entries writes one
//                 32-byte group (u16: the id's low 15 bits) to its bucket's region in HBM.  The
//                 region is shared by all blocks (so only ~2048 lines are ever partly written
//                 and the L2 writes whole lines back), and its cursor is reserved one group
//                 ahead: the thread owning a bucket holds the position of its next group in a
//                 register, so the global atomic's latency is never waited for.  A full ring or
//                 region sends the endpoint straight to deg with an L2 increment: exact on any
//                 degree distribution, only slower on a pathological one.
//   k_deg_order : buckets by decreasing size (the heaviest are counted first: a hub's bucket
//                 is long and its same-address shared atomics serialise).
//   k_deg_count : one block per bucket counts its region in shared memory and adds to deg.
// Traffic: 8m (edges) + 4m (u16 entries out) + 4m (in) + 8n (deg read + write) bytes, against
// 8m per 2^24-id window (4 windows on C4) for the L2-increment count above.  Ids beyond 2^26
// are handled in super-windows of 2^26 ids (one edge-list pass each).
constexpr int DR_SPAN = 15;                       // ids per bucket: 2^15
constexpr uint32_t DR_NB = 2048;                  // buckets per super-window (2^26 ids)
constexpr int DR_CAP = 32;                        // ring entries per bucket (u16, 64 B)
constexpr int DR_THREADS = 1024;
constexpr int DR_VEC = 2;                         // uint4 (two edges) per thread per round
constexpr uint16_t DR_PAD = 0x8000;               // padding entry (counted into a dummy slot)
static_assert(DR_NB == 2 * DR_THREADS, "each k_deg_part thread owns two buckets");
constexpr uint32_t DR_Q = 1024;                   // entries per bucket per epoch of the region layout
struct DegRadix {
  uint16_t* reg;    // bucket regions, epoch-interleaved: entry pos of bucket b at dr_addr(b, pos)
  uint32_t* cur;    // [DR_NB] region cursors (entries reserved)
  uint32_t* order;  // [DR_NB] buckets by decreasing size
  uint32_t C;       // region capacity per bucket (entries, a multiple of DR_Q)
  uint32_t nbk;     // buckets of this super-window
};
// Epoch e holds entries [e*DR_Q, (e+1)*DR_Q) of every bucket, side by side: the buckets fill
// at similar rates, so the blocks' scattered group writes stay within a few MB of address
// space (TLB reach).  One region per bucket, each in its own pages, made the writes 2x slower
// (scripts/micro/deg_part_phases.cu).
CC_DEVI uint64_t dr_addr(const DegRadix& R, uint32_t b, uint32_t pos) {
  return ((uint64_t)(pos / DR_Q) * R.nbk + b) * DR_Q + (pos % DR_Q);
}
// Ring of bucket b: DR_CAP u16 slots (four 16-byte chunks, chunk index XOR-swizzled by bits 1-2
// of b so that rows 64 bytes apart do not share banks) and one packed word
// W[b] = (written-out << 16) | claimed, both renormalised to < 64 at every write-out.
CC_DEVI uint32_t dr_phys(uint32_t b, uint32_t pos) { return (pos & 31u) ^ ((b << 2) & 24u); }
// speculative root level carried by the degree pass (key == nullptr: off; see k_deg_sample)
struct SpecRoot {
  const unsigned long long* key;  // guess = ~(uint32_t)*key; 0: no guess
  uint32_t* S;                    // 2-bit BFS state (the guess already visited)
  uint32_t* next;                 // found bitmap
};
template <bool FULL>  // FULL: every id is in this super-window (lo = 0, n <= 2^26): no range test
__global__ void __launch_bounds__(DR_THREADS, 1)
k_deg_part(const uint4* __restrict__ e2, uint64_t m, uint32_t lo_arg, uint32_t nbk, DegRadix R,
           uint32_t* __restrict__ deg, SpecRoot sp) {
  extern __shared__ __align__(16) uint32_t dsm[];
  uint32_t* s_w = dsm;                                          // [DR_NB]
  uint16_t* s_row = reinterpret_cast<uint16_t*>(dsm + DR_NB);  // [DR_NB][DR_CAP]
  const uint32_t lo = FULL ? 0u : lo_arg;
  bool spec = false;
  uint32_t rg = 0;
  if (sp.key) {
    const unsigned long long k = *sp.key;
    spec = k != 0;
    rg = 0xFFFFFFFFu - (uint32_t)k;
  }
  // the guess's level: claim the other endpoint of every edge at the guess
  auto spec_edge = [&](uint32_t a, uint32_t b) {
    if (a == rg && b != rg) mark2(sp.S, sp.next, b);
    if (b == rg && a != rg) mark2(sp.S, sp.next, a);
  };
  for (uint32_t b = threadIdx.x; b < DR_NB; b += DR_THREADS) s_w[b] = 0;
  // this thread's buckets and the region position of their next 16-entry group
  const uint32_t ob[2] = {threadIdx.x, threadIdx.x + DR_THREADS};
  uint32_t opos[2];
#pragma unroll
  for (int i = 0; i < 2; i++) opos[i] = ob[i] < nbk ? atomicAdd(&R.cur[ob[i]], 16u) : 0xFFFFFFFFu;
  __syncthreads();
  const uint32_t G = gridDim.x, k = blockIdx.x;
  const uint64_t npair = m >> 1;  // uint4 = two edges
  constexpr uint32_t PER_ROUND = DR_THREADS * DR_VEC;
  const uint32_t rounds = (uint32_t)((npair + PER_ROUND - 1) / PER_ROUND);
  const uint32_t full_rounds = (uint32_t)(npair / PER_ROUND);  // rounds with every slot valid
  const uint32_t span_end = nbk << DR_SPAN;
  constexpr uint32_t LOWMASK = (1u << DR_SPAN) - 1;
  auto claim_store = [&](const uint32_t (&v)[4], int nv) {
    uint32_t old[4];
#pragma unroll
    for (int h = 0; h < 4; h++)  // the slot claims in flight together, then the stores
      old[h] = (h < nv && (FULL || v[h] < span_end)) ? atomicAdd(&s_w[v[h] >> DR_SPAN], 1u) : 0xFFFFFFFFu;
#pragma unroll
    for (int h = 0; h < 4; h++) {
      if (old[h] == 0xFFFFFFFFu) continue;
      const uint32_t b = v[h] >> DR_SPAN, w = old[h] & 0xFFFFu;
      if (w - (old[h] >> 16) < DR_CAP) s_row[b * DR_CAP + dr_phys(b, w)] = (uint16_t)(v[h] & LOWMASK);
      else atomicAdd(&deg[v[h] + lo], 1u);  // ring full this round
    }
  };
  if ((m & 1) && k == 0 && threadIdx.x == 0) {  // the last edge of an odd-length list
    const uint2 t = reinterpret_cast<const uint2*>(e2)[m - 1];
    const uint32_t v[4] = {t.x - lo, t.y - lo, 0u, 0u};
    claim_store(v, 2);
    if (spec) spec_edge(t.x, t.y);
  }
  // a thread's DR_VEC = 2 uint4 of a round are adjacent: one 256-bit load
  static_assert(DR_VEC == 2, "one 32-byte load per thread per round");
  auto load = [&](uint4 (&x)[DR_VEC], uint32_t r) {
    const uint4* p = e2 + (uint64_t)r * PER_ROUND + DR_VEC * threadIdx.x;
    if (r < full_rounds) {
      ldg_stream_v8(p, x[0], x[1]);
    } else if (r < rounds) {
#pragma unroll
      for (int j = 0; j < DR_VEC; j++)
        if ((uint64_t)r * PER_ROUND + DR_VEC * threadIdx.x + j < npair) x[j] = ldg_stream(p + j);
    }
  };
  // a full round of a FULL window: every endpoint is valid and in range, so there is no
  // sentinel; the ring store and the (rare) direct count are predicated rather than branched
  // (PTX predicates: ptxas had wrapped each in a BSSY/BRA pair), and the guess test is one
  // predicate per two edges.  k_deg_part on C4 5.78 -> 5.50 ms (profiles/r02/bench_c4_s6_pred*)
  const uint32_t row_base = (uint32_t)__cvta_generic_to_shared(s_row);
  auto insert_full = [&](const uint4 (&x)[DR_VEC]) {
#pragma unroll
    for (int j = 0; j < DR_VEC; j++) {
      const uint32_t v[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
      uint32_t old[4];
#pragma unroll
      for (int h = 0; h < 4; h++) old[h] = atomicAdd(&s_w[v[h] >> DR_SPAN], 1u);
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const uint32_t b = v[h] >> DR_SPAN, w = old[h] & 0xFFFFu;
        const uint32_t sa = row_base + 2u * (b * DR_CAP + dr_phys(b, w));
        // ring slot free: the u16 store; ring full this round: the direct count
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.lt.u32 p, %0, %4;\n\t"
            "@p st.shared.u16 [%1], %2;\n\t"
            "@!p red.global.add.u32 [%3], 1;\n\t}"
            :: "r"(w - (old[h] >> 16)), "r"(sa), "h"((unsigned short)(v[h] & LOWMASK)), "l"(deg + v[h]),
               "n"(DR_CAP) : "memory");
      }
    }
    if (spec) {
#pragma unroll
      for (int j = 0; j < DR_VEC; j++) {
        if (((x[j].x == rg) | (x[j].y == rg) | (x[j].z == rg) | (x[j].w == rg)) != 0) {
          spec_edge(x[j].x, x[j].y);
          spec_edge(x[j].z, x[j].w);
        }
      }
    }
  };
  auto insert_round = [&](const uint4 (&x)[DR_VEC], uint32_t r) {
    if (FULL && r < full_rounds) {
      insert_full(x);
      return;
    }
#pragma unroll
    for (int j = 0; j < DR_VEC; j++) {
      if (r >= full_rounds && (uint64_t)r * PER_ROUND + DR_VEC * threadIdx.x + j >= npair) continue;
      const uint32_t v[4] = {x[j].x - lo, x[j].y - lo, x[j].z - lo, x[j].w - lo};
      claim_store(v, 4);
      if (spec) {
        spec_edge(x[j].x, x[j].y);
        spec_edge(x[j].z, x[j].w);
      }
    }
  };
  // one group of 16 entries of bucket b (in registers) to its reserved region position
  auto put_group = [&](uint32_t b, uint32_t pos, const uint4& r0, const uint4& r1) {
    if (pos < R.C) {  // C and pos are multiples of 16
      st_v8(R.reg + dr_addr(R, b, pos), r0, r1);  // one 32-byte sector per group
    } else {  // region full: count directly
      const uint32_t wv[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
      const uint32_t bs = lo + (b << DR_SPAN);
#pragma unroll
      for (int h = 0; h < 8; h++) {
        if ((wv[h] & 0xFFFFu) != DR_PAD) atomicAdd(&deg[bs + (wv[h] & 0xFFFFu)], 1u);
        if ((wv[h] >> 16) != DR_PAD) atomicAdd(&deg[bs + (wv[h] >> 16)], 1u);
      }
    }
  };
  // write out one 16-entry group of each of this thread's rings holding one
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < 2; i++) {
      const uint32_t b = ob[i];
      const uint32_t wd = s_w[b];
      uint32_t w = wd & 0xFFFFu, f = wd >> 16;
      if (w - f < 16) continue;
      if (w - f > DR_CAP) w = f + DR_CAP;  // claims past the ring went to deg directly
      const uint32_t c0 = f & 16u;         // logical chunks c0/8, c0/8 + 1
      const uint4* row = reinterpret_cast<const uint4*>(s_row + b * DR_CAP);
      const uint4 r0 = row[dr_phys(b, c0) >> 3], r1 = row[dr_phys(b, c0 + 8) >> 3];
      f += 16;
      const uint32_t base = f & ~31u;
      s_w[b] = ((f - base) << 16) | (w - base);
      put_group(b, opos[i], r0, r1);
      opos[i] = atomicAdd(&R.cur[b], 16u);  // the next group's position, needed rounds later
    }
  };
  uint4 xa[DR_VEC], xb[DR_VEC];
  load(xa, k);
  for (uint32_t r = k; r < rounds; r += 2 * G) {
    load(xb, r + G);
    insert_round(xa, r);
    __syncthreads();
    flush();
    __syncthreads();
    if (r + G >= rounds) break;
    load(xa, r + 2 * G);
    insert_round(xb, r + G);
    __syncthreads();
    flush();
    __syncthreads();
  }
  // the ring leftovers (<= 16 per bucket) fill the reserved group, padded with DR_PAD
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const uint32_t b = ob[i];
    if (b >= nbk) continue;
    const uint32_t wd = s_w[b];
    const uint32_t w = wd & 0xFFFFu, f = wd >> 16;
    uint32_t e[16];
#pragma unroll
    for (int q = 0; q < 16; q++)
      e[q] = (f + q < w) ? s_row[b * DR_CAP + dr_phys(b, f + q)] : DR_PAD;
    uint4 r0, r1;
    r0.x = e[0] | (e[1] << 16); r0.y = e[2] | (e[3] << 16); r0.z = e[4] | (e[5] << 16); r0.w = e[6] | (e[7] << 16);
    r1.x = e[8] | (e[9] << 16); r1.y = e[10] | (e[11] << 16); r1.z = e[12] | (e[13] << 16); r1.w = e[14] | (e[15] << 16);
    put_group(b, opos[i], r0, r1);
  }
}
// order[rank] = bucket, by decreasing entry count (ties: smaller bucket first); each block
// ranks DR_ORDER_PER buckets against all of them (one block ranking all 2048 took 120 us)
constexpr uint32_t DR_ORDER_PER = 128;
__global__ void __launch_bounds__(DR_ORDER_PER) k_deg_order(DegRadix R, uint32_t nbk) {
  __shared__ uint32_t s_size[DR_NB];
  for (uint32_t b = threadIdx.x; b < nbk; b += blockDim.x) s_size[b] = min(R.cur[b], R.C);
  __syncthreads();
  for (uint32_t b = blockIdx.x * DR_ORDER_PER + threadIdx.x; b < nbk && b < (blockIdx.x + 1) * DR_ORDER_PER;
       b += blockDim.x) {
    const uint32_t sb = s_size[b];
    uint32_t rank = 0;
    for (uint32_t o = 0; o < nbk; o++) {
      const uint32_t so = s_size[o];
      rank += (so > sb) | ((so == sb) & (o < b));
    }
    R.order[rank] = b;
  }
}
__global__ void __launch_bounds__(DR_THREADS, 1)
k_deg_count(DegRadix R, uint32_t lo, uint64_t n, uint32_t* __restrict__ deg) {
  extern __shared__ __align__(16) uint32_t dsm[];
  uint32_t* s_cnt = dsm;  // [2^DR_SPAN + 1]: slot 2^DR_SPAN absorbs DR_PAD
  const uint32_t b = R.order[blockIdx.x];
  for (uint32_t i = threadIdx.x; i <= (1u << DR_SPAN); i += DR_THREADS) s_cnt[i] = 0;
  __syncthreads();
  // one warp per epoch chunk of this bucket (DR_Q entries = 128 vectors of 16 bytes)
  const uint32_t fill = min(R.cur[b], R.C);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t e = wid; e * DR_Q < fill; e += DR_THREADS / 32) {
    const uint4* src = reinterpret_cast<const uint4*>(R.reg + dr_addr(R, b, e * DR_Q));
    const uint32_t nv = min(DR_Q, fill - e * DR_Q) >> 3;  // a multiple of 2 (groups of 16)
    constexpr int U = DR_Q / 8 / 32;  // 4 vectors per lane
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (lane + u * 32 < nv) v[u] = ldg_stream(src + lane + u * 32);
#pragma unroll
    for (int u = 0; u < U; u++)
      if (lane + u * 32 < nv) {
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int h = 0; h < 4; h++) {
          atomicAdd(&s_cnt[w[h] & 0xFFFFu], 1u);
          atomicAdd(&s_cnt[w[h] >> 16], 1u);
        }
      }
  }
  __syncthreads();
  const uint64_t base = (uint64_t)lo + ((uint64_t)b << DR_SPAN);
  for (uint32_t i = threadIdx.x; i < (1u << DR_SPAN); i += DR_THREADS) {
    const uint32_t c = s_cnt[i];
    if (c && base + i < n) deg[base + i] += c;  // one block per bucket: plain add
  }
}
static bool deg_radix_plan(uint64_t m, uint64_t n, uint64_t scratch_bytes, uint64_t* nbk, uint64_t* C) {
  const uint64_t nb_all = (n + (1u << DR_SPAN) - 1) >> DR_SPAN;
  *nbk = std::min<uint64_t>(nb_all, DR_NB);
  const uint64_t mean = (2 * m + nb_all - 1) / nb_all;  // entries per bucket
  // 4x the mean (R-MAT 26: the heaviest bucket holds ~2.6x), less if the scratch is short; plus
  // the groups reserved ahead and padded (one per bucket per block)
  const uint64_t head = 256 + sizeof(uint32_t) * 2 * DR_NB;
  const uint64_t fit = scratch_bytes > head ? (scratch_bytes - head) / (*nbk * sizeof(uint16_t)) : 0;
  uint64_t c = std::min<uint64_t>(4 * mean + 16 * 160 * 2, fit);
  c = c / DR_Q * DR_Q;
  *C = c;
  return c >= 2 * mean && c < (1ull << 31);
}
static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}
uint64_t degree_radix_scratch(uint64_t m, uint64_t n) {
  const uint64_t nb_all = (n + (1u << DR_SPAN) - 1) >> DR_SPAN;
  const uint64_t nbk = std::min<uint64_t>(nb_all, DR_NB);
  const uint64_t mean = (2 * m + nb_all - 1) / nb_all;
  return 256 + sizeof(uint32_t) * 2 * DR_NB + nbk * sizeof(uint16_t) * (4 * mean + 16 * 160 * 2);
}
uint64_t spec_min_edges() {
  const char* e = getenv("CC_SPEC_MIN_EDGES");  // test hook: exercise the guess on small lists
  return e ? strtoull(e, nullptr, 10) : SPEC_MIN_EDGES;
}
bool launch_degree_radix(const uint2* edges, uint64_t m, uint64_t n, uint32_t* deg, void* scratch,
                         uint64_t scratch_bytes, uint32_t* /*cursor*/, cudaStream_t st, const SpecLevel* spec,
                         bool* spec_ran) {
  *spec_ran = false;
  if (!m || !n) return true;
  uint64_t nbk, C;
  if (!deg_radix_plan(m, n, scratch_bytes, &nbk, &C)) return false;
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch);
  DegRadix R;
  R.C = (uint32_t)C;
  R.nbk = (uint32_t)nbk;
  R.cur = reinterpret_cast<uint32_t*>(p);
  R.order = R.cur + DR_NB;
  R.reg = reinterpret_cast<uint16_t*>(p + 256 + sizeof(uint32_t) * 2 * DR_NB);
  static bool attr = false;
  const int smem_part = DR_NB * sizeof(uint32_t) + DR_NB * DR_CAP * sizeof(uint16_t);
  const int smem_count = ((1 << DR_SPAN) + 1) * sizeof(uint32_t);
  if (!attr) {
    cudaFuncSetAttribute(k_deg_part<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_part);
    cudaFuncSetAttribute(k_deg_part<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_part);
    cudaFuncSetAttribute(k_deg_count, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_count);
    attr = true;
  }
  const int G = sm_count();
  // speculative root level: the prefix [0, m0) is counted by k_deg_sample (and its guess's
  // edges claimed by a root-level pass over it), the degree pass counts [m0, m)
  uint64_t m0 = 0;
  SpecRoot sp{nullptr, nullptr, nullptr};
  if (spec && m >= spec_min_edges()) {
    const char* es = getenv("CC_SPEC_SAMPLE_EDGES");  // test hook
    // a multiple of 4 edges: the degree pass reads the rest with 32-byte loads
    m0 = std::min<uint64_t>(es ? strtoull(es, nullptr, 10) : SPEC_SAMPLE_EDGES, m / 2) & ~3ull;
    auto* gc = reinterpret_cast<unsigned long long*>(spec->gctr);
    k_deg_sample<<<grid_for(m0 / 2, 148 * 4), BLOCK, 0, st>>>(reinterpret_cast<const uint4*>(edges), m0 / 2,
                                                              deg, gc + G_GUESS);
    k_spec_root<<<1, 1, 0, st>>>(gc + G_GUESS, spec->S);
    k_bfs_level<true, false><<<grid_for((m0 + 1) / 2, 148 * 8), BLOCK, 0, st>>>(
        edges, m0, 0u, gc + G_GUESS, spec->S, spec->next, nullptr, gc);
    sp = SpecRoot{gc + G_GUESS, spec->S, spec->next};
    *spec_ran = true;
  }
  const uint4* e2 = reinterpret_cast<const uint4*>(edges + m0);
  const uint64_t mr = m - m0;
  for (uint64_t lo = 0; lo < n; lo += (uint64_t)DR_NB << DR_SPAN) {
    const uint32_t nb = (uint32_t)std::min<uint64_t>(DR_NB, (n - lo + (1u << DR_SPAN) - 1) >> DR_SPAN);
    R.nbk = nb;
    cudaMemsetAsync(R.cur, 0, sizeof(uint32_t) * DR_NB, st);
    if (lo == 0 && n <= ((uint64_t)DR_NB << DR_SPAN))
      k_deg_part<true><<<G, DR_THREADS, smem_part, st>>>(e2, mr, 0u, nb, R, deg, sp);
    else
      k_deg_part<false><<<G, DR_THREADS, smem_part, st>>>(e2, mr, (uint32_t)lo, nb, R, deg,
                                                          lo == 0 ? sp : SpecRoot{nullptr, nullptr, nullptr});
    k_deg_order<<<(nb + DR_ORDER_PER - 1) / DR_ORDER_PER, DR_ORDER_PER, 0, st>>>(R, nb);
    k_deg_count<<<nb, DR_THREADS, smem_count, st>>>(R, (uint32_t)lo, n, deg);
  }
  return true;
}

// Degree distribution D[d] = #{v : deg(v) = d}, d >= 1 (C10), plus n_present and the
// (max degree, smallest argmax) key used for the BFS root (C13).  Shared-memory bins for
// small degrees (where all the mass is), global bins up to 2^20, a tail list beyond.
constexpr int SBINS = 2048;
constexpr int HLOC = 8;  // degrees 1..HLOC are counted in registers (most ids; no atomics)
__global__ void __launch_bounds__(BLOCK) k_deg_hist(const uint32_t* __restrict__ deg, uint64_t n,
                                                    uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ tail,
                                                    unsigned long long* gctr, uint64_t id0) {
  __shared__ uint32_t sh[SBINS];
  for (int i = threadIdx.x; i < SBINS; i += BLOCK) sh[i] = 0;
  __syncthreads();
  uint32_t npres = 0, loc[HLOC];
#pragma unroll
  for (int j = 0; j < HLOC; j++) loc[j] = 0;
  unsigned long long best = 0;
  auto add = [&](uint32_t d, uint64_t v) {
    if (!d) return;
    npres++;
    const unsigned long long key = ((unsigned long long)d << 32) | (0xFFFFFFFFu - (uint32_t)(v + id0));
    best = key > best ? key : best;
    if (d <= HLOC) {
#pragma unroll
      for (int j = 0; j < HLOC; j++) loc[j] += (d == (uint32_t)j + 1);
    } else if (d < SBINS) {
      atomicAdd(&sh[d], 1u);
    } else if (d < HIST_DENSE) {
      atomicAdd(&hist[d], 1u);
    } else {
      const unsigned long long pos = atomicAdd(&gctr[G_TAIL], 1ull);
      if (pos < TAIL_CAP) tail[pos] = d;
    }
  };
  const uint64_t n4 = n >> 2;  // 16-byte loads (deg is 16-byte aligned), two in flight
  const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
  uint64_t q = blockIdx.x * (uint64_t)BLOCK + threadIdx.x;
  for (; q + stride < n4; q += 2 * stride) {
    const uint4 d = reinterpret_cast<const uint4*>(deg)[q];
    const uint4 e = reinterpret_cast<const uint4*>(deg)[q + stride];
    add(d.x, 4 * q); add(d.y, 4 * q + 1); add(d.z, 4 * q + 2); add(d.w, 4 * q + 3);
    const uint64_t r = q + stride;
    add(e.x, 4 * r); add(e.y, 4 * r + 1); add(e.z, 4 * r + 2); add(e.w, 4 * r + 3);
  }
  if (q < n4) {
    const uint4 d = reinterpret_cast<const uint4*>(deg)[q];
    add(d.x, 4 * q); add(d.y, 4 * q + 1); add(d.z, 4 * q + 2); add(d.w, 4 * q + 3);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) add(deg[4 * n4 + threadIdx.x], 4 * n4 + threadIdx.x);
#pragma unroll
  for (int j = 0; j < HLOC; j++) {
    const uint32_t t = warp_sum(loc[j]);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(&sh[j + 1], t);
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
// non-empty dense bins as (degree, count) pairs (unordered): only these reach the host
__global__ void k_hist_pairs(const uint32_t* __restrict__ hist, uint64_t nb, uint2* __restrict__ out,
                             unsigned long long* cnt) {
  for (uint64_t b0 = blockIdx.x * (uint64_t)BLOCK; b0 < nb; b0 += (uint64_t)gridDim.x * BLOCK) {
    const uint64_t d = b0 + threadIdx.x;
    const uint32_t c = (d < nb && d > 0) ? hist[d] : 0u;
    const uint32_t mask = __ballot_sync(0xffffffffu, c != 0);
    if (!mask) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(cnt, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (c) out[base + __popc(mask & ((1u << lane) - 1u))] = make_uint2((uint32_t)d, c);
  }
}
void launch_hist_pairs(const uint32_t* hist, uint64_t nb, uint2* out, uint64_t* cnt, cudaStream_t st) {
  cudaMemsetAsync(cnt, 0, sizeof(uint64_t), st);
  if (nb) k_hist_pairs<<<grid_for(nb, 148 * 4), BLOCK, 0, st>>>(hist, nb, out, reinterpret_cast<unsigned long long*>(cnt));
}
void launch_deg_hist(const uint32_t* deg, uint64_t n, uint32_t* hist, uint32_t* tail,
                     uint64_t* gctr, cudaStream_t st, uint64_t base) {
  if (!n) return;
  k_deg_hist<<<grid_for(n, 148 * 4), BLOCK, 0, st>>>(deg, n, hist, tail,
                                                       reinterpret_cast<unsigned long long*>(gctr), base);
}

// ---------------------------------------------------------------- BFS peel
// Level-synchronous BFS from the root (Alg. 2 lines 7-8) over the edge
// list.  Vertex state is 2 bits (bit 0 visited, bit 1 in the current frontier), 16 ids per
// word, so one random read per endpoint answers both questions; a frontier endpoint claims
// its unvisited neighbour with atomicOr on the visited bit and marks it in `next`.
// Level 1 (frontier = {root}) compares ids instead of reading state.  From the level whose
// frontier holds a fifth of the current arcs (or once most vertices are visited), each level
// also compacts the edge list to the edges that can still matter -- an endpoint unvisited
// after the level (a frontier endpoint's neighbour is visited by then, by this or another
// edge) -- staged per warp in shared memory and written in runs, so later levels and the
// filter stream only those.  (edge-streaming bitmap BFS.)
// root_key (root level only): root = ~(uint32_t)*root_key, no level if 0 (the speculative
// level)
template <bool ROOT, bool COMPACT>
__global__ void __launch_bounds__(BLOCK) k_bfs_level(const uint2* __restrict__ e, uint64_t m,
                                                     uint32_t root, const unsigned long long* root_key,
                                                     uint32_t* S, uint32_t* next,
                                                     uint2* __restrict__ out,
                                                     unsigned long long* gctr) {
  if (ROOT && root_key) {
    const unsigned long long k = *root_key;
    if (!k) return;
    root = 0xFFFFFFFFu - (uint32_t)k;
  }
  // compaction: survivors are staged per warp in shared memory and flushed in runs (one
  // global cursor atomic per run, coalesced stores)
  constexpr int WBUF = COMPACT ? 256 : 1;
  __shared__ uint2 s_buf[BLOCK / 32][WBUF];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t nbuf = 0;  // warp-uniform
  auto flush = [&]() {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&gctr[G_REMAIN], (unsigned long long)nbuf);
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();
    for (uint32_t i = lane; i < nbuf; i += 32) out[base + i] = s_buf[wid][i];
    __syncwarp();
    nbuf = 0;
  };
  // EPT edges per thread per step, one 256-bit load (the list is 32-byte aligned): 2 EPT
  // state reads in flight per thread
  constexpr int EPT = 4;
  const uint64_t stride = (uint64_t)gridDim.x * BLOCK * EPT;
  const uint64_t iters = (m + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; it++) {
    const uint64_t i0 = it * stride + (blockIdx.x * (uint64_t)BLOCK + threadIdx.x) * EPT;
    uint2 x[EPT];
    bool keep[EPT] = {false, false, false, false};
    int cnt = 0;
    if (i0 + EPT <= m) {
      uint4 q0, q1;
      ldg_stream_v8(e + i0, q0, q1);
      x[0] = make_uint2(q0.x, q0.y); x[1] = make_uint2(q0.z, q0.w);
      x[2] = make_uint2(q1.x, q1.y); x[3] = make_uint2(q1.z, q1.w);
      cnt = EPT;
    } else {
#pragma unroll
      for (int j = 0; j < EPT; j++)
        if (i0 + j < m) { x[j] = e[i0 + j]; cnt = j + 1; }
    }
#pragma unroll
    for (int j = 0; j < EPT; j++) {
      if (j >= cnt) continue;
      const uint32_t a = x[j].x, b = x[j].y;
      if (ROOT) {
        if (a == root && b != root) mark2(S, next, b);
        if (b == root && a != root) mark2(S, next, a);
      } else {
        const uint32_t sa = st2(S, a), sb = st2(S, b);
        if ((sa & 2u) && !(sb & 1u)) mark2(S, next, b);
        if ((sb & 2u) && !(sa & 1u)) mark2(S, next, a);
        // after this level a frontier endpoint's neighbour is visited (by this or another
        // edge): an edge whose endpoints are both visited then can no longer matter
        const bool va = (sa & 1u) || (sb & 2u), vb = (sb & 1u) || (sa & 2u);
        keep[j] = !(va && vb);
      }
    }
    if (COMPACT) {
      const uint32_t lt = lanemask_lt();
#pragma unroll
      for (int j = 0; j < EPT; j++) {
        const uint32_t mk = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) s_buf[wid][nbuf + __popc(mk & lt)] = x[j];
        nbuf += __popc(mk);
      }
      if (nbuf > (uint32_t)(COMPACT ? WBUF - 32 * EPT : 0)) flush();
    }
  }
  if (COMPACT && nbuf) flush();
}
// After a level: frontier bits <- next, visited bits |= next (set by this rank's claims
// already; with several ranks `next` also holds the other ranks' finds).
__global__ void k_bfs_advance(uint32_t* S, const uint32_t* __restrict__ next, uint64_t nw2) {
  for (uint64_t w = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; w < nw2; w += (uint64_t)gridDim.x * BLOCK) {
    const uint32_t nb = (next[w >> 1] >> (16 * (w & 1))) & 0xFFFFu;
    // spread 16 bits to the odd positions of 32
    uint32_t x = nb;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    S[w] = (S[w] & 0x55555555u) | x | (x << 1);
  }
}
void launch_bfs_level(bool root_level, bool compact, const uint2* edges, uint64_t m, uint32_t root,
                      uint32_t* S, uint32_t* next, uint2* out, uint64_t* gctr, cudaStream_t st) {
  if (!m) return;
  const unsigned g = grid_for((m + 3) / 4, 148 * 8);
  auto* c = reinterpret_cast<unsigned long long*>(gctr);
  if (root_level) k_bfs_level<true, false><<<g, BLOCK, 0, st>>>(edges, m, root, nullptr, S, next, out, c);
  else if (compact) k_bfs_level<false, true><<<g, BLOCK, 0, st>>>(edges, m, root, nullptr, S, next, out, c);
  else k_bfs_level<false, false><<<g, BLOCK, 0, st>>>(edges, m, root, nullptr, S, next, out, c);
}
void launch_farcs(const uint32_t* next, uint64_t n, const uint32_t* deg, uint64_t* found, uint64_t* farcs,
                  cudaStream_t st) {
  const uint64_t nw = (n + 31) / 32;
  if (nw)
    k_farcs<<<grid_for(nw, 148 * 8), BLOCK, 0, st>>>(next, nw, deg, reinterpret_cast<unsigned long long*>(found),
                                                      reinterpret_cast<unsigned long long*>(farcs));
}
// One pass after a level: the level's found ids (*found += |next|) and their arcs (*farcs),
// S advanced (frontier <- next, visited |= next) and next cleared for the following level
// (replaces k_farcs + k_bfs_advance + a memset of next: one pass over the state instead of three)
__global__ void __launch_bounds__(BLOCK) k_farcs_advance(uint32_t* __restrict__ next, uint32_t* __restrict__ S,
                                                         uint64_t nw, const uint32_t* __restrict__ deg,
                                                         unsigned long long* found, unsigned long long* farcs) {
  unsigned long long s = 0;
  uint32_t c = 0;
  auto spread = [](uint32_t x) {  // 16 bits to the odd positions of 32
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
  };
  for (uint64_t w = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * BLOCK) {
    uint32_t x = next[w];
    if (x) next[w] = 0;
    const uint2 sv = reinterpret_cast<const uint2*>(S)[w];
    const uint32_t lo = spread(x & 0xFFFFu), hi = spread(x >> 16);
    const uint2 nv = make_uint2((sv.x & 0x55555555u) | lo | (lo << 1), (sv.y & 0x55555555u) | hi | (hi << 1));
    if (nv.x != sv.x || nv.y != sv.y) reinterpret_cast<uint2*>(S)[w] = nv;
    c += __popc(x);
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      s += __ldg(&deg[w * 32 + b]);
    }
  }
  s = warp_sum(s);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) {
    atomicAdd(found, (unsigned long long)c);
    atomicAdd(farcs, s);
  }
}
void launch_farcs_advance(uint32_t* next, uint32_t* S, uint64_t n, const uint32_t* deg, uint64_t* found,
                          uint64_t* farcs, cudaStream_t st) {
  const uint64_t nw = (n + 31) / 32;
  if (nw)
    k_farcs_advance<<<grid_for(nw, 148 * 8), BLOCK, 0, st>>>(next, S, nw, deg, reinterpret_cast<unsigned long long*>(found),
                                                             reinterpret_cast<unsigned long long*>(farcs));
}
void launch_bfs_advance(uint32_t* S, const uint32_t* next, uint64_t n, cudaStream_t st) {
  const uint64_t nw2 = (n + 15) / 16;
  if (nw2) k_bfs_advance<<<grid_for(nw2, 148 * 8), BLOCK, 0, st>>>(S, next, nw2);
}

// Filter (Alg. 2 lines 10-11): E <- E \ {(u,v) | u in VI}.  Both arcs of
// an edge are stored, so keeping edges with an unvisited first endpoint removes both
// directions (C15).  Block-aggregated compaction.
__global__ void __launch_bounds__(BLOCK) k_filter(const uint2* __restrict__ e, uint64_t m,
                                                  const uint32_t* __restrict__ S,
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
      keep = !(st2(S, x.x) & 1u);
    }
    uint32_t tot;
    uint32_t off = block_excl_scan<BLOCK>(keep, s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(&gctr[G_REMAIN], (unsigned long long)tot) : 0ull;
    __syncthreads();
    if (keep) out[s_base + off] = x;
    __syncthreads();
  }
}
void launch_filter(const uint2* edges, uint64_t m, const uint32_t* S, uint2* out,
                   uint64_t* gctr, cudaStream_t st) {
  if (!m) return;
  k_filter<<<grid_for(m, 148 * 8), BLOCK, 0, st>>>(edges, m, S, out,
                                                     reinterpret_cast<unsigned long long*>(gctr));
}

// visited bitmap (1 bit per id) from the 2-bit state, for the SV presence test
__global__ void k_vis_bits(const uint32_t* __restrict__ S, uint64_t nw, uint32_t* __restrict__ vis) {
  for (uint64_t w = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * BLOCK) {
    uint32_t lo = S[2 * w] & 0x55555555u, hi = S[2 * w + 1] & 0x55555555u;
    // compress even bits to 16
    auto pack = [](uint32_t x) {
      x = (x | (x >> 1)) & 0x33333333u;
      x = (x | (x >> 2)) & 0x0F0F0F0Fu;
      x = (x | (x >> 4)) & 0x00FF00FFu;
      x = (x | (x >> 8)) & 0x0000FFFFu;
      return x;
    };
    vis[w] = pack(lo) | (pack(hi) << 16);
  }
}
void launch_vis_bits(const uint32_t* S, uint64_t n, uint32_t* vis, cudaStream_t st) {
  const uint64_t nw = (n + 31) / 32;
  if (nw) k_vis_bits<<<grid_for(nw, 148 * 8), BLOCK, 0, st>>>(S, nw, vis);
}

CC_DEVI bool bit(const uint32_t* bm, uint32_t v) { return (__ldg(&bm[v >> 5]) >> (v & 31)) & 1u; }

// L_bfs = min id in VI: first set bit of the visited bitmap.  Each thread's
// first set bit (its words are visited in increasing order), min over the warp, one atomic
// per warp (one per thread serialised ~150 k atomics on one address: 98 us on C4).
__global__ void k_min_visited(const uint32_t* __restrict__ vis, uint64_t nwords,
                              unsigned long long* gctr) {
  unsigned long long mn = ~0ull;
  for (uint64_t w = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; w < nwords;
       w += (uint64_t)gridDim.x * BLOCK) {
    const uint32_t x = vis[w];
    if (x) {
      mn = w * 32 + (__ffs(x) - 1);
      break;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, mn, o);
    mn = y < mn ? y : mn;
  }
  if ((threadIdx.x & 31) == 0 && mn != ~0ull) atomicMin(&gctr[G_MINVIS], mn);
}
void launch_min_visited(const uint32_t* visited, uint64_t n, uint64_t* gctr, cudaStream_t st) {
  uint64_t nw = (n + 31) / 32;
  if (!nw) return;
  k_min_visited<<<grid_for(nw, 148 * 4), BLOCK, 0, st>>>(visited, nw,
                                                           reinterpret_cast<unsigned long long*>(gctr));
}

// label[v] = L_bfs for v in VI, v otherwise (the initial label of every other id, written here
// so the BFS route needs no separate initialisation pass): 4 ids per thread, 16-byte stores
__global__ void k_bfs_labels(const uint32_t* __restrict__ vis, uint64_t n,
                             uint32_t* __restrict__ label, const unsigned long long* gctr) {
  const uint32_t L = (uint32_t)gctr[G_MINVIS];
  const uint64_t n4 = n >> 2;
  for (uint64_t q = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; q < n4; q += (uint64_t)gridDim.x * BLOCK) {
    const uint32_t b = (__ldg(&vis[q >> 3]) >> (4 * (q & 7))) & 15u;
    const uint32_t v = (uint32_t)(4 * q);
    reinterpret_cast<uint4*>(label)[q] =
        make_uint4(b & 1u ? L : v, b & 2u ? L : v + 1, b & 4u ? L : v + 2, b & 8u ? L : v + 3);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const uint32_t v = (uint32_t)(4 * n4 + threadIdx.x);
    label[v] = bit(vis, v) ? L : v;
  }
}
void launch_bfs_labels(const uint32_t* visited, uint64_t n, uint32_t* label, uint64_t* gctr,
                       cudaStream_t st) {
  if (!n) return;
  k_bfs_labels<<<grid_for((n + 3) / 4, 148 * 16), BLOCK, 0, st>>>(
      visited, n, label, reinterpret_cast<const unsigned long long*>(gctr));
}

// components = #{v : label[v] = v} over [lo, hi) (every component has exactly one root,
// its minimum id); added to *cnt
__global__ void k_count_roots_small(const uint32_t* __restrict__ label, uint64_t lo, uint64_t hi,
                                    unsigned long long* cnt) {
  const uint64_t v = lo + threadIdx.x;
  const uint32_t c = warp_sum(v < hi && label[v] == (uint32_t)v ? 1u : 0u);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}
__global__ void k_count_roots(const uint32_t* __restrict__ label, uint64_t lo, uint64_t hi,
                              unsigned long long* cnt) {
  uint32_t c = 0;
  // 16-byte loads over the aligned middle [a, b), single ids at the ends (hi - lo >= 8: a < b)
  const uint64_t a = (lo + 3) & ~3ull, b = hi & ~3ull;
  for (uint64_t q = a / 4 + blockIdx.x * (uint64_t)BLOCK + threadIdx.x; q < b / 4; q += (uint64_t)gridDim.x * BLOCK) {
    const uint4 x = reinterpret_cast<const uint4*>(label)[q];
    const uint32_t v = (uint32_t)(4 * q);
    c += (x.x == v) + (x.y == v + 1) + (x.z == v + 2) + (x.w == v + 3);
  }
  if (blockIdx.x == 0 && threadIdx.x < 8) {
    const uint64_t v = threadIdx.x < 4 ? lo + threadIdx.x : b + (threadIdx.x - 4);
    if (threadIdx.x < 4 ? v < a : v < hi) c += label[v] == (uint32_t)v;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}
void launch_count_roots(const uint32_t* label, uint64_t lo, uint64_t hi, uint64_t* cnt, cudaStream_t st) {
  if (hi <= lo) return;
  if (hi - lo < 8) {  // tiny ranges: one thread per id
    k_count_roots_small<<<1, BLOCK, 0, st>>>(label, lo, hi, reinterpret_cast<unsigned long long*>(cnt));
    return;
  }
  k_count_roots<<<grid_for((hi - lo + 3) / 4, 148 * 8), BLOCK, 0, st>>>(label, lo, hi,
                                                                      reinterpret_cast<unsigned long long*>(cnt));
}

// ------------------------------------------------------------- remainder renumbering
// (DESIGN.md §5.3).  Alg. 1 only compares ids (minima, equality), so running it on the
// remainder's endpoints renumbered in id order gives the same partitions, tuples and counters
// (PAPER.md:133-178); the labels map back through inv.  Saves the id-range-sized passes of the
// SV (slot clears and scans, CSR offsets) when the remainder is small (C4: 21 k of 67 M ids).
__global__ void k_sub_mark(const uint2* __restrict__ e, uint64_t m, uint32_t* bm) {
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < m; i += (uint64_t)gridDim.x * BLOCK) {
    const uint2 x = e[i];
    atomicOr(&bm[x.x >> 5], 1u << (x.x & 31));
    atomicOr(&bm[x.y >> 5], 1u << (x.y & 31));
  }
}
constexpr int SUBW = 16;                       // bitmap words per thread
constexpr uint64_t SUB_TILE = (uint64_t)BLOCK * SUBW;
uint64_t sub_bsum_words(uint64_t nw) { return (nw + SUB_TILE - 1) / SUB_TILE + 1; }
__global__ void __launch_bounds__(BLOCK) k_sub_bsum(const uint32_t* __restrict__ bm, uint64_t nw,
                                                    uint32_t* __restrict__ bsum) {
  __shared__ uint32_t s_scan[BLOCK / 32 + 1];
  const uint64_t w0 = blockIdx.x * SUB_TILE + (uint64_t)threadIdx.x * SUBW;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < SUBW; k++)
    if (w0 + k < nw) c += __popc(bm[w0 + k]);
  uint32_t tot;
  block_excl_scan<BLOCK>(c, s_scan, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(BLOCK) k_sub_rank(const uint32_t* __restrict__ bm, uint64_t nw,
                                                    const uint32_t* __restrict__ bsum,
                                                    uint32_t* __restrict__ wpre,
                                                    unsigned long long* total) {
  __shared__ uint32_t s_scan[BLOCK / 32 + 1];
  // this tile's offset: the sum of the earlier tiles' counts
  uint32_t before = 0;
  for (uint32_t j = threadIdx.x; j < blockIdx.x; j += BLOCK) before += bsum[j];
  uint32_t pref;
  block_excl_scan<BLOCK>(before, s_scan, &pref);
  const uint64_t w0 = blockIdx.x * SUB_TILE + (uint64_t)threadIdx.x * SUBW;
  uint32_t c[SUBW], sum = 0;
#pragma unroll
  for (int k = 0; k < SUBW; k++) {
    c[k] = w0 + k < nw ? __popc(bm[w0 + k]) : 0u;
    sum += c[k];
  }
  uint32_t tot;
  uint32_t run = pref + block_excl_scan<BLOCK>(sum, s_scan, &tot);
#pragma unroll
  for (int k = 0; k < SUBW; k++) {
    if (w0 + k < nw) wpre[w0 + k] = run;
    run += c[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = (unsigned long long)pref + tot;
}
void launch_sub_mark(const uint2* edges, uint64_t m, uint32_t* bm, cudaStream_t st) {
  if (m) k_sub_mark<<<grid_for(m, 148 * 8), BLOCK, 0, st>>>(edges, m, bm);
}
void launch_sub_rank(const uint32_t* bm, uint64_t nw, uint32_t* bsum, uint32_t* wpre, uint64_t* total,
                     cudaStream_t st) {
  if (!nw) return;
  const unsigned tiles = (unsigned)((nw + SUB_TILE - 1) / SUB_TILE);
  k_sub_bsum<<<tiles, BLOCK, 0, st>>>(bm, nw, bsum);
  k_sub_rank<<<tiles, BLOCK, 0, st>>>(bm, nw, bsum, wpre, reinterpret_cast<unsigned long long*>(total));
}
CC_DEVI uint32_t sub_rank_of(const uint32_t* bm, const uint32_t* wpre, uint32_t x) {
  return wpre[x >> 5] + __popc(bm[x >> 5] & ((1u << (x & 31)) - 1u));
}
__global__ void k_sub_edges(const uint2* __restrict__ e, uint64_t m, const uint32_t* __restrict__ bm,
                            const uint32_t* __restrict__ wpre, const uint32_t* __restrict__ deg,
                            uint2* __restrict__ out, uint32_t* __restrict__ inv, uint32_t* __restrict__ sdeg) {
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < m; i += (uint64_t)gridDim.x * BLOCK) {
    const uint2 x = e[i];
    const uint32_t ru = sub_rank_of(bm, wpre, x.x), rv = sub_rank_of(bm, wpre, x.y);
    out[i] = make_uint2(ru, rv);
    // every arc of an endpoint writes the same values (benign)
    inv[ru] = x.x;
    inv[rv] = x.y;
    sdeg[ru] = deg[x.x];
    sdeg[rv] = deg[x.y];
  }
}
void launch_sub_edges(const uint2* edges, uint64_t m, const uint32_t* bm, const uint32_t* wpre,
                      const uint32_t* deg, uint2* out, uint32_t* inv, uint32_t* sdeg, cudaStream_t st) {
  if (m) k_sub_edges<<<grid_for(m, 148 * 8), BLOCK, 0, st>>>(edges, m, bm, wpre, deg, out, inv, sdeg);
}
__global__ void k_sub_labels(const uint32_t* __restrict__ inv, const uint32_t* __restrict__ slabel,
                             uint64_t ns, uint32_t* __restrict__ label) {
  for (uint64_t i = blockIdx.x * (uint64_t)BLOCK + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * BLOCK)
    label[inv[i]] = inv[slabel[i]];
}
void launch_sub_labels(const uint32_t* inv, const uint32_t* slabel, uint64_t ns, uint32_t* label,
                       cudaStream_t st) {
  if (ns) k_sub_labels<<<grid_for(ns, 148 * 8), BLOCK, 0, st>>>(inv, slabel, ns, label);
}

}  // namespace graph
}  // namespace cc
