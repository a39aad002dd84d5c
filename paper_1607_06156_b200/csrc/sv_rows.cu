// sv_rows.cu -- row passes of the r-stationary SV engine.
//
// The tuple array is stored in CSR order (R sorted, vertex bucket VB(u) = one contiguous row,
// see sv_csr.cu).  Because a row is contiguous, the vertex-bucket minimum of Alg. 1
// (lines 9-13 / line 24) is a reduction over one run of the array, and
// the partition-bucket update that consumes it (lines 15-16 / line 25) can
// run in the same pass: q = u_min(r) is never written out and read back.  Each iteration of
// Alg. 1 is two streaming passes over (R, P):
//
//   pass A  (lines 8-16)   p <- PB[p]   (line 25 relabel of the previous iteration, if any)
//                          u_min(r), PC(r) = [min p = max p] per row      (lines 9-13)
//                          PA[p] <- min(PA[p], u_min(r))                   (lines 15-16)
//                          NCP(u_min(r)) for a row that is not PC (see below)
//   pass B  (lines 17-25)  completed(p) = PA[p] = p and not NCP(p): the tuple leaves and its
//                          vertex takes label p (lines 17-21);
//                          otherwise p <- PA[p]                             (line 19)
//                          u_min'(r) over the row plus the temporary <r,_,r> when TB(r)
//                          (line 22 + line 24, fig:doubling PAPER.md:189-197)
//                          PB[p] <- min(PB[p], u_min'(r)); the temporary's own q goes to
//                          PB[r]                                           (line 25)
//
// Completion needs only one flag per non-PC row: a partition p with a tuple in a row whose
// minimum m is below p gets p_min <= m < p and is not completed anyway, so only p = m can
// be completed-but-for-this-row; NCP(m) is the paper's "not all tuples potentially
// completed" for exactly the partitions where it decides.
//
// Work split.  A persistent block stages 2048-tuple tiles (8 per thread) in shared memory by
// TMA, together with R[t0-4, t0) and the 32 tuples past the tile; run minima are branch-free
// segmented scans (thread, warp, block), and a row that continues past the tile edge is
// finished by the tile that holds its head (the last warp reads the extension), so every row
// is reduced and applied by exactly one block.  Rows longer than LONG tuples (hubs) are
// listed once per compaction as segments of at most LSEG tuples and handled by warps in two
// small kernels (segment partials into epoch-tagged 64-bit slots whose newer tags always win
// the atomic, then the apply).  Partition slots PA/PB are n-sized u32 arrays; only slots of
// the iteration's partition list are ever written (k_pstat1/k_pstat2/k_list_from_bits keep
// them clean), updates q = p are skipped (PA preset / k_pstat2's temporary fold), and in hot
// iterations (few partitions per live tuple) each block min-reduces its updates in a
// shared-memory table first.  Every pass is compiled per (pass, hot, relabel, preset/
// exclusion) so each variant carries only its own code and shared memory; with the previous
// iteration's counters (prevctr) both hot variants are launched and the device runs one,
// which lets the host enqueue the next iteration before reading the counters.
#include <algorithm>
#include <cstdlib>

#include "csr.cuh"
#include "sv.cuh"

namespace cc {
namespace csr {

namespace {

constexpr int RB = 256;
constexpr int RITEMS = 8;

constexpr int PB = 256;               // row-pass block: 8 warps, tiles of PB * RITEMS tuples (128: slower)
constexpr int PTILE = PB * RITEMS;
constexpr int RCACHE = 512;
// long-row segment kernels: LU loads of a lane in flight (a warp walks a 1024-tuple segment;
// one dependent load per step left them latency-bound: k_long2 5.5 ms on C4 mode sv)
constexpr int LU = 8;
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr uint32_t DEAD = 0xFFFFFFFFu;
constexpr uint32_t FULL = 0xFFFFFFFFu;
// completed partition p (PA[p] = p and not NCP(p)): k_pstat1 sets this flag on PA[p] so that
// pass B decides the exclusion from its one relabel gather (ids are < 2^30)
constexpr uint32_t CBIT = 0x80000000u;

CC_DEVI bool tbit(const uint32_t* bm, uint32_t i) { return (__ldg(&bm[i >> 5]) >> (i & 31)) & 1u; }

// slot update through the block's cache of pushed values (key p, value in one 64-bit word)
CC_DEVI void push_min(uint32_t* OUT, unsigned long long* s_pc, uint32_t p, uint32_t q) {
  const uint32_t h = (p ^ (p >> 9)) & (RCACHE - 1);
  const unsigned long long e = *(volatile unsigned long long*)&s_pc[h];
  if ((uint32_t)(e >> 32) == p && q >= (uint32_t)e) return;
  atomicMin(&OUT[p], q);  // result unused: compiles to a fire-and-forget reduction
  s_pc[h] = ((unsigned long long)p << 32) | q;
}
// precheck (hot iterations, where many rows share one minimum): read the word first so a
// set bit costs no atomic; otherwise a fire-and-forget atomic (no dependent load)
CC_DEVI void push_bit(uint32_t* BM, uint32_t* s_nc, uint32_t p, bool precheck) {
  const uint32_t h = (p ^ (p >> 9)) & (RCACHE - 1);
  if (*(volatile uint32_t*)&s_nc[h] == p) return;
  s_nc[h] = p;
  const uint32_t b = 1u << (p & 31);
  if (!precheck || !(*(volatile uint32_t*)&BM[p >> 5] & b)) atomicOr(&BM[p >> 5], b);
}
CC_DEVI void set_bit(uint32_t* BM, uint32_t p) {
  const uint32_t b = 1u << (p & 31);
  if (!(*(volatile uint32_t*)&BM[p >> 5] & b)) atomicOr(&BM[p >> 5], b);
}
// epoch-tagged partial slots: min slot hi word = ~tag (newer = smaller), max slot hi = tag
CC_DEVI unsigned long long tmin(uint32_t tag, uint32_t v) {
  return ((unsigned long long)(0xFFFFFFFFu - tag) << 32) | v;
}
CC_DEVI unsigned long long tmax(uint32_t tag, uint32_t v) {
  return ((unsigned long long)tag << 32) | v;
}

CC_DEVI void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
CC_DEVI void store8(uint32_t* X, uint64_t i0, uint64_t L, const uint32_t* x) {
  if (i0 + RITEMS <= L) {  // streaming stores: the next pass reads them back from DRAM anyway
    st_stream(reinterpret_cast<uint4*>(X + i0), make_uint4(x[0], x[1], x[2], x[3]));
    st_stream(reinterpret_cast<uint4*>(X + i0) + 1, make_uint4(x[4], x[5], x[6], x[7]));
  } else {
#pragma unroll
    for (int j = 0; j < RITEMS; j++)
      if (i0 + j < L) X[i0 + j] = x[j];
  }
}

// ---- TMA bulk copies (1-D cp.async.bulk, completion counted on an mbarrier)
CC_DEVI uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
CC_DEVI void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
CC_DEVI void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
CC_DEVI void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
// the tuple stream is read once per pass: evict-first in L2, so the partition slots (the
// random-access working set of the pass) stay resident
CC_DEVI uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
CC_DEVI void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
      "[%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// relabel of one input value: A -> MAP (NULL: identity); B -> PA[p], or DEAD if p completed
template <bool A, bool REL = true>
CC_DEVI uint32_t relabel(uint32_t pv, const uint32_t* __restrict__ MAP, const uint32_t* __restrict__ NCPr,
                         int excl) {
  if (pv == DEAD) return DEAD;
  if (A) return REL ? __ldg(&MAP[pv]) : pv;
  const uint32_t pm = __ldg(&MAP[pv]);
  if (excl && (pm & CBIT)) return DEAD;
  return pm & ~CBIT;
}

}  // namespace

// --------------------------------------------------------------------------- row pass
// A run = a maximal group of equal live keys = one row (or the part of it in the tile).
// Run minima / maxima are computed branch-free: an inclusive forward and a backward
// segmented scan over the thread's 8 items, Kogge-Stone shuffles across the lanes of a warp
// (forward over the threads' last runs, backward over their first runs; keys are sorted and a
// row is contiguous, so equal keys are always connected), and a walk over the 8 warp
// aggregates for runs that cross warps.  A row that continues past the tile end is finished
// by this tile: the last warp reads its extension (< LONG tuples) from global memory, and the
// next tile skips its leading run.  P is double-buffered (Pin -> Pout), so both tiles see
// the pass's input at every position.
struct RunAgg {
  uint32_t key, mn, mx, pad;
};
// REL: pass A relabels through MAP = PB (every iteration but the first) and writes Pout.
// X: pass A -- PA is preset (updates q = p are skipped); pass B -- completed partitions leave.
template <bool A, bool HOT, bool REL, bool X>
__global__ void __launch_bounds__(PB, 2048 / PB / 2) k_rowpass(
    const uint32_t* __restrict__ R, const uint32_t* __restrict__ Pin, uint32_t* __restrict__ Pout,
    uint64_t L, uint32_t ntiles, const uint32_t* __restrict__ MAP,
    const uint32_t* __restrict__ NCPr, const uint32_t* __restrict__ TB, uint32_t* OUT,
    uint32_t* NCPw, uint32_t* __restrict__ label, unsigned long long* ctr, int preset, int excl,
    const unsigned long long* __restrict__ prevctr, int hot_shift, const uint32_t* __restrict__ HW,
    const unsigned long long* __restrict__ hotcnt, int hot_mode) {
  // With prevctr / hotcnt both variants are launched and device counters pick one (so the host
  // can enqueue this pass before reading them): nothing left -> neither runs; few distinct
  // slot targets per live tuple -> the HOT variant.
  if (prevctr && prevctr[sv::C_OUT] == 0) return;
  if (hotcnt || prevctr) {
    const unsigned long long cnt =
        hotcnt ? (hot_mode == 2   ? hotcnt[sv::C_TDIST]
                  : hot_mode == 1 ? hotcnt[sv::C_PARTITIONS] - hotcnt[sv::C_CHANGED] + hotcnt[sv::C_TEMPS]
                                  : hotcnt[0])
               : prevctr[sv::C_PARTITIONS];
    if (((cnt << hot_shift) < L) != HOT) return;
  }
  constexpr bool PRESET = A && X;
  constexpr int EXCL = (A || X) ? 1 : 0;  // (pass A's relabel ignores it)
  (void)excl;
  constexpr int NW = PB / 32;
  // double-buffered tile staging: TMA brings tile i+2 while tile i is processed
  // s_r: R[t0 - 4, t0) (the last one tells whether the tile starts inside a row), the tile,
  // and the XT tuples past it (the first stretch of the last row's extension); s_in: the tile
  // and the XT inputs past it.  Edge reads then cost no global round trip in the tile.
  constexpr int RPRE = 4, XT = 32;
  __shared__ __align__(128) uint32_t s_r[2][RPRE + PTILE + XT];
  __shared__ __align__(128) uint32_t s_in[2][PTILE + XT];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ uint32_t s_last[NW];
  // per warp: last run (prefix), first run (suffix); double-buffered by tile parity, so the
  // next tile can write its aggregates while a slow warp still walks this tile's (the two
  // barriers of the next tile separate a buffer's reuse) -- no end-of-tile barrier
  __shared__ RunAgg s_wt2[2][NW], s_wh2[2][NW + 1];
  __shared__ uint32_t s_kfirst;
  // hot mode: per-block aggregation of slot updates (key claimed once per block, value
  // min-reduced in shared memory, flushed with one global atomic per key at the end)
  constexpr int RAGG = 1024;
  __shared__ uint32_t s_akey[RAGG], s_aval[RAGG];
  __shared__ uint32_t s_nc[A ? RCACHE : 1];
  for (int i = threadIdx.x; i < RAGG; i += PB) {
    s_akey[i] = INF;
    s_aval[i] = INF;
  }
  for (int i = threadIdx.x; i < (A ? RCACHE : 1); i += PB) s_nc[i] = INF;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // the last slot update / NCP flag this thread issued (slots only decrease): repeats are
  // common once a few partitions hold most tuples
  uint32_t last_p = INF, last_q = INF, last_nc = INF;
  auto issue = [&](uint32_t tl, int b) {  // thread 0: stage tile tl into buffer b
    if (tl >= ntiles) return;
    const uint64_t a0 = (uint64_t)tl * PTILE;
    const uint32_t n = (uint32_t)(L - a0 < (uint64_t)PTILE ? L - a0 : (uint64_t)PTILE);
    const uint32_t pre = a0 > 0 ? RPRE : 0;
    // arrays hold >= L + 64 entries: the XT past the end are in bounds (masked by i < L)
    const uint32_t br = ((pre + n + XT) * 4 + 15) & ~15u, bp = ((n + XT) * 4 + 15) & ~15u;
    const uint64_t pol = l2_evict_first_policy();
    mbar_expect_tx(&s_bar[b], br + bp);
    bulk_g2s(s_r[b] + (RPRE - pre), R + a0 - pre, br, &s_bar[b], pol);
    bulk_g2s(s_in[b], Pin + a0, bp, &s_bar[b], pol);
  };
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    issue(blockIdx.x, 0);
    issue(blockIdx.x + gridDim.x, 1);
  }
  uint32_t live = 0;
  uint32_t hid = 0;  // B with row collapse: folded tuples of the rows that leave (HW)
  uint32_t it = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
    const int buf = it & 1;
    const uint64_t t0 = (uint64_t)tile * PTILE;
    const uint32_t tlen = (uint32_t)(L - t0 < (uint64_t)PTILE ? L - t0 : (uint64_t)PTILE);
    const uint64_t i0 = t0 + (uint64_t)threadIdx.x * RITEMS;
    uint32_t r[RITEMS], p[RITEMS];
    mbar_wait(&s_bar[buf], (it >> 1) & 1);
    const uint32_t rprev = (threadIdx.x == 0 && t0 > 0) ? s_r[buf][RPRE - 1] : INF;
    // last warp: R and the relabelled P of tuple t0 + tlen + lane (its gather overlaps the tile)
    uint32_t xr = INF, xm = DEAD;
    if (wid == NW - 1 && t0 + tlen + lane < L) {
      xr = s_r[buf][RPRE + tlen + lane];
      xm = relabel<A, REL>(s_in[buf][tlen + lane], MAP, NCPr, EXCL);
    }
    {
      const uint32_t s0 = threadIdx.x * RITEMS;
      const uint4 a = reinterpret_cast<const uint4*>(s_r[buf] + RPRE + s0)[0];
      const uint4 b = reinterpret_cast<const uint4*>(s_r[buf] + RPRE + s0)[1];
      const uint4 c = reinterpret_cast<const uint4*>(s_in[buf] + s0)[0];
      const uint4 d = reinterpret_cast<const uint4*>(s_in[buf] + s0)[1];
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
      p[0] = c.x; p[1] = c.y; p[2] = c.z; p[3] = c.w; p[4] = d.x; p[5] = d.y; p[6] = d.z; p[7] = d.w;
#pragma unroll
      for (int j = 0; j < RITEMS; j++)
        if (s0 + j >= tlen) { r[j] = INF; p[j] = DEAD; }
    }
    // ---- relabel (A: line 25 of the previous iteration) / exclusion + line 19 (B)
    // Pass A: a relabelled live tuple stays live (its partition has a slot), so the keys below
    // need only the input; the gathers are issued here and first used after the tile's first
    // barrier, so their latency overlaps the barrier wait instead of preceding it (ncu, C4 mode
    // sv iteration 1: 29 % of the stall samples sat at that barrier and 19 % at the first use,
    // profiles/r02/ncu_rowpassA1_c4sv_s7.txt).  C2 5.54 -> 5.49 ms, C3 5.93 -> 5.89 ms (pass A
    // 1.03 -> 0.99 ms per C2 step), C4 mode sv unchanged.
    constexpr bool LATE = A && REL;
    uint32_t gl[LATE ? RITEMS : 1];
    if (LATE) {
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        const bool fresh = p[j] != DEAD && (j == 0 || p[j] != p[j - 1]);
        gl[LATE ? j : 0] = fresh ? __ldg(&MAP[p[j]]) : p[j];
      }
    } else {
      // one gather per run of equal p in the thread's slice: once a few partitions hold most
      // tuples, thousands of threads would otherwise hit the same L2 line at once
      uint32_t m[RITEMS], cpl = 0;
#pragma unroll
      for (int j = 0; j < RITEMS; j++) {
        const bool fresh = p[j] != DEAD && (!A || REL) && (j == 0 || p[j] != p[j - 1]);
        uint32_t g = fresh ? __ldg(&MAP[p[j]]) : p[j];
        if (!A && fresh) {
          cpl |= (g >> 31) << j;  // CBIT: completed partition
          g &= ~CBIT;
        }
        m[j] = g;
      }
#pragma unroll
      for (int j = 1; j < RITEMS; j++)
        if (p[j] != DEAD && (!A || REL) && p[j] == p[j - 1]) {
          m[j] = m[j - 1];
          cpl |= ((cpl >> (j - 1)) & 1u) << j;
        }
      if (!A) {
#pragma unroll
        for (int j = 0; j < RITEMS; j++) {
          if (EXCL && p[j] != DEAD && ((cpl >> j) & 1u)) {
            // completed partition: the whole row leaves, its vertex is labelled p
            if (j == 0 || r[j - 1] != r[j]) {
              label[r[j] & ~R_LONG] = p[j];
              // a collapsed row is one tuple (its own head); other rows have HW = 0
              if (HW) hid += __ldg(&HW[r[j] & ~R_LONG]);
            }
            m[j] = DEAD;
          }
          live += m[j] != DEAD;
        }
      }
#pragma unroll
      for (int j = 0; j < RITEMS; j++) p[j] = m[j];
    }
    if (!LATE && (!A || REL)) store8(Pout, i0, L, p);
    // keys: dead tuples and long rows (k_long1/k_long2) take no part
    uint32_t k[RITEMS];
#pragma unroll
    for (int j = 0; j < RITEMS; j++) k[j] = (p[j] == DEAD || (r[j] & R_LONG)) ? INF : r[j];
    uint32_t prevk = __shfl_up_sync(FULL, k[RITEMS - 1], 1);
    if (lane == 31) s_last[wid] = k[RITEMS - 1];
    // the leading run belongs to the previous tile when the tile starts inside a row
    if (threadIdx.x == 0) s_kfirst = (t0 > 0 && k[0] != INF && rprev == k[0]) ? k[0] : INF;
    // (Tried: skipping the scans of a tile that holds nothing but long-row and dead tuples --
    // 3/4 of C4's tiles in mode sv.  Iteration 2's pass B 9.0 -> 4.9 ms, but iteration 1's
    // pass B 9.8 -> 14.9 ms, pass A unchanged, C2 5.53 -> 5.62 ms: no net gain, removed.
    // profiles/r02/timeline_c4sv_s7_tileskip_rejected.json against timeline_c4sv_s7_final.json)
    __syncthreads();
    const uint32_t kfirst = s_kfirst;
    if (lane == 0) prevk = wid ? s_last[wid - 1] : kfirst;
    if (threadIdx.x == 0) {  // every thread has its items: refill this buffer
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(tile + 2 * gridDim.x, buf);
    }
    if (LATE) {  // the gathered labels: one per run of equal p in the thread's slice
      uint32_t m[RITEMS];
      m[0] = gl[0];
#pragma unroll
      for (int j = 1; j < RITEMS; j++)
        m[j] = (p[j] != DEAD && p[j] == p[j - 1]) ? m[j - 1] : gl[LATE ? j : 0];
#pragma unroll
      for (int j = 0; j < RITEMS; j++) p[j] = m[j];
      store8(Pout, i0, L, p);
    }
    // ---- thread-local scans; the temporary <r,_,r> of line 22 joins VB(r) at the row head
    uint32_t v[RITEMS];
    uint32_t heads = 0;
    // B: the thread's row heads are consecutive ids, almost always inside one TB word
    uint32_t tbi = INF, tbw = 0;
#pragma unroll
    for (int j = 0; j < RITEMS; j++) {
      const uint32_t pk = j ? k[j - 1] : prevk;
      const bool h = k[j] != INF && k[j] != pk;
      heads |= (uint32_t)h << j;
      bool t = false;
      if (!A && h) {
        if ((k[j] >> 5) != tbi) {
          tbi = k[j] >> 5;
          tbw = __ldg(&TB[tbi]);
        }
        t = (tbw >> (k[j] & 31)) & 1u;
      }
      v[j] = t ? min(p[j], k[j]) : p[j];
    }
    uint32_t fmn[RITEMS], fmx[RITEMS], bmn[RITEMS], bmx[RITEMS];
    fmn[0] = v[0]; fmx[0] = p[0];
#pragma unroll
    for (int j = 1; j < RITEMS; j++) {
      const bool c = k[j] == k[j - 1];
      fmn[j] = c ? min(fmn[j - 1], v[j]) : v[j];
      if (A) fmx[j] = c ? max(fmx[j - 1], p[j]) : p[j];
    }
    bmn[RITEMS - 1] = v[RITEMS - 1]; bmx[RITEMS - 1] = p[RITEMS - 1];
#pragma unroll
    for (int j = RITEMS - 2; j >= 0; j--) {
      const bool c = k[j] == k[j + 1];
      bmn[j] = c ? min(bmn[j + 1], v[j]) : v[j];
      if (A) bmx[j] = c ? max(bmx[j + 1], p[j]) : p[j];
    }
    // ---- warp: forward over the threads' last runs, backward over their first runs
    const uint32_t kt = k[RITEMS - 1], kh = k[0];
    uint32_t tmn = fmn[RITEMS - 1], tmx = A ? fmx[RITEMS - 1] : 0u;
    uint32_t hmn = bmn[0], hmx = A ? bmx[0] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t ok = __shfl_up_sync(FULL, kt, d);
      const uint32_t om = __shfl_up_sync(FULL, tmn, d);
      const uint32_t ox = A ? __shfl_up_sync(FULL, tmx, d) : 0u;
      if (lane >= d && ok == kt) { tmn = min(tmn, om); if (A) tmx = max(tmx, ox); }
      const uint32_t nk = __shfl_down_sync(FULL, kh, d);
      const uint32_t nm = __shfl_down_sync(FULL, hmn, d);
      const uint32_t nx = A ? __shfl_down_sync(FULL, hmx, d) : 0u;
      if (lane + d < 32 && nk == kh) { hmn = min(hmn, nm); if (A) hmx = max(hmx, nx); }
    }
    // carries from the neighbouring lanes (their inclusive scans)
    uint32_t cin_k = __shfl_up_sync(FULL, kt, 1), cin_m = __shfl_up_sync(FULL, tmn, 1);
    uint32_t cin_x = A ? __shfl_up_sync(FULL, tmx, 1) : 0u;
    uint32_t cout_k = __shfl_down_sync(FULL, kh, 1), cout_m = __shfl_down_sync(FULL, hmn, 1);
    uint32_t cout_x = A ? __shfl_down_sync(FULL, hmx, 1) : 0u;
    if (lane == 0) cin_k = INF;
    if (lane == 31) cout_k = INF;
    RunAgg* s_wt = s_wt2[buf];
    RunAgg* s_wh = s_wh2[buf];
    if (lane == 31) s_wt[wid] = RunAgg{kt, tmn, tmx, 0u};
    if (lane == 0) s_wh[wid] = RunAgg{kh, hmn, hmx, 0u};
    // ---- extension of the tile's last run into the next tile (last warp)
    if (wid == NW - 1) {
      uint32_t emn = INF, emx = 0, ek = INF;
      const uint32_t klast = __shfl_sync(FULL, kt, 31);
      const uint64_t pos = t0 + tlen;
      if (klast != INF && __shfl_sync(FULL, xr, 0) == klast) {
        ek = klast;
        const bool in0 = xr == klast;  // the prefetched first 32 (live row: not DEAD)
        if (in0) {
          emn = xm;
          emx = xm;
        }
        if (!__ballot_sync(FULL, !in0)) {
          for (uint64_t base = pos + 32; base < pos + LONG; base += 32) {
            const uint64_t i = base + lane;
            const bool in = i < L && __ldg(&R[i]) == klast;
            if (in) {
              const uint32_t pv = relabel<A, REL>(__ldg(&Pin[i]), MAP, NCPr, EXCL);
              emn = min(emn, pv);
              emx = max(emx, pv);
            }
            if (__ballot_sync(FULL, !in)) break;
          }
        }
        emn = __reduce_min_sync(FULL, emn);
        emx = __reduce_max_sync(FULL, emx);
      }
      if (lane == 0) s_wh[NW] = RunAgg{ek, emn, emx, 0u};
    }
    __syncthreads();
    // ---- runs that cross warps: walk the warp aggregates (warp-uniform loops)
    uint32_t wcin_m = INF, wcin_x = 0, wcout_m = INF, wcout_x = 0;
    const uint32_t k0w = __shfl_sync(FULL, kh, 0), k31w = __shfl_sync(FULL, kt, 31);
    for (int w = wid - 1; w >= 0; w--) {
      const RunAgg a = s_wt[w];
      if (a.key != k0w || k0w == INF) break;
      wcin_m = min(wcin_m, a.mn); wcin_x = max(wcin_x, a.mx);
      if (s_wh[w].key != a.key) break;  // warp w is not one run
    }
    for (int w = wid + 1; w <= NW; w++) {
      const RunAgg a = s_wh[w];
      if (a.key != k31w || k31w == INF) break;
      wcout_m = min(wcout_m, a.mn); wcout_x = max(wcout_x, a.mx);
      if (w == NW || s_wt[w].key != a.key) break;
    }
    if (lane == 0) { cin_k = k0w; cin_m = wcin_m; cin_x = wcin_x; }
    else if (cin_k == k0w) { cin_m = min(cin_m, wcin_m); cin_x = max(cin_x, wcin_x); }
    if (lane == 31) { cout_k = k31w; cout_m = wcout_m; cout_x = wcout_x; }
    else if (cout_k == k31w) { cout_m = min(cout_m, wcout_m); cout_x = max(cout_x, wcout_x); }
    // ---- apply: q = u_min(r) to PA/PB[p] (+ NCP(q) of a non-PC row in A, + the
    // temporary's own q in B), skipping the leading run owned by the previous tile
    uint32_t qlast = INF;
#pragma unroll
    for (int j = 0; j < RITEMS; j++) {
      uint32_t q = min(fmn[j], bmn[j]);
      uint32_t x = A ? max(fmx[j], bmx[j]) : 0u;
      if (k[j] == k[0] && cin_k == k[0]) { q = min(q, cin_m); if (A) x = max(x, cin_x); }
      if (k[j] == k[RITEMS - 1] && cout_k == k[RITEMS - 1]) { q = min(q, cout_m); if (A) x = max(x, cout_x); }
      if (k[j] == INF || k[j] == kfirst) continue;
      if (j == RITEMS - 1) qlast = q;
      // (several ranks, owner-computes exchange: pass B writes every value it holds, q = p
      // too, so the slot is requested from its owner -- preset = 1 there)
      if ((A ? PRESET : !preset) && q == p[j]) {
        // A: PA[p] was preset to p (p is a partition of this iteration).  B: every live value
        // p is p_min of a surviving partition, so TB(p) holds and k_pstat2 applies the
        // temporary's own min(PB[p], p).  Either way min(slot, p) changes nothing.
      } else if (!HOT) {
        atomicMin(&OUT[p[j]], q);
      } else if (p[j] != last_p || q < last_q) {  // this thread's last update covers it
        const uint32_t h = (p[j] ^ (p[j] >> 10)) & (RAGG - 1);
        uint32_t key = *(volatile uint32_t*)&s_akey[h];
        if (key == INF) {
          key = atomicCAS(&s_akey[h], INF, p[j]);
          if (key == INF) key = p[j];
        }
        if (key == p[j]) atomicMin(&s_aval[h], q);
        else atomicMin(&OUT[p[j]], q);
        last_p = p[j];
        last_q = q;
      }
      if ((heads >> j) & 1u) {
        if (A) {
          // many non-PC rows share one minimum late in the run: filter through a block cache
          // and a read of the word before the atomic
          if (q != x && (HOT || q != last_nc)) {  // hot: the block cache filters repeats
            push_bit(NCPw, s_nc, q, HOT);
            if (!HOT) last_nc = q;
          }
        } else if (q != k[j] && tbit(TB, k[j])) {  // q = r: k_pstat2's fold covers it
          atomicMin(&OUT[k[j]], q);
        }
      }
    }
    // extension tuples of the last run (owned here): same q as the run
    if (wid == NW - 1 && s_wh[NW].key != INF) {
      const uint32_t q = __shfl_sync(FULL, qlast, 31);
      const uint32_t klast = s_wh[NW].key;
      const uint64_t pos = t0 + tlen;
      const bool in0 = xr == klast;
      if (in0 && (q != xm || (A ? !PRESET : preset))) atomicMin(&OUT[xm], q);  // q = p: see above
      if (!__ballot_sync(FULL, !in0)) {
        for (uint64_t base = pos + 32; base < pos + LONG; base += 32) {
          const uint64_t i = base + lane;
          const bool in = i < L && __ldg(&R[i]) == klast;
          if (in) atomicMin(&OUT[relabel<A, REL>(__ldg(&Pin[i]), MAP, NCPr, EXCL)], q);
          if (__ballot_sync(FULL, !in)) break;
        }
      }
    }
  }
  if (HOT) {  // flush the block's aggregated slot updates
    __syncthreads();
    for (int i = threadIdx.x; i < RAGG; i += PB)
      if (s_akey[i] != INF) atomicMin(&OUT[s_akey[i]], s_aval[i]);
  }
  if (!A) {
    live = warp_sum(live);
    if (lane == 0 && live) atomicAdd(&ctr[sv::C_OUT], (unsigned long long)live);
    if (HW) {
      hid = warp_sum(hid);
      if (lane == 0 && hid) atomicAdd(&ctr[sv::C_HIDDEN_DEAD], (unsigned long long)hid);
    }
  }
}

// --------------------------------------------------------------------------- long rows
// List the segments (<= LSEG tuples) of live rows longer than LONG (R_LONG flag; their
// length is deg + 1, the vertex tuple and one tuple per arc): one thread per row head.
__global__ void __launch_bounds__(RB) k_longlist(const uint32_t* __restrict__ R,
                                                 const uint32_t* __restrict__ P, uint64_t L,
                                                 const uint32_t* __restrict__ deg,
                                                 LongSeg* __restrict__ segs,
                                                 unsigned long long* nsegs, uint64_t cap) {
  // four tuples per thread: one 16-byte load of R when the array is 16-byte aligned
  const bool vec = (reinterpret_cast<uintptr_t>(R) & 15) == 0;
  const uint64_t nq = (L + 3) / 4;
  for (uint64_t q = blockIdx.x * (uint64_t)RB + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * RB) {
    const uint64_t i0 = 4 * q;
    uint32_t r[4];
    if (vec && i0 + 4 <= L) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(R) + q);
      r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) r[j] = i0 + j < L ? R[i0 + j] : 0u;
    }
    if (!((r[0] | r[1] | r[2] | r[3]) & R_LONG)) continue;  // no long-row tuple here
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint64_t i = i0 + j;
      const uint32_t ru = r[j];
      if (i >= L || !(ru & R_LONG)) continue;
      const uint32_t prev = j ? r[j - 1] : (i > 0 ? R[i - 1] : ~ru);
      if (prev == ru || P[i] == DEAD) continue;
      const uint32_t u = ru & ~R_LONG;
      const uint64_t len = (uint64_t)deg[u] + 1, ns = (len + LSEG - 1) / LSEG;
      const uint64_t b = atomicAdd(nsegs, (unsigned long long)ns);
      for (uint64_t s = 0; s < ns && b + s < cap; s++) {
        LongSeg sg;
        sg.u = u;
        sg.start = i + s * LSEG;
        sg.len = (uint32_t)(len - s * LSEG < LSEG ? len - s * LSEG : LSEG);
        segs[b + s] = sg;
      }
    }
  }
}

// Segment partials of long rows (after k_rowpass has written the relabelled values).
template <bool A>
__global__ void __launch_bounds__(RB) k_long1(const uint32_t* __restrict__ P,
                                              const LongSeg* __restrict__ segs,
                                              const unsigned long long* nsegs,
                                              const uint32_t* __restrict__ TB,
                                              unsigned long long* UMIN, unsigned long long* UMAX,
                                              uint32_t tag) {
  const int lane = threadIdx.x & 31;
  const uint64_t cnt = *nsegs;
  for (uint64_t s = (blockIdx.x * (uint64_t)RB + threadIdx.x) >> 5; s < cnt;
       s += ((uint64_t)gridDim.x * RB) >> 5) {
    const LongSeg sg = segs[s];
    uint32_t mn = INF, mx = 0;
    for (uint32_t i0 = lane; i0 < sg.len; i0 += 32 * LU) {
      uint32_t pv[LU];
#pragma unroll
      for (int u = 0; u < LU; u++) pv[u] = i0 + 32u * u < sg.len ? P[sg.start + i0 + 32u * u] : INF;
#pragma unroll
      for (int u = 0; u < LU; u++) {
        mn = min(mn, pv[u]);
        if (pv[u] != DEAD) mx = max(mx, pv[u]);
      }
    }
    mn = __reduce_min_sync(FULL, mn);
    mx = __reduce_max_sync(FULL, mx);
    if (lane == 0 && mn != INF) {
      if (!A && tbit(TB, sg.u)) mn = min(mn, sg.u);
      atomicMin(&UMIN[sg.u], tmin(tag, mn));
      if (A) atomicMax(&UMAX[sg.u], tmax(tag, mx));
    }
  }
}

// Apply of long rows: u_min(r) (and the max) are final in the tagged slots.
template <bool A>
__global__ void __launch_bounds__(RB) k_long2(const uint32_t* __restrict__ P,
                                              const LongSeg* __restrict__ segs,
                                              const unsigned long long* nsegs,
                                              const unsigned long long* __restrict__ UMIN,
                                              const unsigned long long* __restrict__ UMAX,
                                              const uint32_t* __restrict__ TB, uint32_t* OUT,
                                              uint32_t* NCPw, uint32_t tag) {
  __shared__ unsigned long long s_pc[RCACHE];
  for (int i = threadIdx.x; i < RCACHE; i += RB) s_pc[i] = ~0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t cnt = *nsegs;
  for (uint64_t s = (blockIdx.x * (uint64_t)RB + threadIdx.x) >> 5; s < cnt;
       s += ((uint64_t)gridDim.x * RB) >> 5) {
    const LongSeg sg = segs[s];
    const unsigned long long um = UMIN[sg.u];
    if ((uint32_t)(um >> 32) != 0xFFFFFFFFu - tag) continue;  // row left (completed)
    const uint32_t q = (uint32_t)um;
    for (uint32_t i0 = lane; i0 < sg.len; i0 += 32 * LU) {
      uint32_t pv[LU];
#pragma unroll
      for (int u = 0; u < LU; u++)
        if (i0 + 32u * u < sg.len) pv[u] = P[sg.start + i0 + 32u * u];
#pragma unroll
      for (int u = 0; u < LU; u++)
        if (i0 + 32u * u < sg.len) push_min(OUT, s_pc, pv[u], q);
    }
    if (lane == 0) {
      if (A) {
        if (q != (uint32_t)UMAX[sg.u]) set_bit(NCPw, q);
      } else if (tbit(TB, sg.u)) {
        push_min(OUT, s_pc, sg.u, q);
      }
    }
  }
}

// --------------------------------------------------------------------------- slot scans
// After pass A: |P_i|, completed, changed, T_i from PA/NCP; one temporary per surviving
// partition marks TB(p_min) (line 22); PB is cleared for pass B.
// nd (DIST): TB bits this thread set first, i.e. distinct temporary targets p_min = the slots
// pass B will update (its hot-variant choice in iteration 0, which has no earlier counters)
template <bool DIST = false>
CC_DEVI bool pstat1_one(uint32_t pid, uint32_t pm, bool ncp, int temps_all, uint32_t* TB, uint32_t& np,
                        uint32_t& nc, uint32_t& ch, uint32_t& nt, uint32_t& nd) {
  np++;
  ch += pm != pid;
  const bool comp = pm == pid && !ncp;
  nc += comp;
  if (!comp || temps_all) {  // temps_all: completed partitions stay for this iteration
    nt++;
    const uint32_t b = 1u << (pm & 31);
    if (!(*(volatile uint32_t*)&TB[pm >> 5] & b)) {
      if (DIST) nd += !(atomicOr(&TB[pm >> 5], b) & b);
      else atomicOr(&TB[pm >> 5], b);
    }
  }
  return comp;
}
CC_DEVI void pstat1_flush(uint32_t np, uint32_t nc, uint32_t ch, uint32_t nt, unsigned long long* ctr,
                          uint32_t nd = 0) {
  np = warp_sum(np); nc = warp_sum(nc); ch = warp_sum(ch); nt = warp_sum(nt); nd = warp_sum(nd);
  if ((threadIdx.x & 31) == 0) {
    if (np) atomicAdd(&ctr[sv::C_PARTITIONS], (unsigned long long)np);
    if (nc) atomicAdd(&ctr[sv::C_COMPLETED], (unsigned long long)nc);
    if (ch) atomicAdd(&ctr[sv::C_CHANGED], (unsigned long long)ch);
    if (nt) atomicAdd(&ctr[sv::C_TEMPS], (unsigned long long)nt);
    if (nd) atomicAdd(&ctr[sv::C_TDIST], (unsigned long long)nd);
  }
}
// flag: mark completed partitions with CBIT in PA (pass B excludes them)
// base (multiple of 32): PA, NCP, PB start at slot base (an owner block); TB is absolute
__global__ void __launch_bounds__(RB) k_pstat1(uint32_t* __restrict__ PA,
                                               const uint32_t* __restrict__ NCP, uint64_t n4,
                                               uint32_t* TB, uint32_t* __restrict__ PB,
                                               unsigned long long* ctr, int temps_all, int flag,
                                               uint32_t base) {
  uint32_t np = 0, nc = 0, ch = 0, nt = 0, nd = 0;
  for (uint64_t t = blockIdx.x * (uint64_t)RB + threadIdx.x; t < n4; t += (uint64_t)gridDim.x * RB) {
    const uint4 a = reinterpret_cast<const uint4*>(PA)[t];
    reinterpret_cast<uint4*>(PB)[t] = make_uint4(INF, INF, INF, INF);
    if ((a.x & a.y & a.z & a.w) == INF) continue;
    const uint32_t w = __ldg(&NCP[t >> 3]) >> (4 * (t & 7));
    uint32_t v[4] = {a.x, a.y, a.z, a.w};
    uint32_t cm = 0;
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (v[j] != INF && pstat1_one<true>(base + (uint32_t)(4 * t + j), v[j], (w >> j) & 1u, temps_all, TB, np, nc, ch, nt, nd)) {
        v[j] |= CBIT;
        cm = 1;
      }
    if (cm && flag) reinterpret_cast<uint4*>(PA)[t] = make_uint4(v[0], v[1], v[2], v[3]);
  }
  pstat1_flush(np, nc, ch, nt, ctr, nd);
}
// list form: statistics over L_i; PB is cleared over L_i-1 (its written keys lie in P_i-1)
__global__ void __launch_bounds__(RB) k_pstat1_list(uint32_t* __restrict__ PA,
                                                    const uint32_t* __restrict__ NCP,
                                                    const uint32_t* __restrict__ list,
                                                    const unsigned long long* lcnt,
                                                    const uint32_t* __restrict__ prev,
                                                    const unsigned long long* pcnt, uint32_t* TB,
                                                    uint32_t* __restrict__ PB, unsigned long long* ctr,
                                                    int temps_all, int flag) {
  uint32_t np = 0, nc = 0, ch = 0, nt = 0, nd = 0;
  const uint64_t cp = *pcnt;
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < cp; i += (uint64_t)gridDim.x * RB)
    PB[prev[i]] = INF;
  const uint64_t cnt = *lcnt;
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * RB) {
    const uint32_t pid = list[i];
    const uint32_t pm = PA[pid];
    if (pm != INF && pstat1_one(pid, pm, tbit(NCP, pid), temps_all, TB, np, nc, ch, nt, nd) && flag)
      PA[pid] = pm | CBIT;
  }
  pstat1_flush(np, nc, ch, nt, ctr);
}

// After pass B: the temporaries' own element (line 24: <u,_,u>_tmp is in PB(u) with
// q = u_min'(u) <= u; the row part of u_min' was pushed by pass B) -- PB[u] = min(PB[u], u)
// for TB(u) -- then changed2 from PB and PA cleared for the next iteration.
// The next iteration's partition ids: after pass B every live tuple of partition p holds
// v = PA[p], and the next pass A maps it to PB[v].  The values v are exactly the temporaries'
// ids TB (one per surviving partition; with CC_FLAG_NO_EARLY_EXCLUDE a superset, completed
// partitions included), so P_i+1 = { PB[v] : TB(v) } is marked in NX from each slot's own
// word -- no gather.  NCP and TB are cleared by k_list_from_bits, which runs after this kernel.
CC_DEVI void mark(uint32_t* NX, uint32_t v) {
  const uint32_t b = 1u << (v & 31);
  if (!(*(volatile uint32_t*)&NX[v >> 5] & b)) atomicOr(&NX[v >> 5], b);
}
// base (multiple of 32): PB, PA and TB start at slot base (an owner block); NX NULL: no list
__global__ void __launch_bounds__(RB) k_pstat2(uint32_t* __restrict__ PB, uint64_t n4,
                                               uint32_t* __restrict__ PA, const uint32_t* __restrict__ TB,
                                               unsigned long long* ctr, uint32_t* NX, uint32_t base) {
  uint32_t ch = 0;
  for (uint64_t t = blockIdx.x * (uint64_t)RB + threadIdx.x; t < n4; t += (uint64_t)gridDim.x * RB) {
    uint4 b = reinterpret_cast<const uint4*>(PB)[t];
    reinterpret_cast<uint4*>(PA)[t] = make_uint4(INF, INF, INF, INF);
    const uint32_t tw = (TB[t >> 3] >> (4 * (t & 7))) & 15u;
    const uint32_t u0 = base + (uint32_t)(4 * t);
    if (tw) {
      if (tw & 1u) { b.x = min(b.x, u0); if (NX) mark(NX, b.x); }
      if (tw & 2u) { b.y = min(b.y, u0 + 1); if (NX) mark(NX, b.y); }
      if (tw & 4u) { b.z = min(b.z, u0 + 2); if (NX) mark(NX, b.z); }
      if (tw & 8u) { b.w = min(b.w, u0 + 3); if (NX) mark(NX, b.w); }
      reinterpret_cast<uint4*>(PB)[t] = b;
    }
    const uint32_t v[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 4; j++) ch += v[j] != INF && v[j] != u0 + j;
  }
  ch = warp_sum(ch);
  if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&ctr[sv::C_CHANGED2], (unsigned long long)ch);
}
__global__ void __launch_bounds__(RB) k_pstat2_list(uint32_t* __restrict__ PB,
                                                    const uint32_t* __restrict__ list,
                                                    const unsigned long long* lcnt,
                                                    uint32_t* __restrict__ PA, const uint32_t* __restrict__ TB,
                                                    unsigned long long* ctr, uint32_t* NX) {
  uint32_t ch = 0;
  const uint64_t cnt = *lcnt;
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * RB) {
    const uint32_t pid = list[i];
    uint32_t b = PB[pid];
    PA[pid] = INF;
    if ((TB[pid >> 5] >> (pid & 31)) & 1u) {
      if (pid < b) PB[pid] = b = pid;
      mark(NX, b);
    }
    ch += b != INF && b != pid;
  }
  ch = warp_sum(ch);
  if ((threadIdx.x & 31) == 0 && ch) atomicAdd(&ctr[sv::C_CHANGED2], (unsigned long long)ch);
}

// list of the set bits of NX (cleared): one block-wide scan per 256-word chunk, one atomic
// per chunk with set bits
__global__ void __launch_bounds__(RB) k_list_from_bits(uint32_t* NX, uint64_t nw, uint32_t* __restrict__ list,
                                                       unsigned long long* lcnt, uint32_t* __restrict__ NCP,
                                                       uint32_t* __restrict__ TB, uint32_t* __restrict__ PA) {
  __shared__ uint32_t s_w[RB / 32];
  __shared__ unsigned long long s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t w0 = blockIdx.x * (uint64_t)RB; w0 < nw; w0 += (uint64_t)gridDim.x * RB) {
    const uint64_t w = w0 + threadIdx.x;
    uint32_t bits = 0u;
    if (w < nw) {
      bits = NX[w];
      if (bits) NX[w] = 0u;
      NCP[w] = 0u;
      TB[w] = 0u;
    }
    const uint32_t c = __popc(bits);
    uint32_t x = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (int i = 0; i < RB / 32; i++) {
        const uint32_t t = s_w[i];
        s_w[i] = acc;
        acc += t;
      }
      s_base = acc ? atomicAdd(lcnt, (unsigned long long)acc) : 0ull;
    }
    __syncthreads();
    uint64_t pos = s_base + s_w[wid] + x - c;
    while (bits) {  // exact list: each partition id p gets PA[p] = p (pass A skips q = p)
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint32_t id = (uint32_t)(w * 32 + b);
      list[pos++] = id;
      if (PA) PA[id] = id;
    }
    __syncthreads();
  }
}

// Without exclusion (fig:loadbal 'Naive') every row is still in the array at convergence:
// its vertex takes the (now common) partition id of its tuples.
__global__ void k_final_labels(const uint32_t* __restrict__ R, const uint32_t* __restrict__ P, uint64_t L,
                               uint32_t* __restrict__ label) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < L; i += (uint64_t)gridDim.x * RB)
    if (P[i] != DEAD && (i == 0 || R[i - 1] != R[i])) label[R[i] & ~R_LONG] = P[i];
}

// --------------------------------------------------------------------------- exchange helpers
__global__ void k_flip_sign(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < n; i += (uint64_t)gridDim.x * RB)
    a[i] ^= 0x80000000u;
}
__global__ void k_or_parts(const uint32_t* __restrict__ parts, uint64_t words, int world,
                           uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < words; i += (uint64_t)gridDim.x * RB) {
    uint32_t x = 0;
    for (int k = 0; k < world; k++) x |= parts[(uint64_t)k * words + i];
    out[i] = x;
  }
}

// Sparse slot exchange (multi-GPU, late iterations): the touched partition slots of a rank as
// (p, value | NCP(p) << 31) entries (NCP is only ever set on touched slots: the row minimum's
// own tuple touches it), and their application to a rank's copy.
__global__ void k_extract_slots(const uint32_t* __restrict__ S, const uint32_t* __restrict__ BM,
                                uint64_t n, uint2* __restrict__ out, unsigned long long* cnt) {
  for (uint64_t p0 = blockIdx.x * (uint64_t)RB; p0 < n; p0 += (uint64_t)gridDim.x * RB) {
    const uint64_t p = p0 + threadIdx.x;
    const uint32_t v = p < n ? S[p] : INF;
    const bool take = v != INF;
    const uint32_t mask = __ballot_sync(FULL, take);
    if (!mask) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(cnt, (unsigned long long)__popc(mask));
    base = __shfl_sync(FULL, base, leader);
    if (take) {
      const uint32_t ncp = BM ? (BM[p >> 5] >> (p & 31)) & 1u : 0u;
      out[base + __popc(mask & ((1u << lane) - 1u))] = make_uint2((uint32_t)p, v | (ncp << 31));
    }
  }
}
__global__ void k_apply_slots(const uint2* __restrict__ in, uint64_t count, uint32_t* S, uint32_t* BM) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < count; i += (uint64_t)gridDim.x * RB) {
    const uint2 e = in[i];
    if (e.x == INF) continue;  // padding
    const uint32_t v = e.y & 0x7FFFFFFFu;
    if (v < S[e.x]) atomicMin(&S[e.x], v);
    if ((e.y >> 31) && BM) atomicOr(&BM[e.x >> 5], 1u << (e.x & 31));
  }
}

// --------------------------------------------------------------------------- launchers
void extract_slots(const uint32_t* S, const uint32_t* BM, uint64_t n, uint2* out, uint64_t* cnt,
                   cudaStream_t st) {
  cudaMemsetAsync(cnt, 0, sizeof(uint64_t), st);
  if (n)
    k_extract_slots<<<(unsigned)std::min<uint64_t>((n + RB - 1) / RB, 148 * 8), RB, 0, st>>>(
        S, BM, n, out, reinterpret_cast<unsigned long long*>(cnt));
}
void apply_slots(const uint2* in, uint64_t count, uint32_t* S, uint32_t* BM, cudaStream_t st) {
  if (count)
    k_apply_slots<<<(unsigned)std::min<uint64_t>((count + RB - 1) / RB, 148 * 8), RB, 0, st>>>(in, count, S, BM);
}
void final_labels(const uint32_t* R, const uint32_t* P, uint64_t L, uint32_t* label, cudaStream_t st) {
  if (L) k_final_labels<<<(unsigned)std::min<uint64_t>((L + RB - 1) / RB, 148 * 8), RB, 0, st>>>(R, P, L, label);
}
void flip_sign(uint32_t* a, uint64_t n, cudaStream_t st) {
  if (n) k_flip_sign<<<(unsigned)std::min<uint64_t>((n + RB - 1) / RB, 148 * 8), RB, 0, st>>>(a, n);
}
void or_parts(const uint32_t* parts, uint64_t words, int world, uint32_t* out, cudaStream_t st) {
  if (words)
    k_or_parts<<<(unsigned)std::min<uint64_t>((words + RB - 1) / RB, 148 * 8), RB, 0, st>>>(parts, words,
                                                                                            world, out);
}

static unsigned persistent_grid(const void* fn) {
  int ps = 0, sms = 148, dev = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, PB, 0);
  if (ps < 1) ps = 1;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (unsigned)(sms * ps);
}
template <bool A, bool HOT, bool REL, bool X>
static void launch_rowpass_x(const uint32_t* R, const uint32_t* Pin, uint32_t* Pout, uint64_t L, uint64_t nt,
                           const uint32_t* MAP, const uint32_t* NCPr, const uint32_t* TB, uint32_t* OUT,
                           uint32_t* NCPw, uint32_t* label, unsigned long long* c, int preset, int excl,
                           const uint64_t* prevctr, int hot_shift, cudaStream_t st, const uint32_t* HW,
                           const uint64_t* hotcnt, int hot_mode) {
  static unsigned grid = 0;
  if (!grid) grid = persistent_grid((const void*)k_rowpass<A, HOT, REL, X>);
  k_rowpass<A, HOT, REL, X><<<(unsigned)std::min<uint64_t>(nt, grid), PB, 0, st>>>(
      R, Pin, Pout, L, (uint32_t)nt, MAP, NCPr, TB, OUT, NCPw, label, c, preset, excl,
      reinterpret_cast<const unsigned long long*>(prevctr), hot_shift, HW,
      reinterpret_cast<const unsigned long long*>(hotcnt), hot_mode);
}

template <bool A, bool HOT, bool REL>
static void launch_rowpass(const uint32_t* R, const uint32_t* Pin, uint32_t* Pout, uint64_t L, uint64_t nt,
                           const uint32_t* MAP, const uint32_t* NCPr, const uint32_t* TB, uint32_t* OUT,
                           uint32_t* NCPw, uint32_t* label, unsigned long long* c, int preset, int excl,
                           const uint64_t* prevctr, int hot_shift, cudaStream_t st, const uint32_t* HW,
                           const uint64_t* hotcnt = nullptr, int hot_mode = 0) {
  if (A ? preset : excl)
    launch_rowpass_x<A, HOT, REL, true>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, preset, excl,
                                        prevctr, hot_shift, st, HW, hotcnt, hot_mode);
  else
    launch_rowpass_x<A, HOT, REL, false>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, preset, excl,
                                         prevctr, hot_shift, st, HW, hotcnt, hot_mode);
}

uint64_t row_tiles(uint64_t L) { return (L + PTILE - 1) / PTILE; }
uint64_t long_seg_cap(uint64_t L) { return L / LSEG + L / (LONG + 1) + 2; }


void longlist(const uint32_t* R, const uint32_t* P, uint64_t L, const uint32_t* deg, LongSeg* segs,
              uint64_t* nsegs, cudaStream_t st) {
  cudaMemsetAsync(nsegs, 0, sizeof(uint64_t), st);
  if (!L) return;
  const unsigned g = (unsigned)std::min<uint64_t>((L + RB - 1) / RB, 148 * 8);
  k_longlist<<<g, RB, 0, st>>>(R, P, L, deg, segs, reinterpret_cast<unsigned long long*>(nsegs),
                               long_seg_cap(L));
}

void rowpass(bool passA, const uint32_t* R, const uint32_t* Pin, uint32_t* Pout, uint64_t L,
             const uint32_t* MAP, const uint32_t* NCPr, const uint32_t* TB, uint32_t* OUT,
             uint32_t* NCPw, uint32_t* label, uint64_t* UMIN, uint64_t* UMAX, uint32_t tag,
             const LongSeg* segs, const uint64_t* nsegs, bool have_long, bool hot, uint64_t* ctr,
             cudaStream_t st, bool excl, bool preset, const uint64_t* prevctr, int hot_shift,
             const uint32_t* HW, const uint64_t* hotcnt, int hot_mode) {
  if (!L) return;
  const uint64_t nt = row_tiles(L);
  auto* umin = reinterpret_cast<unsigned long long*>(UMIN);
  auto* umax = reinterpret_cast<unsigned long long*>(UMAX);
  auto* ns = reinterpret_cast<const unsigned long long*>(nsegs);
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  const uint32_t* Pv = Pout ? Pout : Pin;  // relabelled values, for the long-row kernels
  // with prevctr both variants go in and the device picks (see k_rowpass)
  const int pre = preset ? 1 : 0, ex = excl ? 1 : 0;
  if (passA && !MAP) {  // the first iteration: identity relabel, no P written, never hot
    launch_rowpass<true, false, false>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, pre, ex, prevctr,
                                       hot_shift, st, passA ? nullptr : HW);
    if (have_long) {
      k_long1<true><<<148 * 4, RB, 0, st>>>(Pv, segs, ns, TB, umin, umax, tag);
      k_long2<true><<<148 * 4, RB, 0, st>>>(Pv, segs, ns, umin, umax, TB, OUT, NCPw, tag);
    }
  } else if (passA) {
    const bool sel = prevctr || hotcnt;
    if (sel || hot)
      launch_rowpass<true, true, true>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, pre, ex, prevctr,
                                       hot_shift, st, passA ? nullptr : HW, hotcnt, hot_mode);
    if (sel || !hot)
      launch_rowpass<true, false, true>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, pre, ex, prevctr,
                                        hot_shift, st, passA ? nullptr : HW, hotcnt, hot_mode);
    if (have_long) {
      k_long1<true><<<148 * 4, RB, 0, st>>>(Pv, segs, ns, TB, umin, umax, tag);
      k_long2<true><<<148 * 4, RB, 0, st>>>(Pv, segs, ns, umin, umax, TB, OUT, NCPw, tag);
    }
  } else {
    const bool sel = prevctr || hotcnt;
    if (sel || hot)
      launch_rowpass<false, true, true>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, pre, ex, prevctr,
                                        hot_shift, st, passA ? nullptr : HW, hotcnt, hot_mode);
    if (sel || !hot)
      launch_rowpass<false, false, true>(R, Pin, Pout, L, nt, MAP, NCPr, TB, OUT, NCPw, label, c, pre, ex, prevctr,
                                         hot_shift, st, passA ? nullptr : HW, hotcnt, hot_mode);
    if (have_long) {
      k_long1<false><<<148 * 4, RB, 0, st>>>(Pv, segs, ns, TB, umin, umax, tag);
      k_long2<false><<<148 * 4, RB, 0, st>>>(Pv, segs, ns, umin, umax, TB, OUT, NCPw, tag);
    }
  }
}

void pstat1(uint32_t* PA, const uint32_t* NCP, uint64_t n, uint32_t* TB, uint32_t* PB,
            uint64_t* ctr, cudaStream_t st, bool temps_all, bool flag, const uint32_t* list,
            const uint64_t* lcnt, const uint32_t* prev, const uint64_t* pcnt) {
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  if (list) {
    if (!prev) cudaMemsetAsync(PB, 0xFF, sizeof(uint32_t) * ((n + 3) / 4 * 4), st);
    k_pstat1_list<<<148 * 8, RB, 0, st>>>(PA, NCP, list, reinterpret_cast<const unsigned long long*>(lcnt),
                                          prev ? prev : list,
                                          reinterpret_cast<const unsigned long long*>(prev ? pcnt : lcnt), TB,
                                          PB, c, temps_all ? 1 : 0, flag ? 1 : 0);
    return;
  }
  const uint64_t n4 = (n + 3) / 4;
  if (!n4) return;
  const unsigned g = (unsigned)std::min<uint64_t>((n4 + RB - 1) / RB, 148 * 8);
  k_pstat1<<<g, RB, 0, st>>>(PA, NCP, n4, TB, PB, c, temps_all ? 1 : 0, flag ? 1 : 0, 0u);
}
void pstat2(uint32_t* PB, uint64_t n, uint32_t* PA, const uint32_t* TB, uint64_t* ctr, cudaStream_t st,
            uint32_t* NX, const uint32_t* list, const uint64_t* lcnt) {
  auto* c = reinterpret_cast<unsigned long long*>(ctr);
  if (list) {
    k_pstat2_list<<<148 * 8, RB, 0, st>>>(PB, list, reinterpret_cast<const unsigned long long*>(lcnt), PA, TB,
                                          c, NX);
    return;
  }
  const uint64_t n4 = (n + 3) / 4;
  if (!n4) return;
  const unsigned g = (unsigned)std::min<uint64_t>((n4 + RB - 1) / RB, 148 * 8);
  k_pstat2<<<g, RB, 0, st>>>(PB, n4, PA, TB, c, NX, 0u);
}
// ------------------------------------------------- iteration 0, pass A by pull (one GPU)
// Pass A pushes u_min(r) to PA[p] for every tuple p of every row r.  In iteration 0 the rows
// are the CSR rows of Alg. 1 line 3 (row r holds r and N(r)), and p is in row r iff r is in
// row p (both arcs of an edge are tuples), so PA[p] = min over the values x of row p of
// u_min(x): the same minima gathered by the row that owns the slot -- random reads of a
// u_min array instead of random reductions into PA (C2: 79 M reductions at the L2 reduction
// rate; C4 in mode sv: 2.2 G reductions into a 268 MB array).  Short rows by a thread each
// (rows are adjacent, so a warp reads one span), long rows by the segment kernels.
__global__ void k_u0(const uint32_t* __restrict__ off, const uint32_t* __restrict__ P, uint64_t n,
                     uint32_t* __restrict__ U, uint32_t* NCP) {
  for (uint64_t r = blockIdx.x * (uint64_t)RB + threadIdx.x; r < n; r += (uint64_t)gridDim.x * RB) {
    const uint32_t a = off[r], b = off[r + 1];
    if (a == b || b - a > LONG) continue;
    uint32_t mn = INF, mx = 0;
    for (uint32_t i = a; i < b; i++) {
      const uint32_t v = P[i];
      mn = min(mn, v);
      mx = max(mx, v);
    }
    U[r] = mn;
    if (mn != mx) set_bit(NCP, mn);  // not PC: 'not potentially completed' at its minimum (R18)
  }
}
// long rows: u_min and the max from k_long1<true>'s segment partials (the row's first segment)
__global__ void k_u0_long(const LongSeg* __restrict__ segs, const unsigned long long* nsegs,
                          const uint32_t* __restrict__ off, const unsigned long long* __restrict__ UMIN,
                          const unsigned long long* __restrict__ UMAX, uint32_t* __restrict__ U, uint32_t* NCP) {
  const uint64_t cnt = *nsegs;
  for (uint64_t s = blockIdx.x * (uint64_t)RB + threadIdx.x; s < cnt; s += (uint64_t)gridDim.x * RB) {
    const LongSeg sg = segs[s];
    if (sg.start != off[sg.u]) continue;
    const uint32_t mn = (uint32_t)UMIN[sg.u], mx = (uint32_t)UMAX[sg.u];
    U[sg.u] = mn;
    if (mn != mx) set_bit(NCP, mn);
  }
}
// WIN: one id window [lo, lo + span) of U per launch (n-sized U beyond the L2: the gathers of a
// window hit the L2 while P streams past it with evict-first loads; PA[p] accumulates the
// windows' minima -- still the slot's only writer)
template <bool WIN>
__global__ void k_pull0(const uint32_t* __restrict__ off, const uint32_t* __restrict__ P, uint64_t n,
                        const uint32_t* __restrict__ U, uint32_t* __restrict__ PA, uint32_t lo, uint32_t span) {
  for (uint64_t p = blockIdx.x * (uint64_t)RB + threadIdx.x; p < n; p += (uint64_t)gridDim.x * RB) {
    const uint32_t a = off[p], b = off[p + 1];
    if (a == b || b - a > LONG) continue;
    uint32_t mn = INF, i = a;
    if (WIN) {
      for (; i + 4 <= b; i += 4) {
        const uint32_t p0 = __ldcs(&P[i]), p1 = __ldcs(&P[i + 1]), p2 = __ldcs(&P[i + 2]), p3 = __ldcs(&P[i + 3]);
        const uint32_t u0 = p0 - lo < span ? __ldg(&U[p0]) : INF, u1 = p1 - lo < span ? __ldg(&U[p1]) : INF;
        const uint32_t u2 = p2 - lo < span ? __ldg(&U[p2]) : INF, u3 = p3 - lo < span ? __ldg(&U[p3]) : INF;
        mn = min(mn, min(min(u0, u1), min(u2, u3)));
      }
      for (; i < b; i++) {
        const uint32_t p0 = __ldcs(&P[i]);
        if (p0 - lo < span) mn = min(mn, __ldg(&U[p0]));
      }
      if (mn != INF) PA[p] = min(PA[p], mn);
    } else {
      for (; i + 4 <= b; i += 4) {  // four gathers in flight
        const uint32_t p0 = P[i], p1 = P[i + 1], p2 = P[i + 2], p3 = P[i + 3];
        const uint32_t u0 = __ldg(&U[p0]), u1 = __ldg(&U[p1]), u2 = __ldg(&U[p2]), u3 = __ldg(&U[p3]);
        mn = min(mn, min(min(u0, u1), min(u2, u3)));
      }
      for (; i < b; i++) mn = min(mn, __ldg(&U[P[i]]));
      PA[p] = mn;  // the slot's only writer
    }
  }
}
template <bool WIN>
__global__ void k_pull0_long(const uint32_t* __restrict__ P, const LongSeg* __restrict__ segs,
                             const unsigned long long* nsegs, const uint32_t* __restrict__ U, uint32_t* PA,
                             uint32_t lo, uint32_t span) {
  const int lane = threadIdx.x & 31;
  const uint64_t cnt = *nsegs;
  for (uint64_t s = (blockIdx.x * (uint64_t)RB + threadIdx.x) >> 5; s < cnt; s += ((uint64_t)gridDim.x * RB) >> 5) {
    const LongSeg sg = segs[s];
    uint32_t mn = INF;
    for (uint32_t i0 = lane; i0 < sg.len; i0 += 32 * LU) {
      uint32_t pv[LU], uv[LU];
#pragma unroll
      for (int u = 0; u < LU; u++)
        pv[u] = i0 + 32u * u < sg.len ? (WIN ? __ldcs(&P[sg.start + i0 + 32u * u]) : P[sg.start + i0 + 32u * u]) : INF;
#pragma unroll
      for (int u = 0; u < LU; u++)
        uv[u] = (WIN ? pv[u] - lo < span : pv[u] != INF) ? __ldg(&U[pv[u]]) : INF;
#pragma unroll
      for (int u = 0; u < LU; u++) mn = min(mn, uv[u]);
    }
    mn = __reduce_min_sync(FULL, mn);
    if (lane == 0 && mn != INF) atomicMin(&PA[sg.u], mn);
  }
}
// CC_PULLW: log2 of the window's id count (0: no windows); default 2^24 ids = 64 MB of U
static int pull_window_log2() {
  const char* e = getenv("CC_PULLW");  // read per run, so a test can switch it
  const int x = e && *e ? atoi(e) : 24;
  return x < 0 || x > 31 ? 0 : x;
}
void rowpass_a0_pull(const uint32_t* off, const uint32_t* P, uint64_t n, uint32_t* U, uint32_t* PA, uint32_t* NCP,
                     uint64_t* UMIN, uint64_t* UMAX, uint32_t tag, const LongSeg* segs, const uint64_t* nsegs,
                     bool have_long, cudaStream_t st) {
  if (!n) return;
  auto* umin = reinterpret_cast<unsigned long long*>(UMIN);
  auto* umax = reinterpret_cast<unsigned long long*>(UMAX);
  auto* ns = reinterpret_cast<const unsigned long long*>(nsegs);
  const unsigned g = (unsigned)std::min<uint64_t>((n + RB - 1) / RB, 148 * 8);
  k_u0<<<g, RB, 0, st>>>(off, P, n, U, NCP);
  if (have_long) {
    k_long1<true><<<148 * 4, RB, 0, st>>>(P, segs, ns, nullptr, umin, umax, tag);
    k_u0_long<<<148 * 2, RB, 0, st>>>(segs, ns, off, umin, umax, U, NCP);
  }
  // U beyond the L2 (C4 in mode sv: 268 MB): the gathers by windows of 2^pull_window_log2 ids
  const int wl = pull_window_log2();
  if (wl > 0 && n > (3ull << wl) / 2) {
    const uint32_t span = 1u << wl;
    // Short rows in one pass unless CC_PULLW_SHORT=1: a thread walks its row, so each window
    // costs the whole latency-bound walk again (C4 mode sv: 4 x 4.5 ms against 8.3 ms),
    // while the long rows' warps stream P at full rate (4 x 1.9 ms against 16.6 ms).
    const char* ws = getenv("CC_PULLW_SHORT");
    const bool win_short = ws && ws[0] == '1';
    if (!win_short) k_pull0<false><<<g, RB, 0, st>>>(off, P, n, U, PA, 0u, 0u);
    for (uint64_t lo = 0; lo < n; lo += span) {
      if (win_short) k_pull0<true><<<g, RB, 0, st>>>(off, P, n, U, PA, (uint32_t)lo, span);
      if (have_long) k_pull0_long<true><<<148 * 4, RB, 0, st>>>(P, segs, ns, U, PA, (uint32_t)lo, span);
    }
    return;
  }
  k_pull0<false><<<g, RB, 0, st>>>(off, P, n, U, PA, 0u, 0u);
  if (have_long) k_pull0_long<false><<<148 * 4, RB, 0, st>>>(P, segs, ns, U, PA, 0u, 0u);
}

void pstat1_block(uint32_t* PA, const uint32_t* NCP, uint64_t lo, uint64_t hi, uint32_t* TB, uint32_t* PB,
                  uint64_t* ctr, cudaStream_t st) {
  const uint64_t n4 = (hi - lo + 3) / 4;
  if (!n4) return;
  const unsigned g = (unsigned)std::min<uint64_t>((n4 + RB - 1) / RB, 148 * 8);
  k_pstat1<<<g, RB, 0, st>>>(PA + lo, NCP + lo / 32, n4, TB, PB + lo, reinterpret_cast<unsigned long long*>(ctr),
                             0, 1, (uint32_t)lo);
}
void pstat2_block(uint32_t* PB, uint64_t lo, uint64_t hi, uint32_t* PA, const uint32_t* TB, uint64_t* ctr,
                  cudaStream_t st) {
  const uint64_t n4 = (hi - lo + 3) / 4;
  if (!n4) return;
  const unsigned g = (unsigned)std::min<uint64_t>((n4 + RB - 1) / RB, 148 * 8);
  k_pstat2<<<g, RB, 0, st>>>(PB + lo, n4, PA + lo, TB + lo / 32, reinterpret_cast<unsigned long long*>(ctr),
                             nullptr, (uint32_t)lo);
}

// ------------------------------------------------------- owner-computes slot exchange (NEXT-1)
// Entries (slot, value | flag << 31) of the slots this rank touched outside its own block,
// grouped by the owner of the slot (owner k holds [k*blk, (k+1)*blk)).  S != NULL: slots
// with S[p] != INF, flag = BM bit (NCP); S == NULL: the set bits of BM, value 0, flag 1 (TB).
CC_DEVI bool oc_take(const uint32_t* S, const uint32_t* BM, uint64_t p, uint64_t n, uint64_t lo, uint64_t hi,
                     uint32_t* v) {
  if (p >= n || (p >= lo && p < hi)) return false;
  if (S) {
    *v = S[p];
    if (*v == INF) return false;
    if (BM) *v |= ((BM[p >> 5] >> (p & 31)) & 1u) << 31;
    return true;
  }
  *v = 0x80000000u;
  return (BM[p >> 5] >> (p & 31)) & 1u;
}
__global__ void k_oc_count(const uint32_t* __restrict__ S, const uint32_t* __restrict__ BM, uint64_t n,
                           uint64_t lo, uint64_t hi, uint64_t blk, int world, unsigned long long* cnt) {
  __shared__ uint32_t s[256];
  for (int i = threadIdx.x; i < world; i += RB) s[i] = 0;
  __syncthreads();
  for (uint64_t p = blockIdx.x * (uint64_t)RB + threadIdx.x; p < n; p += (uint64_t)gridDim.x * RB) {
    uint32_t v;
    if (oc_take(S, BM, p, n, lo, hi, &v)) atomicAdd(&s[p / blk], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < world; i += RB)
    if (s[i]) atomicAdd(&cnt[i], (unsigned long long)s[i]);
}
__global__ void k_oc_scatter(const uint32_t* __restrict__ S, const uint32_t* __restrict__ BM, uint64_t n,
                             uint64_t lo, uint64_t hi, uint64_t blk, unsigned long long* cursor,
                             uint2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (uint64_t p0 = blockIdx.x * (uint64_t)RB; p0 < n; p0 += (uint64_t)gridDim.x * RB) {
    const uint64_t p = p0 + threadIdx.x;
    uint32_t v = 0;
    const bool take = oc_take(S, BM, p, n, lo, hi, &v);
    const uint32_t own = take ? (uint32_t)(p / blk) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(FULL, own);
    if (take) {
      const int leader = __ffs(peers) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(&cursor[own], (unsigned long long)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      out[base + __popc(peers & ((1u << lane) - 1u))] = make_uint2((uint32_t)p, v);
    }
  }
}
// owner side: S[p] = min(S[p], value), BM bit p |= flag
__global__ void k_oc_apply(const uint2* __restrict__ in, uint64_t count, uint32_t* S, uint32_t* BM) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < count; i += (uint64_t)gridDim.x * RB) {
    const uint2 e = in[i];
    if (S) {
      const uint32_t v = e.y & 0x7FFFFFFFu;
      if (v < S[e.x]) atomicMin(&S[e.x], v);
    }
    if ((e.y >> 31) && BM) set_bit(BM, e.x);
  }
}
// owner side: the final value of every received slot, in receive order
__global__ void k_oc_gather(const uint2* __restrict__ in, uint64_t count, const uint32_t* __restrict__ S,
                            uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < count; i += (uint64_t)gridDim.x * RB)
    out[i] = S[in[i].x];
}
// requester side: S[sent[i].slot] = vals[i] (vals == NULL: INF, the clear)
__global__ void k_oc_put(const uint2* __restrict__ sent, uint64_t count, const uint32_t* __restrict__ vals,
                         uint32_t* S) {
  for (uint64_t i = blockIdx.x * (uint64_t)RB + threadIdx.x; i < count; i += (uint64_t)gridDim.x * RB)
    S[sent[i].x] = vals ? vals[i] : INF;
}
static unsigned oc_grid(uint64_t work) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + RB - 1) / RB, 148 * 8)); }
void oc_count(const uint32_t* S, const uint32_t* BM, uint64_t n, uint64_t lo, uint64_t hi, uint64_t blk, int world,
              uint64_t* cnt, cudaStream_t st) {
  if (n) k_oc_count<<<oc_grid(n), RB, 0, st>>>(S, BM, n, lo, hi, blk, world, reinterpret_cast<unsigned long long*>(cnt));
}
void oc_scatter(const uint32_t* S, const uint32_t* BM, uint64_t n, uint64_t lo, uint64_t hi, uint64_t blk,
                uint64_t* cursor, uint2* out, cudaStream_t st) {
  if (n) k_oc_scatter<<<oc_grid(n), RB, 0, st>>>(S, BM, n, lo, hi, blk, reinterpret_cast<unsigned long long*>(cursor), out);
}
void oc_apply(const uint2* in, uint64_t count, uint32_t* S, uint32_t* BM, cudaStream_t st) {
  if (count) k_oc_apply<<<oc_grid(count), RB, 0, st>>>(in, count, S, BM);
}
void oc_gather(const uint2* in, uint64_t count, const uint32_t* S, uint32_t* out, cudaStream_t st) {
  if (count) k_oc_gather<<<oc_grid(count), RB, 0, st>>>(in, count, S, out);
}
void oc_put(const uint2* sent, uint64_t count, const uint32_t* vals, uint32_t* S, cudaStream_t st) {
  if (count) k_oc_put<<<oc_grid(count), RB, 0, st>>>(sent, count, vals, S);
}

void list_from_bits(uint32_t* NX, uint64_t n, uint32_t* list, uint64_t* lcnt, uint32_t* NCP, uint32_t* TB,
                    uint32_t* PA, cudaStream_t st) {
  cudaMemsetAsync(lcnt, 0, sizeof(uint64_t), st);
  const uint64_t nw = (n + 31) / 32 + 2;  // the bitmaps' padding words too
  const unsigned g = (unsigned)std::min<uint64_t>((nw + RB - 1) / RB, 148 * 8);
  k_list_from_bits<<<g, RB, 0, st>>>(NX, nw, list, reinterpret_cast<unsigned long long*>(lcnt), NCP, TB, PA);
}

}  // namespace csr
}  // namespace cc
