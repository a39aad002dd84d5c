// csr.cuh -- launchers of the r-stationary SV engine (sv_csr.cu).
#pragma once
#include "scan.cuh"

namespace cc {
namespace csr {

// CSR build (counting regroup by r): off[v] / cur[v] from degrees; ctr[C_VT_OUT] = A_0.
int group_shift(uint64_t n, uint64_t tuples);
// count_groups: also accumulate per-group arc counts into garc (false when bucket_degrees
// already produced them).
void build(const uint2* edges, uint64_t m, const uint32_t* deg, const uint32_t* vis, uint64_t n,
           uint32_t* off, uint32_t* cur, uint32_t* garc, int gshift, scan::State& ss, uint64_t* ctr,
           cudaStream_t st, bool count_groups = true);
// Full-graph CSR path (n <= 2^26): gshift for groups of <= 2^15 ids (-1: n too large).
int group_shift_full(uint64_t n);
// Bucket both arcs of every edge by the group of r into tmp (2m uint2) and count degrees per
// group in shared memory (Alg. 2 line 2 without global atomics); garc/gcur: group scratch.
void bucket_degrees(const uint2* edges, uint64_t m, uint64_t n, int gshift, uint32_t* garc,
                    uint64_t* gcur, uint2* tmp, uint32_t* deg, cudaStream_t st);
// R, vertex tuples and the row scatter of the bucketed arcs (after build with the same deg).
void fill_from_buckets(const uint32_t* off, uint32_t* cur, uint64_t n, uint64_t A, uint32_t* R,
                       uint32_t* P, const uint2* tmp, uint64_t na, uint32_t* longlist, uint64_t* nlong,
                       cudaStream_t st);
// R fill, vertex tuples, and the arc placement: bucket by vertex group, re-bucket by
// subgroup of 2^13 ids into P-aligned scratch, place rows with shared-memory cursors.  R and
// P must be the two halves of one allocation (P - R >= 2m; the group buckets use it), tmp
// is cap uint2 of scratch; longlist: n uint32 scratch; garc/gcur: group entries.  `directed`:
// `edges` holds m arcs (r, p) instead of m undirected edges (two arcs each).
void fill(const uint2* edges, uint64_t m, const uint32_t* off, uint32_t* cur, uint64_t n, uint64_t A,
          uint32_t* R, uint32_t* P, const uint32_t* garc, int gshift, uint64_t* gcur, uint2* tmp,
          uint32_t* longlist, uint64_t* nlong, cudaStream_t st, bool directed = false);
// Row passes (sv_rows.cu).  Rows longer than LONG tuples (R_LONG set in R) are handled as
// segments of at most LSEG tuples by warps (k_long1/k_long2); the segment list is rebuilt
// after each compaction.
constexpr uint32_t LONG = 256;
constexpr uint32_t LSEG = 1024;
constexpr uint32_t R_LONG = 0x80000000u;  // flag in R of the tuples of long rows (ids < 2^30)
struct LongSeg {
  uint64_t start;
  uint32_t u, len;
};
uint64_t row_tiles(uint64_t L);
uint64_t long_seg_cap(uint64_t L);
void longlist(const uint32_t* R, const uint32_t* P, uint64_t L, const uint32_t* deg, LongSeg* segs,
              uint64_t* nsegs, cudaStream_t st);
// P is read from Pin and the relabelled values written to Pout (NULL: pass A without MAP).
// pass A (MAP = PB of the previous iteration or NULL; OUT = PA; NCPw = NCP) or pass B
// (MAP = PA, NCPr = NCP, TB; OUT = PB; label; ctr[C_OUT] += live tuples; excl: completed
// partitions leave, else they stay).  `tag` must
// increase with every call (tagged long-row partial slots UMIN/UMAX).  `hot`: few distinct
// partitions per tuple, filter slot updates through the block's cache.
void rowpass(bool passA, const uint32_t* R, const uint32_t* Pin, uint32_t* Pout, uint64_t L,
             const uint32_t* MAP, const uint32_t* NCPr, const uint32_t* TB, uint32_t* OUT,
             uint32_t* NCPw, uint32_t* label, uint64_t* UMIN, uint64_t* UMAX, uint32_t tag,
             const LongSeg* segs, const uint64_t* nsegs, bool have_long, bool hot, uint64_t* ctr,
             cudaStream_t st, bool excl = true, bool preset = false, const uint64_t* prevctr = nullptr,
             int hot_shift = 0, const uint32_t* HW = nullptr, const uint64_t* hotcnt = nullptr,
             int hot_mode = 0);
// HW (pass B, row collapse): HW[r] = tuples folded into row r by collapse(); a row that leaves
// adds them to ctr[C_HIDDEN_DEAD] (NULL before the first collapse of a run)
// prevctr (device, the previous iteration's sv counters): the pass returns at once when it
// left no live tuple, and is hot when |P_prev| << hot_shift < L (overrides `hot`).
// hotcnt (device; overrides prevctr's count, and selects on the device in the first iteration
// too): the number of distinct slots the pass updates, hot when count << hot_shift < L --
// hot_mode 0: hotcnt[0] (pass A: |P_i|, the partition list's length); 1: hotcnt is this
// iteration's sv counters after pstat1, count = |P_i| - changed + T_i (pass B's targets:
// the unchanged partitions and the distinct p_min of the changed ones)
// partition statistics after pass A (sets TB, clears PB); slot arrays padded to 4*ceil(n/4)
// temps_all: a temporary for every partition, completed ones included (their tuples leave at
// the end of the iteration or never)
// list / lcnt (device): scan only the slots of the partition-id superset L_i (all slot writes
// of iteration i land in P_i, a subset of L_i, and L_i+1 is a subset of L_i);
// PB is then cleared over prev = L_i-1 (NULL: all of it).  list NULL: all n slots
// flag: completed partitions get bit 31 set in PA (pass B reads it in its relabel gather)
void pstat1(uint32_t* PA, const uint32_t* NCP, uint64_t n, uint32_t* TB, uint32_t* PB,
            uint64_t* ctr, cudaStream_t st, bool temps_all, bool flag, const uint32_t* list = nullptr,
            const uint64_t* lcnt = nullptr, const uint32_t* prev = nullptr, const uint64_t* pcnt = nullptr);
// labels of the rows still in the array (no-exclusion variant)
void final_labels(const uint32_t* R, const uint32_t* P, uint64_t L, uint32_t* label, cudaStream_t st);
// after pass B: the temporaries' own element (PB[u] = min(PB[u], u) for TB(u)), changed2,
// PA cleared; marks in NX the next iteration's partition ids { PB[v] : TB(v) } (exact unless
// CC_FLAG_NO_EARLY_EXCLUDE, where TB also holds completed partitions); list variant over L_i
void pstat2(uint32_t* PB, uint64_t n, uint32_t* PA, const uint32_t* TB, uint64_t* ctr, cudaStream_t st,
            uint32_t* NX, const uint32_t* list = nullptr, const uint64_t* lcnt = nullptr);
// list[0..*lcnt) = ids of the set bits of NX (bitmap of n bits, cleared on the way); with PA
// (exact list) each id gets PA[id] = id preset (pass A then skips updates q = p); clears the
// NCP and TB bitmaps for the next iteration
void list_from_bits(uint32_t* NX, uint64_t n, uint32_t* list, uint64_t* lcnt, uint32_t* NCP, uint32_t* TB,
                    uint32_t* PA, cudaStream_t st);
// multi-GPU sparse slot exchange: touched slots as (p, value | NCP(p) << 31) entries (*cnt =
// their number), and min / OR application of a list (entries with p = ~0 are padding)
void extract_slots(const uint32_t* S, const uint32_t* BM, uint64_t n, uint2* out, uint64_t* cnt,
                   cudaStream_t st);
void apply_slots(const uint2* in, uint64_t count, uint32_t* S, uint32_t* BM, cudaStream_t st);
// Iteration 0's pass A by pull (one GPU, the tuple array still in CSR order with offsets
// off[0..n]): U[r] = u_min(r), NCP(u_min) of non-PC rows, PA[p] = min over row p's values x
// of U[x]; U is n-sized scratch (PB: k_pstat1 clears it next), tag the long-row epoch
void rowpass_a0_pull(const uint32_t* off, const uint32_t* P, uint64_t n, uint32_t* U, uint32_t* PA, uint32_t* NCP,
                     uint64_t* UMIN, uint64_t* UMAX, uint32_t tag, const LongSeg* segs, const uint64_t* nsegs,
                     bool have_long, cudaStream_t st);
// multi-GPU owner-computes exchange (NEXT-1; cc_api.cu sv_iterate).  pstat1/pstat2 over one
// owner block [lo, hi) (lo a multiple of 32; TB absolute in pstat1, ids offset by lo; no list)
void pstat1_block(uint32_t* PA, const uint32_t* NCP, uint64_t lo, uint64_t hi, uint32_t* TB, uint32_t* PB,
                  uint64_t* ctr, cudaStream_t st);
void pstat2_block(uint32_t* PB, uint64_t lo, uint64_t hi, uint32_t* PA, const uint32_t* TB, uint64_t* ctr,
                  cudaStream_t st);
// entries (p, value | flag << 31) of the touched slots outside [lo, hi), grouped by owner p / blk:
// S != NULL: S[p] != INF (flag: the BM bit); S == NULL: set bits of BM.  oc_count adds the
// per-owner counts to cnt[world]; oc_scatter writes them at cursor[owner]++ (exclusive offsets)
void oc_count(const uint32_t* S, const uint32_t* BM, uint64_t n, uint64_t lo, uint64_t hi, uint64_t blk, int world,
              uint64_t* cnt, cudaStream_t st);
void oc_scatter(const uint32_t* S, const uint32_t* BM, uint64_t n, uint64_t lo, uint64_t hi, uint64_t blk,
                uint64_t* cursor, uint2* out, cudaStream_t st);
// owner: S[p] = min(S[p], value) (S may be NULL), BM bit |= flag; out[i] = S[in[i].p]
void oc_apply(const uint2* in, uint64_t count, uint32_t* S, uint32_t* BM, cudaStream_t st);
void oc_gather(const uint2* in, uint64_t count, const uint32_t* S, uint32_t* out, cudaStream_t st);
// requester: S[sent[i].p] = vals[i] (vals NULL: INF)
void oc_put(const uint2* sent, uint64_t count, const uint32_t* vals, uint32_t* S, cudaStream_t st);
// multi-GPU slot exchange helpers: a[i] ^= 0x80000000; out[i] = OR_k parts[k*words + i]
void flip_sign(uint32_t* a, uint64_t n, cudaStream_t st);
void or_parts(const uint32_t* parts, uint64_t words, int world, uint32_t* out, cudaStream_t st);
// ordered compaction that also collapses every potentially-completed row (all live p equal,
// PAPER.md:150-155) that lies inside one compaction tile and is not a long row to its head
// tuple: such a row stays PC for good (one relabel maps its equal values to one value), so its
// other tuples repeat the head's bucket updates (min is idempotent).  HW[r] += the tuples
// folded into row r, *hidden += their total, *out_len = the output length.  Partition sets,
// completion, temporaries and every trace counter are unchanged; A_i = live + hidden.
void collapse(const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* R2, uint32_t* P2, uint32_t* HW,
              uint64_t* hidden, uint64_t* out_len, scan::State& ss, cudaStream_t st);
// ordered compaction of live tuples (R order kept); output count = live count
void compact(const uint32_t* R, const uint32_t* P, uint64_t A, uint32_t* R2, uint32_t* P2,
             scan::State& ss, cudaStream_t st);

}  // namespace csr
}  // namespace cc
