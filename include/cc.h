/*
 * cc.h -- C ABI of the B200-native adaptive connected-components library (libcc.so).
 *
 * Method: Jain, Flick, Pan, Green, Aluru, "An Adaptive Parallel Algorithm for Computing
 * Connected Components" (arXiv 1607.06156).  References below are to that paper's
 * LaTeX source (PAPER.md:<line>) and to SURVEY.md §8(b), which fixes this boundary.
 *
 * What cc_run computes (PAPER.md:28 definition, PAPER.md:197 projection):
 *   label(v) = min { u : u is connected to v }   (the component's minimum vertex id)
 * via Alg. 2: degree distribution -> power-law gate -> optionally one
 * BFS that peels the giant component -> edge-tuple Shiloach-Vishkin (Alg. 1,
 * PAPER.md:133-178) with completed-partition exclusion on the rest.
 *
 * Conventions (all entry points):
 *  - Status codes only; nothing aborts, exits or throws across the ABI.  Details of the
 *    last failure are in cc_last_error(ctx).
 *  - Pointers are plain host or device pointers, sizes are element counts.  Input
 *    buffers are borrowed for the duration of the call only (copied).  Output buffers are
 *    caller-allocated.  cc_report.iters is owned by the context and valid until the next
 *    cc_run / cc_destroy.
 *  - All device work is enqueued on cfg.stream (a cudaStream_t, NULL = legacy default);
 *    cc_run and cc_labels_* return after their results are complete (they synchronise
 *    that stream).
 *  - Device memory comes from cfg.alloc/cfg.free when set (e.g. the PyTorch caching
 *    allocator), else from cudaMallocAsync on cfg.stream.
 *  - One context per thread per GPU.
 */
#ifndef CC_H_
#define CC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cc_ctx cc_ctx; /* opaque; owns all device buffers */

typedef enum {
  CC_OK = 0,
  CC_ERR_INVALID = 1, /* bad argument (NULL pointer, bad mode, n too large, ...) */
  CC_ERR_RANGE = 2,   /* u32 mode: an edge endpoint >= n_vertices (checked on device) */
  CC_ERR_NOMEM = 3,   /* device allocation failed */
  CC_ERR_CUDA = 4,    /* a CUDA runtime error (message in cc_last_error) */
  CC_ERR_COMM = 5,    /* multi-GPU exchange failed */
  CC_ERR_STATE = 6,   /* call out of order, e.g. cc_run before cc_load_edges */
  CC_ERR_NOCONV = 7   /* SV did not converge within 2*ceil(log2 n)+8 iterations */
} cc_status;

typedef enum {
  CC_MODE_AUTO = 0,   /* Alg. 2: the gate decides whether to run the BFS peel */
  CC_MODE_SV = 1,     /* hard-coded: SV only (fig:dynamic 'never BFS')        */
  CC_MODE_BFS_SV = 2  /* hard-coded: BFS peel, then SV on the remainder       */
} cc_mode;

typedef enum { CC_U32 = 0, CC_U64 = 1 } cc_idw;

/* cc_config.flags */
#define CC_FLAG_TRACE 0x1u           /* also fit the histogram + K-S in forced modes        */
#define CC_FLAG_GATE_KS 0x2u         /* decide with the paper's K-S < tau
                                        instead of gate G (least-squares fit)  */
#define CC_FLAG_NO_EARLY_EXCLUDE 0x4u /* csr engine: completed partitions leave at the end of
                                        the iteration (the paper's timing; their
                                        temporaries are made, T_i = |P_i|) -- SURVEY C4    */
#define CC_FLAG_PERMUTE_IDS 0x100u   /* u64 ids: run on ids permuted by a 64-bit invertible
                                        mix, labels mapped back to the minimum
                                        original id of each component (C1)               */
#define CC_FLAG_NO_EXCLUDE 0x80u     /* csr engine: completed partitions never leave
                                        (fig:loadbal 'Naive'): iterate until no
                                        partition changes in either partition pass         */
/* SV regroup engine (all three compute identical sets and counters):
 *   default : r-stationary -- tuples regrouped by r once (CSR build), partition buckets
 *             addressed directly in L2-resident slots, ordered compaction
 *   SORT    : the paper's four radix-sort regroups per iteration
 *   DIRECT  : no regroup at all; both bucket kinds addressed directly (ablation)        */
#define CC_FLAG_REGROUP_SORT 0x8u
#define CC_FLAG_REGROUP_DIRECT 0x20u
#define CC_FLAG_PROFILE 0x10u        /* CUDA-event timing of kernel families (cc_kernel_stats) */
#define CC_FLAG_NO_COLLAPSE 0x200u   /* csr engine: never collapse potentially-completed rows
                                        to one tuple (ablation; DESIGN.md §5.2 row collapse) */
#define CC_FLAG_NO_RENUMBER 0x400u   /* BFS route: run the SV on the remainder with the original
                                        id range instead of its endpoints renumbered densely in
                                        id order (ablation)                   */
#define CC_FLAG_BALANCE 0x800u      /* several ranks, csr engine with exclusion: the paper's
                                        'balanced' variant -- the live rows are
                                        redistributed evenly over the ranks after an iteration
                                        whose most loaded rank holds > 1/16 above the mean  */
#define CC_FLAG_DENSE_EXCHANGE 0x1000u /* several ranks: combine the partition slots by dense
                                        n-slot all-reduces (and a sparse all-gather late)
                                        instead of the owner-computes exchange (
                                        ablation)                                            */
#define CC_FLAG_BFS_CSR 0x40u        /* csr engine: degrees from the bucketed CSR build and a
                                        direction-optimising (top-down / bottom-up) BFS on the
                                        CSR rows instead of the edge-streaming BFS            */

/* ---- multi-GPU exchange (world_size > 1).  The library runs one process per GPU.  Two ways
 * to connect the ranks:
 *  (1) library-owned NCCL: rank 0 calls cc_get_unique_id, the caller
 *      broadcasts the 128 bytes (e.g. torch.distributed.broadcast_object_list), and every
 *      rank passes them as cfg.nccl_id.  cc_init then creates an NCCL communicator
 *      (ncclCommInitRank; collective: all ranks must be inside cc_init together) and every
 *      exchange is an NCCL call enqueued on cfg.stream -- no host synchronisation per
 *      collective, no callback into the caller.  libnccl.so.2 is loaded at run time (the
 *      copy already in the process if any; CC_NCCL_LIB=path overrides).  world_size == 1
 *      with nccl_id runs the sharded driver on a 1-rank communicator (tests).
 *  (2) caller callbacks (cfg.comm, below; used when nccl_id is NULL), e.g.
 *      torch.distributed over gloo in the CPU-side tests.  Every
 * callback is entered with all earlier work on `stream` complete and must return 0 only once
 * its result is in place in the (device) buffers; nonzero -> CC_ERR_COMM.  All ranks call the
 * same sequence of collectives (SPMD).  Element types follow cc_dtype; the library maps its
 * unsigned slot values to an order-preserving signed form before MIN / MAX. */
typedef enum { CC_DT_I32 = 0, CC_DT_I64 = 1, CC_DT_U8 = 2 } cc_dtype;
typedef enum { CC_OP_SUM = 0, CC_OP_MIN = 1, CC_OP_MAX = 2 } cc_redop;
typedef struct {
  void* user;
  /* in place: buf[i] <- op over ranks of buf[i], i < count */
  int (*allreduce)(void* user, void* buf, uint64_t count, int dtype, int op, void* stream);
  /* recv (world_size * bytes) <- concatenation, rank-major, of every rank's `bytes` at send */
  int (*allgather)(void* user, const void* send, void* recv, uint64_t bytes, void* stream);
  /* send: world_size consecutive blocks, send_bytes[k] for rank k; recv: recv_bytes[k] from
   * rank k, rank-major.  The byte-count arrays are host arrays of world_size entries. */
  int (*alltoallv)(void* user, const void* send, const uint64_t* send_bytes, void* recv,
                   const uint64_t* recv_bytes, void* stream);
} cc_comm;

typedef void* (*cc_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*cc_free_fn)(void* ptr, size_t bytes, void* stream, void* user);

typedef struct {
  int device;          /* CUDA device ordinal                                         */
  void* stream;        /* cudaStream_t; NULL = legacy default stream                   */
  int rank, world_size;/* SPMD position; world_size == 1 for a single GPU              */
  const cc_comm* comm; /* collectives for world_size > 1 (borrowed; must outlive ctx)  */
  cc_alloc_fn alloc;   /* optional device allocator hooks (NULL => cudaMallocAsync)     */
  cc_free_fn free;
  void* alloc_user;
  double tau;          /* K-S threshold for CC_FLAG_GATE_KS; <= 0 => 0.05*/
  uint64_t seed;       /* reserved (deterministic run; no randomness is drawn)         */
  uint32_t flags;      /* CC_FLAG_*                                                    */
  const void* nccl_id; /* CC_UNIQUE_ID_BYTES from cc_get_unique_id (rank 0, broadcast), or
                          NULL.  Non-NULL: library-owned NCCL communicator (cfg.comm ignored) */
} cc_config;

#define CC_UNIQUE_ID_BYTES 128

/* 128-byte NCCL unique id for cfg.nccl_id (call on rank 0 only, broadcast the bytes to the
 * other ranks).  CC_ERR_COMM if libnccl cannot be loaded or fails (cc_last_error(NULL) is
 * not available: the reason is written to `why` when non-NULL, up to why_len bytes). */
cc_status cc_get_unique_id(void* out128, char* why, size_t why_len);

/* One SV iteration (counters of SURVEY.md §8(c) "Trace oracle"). */
typedef struct {
  uint64_t active_in;  /* A_i: non-temporary tuples entering the iteration             */
  uint64_t partitions; /* |P_i| at the first partition pass                            */
  uint64_t temps;      /* T_i: temporary tuples <p_min,_,p_min>_tmp appended    */
  uint64_t completed;  /* partitions found completed                    */
  uint64_t changed;    /* #{p : p_min != p} at the first partition pass        */
  uint64_t changed2;   /* same count at the second partition pass             */
  uint64_t active_min; /* live tuples entering the iteration on the least / most loaded */
  uint64_t active_max; /* rank (fig:loadbal); = active_in on one GPU.  With
                          several ranks they are reduced only under CC_FLAG_TRACE (two
                          extra all-reduces per iteration); otherwise this rank's count */
  double ms;           /* device time of the iteration                                 */
} cc_iter_stat;

typedef struct {
  int ran_bfs;                        /* route taken by Alg. 2                          */
  double ls_alpha, ls_r2;             /* gate G: log-log least-squares fit              */
  double ks_stat, ks_alpha;           /* paper's K-S statistic and alpha-hat (reported) */
  uint32_t ks_xmin;
  uint64_t max_degree;
  uint64_t n_present;                 /* ids touched by an edge                         */
  uint64_t m_edges;                   /* undirected edge records (incl. dups, loops)    */
  uint64_t components;                /* number of components (isolated ids included)   */
  uint64_t bfs_root, bfs_visited, bfs_levels, remainder_edges;
  uint32_t sv_iterations;
  double ms_total, ms_prediction, ms_relabel, ms_bfs, ms_filter, ms_sv, ms_finalize;
  const cc_iter_stat* iters;          /* sv_iterations entries (CC_FLAG_TRACE)          */
  uint32_t n_iters;
  int bfs_spec_root;                  /* 1: the BFS root's level ran inside the degree
                                         pass on a guessed root that proved exact (large
                                         lists); labels are unaffected  */
  uint64_t sv_ids;                    /* id range the SV ran on: n, or n' (the remainder's
                                         endpoints renumbered densely in id order, BFS
                                         route); 0 if no SV ran           */
} cc_report;

/* Library version string. */
const char* cc_version(void);

/* Create a context on cfg->device.  cfg is copied.  Returns CC_ERR_INVALID for a NULL
 * argument, a bad rank / world_size, or world_size > 1 with neither cfg->nccl_id nor
 * cfg->comm; CC_ERR_CUDA if the device cannot be used; CC_ERR_COMM if the NCCL communicator
 * cannot be created (collective with nccl_id: every rank calls cc_init).  In multi-GPU contexts (world_size > 1) cc_load_edges,
 * cc_run are collective (every rank calls them, each with its own block of edges). */
cc_status cc_init(const cc_config* cfg, cc_ctx** out);

/* Load an undirected edge list (the input G(V,E) of Alg. 1/2; PAPER.md:205 block
 * distributed edge list, here one block per rank).
 *   w          CC_U32: ids are uint32 < n_vertices; CC_U64: ids are arbitrary uint64
 *   pairs      interleaved endpoints (u0,v0,u1,v1,...): 2*m_local ids of width w
 *   m_local    number of undirected edge records on this rank (duplicates and
 *              self-loops are legal and kept)
 *   n_vertices u32: id bound n (V = [0,n), isolated ids are singleton components);
 *              u64: must be 0 (V = ids that appear in the edge list)
 *   pairs_on_device  nonzero if `pairs` is a device pointer
 * Ids >= n in u32 mode -> CC_ERR_RANGE (detected on device).  n > 2^30 -> CC_ERR_INVALID.
 * u64 mode: cc_run first relabels the ids to dense [0, |V|) in id order (Alg. 2 line 4,
 * PAPER.md:260, :277; timed as ms_relabel); more than 2^30 distinct ids -> CC_ERR_INVALID.
 * Replaces any previously loaded graph. */
cc_status cc_load_edges(cc_ctx* ctx, cc_idw w, const void* pairs, uint64_t m_local,
                        uint64_t n_vertices, int pairs_on_device);

/* Compute component labels (Alg. 2 with `mode`), fill *out if non-NULL.  Labels stay on
 * the device for cc_labels_*.  CC_ERR_STATE if no graph is loaded. */
cc_status cc_run(cc_ctx* ctx, cc_mode mode, cc_report* out);

/* u32 mode: labels of ids [0, n), or of this rank's block [lo, hi) (cc_block_range) when
 * world_size > 1.  `out` has room for `cap` labels; *count receives the label count.
 * CC_ERR_INVALID if cap is smaller. */
cc_status cc_labels_u32(cc_ctx* ctx, uint32_t* out, uint64_t cap, uint64_t* count,
                        int out_on_device);

/* u64 mode: the distinct ids (ascending) into `ids` and the label of each (the minimum id
 * of its component) into `labels`; both have room for `cap` entries, *count receives the
 * number of distinct ids.  CC_ERR_STATE on a u32 graph (and cc_labels_u32 on a u64 one).
 * world_size > 1: the ids are relabelled over all ranks by a distributed sort-unique
 * (sample-sort splitters, two all-to-all-v exchanges), rank k owns the
 * block [lo, hi) of the dense ids (cc_block_range) and receives the original ids of that
 * block with their labels (*count = hi - lo; the ranks' outputs concatenate to the global
 * sorted id list).  Collective then: every rank calls it with buffers (a call with NULL
 * buffers only reports *count and returns CC_ERR_INVALID, without communicating).
 * CC_FLAG_PERMUTE_IDS is single-GPU (CC_ERR_INVALID from cc_load_edges otherwise). */
cc_status cc_labels_u64(cc_ctx* ctx, uint64_t* ids, uint64_t* labels, uint64_t cap,
                        uint64_t* count, int out_on_device);

/* The degree distribution D of the last cc_run (Alg. 2 line 2): the
 * non-empty bins (d, D[d]), d >= 1 ascending, with D[d] = #{v : deg(v) = d} and deg(v) = arcs
 * with source v (a self-loop counts 2) -- exactly the input the power-law
 * gate (line 3) was fitted on.  Summed over all ranks when world_size > 1.  `degrees` and
 * `counts` (host) have room for `cap` bins; *count receives the bin count.  CC_ERR_STATE if the
 * last cc_run did not build it (it does in CC_MODE_AUTO or under CC_FLAG_TRACE);
 * CC_ERR_INVALID if cap is smaller. */
cc_status cc_degree_histogram(cc_ctx* ctx, uint64_t* degrees, uint64_t* counts, uint64_t cap,
                              uint64_t* count);

/* deg(v) for every id v in [0, n) (Alg. 2 line 2; same kernels and dispatch as the prediction
 * stage of cc_run) into `out` (room for `cap`, host or device per out_on_device); *count = n.
 * u32 graphs on one GPU (CC_ERR_INVALID otherwise); CC_ERR_STATE before cc_load_edges.  Uses
 * the context's tuple scratch: labels of an earlier cc_run are invalidated (CC_ERR_STATE from
 * cc_labels_* until the next cc_run). */
cc_status cc_degrees_u32(cc_ctx* ctx, uint32_t* out, uint64_t cap, uint64_t* count, int out_on_device);

/* Multi-GPU (world_size > 1): rank k owns the vertex block [k*B, min((k+1)*B, n)) with
 * B = 32*ceil(n / (32*world_size)) -- its CSR rows (owner-computes) and its
 * labels.  Writes the block of this rank (lo = 0, hi = n on one GPU). */
cc_status cc_block_range(const cc_ctx* ctx, uint64_t* lo, uint64_t* hi);

/* BFS eccentricity (depth of the BFS tree within the seed's component) of each of `count`
 * seeds into ecc[i]: the paper's approximate diameter is the maximum over random seeds
 * (PAPER.md:307).  u32 graphs on one GPU, n <= 2^26 (CC_ERR_INVALID otherwise); seeds >= n ->
 * CC_ERR_RANGE.  Uses the direction-optimising BFS on the CSR rows; invalidates the labels of
 * an earlier cc_run (CC_ERR_STATE from cc_labels_* until the next cc_run). */
cc_status cc_bfs_eccentricity(cc_ctx* ctx, const uint64_t* seeds, uint32_t count, uint64_t* ecc);

/* The paper's approximate diameter (approximated "by executing a total of 100
 * BFS runs from a set of random seed vertices"; read as the largest depth found): the maximum of cc_bfs_eccentricity over the `count` seeds the caller drew (host
 * array; the draw is the caller's so that a test passes the same seeds to its oracle) into
 * *diameter (0 with no seed).  Same limits, errors and side effects as cc_bfs_eccentricity. */
cc_status cc_approx_diameter(cc_ctx* ctx, const uint64_t* seeds, uint32_t count, uint64_t* diameter);

/* Stable LSD radix sort (the onesweep regroup primitive of the sort engine, PAPER.md:207
 * "the bulk step of the algorithm is the sorting of tuples") of n 64-bit keys by their bits
 * [0, key_bits), key_bits in 1..64 (keys must be < 2^key_bits), carrying a u32 payload.  keys/vals: device arrays of n,
 * sorted in place; tmp_keys/tmp_vals: device scratch of n each.  Enqueued on `stream`
 * (cudaStream_t) and synchronised; its look-back workspace (8 B x 256 per 4096 keys) comes
 * from cudaMallocAsync.  For the SURVEY NEXT-3 sort microbenchmark (scripts/sort_bench.py). */
cc_status cc_radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t* tmp_keys, uint32_t* tmp_vals,
                              uint64_t n, int key_bits, void* stream);

/* Device pointer of the label array (u32 mode), valid until the next load/destroy, and
 * the device stream all work is enqueued on.  For zero-copy consumers. */
cc_status cc_labels_device(cc_ctx* ctx, const uint32_t** labels, uint64_t* count);

/* Switch the CC_FLAG_PROFILE event timing on (nonzero) or off for the following cc_run calls
 * (bench.py times the step without events, then the per-kernel breakdown with them). */
cc_status cc_set_profiling(cc_ctx* ctx, int on);

/* Number of kernel launches enqueued by the last cc_run (evidence for bench.py). */
uint64_t cc_last_launch_count(const cc_ctx* ctx);

/* Device time (ms, CUDA events on cfg.stream around each launch) of kernel family
 * `which` in the last cc_run, recorded only under CC_FLAG_PROFILE, with the family's
 * algorithmic bytes (DESIGN.md §6 byte model) and launch count.  Families are numbered
 * 0..N-1; cc_kernel_name(which) names them and returns NULL past the last one.
 * CC_ERR_INVALID for a bad index. */
cc_status cc_kernel_stats(const cc_ctx* ctx, int which, double* ms, double* bytes,
                          uint64_t* launches);
const char* cc_kernel_name(int which);
/* The random accesses family `which` made in the last cc_run under CC_FLAG_PROFILE (its
 * algorithmic count, e.g. 2 L2 reads per edge of a BFS level, 2 shared-memory atomics per arc
 * of the bucketed degree count) and their unit ("" if the family is not access-bound), for a
 * request-rate roofline beside the bytes of cc_kernel_stats.  CC_ERR_INVALID for a bad index. */
cc_status cc_kernel_ops(const cc_ctx* ctx, int which, double* ops, const char** unit);

cc_status cc_destroy(cc_ctx* ctx);

const char* cc_status_string(cc_status s);
const char* cc_last_error(const cc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* CC_H_ */
