// relabel.cuh -- u64 -> dense u32 relabel (Alg. 2 line 4) launchers.
#pragma once
#include "radix.cuh"
#include "scan.cuh"

namespace cc {
namespace relabel {

typedef int cc_status_t;

// ids: k = 2m endpoints (device).  Sorts (id, position) with the onesweep radix sort in
// keys/vals (two buffers each of k), writes dense[position] = rank of the id among the
// distinct ids and uids[rank] = id; *total (device u64) = number of distinct ids.
cc_status_t run(const uint64_t* ids, uint64_t k, uint64_t* keys[2], uint32_t* vals[2],
                radix::Workspace& rws, scan::State& ss, uint32_t* dense, uint64_t* uids,
                uint64_t* total, cudaStream_t st, uint64_t* launches);
// Same outputs as run() through a hash table of up to hash_slots(k) + 1 u64 entries (`table`,
// clobbered): only the distinct ids are sorted (keys/vals need room for them).  scratch: 3
// device u64.  Synchronises the stream (table overflow check; the distinct count sizes the sort).
// hash_slots(k) = 0: k too large for u32 slot indices at load < 0.9 -- use run().
// The first attempt needs hash_first_slots(k) + 1 entries; after a probe overflow run_hash
// needs hash_slots(k) + 1: it returns 1 when `table_slots` is short (the caller grows the table
// and calls again with start_full).
uint64_t hash_slots(uint64_t k);
uint64_t hash_first_slots(uint64_t k);
cc_status_t run_hash(const uint64_t* ids, uint64_t k, uint64_t* table, uint64_t table_slots, bool start_full,
                     uint64_t* keys[2], uint32_t* vals[2], radix::Workspace& rws, uint32_t* dense, uint64_t* uids,
                     uint64_t* total, uint64_t* scratch, cudaStream_t st, uint64_t* launches);
// Id permutation: out[i] = mix64(uids[i]); e[i] = pi[e[i]];
// canonicalize: out[v] = min { w : label[pi[w]] = label[pi[v]] } (v, w original dense ranks)
void mix(const uint64_t* uids, uint64_t n, uint64_t* out, cudaStream_t st);
void apply(uint32_t* e, uint64_t k, const uint32_t* pi, cudaStream_t st);
void canonicalize(const uint32_t* pi, const uint32_t* label, uint64_t n, uint32_t* mino, uint32_t* out,
                  cudaStream_t st);
// out[i] = uids[label[i]] for the n dense ids
void labels(const uint64_t* uids, const uint32_t* label, uint64_t n, uint64_t* out, cudaStream_t st);

}  // namespace relabel
}  // namespace cc
