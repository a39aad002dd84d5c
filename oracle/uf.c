/*
 * oracle/uf.c -- CPU union-find oracle for connected-component labels.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this.  It shares no code with the
 * CUDA path (paper_1607_06156_b200/).
 *
 * Plain definition ("two vertices belong to the same connected component
 * iff there is a path"; "the unique connected component label c ... projected
 * from any tuple <c,_,u>"): label(v) = min{u : u connected to v}.
 *
 * Algorithm ("union-find based algorithm, where each vertex is initially
 * assumed to be a different graph component and components connected by an edge are
 * iteratively merged"; PAPER.md:431 union-find is the best sequential method):
 *   parent[v] = v; for each edge (a,b): ra=find(a), rb=find(b); if ra!=rb link the
 *   larger root under the smaller.  Roots are therefore always their set's minimum, so
 *   label[v] = find(v) needs no canonicalisation.  find() uses path halving.
 * Single-threaded on purpose (it is also the timed CPU baseline).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint32_t find32(uint32_t* parent, uint32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]]; /* path halving */
    x = parent[x];
  }
  return x;
}

/* u32 mode: ids in [0,n); edges interleaved (a0,b0,a1,b1,...).  Returns -1 if an id
 * is out of range, else the number of components (including isolated ids). */
int64_t oracle_uf_labels_u32(uint64_t n, const uint32_t* edges, uint64_t m, uint32_t* label) {
  uint32_t* parent = label; /* reuse the output buffer as the forest */
  for (uint64_t v = 0; v < n; v++) parent[v] = (uint32_t)v;
  for (uint64_t e = 0; e < m; e++) {
    uint32_t a = edges[2 * e], b = edges[2 * e + 1];
    if (a >= n || b >= n) return -1;
    uint32_t ra = find32(parent, a), rb = find32(parent, b);
    if (ra != rb) {
      if (ra < rb) parent[rb] = ra; else parent[ra] = rb;
    }
  }
  int64_t comps = 0;
  for (uint64_t v = 0; v < n; v++) {
    label[v] = find32(parent, (uint32_t)v);
    comps += (label[v] == v);
  }
  return comps;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

static uint64_t lower_bound(const uint64_t* a, uint64_t n, uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) { uint64_t mid = lo + (hi - lo) / 2; if (a[mid] < key) lo = mid + 1; else hi = mid; }
  return lo;
}

/* u64 mode: V = ids that appear in the edge list.  ids_out receives the
 * sorted distinct ids (capacity 2m), labels_out[i] the label (an id) of ids_out[i].
 * Returns the number of distinct ids.  The id->index map is order preserving, so the
 * minimum index of a set is the index of its minimum id. */
int64_t oracle_uf_labels_u64(const uint64_t* edges, uint64_t m, uint64_t* ids_out,
                             uint64_t* labels_out) {
  uint64_t k = 2 * m;
  memcpy(ids_out, edges, sizeof(uint64_t) * k);
  qsort(ids_out, k, sizeof(uint64_t), cmp_u64);
  uint64_t nv = 0;
  for (uint64_t i = 0; i < k; i++)
    if (nv == 0 || ids_out[nv - 1] != ids_out[i]) ids_out[nv++] = ids_out[i];
  if (nv >= 0xffffffffULL) return -1;
  uint32_t* parent = (uint32_t*)malloc(sizeof(uint32_t) * (nv ? nv : 1));
  for (uint64_t v = 0; v < nv; v++) parent[v] = (uint32_t)v;
  for (uint64_t e = 0; e < m; e++) {
    uint32_t a = (uint32_t)lower_bound(ids_out, nv, edges[2 * e]);
    uint32_t b = (uint32_t)lower_bound(ids_out, nv, edges[2 * e + 1]);
    uint32_t ra = find32(parent, a), rb = find32(parent, b);
    if (ra != rb) {
      if (ra < rb) parent[rb] = ra; else parent[ra] = rb;
    }
  }
  for (uint64_t v = 0; v < nv; v++) labels_out[v] = ids_out[find32(parent, (uint32_t)v)];
  free(parent);
  return (int64_t)nv;
}
