/*
 * graphgen/gen.c -- seeded synthetic graph generators (inputs only).
 *
 * This module holds NO arithmetic of the connected-components method: it only
 * draws edge lists.  It is the one piece of code shared by the oracle side
 * (oracle/, tests/) and the CUDA side (bench.py, GPU tests), as DESIGN.md §3
 * allows.  Every draw is a pure function R(seed, stream, index) of a
 * counter-based splitmix64 mix, so a graph is fully determined by its
 * parameters and seed, independent of thread count.
 *
 * Workloads (BASELINE.json configs; SURVEY.md §8(d) "Synthetic inputs"; the
 * paper's datasets tab:data PAPER.md:286-304 are not available, these stand in):
 *   gg_blocks : C1 forest-of-blocks        (stand-in for many-small-component M3/M4)
 *   gg_paths  : C2 de Bruijn-like paths    (stand-in for metagenomic M1/M2)
 *   gg_grid   : C3 thinned 2-D lattice     (stand-in for road network G3)
 *   gg_rmat   : C4 R-MAT / Kronecker       (stand-in for K1/K2, G1/G2)
 *   gg_er     : Erdos-Renyi (tests only)
 * Vertex ids are scrambled by a seeded Feistel bijection on [0,n) (cycle
 * walking), and edge order by a second bijection on [0,m).
 *
 * Output format everywhere: interleaved uint32 pairs (u0,v0,u1,v1,...).
 * Two-phase API where the edge count is data dependent: call with out==NULL
 * to get the counts, then again with a buffer of 2*m uint32.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

static inline uint64_t gg_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* counter-based generator: R(seed, stream, i) */
uint64_t gg_rand(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t k = gg_mix(seed ^ gg_mix(stream * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL));
  return gg_mix(k + (i + 1) * 0x9E3779B97F4A7C15ULL);
}

/* ---- seeded bijection on [0, n): balanced Feistel + cycle walking ---- */
typedef struct { uint64_t n; uint32_t h; uint64_t mask; uint64_t key[4]; } gg_perm;

static void perm_init(gg_perm* p, uint64_t n, uint64_t seed, uint64_t stream) {
  uint32_t w = 2;
  while (w < 64 && (1ULL << w) < n) w++;
  if (w & 1) w++;
  p->n = n; p->h = w / 2; p->mask = (p->h >= 64) ? ~0ULL : ((1ULL << p->h) - 1);
  for (int i = 0; i < 4; i++) p->key[i] = gg_rand(seed, stream, (uint64_t)i);
}
static inline uint64_t perm_round(const gg_perm* p, uint64_t x) {
  uint64_t l = x >> p->h, r = x & p->mask;
  for (int i = 0; i < 4; i++) {
    uint64_t f = gg_mix(r ^ p->key[i]) & p->mask;
    uint64_t nl = r, nr = l ^ f;
    l = nl; r = nr;
  }
  return (l << p->h) | r;
}
static inline uint64_t perm_apply(const gg_perm* p, uint64_t x) {
  if (p->n <= 1) return x;
  do { x = perm_round(p, x); } while (x >= p->n);
  return x;
}

uint64_t gg_perm_value(uint64_t n, uint64_t seed, uint64_t stream, uint64_t x) {
  gg_perm p; perm_init(&p, n, seed, stream); return perm_apply(&p, x);
}

/* relabel all endpoints by the id bijection, then permute edge order */
static void finish(uint32_t* out, uint64_t m, uint64_t n, uint64_t seed, int permute_ids,
                   int permute_order) {
  if (permute_ids) {
    gg_perm p; perm_init(&p, n, seed, 1001);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)(2 * m); i++) out[i] = (uint32_t)perm_apply(&p, out[i]);
  }
  if (permute_order && m > 1) {
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * 2 * m);
    gg_perm p; perm_init(&p, m, seed, 1002);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)m; e++) {
      uint64_t s = perm_apply(&p, (uint64_t)e);
      tmp[2 * e] = out[2 * s]; tmp[2 * e + 1] = out[2 * s + 1];
    }
    memcpy(out, tmp, sizeof(uint32_t) * 2 * m);
    free(tmp);
  }
}

/* C1: n vertices in n/block equal blocks; each edge picks a block uniformly and two
 * endpoints uniformly inside it (self-loops kept). */
int gg_blocks(uint64_t seed, uint64_t n, uint64_t m, uint64_t block, uint32_t* out) {
  if (block == 0 || n % block) return -1;
  uint64_t nb = n / block;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < (int64_t)m; e++) {
    uint64_t b = gg_rand(seed, 1, e) % nb;
    uint64_t r = gg_rand(seed, 2, e);
    out[2 * e] = (uint32_t)(b * block + (r & 0xffffffffULL) % block);
    out[2 * e + 1] = (uint32_t)(b * block + (r >> 32) % block);
  }
  finish(out, m, n, seed, 1, 1);
  return 0;
}

/* Erdos-Renyi-like multigraph: m uniform pairs (tests). */
int gg_er(uint64_t seed, uint64_t n, uint64_t m, uint32_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < (int64_t)m; e++) {
    out[2 * e] = (uint32_t)(gg_rand(seed, 3, e) % n);
    out[2 * e + 1] = (uint32_t)(gg_rand(seed, 4, e) % n);
  }
  return 0;
}

/* C2: n_paths simple paths, lengths 1+Geometric(1/mean) vertices; bubbles (s, s+d),
 * d in [2,8] inside a path (bubble_ppm per million path edges; dropped when they run
 * past the path end); joins between uniform vertices (join_ppm per million path edges).
 * counts[0]=n, counts[1]=m. */
int gg_paths(uint64_t seed, uint64_t n_paths, double mean_len, uint64_t bubble_ppm,
             uint64_t join_ppm, uint64_t* counts, uint32_t* out) {
  uint64_t* start = (uint64_t*)malloc(sizeof(uint64_t) * (n_paths + 1));
  double q = 1.0 - 1.0 / mean_len;
  uint64_t n = 0;
  for (uint64_t k = 0; k < n_paths; k++) {
    double u = ((gg_rand(seed, 10, k) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    uint64_t L = 1 + (uint64_t)floor(log(u) / log(q));
    start[k] = n; n += L;
  }
  start[n_paths] = n;
  uint64_t n_path_edges = n - n_paths;
  uint64_t nb = n_path_edges * bubble_ppm / 1000000ULL;
  uint64_t nj = n_path_edges * join_ppm / 1000000ULL;
  /* bubbles: draw a vertex s uniformly, keep iff s+d stays inside its path */
  uint8_t* keep = (uint8_t*)malloc(nb ? nb : 1);
  uint64_t* bs = (uint64_t*)malloc(sizeof(uint64_t) * (nb ? nb : 1));
  uint32_t* bd = (uint32_t*)malloc(sizeof(uint32_t) * (nb ? nb : 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)nb; i++) {
    uint64_t s = gg_rand(seed, 11, i) % n;
    uint32_t d = 2 + (uint32_t)(gg_rand(seed, 12, i) % 7);
    /* path of s: binary search */
    uint64_t lo = 0, hi = n_paths;
    while (hi - lo > 1) { uint64_t mid = (lo + hi) / 2; if (start[mid] <= s) lo = mid; else hi = mid; }
    keep[i] = (s + d < start[lo + 1]);
    bs[i] = s; bd[i] = d;
  }
  uint64_t nbk = 0;
  for (uint64_t i = 0; i < nb; i++) nbk += keep[i];
  uint64_t m = n_path_edges + nbk + nj;
  counts[0] = n; counts[1] = m;
  if (out) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t k = 0; k < (int64_t)n_paths; k++) {
      uint64_t s = start[k], e = start[k + 1];
      uint64_t pos = s - (uint64_t)k; /* edges before path k */
      for (uint64_t v = s; v + 1 < e; v++, pos++) { out[2 * pos] = (uint32_t)v; out[2 * pos + 1] = (uint32_t)(v + 1); }
    }
    uint64_t pos = n_path_edges;
    for (uint64_t i = 0; i < nb; i++)
      if (keep[i]) { out[2 * pos] = (uint32_t)bs[i]; out[2 * pos + 1] = (uint32_t)(bs[i] + bd[i]); pos++; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)nj; i++) {
      out[2 * (pos + i)] = (uint32_t)(gg_rand(seed, 13, i) % n);
      out[2 * (pos + i) + 1] = (uint32_t)(gg_rand(seed, 14, i) % n);
    }
    finish(out, m, n, seed, 1, 1);
  }
  free(start); free(keep); free(bs); free(bd);
  return 0;
}

/* C3: side x side lattice, right/down edges kept with probability keep32/2^32, plus
 * n_diag diagonals at uniform cells (x,y <= side-2) with a random orientation.
 * counts[0]=n, counts[1]=m. */
int gg_grid(uint64_t seed, uint64_t side, uint32_t keep32, uint64_t n_diag, uint64_t* counts,
            uint32_t* out) {
  uint64_t n = side * side;
  uint64_t nlat = 2 * side * (side - 1); /* right edges then down edges */
  /* count kept edges per row for positions */
  uint64_t* rowcnt = (uint64_t*)calloc(side + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(static)
  for (int64_t y = 0; y < (int64_t)side; y++) {
    uint64_t c = 0;
    for (uint64_t x = 0; x + 1 < side; x++) c += ((uint32_t)gg_rand(seed, 20, y * side + x) < keep32);
    if ((uint64_t)y + 1 < side)
      for (uint64_t x = 0; x < side; x++) c += ((uint32_t)gg_rand(seed, 21, y * side + x) < keep32);
    rowcnt[y + 1] = c;
  }
  for (uint64_t y = 0; y < side; y++) rowcnt[y + 1] += rowcnt[y];
  uint64_t nkept = rowcnt[side];
  uint64_t m = nkept + n_diag;
  counts[0] = n; counts[1] = m;
  (void)nlat;
  if (out) {
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < (int64_t)side; y++) {
      uint64_t pos = rowcnt[y];
      for (uint64_t x = 0; x + 1 < side; x++)
        if ((uint32_t)gg_rand(seed, 20, y * side + x) < keep32) {
          out[2 * pos] = (uint32_t)(y * side + x); out[2 * pos + 1] = (uint32_t)(y * side + x + 1); pos++;
        }
      if ((uint64_t)y + 1 < side)
        for (uint64_t x = 0; x < side; x++)
          if ((uint32_t)gg_rand(seed, 21, y * side + x) < keep32) {
            out[2 * pos] = (uint32_t)(y * side + x); out[2 * pos + 1] = (uint32_t)((y + 1) * side + x); pos++;
          }
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n_diag; i++) {
      uint64_t r = gg_rand(seed, 22, i);
      uint64_t x = (r & 0xffffffffULL) % (side - 1), y = ((r >> 32) & 0x7fffffffULL) % (side - 1);
      int orient = (int)(r >> 63);
      uint64_t a = orient ? (y * side + x + 1) : (y * side + x);
      uint64_t b = orient ? ((y + 1) * side + x) : ((y + 1) * side + x + 1);
      out[2 * (nkept + i)] = (uint32_t)a; out[2 * (nkept + i) + 1] = (uint32_t)b;
    }
    finish(out, m, n, seed, 1, 1);
  }
  free(rowcnt);
  return 0;
}

/* C4: R-MAT scale s, m edges; per level a 32-bit draw picks a quadrant with integer
 * thresholds ta < tab < tabc (a, a+b, a+b+c scaled by 2^32). Ids then permuted on
 * [0, 2^s). Duplicates and self-loops kept. */
int gg_rmat(uint64_t seed, uint32_t scale, uint64_t m, uint32_t ta, uint32_t tab, uint32_t tabc,
            int permute_ids, uint32_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < (int64_t)m; e++) {
    uint64_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; l += 2) {
      uint64_t r = gg_rand(seed, 30, (uint64_t)e * 32 + l / 2);
      for (int h = 0; h < 2 && l + h < scale; h++) {
        uint32_t x = (uint32_t)(h ? (r >> 32) : r);
        uint32_t ub = (x >= tab), vb = (x >= ta && x < tab) || (x >= tabc);
        u = (u << 1) | ub; v = (v << 1) | vb;
      }
    }
    out[2 * e] = (uint32_t)u; out[2 * e + 1] = (uint32_t)v;
  }
  finish(out, m, 1ULL << scale, seed, permute_ids, 0);
  return 0;
}

int gg_num_threads(void) { return omp_get_max_threads(); }

/* ---- C5: union of an R-MAT part and a path part on disjoint dense indices, relabelled to
 * u64 ids by a 64-bit bijective integer mix (Thomas Wang / Jenkins style 7-step hash; the
 * id space of the configs' "u64 ids"), edge order scrambled by a seeded bijection.
 * in:  a (ma pairs, indices < na) and b (mb pairs, indices < nb, offset by na)
 * out: 2*(ma+mb) uint64 ids.                                                              */
static inline uint64_t gg_mix64(uint64_t k) {
  k = (~k) + (k << 21);
  k = k ^ (k >> 24);
  k = (k + (k << 3)) + (k << 8);
  k = k ^ (k >> 14);
  k = (k + (k << 2)) + (k << 4);
  k = k ^ (k >> 28);
  k = k + (k << 31);
  return k;
}
uint64_t gg_mix64_value(uint64_t k) { return gg_mix64(k); }
int gg_union_u64(uint64_t seed, const uint32_t* a, uint64_t ma, uint64_t na, const uint32_t* b,
                 uint64_t mb, uint64_t* out) {
  const uint64_t m = ma + mb;
  gg_perm pe;
  perm_init(&pe, m ? m : 1, seed, 9);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)m; i++) {
    uint64_t j = perm_apply(&pe, (uint64_t)i);
    uint64_t u, v;
    if (j < ma) { u = a[2 * j]; v = a[2 * j + 1]; }
    else { j -= ma; u = na + b[2 * j]; v = na + b[2 * j + 1]; }
    out[2 * i] = gg_mix64(u);
    out[2 * i + 1] = gg_mix64(v);
  }
  return 0;
}

/* C5, one rank's block of the output: edge records [i0, i1) of gg_union_u64's list over the
 * R-MAT part (scale `scale`, ma edges, thresholds as gg_rmat, ids permuted) and the path part
 * b (mb pairs) -- R-MAT edges are drawn on the fly (each is a pure function of (seed, j)),
 * so a rank never holds the other ranks' R-MAT edges.  Identical to the same rows of
 * gg_union_u64(seed, rmat(...), 2^scale, b).                                              */
int gg_c5_block(uint64_t seed, uint64_t rseed, uint32_t scale, uint64_t ma, uint32_t ta, uint32_t tab,
                uint32_t tabc, const uint32_t* b, uint64_t mb, uint64_t i0, uint64_t i1, uint64_t* out) {
  const uint64_t m = ma + mb, na = 1ULL << scale;
  gg_perm pe, pid;
  perm_init(&pe, m ? m : 1, seed, 9);
  perm_init(&pid, na, rseed, 1001);
#pragma omp parallel for schedule(static)
  for (int64_t i = (int64_t)i0; i < (int64_t)i1; i++) {
    uint64_t j = perm_apply(&pe, (uint64_t)i);
    uint64_t u = 0, v = 0;
    if (j < ma) {
      for (uint32_t l = 0; l < scale; l += 2) {
        uint64_t r = gg_rand(rseed, 30, j * 32 + l / 2);
        for (int h = 0; h < 2 && l + h < scale; h++) {
          uint32_t x = (uint32_t)(h ? (r >> 32) : r);
          uint32_t ub = (x >= tab), vb = (x >= ta && x < tab) || (x >= tabc);
          u = (u << 1) | ub; v = (v << 1) | vb;
        }
      }
      u = perm_apply(&pid, u);
      v = perm_apply(&pid, v);
    } else {
      j -= ma;
      u = na + b[2 * j];
      v = na + b[2 * j + 1];
    }
    out[2 * (i - i0)] = gg_mix64(u);
    out[2 * (i - i0) + 1] = gg_mix64(v);
  }
  return 0;
}
