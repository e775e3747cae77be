/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product or a fallback.
 *
 * Plain-C restatement of the reference (rowgcn, /root/reference/proj) algorithm for the MG-GCN
 * full-batch training step, used by tests/ to check the CUDA path and pinned against the compiled
 * reference (oracle/_ref) and the golden fixtures in tests/golden/ (tests/test_oracle.py).
 * Every function cites the reference lines it restates ("inc/" = proj/include/rowgcn/).
 *
 * Built twice by oracle/build_oracle.sh: OR_S=float (liboracle_f32.so) and OR_S=double
 * (liboracle_f64.so), with -O2 -ffp-contract=off so `out += a*b` stays a separate multiply and add,
 * exactly like the reference's canonical build (0 FMA instructions).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef OR_S
#define OR_S float
#endif
typedef OR_S S;
typedef int64_t idx_t; /* inc/dense.hpp:18 index_t = int64 */

#define OR_CAT2(a, b) a##b
#define OR_CAT(a, b) OR_CAT2(a, b)
#ifdef OR_F64
#define FN(name) OR_CAT(name, _f64)
#else
#define FN(name) OR_CAT(name, _f32)
#endif

/* ------------------------------------------------------------------ mt19937_64 + Rng
 * inc/rng.hpp:13-28: std::mt19937_64 (standard-mandated sequence), below(n) = gen() % n,
 * uniform() = (gen() >> 11) * 2^-53, uniform(lo, hi) = lo + (hi - lo) * uniform(). */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_rng;

static void rng_seed(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t rng_next(or_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

static uint64_t rng_below(or_rng* r, uint64_t n) { return rng_next(r) % n; }
static double rng_uniform(or_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform_ab(or_rng* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }

uint64_t FN(or_rng_first)(uint64_t seed, int32_t count, uint64_t* out) {
  or_rng r;
  rng_seed(&r, seed);
  for (int i = 0; i < count; ++i) out[i] = rng_next(&r);
  return count > 0 ? out[0] : 0;
}

/* ------------------------------------------------------------------ partitioner */

/* inc/partition.hpp:69-79: Fisher-Yates over inverse (i = n-1..1, j = below(i+1)), then
 * forward[inverse[i]] = i. */
void FN(or_random_permutation)(idx_t n, uint64_t seed, idx_t* forward, idx_t* inverse) {
  or_rng r;
  rng_seed(&r, seed);
  for (idx_t i = 0; i < n; ++i) inverse[i] = i;
  for (idx_t i = n - 1; i > 0; --i) {
    const idx_t j = (idx_t)rng_below(&r, (uint64_t)i + 1);
    const idx_t t = inverse[i];
    inverse[i] = inverse[j];
    inverse[j] = t;
  }
  for (idx_t i = 0; i < n; ++i) forward[inverse[i]] = i;
}

/* inc/partition.hpp:42-49: bounds[i] = i * n / P (int64 floor). */
void FN(or_uniform_partition)(idx_t n, int32_t parts, idx_t* bounds) {
  for (int i = 0; i <= parts; ++i) bounds[i] = (idx_t)i * n / parts;
}

/* inc/partition.hpp:35-38 part_of: upper_bound(bounds, v) - 1 (empty parts skipped). */
static int part_of(const idx_t* bounds, int parts, idx_t v) {
  int lo = 0, hi = parts + 1; /* first index with bounds[k] > v */
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (bounds[mid] > v) hi = mid; else lo = mid + 1;
  }
  return lo - 1;
}

typedef struct {
  idx_t rows, cols;
  idx_t* row_ptr;
  idx_t* col_idx;
  S* values;
} or_csr;

static void csr_alloc(or_csr* m, idx_t rows, idx_t cols, idx_t nnz) {
  m->rows = rows;
  m->cols = cols;
  m->row_ptr = (idx_t*)calloc((size_t)rows + 1, sizeof(idx_t));
  m->col_idx = (idx_t*)malloc(sizeof(idx_t) * (size_t)(nnz > 0 ? nnz : 1));
  m->values = (S*)malloc(sizeof(S) * (size_t)(nnz > 0 ? nnz : 1));
}
static void csr_free(or_csr* m) {
  free(m->row_ptr);
  free(m->col_idx);
  free(m->values);
  memset(m, 0, sizeof(*m));
}

/* Sort (col, val) pairs of one row by column: insertion sort over small rows, heap-free
 * shell sort otherwise. Rows of a valid CSR are duplicate-free, so a plain key sort reproduces
 * from_coo's (src, dst) ordering (inc/sparse.hpp:59-90). */
static void sort_row(idx_t* c, S* v, idx_t len) {
  for (idx_t gap = len / 2; gap > 0; gap = gap == 2 ? 1 : (idx_t)(gap / 2.2)) {
    for (idx_t i = gap; i < len; ++i) {
      const idx_t kc = c[i];
      const S kv = v[i];
      idx_t j = i;
      while (j >= gap && c[j - gap] > kc) {
        c[j] = c[j - gap];
        v[j] = v[j - gap];
        j -= gap;
      }
      c[j] = kc;
      v[j] = kv;
    }
    if (gap == 1) break;
  }
}

/* inc/partition.hpp:101-116 permute_graph: a'(pi(u), pi(v)) = a(u, v), rebuilt through from_coo
 * (sorted by (src, dst)); counting sort by new row then per-row column sort gives the same CSR. */
static void permute_graph(const or_csr* a, const idx_t* fwd, or_csr* out) {
  const idx_t n = a->rows, nnz = a->row_ptr[n];
  csr_alloc(out, n, n, nnz);
  for (idx_t u = 0; u < n; ++u) out->row_ptr[fwd[u] + 1] = a->row_ptr[u + 1] - a->row_ptr[u];
  for (idx_t u = 0; u < n; ++u) out->row_ptr[u + 1] += out->row_ptr[u];
  for (idx_t u = 0; u < n; ++u) {
    idx_t pos = out->row_ptr[fwd[u]];
    for (idx_t e = a->row_ptr[u]; e < a->row_ptr[u + 1]; ++e, ++pos) {
      out->col_idx[pos] = fwd[a->col_idx[e]];
      out->values[pos] = a->values[e];
    }
  }
  for (idx_t u = 0; u < n; ++u)
    sort_row(out->col_idx + out->row_ptr[u], out->values + out->row_ptr[u], out->row_ptr[u + 1] - out->row_ptr[u]);
}

/* inc/sparse.hpp:94-107 normalize_in_degree: column sums accumulated in CSR edge order, then
 * value / sum (zero-in-degree columns stay 0). In place. */
static void normalize_in_degree(or_csr* a) {
  const idx_t nnz = a->row_ptr[a->rows];
  S* col_sum = (S*)calloc((size_t)a->cols, sizeof(S));
  for (idx_t e = 0; e < nnz; ++e) col_sum[a->col_idx[e]] += a->values[e];
  for (idx_t e = 0; e < nnz; ++e) {
    const S s = col_sum[a->col_idx[e]];
    a->values[e] = s != (S)0 ? a->values[e] / s : (S)0;
  }
  free(col_sum);
}

/* inc/sparse.hpp:110-129 transpose: stable counting sort over target rows. */
static void transpose(const or_csr* a, or_csr* t) {
  const idx_t nnz = a->row_ptr[a->rows];
  csr_alloc(t, a->cols, a->rows, nnz);
  for (idx_t e = 0; e < nnz; ++e) t->row_ptr[a->col_idx[e] + 1]++;
  for (idx_t v = 0; v < t->rows; ++v) t->row_ptr[v + 1] += t->row_ptr[v];
  idx_t* fill = (idx_t*)malloc(sizeof(idx_t) * (size_t)(t->rows > 0 ? t->rows : 1));
  memcpy(fill, t->row_ptr, sizeof(idx_t) * (size_t)t->rows);
  for (idx_t u = 0; u < a->rows; ++u)
    for (idx_t e = a->row_ptr[u]; e < a->row_ptr[u + 1]; ++e) {
      const idx_t pos = fill[a->col_idx[e]]++;
      t->col_idx[pos] = u;
      t->values[pos] = a->values[e];
    }
  free(fill);
}

/* inc/partition.hpp:173-225 tile_rows: tiles[i][j] = rows of part i, columns of part j, local
 * column index v - begin(j), column order kept. tiles is an array of parts*parts CSRs. */
static void tile_rows(const or_csr* a, const idx_t* bounds, int parts, or_csr* tiles) {
  for (int i = 0; i < parts; ++i) {
    const idx_t r0 = bounds[i], r1 = bounds[i + 1];
    for (int j = 0; j < parts; ++j) {
      or_csr* t = &tiles[i * parts + j];
      idx_t cnt = 0;
      for (idx_t u = r0; u < r1; ++u)
        for (idx_t e = a->row_ptr[u]; e < a->row_ptr[u + 1]; ++e)
          if (a->col_idx[e] >= bounds[j] && a->col_idx[e] < bounds[j + 1]) ++cnt;
      csr_alloc(t, r1 - r0, bounds[j + 1] - bounds[j], cnt);
      idx_t pos = 0;
      for (idx_t u = r0; u < r1; ++u) {
        for (idx_t e = a->row_ptr[u]; e < a->row_ptr[u + 1]; ++e) {
          const idx_t v = a->col_idx[e];
          if (part_of(bounds, parts, v) != j) continue;
          t->col_idx[pos] = v - bounds[j];
          t->values[pos] = a->values[e];
          ++pos;
        }
        t->row_ptr[u - r0 + 1] = pos;
      }
    }
  }
}

/* ------------------------------------------------------------------ synthetic generator
 * inc/dataset.hpp:287-334 synth_graph: weights (u+1)^-exponent, stochastic rounding of
 * stubs_total * w / wsum, uniform endpoints (self loops dropped), symmetrised, sorted + dedup,
 * unit values; then features U(-1,1) and labels below(classes) from the same stream. The pair list
 * is bucketed by source and each bucket sorted + deduplicated, which equals sort + unique. */
typedef struct {
  idx_t n, d0;
  or_csr graph;
  S* features;
  int32_t* labels;
} or_dataset;


static int cmp_idx(const void* a, const void* b) {
  const idx_t x = *(const idx_t*)a, y = *(const idx_t*)b;
  return x < y ? -1 : x > y;
}

static or_dataset* ds_alloc(idx_t n, idx_t d0) {
  or_dataset* ds = (or_dataset*)calloc(1, sizeof(or_dataset));
  ds->n = n;
  ds->d0 = d0;
  ds->features = (S*)calloc((size_t)(n * d0 > 0 ? n * d0 : 1), sizeof(S));
  ds->labels = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  return ds;
}

/* ------------------------------------------------------------------ synthetic generator
 * inc/dataset.hpp:287-334 synth_graph: weights (u+1)^-exponent, stochastic rounding of
 * stubs_total * w / wsum, uniform endpoints (self loops dropped), symmetrised, sorted + dedup,
 * unit values; then features U(-1,1) and labels below(classes) from the same stream. The pair list
 * is bucketed by source and each bucket sorted + deduplicated, which equals sort + unique. */
void* FN(or_synth_graph)(idx_t n, double avg_degree, double exponent, uint64_t seed, idx_t feature_dim,
                         int32_t classes) {
  if (n < 2 || avg_degree < 1.0 || avg_degree >= (double)(n - 1)) return NULL;
  or_rng r;
  rng_seed(&r, seed);
  double* weight = (double*)malloc(sizeof(double) * (size_t)n);
  double wsum = 0;
  for (idx_t u = 0; u < n; ++u) {
    weight[u] = pow((double)(u + 1), -exponent);
    wsum += weight[u];
  }
  const double stubs_total = avg_degree * (double)n / 2.0;
  size_t cap = (size_t)(stubs_total * 1.2) + 16, cnt = 0;
  idx_t* su = (idx_t*)malloc(sizeof(idx_t) * cap);
  idx_t* sv = (idx_t*)malloc(sizeof(idx_t) * cap);
  for (idx_t u = 0; u < n; ++u) {
    const double exact = stubs_total * weight[u] / wsum;
    idx_t k = (idx_t)exact;
    if (rng_uniform(&r) < exact - (double)k) ++k;
    if (k > n - 1) k = n - 1;
    for (idx_t t = 0; t < k; ++t) {
      const idx_t v = (idx_t)rng_below(&r, (uint64_t)n);
      if (v == u) continue;
      if (cnt == cap) {
        cap *= 2;
        su = (idx_t*)realloc(su, sizeof(idx_t) * cap);
        sv = (idx_t*)realloc(sv, sizeof(idx_t) * cap);
      }
      su[cnt] = u;
      sv[cnt] = v;
      ++cnt;
    }
  }
  free(weight);
  idx_t* start = (idx_t*)calloc((size_t)n + 1, sizeof(idx_t));
  for (size_t i = 0; i < cnt; ++i) {
    start[su[i] + 1]++;
    start[sv[i] + 1]++;
  }
  for (idx_t u = 0; u < n; ++u) start[u + 1] += start[u];
  idx_t* adj = (idx_t*)malloc(sizeof(idx_t) * (size_t)(start[n] > 0 ? start[n] : 1));
  idx_t* fill = (idx_t*)malloc(sizeof(idx_t) * (size_t)n);
  memcpy(fill, start, sizeof(idx_t) * (size_t)n);
  for (size_t i = 0; i < cnt; ++i) {
    adj[fill[su[i]]++] = sv[i];
    adj[fill[sv[i]]++] = su[i];
  }
  free(su);
  free(sv);
  idx_t* uniq = fill; /* reuse: unique count per row */
  idx_t total = 0;
  for (idx_t u = 0; u < n; ++u) {
    idx_t* row = adj + start[u];
    const idx_t len = start[u + 1] - start[u];
    qsort(row, (size_t)len, sizeof(idx_t), cmp_idx);
    idx_t w = 0;
    for (idx_t i = 0; i < len; ++i)
      if (w == 0 || row[i] != row[w - 1]) row[w++] = row[i];
    uniq[u] = w;
    total += w;
  }
  or_dataset* ds = ds_alloc(n, feature_dim);
  csr_alloc(&ds->graph, n, n, total);
  idx_t pos = 0;
  for (idx_t u = 0; u < n; ++u) {
    for (idx_t i = 0; i < uniq[u]; ++i, ++pos) {
      ds->graph.col_idx[pos] = adj[start[u] + i];
      ds->graph.values[pos] = (S)1;
    }
    ds->graph.row_ptr[u + 1] = pos;
  }
  free(adj);
  free(start);
  free(fill);
  for (idx_t i = 0; i < n * feature_dim; ++i) ds->features[i] = (S)rng_uniform_ab(&r, -1.0, 1.0);
  for (idx_t i = 0; i < n; ++i) ds->labels[i] = (int32_t)rng_below(&r, (uint64_t)classes);
  return ds;
}

void* FN(or_ds_from_arrays)(idx_t n, const idx_t* rp, const idx_t* ci, const S* v, idx_t d0, const S* feats,
                            const int32_t* labels) {
  or_dataset* ds = ds_alloc(n, d0);
  csr_alloc(&ds->graph, n, n, rp[n]);
  memcpy(ds->graph.row_ptr, rp, sizeof(idx_t) * (size_t)(n + 1));
  memcpy(ds->graph.col_idx, ci, sizeof(idx_t) * (size_t)rp[n]);
  memcpy(ds->graph.values, v, sizeof(S) * (size_t)rp[n]);
  memcpy(ds->features, feats, sizeof(S) * (size_t)(n * d0));
  memcpy(ds->labels, labels, sizeof(int32_t) * (size_t)n);
  return ds;
}

void FN(or_ds_info)(void* h, idx_t* n, idx_t* nnz, idx_t* d0) {
  const or_dataset* ds = (const or_dataset*)h;
  *n = ds->n;
  *nnz = ds->graph.row_ptr[ds->n];
  *d0 = ds->d0;
}

void FN(or_ds_export)(void* h, idx_t* rp, idx_t* ci, S* v, S* feats, int32_t* labels) {
  const or_dataset* ds = (const or_dataset*)h;
  const idx_t nnz = ds->graph.row_ptr[ds->n];
  if (rp) memcpy(rp, ds->graph.row_ptr, sizeof(idx_t) * (size_t)(ds->n + 1));
  if (ci) memcpy(ci, ds->graph.col_idx, sizeof(idx_t) * (size_t)nnz);
  if (v) memcpy(v, ds->graph.values, sizeof(S) * (size_t)nnz);
  if (feats) memcpy(feats, ds->features, sizeof(S) * (size_t)(ds->n * ds->d0));
  if (labels) memcpy(labels, ds->labels, sizeof(int32_t) * (size_t)ds->n);
}

void FN(or_ds_free)(void* h) {
  or_dataset* ds = (or_dataset*)h;
  if (!ds) return;
  csr_free(&ds->graph);
  free(ds->features);
  free(ds->labels);
  free(ds);
}

/* ------------------------------------------------------------------ prepare_data
 * inc/driver.hpp:87-117: permutation (seed = cfg.seed) of features/labels/mask, uniform
 * partition, permute_graph -> normalize_in_degree -> transpose; fwd tiles = tile_rows(A_hat^T),
 * bwd tiles = tile_rows(A_hat). The full A_hat / A_hat^T are kept for the model below (the staged
 * SpMM equals the monolithic one bitwise, inc/dist_spmm.hpp:55-56). */
typedef struct {
  idx_t n, d0, mask_count;
  int parts;
  idx_t* bounds;
  idx_t* perm_fwd;
  S* features;
  int32_t* labels;
  uint8_t* mask;
  or_csr ahat, ahat_t;
  or_csr* fwd_tiles; /* parts*parts */
  or_csr* bwd_tiles;
} or_prepared;

void* FN(or_prepare)(void* dsh, const uint8_t* train_mask, int32_t permute, uint64_t seed, int32_t workers) {
  const or_dataset* ds = (const or_dataset*)dsh;
  const idx_t n = ds->n, d0 = ds->d0;
  or_prepared* p = (or_prepared*)calloc(1, sizeof(or_prepared));
  p->n = n;
  p->d0 = d0;
  p->parts = workers;
  p->perm_fwd = (idx_t*)malloc(sizeof(idx_t) * (size_t)n);
  idx_t* inv = (idx_t*)malloc(sizeof(idx_t) * (size_t)n);
  if (permute) {
    FN(or_random_permutation)(n, seed, p->perm_fwd, inv);
  } else {
    for (idx_t i = 0; i < n; ++i) p->perm_fwd[i] = i;
  }
  free(inv);
  p->features = (S*)malloc(sizeof(S) * (size_t)(n * d0 > 0 ? n * d0 : 1));
  p->labels = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  p->mask = (uint8_t*)malloc((size_t)n);
  for (idx_t u = 0; u < n; ++u) { /* inc/partition.hpp:118-140 permute_rows / permute_values */
    const idx_t v = p->perm_fwd[u];
    memcpy(p->features + v * d0, ds->features + u * d0, sizeof(S) * (size_t)d0);
    p->labels[v] = ds->labels[u];
    p->mask[v] = train_mask ? train_mask[u] : 1; /* inc/dataset.hpp:46-49 effective_mask */
  }
  for (idx_t u = 0; u < n; ++u) p->mask_count += p->mask[u] ? 1 : 0;
  p->bounds = (idx_t*)malloc(sizeof(idx_t) * (size_t)(workers + 1));
  FN(or_uniform_partition)(n, workers, p->bounds);
  if (permute) {
    permute_graph(&ds->graph, p->perm_fwd, &p->ahat);
  } else {
    csr_alloc(&p->ahat, n, n, ds->graph.row_ptr[n]);
    memcpy(p->ahat.row_ptr, ds->graph.row_ptr, sizeof(idx_t) * (size_t)(n + 1));
    memcpy(p->ahat.col_idx, ds->graph.col_idx, sizeof(idx_t) * (size_t)ds->graph.row_ptr[n]);
    memcpy(p->ahat.values, ds->graph.values, sizeof(S) * (size_t)ds->graph.row_ptr[n]);
  }
  normalize_in_degree(&p->ahat);
  transpose(&p->ahat, &p->ahat_t);
  p->fwd_tiles = (or_csr*)calloc((size_t)(workers * workers), sizeof(or_csr));
  p->bwd_tiles = (or_csr*)calloc((size_t)(workers * workers), sizeof(or_csr));
  tile_rows(&p->ahat_t, p->bounds, workers, p->fwd_tiles);
  tile_rows(&p->ahat, p->bounds, workers, p->bwd_tiles);
  return p;
}

void FN(or_prep_info)(void* h, idx_t* mask_count, idx_t* bounds) {
  const or_prepared* p = (const or_prepared*)h;
  *mask_count = p->mask_count;
  memcpy(bounds, p->bounds, sizeof(idx_t) * (size_t)(p->parts + 1));
}

void FN(or_prep_tile_info)(void* h, int32_t dir, int32_t i, int32_t j, idx_t* rows, idx_t* cols, idx_t* nnz) {
  const or_prepared* p = (const or_prepared*)h;
  const or_csr* t = &(dir == 0 ? p->fwd_tiles : p->bwd_tiles)[i * p->parts + j];
  *rows = t->rows;
  *cols = t->cols;
  *nnz = t->row_ptr[t->rows];
}

void FN(or_prep_tile_export)(void* h, int32_t dir, int32_t i, int32_t j, idx_t* rp, idx_t* ci, S* v) {
  const or_prepared* p = (const or_prepared*)h;
  const or_csr* t = &(dir == 0 ? p->fwd_tiles : p->bwd_tiles)[i * p->parts + j];
  memcpy(rp, t->row_ptr, sizeof(idx_t) * (size_t)(t->rows + 1));
  memcpy(ci, t->col_idx, sizeof(idx_t) * (size_t)t->row_ptr[t->rows]);
  memcpy(v, t->values, sizeof(S) * (size_t)t->row_ptr[t->rows]);
}

void FN(or_prep_rows_export)(void* h, S* feats, int32_t* labels, uint8_t* mask, idx_t* perm_fwd) {
  const or_prepared* p = (const or_prepared*)h;
  if (feats) memcpy(feats, p->features, sizeof(S) * (size_t)(p->n * p->d0));
  if (labels) memcpy(labels, p->labels, sizeof(int32_t) * (size_t)p->n);
  if (mask) memcpy(mask, p->mask, (size_t)p->n);
  if (perm_fwd) memcpy(perm_fwd, p->perm_fwd, sizeof(idx_t) * (size_t)p->n);
}

void FN(or_prep_free)(void* h) {
  or_prepared* p = (or_prepared*)h;
  if (!p) return;
  for (int k = 0; k < p->parts * p->parts; ++k) {
    csr_free(&p->fwd_tiles[k]);
    csr_free(&p->bwd_tiles[k]);
  }
  free(p->fwd_tiles);
  free(p->bwd_tiles);
  csr_free(&p->ahat);
  csr_free(&p->ahat_t);
  free(p->bounds);
  free(p->perm_fwd);
  free(p->features);
  free(p->labels);
  free(p->mask);
  free(p);
}

/* ------------------------------------------------------------------ kernels */

#ifdef OR_F64
#define OR_EXP exp
#define OR_LOG log
#define OR_SQRT sqrt
#else
#define OR_EXP expf
#define OR_LOG logf
#define OR_SQRT sqrtf
#endif

/* inc/sparse.hpp:140-154 spmm_rows: out[u] = (acc ? out[u] : 0) + sum over row u in column order
 * of val * h[col] (separate multiply and add). */
static void spmm_core(idx_t rows, const idx_t* rp, const idx_t* ci, const S* v, const S* h, idx_t w, int acc, S* out) {
  for (idx_t u = 0; u < rows; ++u) {
    S* o = out + u * w;
    if (!acc)
      for (idx_t j = 0; j < w; ++j) o[j] = (S)0;
    for (idx_t e = rp[u]; e < rp[u + 1]; ++e) {
      const S val = v[e];
      const S* hr = h + ci[e] * w;
      for (idx_t j = 0; j < w; ++j) o[j] += val * hr[j];
    }
  }
}

int FN(or_spmm)(idx_t rows, idx_t cols, const idx_t* rp, const idx_t* ci, const S* v, const S* h, idx_t w,
                int32_t acc, S* out) {
  (void)cols;
  spmm_core(rows, rp, ci, v, h, w, acc, out);
  return 0;
}

/* inc/dense.hpp:140-204 gemm: out = (acc ? out : 0) + op(a) op(b); k ascending; NN and TN skip
 * zero a-entries (:165, :177); NT/TT form a row dot product then add it to out (:189-191). */
static void gemm_core(const S* a, idx_t ar, idx_t ac, const S* b, idx_t br, idx_t bc, int ta, int tb, int acc,
                      S* out) {
  const idx_t m = ta ? ac : ar, k = ta ? ar : ac, n = tb ? br : bc;
  (void)br;
  (void)bc;
  if (!acc)
    for (idx_t i = 0; i < m * n; ++i) out[i] = (S)0;
  if (!ta && !tb) {
    for (idx_t i = 0; i < m; ++i) {
      S* orow = out + i * n;
      const S* arow = a + i * k;
      for (idx_t p = 0; p < k; ++p) {
        const S aik = arow[p];
        if (aik == (S)0) continue;
        const S* brow = b + p * n;
        for (idx_t j = 0; j < n; ++j) orow[j] += aik * brow[j];
      }
    }
  } else if (ta && !tb) {
    for (idx_t p = 0; p < k; ++p) {
      const S* arow = a + p * m;
      const S* brow = b + p * n;
      for (idx_t i = 0; i < m; ++i) {
        const S api = arow[i];
        if (api == (S)0) continue;
        S* orow = out + i * n;
        for (idx_t j = 0; j < n; ++j) orow[j] += api * brow[j];
      }
    }
  } else if (!ta && tb) {
    for (idx_t i = 0; i < m; ++i) {
      const S* arow = a + i * k;
      S* orow = out + i * n;
      for (idx_t j = 0; j < n; ++j) {
        const S* brow = b + j * k;
        S s = 0;
        for (idx_t p = 0; p < k; ++p) s += arow[p] * brow[p];
        orow[j] += s;
      }
    }
  } else {
    for (idx_t i = 0; i < m; ++i)
      for (idx_t j = 0; j < n; ++j) {
        S s = 0;
        for (idx_t p = 0; p < k; ++p) s += a[p * m + i] * b[j * k + p];
        out[i * n + j] += s;
      }
  }
}

int FN(or_gemm)(const S* a, idx_t ar, idx_t ac, const S* b, idx_t br, idx_t bc, int32_t ta, int32_t tb,
                int32_t acc, S* out) {
  gemm_core(a, ar, ac, b, br, bc, ta, tb, acc, out);
  return 0;
}

/* inc/dense.hpp:241-277 softmax_xent_sum: masked rows get (softmax - onehot) / denom, unmasked rows
 * zero; returns the loss SUM in S arithmetic (serial). grad may alias logits. */
static S softmax_xent_core(const S* logits, idx_t rows, idx_t c, const int32_t* labels, const uint8_t* mask,
                           S* grad, idx_t denom) {
  const S inv_denom = (S)1 / (S)denom;
  S loss_sum = 0;
  for (idx_t v = 0; v < rows; ++v) {
    S* g = grad + v * c;
    if (!mask[v]) {
      for (idx_t j = 0; j < c; ++j) g[j] = (S)0;
      continue;
    }
    const int32_t label = labels[v];
    const S* row = logits + v * c;
    S row_max = row[0];
    for (idx_t j = 1; j < c; ++j) row_max = row_max < row[j] ? row[j] : row_max; /* std::max */
    S sum_exp = 0;
    for (idx_t j = 0; j < c; ++j) sum_exp += OR_EXP(row[j] - row_max);
    loss_sum += OR_LOG(sum_exp) - (row[label] - row_max);
    for (idx_t j = 0; j < c; ++j) g[j] = OR_EXP(row[j] - row_max) / sum_exp * inv_denom;
    g[label] -= inv_denom;
  }
  return loss_sum;
}

int FN(or_softmax_xent_sum)(const S* logits, idx_t rows, idx_t cols, const int32_t* labels, const uint8_t* mask,
                            S* grad, idx_t denom, double* loss_sum) {
  for (idx_t v = 0; v < rows; ++v)
    if (mask[v] && (labels[v] < 0 || labels[v] >= cols)) return 2; /* ValueError, inc/dense.hpp:263-265 */
  if (denom <= 0) return 2;
  *loss_sum = (double)softmax_xent_core(logits, rows, cols, labels, mask, grad, denom);
  return 0;
}

/* inc/gcn.hpp:61-85 adam_step: S-typed constants, bias corrections 1 - (S)pow(beta, t) in double,
 * grads zeroed afterwards. */
static void adam_core(S* w, S* g, S* m, S* v, idx_t size, int t, double lr_d, double b1_d, double b2_d,
                      double eps_d) {
  const S b1 = (S)b1_d, b2 = (S)b2_d, lr = (S)lr_d, eps = (S)eps_d;
  const S corr1 = (S)1 - (S)pow(b1_d, t);
  const S corr2 = (S)1 - (S)pow(b2_d, t);
  for (idx_t i = 0; i < size; ++i) {
    m[i] = b1 * m[i] + ((S)1 - b1) * g[i];
    v[i] = b2 * v[i] + ((S)1 - b2) * g[i] * g[i];
    const S mhat = m[i] / corr1;
    const S vhat = v[i] / corr2;
    w[i] -= lr * mhat / (OR_SQRT(vhat) + eps);
  }
  for (idx_t i = 0; i < size; ++i) g[i] = (S)0;
}

int FN(or_adam)(S* w, S* g, S* m, S* v, idx_t size, int32_t t, double lr, double b1, double b2, double eps) {
  if (t < 1) return 2;
  adam_core(w, g, m, v, size, t, lr, b1, b2, eps);
  return 0;
}

/* ------------------------------------------------------------------ model (GcnWorker, inc/gcn.hpp)
 * Global-row restatement of P workers: row-local ops (GeMM, ReLU, loss rows) are the concatenation
 * of the workers' local ops; the staged SpMM is the monolithic SpMM (bitwise, inc/dist_spmm.hpp:55);
 * the cross-worker reductions (loss stats, W-grad staging) are reproduced per worker and summed in
 * rank order exactly as DeviceGroup::all_reduce_sum (inc/collectives.hpp:76-94, no-op at P=1). */
typedef struct {
  const or_prepared* prep;
  int L;
  idx_t* dims;
  double lr, b1, b2, eps;
  int skip_first, order_swap;
  S** w;
  S** wg;
  S** m;
  S** v;
  S** ahw;  /* L buffers n x d_{l+1} */
  S* hw;    /* n x w_max */
  S* x;     /* permuted features */
  idx_t wblocks[9];
  double last_acc;
} or_model;

void* FN(or_model_create)(void* prep_h, const idx_t* dims, int32_t n_dims, double lr, double b1, double b2,
                          double eps, uint64_t seed, int32_t skip_first, int32_t order_swap) {
  const or_prepared* p = (const or_prepared*)prep_h;
  or_model* M = (or_model*)calloc(1, sizeof(or_model));
  M->prep = p;
  M->L = n_dims - 1;
  M->dims = (idx_t*)malloc(sizeof(idx_t) * (size_t)n_dims);
  memcpy(M->dims, dims, sizeof(idx_t) * (size_t)n_dims);
  M->lr = lr;
  M->b1 = b1;
  M->b2 = b2;
  M->eps = eps;
  M->skip_first = skip_first;
  M->order_swap = order_swap;
  const idx_t n = p->n;
  idx_t wmax = dims[0];
  for (int l = 1; l < n_dims; ++l) wmax = dims[l] > wmax ? dims[l] : wmax;
  M->w = (S**)calloc((size_t)M->L, sizeof(S*));
  M->wg = (S**)calloc((size_t)M->L, sizeof(S*));
  M->m = (S**)calloc((size_t)M->L, sizeof(S*));
  M->v = (S**)calloc((size_t)M->L, sizeof(S*));
  M->ahw = (S**)calloc((size_t)M->L, sizeof(S*));
  or_rng r; /* init_params, inc/gcn.hpp:163-173: one Rng(seed) across layers, Glorot uniform */
  rng_seed(&r, seed);
  for (int l = 0; l < M->L; ++l) {
    const idx_t sz = dims[l] * dims[l + 1];
    M->w[l] = (S*)calloc((size_t)sz, sizeof(S));
    M->wg[l] = (S*)calloc((size_t)sz, sizeof(S));
    M->m[l] = (S*)calloc((size_t)sz, sizeof(S));
    M->v[l] = (S*)calloc((size_t)sz, sizeof(S));
    M->ahw[l] = (S*)calloc((size_t)(n * dims[l + 1]), sizeof(S));
    const double limit = sqrt(6.0 / (double)(dims[l] + dims[l + 1]));
    for (idx_t i = 0; i < sz; ++i) M->w[l][i] = (S)rng_uniform_ab(&r, -limit, limit);
  }
  M->hw = (S*)calloc((size_t)(n * wmax), sizeof(S));
  M->x = p->features;
  FN(or_uniform_partition)(n, 8, M->wblocks); /* inc/driver.hpp:156 canonical W-grad blocks */
  return M;
}

void FN(or_model_free)(void* h) {
  or_model* M = (or_model*)h;
  if (!M) return;
  for (int l = 0; l < M->L; ++l) {
    free(M->w[l]);
    free(M->wg[l]);
    free(M->m[l]);
    free(M->v[l]);
    free(M->ahw[l]);
  }
  free(M->w);
  free(M->wg);
  free(M->m);
  free(M->v);
  free(M->ahw);
  free(M->hw);
  free(M->dims);
  free(M);
}

void FN(or_model_get_w)(void* h, S* out) {
  or_model* M = (or_model*)h;
  idx_t off = 0;
  for (int l = 0; l < M->L; ++l) {
    const idx_t sz = M->dims[l] * M->dims[l + 1];
    memcpy(out + off, M->w[l], sizeof(S) * (size_t)sz);
    off += sz;
  }
}

void FN(or_model_set_w)(void* h, const S* in) {
  or_model* M = (or_model*)h;
  idx_t off = 0;
  for (int l = 0; l < M->L; ++l) {
    const idx_t sz = M->dims[l] * M->dims[l + 1];
    memcpy(M->w[l], in + off, sizeof(S) * (size_t)sz);
    off += sz;
  }
}

/* inc/gcn.hpp:238-267 submit_forward */
static void model_forward(or_model* M) {
  const or_prepared* p = M->prep;
  const idx_t n = p->n;
  for (int l = 0; l < M->L; ++l) {
    const idx_t dl = M->dims[l], dl1 = M->dims[l + 1];
    const S* h_in = l == 0 ? M->x : M->ahw[l - 1];
    const int swap = M->order_swap && dl < dl1; /* gcn.hpp:145-148 */
    if (!swap) {
      gemm_core(h_in, n, dl, M->w[l], dl, dl1, 0, 0, 0, M->hw);
      spmm_core(n, p->ahat_t.row_ptr, p->ahat_t.col_idx, p->ahat_t.values, M->hw, dl1, 0, M->ahw[l]);
    } else {
      spmm_core(n, p->ahat_t.row_ptr, p->ahat_t.col_idx, p->ahat_t.values, h_in, dl, 0, M->hw);
      gemm_core(M->hw, n, dl, M->w[l], dl, dl1, 0, 0, 0, M->ahw[l]);
    }
    if (l < M->L - 1) /* inc/dense.hpp:208-215 relu_forward in place */
      for (idx_t i = 0; i < n * dl1; ++i) M->ahw[l][i] = M->ahw[l][i] > (S)0 ? M->ahw[l][i] : (S)0;
  }
}

/* inc/gcn.hpp:271-290 submit_loss_grad: per-worker argmax count + softmax_xent_sum, then the rank-order
 * all-reduce of the two S stats. Returns loss = sum / mask_count (S). */
static S model_loss_grad(or_model* M) {
  const or_prepared* p = M->prep;
  const idx_t C = M->dims[M->L];
  S* logits = M->ahw[M->L - 1];
  S tot0 = 0, tot1 = 0;
  for (int r = 0; r < p->parts; ++r) {
    const idx_t r0 = p->bounds[r], r1 = p->bounds[r + 1];
    S s1 = 0;
    for (idx_t i = r0; i < r1; ++i) {
      if (!p->mask[i]) continue;
      const S* row = logits + i * C;
      idx_t arg = 0;
      for (idx_t j = 1; j < C; ++j)
        if (row[j] > row[arg]) arg = j;
      if (arg == p->labels[i]) s1 += (S)1;
    }
    const S s0 = softmax_xent_core(logits + r0 * C, r1 - r0, C, p->labels + r0, p->mask + r0, logits + r0 * C,
                                   p->mask_count);
    if (p->parts == 1) {
      tot0 = s0;
      tot1 = s1;
    } else {
      tot0 += s0;
      tot1 += s1;
    }
  }
  M->last_acc = (double)tot1 / (double)p->mask_count;
  return tot0 / (S)p->mask_count;
}

/* inc/gcn.hpp:292-350 submit_backward + :365-377 finalize_wgrad */
static void model_backward(or_model* M) {
  const or_prepared* p = M->prep;
  const idx_t n = p->n;
  for (int l = M->L - 1; l >= 0; --l) {
    const idx_t dl = M->dims[l], dl1 = M->dims[l + 1];
    const S* grad_rows = M->ahw[l];
    if (!(l == 0 && M->skip_first)) {
      spmm_core(n, p->ahat.row_ptr, p->ahat.col_idx, p->ahat.values, M->ahw[l], dl1, 0, M->hw);
      grad_rows = M->hw;
    }
    const S* h_in = l == 0 ? M->x : M->ahw[l - 1];
    /* W-grad staging: every worker fills its own 8-block stage, then rank-order all-reduce */
    const idx_t bs = dl * dl1;
    S* stage = (S*)calloc((size_t)(8 * bs), sizeof(S));
    S* part = (S*)calloc((size_t)(8 * bs), sizeof(S));
    for (int r = 0; r < p->parts; ++r) {
      const idx_t r0 = p->bounds[r], r1 = p->bounds[r + 1];
      memset(part, 0, sizeof(S) * (size_t)(8 * bs));
      for (int g = 0; g < 8; ++g) {
        const idx_t a = M->wblocks[g] > r0 ? M->wblocks[g] : r0;
        const idx_t b = M->wblocks[g + 1] < r1 ? M->wblocks[g + 1] : r1;
        if (a >= b) continue;
        gemm_core(h_in + a * dl, b - a, dl, grad_rows + a * dl1, b - a, dl1, 1, 0, 0, part + g * bs);
      }
      if (p->parts == 1) {
        memcpy(stage, part, sizeof(S) * (size_t)(8 * bs));
      } else {
        for (idx_t i = 0; i < 8 * bs; ++i) stage[i] += part[i];
      }
    }
    for (idx_t i = 0; i < bs; ++i) M->wg[l][i] = (S)0;
    for (int g = 0; g < 8; ++g)
      for (idx_t i = 0; i < bs; ++i) M->wg[l][i] += stage[g * bs + i];
    free(stage);
    free(part);
    if (l > 0) { /* H-grad = grad_rows W^T (NT), then relu_backward into ahw[l-1] */
      S* hg = (S*)calloc((size_t)(n * dl), sizeof(S));
      gemm_core(grad_rows, n, dl1, M->w[l], dl, dl1, 0, 1, 0, hg);
      S* below = M->ahw[l - 1];
      for (idx_t i = 0; i < n * dl; ++i) below[i] = below[i] > (S)0 ? hg[i] : (S)0;
      free(hg);
    }
  }
}

/* mode 0: train_step(t) (gcn.hpp:175-184); 1: compute_gradients (:208-217); 2: loss_only (:189-205).
 * Optional dumps (global permuted rows): ahw_fwd = concat_l n x d_{l+1} after forward, loss_grad =
 * n x C, ahw_bwd = the pool after backward, wgrad = concat of W_G. */
int FN(or_model_step)(void* h, int32_t t, int32_t mode, double* loss, double* acc, S* ahw_fwd, S* loss_grad,
                      S* ahw_bwd, S* wgrad) {
  or_model* M = (or_model*)h;
  const idx_t n = M->prep->n;
  model_forward(M);
  if (ahw_fwd) {
    idx_t off = 0;
    for (int l = 0; l < M->L; ++l) {
      memcpy(ahw_fwd + off, M->ahw[l], sizeof(S) * (size_t)(n * M->dims[l + 1]));
      off += n * M->dims[l + 1];
    }
  }
  if (mode == 2) {
    /* loss_only: same arithmetic as the loss sum, logits untouched */
    const or_prepared* p = M->prep;
    const idx_t C = M->dims[M->L];
    S tot = 0;
    for (int r = 0; r < p->parts; ++r) {
      S s = 0;
      for (idx_t i = p->bounds[r]; i < p->bounds[r + 1]; ++i) {
        if (!p->mask[i]) continue;
        const S* row = M->ahw[M->L - 1] + i * C;
        S mx = row[0];
        for (idx_t j = 1; j < C; ++j) mx = mx < row[j] ? row[j] : mx;
        S se = 0;
        for (idx_t j = 0; j < C; ++j) se += OR_EXP(row[j] - mx);
        s += OR_LOG(se) - (row[p->labels[i]] - mx);
      }
      tot = p->parts == 1 ? s : tot + s;
    }
    *loss = (double)(tot / (S)p->mask_count);
    return 0;
  }
  *loss = (double)model_loss_grad(M);
  *acc = M->last_acc;
  if (loss_grad) memcpy(loss_grad, M->ahw[M->L - 1], sizeof(S) * (size_t)(n * M->dims[M->L]));
  model_backward(M);
  if (ahw_bwd) {
    idx_t off = 0;
    for (int l = 0; l < M->L; ++l) {
      memcpy(ahw_bwd + off, M->ahw[l], sizeof(S) * (size_t)(n * M->dims[l + 1]));
      off += n * M->dims[l + 1];
    }
  }
  if (wgrad) {
    idx_t off = 0;
    for (int l = 0; l < M->L; ++l) {
      memcpy(wgrad + off, M->wg[l], sizeof(S) * (size_t)(M->dims[l] * M->dims[l + 1]));
      off += M->dims[l] * M->dims[l + 1];
    }
  }
  if (mode == 0) {
    if (t < 1) return 2;
    for (int l = 0; l < M->L; ++l)
      adam_core(M->w[l], M->wg[l], M->m[l], M->v[l], M->dims[l] * M->dims[l + 1], t, M->lr, M->b1, M->b2, M->eps);
  }
  return 0;
}
