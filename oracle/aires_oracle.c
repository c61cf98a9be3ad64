/*
 * aires_oracle.c -- TEST INFRASTRUCTURE ONLY (see aires_oracle.h).
 *
 * CPU restatement of the reference AIRES hot path.  Built with the reference's
 * own arithmetic contract: -O2/-O3, no -march, -ffp-contract=off, so every
 * `sum += a*b` is one IEEE multiply then one IEEE add.
 */
#include "aires_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

void ao_free(ao_csr* m) {
  if (!m) return;
  free(m->ptr);
  free(m->idx);
  free(m->val);
  m->ptr = NULL;
  m->idx = NULL;
  m->val = NULL;
}

static void* xmalloc(size_t n) { return malloc(n ? n : 1); }
static void* xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s ? s : 1); }

/* sparse.hpp:119-140 */
int ao_csr_to_csc(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                  const uint64_t* col_idx, const double* values, ao_csr* b) {
  uint64_t nnz = row_ptr[n_rows];
  b->n_rows = n_rows;
  b->n_cols = n_cols;
  b->nnz = nnz;
  b->ptr = (uint64_t*)xcalloc(n_cols + 1, sizeof(uint64_t));
  b->idx = (uint64_t*)xmalloc(nnz * sizeof(uint64_t));
  b->val = (double*)xmalloc(nnz * sizeof(double));
  for (uint64_t k = 0; k < nnz; k++) b->ptr[col_idx[k] + 1]++;
  for (uint64_t c = 0; c < n_cols; c++) b->ptr[c + 1] += b->ptr[c];
  uint64_t* cursor = (uint64_t*)xmalloc(n_cols * sizeof(uint64_t));
  memcpy(cursor, b->ptr, n_cols * sizeof(uint64_t));
  for (uint64_t r = 0; r < n_rows; r++)
    for (uint64_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) {
      uint64_t c = col_idx[k];
      b->idx[cursor[c]] = r;
      b->val[cursor[c]] = values[k];
      cursor[c]++;
    }
  free(cursor);
  return AO_OK;
}

/* sparse.hpp:142-163 */
int ao_csc_to_csr(uint64_t n_rows, uint64_t n_cols, const uint64_t* col_ptr,
                  const uint64_t* row_idx, const double* values, ao_csr* a) {
  uint64_t nnz = col_ptr[n_cols];
  a->n_rows = n_rows;
  a->n_cols = n_cols;
  a->nnz = nnz;
  a->ptr = (uint64_t*)xcalloc(n_rows + 1, sizeof(uint64_t));
  a->idx = (uint64_t*)xmalloc(nnz * sizeof(uint64_t));
  a->val = (double*)xmalloc(nnz * sizeof(double));
  for (uint64_t k = 0; k < nnz; k++) a->ptr[row_idx[k] + 1]++;
  for (uint64_t r = 0; r < n_rows; r++) a->ptr[r + 1] += a->ptr[r];
  uint64_t* cursor = (uint64_t*)xmalloc(n_rows * sizeof(uint64_t));
  memcpy(cursor, a->ptr, n_rows * sizeof(uint64_t));
  for (uint64_t c = 0; c < n_cols; c++)
    for (uint64_t k = col_ptr[c]; k < col_ptr[c + 1]; k++) {
      uint64_t r = row_idx[k];
      a->idx[cursor[r]] = c;
      a->val[cursor[r]] = values[k];
      cursor[r]++;
    }
  free(cursor);
  return AO_OK;
}

/* spgemm.hpp:21-42 detail::dot_row_col */
static int dot_row_col(const uint64_t* ac, const double* av, uint64_t an, const uint64_t* br,
                       const double* bv, uint64_t bn, double* out, uint64_t* macs) {
  uint64_t i = 0, j = 0;
  int hit = 0;
  double sum = 0.0;
  while (i < an && j < bn) {
    if (ac[i] < br[j]) {
      i++;
    } else if (ac[i] > br[j]) {
      j++;
    } else {
      sum += av[i] * bv[j];
      (*macs)++;
      hit = 1;
      i++;
      j++;
    }
  }
  if (hit) *out = sum;
  return hit;
}

/* spgemm.hpp:60-132 spgemm_block (inner product, symbolic + exact alloc + numeric) */
int ao_spgemm_inner(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                    uint64_t rows, uint64_t a_n_cols, uint64_t b_n_rows, uint64_t b_n_cols,
                    const uint64_t* b_col_ptr, const uint64_t* b_row_idx,
                    const double* b_values, uint64_t tile_cols, ao_csr* c, uint64_t* macs_out) {
  if (a_n_cols != b_n_rows) return AO_DIMENSION_MISMATCH; /* spgemm.hpp:66-68 */
  if (tile_cols == 0) tile_cols = 256;                     /* spgemm.hpp:69 */
  c->n_rows = rows;
  c->n_cols = b_n_cols;
  c->ptr = (uint64_t*)xcalloc(rows + 1, sizeof(uint64_t));
  uint64_t macs = 0;
  for (uint64_t r = 0; r < rows; r++) { /* symbolic :94-109 */
    uint64_t count = 0;
    const uint64_t* ac = col_idx + row_ptr[r];
    const double* av = values + row_ptr[r];
    uint64_t an = row_ptr[r + 1] - row_ptr[r];
    for (uint64_t jt = 0; jt < b_n_cols; jt += tile_cols) {
      uint64_t jend = jt + tile_cols < b_n_cols ? jt + tile_cols : b_n_cols;
      for (uint64_t j = jt; j < jend; j++) {
        double v;
        if (dot_row_col(ac, av, an, b_row_idx + b_col_ptr[j], b_values + b_col_ptr[j],
                        b_col_ptr[j + 1] - b_col_ptr[j], &v, &macs))
          count++;
      }
    }
    c->ptr[r + 1] = c->ptr[r] + count;
  }
  c->nnz = c->ptr[rows];
  c->idx = (uint64_t*)xmalloc(c->nnz * sizeof(uint64_t)); /* exact alloc :111-112 */
  c->val = (double*)xmalloc(c->nnz * sizeof(double));
  uint64_t dummy = 0;
  for (uint64_t r = 0; r < rows; r++) { /* numeric :114-130 */
    uint64_t at = c->ptr[r];
    const uint64_t* ac = col_idx + row_ptr[r];
    const double* av = values + row_ptr[r];
    uint64_t an = row_ptr[r + 1] - row_ptr[r];
    for (uint64_t jt = 0; jt < b_n_cols; jt += tile_cols) {
      uint64_t jend = jt + tile_cols < b_n_cols ? jt + tile_cols : b_n_cols;
      for (uint64_t j = jt; j < jend; j++) {
        double v;
        if (dot_row_col(ac, av, an, b_row_idx + b_col_ptr[j], b_values + b_col_ptr[j],
                        b_col_ptr[j + 1] - b_col_ptr[j], &v, &dummy)) {
          c->idx[at] = j;
          c->val[at] = v;
          at++;
        }
      }
    }
  }
  *macs_out = macs;
  return AO_OK;
}

/* ---- row-wise restatement with identical bits ---------------------------- */

typedef struct {
  const uint64_t *row_ptr, *col_idx;
  const double* values;
  uint64_t r0, r1, b_n_rows, b_n_cols;
  const uint64_t *b_row_ptr, *b_col_idx;
  const double* b_values;
  /* output */
  uint64_t* counts; /* per row, length r1-r0 */
  uint64_t *idx, nnz, cap;
  double* val;
  uint64_t macs;
} rw_job;

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

static void* rw_run(void* arg) {
  rw_job* j = (rw_job*)arg;
  double* acc = (double*)xcalloc(j->b_n_cols, sizeof(double));
  unsigned char* seen = (unsigned char*)xcalloc(j->b_n_cols, 1);
  uint64_t* touched = (uint64_t*)xmalloc((j->b_n_cols ? j->b_n_cols : 1) * sizeof(uint64_t));
  j->cap = 1024;
  j->idx = (uint64_t*)xmalloc(j->cap * sizeof(uint64_t));
  j->val = (double*)xmalloc(j->cap * sizeof(double));
  j->nnz = 0;
  j->macs = 0;
  for (uint64_t r = j->r0; r < j->r1; r++) {
    uint64_t nt = 0;
    for (uint64_t p = j->row_ptr[r]; p < j->row_ptr[r + 1]; p++) { /* ascending k */
      uint64_t k = j->col_idx[p];
      if (k >= j->b_n_rows) continue; /* never intersects any B column */
      double a = j->values[p];
      for (uint64_t q = j->b_row_ptr[k]; q < j->b_row_ptr[k + 1]; q++) {
        uint64_t col = j->b_col_idx[q];
        if (!seen[col]) {
          seen[col] = 1;
          acc[col] = 0.0; /* dot_row_col: sum = 0.0 */
          touched[nt++] = col;
        }
        acc[col] += a * j->b_values[q]; /* one IEEE mul, one IEEE add */
        j->macs++;
      }
    }
    qsort(touched, nt, sizeof(uint64_t), cmp_u64);
    if (j->nnz + nt > j->cap) {
      while (j->nnz + nt > j->cap) j->cap *= 2;
      j->idx = (uint64_t*)realloc(j->idx, j->cap * sizeof(uint64_t));
      j->val = (double*)realloc(j->val, j->cap * sizeof(double));
    }
    for (uint64_t t = 0; t < nt; t++) {
      j->idx[j->nnz] = touched[t];
      j->val[j->nnz] = acc[touched[t]];
      seen[touched[t]] = 0;
      j->nnz++;
    }
    j->counts[r - j->r0] = nt;
  }
  free(acc);
  free(seen);
  free(touched);
  return NULL;
}

int ao_spgemm_rowwise(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                      uint64_t rows, uint64_t a_n_cols, uint64_t b_n_rows, uint64_t b_n_cols,
                      const uint64_t* b_row_ptr, const uint64_t* b_col_idx,
                      const double* b_values, int nthreads, ao_csr* c, uint64_t* macs_out) {
  if (a_n_cols != b_n_rows) return AO_DIMENSION_MISMATCH;
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > rows) nthreads = rows ? (int)rows : 1;
  uint64_t* counts = (uint64_t*)xcalloc(rows + 1, sizeof(uint64_t));
  rw_job* jobs = (rw_job*)xcalloc((size_t)nthreads, sizeof(rw_job));
  pthread_t* th = (pthread_t*)xcalloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; t++) {
    rw_job* j = &jobs[t];
    j->row_ptr = row_ptr;
    j->col_idx = col_idx;
    j->values = values;
    j->r0 = rows * (uint64_t)t / (uint64_t)nthreads;
    j->r1 = rows * (uint64_t)(t + 1) / (uint64_t)nthreads;
    j->b_n_rows = b_n_rows;
    j->b_n_cols = b_n_cols;
    j->b_row_ptr = b_row_ptr;
    j->b_col_idx = b_col_idx;
    j->b_values = b_values;
    j->counts = counts + 1 + j->r0;
    if (nthreads == 1)
      rw_run(j);
    else
      pthread_create(&th[t], NULL, rw_run, j);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  c->n_rows = rows;
  c->n_cols = b_n_cols;
  c->ptr = counts;
  for (uint64_t r = 0; r < rows; r++) counts[r + 1] += counts[r];
  c->nnz = counts[rows];
  c->idx = (uint64_t*)xmalloc(c->nnz * sizeof(uint64_t));
  c->val = (double*)xmalloc(c->nnz * sizeof(double));
  uint64_t macs = 0;
  for (int t = 0; t < nthreads; t++) {
    rw_job* j = &jobs[t];
    memcpy(c->idx + counts[j->r0], j->idx, j->nnz * sizeof(uint64_t));
    memcpy(c->val + counts[j->r0], j->val, j->nnz * sizeof(double));
    macs += j->macs;
    free(j->idx);
    free(j->val);
  }
  free(jobs);
  free(th);
  *macs_out = macs;
  return AO_OK;
}

/* ---- memory model (memory_model.hpp) ------------------------------------- */

uint64_t ao_calc_mem(uint64_t k, uint64_t q, uint64_t I, uint64_t V) {
  return (k + 1) * I + q * (I + V); /* :84-86 */
}

double ao_sparsity_percent(uint64_t n_rows, uint64_t n_cols, uint64_t nnz) {
  if (n_rows == 0 || n_cols == 0) return 100.0; /* :32-36 */
  double cells = (double)n_rows * (double)n_cols;
  return 100.0 * (1.0 - (double)nnz / cells);
}

uint64_t ao_estimate_output_memory(uint64_t alpha_a, double s_a, uint64_t alpha_b,
                                   double s_b) { /* :61-70 */
  if (alpha_a == 0) return 0;
  double x = 3.0 * (double)alpha_a * ((100.0 - s_a) / 100.0) *
             (1.0 + (double)alpha_b / (double)alpha_a + (100.0 - s_b) / 100.0);
  double snapped = round(x);
  double ax = fabs(x);
  if (fabs(x - snapped) <= 1e-9 * (ax > 1.0 ? ax : 1.0)) x = snapped;
  return (uint64_t)ceil(x);
}

int ao_block_budget(uint64_t device_total, uint64_t m_c, uint64_t m_b, uint64_t* p,
                    uint64_t* m_a) { /* :95-106 */
  if (device_total <= m_c + m_b) return AO_INSUFFICIENT_DEVICE_MEMORY;
  *m_a = device_total - m_c - m_b;
  *p = *m_a / 3;
  return AO_OK;
}

/* ---- RoBW Alg. 1 (partition.hpp:52-74) ----------------------------------- */

int ao_robw_cuts(const uint64_t* row_ptr, uint64_t n_rows, uint64_t m_a, uint64_t I,
                 uint64_t V, uint64_t* cuts, uint64_t* n_segs, uint64_t* bad_row) {
  uint64_t r = 0, s = 0;
  cuts[0] = 0;
  while (r < n_rows) {
    uint64_t k = 0, q = 0;
    while (r < n_rows) {
      uint64_t rn = row_ptr[r + 1] - row_ptr[r];
      if (ao_calc_mem(k + 1, q + rn, I, V) > m_a) break;
      k++;
      q += rn;
      r++;
    }
    if (k == 0) {
      *bad_row = r;
      *n_segs = s;
      return AO_ROW_TOO_LARGE;
    }
    cuts[++s] = r;
  }
  *n_segs = s;
  return AO_OK;
}

/* ---- FNV-1a 64 and checksum (serialize.hpp:22-59) ------------------------ */

#define FNV_OFF 14695981039346656037ULL
#define FNV_PRIME 1099511628211ULL

uint64_t ao_fnv1a64(const void* data, uint64_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = FNV_OFF;
  for (uint64_t i = 0; i < n; i++) {
    h ^= p[i];
    h *= FNV_PRIME;
  }
  return h;
}

static uint64_t fnv_u64(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; i++) {
    h ^= (unsigned char)(v >> (8 * i));
    h *= FNV_PRIME;
  }
  return h;
}

uint64_t ao_checksum(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, const uint64_t* row_ptr,
                     const uint64_t* col_idx, const double* values) {
  uint64_t h = FNV_OFF;
  h = fnv_u64(h, n_rows);
  h = fnv_u64(h, n_cols);
  h = fnv_u64(h, nnz);
  for (uint64_t i = 0; i <= n_rows; i++) h = fnv_u64(h, row_ptr[i]);
  for (uint64_t i = 0; i < nnz; i++) h = fnv_u64(h, col_idx[i]);
  for (uint64_t i = 0; i < nnz; i++) {
    uint64_t bits;
    memcpy(&bits, &values[i], 8);
    h = fnv_u64(h, bits);
  }
  return h;
}

/* ---- std::mt19937_64 restated, synth.hpp generators ---------------------- */

typedef struct {
  uint64_t mt[312];
  int i;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; i++)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->i = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->i >= 312) {
    for (int i = 0; i < 312; i++) {
      uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->i = 0;
  }
  uint64_t x = s->mt[s->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; } /* :14-16 */

int ao_gen_sparse(uint64_t rows, uint64_t cols, double density, uint64_t seed, double lo,
                  double hi, ao_csr* m) { /* synth.hpp:49-69 */
  if (!(density > 0.0) || density > 1.0) return AO_INVALID_DENSITY;
  mt64* rng = (mt64*)xmalloc(sizeof(mt64));
  mt64_seed(rng, seed);
  uint64_t cap = 1024;
  m->n_rows = rows;
  m->n_cols = cols;
  m->ptr = (uint64_t*)xcalloc(rows + 1, sizeof(uint64_t));
  m->idx = (uint64_t*)xmalloc(cap * sizeof(uint64_t));
  m->val = (double*)xmalloc(cap * sizeof(double));
  uint64_t nnz = 0;
  for (uint64_t i = 0; i < rows; i++) {
    for (uint64_t j = 0; j < cols; j++) {
      if (uniform01(rng) < density) {
        double v = lo + (hi - lo) * uniform01(rng);
        if (v == 0.0) continue;
        if (nnz == cap) {
          cap *= 2;
          m->idx = (uint64_t*)realloc(m->idx, cap * sizeof(uint64_t));
          m->val = (double*)realloc(m->val, cap * sizeof(double));
        }
        m->idx[nnz] = j;
        m->val[nnz] = v;
        nnz++;
      }
    }
    m->ptr[i + 1] = nnz;
  }
  m->nnz = nnz;
  free(rng);
  return AO_OK;
}

int ao_gen_features(uint64_t n_nodes, uint64_t dim, double sparsity_pct, uint64_t seed,
                    ao_csr* out) { /* synth.hpp:73-78 */
  if (sparsity_pct < 0.0 || sparsity_pct >= 100.0) return AO_INVALID_DENSITY;
  return ao_gen_sparse(n_nodes, dim, (100.0 - sparsity_pct) / 100.0, seed, 0.1, 1.0, out);
}

/* ---- gcn.hpp:29-72 normalize_adjacency ----------------------------------- */

int ao_normalize_adjacency(uint64_t n, const uint64_t* row_ptr, const uint64_t* col_idx,
                           const double* values, ao_csr* ah) {
  uint64_t nnz = row_ptr[n];
  for (uint64_t k = 0; k < nnz; k++)
    if (values[k] < 0.0) return AO_NEGATIVE_WEIGHT;
  ah->n_rows = ah->n_cols = n;
  ah->ptr = (uint64_t*)xcalloc(n + 1, sizeof(uint64_t));
  ah->idx = (uint64_t*)xmalloc((nnz + n) * sizeof(uint64_t));
  ah->val = (double*)xmalloc((nnz + n) * sizeof(double));
  uint64_t w = 0;
  for (uint64_t r = 0; r < n; r++) { /* A + I, diagonal merged in column order */
    int placed = 0;
    for (uint64_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) {
      uint64_t c = col_idx[k];
      if (!placed && c >= r) {
        ah->idx[w] = r;
        ah->val[w] = (c == r) ? values[k] + 1.0 : 1.0;
        w++;
        placed = 1;
        if (c == r) continue;
      }
      ah->idx[w] = c;
      ah->val[w] = values[k];
      w++;
    }
    if (!placed) {
      ah->idx[w] = r;
      ah->val[w] = 1.0;
      w++;
    }
    ah->ptr[r + 1] = w;
  }
  ah->nnz = w;
  double* degree = (double*)xcalloc(n, sizeof(double));
  for (uint64_t r = 0; r < n; r++)
    for (uint64_t k = ah->ptr[r]; k < ah->ptr[r + 1]; k++) degree[r] += ah->val[k];
  for (uint64_t r = 0; r < n; r++)
    for (uint64_t k = ah->ptr[r]; k < ah->ptr[r + 1]; k++)
      ah->val[k] = ah->val[k] / sqrt(degree[r] * degree[ah->idx[k]]);
  free(degree);
  return AO_OK;
}

/* synth.hpp:81-86 gen_weights: row-major in_dim x out_dim, uniform01 - 0.5 */
int ao_gen_weights(uint64_t in_dim, uint64_t out_dim, uint64_t seed, double* out) {
  mt64 st;
  mt64_seed(&st, seed);
  for (uint64_t i = 0; i < in_dim * out_dim; i++) out[i] = uniform01(&st) - 0.5;
  return AO_OK;
}

/* gcn.hpp:90-116 combine: per row, acc[j] = sum_k v_k * W[in_k][j] in ascending k from 0.0
   (separate multiply and add; the build uses -ffp-contract=off), keep acc[j] > 0. */
int ao_combine(uint64_t rows, uint64_t x_cols, const uint64_t* row_ptr, const uint64_t* col_idx,
               const double* values, const double* w, uint64_t w_rows, uint64_t w_cols, ao_csr* out) {
  if (x_cols != w_rows) return AO_DIMENSION_MISMATCH;
  double* acc = (double*)xmalloc(w_cols * sizeof(double));
  uint64_t cap = 1024, nnz = 0;
  out->n_rows = rows;
  out->n_cols = w_cols;
  out->ptr = (uint64_t*)xcalloc(rows + 1, sizeof(uint64_t));
  out->idx = (uint64_t*)xmalloc(cap * sizeof(uint64_t));
  out->val = (double*)xmalloc(cap * sizeof(double));
  for (uint64_t r = 0; r < rows; r++) {
    for (uint64_t j = 0; j < w_cols; j++) acc[j] = 0.0;
    for (uint64_t k = row_ptr[r]; k < row_ptr[r + 1]; k++) {
      const uint64_t in = col_idx[k];
      const double v = values[k];
      for (uint64_t j = 0; j < w_cols; j++) acc[j] += v * w[in * w_cols + j];
    }
    for (uint64_t j = 0; j < w_cols; j++)
      if (acc[j] > 0.0) {
        if (nnz == cap) {
          cap *= 2;
          out->idx = (uint64_t*)realloc(out->idx, cap * sizeof(uint64_t));
          out->val = (double*)realloc(out->val, cap * sizeof(double));
        }
        out->idx[nnz] = j;
        out->val[nnz] = acc[j];
        nnz++;
      }
    out->ptr[r + 1] = nnz;
  }
  out->nnz = nnz;
  free(acc);
  return AO_OK;
}

/* ---- benchmark inputs for the reference arm (bench.py --impl reference) ----------------------
 * A restatement of the B200 library's Chung-Lu generator (paper_2507_02006_b200/csrc/ab2_synth.cpp,
 * aires_b200_synth_graph; BASELINE.md §4 / SURVEY.md §8(d) "Synthetic inputs"), so the reference
 * arm builds the identical Ã without loading libaires_b200.so.  Same arithmetic, draw for draw:
 * splitmix64 hashes of the pair index, the continuous power law on [0, n) with density
 * (x + i0)^-alpha, i0 bisected on a log scale so the heaviest node's expected degree is the cap,
 * the std::mt19937_64 Fisher-Yates relabel, up to four sampling rounds rescaling the pair count,
 * and normalize_adjacency's (gcn.hpp:29-72) D^-1/2 (A+I) D^-1/2 values.  Rows are sorted and
 * de-duplicated, so the multi-threaded counting pass is deterministic.  Pinned byte for byte
 * against aires_b200_synth_graph by tests/test_oracle.py::test_synth_graph_restatement. */
static uint64_t sg_splitmix(uint64_t x) {
  uint64_t z = x + 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double sg_u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

typedef struct {
  double alpha, i0, a1, lo, hi;
  uint64_t n;
} sg_plaw;

static sg_plaw sg_plaw_make(uint64_t n, double alpha, double i0) {
  sg_plaw p;
  p.alpha = alpha;
  p.i0 = i0;
  p.n = n;
  p.a1 = 1.0 - alpha;
  p.lo = pow(i0, p.a1);
  p.hi = pow((double)n + i0, p.a1);
  return p;
}
static uint64_t sg_plaw_sample(const sg_plaw* p, double u) {
  double t = p->lo + u * (p->hi - p->lo);
  double x = pow(t, 1.0 / p->a1) - p->i0;
  if (!(x >= 0)) x = 0;
  uint64_t i = (uint64_t)x;
  return i >= p->n ? p->n - 1 : i;
}
static double sg_plaw_mass(const sg_plaw* p, double a, double b) {
  return (pow(b + p->i0, p->a1) - pow(a + p->i0, p->a1)) / (p->hi - p->lo);
}
static double sg_top(uint64_t n, double alpha, double pairs, double i0) {
  sg_plaw p = sg_plaw_make(n, alpha, i0);
  return 2.0 * pairs * sg_plaw_mass(&p, 0.0, 1.0);
}
static double sg_solve_i0(uint64_t n, double alpha, double pairs, double cap) {
  if (sg_top(n, alpha, pairs, 1e-9) <= cap) return 1e-9;
  double lo = 1e-9, hi = (double)n;
  for (int it = 0; it < 200; it++) {
    double mid = sqrt(lo * hi);
    if (sg_top(n, alpha, pairs, mid) > cap)
      lo = mid;
    else
      hi = mid;
  }
  return hi;
}

typedef struct {
  const sg_plaw* pl;
  const uint32_t* perm;
  uint64_t seed, p0, p1, r0, r1;
  uint32_t* deg;      /* atomic adds */
  uint64_t* cur;      /* atomic cursors */
  uint32_t* raw;
  const uint64_t* off;
  uint64_t* cnt;
  int phase;
} sg_job;

static void sg_pair(const sg_job* j, uint64_t p, uint32_t* u, uint32_t* v) {
  uint64_t h1 = sg_splitmix(j->seed * 0x100000001b3ULL + 2 * p);
  uint64_t h2 = sg_splitmix(j->seed * 0x100000001b3ULL + 2 * p + 1);
  uint64_t a = sg_plaw_sample(j->pl, sg_u01(h1)), b = sg_plaw_sample(j->pl, sg_u01(h2));
  *u = j->perm ? j->perm[a] : (uint32_t)a;
  *v = j->perm ? j->perm[b] : (uint32_t)b;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

static void* sg_run(void* arg) {
  sg_job* j = (sg_job*)arg;
  if (j->phase == 0) {
    for (uint64_t p = j->p0; p < j->p1; p++) {
      uint32_t u, v;
      sg_pair(j, p, &u, &v);
      if (u == v) continue;
      __atomic_fetch_add(&j->deg[u], 1u, __ATOMIC_RELAXED);
      __atomic_fetch_add(&j->deg[v], 1u, __ATOMIC_RELAXED);
    }
  } else if (j->phase == 1) {
    for (uint64_t p = j->p0; p < j->p1; p++) {
      uint32_t u, v;
      sg_pair(j, p, &u, &v);
      if (u == v) continue;
      j->raw[__atomic_fetch_add(&j->cur[u], 1ull, __ATOMIC_RELAXED)] = v;
      j->raw[__atomic_fetch_add(&j->cur[v], 1ull, __ATOMIC_RELAXED)] = u;
    }
  } else {
    for (uint64_t r = j->r0; r < j->r1; r++) { /* sort + unique per row */
      uint32_t* s = j->raw + j->off[r];
      uint64_t m = j->off[r + 1] - j->off[r], w = 0;
      qsort(s, m, sizeof(uint32_t), cmp_u32);
      for (uint64_t i = 0; i < m; i++)
        if (w == 0 || s[i] != s[w - 1]) s[w++] = s[i];
      j->cnt[r + 1] = w;
    }
  }
  return NULL;
}

static void sg_parallel(sg_job* proto, int phase, uint64_t n_items, int threads) {
  if (threads < 1) threads = 1;
  if (n_items < 4096) threads = 1;
  sg_job* jobs = (sg_job*)xcalloc((size_t)threads, sizeof(sg_job));
  pthread_t* th = (pthread_t*)xcalloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; t++) {
    jobs[t] = *proto;
    jobs[t].phase = phase;
    uint64_t a = n_items * (uint64_t)t / (uint64_t)threads, b = n_items * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].p0 = jobs[t].r0 = a;
    jobs[t].p1 = jobs[t].r1 = b;
    if (threads == 1)
      sg_run(&jobs[t]);
    else
      pthread_create(&th[t], NULL, sg_run, &jobs[t]);
  }
  if (threads > 1)
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
}

/* One sampling round: M pairs -> symmetric, loop-free, duplicate-free CSR (ptr n+1, col u32). */
static void sg_build(uint64_t n, uint64_t M, const sg_plaw* pl, const uint32_t* perm, uint64_t seed,
                     int threads, uint64_t** ptr_out, uint32_t** col_out) {
  sg_job j;
  memset(&j, 0, sizeof j);
  j.pl = pl;
  j.perm = perm;
  j.seed = seed;
  j.deg = (uint32_t*)xcalloc(n, sizeof(uint32_t));
  sg_parallel(&j, 0, M, threads);
  uint64_t* off = (uint64_t*)xcalloc(n + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; i++) off[i + 1] = off[i] + j.deg[i];
  free(j.deg);
  j.deg = NULL;
  j.raw = (uint32_t*)xmalloc(off[n] * sizeof(uint32_t));
  j.cur = (uint64_t*)xmalloc(n * sizeof(uint64_t));
  memcpy(j.cur, off, n * sizeof(uint64_t));
  sg_parallel(&j, 1, M, threads);
  free(j.cur);
  j.off = off;
  j.cnt = (uint64_t*)xcalloc(n + 1, sizeof(uint64_t));
  sg_parallel(&j, 2, n, threads);
  uint64_t* ptr = j.cnt; /* cnt[r+1] -> prefix */
  for (uint64_t i = 0; i < n; i++) ptr[i + 1] += ptr[i];
  uint32_t* col = (uint32_t*)xmalloc((ptr[n] ? ptr[n] : 1) * sizeof(uint32_t));
  for (uint64_t r = 0; r < n; r++) memcpy(col + ptr[r], j.raw + off[r], (ptr[r + 1] - ptr[r]) * sizeof(uint32_t));
  free(j.raw);
  free(off);
  *ptr_out = ptr;
  *col_out = col;
}

int ao_synth_graph(uint64_t n, uint64_t target_nnz, double alpha, uint64_t degree_cap, uint64_t seed,
                   uint64_t relabel_seed, int relabel, int normalize, int threads, ao_csr* out, double* stats) {
  if (n == 0 || n >= (1ull << 32) || !(alpha > 0.0 && alpha < 1.0)) return AO_INDEX_OUT_OF_RANGE;
  if (threads < 1) threads = 1;
  uint32_t* perm = NULL;
  if (relabel) {
    perm = (uint32_t*)xmalloc(n * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
    mt64* rng = (mt64*)xmalloc(sizeof(mt64));
    mt64_seed(rng, relabel_seed);
    for (uint64_t i = n - 1; i > 0; i--) {
      uint64_t k = mt64_next(rng) % (i + 1);
      uint32_t t = perm[i];
      perm[i] = perm[k];
      perm[k] = t;
    }
    free(rng);
  }
  double pairs = (double)target_nnz / 2.0;
  if (pairs < 1.0) pairs = 1.0;
  double cap = degree_cap ? (double)degree_cap : (double)n;
  uint64_t* gp = NULL;
  uint32_t* gc = NULL;
  int rounds = 0;
  double i0 = 0;
  for (; rounds < 4; rounds++) {
    i0 = sg_solve_i0(n, alpha, pairs, cap);
    sg_plaw pl = sg_plaw_make(n, alpha, i0);
    free(gp);
    free(gc);
    sg_build(n, (uint64_t)pairs, &pl, perm, seed, threads, &gp, &gc);
    double got = (double)gp[n];
    if (target_nnz == 0 || got <= 0) break;
    double ratio = (double)target_nnz / got;
    if (fabs(ratio - 1.0) < 0.005) break;
    pairs *= ratio * (ratio > 1 ? 1.02 : 1.0);
  }
  free(perm);
  const uint64_t nnz_a = gp[n];
  uint64_t maxdeg = 0;
  for (uint64_t r = 0; r < n; r++)
    if (gp[r + 1] - gp[r] > maxdeg) maxdeg = gp[r + 1] - gp[r];
  const uint64_t nnz = normalize ? nnz_a + n : nnz_a;
  out->n_rows = n;
  out->n_cols = n;
  out->nnz = nnz;
  out->ptr = (uint64_t*)xmalloc((n + 1) * sizeof(uint64_t));
  out->idx = (uint64_t*)xmalloc(nnz * sizeof(uint64_t));
  out->val = (double*)xmalloc(nnz * sizeof(double));
  out->ptr[0] = 0;
  for (uint64_t r = 0; r < n; r++) out->ptr[r + 1] = out->ptr[r] + (gp[r + 1] - gp[r]) + (normalize ? 1 : 0);
  /* gcn.hpp:29-72 with unit weights and no loops: d_i = deg_i + 1, diagonal in column order */
  for (uint64_t r = 0; r < n; r++) {
    uint64_t w = out->ptr[r];
    const double dr = (double)(gp[r + 1] - gp[r] + 1);
    int placed = !normalize;
    for (uint64_t k = gp[r]; k <= gp[r + 1]; k++) {
      uint64_t c = k < gp[r + 1] ? gc[k] : UINT64_MAX;
      if (!placed && c > r) {
        out->idx[w] = r;
        out->val[w++] = 1.0 / sqrt(dr * dr);
        placed = 1;
      }
      if (k == gp[r + 1]) break;
      out->idx[w] = c;
      out->val[w++] = normalize ? 1.0 / sqrt(dr * (double)(gp[c + 1] - gp[c] + 1)) : 1.0;
    }
  }
  if (stats) {
    stats[0] = (double)nnz_a;
    stats[1] = (double)maxdeg;
    stats[2] = (double)nnz_a / (double)n;
    stats[3] = (double)(rounds + 1);
    stats[4] = 0.0;
    stats[5] = i0;
    stats[6] = stats[7] = 0.0;
  }
  free(gp);
  free(gc);
  return AO_OK;
}

/* Sum over rows[] of FNV-1a 64 (serialize.hpp:22-48) of (row id, col_idx..., value bits...) --
 * the row hash oracle/ref_shim.cpp:ref_spgemm_rows_timed reports for the reference's sampled rows,
 * computed here over any CSR (e.g. the B200 product read back) for the same rows. */
uint64_t ao_rows_hash(const uint64_t* row_ptr, const uint64_t* col_idx, const double* values,
                      const uint64_t* rows, uint64_t n_sample) {
  uint64_t tot = 0;
  for (uint64_t i = 0; i < n_sample; i++) {
    uint64_t r = rows[i], h = 0xcbf29ce484222325ULL;
    h = fnv_u64(h, r);
    for (uint64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) h = fnv_u64(h, col_idx[p]);
    for (uint64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++) {
      uint64_t b;
      memcpy(&b, &values[p], 8);
      h = fnv_u64(h, b);
    }
    tot += h;
  }
  return tot;
}
