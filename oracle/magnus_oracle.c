/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the MAGNUS SpGEMM hot path.
 *
 * A plain-C restatement of the reference's Python/numpy algorithm
 * (/root/reference/pkg/src/spgemm/{magnus,accumulators,planner,gustavson,
 * matrix,util}.py).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * path (paper_2501_07056_b200/) never does.
 *
 * The summation association of the reference lives in numpy (pinned as
 * numpy>=1.24 by the reference's pyproject.toml:10; validated here against
 * numpy 2.3.5 golden vectors, tests/golden/):
 *   - np.bincount(weights) / np.add.at (accumulators.py:90,93): sequential,
 *     starting from +0.0, in input order;
 *   - np.add.reduceat (accumulators.py:129): out = x0; out += pairwise(x1..),
 *     numpy's published pairwise summation (block 128, 8 accumulators).
 * Both are restated below; every function cites the reference line it follows.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "magnus_oracle.h"

static _Thread_local char g_err[512];
const char* oracle_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ---------------------------------------------------------------- util.py */
/* ceil_pow2 util.py:6-10 */
static int64_t ceil_pow2(int64_t x) { int64_t p = 1; while (p < x) p <<= 1; return p; }
/* floor_pow2 util.py:13-17 */
static int64_t floor_pow2_u(unsigned __int128 x) {
  unsigned __int128 p = 1; while ((p << 1) <= x) p <<= 1; return (int64_t)p;
}
/* exact_log2 util.py:20-25 */
static int64_t exact_log2(int64_t x) { int64_t k = 0; while (((int64_t)1 << k) < x) ++k; return k; }
/* round_pow2_of_sqrt util.py:28-44 (integer-only, ties round up) */
static int64_t round_pow2_of_sqrt(unsigned __int128 num, unsigned __int128 den) {
  if (num < den) return 1;
  int k = 0;
  while (num >= (den << (2 * (k + 1)))) ++k;
  if (num >= (den << (2 * k + 1))) ++k;
  return (int64_t)1 << k;
}

/* ------------------------------------------------------------- planner.py */
/* compute_chunk_plan planner.py:106-152 (+ max_l2_cols :100-103) */
int oracle_compute_chunk_plan(const oracle_sys* sys, int64_t m_c, int numeric, int allow_coarse, oracle_plan* out) {
  if (m_c < 1) return fail(ORACLE_INPUT, "m_c must be >= 1");
  int64_t plan_cols = ceil_pow2(m_c);
  int64_t sda = numeric ? sys->val_bytes + 1 : 1;                       /* dense_accum_bytes :74-76 */
  int64_t scf = sys->histo_type_bytes + sys->prefix_sum_type_bytes + 2 * sys->cache_line_bytes; /* :71-72 */
  unsigned __int128 raw = (unsigned __int128)sys->l2_bytes * (unsigned __int128)sys->l2_bytes / (unsigned __int128)(4 * 1 * scf);
  int64_t m_max = raw >= 1 ? floor_pow2_u(raw) : 1;
  int use_coarse = allow_coarse && plan_cols > m_max;
  int64_t span = use_coarse ? m_max : plan_cols;
  int64_t n_fine = round_pow2_of_sqrt((unsigned __int128)span * sda, scf);
  int64_t min_len = sys->cache_line_bytes / 4; if (min_len < 1) min_len = 1;
  int64_t lim = span / min_len; if (lim < 1) lim = 1;
  if (n_fine > lim) n_fine = lim;
  if (n_fine > span) n_fine = span;
  if (n_fine < 1) n_fine = 1;
  int64_t chunk_len = span / n_fine;
  out->plan_cols = plan_cols; out->s_dense_accum = sda; out->s_chunk_fine = scf;
  out->n_chunks_fine = n_fine; out->chunk_len_fine = chunk_len; out->shift_fine = exact_log2(chunk_len);
  out->m_max_l2 = m_max; out->use_coarse = use_coarse;
  out->n_chunks_coarse = use_coarse ? plan_cols / m_max : 1;
  out->chunk_len_coarse = use_coarse ? m_max : plan_cols;
  out->shift_coarse = exact_log2(out->chunk_len_coarse);
  return ORACLE_OK;
}

/* ------------------------------------------------------------ gustavson.py */
/* row_intermediate_stats gustavson.py:97-134 */
static void row_stats(const oracle_csr* A, const oracle_csr* B, int64_t* inter, int64_t* mn, int64_t* mx) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < A->n_rows; ++i) {
    int64_t s = 0, lo = B->n_cols, hi = -1;
    for (int64_t j = A->row_ptr[i]; j < A->row_ptr[i + 1]; ++j) {
      int64_t k = A->col[j];
      int64_t b0 = B->row_ptr[k], b1 = B->row_ptr[k + 1];
      s += b1 - b0;
      if (b1 > b0) {
        if ((int64_t)B->col[b0] < lo) lo = B->col[b0];
        if ((int64_t)B->col[b1 - 1] > hi) hi = B->col[b1 - 1];
      }
    }
    inter[i] = s;
    mn[i] = s > 0 ? lo : 0;
    mx[i] = s > 0 ? hi : -1;
  }
}

/* --------------------------------------------------------- numpy restated */
/* numpy pairwise summation (restated from numpy's published algorithm;
 * reached through np.add.reduceat at accumulators.py:129). */
static double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
  }
}

typedef struct { int64_t key; int64_t pos; double val; } kv_t;
static int kv_cmp(const void* x, const void* y) {
  const kv_t* a = (const kv_t*)x; const kv_t* b = (const kv_t*)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->pos < b->pos ? -1 : (a->pos > b->pos);
}

/* per-thread scratch (WorkerScratch magnus.py:97-109) */
typedef struct {
  kv_t* kv; int64_t kv_cap;
  double* tmp; int64_t tmp_cap;
  double* dbuf; unsigned char* dmark; int64_t d_cap;     /* DenseAccumulator accumulators.py:44-60 */
  int64_t* touched; int64_t t_cap;
  int64_t* colf; double* valf; int64_t f_cap;             /* fine-level reorder buffers */
  int64_t* counts; int64_t* offsets; int64_t* heads; int64_t c_cap;
  int64_t* groups; int64_t g_cap;
} scratch_t;

#define GROW(p, cap, need, T) do { if ((need) > (cap)) { int64_t nc_ = (need) * 2 + 16; \
  (p) = (T*)realloc((p), (size_t)nc_ * sizeof(T)); (cap) = nc_; } } while (0)

/* counts / offsets / heads share one allocation of 3*n entries */
static void chunk_arrays(scratch_t* s, int64_t n) {
  if (n > s->c_cap) {
    free(s->counts);
    s->c_cap = 2 * n + 16;
    s->counts = (int64_t*)malloc((size_t)(3 * s->c_cap) * sizeof(int64_t));
  }
  s->offsets = s->counts + s->c_cap;
  s->heads = s->counts + 2 * s->c_cap;
}

static void scratch_free(scratch_t* s) {
  free(s->kv); free(s->tmp); free(s->dbuf); free(s->dmark); free(s->touched);
  free(s->colf); free(s->valf); free(s->counts); free(s->groups);
  memset(s, 0, sizeof *s);
}

/* sort_accumulate accumulators.py:113-129: stable argsort on cols, merge with
 * np.add.reduceat (x0 + pairwise(rest)).  Writes ascending distinct cols.
 * If vals == NULL returns only the distinct count (np.unique, magnus.py:190,411). */
static int64_t sort_accumulate(scratch_t* s, const int64_t* cols, const double* vals, int64_t n,
                               int64_t* out_c, double* out_v) {
  if (n == 0) return 0;
  GROW(s->kv, s->kv_cap, n, kv_t);
  for (int64_t i = 0; i < n; ++i) { s->kv[i].key = cols[i]; s->kv[i].pos = i; s->kv[i].val = vals ? vals[i] : 0.0; }
  qsort(s->kv, (size_t)n, sizeof(kv_t), kv_cmp);   /* (key,pos) unique => equals a stable sort */
  int64_t m = 0;
  for (int64_t i = 0; i < n;) {
    int64_t j = i + 1;
    while (j < n && s->kv[j].key == s->kv[i].key) ++j;
    if (out_c) {
      out_c[m] = s->kv[i].key;
      if (vals) {
        GROW(s->tmp, s->tmp_cap, j - i, double);
        for (int64_t t = i + 1; t < j; ++t) s->tmp[t - i - 1] = s->kv[t].val;
        double x = s->kv[i].val;
        if (j - i > 1) x += pairwise_sum(s->tmp, j - i - 1);
        out_v[m] = x;
      }
    }
    ++m; i = j;
  }
  return m;
}

static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y; return a < b ? -1 : (a > b);
}

/* dense_accumulate accumulators.py:68-97 followed by the caller's argsort
 * (magnus.py:164,500): sums are sequential from +0.0 in input order
 * (np.bincount / np.add.at); output ascending.  vals == NULL: distinct count
 * only (dense_accumulate_symbolic accumulators.py:100-110). */
static int64_t dense_accumulate(scratch_t* s, const int64_t* cols, const double* vals, int64_t n, int64_t capacity,
                                int64_t* out_c, double* out_v, int* err) {
  if (n == 0) return 0;
  if (capacity > s->d_cap) {
    free(s->dbuf); free(s->dmark);
    s->dbuf = (double*)calloc((size_t)capacity, sizeof(double));
    s->dmark = (unsigned char*)calloc((size_t)capacity, 1);
    s->d_cap = capacity;
  }
  GROW(s->touched, s->t_cap, n, int64_t);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = cols[i];
    if (c < 0 || c >= capacity) { *err = 1; return 0; }
    if (!s->dmark[c]) { s->dmark[c] = 1; s->dbuf[c] = 0.0; s->touched[m++] = c; }
    if (vals) s->dbuf[c] += vals[i];
  }
  qsort(s->touched, (size_t)m, sizeof(int64_t), cmp_i64);
  for (int64_t t = 0; t < m; ++t) {
    int64_t c = s->touched[t];
    if (out_c) { out_c[t] = c; if (vals) out_v[t] = s->dbuf[c]; }
    s->dmark[c] = 0; s->dbuf[c] = 0.0;
  }
  return m;
}

/* merge_chunks_for_sort accumulators.py:137-157 (greedy toward target) */
static int64_t merge_chunks_for_sort(const int64_t* sizes, int64_t n, int64_t target, int64_t* bounds) {
  int64_t nb = 0;
  bounds[nb++] = 0;
  if (n == 0) return nb;
  int64_t total = sizes[0];
  for (int64_t i = 1; i < n; ++i) {
    int64_t a = total + sizes[i] - target; if (a < 0) a = -a;
    int64_t b = total - target; if (b < 0) b = -b;
    if (a < b) total += sizes[i];
    else { bounds[nb++] = i; total = sizes[i]; }
  }
  bounds[nb++] = n;
  return nb;
}

typedef struct {
  const oracle_sys* sys; const oracle_thresholds* th;
  const oracle_plan* plan;
  /* emitter (_RowEmitter magnus.py:112-141) */
  uint32_t* c_col; double* c_val; int64_t pos, end; int numeric; int err;
} emit_t;

static void emit(emit_t* e, int64_t base, const int64_t* cols, const double* vals, int64_t k) {
  if (!e->numeric) return;
  if (e->pos + k > e->end) { e->err = 2; return; }
  for (int64_t t = 0; t < k; ++t) { e->c_col[e->pos + t] = (uint32_t)(cols[t] + base); e->c_val[e->pos + t] = vals[t]; }
  e->pos += k;
}

/* _accumulate_chunks magnus.py:144-192 */
static int64_t accumulate_chunks(scratch_t* s, emit_t* e, const int64_t* col_f, const double* val_f,
                                 const int64_t* offsets, int64_t base) {
  const oracle_plan* plan = e->plan;
  int64_t n = plan->n_chunks_fine, cl = plan->chunk_len_fine;
  int64_t total = 0;
  GROW(s->groups, s->g_cap, n + 2, int64_t);
  /* output staging reuses a per-call buffer */
  int64_t* oc = NULL; double* ov = NULL;
  int64_t i = 0;
  while (i < n) {
    int64_t sz = offsets[i + 1] - offsets[i];
    if (sz >= e->th->sort_dense_crossover) {                 /* Accum.DENSE (select_accumulator :132-134) */
      int64_t st = offsets[i];
      oc = (int64_t*)malloc((size_t)sz * sizeof(int64_t)); ov = (double*)malloc((size_t)sz * sizeof(double));
      int derr = 0;
      int64_t m = dense_accumulate(s, col_f + st, e->numeric ? val_f + st : NULL, sz, cl, oc, ov, &derr);
      if (derr) e->err = 2;
      emit(e, base + i * cl, oc, ov, m);
      total += m; free(oc); free(ov);
      ++i; continue;
    }
    int64_t j = i;
    while (j < n && (offsets[j + 1] - offsets[j]) < e->th->sort_dense_crossover) ++j;
    int64_t* sizes = (int64_t*)malloc((size_t)(j - i) * sizeof(int64_t));
    for (int64_t t = i; t < j; ++t) sizes[t - i] = offsets[t + 1] - offsets[t];
    int64_t* bounds = (int64_t*)malloc((size_t)(j - i + 2) * sizeof(int64_t));
    int64_t nb = merge_chunks_for_sort(sizes, j - i, e->th->sort_sweet_spot, bounds);
    for (int64_t g = 0; g + 1 < nb; ++g) {
      int64_t a = bounds[g], b = bounds[g + 1];
      int64_t st = offsets[i + a], en = offsets[i + b];
      if (st == en) continue;
      int64_t len = en - st;
      int64_t* keys = (int64_t*)malloc((size_t)len * sizeof(int64_t));
      /* composite keys col + chunk_offset*len (magnus.py:179-184) */
      for (int64_t q = a; q < b; ++q)
        for (int64_t t = offsets[i + q]; t < offsets[i + q + 1]; ++t) keys[t - st] = col_f[t] + (q - a) * cl;
      oc = (int64_t*)malloc((size_t)len * sizeof(int64_t)); ov = (double*)malloc((size_t)len * sizeof(double));
      int64_t m = sort_accumulate(s, keys, e->numeric ? val_f + st : NULL, len, oc, ov);
      emit(e, base + (i + a) * cl, oc, ov, m);
      total += m;
      free(keys); free(oc); free(ov);
    }
    free(sizes); free(bounds);
    i = j;
  }
  return total;
}

/* fine_level_chunk magnus.py:195-221 (chunk-local cols in, stable reorder) */
static int64_t fine_level_chunk(scratch_t* s, emit_t* e, const int64_t* cols, const double* vals, int64_t n, int64_t base) {
  if (n == 0) return 0;
  const oracle_plan* plan = e->plan;
  int64_t nf = plan->n_chunks_fine;
  chunk_arrays(s, nf + 1);
  memset(s->counts, 0, (size_t)nf * sizeof(int64_t));
  for (int64_t t = 0; t < n; ++t) {
    int64_t ch = cols[t] >> plan->shift_fine;
    if (ch >= nf || cols[t] < 0) { e->err = 2; return 0; }
    s->counts[ch]++;
  }
  s->offsets[0] = 0;
  for (int64_t c = 0; c < nf; ++c) s->offsets[c + 1] = s->offsets[c] + s->counts[c];
  memcpy(s->heads, s->offsets, (size_t)nf * sizeof(int64_t));
  int64_t* colf = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  double* valf = e->numeric ? (double*)malloc((size_t)n * sizeof(double)) : NULL;
  for (int64_t t = 0; t < n; ++t) {                      /* stable_scatter_positions matrix.py:187-204 */
    int64_t ch = cols[t] >> plan->shift_fine;
    int64_t p = s->heads[ch]++;
    colf[p] = cols[t] & (plan->chunk_len_fine - 1);
    if (valf) valf[p] = vals[t];
  }
  int64_t* offs = (int64_t*)malloc((size_t)(nf + 1) * sizeof(int64_t));
  memcpy(offs, s->offsets, (size_t)(nf + 1) * sizeof(int64_t));
  int64_t r = accumulate_chunks(s, e, colf, valf, offs, base);
  free(colf); free(valf); free(offs);
  return r;
}

/* fine_level_row magnus.py:224-262: two passes over the referenced B rows */
static int64_t fine_level_row(scratch_t* s, emit_t* e, const oracle_csr* A, const oracle_csr* B, int64_t row) {
  const oracle_plan* plan = e->plan;
  int64_t a0 = A->row_ptr[row], a1 = A->row_ptr[row + 1];
  if (a0 == a1) return 0;
  int64_t nf = plan->n_chunks_fine, cl = plan->chunk_len_fine;
  chunk_arrays(s, nf + 1);
  memset(s->counts, 0, (size_t)nf * sizeof(int64_t));
  for (int64_t t = a0; t < a1; ++t) {                    /* pass 1: histogram :241-247 */
    int64_t k = A->col[t];
    for (int64_t p = B->row_ptr[k]; p < B->row_ptr[k + 1]; ++p) {
      int64_t ch = (int64_t)B->col[p] >> plan->shift_fine;
      if (ch >= nf) { e->err = 2; return 0; }
      s->counts[ch]++;
    }
  }
  s->offsets[0] = 0;
  for (int64_t c = 0; c < nf; ++c) s->offsets[c + 1] = s->offsets[c] + s->counts[c];
  int64_t total = s->offsets[nf];
  if (total == 0) return 0;
  GROW(s->colf, s->f_cap, total, int64_t);
  if (e->numeric) { free(s->valf); s->valf = (double*)malloc((size_t)total * sizeof(double)); }
  memcpy(s->heads, s->offsets, (size_t)nf * sizeof(int64_t));
  for (int64_t t = a0; t < a1; ++t) {                    /* pass 2: stable scatter :255-261 */
    int64_t k = A->col[t];
    double av = A->val[t];
    for (int64_t p = B->row_ptr[k]; p < B->row_ptr[k + 1]; ++p) {
      int64_t c = B->col[p];
      int64_t q = s->heads[c >> plan->shift_fine]++;
      s->colf[q] = c & (cl - 1);
      if (e->numeric) s->valf[q] = av * B->val[p];
    }
  }
  int64_t* offs = (int64_t*)malloc((size_t)(nf + 1) * sizeof(int64_t));
  memcpy(offs, s->offsets, (size_t)(nf + 1) * sizeof(int64_t));
  int64_t r = accumulate_chunks(s, e, s->colf, e->numeric ? s->valf : NULL, offs, 0);
  free(offs);
  return r;
}

/* gather_row_product gustavson.py:44-59 (Gustavson order) */
static int64_t gather_row(const oracle_csr* A, const oracle_csr* B, int64_t i, int64_t* cols, double* vals) {
  int64_t m = 0;
  for (int64_t t = A->row_ptr[i]; t < A->row_ptr[i + 1]; ++t) {
    int64_t k = A->col[t];
    double av = A->val[t];
    for (int64_t p = B->row_ptr[k]; p < B->row_ptr[k + 1]; ++p) {
      cols[m] = B->col[p];
      if (vals) vals[m] = B->val[p] * av;
      ++m;
    }
  }
  return m;
}

/* build_coarse_batches magnus.py:277-314.  Returns number of batches; batch
 * boundaries (indices into coarse_rows) in *bounds (size nb+1). */
static int build_coarse_batches(const int64_t* rows, int64_t n, const int64_t* inter, const oracle_plan* plan,
                                const oracle_sys* sys, int64_t bpe, int64_t** bounds_out, int64_t* nb_out) {
  int64_t ncc = plan->n_chunks_coarse, budget = sys->memory_budget_bytes;
  int64_t* bounds = (int64_t*)malloc((size_t)(n + 2) * sizeof(int64_t));
  int64_t nb = 0; bounds[0] = 0;
  int64_t cur_n = 0, cur_bytes = 0, cur_meta = 0;
  for (int64_t t = 0; t < n; ++t) {
    int64_t isz = inter[rows[t]];
    int64_t row_bytes = isz * bpe;
    if (row_bytes > budget) {
      free(bounds);
      char msg[256];
      snprintf(msg, sizeof msg, "row %lld: buffering %lld intermediate elements needs %lld bytes, over the %lld-byte memory budget",
               (long long)rows[t], (long long)isz, (long long)row_bytes, (long long)budget);
      return fail(ORACLE_OVER_BUDGET, msg);
    }
    int64_t row_meta = ncc * sys->histo_type_bytes + (ncc + 1) * sys->prefix_sum_type_bytes +
                       2 * sys->cache_line_bytes * (ncc < isz ? ncc : isz);
    if (cur_n && (cur_bytes + row_bytes > budget || cur_meta + row_meta > sys->l2_bytes)) {
      bounds[++nb] = t; cur_n = 0; cur_bytes = 0; cur_meta = 0;
    }
    cur_n++; cur_bytes += row_bytes; cur_meta += row_meta;
  }
  if (cur_n) bounds[++nb] = n;
  *bounds_out = bounds; *nb_out = nb;
  return ORACLE_OK;
}

/* build_coarse_chunks magnus.py:317-376 + coarse_level_batch :379-406.
 * csr_rows_to_csc (matrix.py:153-184) restated as a counting sort over the
 * batch rows; B rows visited ascending, A rows inner, B columns innermost. */
static int coarse_level_batch(scratch_t* s, emit_t* e, const oracle_csr* A, const oracle_csr* B,
                              const int64_t* brows, int64_t nbr, int64_t* counts_out, const int64_t* row_ptr_c) {
  const oracle_plan* plan = e->plan;
  int64_t ncc = plan->n_chunks_coarse, clc = plan->chunk_len_coarse;
  /* CSC of the batch (csr_rows_to_csc): col_ptr over B rows */
  int64_t nnz = 0;
  for (int64_t t = 0; t < nbr; ++t) nnz += A->row_ptr[brows[t] + 1] - A->row_ptr[brows[t]];
  int64_t* cptr = (int64_t*)calloc((size_t)(A->n_cols + 1), sizeof(int64_t));
  int64_t* crow = (int64_t*)malloc((size_t)(nnz + 1) * sizeof(int64_t));
  double* cval = (double*)malloc((size_t)(nnz + 1) * sizeof(double));
  for (int64_t t = 0; t < nbr; ++t)
    for (int64_t j = A->row_ptr[brows[t]]; j < A->row_ptr[brows[t] + 1]; ++j) cptr[A->col[j] + 1]++;
  for (int64_t c = 0; c < A->n_cols; ++c) cptr[c + 1] += cptr[c];
  int64_t* head = (int64_t*)malloc((size_t)(A->n_cols + 1) * sizeof(int64_t));
  memcpy(head, cptr, (size_t)(A->n_cols + 1) * sizeof(int64_t));
  for (int64_t t = 0; t < nbr; ++t)
    for (int64_t j = A->row_ptr[brows[t]]; j < A->row_ptr[brows[t] + 1]; ++j) {
      int64_t q = head[A->col[j]]++;
      crow[q] = t; cval[q] = A->val[j];
    }
  free(head);
  /* histogram over (local row, coarse chunk) :332-342 */
  int64_t nbk = nbr * ncc;
  int64_t* cnt = (int64_t*)calloc((size_t)nbk + 1, sizeof(int64_t));
  for (int64_t k = 0; k < A->n_cols; ++k) {
    if (cptr[k] == cptr[k + 1]) continue;
    for (int64_t p = B->row_ptr[k]; p < B->row_ptr[k + 1]; ++p) {
      int64_t ch = (int64_t)B->col[p] >> plan->shift_coarse;
      if (ch >= ncc) { e->err = 2; goto out; }
      for (int64_t q = cptr[k]; q < cptr[k + 1]; ++q) cnt[crow[q] * ncc + ch]++;
    }
  }
  {
    int64_t* off = (int64_t*)malloc((size_t)(nbk + 1) * sizeof(int64_t));   /* row-linked flat cumsum :344-345 */
    off[0] = 0;
    for (int64_t b = 0; b < nbk; ++b) off[b + 1] = off[b] + cnt[b];
    int64_t total = off[nbk];
    int64_t* colc = (int64_t*)malloc((size_t)(total + 1) * sizeof(int64_t));
    double* valc = e->numeric ? (double*)malloc((size_t)(total + 1) * sizeof(double)) : NULL;
    int64_t* hd = (int64_t*)malloc((size_t)(nbk + 1) * sizeof(int64_t));
    memcpy(hd, off, (size_t)(nbk + 1) * sizeof(int64_t));
    for (int64_t k = 0; k < A->n_cols; ++k) {                               /* stable scatter :350-363 */
      if (cptr[k] == cptr[k + 1]) continue;
      for (int64_t q = cptr[k]; q < cptr[k + 1]; ++q) {
        int64_t lr = crow[q];
        for (int64_t p = B->row_ptr[k]; p < B->row_ptr[k + 1]; ++p) {
          int64_t c = B->col[p];
          int64_t dst = hd[lr * ncc + (c >> plan->shift_coarse)]++;
          colc[dst] = c & (clc - 1);
          if (valc) valc[dst] = cval[q] * B->val[p];
        }
      }
    }
    free(hd);
    /* depth-first fine level per (row, coarse chunk) :392-405 */
    for (int64_t li = 0; li < nbr; ++li) {
      int64_t r = brows[li];
      if (e->numeric) { e->pos = row_ptr_c[r]; e->end = row_ptr_c[r + 1]; }
      int64_t c = 0;
      for (int64_t j = 0; j < ncc; ++j) {
        int64_t st = off[li * ncc + j], en = off[li * ncc + j + 1];
        if (st == en) continue;
        c += fine_level_chunk(s, e, colc + st, valc ? valc + st : NULL, en - st, j * clc);
      }
      counts_out[li] = c;
      if (e->numeric && e->pos != e->end) e->err = 2;
    }
    free(off); free(colc); free(valc);
  }
out:
  free(cptr); free(crow); free(cval); free(cnt);
  return e->err ? fail(ORACLE_CONTRACT, "coarse level contract violation") : ORACLE_OK;
}

/* categorize_rows magnus.py:68-94 (first match wins) */
static void categorize(const int64_t* inter, const int64_t* mn, const int64_t* mx, int64_t n, const oracle_plan* plan_sym,
                       const oracle_sys* sys, const oracle_thresholds* th, int8_t* cat) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t range = mx[i] - mn[i] + 1;
    if (inter[i] < th->sort_dense_crossover) cat[i] = ORACLE_CAT_SORT;
    else if (range * (sys->val_bytes + 1) <= sys->l2_bytes) cat[i] = ORACLE_CAT_DENSE;
    else cat[i] = plan_sym->use_coarse ? ORACLE_CAT_COARSE : ORACLE_CAT_FINE;
  }
}

typedef struct {
  int64_t *inter, *mn, *mx; int8_t* cat;
  oracle_plan plan_sym, plan_num;
  int64_t* rows[4]; int64_t nrows[4];
} setup_t;

static void setup_free(setup_t* st) {
  free(st->inter); free(st->mn); free(st->mx); free(st->cat);
  for (int c = 0; c < 4; ++c) free(st->rows[c]);
}

static int setup(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                 int force_fine_only, setup_t* st) {
  memset(st, 0, sizeof *st);
  if (A->n_cols != B->n_rows) return fail(ORACLE_INPUT, "dimension mismatch");   /* _check_dims gustavson.py:39-41 */
  int64_t n = A->n_rows;
  st->inter = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  st->mn = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  st->mx = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  st->cat = (int8_t*)malloc((size_t)(n + 1));
  row_stats(A, B, st->inter, st->mn, st->mx);
  int64_t m_c = B->n_cols > 1 ? B->n_cols : 1;                                   /* magnus.py:565 */
  int rc = oracle_compute_chunk_plan(sys, m_c, 0, !force_fine_only, &st->plan_sym);
  if (rc) return rc;
  rc = oracle_compute_chunk_plan(sys, m_c, 1, !force_fine_only, &st->plan_num);
  if (rc) return rc;
  categorize(st->inter, st->mn, st->mx, n, &st->plan_sym, sys, th, st->cat);
  for (int c = 0; c < 4; ++c) { st->rows[c] = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t)); st->nrows[c] = 0; }
  for (int64_t i = 0; i < n; ++i) { int c = st->cat[i]; st->rows[c][st->nrows[c]++] = i; }
  return ORACLE_OK;
}

static int64_t coarse_bpe(const oracle_csr* B, const oracle_sys* sys) {          /* magnus.py:414-417 */
  return (B->n_cols <= ((int64_t)1 << 32) ? 4 : 8) + sys->val_bytes;
}

/* magnus_symbolic magnus.py:420-456 and magnus_numeric magnus.py:459-542 */
static int run_phase(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                     setup_t* st, int numeric, int64_t* row_ptr, uint32_t* c_col, double* c_val, int64_t* info, int threads) {
  int64_t n = A->n_rows;
  const oracle_plan* plan = numeric ? &st->plan_num : &st->plan_sym;
  int64_t* counts = NULL;
  if (!numeric) counts = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
  int err = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  /* direct rows: sort then dense (magnus.py:425-433 / :483-503) */
  for (int c = ORACLE_CAT_SORT; c <= ORACLE_CAT_DENSE; ++c) {
    int64_t nr = st->nrows[c];
    const int64_t* rows = st->rows[c];
    #pragma omp parallel
    {
      scratch_t s; memset(&s, 0, sizeof s);
      int64_t* cols = NULL; double* vals = NULL; int64_t cap = 0;
      int64_t* oc = NULL; double* ov = NULL; int64_t ocap = 0;
      #pragma omp for schedule(dynamic, 64)
      for (int64_t t = 0; t < nr; ++t) {
        int64_t r = rows[t];
        int64_t isz = st->inter[r];
        if (isz > cap) { free(cols); free(vals); cap = isz * 2; cols = (int64_t*)malloc((size_t)cap * 8); vals = (double*)malloc((size_t)cap * 8); }
        if (isz > ocap) { free(oc); free(ov); ocap = isz * 2; oc = (int64_t*)malloc((size_t)ocap * 8); ov = (double*)malloc((size_t)ocap * 8); }
        int64_t m = gather_row(A, B, r, cols, numeric ? vals : NULL);
        int64_t got;
        if (c == ORACLE_CAT_SORT) {
          got = sort_accumulate(&s, cols, numeric ? vals : NULL, m, oc, ov);
        } else {
          int64_t mn = st->mn[r];
          int64_t cap_w = ceil_pow2(st->mx[r] - mn + 1 > 1024 ? st->mx[r] - mn + 1 : 1024);   /* window_dense magnus.py:105-109 */
          for (int64_t q = 0; q < m; ++q) cols[q] -= mn;
          int derr = 0;
          got = dense_accumulate(&s, cols, numeric ? vals : NULL, m, cap_w, oc, ov, &derr);
          for (int64_t q = 0; q < got; ++q) oc[q] += mn;
          if (derr) { _Pragma("omp atomic write") err = 2; }
        }
        if (numeric) {                                                        /* write_row magnus.py:474-481 */
          int64_t c0 = row_ptr[r], c1 = row_ptr[r + 1];
          if (got != c1 - c0) { _Pragma("omp atomic write") err = 2; }
          else for (int64_t q = 0; q < got; ++q) { c_col[c0 + q] = (uint32_t)oc[q]; c_val[c0 + q] = ov[q]; }
        } else counts[r] = got;
      }
      free(cols); free(vals); free(oc); free(ov); scratch_free(&s);
    }
  }
  /* fine rows magnus.py:435-441 / :505-515 */
  {
    int64_t nr = st->nrows[ORACLE_CAT_FINE];
    const int64_t* rows = st->rows[ORACLE_CAT_FINE];
    #pragma omp parallel
    {
      scratch_t s; memset(&s, 0, sizeof s);
      emit_t e = {sys, th, plan, c_col, c_val, 0, 0, numeric, 0};
      #pragma omp for schedule(dynamic, 16)
      for (int64_t t = 0; t < nr; ++t) {
        int64_t r = rows[t];
        if (numeric) { e.pos = row_ptr[r]; e.end = row_ptr[r + 1]; }
        int64_t got = fine_level_row(&s, &e, A, B, r);
        if (numeric) { if (e.pos != e.end) e.err = 2; }
        else counts[r] = got;
      }
      if (e.err) { _Pragma("omp atomic write") err = 2; }
      scratch_free(&s);
    }
  }
  /* coarse rows magnus.py:443-452 / :517-534 */
  int64_t n_batches = 0;
  if (st->nrows[ORACLE_CAT_COARSE]) {
    int64_t* bounds = NULL; int64_t nb = 0;
    int rc = build_coarse_batches(st->rows[ORACLE_CAT_COARSE], st->nrows[ORACLE_CAT_COARSE], st->inter, plan, sys,
                                  coarse_bpe(B, sys), &bounds, &nb);
    if (rc) { free(counts); return rc; }
    n_batches = nb;
    const int64_t* rows = st->rows[ORACLE_CAT_COARSE];
    #pragma omp parallel
    {
      scratch_t s; memset(&s, 0, sizeof s);
      emit_t e = {sys, th, plan, c_col, c_val, 0, 0, numeric, 0};
      #pragma omp for schedule(dynamic, 1)
      for (int64_t b = 0; b < nb; ++b) {
        int64_t lo = bounds[b], hi = bounds[b + 1];
        int64_t* cnt = (int64_t*)malloc((size_t)(hi - lo + 1) * sizeof(int64_t));
        coarse_level_batch(&s, &e, A, B, rows + lo, hi - lo, cnt, row_ptr);
        if (!numeric) for (int64_t q = lo; q < hi; ++q) counts[rows[q]] = cnt[q - lo];
        free(cnt);
      }
      if (e.err) { _Pragma("omp atomic write") err = 2; }
      scratch_free(&s);
    }
    free(bounds);
  }
  if (!numeric) {                                                              /* cumsum magnus.py:454-456 */
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + counts[i];
    free(counts);
  }
  if (info) {
    int64_t sum = 0;
    for (int64_t i = 0; i < n; ++i) sum += st->inter[i];
    info[0] = row_ptr[n]; info[1] = sum; info[2] = n_batches;
    for (int c = 0; c < 4; ++c) info[3 + c] = st->nrows[c];
  }
  if (err) return fail(ORACLE_CONTRACT, "numeric phase count differs from the symbolic count");
  return ORACLE_OK;
}

int oracle_symbolic(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                    int force_fine_only, int threads, int64_t* row_ptr, int64_t* info) {
  setup_t st;
  int rc = setup(A, B, sys, th, force_fine_only, &st);
  if (!rc) rc = run_phase(A, B, sys, th, &st, 0, row_ptr, NULL, NULL, info, threads);
  setup_free(&st);
  return rc;
}

int oracle_numeric(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                   int force_fine_only, int threads, const int64_t* row_ptr, uint32_t* c_col, double* c_val, int64_t* info) {
  setup_t st;
  int rc = setup(A, B, sys, th, force_fine_only, &st);
  if (!rc) {
    if (row_ptr[0] != 0) rc = fail(ORACLE_CONTRACT, "row_ptr does not come from a symbolic pass of (A, B)");
    else rc = run_phase(A, B, sys, th, &st, 1, (int64_t*)row_ptr, c_col, c_val, info, threads);
  }
  setup_free(&st);
  return rc;
}

/* row_intermediate_stats + categorize_rows exposed for host-logic tests */
int oracle_setup(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                 int force_fine_only, int64_t* inter, int64_t* mn, int64_t* mx, int8_t* cat) {
  setup_t st;
  int rc = setup(A, B, sys, th, force_fine_only, &st);
  if (!rc) {
    memcpy(inter, st.inter, (size_t)A->n_rows * 8); memcpy(mn, st.mn, (size_t)A->n_rows * 8);
    memcpy(mx, st.mx, (size_t)A->n_rows * 8); memcpy(cat, st.cat, (size_t)A->n_rows);
  }
  setup_free(&st);
  return rc;
}

double oracle_pairwise_sum(const double* a, int64_t n) { return pairwise_sum(a, n); }

/* --------------------------------------------------------- Gustavson baselines */
/* gustavson_dense_symbolic gustavson.py:155-170 (np.unique of the row's product),
 * gustavson_dense_numeric gustavson.py:184-220 (DenseAccumulator over all n_cols:
 * sequential from +0.0 in Gustavson order, then canonicalize_csr sorts the row),
 * gustavson_esc_numeric gustavson.py:223-250 (sort_accumulate: x0 + pairwise(rest)).
 * phase 0: row_ptr (n+1) out.  phase 1 (dense) / 2 (esc): col/val filled for row_ptr. */
int oracle_gustavson(const oracle_csr* A, const oracle_csr* B, int phase, int threads, int64_t* row_ptr, uint32_t* c_col,
                     double* c_val) {
  if (A->n_cols != B->n_rows) return fail(ORACLE_INPUT, "dimension mismatch");
  const int64_t n = A->n_rows;
  if (phase && row_ptr[0] != 0) return fail(ORACLE_CONTRACT, "row_ptr does not come from a symbolic pass of (A, B)");
  int64_t* counts = phase ? NULL : (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
  int err = 0;
  if (threads > 0) omp_set_num_threads(threads);
  #pragma omp parallel
  {
    scratch_t s;
    memset(&s, 0, sizeof s);
    int64_t cap = 0;
    int64_t* cols = NULL; double* vals = NULL; int64_t* oc = NULL; double* ov = NULL;
    #pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
      int64_t m = 0;
      for (int64_t t = A->row_ptr[i]; t < A->row_ptr[i + 1]; ++t) m += B->row_ptr[A->col[t] + 1] - B->row_ptr[A->col[t]];
      if (m > cap) {
        cap = m * 2 + 16;
        cols = (int64_t*)realloc(cols, (size_t)cap * 8); vals = (double*)realloc(vals, (size_t)cap * 8);
        oc = (int64_t*)realloc(oc, (size_t)cap * 8); ov = (double*)realloc(ov, (size_t)cap * 8);
      }
      gather_row(A, B, i, cols, phase ? vals : NULL);
      int derr = 0;
      int64_t got;
      if (phase == 2) got = sort_accumulate(&s, cols, vals, m, oc, ov);
      else got = dense_accumulate(&s, cols, phase ? vals : NULL, m, B->n_cols > 0 ? B->n_cols : 1, phase ? oc : NULL,
                                  phase ? ov : NULL, &derr);
      if (!phase) { counts[i] = got; continue; }
      if (derr || got != row_ptr[i + 1] - row_ptr[i]) { _Pragma("omp atomic write") err = 1; continue; }
      for (int64_t t = 0; t < got; ++t) { c_col[row_ptr[i] + t] = (uint32_t)oc[t]; c_val[row_ptr[i] + t] = ov[t]; }
    }
    free(cols); free(vals); free(oc); free(ov);
    scratch_free(&s);
  }
  if (!phase) {
    row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + counts[i];
    free(counts);
  }
  if (err) return fail(ORACLE_CONTRACT, "numeric phase count differs from the symbolic count");
  return ORACLE_OK;
}
