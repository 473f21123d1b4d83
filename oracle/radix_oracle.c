/*
 * radix_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline), never the
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.
 *
 * A C restatement of the reference's fastest CPU counting path, the level-wise MSD radix
 * partition of countstream (reference pkg/src/countstream/radix.py):
 *   - partition_level   <- _partition_level (radix.py:33-79): per-segment counting sort of
 *                          row ids on one column, empty buckets dropped, singleton segments
 *                          harvested instead of re-partitioned;
 *   - radix_query_one   <- radix_query (radix.py:113-156): parents in the given order, then
 *                          the target; N_ij from the parent bucket of each target bucket
 *                          (:130-137); harvested singletons contribute (1, 1) cells (:154-156);
 *   - LL accumulation   <- LogLikelihood.accept_block (aggregators.py:147-157);
 *   - bitmap pack/count <- bitmap._pack / bitmap_count (bitmap.py:29-31, 131-136).
 * The reference streams cells into an aggregator; this restatement writes each cell into a
 * dense table at the mixed-radix index of baselines._config_keys (baselines.py:51-57) with
 * the target as least significant digit, so GPU tables can be compared cell by cell.
 * Multi-threaded over queries with pthreads (the reference is single-core; the CPU
 * baseline states the thread count it used).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t *rows, *spare;      /* row ids of the live buckets, packed */
  int64_t *starts, *sstarts;  /* bucket boundaries (nb + 1) */
  int32_t *finished;          /* harvested singleton rows */
  int64_t nb, nf, m;
  int64_t local[256];
} level_buf;

static int lb_init(level_buf* b, int64_t m) {
  b->m = m;
  b->rows = malloc(sizeof(int32_t) * (size_t)m);
  b->spare = malloc(sizeof(int32_t) * (size_t)m);
  b->starts = malloc(sizeof(int64_t) * (size_t)(m + 1));
  b->sstarts = malloc(sizeof(int64_t) * (size_t)(m + 1));
  b->finished = malloc(sizeof(int32_t) * (size_t)m);
  return b->rows && b->spare && b->starts && b->sstarts && b->finished ? 0 : -1;
}

static void lb_free(level_buf* b) {
  free(b->rows);
  free(b->spare);
  free(b->starts);
  free(b->sstarts);
  free(b->finished);
}

static void lb_reset(level_buf* b) {
  for (int64_t i = 0; i < b->m; ++i) b->rows[i] = (int32_t)i;
  b->starts[0] = 0;
  b->starts[1] = b->m;
  b->nb = 1;
  b->nf = 0;
}

/* one counting-sort level over every live segment (radix.py:33-79) */
static void partition_level(level_buf* b, const uint8_t* col, int r) {
  int64_t nb_out = 0, out = 0;
  b->sstarts[0] = 0;
  for (int64_t s = 0; s < b->nb; ++s) {
    const int64_t lo = b->starts[s], hi = b->starts[s + 1];
    if (hi - lo == 1) { /* singleton: harvest (radix.py:57-60) */
      b->finished[b->nf++] = b->rows[lo];
      continue;
    }
    for (int j = 0; j < r; ++j) b->local[j] = 0;
    for (int64_t p = lo; p < hi; ++p) b->local[col[b->rows[p]]]++;
    int64_t acc = out;
    for (int j = 0; j < r; ++j) {
      const int64_t c = b->local[j];
      if (c > 0) b->sstarts[++nb_out] = acc + c;
      b->local[j] = acc;
      acc += c;
    }
    for (int64_t p = lo; p < hi; ++p) {
      const int k = col[b->rows[p]];
      b->spare[b->local[k]++] = b->rows[p];
    }
    out += hi - lo;
  }
  int32_t* t = b->rows;
  b->rows = b->spare;
  b->spare = t;
  int64_t* u = b->starts;
  b->starts = b->sstarts;
  b->sstarts = u;
  b->nb = nb_out;
}

static uint64_t cell_of_row(const uint8_t* cols, int64_t ld, const int32_t* v, const int64_t* stride,
                            int k, int64_t row) {
  uint64_t idx = 0;
  for (int t = 0; t < k; ++t) idx += (uint64_t)cols[(int64_t)v[t] * ld + row] * (uint64_t)stride[t];
  return idx;
}

/* radix_query (radix.py:113-156) for one query: vars[0] = target, vars[1..] = parents */
static void radix_query_one(level_buf* b, const uint8_t* cols, int64_t ld, const int32_t* arity,
                            const int32_t* v, int k, uint32_t* table, double* ll, int64_t* nnz) {
  int64_t stride[64];
  int64_t s = 1;
  for (int t = 0; t < k && t < 64; ++t) {
    stride[t] = s;
    s *= arity[v[t]];
  }
  lb_reset(b);
  for (int t = 1; t < k; ++t) partition_level(b, cols + (int64_t)v[t] * ld, arity[v[t]]);
  /* parent bucket sizes before the target level (radix.py:130) */
  const int64_t np = b->nb;
  int64_t* psize = malloc(sizeof(int64_t) * (size_t)(np > 0 ? np : 1));
  for (int64_t j = 0; j < np; ++j) psize[j] = b->starts[j + 1] - b->starts[j];
  /* target level: remember which parent bucket each child came from */
  const int rt = arity[v[0]];
  const uint8_t* tc = cols + (int64_t)v[0] * ld;
  int64_t* parent_of = malloc(sizeof(int64_t) * (size_t)(b->m + 1));
  {
    int64_t nb_out = 0, out = 0;
    b->sstarts[0] = 0;
    for (int64_t sg = 0; sg < b->nb; ++sg) {
      const int64_t lo = b->starts[sg], hi = b->starts[sg + 1];
      if (hi - lo == 1) {
        b->finished[b->nf++] = b->rows[lo];
        continue;
      }
      for (int j = 0; j < rt; ++j) b->local[j] = 0;
      for (int64_t p = lo; p < hi; ++p) b->local[tc[b->rows[p]]]++;
      int64_t acc = out;
      for (int j = 0; j < rt; ++j) {
        const int64_t c = b->local[j];
        if (c > 0) {
          parent_of[nb_out] = sg;
          b->sstarts[++nb_out] = acc + c;
        }
        b->local[j] = acc;
        acc += c;
      }
      for (int64_t p = lo; p < hi; ++p) {
        const int kk = tc[b->rows[p]];
        b->spare[b->local[kk]++] = b->rows[p];
      }
      out += hi - lo;
    }
    int32_t* t = b->rows;
    b->rows = b->spare;
    b->spare = t;
    int64_t* u = b->starts;
    b->starts = b->sstarts;
    b->sstarts = u;
    b->nb = nb_out;
  }
  double total = 0.0;
  int64_t cnt = 0;
  for (int64_t c = 0; c < b->nb; ++c) {
    const int64_t n_ijk = b->starts[c + 1] - b->starts[c];
    const int64_t n_ij = psize[parent_of[c]];
    const uint64_t idx = cell_of_row(cols, ld, v, stride, k, b->rows[b->starts[c]]);
    if (table) table[idx] = (uint32_t)n_ijk;
    const double x = (double)n_ijk;
    total += x * log(x / (double)n_ij);
    ++cnt;
  }
  for (int64_t f = 0; f < b->nf; ++f) { /* harvested singletons: (1, 1) cells, ln 1 = 0 */
    const uint64_t idx = cell_of_row(cols, ld, v, stride, k, b->finished[f]);
    if (table) table[idx] = 1u;
    ++cnt;
  }
  free(psize);
  free(parent_of);
  if (ll) *ll = total;
  if (nnz) *nnz = cnt;
}

typedef struct {
  const uint8_t* cols;
  int64_t ld, m;
  const int32_t* arity;
  int32_t nq;
  const int32_t *var_off, *vars;
  const int64_t* table_off;
  uint32_t* tables;
  double* loglik;
  int64_t* nnz;
  int32_t next;
  pthread_mutex_t mu;
  int err;
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  level_buf b;
  if (lb_init(&b, J->m) != 0) {
    J->err = -3;
    lb_free(&b);
    return NULL;
  }
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int32_t q = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (q >= J->nq) break;
    const int32_t o = J->var_off[q], k = J->var_off[q + 1] - o;
    radix_query_one(&b, J->cols, J->ld, J->arity, J->vars + o, k,
                    J->tables ? J->tables + J->table_off[q] : NULL, J->loglik ? J->loglik + q : NULL,
                    J->nnz ? J->nnz + q : NULL);
  }
  lb_free(&b);
  return NULL;
}

/* Dense tables (zeroed by the caller), LL and non-zero counts for nq queries.
 * cols: n x ld uint8 variable-major.  Returns 0 or a negative error. */
int oracle_radix_tables(const uint8_t* cols, int64_t ld, int64_t m, const int32_t* arity, int32_t nq,
                        const int32_t* var_off, const int32_t* vars, const int64_t* table_off,
                        uint32_t* tables, double* loglik, int64_t* nnz, int32_t nthreads) {
  if (m >= ((int64_t)1 << 31)) return -1;
  job_t J = {cols, ld, m, arity, nq, var_off, vars, table_off, tables, loglik, nnz, 0,
             PTHREAD_MUTEX_INITIALIZER, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return J.err;
}

/* bitmap._pack (bitmap.py:29-31): bit t of word t/32 = (col[t] == state) */
void oracle_bitmap_pack(const uint8_t* col, int64_t m, int32_t state, uint32_t* words) {
  const int64_t nw = (m + 31) / 32;
  memset(words, 0, sizeof(uint32_t) * (size_t)nw);
  for (int64_t t = 0; t < m; ++t)
    if (col[t] == (uint8_t)state) words[t >> 5] |= 1u << (t & 31);
}

typedef struct {
  const uint32_t* const* planes; /* per query item lists flattened */
  const int32_t* off;
  int64_t nwords, m;
  int32_t nq;
  int64_t* counts;
  int32_t next;
  pthread_mutex_t mu;
} cnt_job;

static void* cnt_worker(void* arg) {
  cnt_job* J = (cnt_job*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int32_t q = J->next;
    J->next += 64;
    pthread_mutex_unlock(&J->mu);
    if (q >= J->nq) break;
    const int32_t qe = q + 64 < J->nq ? q + 64 : J->nq;
    for (int32_t i = q; i < qe; ++i) {
      const int32_t b = J->off[i], k = J->off[i + 1] - b;
      if (k == 0) {
        J->counts[i] = J->m;
        continue;
      }
      int64_t c = 0;
      for (int64_t w = 0; w < J->nwords; ++w) {
        uint32_t x = J->planes[b][w];
        for (int j = 1; j < k; ++j) x &= J->planes[b + j][w];
        c += __builtin_popcount(x);
      }
      J->counts[i] = c;
    }
  }
  return NULL;
}

/* bitmap_count (bitmap.py:131-136) for nq assignments given as plane pointer lists */
int oracle_bitmap_counts(const uint32_t* const* planes, const int32_t* off, int32_t nq, int64_t nwords,
                         int64_t m, int64_t* counts, int32_t nthreads) {
  cnt_job J = {planes, off, nwords, m, nq, counts, 0, PTHREAD_MUTEX_INITIALIZER};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, cnt_worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}
