/* TEST INFRASTRUCTURE ONLY -- second, independent restatement of the counting path, used by the
 * full-size parity tests (tests/test_gpu_fullsize.py) where the level-wise radix port
 * (radix_oracle.c) would take minutes.  Never linked into the product library.
 *
 * oracle_dense_tables: the reference's joint-key convention (baselines.py:51-57,
 *   key = s_0 + r_0 * s_1 + r_0 r_1 * s_2 ..., target first) counted straight into a dense
 *   table -- hash_query (baselines.py:77-89) with an array in place of the dict -- then
 *   LogLikelihood (aggregators.py:147-157: sum x ln(x / n_ij) over non-zero cells), the
 *   survey 8(a) MI definition and the non-zero count (NullSink).
 * oracle_itemset_enum: supports of every 2- and 3-subset of a list of binary items, counted
 *   record by record (each record adds 1 to every subset of the items it holds) -- the
 *   definition oracle_count (oracle.py:59-65) evaluates, organised per record instead of per
 *   itemset.
 *
 * Both are pinned against the golden vectors and the radix / bitmap ports by
 * tests/test_oracle_golden.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const uint8_t* cols;
  int64_t ld, m;
  const int32_t* arity;
  int32_t nq;
  const int32_t *var_off, *vars;
  const int64_t* table_off;
  uint32_t* tables;
  double *loglik, *mi;
  int64_t* nnz;
  int32_t next;
  pthread_mutex_t mu;
  int err;
} dense_job;

enum { BLK = 4096 };

static void dense_one(const dense_job* J, int32_t q, uint32_t* tab, int64_t cells) {
  const int32_t o = J->var_off[q], k = J->var_off[q + 1] - o;
  const int32_t* v = J->vars + o;
  int64_t stride[64];
  int64_t s = 1;
  for (int t = 0; t < k && t < 64; ++t) {
    stride[t] = s;
    s *= J->arity[v[t]];
  }
  memset(tab, 0, sizeof(uint32_t) * (size_t)cells);
  /* rows in blocks: the key of a block is accumulated column by column (sequential reads) */
  uint32_t key[BLK];
  for (int64_t r0 = 0; r0 < J->m; r0 += BLK) {
    const int64_t nb = J->m - r0 < BLK ? J->m - r0 : BLK;
    const uint8_t* c0 = J->cols + (int64_t)v[0] * J->ld + r0;
    for (int64_t i = 0; i < nb; ++i) key[i] = c0[i];
    for (int t = 1; t < k; ++t) {
      const uint8_t* c = J->cols + (int64_t)v[t] * J->ld + r0;
      const uint32_t st = (uint32_t)stride[t];
      for (int64_t i = 0; i < nb; ++i) key[i] += (uint32_t)c[i] * st;
    }
    for (int64_t i = 0; i < nb; ++i) tab[key[i]]++;
  }
  const int rt = J->arity[v[0]];
  const int64_t J_cfg = cells / rt;
  double ll = 0.0;
  int64_t nz = 0;
  /* target marginals for MI */
  int64_t nk[256];
  memset(nk, 0, sizeof nk);
  for (int64_t c = 0; c < cells; ++c) nk[c % rt] += tab[c];
  double mi = 0.0;
  const double m = (double)J->m;
  for (int64_t j = 0; j < J_cfg; ++j) {
    int64_t nij = 0;
    for (int kk = 0; kk < rt; ++kk) nij += tab[j * rt + kk];
    if (!nij) continue;
    for (int kk = 0; kk < rt; ++kk) {
      const uint32_t x = tab[j * rt + kk];
      if (!x) continue;
      ++nz;
      const double xd = (double)x;
      ll += xd * log(xd / (double)nij);
      mi += (xd / m) * log(m * xd / ((double)nij * (double)nk[kk]));
    }
  }
  if (J->loglik) J->loglik[q] = ll;
  if (J->mi) J->mi[q] = mi;
  if (J->nnz) J->nnz[q] = nz;
}

static void* dense_worker(void* arg) {
  dense_job* J = (dense_job*)arg;
  uint32_t* own = NULL;
  int64_t own_cells = 0;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const int32_t q = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (q >= J->nq) break;
    const int32_t o = J->var_off[q], k = J->var_off[q + 1] - o;
    int64_t cells = 1;
    for (int t = 0; t < k; ++t) cells *= J->arity[J->vars[o + t]];
    uint32_t* tab;
    if (J->tables) {
      tab = J->tables + J->table_off[q];
    } else {
      if (cells > own_cells) {
        free(own);
        own = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)cells);
        own_cells = own ? cells : 0;
        if (!own) {
          J->err = -3;
          break;
        }
      }
      tab = own;
    }
    dense_one(J, q, tab, cells);
  }
  free(own);
  return NULL;
}

/* Dense tables (optional), LL, MI and non-zero counts for nq queries over n x ld uint8 columns
 * (rows [0, m)).  Joint state spaces must fit 32-bit keys (< 2^32 cells). */
int oracle_dense_tables(const uint8_t* cols, int64_t ld, int64_t m, const int32_t* arity, int32_t nq,
                        const int32_t* var_off, const int32_t* vars, const int64_t* table_off,
                        uint32_t* tables, double* loglik, double* mi, int64_t* nnz, int32_t nthreads) {
  for (int32_t q = 0; q < nq; ++q) {
    int64_t c = 1;
    for (int32_t i = var_off[q]; i < var_off[q + 1]; ++i) c *= arity[vars[i]];
    if (c >= ((int64_t)1 << 32) || var_off[q + 1] - var_off[q] > 64) return -1;
  }
  dense_job J = {cols, ld, m, arity, nq, var_off, vars, table_off, tables, loglik, mi, nnz, 0,
                 PTHREAD_MUTEX_INITIALIZER, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, dense_worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return J.err;
}

/* ---------------------------------------------------------------------------------------- */

typedef struct {
  const uint8_t* cols; /* nitems x ld, one column per item (state 1 = present) */
  int64_t ld, m;
  int32_t n;
  const int64_t* off2; /* n x n: combinations index of (a, b, b + 1) */
  int64_t ntri;
  int64_t *pairs, *triples; /* shared outputs (n x n, ntri) */
  int32_t nthreads, tid_next;
  pthread_mutex_t mu;
  int err;
} enum_job;

static void* enum_worker(void* arg) {
  enum_job* J = (enum_job*)arg;
  pthread_mutex_lock(&J->mu);
  const int tid = J->tid_next++;
  pthread_mutex_unlock(&J->mu);
  const int n = J->n;
  const int64_t r0 = J->m * tid / J->nthreads, r1 = J->m * (tid + 1) / J->nthreads;
  uint32_t* tri = (uint32_t*)calloc((size_t)(J->ntri > 0 ? J->ntri : 1), sizeof(uint32_t));
  uint64_t* pr = (uint64_t*)calloc((size_t)n * n, sizeof(uint64_t));
  const int W = (n + 63) / 64;
  uint64_t* mask = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)BLK * W);
  if (!tri || !pr || !mask) {
    J->err = -3;
    free(tri);
    free(pr);
    free(mask);
    return NULL;
  }
  int32_t list[4096];
  for (int64_t b0 = r0; b0 < r1; b0 += BLK) {
    const int64_t nb = r1 - b0 < BLK ? r1 - b0 : BLK;
    memset(mask, 0, sizeof(uint64_t) * (size_t)BLK * W);
    for (int i = 0; i < n; ++i) {
      const uint8_t* c = J->cols + (int64_t)i * J->ld + b0;
      const uint64_t bit = 1ull << (i & 63);
      uint64_t* mw = mask + (i >> 6);
      for (int64_t r = 0; r < nb; ++r)
        if (c[r] == 1) mw[r * W] |= bit;
    }
    for (int64_t r = 0; r < nb; ++r) {
      int cnt = 0;
      for (int w = 0; w < W; ++w) {
        uint64_t x = mask[r * W + w];
        while (x) {
          list[cnt++] = w * 64 + __builtin_ctzll(x);
          x &= x - 1;
        }
      }
      for (int a = 0; a < cnt; ++a)
        for (int b = a + 1; b < cnt; ++b) {
          const int ia = list[a], ib = list[b];
          pr[(int64_t)ia * n + ib]++;
          const int64_t base = J->off2[(int64_t)ia * n + ib] - ib - 1;
          for (int c = b + 1; c < cnt; ++c) tri[base + list[c]]++;
        }
    }
  }
  pthread_mutex_lock(&J->mu);
  for (int64_t t = 0; t < J->ntri; ++t) J->triples[t] += tri[t];
  for (int64_t t = 0; t < (int64_t)n * n; ++t) J->pairs[t] += (int64_t)pr[t];
  pthread_mutex_unlock(&J->mu);
  free(tri);
  free(pr);
  free(mask);
  return NULL;
}

/* pairs[a * n + b] (a < b) and triples (itertools.combinations order of positions) of the
 * n item columns; outputs zeroed by the caller.  n <= 4096. */
int oracle_itemset_enum(const uint8_t* cols, int64_t ld, int64_t m, int32_t n, int64_t* pairs,
                        int64_t* triples, int32_t nthreads) {
  if (n < 0 || n > 4096) return -1;
  const int64_t ntri = (int64_t)n * (n - 1) * (n - 2) / 6;
  int64_t* off2 = (int64_t*)calloc((size_t)n * n + 1, sizeof(int64_t));
  if (!off2) return -3;
  int64_t idx = 0;
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b) {
      off2[(int64_t)a * n + b] = idx;
      idx += n - 1 - b;
    }
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  enum_job J = {cols, ld, m, n, off2, ntri, pairs, triples, nthreads, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, enum_worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(off2);
  return J.err;
}
