// cs_kernels.cuh -- sm_100a kernels of the counting-query engine.
//
//   K1 k_hist          batched joint histogram: persistent CTAs pull (query, row-segment)
//                      work items; 16-row uint4 column loads; mixed-radix joint index in
//                      SIMD byte / 16-bit lanes; SMEM-privatised, lane-replicated uint32
//                      tables (conflict-free ATOMS); fused fp64 score epilogue.
//                      Replaces radix._partition_level / radix_query (radix.py:33-156).
//   K1g k_hist_generic queries with more than CS_MAXK variables (runtime digit loop).
//   K2 k_score         fp64 LL / MI / nnz over merged global tables (aggregators.py:147-157).
//   K3 k_bitmap_build  per-(variable, state) bit planes (bitmap.py:29-66).
//   K4 k_points_*      AND + popcount point counts (bitmap.py:131-136) / byte-scan fallback
//                      when no planes exist (radix.py:181-193 semantics).
//   K5 k_compact       non-zero cell stream (n_ijk, n_ij, cell) for record aggregators.
//      k_generate      counter-based column generator (device twin of oracle/gen_twin.py).
#pragma once
#include "cs_common.cuh"

namespace cs {

// ------------------------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ uint4 ldg_stream16(const uint8_t* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t word_of(const uint4& w, int j) {
  return j == 0 ? w.x : (j == 1 ? w.y : (j == 2 ? w.z : w.w));
}

// block-wide sums; result valid in thread 0.  s_red needs 32 slots.
__device__ __forceinline__ double block_sum(double v, double* s_red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) s_red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (l < (int)(blockDim.x >> 5)) ? s_red[l] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v,
                                                            unsigned long long* s_red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) s_red[w] = v;
  __syncthreads();
  unsigned long long r = 0;
  if (w == 0) {
    r = (l < (int)(blockDim.x >> 5)) ? s_red[l] : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;
}

// ------------------------------------------------------------------------------------------
// fused score epilogue (K2 body).  `cell(c)` returns N for table cell c.  All threads of the
// block must call it.  Follows LogLikelihood.accept_block (aggregators.py:147-157):
//   LL  = sum_{n_ijk > 0} n_ijk * ln(n_ijk / n_ij)
//   MI  = (1/m) sum n_ijk * ln(m * n_ijk / (n_ij * n_k))        (survey 8a, new)
//   nnz = number of non-zero cells (what NullSink counts, aggregators.py:80-93)

struct ScoreSmem {
  unsigned long long marg[CS_MAX_ARITY];
  double red[32];
  unsigned long long redu[32];
};

template <class CellFn>
__device__ void score_table(CellFn cell, uint32_t C, int rt, double m_total, uint32_t flags,
                            int q, double* ll_out, double* mi_out, int64_t* nnz_out,
                            ScoreSmem& ss) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const bool want_mi = (flags & F_MI) != 0;
  if (want_mi) {
    for (int k = tid; k < rt; k += nt) ss.marg[k] = 0ull;
    __syncthreads();
    for (uint32_t c = tid; c < C; c += nt) {
      const uint32_t v = cell(c);
      if (v) atomicAdd(&ss.marg[c % (uint32_t)rt], (unsigned long long)v);
    }
    __syncthreads();
  }
  double ll = 0.0, mi = 0.0;
  unsigned long long nz = 0;
  const uint32_t J = C / (uint32_t)rt;
  for (uint32_t j = tid; j < J; j += nt) {
    const uint32_t base = j * (uint32_t)rt;
    unsigned long long nij = 0;
    for (int k = 0; k < rt; ++k) nij += cell(base + k);
    if (nij == 0) continue;
    const double dnij = (double)nij;
    for (int k = 0; k < rt; ++k) {
      const uint32_t n = cell(base + k);
      if (n) {
        const double x = (double)n;
        ll += (flags & F_NLOGN) ? x * log(x) : x * log(x / dnij);
        ++nz;
        if (want_mi) mi += x * log((x * m_total) / (dnij * (double)ss.marg[k]));
      }
    }
  }
  const double tll = block_sum(ll, ss.red);
  const double tmi = want_mi ? block_sum(mi, ss.red) : 0.0;
  const unsigned long long tnz = block_sum_u64(nz, ss.redu);
  if (tid == 0) {
    if (ll_out) ll_out[q] = tll;
    if (mi_out) mi_out[q] = want_mi ? tmi / m_total : 0.0;
    if (nnz_out) nnz_out[q] = (int64_t)tnz;
  }
}

// ------------------------------------------------------------------------------------------
// K1 inner loop: count rows [r0, r1) of one query.
//
// MODE 0 (C <= 256): every 32-bit word carries 4 rows in byte lanes; digit d contributes
//   word_d * stride_d with no carry between lanes because the running index stays < 256.
// MODE 1 (C <= 65536): leading digits with cumulative product <= 256 are combined in byte
//   lanes, then split into two words of 16-bit lanes (PRMT) for the remaining digits.
// MODE 2: scalar 32-bit index per row.
// SMEM=true : ATOMS into lane-replicated table sh[(idx << rlog) | (lane & (R-1))].
// SMEM=false: RED.ADD into the global table gtab[idx] (tables too large for SMEM).

// SMEM class, C * R * 4 <= 65536: the *byte offset* of each row's replica counter,
// (idx * R + rep) * 4, is built directly in 16-bit SIMD lanes (two rows per 32-bit word):
// digits with cumulative product <= 256 are combined in byte lanes (one IMAD per digit per
// 4 rows), split to 16-bit lanes (2 PRMT), remaining digits added per lane pair, and one
// IMAD per 2 rows applies the x(4R) scale and adds the thread's replica offset.  Each row
// then costs one extract (LOP3/SHF) and one ATOMS.  Rows past the end of the last vector
// read zero padding; they are counted into cell 0 of the thread's replica and subtracted
// once after the loop (no per-row tail predicate).

template <int K>
__device__ __forceinline__ void load_vec16(uint32_t (&x)[K][4], const uint8_t* p,
                                           const uint32_t (&co)[K]) {
#pragma unroll
  for (int v = 0; v < K; ++v) {
    const uint4 t = ldg_stream16(p + ((uint64_t)co[v] << 8));
    x[v][0] = t.x;
    x[v][1] = t.y;
    x[v][2] = t.z;
    x[v][3] = t.w;
  }
}

template <int K>
__device__ __forceinline__ void count_vec16(const uint32_t (&x)[K][4], const uint32_t (&st)[K],
                                            int nbyte, uint32_t scale, uint32_t rep_pair,
                                            char* shb) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t a8 = x[0][j];
#pragma unroll
    for (int v = 1; v < K; ++v)
      if (v < nbyte) a8 += x[v][j] * st[v];
    uint32_t lo = __byte_perm(a8, 0u, 0x4140);
    uint32_t hi = __byte_perm(a8, 0u, 0x4342);
#pragma unroll
    for (int v = 1; v < K; ++v) {
      if (v >= nbyte) {
        lo += __byte_perm(x[v][j], 0u, 0x4140) * st[v];
        hi += __byte_perm(x[v][j], 0u, 0x4342) * st[v];
      }
    }
    lo = lo * scale + rep_pair;
    hi = hi * scale + rep_pair;
    atomicAdd(reinterpret_cast<uint32_t*>(shb + (lo & 0xffffu)), 1u);
    atomicAdd(reinterpret_cast<uint32_t*>(shb + (lo >> 16)), 1u);
    atomicAdd(reinterpret_cast<uint32_t*>(shb + (hi & 0xffffu)), 1u);
    atomicAdd(reinterpret_cast<uint32_t*>(shb + (hi >> 16)), 1u);
  }
}

template <int K, bool PF>
__device__ __forceinline__ void hist_smem_lane16(const QDesc& q, int64_t r0, int64_t r1,
                                                 uint32_t* sh) {
  const uint8_t* rowp = q.base + r0;
  uint32_t co[K], st[K];
#pragma unroll
  for (int v = 0; v < K; ++v) {
    co[v] = q.coff[v];
    st[v] = q.stride[v];
  }
  const int nbyte = q.nbyte;
  const int rlog = q.rlog;
  const uint32_t scale = 4u << rlog;
  const uint32_t rep4 = (threadIdx.x & ((1u << rlog) - 1u)) * 4u;
  const uint32_t rep_pair = rep4 | (rep4 << 16);
  char* shb = reinterpret_cast<char*>(sh);
  const int64_t nrows = r1 - r0;
  const int64_t nvec = (nrows + 15) >> 4;
  const int64_t bd = blockDim.x;
  int64_t vi = threadIdx.x;
  if (PF && K <= 4) {
    // ping-pong: vector i+1's K loads are in flight while vector i is counted
    uint32_t a[K][4], b[K][4];
    if (vi < nvec) load_vec16<K>(a, rowp + (vi << 4), co);
    for (; vi < nvec; vi += 2 * bd) {
      const bool hb = vi + bd < nvec;
      if (hb) load_vec16<K>(b, rowp + ((vi + bd) << 4), co);
      count_vec16<K>(a, st, nbyte, scale, rep_pair, shb);
      if (!hb) break;
      if (vi + 2 * bd < nvec) load_vec16<K>(a, rowp + ((vi + 2 * bd) << 4), co);
      count_vec16<K>(b, st, nbyte, scale, rep_pair, shb);
    }
  } else {
    for (; vi < nvec; vi += bd) {
      uint32_t a[K][4];
      load_vec16<K>(a, rowp + (vi << 4), co);
      count_vec16<K>(a, st, nbyte, scale, rep_pair, shb);
    }
  }
  const int64_t pad = (nvec << 4) - nrows;  // padding rows counted into cell 0
  if (pad > 0 && (int64_t)threadIdx.x == ((nvec - 1) % bd))
    atomicSub(reinterpret_cast<uint32_t*>(shb + rep4), (uint32_t)pad);
}

// Other classes: scalar 32-bit index per row.
//   SMEM=true : SMEM tables too large for 16-bit byte offsets (C*R*4 > 65536);
//   SMEM=false: RED.ADD into the global table (tables too large for SMEM).
// MODE 1 builds the index in 16-bit lanes (C <= 65536), MODE 2 per row in 32 bits.
template <int K, int MODE, bool SMEM>
__device__ __forceinline__ void hist_rows(const QDesc& q, int64_t r0, int64_t r1, uint32_t* sh,
                                          uint32_t* gtab) {
  const uint8_t* rowp = q.base + r0;
  uint32_t co[K], st[K];
#pragma unroll
  for (int v = 0; v < K; ++v) {
    co[v] = q.coff[v];
    st[v] = q.stride[v];
  }
  const int nbyte = q.nbyte;
  const int rlog = q.rlog;
  const uint32_t rep = threadIdx.x & ((1u << rlog) - 1u);
  const int64_t nrows = r1 - r0;
  const int64_t nvec = (nrows + 15) >> 4;
  uint32_t* base = SMEM ? sh : gtab;
  // SMEM: byte address of a row's counter = idx * (4R) + (4 rep + table base): one IMAD
  const uint32_t scale = 4u << rlog;
  char* rbase = reinterpret_cast<char*>(sh) + 4u * rep;
  for (int64_t vi = threadIdx.x; vi < nvec; vi += blockDim.x) {
    uint4 w[K];
#pragma unroll
    for (int v = 0; v < K; ++v) w[v] = ldg_stream16(rowp + (vi << 4) + ((uint64_t)co[v] << 8));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t idx[4];
      if (MODE == 1) {
        uint32_t a8 = word_of(w[0], j);
#pragma unroll
        for (int v = 1; v < K; ++v)
          if (v < nbyte) a8 += word_of(w[v], j) * st[v];
        uint32_t lo = __byte_perm(a8, 0u, 0x4140);
        uint32_t hi = __byte_perm(a8, 0u, 0x4342);
#pragma unroll
        for (int v = 1; v < K; ++v) {
          if (v >= nbyte) {
            const uint32_t x = word_of(w[v], j);
            lo += __byte_perm(x, 0u, 0x4140) * st[v];
            hi += __byte_perm(x, 0u, 0x4342) * st[v];
          }
        }
        idx[0] = lo & 0xffffu;
        idx[1] = lo >> 16;
        idx[2] = hi & 0xffffu;
        idx[3] = hi >> 16;
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          uint32_t acc = 0;
#pragma unroll
          for (int v = 0; v < K; ++v) acc += __byte_perm(word_of(w[v], j), 0u, 0x4440 + b) * st[v];
          idx[b] = acc;
        }
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (SMEM) atomicAdd(reinterpret_cast<uint32_t*>(rbase + idx[b] * scale), 1u);
        else atomicAdd(base + idx[b], 1u);
      }
    }
  }
  const int64_t pad = (nvec << 4) - nrows;
  if (pad > 0 && (int64_t)threadIdx.x == ((nvec - 1) % (int64_t)blockDim.x))
    atomicSub(base + (SMEM ? rep : 0u), (uint32_t)pad);
}

template <bool SMEM, bool PF = false>
__device__ __forceinline__ void dispatch_rows(const QDesc& q, int64_t r0, int64_t r1, uint32_t* sh,
                                              uint32_t* gtab) {
#define CS_CASE_K(KK)                                                        \
  case KK:                                                                   \
    if (SMEM) {                                                              \
      if (q.mode == 0) hist_smem_lane16<KK, PF>(q, r0, r1, sh);              \
      else hist_rows<KK, 1, true>(q, r0, r1, sh, gtab);                      \
    } else {                                                                 \
      if (q.mode <= 1) hist_rows<KK, 1, false>(q, r0, r1, sh, gtab);         \
      else hist_rows<KK, 2, false>(q, r0, r1, sh, gtab);                     \
    }                                                                        \
    break;
  switch (q.k) {
    CS_CASE_K(1)
    CS_CASE_K(2)
    CS_CASE_K(3)
    CS_CASE_K(4)
    CS_CASE_K(5)
    CS_CASE_K(6)
    CS_CASE_K(7)
    CS_CASE_K(8)
    default:
      break;
  }
#undef CS_CASE_K
}

// Persistent K1.  items are sorted by descending cost on the host; CTAs pull them from
// *head.  kind 0 (SMEM) items finish with the fused epilogue: a single-segment query writes
// its table and scores straight from SMEM; a multi-segment query adds its partial table into
// global memory and the last segment to arrive (done[] counter) scores the merged table.
template <int THREADS, int MINB, bool PF>
__global__ void __launch_bounds__(THREADS, MINB)
    k_hist(const QDesc* __restrict__ qd, const WItem* __restrict__ items, int nitems,
           int* __restrict__ head, uint32_t* tables, uint32_t* __restrict__ done, double* ll_out,
           double* mi_out, int64_t* nnz_out, uint32_t flags, double m_total) {
  extern __shared__ uint32_t sh[];
  __shared__ QDesc s_q;
  __shared__ int s_item, s_last;
  __shared__ ScoreSmem ss;
  const bool want_score = !(flags & F_PARTIAL) && (flags & (F_LOGLIK | F_MI | F_NNZ));
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(head, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) return;
    const WItem wi = items[it];
    if (threadIdx.x < (int)(sizeof(QDesc) / 16))
      reinterpret_cast<int4*>(&s_q)[threadIdx.x] =
          reinterpret_cast<const int4*>(qd + wi.q)[threadIdx.x];
    __syncthreads();
    const QDesc& q = s_q;
    const int rl = q.rlog;
    const uint32_t R = 1u << rl;
    const uint32_t C = q.cells;
    const uint32_t nw = C << rl;
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    dispatch_rows<true, PF>(q, wi.r0, wi.r1, sh, nullptr);
    __syncthreads();
    auto cell = [&](uint32_t c) -> uint32_t {
      uint32_t s = 0;
      for (uint32_t r = 0; r < R; ++r) s += sh[(c << rl) | ((r + c) & (R - 1u))];
      return s;
    };
    if (q.nseg == 1) {
      if (tables) {
        uint32_t* t = tables + q.table_off;
        for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) t[c] = cell(c);
      }
      if (want_score)
        score_table(cell, C, q.r_target, m_total, flags, wi.q, ll_out, mi_out, nnz_out, ss);
    } else {
      uint32_t* t = tables + q.table_off;
      for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
        const uint32_t v = cell(c);
        if (v) atomicAdd(t + c, v);
      }
      if (want_score) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = (atomicAdd(done + wi.q, 1u) == (uint32_t)(q.nseg - 1));
        __syncthreads();
        if (s_last) {
          __threadfence();
          auto gcell = [&](uint32_t c) -> uint32_t { return __ldcg(t + c); };
          score_table(gcell, C, q.r_target, m_total, flags, wi.q, ll_out, mi_out, nnz_out, ss);
        }
      }
    }
  }
}

// K1 global class: tables too large for SMEM; RED.ADD into the (pre-zeroed) global table.
// Same persistent work-queue scheme as k_hist, no shared memory.
__global__ void __launch_bounds__(512, 2)
    k_hist_global(const QDesc* __restrict__ qd, const WItem* __restrict__ items, int nitems,
                  int* __restrict__ head, uint32_t* tables) {
  __shared__ QDesc s_q;
  __shared__ int s_item;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(head, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) return;
    const WItem wi = items[it];
    if (threadIdx.x < (int)(sizeof(QDesc) / 16))
      reinterpret_cast<int4*>(&s_q)[threadIdx.x] =
          reinterpret_cast<const int4*>(qd + wi.q)[threadIdx.x];
    __syncthreads();
    dispatch_rows<false>(s_q, wi.r0, wi.r1, nullptr, tables + s_q.table_off);
    __syncthreads();
  }
}

// K1g: queries with more than CS_MAXK variables.  grid = (row blocks, listed queries).
__global__ void k_hist_generic(const QDesc* __restrict__ qd, const int32_t* __restrict__ qlist,
                               const int32_t* __restrict__ gvars,
                               const uint32_t* __restrict__ gstride, const uint8_t* __restrict__ cols,
                               int64_t ld, int64_t m, uint32_t* tables) {
  const QDesc q = qd[qlist[blockIdx.y]];
  uint32_t* t = tables + q.table_off;
  const int32_t* vv = gvars + q.var_base;
  const uint32_t* ss = gstride + q.var_base;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    uint32_t idx = 0;
    for (int v = 0; v < q.k; ++v) idx += (uint32_t)__ldg(cols + (int64_t)vv[v] * ld + row) * ss[v];
    atomicAdd(t + idx, 1u);
  }
}

// K2: scores of global tables, one CTA per listed query.
__global__ void k_score(const QDesc* __restrict__ qd, const int32_t* __restrict__ qlist,
                        const uint32_t* __restrict__ tables, double* ll_out, double* mi_out,
                        int64_t* nnz_out, uint32_t flags, double m_total) {
  __shared__ ScoreSmem ss;
  const int q = qlist ? qlist[blockIdx.x] : (int)blockIdx.x;
  const QDesc& d = qd[q];
  const uint32_t* t = tables + d.table_off;
  auto cell = [&](uint32_t c) -> uint32_t { return t[c]; };
  score_table(cell, d.cells, d.r_target, m_total, flags, q, ll_out, mi_out, nnz_out, ss);
}

// family scores for the batched learn_parents driver (harness.py:296-348 semantics):
//   LL(X | Pa) = sum n ln n over joint(X u Pa) - sum n ln n over joint(Pa)
// (the second term is m ln m for Pa = {}), MDL = -LL + penalty (aggregators.py:191-193).
__global__ void k_family(int64_t nfam, const double* __restrict__ nlogn,
                         const int32_t* __restrict__ s_idx, const int32_t* __restrict__ p_idx,
                         const double* __restrict__ penalty, double m_ln_m, double* ll, double* mdl) {
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nfam;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pi = p_idx[f];
    const double v = nlogn[s_idx[f]] - (pi >= 0 ? nlogn[pi] : m_ln_m);
    if (ll) ll[f] = v;
    if (mdl) mdl[f] = -v + penalty[f];
  }
}

// K5: non-zero cells of each table in ascending cell order.  One CTA per query.
__global__ void k_compact(const QDesc* __restrict__ qd, const uint32_t* __restrict__ tables,
                          const int64_t* __restrict__ out_off, int64_t* cidx, int64_t* nijk,
                          int64_t* nij) {
  __shared__ int s_warp[32];
  __shared__ int64_t s_base;
  const int q = blockIdx.x;
  const QDesc& d = qd[q];
  const uint32_t* t = tables + d.table_off;
  const int rt = d.r_target;
  const uint32_t J = d.cells / (uint32_t)rt;
  if (threadIdx.x == 0) s_base = out_off[q];
  __syncthreads();
  for (uint32_t j0 = 0; j0 < J; j0 += blockDim.x) {
    const uint32_t j = j0 + threadIdx.x;
    int cnt = 0;
    unsigned long long tot = 0;
    if (j < J) {
      for (int k = 0; k < rt; ++k) {
        const uint32_t v = t[(uint64_t)j * rt + k];
        tot += v;
        cnt += (v != 0);
      }
    }
    // block exclusive scan of cnt
    int x = cnt;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
      int s = (lane < (int)(blockDim.x >> 5)) ? s_warp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      s_warp[lane] = s;
    }
    __syncthreads();
    const int excl = x - cnt + (w > 0 ? s_warp[w - 1] : 0);
    const int total = s_warp[(blockDim.x >> 5) - 1];
    if (cnt) {
      int64_t pos = s_base + excl;
      for (int k = 0; k < rt; ++k) {
        const uint32_t v = t[(uint64_t)j * rt + k];
        if (v) {
          cidx[pos] = (int64_t)j * rt + k;
          nijk[pos] = v;
          nij[pos] = (int64_t)tot;
          ++pos;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// generator: column var, rows [0, m) of this shard = global rows row_offset + row.
__global__ void k_generate(uint8_t* __restrict__ col, int64_t m, uint64_t key, int64_t row_offset,
                           int np, const uint8_t* const* __restrict__ pcols,
                           const uint32_t* __restrict__ pstride, const uint32_t* __restrict__ thr,
                           int rm1) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    uint32_t pcfg = 0;
    for (int t = 0; t < np; ++t) pcfg += (uint32_t)pcols[t][row] * pstride[t];
    const uint32_t u = hash32(key, (uint64_t)(row_offset + row));
    const uint32_t* th = thr + (uint64_t)pcfg * rm1;
    int s = 0;
    for (int t = 0; t < rm1; ++t) s += (u >= __ldg(th + t)) ? 1 : 0;
    col[row] = (uint8_t)s;
  }
}

// state validation: bad[var] = first row whose state >= arity (or INT64_MAX)
__global__ void k_check_states(const uint8_t* __restrict__ cols, int64_t ld, int64_t m,
                               const int32_t* __restrict__ arity, unsigned long long* bad) {
  const int var = blockIdx.y;
  const uint32_t r = (uint32_t)arity[var];
  const uint8_t* c = cols + (int64_t)var * ld;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < m;
       row += (int64_t)gridDim.x * blockDim.x) {
    if ((uint32_t)c[row] >= r) atomicMin(bad + var, (unsigned long long)row);
  }
}

// ------------------------------------------------------------------------------------------
// K3: bit planes.  grid = (word blocks, listed vars); thread per 32-row word.
__device__ __forceinline__ uint32_t eq_bits4(uint32_t x, uint32_t pat) {
  const uint32_t e = __vcmpeq4(x, pat) & 0x01010101u;  // 1 per equal byte
  return ((e * 0x00204081u) >> 21) & 0xfu;              // byte b -> bit b
}

__global__ void k_bitmap_build(const uint8_t* __restrict__ cols, int64_t ld, int64_t m,
                               const int32_t* __restrict__ vars, const int32_t* __restrict__ arity,
                               const int64_t* __restrict__ plane_off, uint32_t* planes,
                               int64_t words) {
  const int vi = blockIdx.y;
  const int var = vars[vi];
  const int r = arity[var];
  const uint8_t* c = cols + (int64_t)var * ld;
  uint32_t* out = planes + plane_off[vi];
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row0 = w * 32;
    uint32_t valid;
    if (row0 >= m) valid = 0u;
    else if (m - row0 >= 32) valid = 0xffffffffu;
    else valid = (1u << (uint32_t)(m - row0)) - 1u;
    uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
    if (valid) {
      a = *reinterpret_cast<const uint4*>(c + row0);
      b = *reinterpret_cast<const uint4*>(c + row0 + 16);
    }
    for (int s = 0; s < r; ++s) {
      const uint32_t pat = 0x01010101u * (uint32_t)s;
      uint32_t bits = eq_bits4(a.x, pat) | (eq_bits4(a.y, pat) << 4) | (eq_bits4(a.z, pat) << 8) |
                      (eq_bits4(a.w, pat) << 12) | (eq_bits4(b.x, pat) << 16) |
                      (eq_bits4(b.y, pat) << 20) | (eq_bits4(b.z, pat) << 24) |
                      (eq_bits4(b.w, pat) << 28);
      out[(int64_t)s * words + w] = bits & valid;
    }
  }
}

// K4 (bitmap): counts[q] += popc(AND_j plane_j) over a word chunk.  grid = (chunks, nq).
// plist holds, per query, k plane offsets starting at poff[q].
__global__ void k_points_bitmap(const int32_t* __restrict__ poff, const int64_t* __restrict__ plist,
                                const uint32_t* __restrict__ planes, int64_t words,
                                int64_t words_per_chunk, unsigned long long* counts) {
  __shared__ unsigned long long s_red[32];
  const int q = blockIdx.y;
  const int b = poff[q], k = poff[q + 1] - b;
  const int64_t w0 = (int64_t)blockIdx.x * words_per_chunk;
  const int64_t w1 = min(words, w0 + words_per_chunk);
  unsigned long long acc = 0;
  for (int64_t w = w0 + 4 * (int64_t)threadIdx.x; w < w1; w += 4 * (int64_t)blockDim.x) {
    uint4 x = *reinterpret_cast<const uint4*>(planes + plist[b] + w);
    for (int j = 1; j < k; ++j) {
      const uint4 y = *reinterpret_cast<const uint4*>(planes + plist[b + j] + w);
      x.x &= y.x; x.y &= y.y; x.z &= y.z; x.w &= y.w;
    }
    acc += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
  }
  const unsigned long long t = block_sum_u64(acc, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(counts + q, t);
}

// K4 (byte scan): rows where every listed column equals its state.  grid = (chunks, nq).
__global__ void k_points_scan(const int32_t* __restrict__ poff, const int32_t* __restrict__ pvar,
                              const int32_t* __restrict__ pstate, const uint8_t* __restrict__ cols,
                              int64_t ld, int64_t m, int64_t rows_per_chunk,
                              unsigned long long* counts) {
  __shared__ unsigned long long s_red[32];
  const int q = blockIdx.y;
  const int b = poff[q], k = poff[q + 1] - b;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_chunk;
  const int64_t r1 = min(m, r0 + rows_per_chunk);
  unsigned long long acc = 0;
  for (int64_t row = r0 + 16 * (int64_t)threadIdx.x; row < r1; row += 16 * (int64_t)blockDim.x) {
    uint4 mk = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    for (int j = 0; j < k; ++j) {
      const uint4 x = *reinterpret_cast<const uint4*>(cols + (int64_t)pvar[b + j] * ld + row);
      const uint32_t pat = 0x01010101u * (uint32_t)pstate[b + j];
      mk.x &= __vcmpeq4(x.x, pat); mk.y &= __vcmpeq4(x.y, pat);
      mk.z &= __vcmpeq4(x.z, pat); mk.w &= __vcmpeq4(x.w, pat);
    }
    const int64_t left = r1 - row;
    if (left < 16) {
      // keep only the first `left` byte lanes
      uint32_t lanes[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t keep = left - 4 * j;
        if (keep <= 0) lanes[j] = 0;
        else if (keep < 4) lanes[j] &= (1u << (8 * keep)) - 1u;
      }
      mk = make_uint4(lanes[0], lanes[1], lanes[2], lanes[3]);
    }
    acc += __popc(mk.x) + __popc(mk.y) + __popc(mk.z) + __popc(mk.w);
  }
  const unsigned long long t = block_sum_u64(acc, s_red);
  if (threadIdx.x == 0 && t) atomicAdd(counts + q, t);
}

}  // namespace cs
