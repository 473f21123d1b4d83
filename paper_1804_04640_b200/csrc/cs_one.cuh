// cs_one.cuh -- K8, the single-query latency class behind cs_query_one (the drop-in
// Strategy.query path: reference radix.py:113-156 / bitmap.py:69-128 answer one query per
// call, and harness.py:222-275 times exactly that).
//
// A batch plan costs a descriptor upload, several launches and a device sync; for one small
// query that fixed cost dwarfs the counting.  Here the whole query travels as a kernel
// parameter (no upload), one CTA counts every row into an SMEM table, scores it with the
// shared fp64 epilogue (score_table) and stores the results -- scalars and, when asked, the
// dense table -- straight into page-locked, device-mapped host memory: one launch and one
// stream sync per query.
#pragma once
#include <cstdint>

#include "cs_common.cuh"
#include "cs_kernels.cuh"

namespace cs {

constexpr int ONE_THREADS = 1024;
constexpr uint32_t ONE_MAX_CELLS = 48 * 1024;  // 192 KB of SMEM counters

struct OneQ {
  const uint8_t* col[CS_MAXK];  // uint8 column of digit v (target first)
  uint32_t stride[CS_MAXK];
  int32_t k, r_t;
  uint32_t cells;
  uint32_t flags;
  int64_t m;
  double m_total;
  uint32_t* table;  // mapped host (or device) dense table, or NULL
  int64_t* cells_out;  // mapped host: [3][cells] cell index, N_ijk, N_ij of the non-zero cells in
                       // cell order (the record stream), or NULL; their count goes to out[2]
  double* out;      // [0] LL, [1] MI, [2] nnz (int64 bits)
  volatile uint32_t* done;  // mapped host word: set to `seq` once every result above is visible
  uint32_t seq;
};

__global__ void __launch_bounds__(ONE_THREADS, 1) k_query_one(const OneQ q) {
  extern __shared__ __align__(16) uint32_t one_tab[];
  __shared__ ScoreSmem ss;
  const int tid = threadIdx.x;
  for (uint32_t c = tid; c < q.cells; c += ONE_THREADS) one_tab[c] = 0;
  __syncthreads();
  // 4 rows per thread step: one 32-bit load per column (columns are 256-B aligned and padded)
  for (int64_t r0 = (int64_t)tid * 4; r0 < q.m; r0 += 4 * ONE_THREADS) {
    uint32_t idx[4] = {0, 0, 0, 0};
    for (int v = 0; v < q.k; ++v) {
      const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(q.col[v] + r0));
      const uint32_t s = q.stride[v];
#pragma unroll
      for (int r = 0; r < 4; ++r) idx[r] += ((w >> (8 * r)) & 0xffu) * s;
    }
    const int nr = q.m - r0 >= 4 ? 4 : (int)(q.m - r0);
    for (int r = 0; r < nr; ++r) atomicAdd(&one_tab[idx[r]], 1u);
  }
  __syncthreads();
  if (q.table)
    for (uint32_t c = tid; c < q.cells; c += ONE_THREADS) q.table[c] = one_tab[c];
  if (q.cells_out) {
    // non-zero cells in cell order: each thread owns a contiguous run of whole configurations
    // (r_t cells), counts its non-zeros, a block scan places them
    __shared__ uint32_t s_wsum[ONE_THREADS / 32];
    const uint32_t J = q.cells / (uint32_t)q.r_t;
    const uint32_t per = (J + ONE_THREADS - 1) / ONE_THREADS;
    const uint32_t j0 = min(J, tid * per), j1 = min(J, j0 + per);
    uint32_t mine = 0;
    for (uint32_t c = j0 * q.r_t; c < j1 * q.r_t; ++c) mine += one_tab[c] != 0;
    uint32_t incl = mine;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
    for (int w = 0; w < ONE_THREADS / 32; ++w) {
      if (w < warp) pre += s_wsum[w];
      tot += s_wsum[w];
    }
    uint32_t pos = pre + incl - mine;
    int64_t* oi = q.cells_out;
    int64_t* on = oi + q.cells;
    int64_t* oj = on + q.cells;
    for (uint32_t j = j0; j < j1; ++j) {
      uint32_t nij = 0;
      for (int k = 0; k < q.r_t; ++k) nij += one_tab[j * q.r_t + k];
      for (int k = 0; k < q.r_t; ++k) {
        const uint32_t c = j * q.r_t + k, x = one_tab[c];
        if (x) {
          oi[pos] = c;
          on[pos] = x;
          oj[pos] = nij;
          ++pos;
        }
      }
    }
    if (tid == 0) reinterpret_cast<int64_t*>(q.out)[2] = tot;
  }
  if (q.flags & (F_LOGLIK | F_MI | F_NNZ)) {
    auto cell = [&](uint32_t c) { return one_tab[c]; };
    score_table(cell, q.cells, q.r_t, q.m_total, q.flags, 0, q.out, q.out + 1,
                reinterpret_cast<int64_t*>(q.out + 2), ss);
  }
  // completion word: the host polls it instead of a stream synchronisation (lower latency);
  // every thread's stores are fenced to system scope before thread 0 publishes
  __threadfence_system();
  __syncthreads();
  if (tid == 0) *q.done = q.seq;
}

}  // namespace cs
