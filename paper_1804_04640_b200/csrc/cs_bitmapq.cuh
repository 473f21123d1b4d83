// cs_bitmapq.cuh -- K7, the bitmap query class (survey 8(f)3): the reference's Alg. 1
// (bitmap.py:69-128) for queries whose variables are all binary and few
// (<= 4 digits, <= 16 cells).  Such a table is answered from the variables' state-1 bit planes
// (bitmap.py:29-31 order, cs_bitmap_build) with AND + popcount instead of a per-row histogram.
//
// The reference walks the parent configurations depth first, ANDing one bitset per level and
// popcounting the target states at the leaves.  Here every 32-record word is handled by one
// lane at once for all configurations, and the complement planes (state 0) are never formed:
// for every non-empty digit subset S the kernel counts
//       f(S) = #records whose digits in S are all 1 = popc(AND_{v in S} plane_v)
// (2^K - 1 popcounts per word, the ANDs shared along a subset tree), and k_bitmap_mobius turns
// those superset sums into the table in place (f(0) = m; for each digit v, N(c) = f(c) -
// f(c | bit v) over cells without v) -- exact integer arithmetic, the same table the histogram
// classes produce.  Planes are bytes-thin (K / 8 B per record versus K / 4 for the 2-bit column
// copy), so the bound is the L2 / HBM stream or the POPC pipe, not SMEM atomics.
//
// Pipeline (the north-star's "TMA-staged AND plus popc with warp-shuffle reductions"): a producer
// warp pulls (query, tile range) items and stages each tile of the K planes into shared memory
// with cp.async.bulk (the TMA bulk-copy engine) on an mbarrier ring; 8 consumer warps AND /
// popcount out of SMEM and reduce each item's counts with redux.sync before one global atomic
// per (warp, subset).
#pragma once
#include <cstdint>

#include "cs_common.cuh"

namespace cs {

constexpr int BQ_TILE = 1024;      // plane words per stage per digit (4 KB)
constexpr int BQ_STAGES = 8;       // mbarrier ring depth
constexpr int BQ_CONSUMERS = 256;  // 8 consumer warps: one 16-B word vector per thread per tile
constexpr int BQ_THREADS = BQ_CONSUMERS + 32;
constexpr int BQ_MAXK = 4;

struct BDesc {
  const uint32_t* plane[BQ_MAXK];  // state-1 plane of digit v (target first, then parents)
  int64_t table_off;
  int32_t k;
  int32_t pad;
};

struct BItem {
  int32_t d;       // BDesc index
  int32_t t0, t1;  // tiles [t0, t1) of BQ_TILE words
};

struct BStage {
  int32_t d;      // BDesc of the tile, -1 = end of work
  int32_t words;  // valid words in the tile (multiple of 32)
  int32_t flush;  // last tile of its item: consumers reduce and publish
  int32_t pad;
};

__device__ __forceinline__ uint32_t bq_smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bq_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "BQ_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra BQ_WAIT;\n\t}" ::"r"(bar),
      "r"(parity), "r"(0x10000u)
      : "memory");
}

template <int K>
__device__ __forceinline__ void bq_count_word(const uint32_t (&p)[K], uint32_t (&acc)[1 << K]) {
  // subset products along a tree: prod(S) = prod(S without its highest digit) & plane(highest)
  uint32_t prod[1 << K];
#pragma unroll
  for (int S = 1; S < (1 << K); ++S) {
    const int hi = 31 - __clz(S);
    const int rest = S ^ (1 << hi);
    prod[S] = rest ? (prod[rest] & p[hi]) : p[hi];
    acc[S] += __popc(prod[S]);
  }
}

template <int K>
__global__ void __launch_bounds__(BQ_THREADS)
    k_bitmap_query(const BDesc* __restrict__ bd, const BItem* __restrict__ items, int nitems, int* head,
                   int64_t words, uint32_t* tables) {
  extern __shared__ __align__(128) uint32_t bq_buf[];  // [BQ_STAGES][K][BQ_TILE]
  __shared__ __align__(8) uint64_t full[BQ_STAGES], empty[BQ_STAGES];
  __shared__ BStage meta[BQ_STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < BQ_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bq_smem_addr(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bq_smem_addr(&empty[s])),
                   "r"(BQ_CONSUMERS / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == BQ_CONSUMERS / 32) {
    // producer: one lane issues the bulk copies
    if (lane != 0) return;
    int s = 0;
    uint32_t iter = 0;
    for (;;) {
      const int it = atomicAdd(head, 1);
      const bool done = it >= nitems;
      BItem item = done ? BItem{0, 0, 1} : items[it];
      for (int t = item.t0; t < item.t1; ++t) {
        if (iter >= (uint32_t)BQ_STAGES) bq_wait(bq_smem_addr(&empty[s]), ((iter / BQ_STAGES) - 1) & 1);
        const uint32_t fb = bq_smem_addr(&full[s]);
        if (done) {
          meta[s] = BStage{-1, 0, 0, 0};
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
          break;
        }
        const BDesc& d = bd[item.d];
        const int64_t w0 = (int64_t)t * BQ_TILE;
        const int nw = (int)min((int64_t)BQ_TILE, words - w0);
        meta[s] = BStage{item.d, nw, t + 1 == item.t1, 0};
        const uint32_t bytes = (uint32_t)nw * 4u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(bytes * K) : "memory");
        uint32_t* st = bq_buf + (size_t)s * K * BQ_TILE;
#pragma unroll
        for (int v = 0; v < K; ++v)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           bq_smem_addr(st + v * BQ_TILE)),
                       "l"(d.plane[v] + w0), "r"(bytes), "r"(fb)
                       : "memory");
        ++iter;
        s = s + 1 == BQ_STAGES ? 0 : s + 1;
      }
      if (done) break;
    }
    return;
  }
  // consumers
  uint32_t acc[1 << K];
#pragma unroll
  for (int S = 0; S < (1 << K); ++S) acc[S] = 0;
  int s = 0;
  uint32_t iter = 0;
  for (;;) {
    bq_wait(bq_smem_addr(&full[s]), (iter / BQ_STAGES) & 1);
    const BStage mt = meta[s];
    if (mt.d < 0) break;
    const uint32_t* st = bq_buf + (size_t)s * K * BQ_TILE;
    const int w = tid * 4;
    if (w < mt.words) {
      uint4 x[K];
#pragma unroll
      for (int v = 0; v < K; ++v) x[v] = *reinterpret_cast<const uint4*>(st + v * BQ_TILE + w);
      uint32_t p[K];
#pragma unroll
      for (int v = 0; v < K; ++v) p[v] = x[v].x;
      bq_count_word<K>(p, acc);
#pragma unroll
      for (int v = 0; v < K; ++v) p[v] = x[v].y;
      bq_count_word<K>(p, acc);
#pragma unroll
      for (int v = 0; v < K; ++v) p[v] = x[v].z;
      bq_count_word<K>(p, acc);
#pragma unroll
      for (int v = 0; v < K; ++v) p[v] = x[v].w;
      bq_count_word<K>(p, acc);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bq_smem_addr(&empty[s])) : "memory");
    if (mt.flush) {
      uint32_t* t = tables + bd[mt.d].table_off;
#pragma unroll
      for (int S = 1; S < (1 << K); ++S) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, acc[S]);
        if (lane == 0 && v) atomicAdd(t + S, v);
        acc[S] = 0;
      }
    }
    ++iter;
    s = s + 1 == BQ_STAGES ? 0 : s + 1;
  }
}

// superset sums -> cells, in place, one thread per bitmap-class query: f(0) = m records, then
// N(c) = f(c) - f(c | 2^v) for every digit v over the cells without v
__global__ void k_bitmap_mobius(const BDesc* __restrict__ bd, int nq, uint32_t m, uint32_t* tables) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  const BDesc d = bd[i];
  uint32_t* t = tables + d.table_off;
  const int C = 1 << d.k;
  t[0] = m;
  for (int v = 0; v < d.k; ++v)
    for (int c = 0; c < C; ++c)
      if (!(c & (1 << v))) t[c] -= t[c | (1 << v)];
}

}  // namespace cs
