// cs_itemsets_sel.cuh -- K4d: 2-/3-itemset supports by rarest-item selection (sparse data).
//
// The reference's bitmap query (bitmap.py:69-128, Alg. 1 of the paper) walks the variables in
// ascending-entropy order and prunes the AND tree as soon as a prefix is empty: the rare items
// decide which records matter.  Applied to all itemsets at once: every itemset {x, y, z} is
// counted exactly once, under its LEAST frequent item s (the "selector"), over only the records
// that contain s:
//     supp(s, y)    = #{t : s in t, y in t}          y more frequent than s
//     supp(s, y, z) = #{t : s in t, y in t, z in t}  y, z more frequent than s
// so the work is a Gram matrix of only supp(s) records per selector: sum_s supp(s) r_s^2 / 64
// popcounts (r_s = the selector's frequency rank) -- for Zipf-distributed transactions
// (BASELINE configs[3]) tens of times less than the dense bit-GEMM (K4b/K4c) that ANDs every
// pair plane with every item plane over all m records.  The host picks this class when its cost model says so
// (cs_itemset_supports); results are identical.
//
//   k_sel_support   supports of the n items (popcount of the state-1 planes)
//   k_sel_rowmask   record-major membership masks over the items in RANK order (rank 0 = most
//                   frequent): rm[t][j] bit b = item of rank 32 j + b is in record t.  Warp per
//                   32-record plane word: lane i loads the word of rank 32 j + i, 32 ballots
//                   transpose it, lane t stores record t's wr words (one coalesced 1 KB store)
//   k_sel_gram      (selector rank r, plane-word range) units: Gram of the records holding the
//                   selector over their masks below rank r (see the kernel's comment)
#pragma once
#include "cs_common.cuh"

namespace cs {

constexpr int SEL_THREADS = 512;
constexpr int SEL_WARPS = SEL_THREADS / 32;
constexpr int SEL_MAXN = 248;  // items (ranks) on this path: (248/8)(248/8+1)/2 = 496 Gram blocks <= 512 threads

struct SelUnit {
  int32_t r;      // selector rank
  int32_t pad;
  int64_t w0, w1;  // plane words [w0, w1), multiples of 32
};

__global__ void k_sel_support(const uint32_t* const* __restrict__ plane, int64_t words,
                              unsigned long long* __restrict__ supp) {
  const uint4* p = reinterpret_cast<const uint4*>(plane[blockIdx.y]);
  const int64_t nv = words >> 2;
  uint32_t c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = __ldg(p + i);
    c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(supp + blockIdx.y, (unsigned long long)c);
}

// rank_plane[k] = state-1 plane of the item of rank k (k < n); wr = words per record mask (1..8)
__global__ void __launch_bounds__(256) k_sel_rowmask(const uint32_t* const* __restrict__ rank_plane, int n,
                                                     int64_t words, int wr, uint32_t* __restrict__ rm) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < words; w += nwarps) {
    uint32_t mine[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      mine[j] = 0;
      if (j < wr) {
        const int k = 32 * j + lane;
        const uint32_t x = k < n ? __ldg(rank_plane[k] + w) : 0u;
#pragma unroll 8
        for (int t = 0; t < 32; ++t) {
          const uint32_t b = __ballot_sync(0xffffffffu, (x >> t) & 1u);
          if (lane == t) mine[j] = b;
        }
      }
    }
    uint32_t* dst = rm + (w * 32 + lane) * wr;
    if (wr == 8) {
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(mine[0], mine[1], mine[2], mine[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(mine[4], mine[5], mine[6], mine[7]);
    } else if (wr == 4) {
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(mine[0], mine[1], mine[2], mine[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < wr) dst[j] = mine[j];
    }
  }
}

__device__ __forceinline__ int64_t sel_triple_index(int n, int a, int b, int c) {
  auto c3 = [](int64_t x) { return x >= 3 ? x * (x - 1) * (x - 2) / 6 : 0; };
  auto c2 = [](int64_t x) { return x >= 2 ? x * (x - 1) / 2 : 0; };
  return c3(n) - c3(n - a) + c2(n - a - 1) - c2(n - b) + (c - b - 1);
}

constexpr int SEL_LCAP = 4096;           // compacted records per round
constexpr int SEL_MAXB = SEL_LCAP / 32;  // 32-record batches per round

// K4d main kernel, one persistent 512-thread CTA per SM pulling (selector rank r, plane-word
// range) units.  Per unit, rounds of
//   A1  warps scan 32-word chunks of the selector's plane and append the records holding it
//       to a CTA list (exact CAS reservations; a warp whose chunk does not fit ends the round)
//   A2  per 32-record batch: each lane gathers its record's mask words below rank r, 32
//       ballots per mask word transpose the batch into bit words Y[b][y] (bit l = record l of
//       the batch holds rank y)
//   B   Gram of the batches: thread (by, bz, g), by <= bz, owns an 8 x 8 block of (y, z)
//       counters in registers, acc += popc(Y[b][y] & Y[b][z]) over the batches b = g mod G
//       (G = 512 / #blocks thread groups, so small-r units keep every thread busy)
// and at the unit's end the non-zero counters with y <= z < r go to the global arrays:
// y == z -> pair (s, y), y < z -> triple (s, y, z).  A record holding k more frequent items
// costs ~(r/8)^2 x 64 / 32 popcounts regardless of k, so this is the dense Gram of the
// selected records only: POPC-issue bound, no atomics, no per-record divergence.
// dynamic SMEM: list (SEL_LCAP uint32) | Y (SEL_MAXB x R uint32), R = round_up(rmax, 8)
__global__ void __launch_bounds__(SEL_THREADS, 1) k_sel_gram(
    const uint32_t* const* __restrict__ rank_plane, const uint32_t* __restrict__ rm, int wr,
    const int16_t* __restrict__ rank_item, int n, const SelUnit* __restrict__ units, int nunits,
    int* __restrict__ head, int R, unsigned long long* __restrict__ pairs,
    unsigned long long* __restrict__ triples) {
  extern __shared__ __align__(16) uint32_t sel_smem[];
  uint32_t* list = sel_smem;
  uint32_t* Y = sel_smem + SEL_LCAP;
  __shared__ int s_unit, s_cnt;
  __shared__ int16_t s_item[SEL_MAXN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < n; k += SEL_THREADS) s_item[k] = rank_item[k];
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(head, 1);
    __syncthreads();
    const int ui = s_unit;
    if (ui >= nunits) return;
    const SelUnit u = units[ui];
    const int r = u.r;
    const int nb = (r + 7) >> 3;
    // thread -> (Gram block, batch group): with few blocks (frequent selectors, small r) several
    // threads share a block and split the batches, each keeping its own partial counters
    const int nblk = nb * (nb + 1) / 2;
    const int ngrp = SEL_THREADS / nblk;
    const int grp = threadIdx.x / nblk;
    int by = -1, bz = -1;
    if (grp < ngrp) {
      int t = threadIdx.x - grp * nblk;
      for (int y = 0; y < nb; ++y) {
        if (t < nb - y) {
          by = y;
          bz = y + t;
          break;
        }
        t -= nb - y;
      }
    }
    uint32_t acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0;
    const int nwr = (r + 31) >> 5;
    const uint32_t lastmask = (r & 31) ? (1u << (r & 31)) - 1 : 0xffffffffu;
    const uint32_t* sp = rank_plane[r];
    int64_t wnext = u.w0 + 32 * warp;
    for (;;) {
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
      // A1: append selected records until the range ends or a chunk does not fit
      while (wnext < u.w1) {
        uint32_t x = sp[wnext + lane];
        const int c = __popc(x);
        int pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += y;
        }
        const int total = __shfl_sync(0xffffffffu, pre, 31);
        int base = 0, ok = 1;
        if (lane == 0) {
          int old = *reinterpret_cast<volatile int*>(&s_cnt);
          for (;;) {
            if (old + total > SEL_LCAP) {
              ok = 0;
              break;
            }
            const int prev = atomicCAS(&s_cnt, old, old + total);
            if (prev == old) {
              base = old;
              break;
            }
            old = prev;
          }
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        base = __shfl_sync(0xffffffffu, base, 0);
        int pos = base + pre - c;
        const uint32_t rec0 = (uint32_t)((wnext + lane) * 32);
        while (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1;
          list[pos++] = rec0 + b;
        }
        wnext += 32 * SEL_WARPS;
      }
      const bool done = __syncthreads_and(wnext >= u.w1);
      const int cnt = s_cnt;
      const int nbatch = (cnt + 31) >> 5;
      // A2: batch transposes (masks below rank r only; y in [r, R) comes out zero)
      for (int b = warp; b < nbatch; b += SEL_WARPS) {
        const int i = 32 * b + lane;
        const uint32_t* mrow = rm + (int64_t)(i < cnt ? list[i] : 0) * wr;
        uint32_t mw[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          mw[j] = (i < cnt && j < nwr) ? mrow[j] & (j == nwr - 1 ? lastmask : 0xffffffffu) : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < nwr) {
            uint32_t mine = 0;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const uint32_t bal = __ballot_sync(0xffffffffu, (mw[j] >> t) & 1u);
              if (lane == t) mine = bal;
            }
            if (32 * j + lane < R) Y[b * R + 32 * j + lane] = mine;
          }
        }
      }
      __syncthreads();
      // B: Gram of the batches
      if (by >= 0) {
        for (int b = grp; b < nbatch; b += ngrp) {
          const uint4* yp = reinterpret_cast<const uint4*>(Y + b * R + 8 * by);
          const uint4* zp = reinterpret_cast<const uint4*>(Y + b * R + 8 * bz);
          const uint4 y0 = yp[0], y1 = yp[1], z0 = zp[0], z1 = zp[1];
          const uint32_t ya[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
          const uint32_t za[8] = {z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w};
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[a * 8 + c] += __popc(ya[a] & za[c]);
        }
      }
      __syncthreads();
      if (done) break;
    }
    // flush: y <= z < r
    if (by >= 0) {
      const int s = s_item[r];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int y = 8 * by + a, z = 8 * bz + c;
          const uint32_t v = acc[a * 8 + c];
          if (!v || y > z || z >= r) continue;
          const int iy = s_item[y];
          if (y == z) {
            const int lo = min(iy, s), hi = max(iy, s);
            atomicAdd(pairs + (int64_t)lo * n + hi, (unsigned long long)v);
          } else {
            int p0 = s, p1 = iy, p2 = s_item[z];
            if (p0 > p1) { const int t = p0; p0 = p1; p1 = t; }
            if (p1 > p2) { const int t = p1; p1 = p2; p2 = t; }
            if (p0 > p1) { const int t = p0; p0 = p1; p1 = t; }
            atomicAdd(triples + sel_triple_index(n, p0, p1, p2), (unsigned long long)v);
          }
        }
    }
  }
}

}  // namespace cs
