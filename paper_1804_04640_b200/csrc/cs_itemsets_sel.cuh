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
//   (item supports = the state-1 plane counts recorded by cs_bitmap_build, k_plane_popc)
//   k_sel_rowmask   record-major membership masks over the items in RANK order (rank 0 = most
//                   frequent): rm[t][j] bit b = item of rank 32 j + b is in record t.  Warp per
//                   32-record plane word: lane i loads the word of rank 32 j + i, 32 ballots
//                   transpose it, lane t stores record t's wr words (one coalesced 1 KB store)
//   k_sel_gram      (selector rank r, plane-word range) units: Gram of the records holding the
//                   selector over their masks below rank r (see the kernel's comment)
#pragma once
#include "cs_common.cuh"

namespace cs {

constexpr int SEL_THREADS = 512;  // two CTAs per SM (64 registers per thread)
constexpr int SEL_WARPS = SEL_THREADS / 32;
constexpr int SEL_MAXN = 248;  // items (ranks) on this path (rank -> item table in static SMEM)

struct SelUnit {
  int32_t r;       // selector rank
  int16_t blk0;    // Gram blocks [blk0, blk1) of this rank computed by the unit (<= SEL_THREADS)
  int16_t blk1;
  int64_t w0, w1;  // plane words [w0, w1), multiples of 32 x SEL_WARPS
};

// record count of each of the bitmap index's planes (contiguous, `words` uint32 each): the
// index's state counts, taken once when it is built
__global__ void k_plane_popc(const uint32_t* __restrict__ planes, int64_t words, unsigned long long* __restrict__ cnt,
                             int64_t nplanes) {
  for (int64_t pl = blockIdx.y; pl < nplanes; pl += gridDim.y) {
    const uint4* p = reinterpret_cast<const uint4*>(planes + pl * words);
    const int64_t nv = words >> 2;
    uint32_t c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
      const uint4 x = __ldg(p + i);
      c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt + pl, (unsigned long long)c);
  }
}

// rank_plane[k] = state-1 plane of the item of rank k (k < n); wr = words per record mask (1..8).
// Warp per 8 plane words (256 records): lane i loads the 32-B sector of rank 32 j + i for every
// rank block j, one butterfly transpose per (word, block) leaves record 32 q + lane's mask word
// j in lane `lane`, and each record's wr words go out as one vector store (1 KB per warp).
__global__ void __launch_bounds__(256) k_sel_rowmask(const uint32_t* const* __restrict__ rank_plane, int n,
                                                     int64_t words, int wr, uint32_t* __restrict__ rm);

// 32 x 32 bit transpose across a warp: lane r holds row r (bit c = element (r, c)); afterwards
// lane c holds column c (bit r = element (r, c)).  Five butterfly stages, each swapping the
// off-diagonal j x j blocks with the partner lane r ^ j.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  uint32_t m = 0x0000ffffu;
#pragma unroll
  for (int j = 16; j; j >>= 1, m ^= m << j) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? (x & ~m) | ((y >> j) & m) : (x & m) | ((y << j) & ~m);
  }
  return x;
}

__global__ void __launch_bounds__(256) k_sel_rowmask(const uint32_t* const* __restrict__ rank_plane, int n,
                                                     int64_t words, int wr, uint32_t* __restrict__ rm) {
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = words >> 3;  // words is a multiple of 32
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < ngroups; g += nwarps) {
    const int64_t w0 = g * 8;
    uint32_t out[8][8];  // [word q][block j] for record 32 (w0 + q) + lane
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < wr) {
        const int k = 32 * j + lane;
        uint4 a0 = make_uint4(0, 0, 0, 0), a1 = make_uint4(0, 0, 0, 0);
        if (k < n) {
          const uint4* src = reinterpret_cast<const uint4*>(rank_plane[k] + w0);
          a0 = __ldg(src);
          a1 = __ldg(src + 1);
        }
        const uint32_t x[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) out[q][j] = warp_transpose32(x[q], lane);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) out[q][j] = 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t* dst = rm + ((w0 + q) * 32 + lane) * wr;
      if (wr == 8) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(out[q][0], out[q][1], out[q][2], out[q][3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(out[q][4], out[q][5], out[q][6], out[q][7]);
      } else if (wr == 4) {
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(out[q][0], out[q][1], out[q][2], out[q][3]);
      } else if (wr == 2) {
        reinterpret_cast<uint2*>(dst)[0] = make_uint2(out[q][0], out[q][1]);
      } else {
        dst[0] = out[q][0];
      }
    }
  }
}

__device__ __forceinline__ int64_t sel_triple_index(int n, int a, int b, int c) {
  auto c3 = [](int64_t x) { return x >= 3 ? x * (x - 1) * (x - 2) / 6 : 0; };
  auto c2 = [](int64_t x) { return x >= 2 ? x * (x - 1) / 2 : 0; };
  return c3(n) - c3(n - a) + c2(n - a - 1) - c2(n - b) + (c - b - 1);
}

constexpr int SEL_LCAP = 3072;           // compacted records per round (2 CTAs x ~89 KB SMEM per SM)
constexpr int SEL_MAXB = SEL_LCAP / 32;  // 32-record batches per round

// A2 of k_sel_gram for units whose masks below rank r span NWR words: warp per 32-record
// batch, lane l gathers record l's NWR mask words (vector loads when the row is 16-B aligned),
// one butterfly transpose per word, Y[b][32 j + lane] = batch bits of rank 32 j + lane.
template <int NWR>
__device__ __forceinline__ void sel_batches(const uint32_t* __restrict__ rm, int wr, const uint32_t* list, int cnt,
                                            int nbatch, uint32_t lastmask, int R, uint32_t* Y, int warp,
                                            int lane) {
  for (int b = warp; b < nbatch; b += SEL_WARPS) {
    const int i = 32 * b + lane;
    // the warp's next batch: pull its records' mask rows into L2 now (no registers held)
    const int i2 = i + 32 * SEL_WARPS;
    if (i2 < cnt) asm volatile("prefetch.global.L2 [%0];" ::"l"(rm + (int64_t)list[i2] * wr));
    uint32_t mw[NWR];
#pragma unroll
    for (int j = 0; j < NWR; ++j) mw[j] = 0u;
    if (i < cnt) {
      const uint32_t* mrow = rm + (int64_t)list[i] * wr;
      if (wr >= 4) {
#pragma unroll
        for (int v = 0; v < (NWR + 3) / 4; ++v) {
          const uint4 x = reinterpret_cast<const uint4*>(mrow)[v];
          const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (4 * v + j < NWR) mw[4 * v + j] = xs[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < NWR; ++j) mw[j] = mrow[j];
      }
      mw[NWR - 1] &= lastmask;
    }
#pragma unroll
    for (int j = 0; j < NWR; ++j) {
      const uint32_t col = warp_transpose32(mw[j], lane);  // bit l: record l holds rank 32 j + lane
      if (32 * j + lane < R) Y[b * R + 32 * j + lane] = col;
    }
  }
}

// K4d main kernel, two persistent 512-thread CTAs per SM (their barrier phases interleave) pulling (selector rank r, plane-word
// range) units.  Per unit, rounds of
//   A1  warps scan 32-word chunks of the selector's plane and append the records holding it
//       to a CTA list (exact CAS reservations; a warp whose chunk does not fit ends the round)
//   A2  per 32-record batch: each lane gathers its record's mask words below rank r; a warp
//       butterfly transpose per mask word turns the batch into bit words Y[b][y] (bit l =
//       record l of the batch holds rank y)
//   B   Gram of the batches: thread (by, bz, g) owns an 8 x 4 block of (y, z) counters
//       (ranks 8 by.., 4 bz..; only blocks with some y <= z) in registers, acc += popc(Y[b][y] & Y[b][z]) over the batches b = g mod G
//       (G = 512 / #blocks thread groups, so small-r units keep every thread busy)
// and at the unit's end the non-zero counters with y <= z < r go to the global arrays:
// y == z -> pair (s, y), y < z -> triple (s, y, z).  A record holding k more frequent items
// costs ~(r/8)^2 x 64 / 32 popcounts regardless of k, so this is the dense Gram of the
// selected records only: POPC-issue bound, no atomics, no per-record divergence.
// dynamic SMEM: list (SEL_LCAP uint32) | Y (SEL_MAXB x R uint32), R = round_up(rmax, 8)
__global__ void __launch_bounds__(SEL_THREADS, 2) k_sel_gram(
    const uint32_t* const* __restrict__ rank_plane, const uint32_t* __restrict__ rm, int wr,
    const int16_t* __restrict__ rank_item, int n, const SelUnit* __restrict__ units, int nunits,
    int* __restrict__ head, int R, unsigned long long* __restrict__ pairs,
    unsigned long long* __restrict__ triples, int dbg) {
  extern __shared__ __align__(16) uint32_t sel_smem[];
  uint32_t* list = sel_smem;
  uint32_t* Y = sel_smem + SEL_LCAP;
  __shared__ int s_unit, s_cnt, s_end;
  __shared__ int16_t s_item[SEL_MAXN];
  // triple_index(n, a, b, c) = t3[a] - t2[b] + (c - b - 1) for a < b < c
  __shared__ long long s_t3[SEL_MAXN], s_t2[SEL_MAXN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < n; k += SEL_THREADS) {
    s_item[k] = rank_item[k];
    const auto c3 = [](long long x) { return x >= 3 ? x * (x - 1) * (x - 2) / 6 : 0ll; };
    const auto c2 = [](long long x) { return x >= 2 ? x * (x - 1) / 2 : 0ll; };
    s_t3[k] = c3(n) - c3(n - k) + c2(n - k - 1);
    s_t2[k] = c2(n - k);
  }
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(head, 1);
    __syncthreads();
    const int ui = s_unit;
    if (ui >= nunits) return;
    const SelUnit u = units[ui];
    const int r = u.r & 0xffff;
    const bool direct = (u.r >> 30) & 1;  // dense selector: batches = plane words, no compaction
    // Gram blocks: 8 ranks (y) x 4 ranks (z), only blocks holding some y <= z (bz >= 2 by)
    const int nby = (r + 7) >> 3, nbz = (r + 3) >> 2;
    // this unit's Gram blocks: [blk0, blk1) of the rank's 8 x 4 blocks holding some y <= z
    // (bz >= 2 by), enumerated by y block; ranks with more blocks than threads are split into
    // several units over the same records
    const int nblk = u.blk1 - u.blk0;
    // thread -> (Gram block, batch group): with few blocks (frequent selectors, small r) several
    // threads share a block and split the batches, each keeping its own partial counters
    const int ngrp = SEL_THREADS / nblk;
    const int grp = threadIdx.x / nblk;
    int by = -1, bz = -1;
    if (grp < ngrp) {
      int t = u.blk0 + threadIdx.x - grp * nblk;
      for (int y = 0; y < nby; ++y) {
        const int len = nbz - 2 * y;
        if (t < len) {
          by = y;
          bz = 2 * y + t;
          break;
        }
        t -= len;
      }
    }
    uint32_t acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0;
    const int nwr = (r + 31) >> 5;
    const uint32_t lastmask = (r & 31) ? (1u << (r & 31)) - 1 : 0xffffffffu;
    const uint32_t* sp = rank_plane[r];
    int64_t wnext = u.w0 + 128 * warp;
    int64_t wdir = u.w0;  // direct mode: next plane word
    for (;;) {
      bool done;
      int nbatch;
      if (direct) {
        // batch b = plane word wdir + b: Y[b][y] = P_y & P_s (records of the word holding both);
        // ranks [r, 8 nby) are zeroed for the last Gram block row
        nbatch = (int)(u.w1 - wdir < SEL_MAXB ? u.w1 - wdir : SEL_MAXB);
        const int ny = min(R, 8 * nby);
        for (int i = threadIdx.x; i < ny * nbatch; i += SEL_THREADS) {
          const int y = i / nbatch, b = i - y * nbatch;
          Y[b * R + y] = y < r ? __ldg(rank_plane[y] + wdir + b) & __ldg(sp + wdir + b) : 0u;
        }
        wdir += nbatch;
        done = wdir >= u.w1;
        __syncthreads();
      } else {
      if (threadIdx.x == 0) {
        s_cnt = 0;
        s_end = SEL_LCAP;
      }
      __syncthreads();
      // A1: append selected records until the range ends or a chunk does not fit
      // A1 chunks: 4 words (128 records) per lane, 128 words per warp; the next two chunks'
      // selector words are in flight while one is compacted (the scan is latency-bound: one
      // 128-B request per warp kept only ~0.6 TB/s of plane reads in flight)
      auto load4 = [&](int64_t w) -> uint4 {
        if (w + 4 <= u.w1) return __ldg(reinterpret_cast<const uint4*>(sp + w));
        uint4 v = make_uint4(0, 0, 0, 0);
        if (w < u.w1) v.x = sp[w];
        if (w + 1 < u.w1) v.y = sp[w + 1];
        if (w + 2 < u.w1) v.z = sp[w + 2];
        return v;
      };
      const int64_t stride = 128 * SEL_WARPS;
      uint4 xa = load4(wnext + 4 * lane), xb = load4(wnext + stride + 4 * lane);
      while (wnext < u.w1) {
        const uint4 xc = xa;
        xa = xb;
        xb = load4(wnext + 2 * stride + 4 * lane);
        uint32_t xs[4] = {xc.x, xc.y, xc.z, xc.w};
        const int c = __popc(xs[0]) + __popc(xs[1]) + __popc(xs[2]) + __popc(xs[3]);
        int pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += y;
        }
        const int total = __shfl_sync(0xffffffffu, pre, 31);
        // reserve with one atomicAdd; a reservation past SEL_LCAP fails (every later one does
        // too), and the round's list ends at the smallest failed base (s_end)
        int base = 0;
        if (lane == 0 && total) base = atomicAdd(&s_cnt, total);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base + total > SEL_LCAP) {
          if (lane == 0) atomicMin(&s_end, base);
          // the two loads in flight are dropped; the next round reloads from wnext
          break;
        }
        int pos = base + pre - c;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t x = xs[j];
          const uint32_t rec0 = (uint32_t)((wnext + 4 * lane + j) * 32);
          while (x) {
            const int bit = __ffs(x) - 1;
            x &= x - 1;
            list[pos++] = rec0 + bit;
          }
        }
        wnext += stride;
      }
      done = __syncthreads_and(wnext >= u.w1);
      const int cnt = min(s_cnt, s_end);
      nbatch = (cnt + 31) >> 5;
      // A2: batch transposes (masks below rank r only; y in [r, R) comes out zero), unrolled
      // for the unit's mask-word count
      if (!(dbg & 2)) switch (nwr) {
        case 1: sel_batches<1>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        case 2: sel_batches<2>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        case 3: sel_batches<3>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        case 4: sel_batches<4>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        case 5: sel_batches<5>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        case 6: sel_batches<6>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        case 7: sel_batches<7>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
        default: sel_batches<8>(rm, wr, list, cnt, nbatch, lastmask, R, Y, warp, lane); break;
      }
      __syncthreads();
      }  // compacted mode
      // B: Gram of the batches
      if (by >= 0 && !(dbg & 1)) {
        for (int b = grp; b < nbatch; b += ngrp) {
          const uint4* yp = reinterpret_cast<const uint4*>(Y + b * R + 8 * by);
          const uint4 y0 = yp[0], y1 = yp[1], z0 = *reinterpret_cast<const uint4*>(Y + b * R + 4 * bz);
          const uint32_t ya[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
          const uint32_t za[4] = {z0.x, z0.y, z0.z, z0.w};
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a * 4 + c] += __popc(ya[a] & za[c]);
        }
      }
      __syncthreads();
      if (done) break;
    }
    // flush: y <= z < r
    if (by >= 0 && !(dbg & 4)) {
      const int s = s_item[r];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int y = 8 * by + a, z = 4 * bz + c;
          const uint32_t v = acc[a * 4 + c];
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
            atomicAdd(triples + (s_t3[p0] - s_t2[p1] + (p2 - p1 - 1)), (unsigned long long)v);
          }
        }
    }
  }
}

}  // namespace cs
