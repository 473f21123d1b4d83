// cs_itemsets.cuh -- K4b: supports of all 2- and 3-itemsets of n binary items (BASELINE
// configs[3]; reference semantics: mine_rules' support_of -> bitmap_count, harness.py:390-392,
// bitmap.py:131-136, i.e. popcount of the AND of the items' state-1 bit planes).
//
// Formulated as a bit-level GEMM:   S[r, c] = sum_w popc( X_r[w] & P_c[w] )
//   rows r : the item pairs (a, b), a < b, with X_r = P_a & P_b   -> triple supports (a, b, c)
//            plus the singles (a, a), X_r = P_a                    -> pair supports   (a, c)
//   cols c : items, only c > max(a, b) is computed/written.
// Rows are sorted by b so a row block needs only a short column range.  A CTA computes a
// 128-row x 32-column tile over a slice of the words (split-K units are pulled from a work
// queue; partial sums are added with 64-bit atomics).  Per k-step, 32 words of the 128 X
// rows (ANDed while staging) and of the 32 columns go to shared memory; each lane owns 4 rows
// x 4 columns.  The popcounts use a Harley-Seal carry-save adder over 4-word groups: per
// (output, word) one AND and 0.75 CSA (two LOP3 each) plus 1/4 POPC, because POPC issues at
// 16/clk/SM on B200 while LOP3 issues at ~90-128/clk/SM (tools/microbench.cu).
#pragma once
#include "cs_common.cuh"

namespace cs {

constexpr int IS_ROWS = 128;   // rows per tile (32 lanes x 4)
constexpr int IS_COLS = 32;    // columns per tile (8 warps x 4)
constexpr int IS_TW = 32;      // words per k-step
constexpr int IS_XS = IS_TW + 2;  // padded smem row stride: lane-per-row LDS.64 conflict-free
constexpr int IS_THREADS = 256;

struct ISRow {
  int16_t a, b;  // a == b: single row (pair supports)
};

struct ISUnit {
  int32_t row0;  // first row of the tile (multiple of IS_ROWS in the sorted row list)
  int32_t col0;  // first column of the tile
  int64_t w0, w1;  // word slice
};

__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

__device__ __forceinline__ int64_t triple_index(int n, int a, int b, int c) {
  auto c3 = [](int64_t x) { return x >= 3 ? x * (x - 1) * (x - 2) / 6 : 0; };
  auto c2 = [](int64_t x) { return x >= 2 ? x * (x - 1) / 2 : 0; };
  return c3(n) - c3(n - a) + c2(n - a - 1) - c2(n - b) + (c - b - 1);
}

__global__ void __launch_bounds__(IS_THREADS, 2)
    k_itemsets(const uint32_t* const* __restrict__ plane, const ISRow* __restrict__ rows, int nrows,
               int n, const ISUnit* __restrict__ units, int nunits, int* __restrict__ head,
               unsigned long long* pairs, unsigned long long* triples) {
  __shared__ __align__(16) uint32_t xs[IS_ROWS * IS_XS];
  __shared__ __align__(16) uint32_t ys[IS_COLS * IS_TW];
  __shared__ int s_unit;
  __shared__ ISRow s_rows[IS_ROWS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(head, 1);
    __syncthreads();
    const int ui = s_unit;
    if (ui >= nunits) return;
    const ISUnit u = units[ui];
    if (threadIdx.x < IS_ROWS) {
      const int r = u.row0 + threadIdx.x;
      s_rows[threadIdx.x] = r < nrows ? rows[r] : ISRow{-1, -1};
    }
    __syncthreads();
    // per-lane accumulators: 4 rows (lane, lane+32, +64, +96) x 4 columns (warp*4 + j).
    // Carry-save state per output: ones, twos (bit-sliced partial sums) and cnt (# of 4s).
    uint32_t ones[16], twos[16], cnt[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) ones[i] = twos[i] = cnt[i] = 0u;
    for (int64_t w0 = u.w0; w0 < u.w1; w0 += IS_TW) {
      // stage X (AND of the row's two planes) and Y, 4 words per thread-load
      for (int e = threadIdx.x; e < IS_ROWS * (IS_TW / 4); e += IS_THREADS) {
        const int r = e / (IS_TW / 4), q = e % (IS_TW / 4);
        const ISRow rr = s_rows[r];
        uint4 x = make_uint4(0u, 0u, 0u, 0u);
        if (rr.a >= 0) {
          const uint4 pa = *reinterpret_cast<const uint4*>(plane[rr.a] + w0 + 4 * q);
          const uint4 pb = *reinterpret_cast<const uint4*>(plane[rr.b] + w0 + 4 * q);
          x = make_uint4(pa.x & pb.x, pa.y & pb.y, pa.z & pb.z, pa.w & pb.w);
        }
        uint2* d = reinterpret_cast<uint2*>(xs + r * IS_XS + 4 * q);
        d[0] = make_uint2(x.x, x.y);
        d[1] = make_uint2(x.z, x.w);
      }
      for (int e = threadIdx.x; e < IS_COLS * (IS_TW / 4); e += IS_THREADS) {
        const int c = e / (IS_TW / 4), q = e % (IS_TW / 4);
        const int item = u.col0 + c;
        uint4 y = make_uint4(0u, 0u, 0u, 0u);
        if (item < n) y = *reinterpret_cast<const uint4*>(plane[item] + w0 + 4 * q);
        *reinterpret_cast<uint4*>(ys + c * IS_TW + 4 * q) = y;
      }
      __syncthreads();
#pragma unroll 2
      for (int k = 0; k < IS_TW; k += 4) {
        // Harley-Seal over 4 words: ones/twos absorb z_k..z_k+3, every carry into the
        // "fours" place is popcounted once.
        uint32_t tA[16];
        {
          uint32_t x0[4], x1[4], y0[4], y1[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint2 t = *reinterpret_cast<const uint2*>(xs + (lane + 32 * i) * IS_XS + k);
            x0[i] = t.x;
            x1[i] = t.y;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint2 t = *reinterpret_cast<const uint2*>(ys + (warp * 4 + j) * IS_TW + k);
            y0[j] = t.x;
            y1[j] = t.y;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              csa(tA[4 * i + j], ones[4 * i + j], ones[4 * i + j], x0[i] & y0[j], x1[i] & y1[j]);
        }
        {
          uint32_t x2[4], x3[4], y2[4], y3[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint2 t = *reinterpret_cast<const uint2*>(xs + (lane + 32 * i) * IS_XS + k + 2);
            x2[i] = t.x;
            x3[i] = t.y;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint2 t = *reinterpret_cast<const uint2*>(ys + (warp * 4 + j) * IS_TW + k + 2);
            y2[j] = t.x;
            y3[j] = t.y;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int o = 4 * i + j;
              uint32_t tB, f;
              csa(tB, ones[o], ones[o], x2[i] & y2[j], x3[i] & y3[j]);
              csa(f, twos[o], twos[o], tA[o], tB);
              cnt[o] += __popc(f);
            }
        }
      }
      __syncthreads();
    }
    // totals and writes
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = lane + 32 * i;
      const ISRow rr = s_rows[rl];
      if (rr.a < 0) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int o = 4 * i + j;
        const int c = u.col0 + warp * 4 + j;
        if (c >= n || c <= rr.b) continue;
        const unsigned long long tot =
            4ull * cnt[o] + 2ull * __popc(twos[o]) + (unsigned long long)__popc(ones[o]);
        if (!tot) continue;
        if (rr.a == rr.b) atomicAdd(pairs + (int64_t)rr.a * n + c, tot);
        else atomicAdd(triples + triple_index(n, rr.a, rr.b, c), tot);
      }
    }
    __syncthreads();
  }
}

}  // namespace cs
