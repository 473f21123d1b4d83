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

// ---------------------------------------------------------------------------------------------
// K4c: the same bit-GEMM on the 5th-generation tensor cores (tcgen05.mma kind::i8).
//
// Bits are expanded to 0/1 bytes and multiplied as u8 x u8 -> s32:  S[r, c] = sum_k X_r[k] P_c[k].
// Per 256-row step a CTA expands its 128 pair rows (A, M = 128) straight into TMEM with
// tcgen05.st and its N <= 256 item columns (B) into a K-major SWIZZLE_NONE core-matrix stage in
// shared memory; one thread issues eight 128 x N x 32 MMAs into a TMEM accumulator (int32,
// columns 0..N-1, lane = pair row).  K order inside a step is permuted so the expansion is two
// ops per 4 bytes: byte j of 32-bit column 8q + i holds bit 8j + i of the step's word q (both
// operands use the same permutation, so the dot products are unchanged).
//
// Roles (416 threads, one CTA per SM, 512 TMEM columns):
//   warps 0-3  : A producers (thread t owns TMEM lane t = pair row t), then the epilogue
//                (tcgen05.ld of the accumulator, 64-bit atomics into pairs / triples)
//   warps 4-11 : B producers (item planes -> expanded SMEM stage, fence.proxy.async)
//   warp 12    : MMA issuer (lane 0)
// Pipelining: TC_STAGES stages; full[s] (384 producer arrivals) -> MMA -> tcgen05.commit ->
// empty[s]; the last MMA of a unit commits to d_full, the epilogue arrives on d_empty.
// Units (row block, column chunk, word range) are planned on the host: equal-cost split-K
// pieces, LPT-assigned per CTA and sorted by word offset so the SMs sweep the planes together.
constexpr int TC_KT = 256;            // data rows (bits) per step = 8 words per plane
constexpr int TC_STAGES = 3;
constexpr int TC_NMAX = 256;
constexpr int TC_STAGE_BYTES = TC_NMAX * TC_KT;  // 64 KB
constexpr int TC_THREADS = 416;
constexpr int TC_A_THREADS = 128, TC_B_THREADS = 256;
constexpr uint32_t TC_A_COL = 256;    // first TMEM column of the A stages (64 columns each)

struct TCUnit {
  int32_t row0;   // first pair row (multiple of 128 in the sorted row list)
  int16_t col0;   // first item column
  int16_t ncols;  // N: multiple of 16, <= 256
  int64_t w0, w1; // word range (multiples of 8)
};

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tc_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void tc_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ uint64_t tc_sdesc(uint32_t addr) {
  // K-major, no swizzle: LBO = 128 B (next 16-byte K chunk), SBO = 2048 B (next 8-row group)
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ uint4 tc_ld4(const uint32_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_itemsets_tc(const uint32_t* const* __restrict__ plane, const ISRow* __restrict__ rows, int nrows, int n,
                  const TCUnit* __restrict__ units, const int32_t* __restrict__ cta_off,
                  unsigned long long* pairs, unsigned long long* triples) {
  extern __shared__ __align__(16) uint8_t tc_stage[];  // 16 B suffices for SWIZZLE_NONE (and a
  // larger alignment here would pad the static SMEM of every kernel in this translation unit)
  __shared__ __align__(8) uint64_t bar_full[TC_STAGES], bar_empty[TC_STAGES], bar_dfull, bar_dempty;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < TC_STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_full[s])),
                   "r"(TC_A_THREADS + TC_B_THREADS));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_empty[s])), "r"(1));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_dfull)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_dempty)), "r"(TC_A_THREADS));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const int u_begin = cta_off[blockIdx.x], u_end = cta_off[blockIdx.x + 1];
  const uint32_t stage0 = tc_smem(tc_stage);

  if (warp < 4) {
    // ---------------- A producers + epilogue ----------------
    uint32_t g = 0;  // global step counter of this CTA
    int uc = 0;
    for (int ui = u_begin; ui < u_end; ++ui, ++uc) {
      const TCUnit u = units[ui];
      const int r = u.row0 + tid;
      const ISRow rr = r < nrows ? rows[r] : ISRow{-1, -1};
      const uint32_t* pa = rr.a >= 0 ? plane[rr.a] : nullptr;
      const uint32_t* pb = rr.a >= 0 ? plane[rr.b] : nullptr;
      uint4 c0 = make_uint4(0, 0, 0, 0), c1 = c0;
      if (pa) {
        const uint4 a0 = tc_ld4(pa + u.w0), a1 = tc_ld4(pa + u.w0 + 4), b0 = tc_ld4(pb + u.w0),
                    b1 = tc_ld4(pb + u.w0 + 4);
        c0 = make_uint4(a0.x & b0.x, a0.y & b0.y, a0.z & b0.z, a0.w & b0.w);
        c1 = make_uint4(a1.x & b1.x, a1.y & b1.y, a1.z & b1.z, a1.w & b1.w);
      }
      for (int64_t w = u.w0; w < u.w1; w += 8, ++g) {
        uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0;
        if (pa && w + 8 < u.w1) {
          const uint4 a0 = tc_ld4(pa + w + 8), a1 = tc_ld4(pa + w + 12), b0 = tc_ld4(pb + w + 8),
                      b1 = tc_ld4(pb + w + 12);
          n0 = make_uint4(a0.x & b0.x, a0.y & b0.y, a0.z & b0.z, a0.w & b0.w);
          n1 = make_uint4(a1.x & b1.x, a1.y & b1.y, a1.z & b1.z, a1.w & b1.w);
        }
        const uint32_t s = g % TC_STAGES;
        tc_wait(tc_smem(&bar_empty[s]), ((g / TC_STAGES) & 1) ^ 1);
        const uint32_t x[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + TC_A_COL + s * 64;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t v[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            v[i] = (x[2 * h] >> i) & 0x01010101u;
            v[8 + i] = (x[2 * h + 1] >> i) & 0x01010101u;
          }
          tc_st16(ta + 16 * h, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        tc_arrive(tc_smem(&bar_full[s]));
        c0 = n0;
        c1 = n1;
      }
      // epilogue: accumulator lane tid = pair row, columns 0..ncols-1 = items col0..
      tc_wait(tc_smem(&bar_dfull), uc & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t td = tmem + ((uint32_t)(warp * 32) << 16);
      for (int j0 = 0; j0 < u.ncols; j0 += 16) {
        uint32_t v[16];
        tc_ld16(td + j0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (rr.a < 0) continue;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = u.col0 + j0 + i;
          if (c <= rr.b || c >= n || v[i] == 0) continue;
          if (rr.a == rr.b) atomicAdd(pairs + (int64_t)rr.a * n + c, (unsigned long long)v[i]);
          else atomicAdd(triples + triple_index(n, rr.a, rr.b, c), (unsigned long long)v[i]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      tc_arrive(tc_smem(&bar_dempty));
    }
  } else if (warp < 12) {
    // ---------------- B producers ----------------
    const int bt = tid - TC_A_THREADS;
    uint32_t g = 0;
    for (int ui = u_begin; ui < u_end; ++ui) {
      const TCUnit u = units[ui];
      const int N = u.ncols;
      // tasks e = bt, bt + 256 over (item il = e % N, half h = e / N): 4 words -> 32 bytes x 4
      const uint32_t* src[2];
      uint32_t dst[2];
      int h4[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int e = bt + TC_B_THREADS * k;
        src[k] = nullptr;
        dst[k] = 0xffffffffu;
        h4[k] = 0;
        if (e < 2 * N) {
          const int il = e % N, h = e / N, item = u.col0 + il;
          h4[k] = 4 * h;
          dst[k] = (uint32_t)((il >> 3) * 2048 + (il & 7) * 16);
          if (item < n) src[k] = plane[item] + 4 * h;
        }
      }
      uint4 cur[2], nxt[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) cur[k] = src[k] ? tc_ld4(src[k] + u.w0) : make_uint4(0, 0, 0, 0);
      for (int64_t w = u.w0; w < u.w1; w += 8, ++g) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
          nxt[k] = (src[k] && w + 8 < u.w1) ? tc_ld4(src[k] + w + 8) : make_uint4(0, 0, 0, 0);
        const uint32_t s = g % TC_STAGES;
        tc_wait(tc_smem(&bar_empty[s]), ((g / TC_STAGES) & 1) ^ 1);
        uint8_t* st = tc_stage + (size_t)s * TC_STAGE_BYTES;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          if (dst[k] == 0xffffffffu) continue;
          const uint32_t x[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int q = h4[k] + qq;  // word of the step -> chunks 2q, 2q + 1
            uint4 lo, hi;
            lo.x = x[qq] & 0x01010101u;
            lo.y = (x[qq] >> 1) & 0x01010101u;
            lo.z = (x[qq] >> 2) & 0x01010101u;
            lo.w = (x[qq] >> 3) & 0x01010101u;
            hi.x = (x[qq] >> 4) & 0x01010101u;
            hi.y = (x[qq] >> 5) & 0x01010101u;
            hi.z = (x[qq] >> 6) & 0x01010101u;
            hi.w = (x[qq] >> 7) & 0x01010101u;
            *reinterpret_cast<uint4*>(st + dst[k] + (2 * q) * 128) = lo;
            *reinterpret_cast<uint4*>(st + dst[k] + (2 * q + 1) * 128) = hi;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_arrive(tc_smem(&bar_full[s]));
        cur[0] = nxt[0];
        cur[1] = nxt[1];
      }
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer ----------------
    uint32_t g = 0;
    int uc = 0;
    for (int ui = u_begin; ui < u_end; ++ui, ++uc) {
      const TCUnit u = units[ui];
      // idesc: D s32 (bits 4-5 = 2), A/B u8, K-major, N >> 3 at bit 17, M >> 4 at bit 24
      const uint32_t idesc = (2u << 4) | ((uint32_t)(u.ncols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      tc_wait(tc_smem(&bar_dempty), (uc & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      bool first = true;
      for (int64_t w = u.w0; w < u.w1; w += 8, ++g) {
        const uint32_t s = g % TC_STAGES;
        tc_wait(tc_smem(&bar_full[s]), (g / TC_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem + TC_A_COL + s * 64;
        const uint32_t sb = stage0 + s * TC_STAGE_BYTES;
#pragma unroll
        for (int j = 0; j < TC_KT / 32; ++j) {
          const uint32_t acc = (first && j == 0) ? 0u : 1u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(ta + 8u * j), "l"(tc_sdesc(sb + 256u * j)), "r"(idesc), "r"(acc)
              : "memory");
        }
        first = false;
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         tc_smem(&bar_empty[s]))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tc_smem(&bar_dfull))
                   : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace cs
