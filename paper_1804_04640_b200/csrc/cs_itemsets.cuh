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
// Input: the items' state-1 planes transposed step-major, pmt[step][item] = 32 bytes (one
// 256-row step of one item; k_pmt_transpose), so every contiguous item range of a step is one
// contiguous chunk.  A loader thread moves each step's chunks -- the B column range and the
// row block's merged a/b item segments (TCSeg) -- with cp.async.bulk into a raw ring
// (mbarrier complete_tx), far ahead of the producers.
//
// Roles (one CTA per SM, 512 TMEM columns).  Producer groups take interleaved steps so several
// per-step latency chains are in flight: an A group's chain is dominated by the completion of
// its tcgen05.st (~800 cycles measured), so up to TC_GA = 4 A groups run (ga <= nb per launch,
// which keeps the stage ring's parity waits unambiguous); TC_GB = 2 B groups.
//   warps 0 .. 4GA-1          : A producers (warp w owns TMEM lanes 32 (w % 4) .. +31 = pair
//                               rows), then the epilogue (tcgen05.ld of the accumulator, 64-bit
//                               atomics into pairs / triples; the groups split the columns)
//   warps 4GA .. 4(GA+GB)-1   : B producers (raw item words -> expanded SMEM stage, fence.proxy.async)
//   warp 4(GA+GB)             : MMA issuer (whole warp, elected lane)
//   warps 4(GA+GB)+1 ..       : TC_LOADERS bulk-copy loaders (elected lane; loader j takes steps g % L == j)
// Pipelines: raw ring raw_full[r] (complete_tx) -> one group's producers -> raw_empty[r];
// operand stages full[s] (one group's 256 arrivals) -> MMA -> tcgen05.commit -> empty[s]; the last MMA of
// a unit commits to d_full, the epilogue arrives on d_empty.  Units (row block, column chunk,
// step range) are planned on the host (cs_itemset_supports): the step axis is cut into
// L2-sized windows and each window's work is split into equal per-CTA pieces, so all SMs
// sweep the same window together.
constexpr int TC_KT = 256;            // data rows (bits) per step = 8 words per plane
constexpr int TC_NMAX = 256;
constexpr int TC_GA = 2;  // A producer groups (4 warps each; per launch ga <= min(TC_GA, nb) are used)
constexpr int TC_GB = 2;  // B producer groups (4 warps each)
constexpr int TC_A_THREADS = 128, TC_B_THREADS = 128;  // per group
constexpr int TC_BT = 2 * TC_NMAX / TC_B_THREADS;       // B tasks per thread per step
constexpr int TC_LOADERS = 4;          // bulk-copy issuing warps (one issue batch per ~700 cycles
                                       // per warp, tools/microbench5.cu)
constexpr int TC_THREADS = TC_GA * TC_A_THREADS + TC_GB * TC_B_THREADS + 32 + 32 * TC_LOADERS;
constexpr int TC_RAWA = 256 * 32;     // max raw A bytes per step: <= 256 item slots
constexpr int TC_MAXSEG = 8;
constexpr int TC_MAXNB = 8, TC_MAXNR = 16;  // operand stages / raw ring slots (runtime <= these;
                                            // the host keeps nr a multiple of TC_LOADERS)

// ring position: slot index and the parity of the slot's current phase
struct TCRing {
  uint32_t slot = 0, phase = 0;
  __device__ __forceinline__ void next(uint32_t n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1;
    }
  }
  __device__ __forceinline__ void step(uint32_t k, uint32_t n) {  // k <= n
    slot += k;
    if (slot >= n) {
      slot -= n;
      phase ^= 1;
    }
  }
  __device__ __forceinline__ TCRing plus(uint32_t k, uint32_t n) const {  // any k
    TCRing r;
    const uint32_t t = slot + k;
    r.slot = t % n;
    r.phase = phase ^ ((t / n) & 1);
    return r;
  }
};

struct TCUnit {
  int32_t row0;   // first pair row (multiple of 128 in the sorted row list)
  int16_t col0;   // first item column
  int16_t ncols;  // N: multiple of 16, <= 256
  int32_t s0, s1; // step range
};

struct TCSeg {    // per row block: the items its rows touch, as contiguous ranges
  int32_t nseg;
  int32_t src[TC_MAXSEG], len[TC_MAXSEG], dst[TC_MAXSEG];  // item, count, raw slot
};

struct TCSlot {
  int16_t sa, sb;  // raw slots of the row's two items
};

__global__ void k_pmt_transpose(const uint32_t* const* __restrict__ plane, int n, int64_t nsteps,
                                uint4* __restrict__ pmt) {
  const int64_t total = nsteps * n * 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int h = (int)(i & 1);
    const int64_t t = i >> 1;
    const int item = (int)(t % n);
    const int64_t st = t / n;
    pmt[i] = __ldg(reinterpret_cast<const uint4*>(plane[item] + st * 8 + 4 * h));
  }
}

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// The spin loop lives inside the asm (CUTLASS's pattern): a C loop over an asm output makes
// the compiler treat everything after it as divergent, which moves every MMA / bulk-copy
// operand through R2UR on each use.
__device__ __forceinline__ void tc_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TC_WAIT;\n\t}" ::"r"(bar),
      "r"(parity), "r"(0x10000u)  // suspend-time hint (ns): sleep instead of spinning
      : "memory");
}

// diagnostic wait (-DCS_TC_PROFILE): adds the cycles spent blocked to acc
__device__ __forceinline__ void tc_wait_t(uint32_t bar, uint32_t parity, long long& acc) {
#ifdef CS_TC_PROFILE
  const long long t0 = clock64();
  tc_wait(bar, parity);
  acc += clock64() - t0;
#else
  tc_wait(bar, parity);
#endif
}

__device__ __forceinline__ long long tc_clock() {
#ifdef CS_TC_PROFILE
  return clock64();
#else
  return 0;
#endif
}

__device__ __forceinline__ void tc_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// one arrival per warp: each lane has ordered its own accesses (fences) before this point;
// __syncwarp orders them before lane 0's release-arrive.  256 per-thread arrivals on one SMEM
// word per step serialised the producers (measured ~1400 cycles per step).
__device__ __forceinline__ void tc_arrive_warp(uint32_t bar, int lane) {
  __syncwarp();
  if (lane == 0) tc_arrive(bar);
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

__device__ __forceinline__ void tc_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_itemsets_tc(const uint4* __restrict__ pmt, int n, const ISRow* __restrict__ rows,
                  const TCSlot* __restrict__ slots, int nrows, const TCSeg* __restrict__ segs,
                  const TCUnit* __restrict__ units, const int32_t* __restrict__ cta_off, int ga, int nb, int cpc,
                  int a_col, int nr, int stage_bytes, int rawa_bytes, int rawb_bytes, unsigned long long* pairs,
                  unsigned long long* triples, int dbg, long long* prof) {
  extern __shared__ __align__(16) uint8_t tc_smem_buf[];  // 16 B suffices for SWIZZLE_NONE (and a
  // larger alignment here would pad the static SMEM of every kernel in this translation unit)
  __shared__ __align__(8) uint64_t bar_full[TC_MAXNB], bar_empty[TC_MAXNB], bar_rfull[TC_MAXNR],
      bar_rempty[TC_MAXNR], bar_dfull, bar_dempty;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t_start = tc_clock();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < nb; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_full[s])),
                   "r"((TC_A_THREADS + TC_B_THREADS) / 32));
      if (s % cpc == 0)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_empty[s / cpc])), "r"(1));
    }
    for (int r = 0; r < nr; ++r) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_rfull[r])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_rempty[r])),
                   "r"((TC_A_THREADS + TC_B_THREADS) / 32));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_dfull)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(&bar_dempty)), "r"(TC_GA * TC_A_THREADS / 32));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const int u_begin = cta_off[blockIdx.x], u_end = cta_off[blockIdx.x + 1];
  uint8_t* const stages = tc_smem_buf;
  uint8_t* const raw = tc_smem_buf + (size_t)nb * stage_bytes;
  const int raw_bytes = rawa_bytes + rawb_bytes;

  if (warp < 4 * TC_GA) {
    // ---------------- A producers (group grp takes steps g % G == grp) + epilogue ----------------
    const int grp = warp >> 2, quad = warp & 3, row = quad * 32 + lane;
    long long pa_raw = 0, pa_empty = 0, pa_dfull = 0, pa_epi = 0, pa_st = 0, pa_lds = 0;
    TCRing rr0, sr0;  // ring positions at the start of the current unit
    uint32_t g = 0;     // CTA step counter at the start of the current unit
    int uc = 0;
    for (int ui = u_begin; ui < u_end; ++ui, ++uc) {
      const TCUnit u = units[ui];
      const int r = u.row0 + row;
      const ISRow rr = r < nrows ? rows[r] : ISRow{-1, -1};
      const TCSlot sl = r < nrows ? slots[r] : TCSlot{0, 0};
      const uint32_t skip = ((uint32_t)grp + ga - g % ga) % ga;  // first own step of the unit
      TCRing rr_ = rr0.plus(skip, nr), sr_ = sr0.plus(skip, nb);
      for (int st = u.s0 + (int)skip; st < u.s1; st += ga, rr_.step(ga, nr), sr_.step(ga, nb)) {
        tc_wait_t(tc_smem(&bar_rfull[rr_.slot]), rr_.phase, pa_raw);
        const long long tq0 = tc_clock();
        const uint8_t* ra = raw + (size_t)rr_.slot * raw_bytes;
        const uint4 a0 = *reinterpret_cast<const uint4*>(ra + sl.sa * 32);
        const uint4 a1 = *reinterpret_cast<const uint4*>(ra + sl.sa * 32 + 16);
        const uint4 b0 = *reinterpret_cast<const uint4*>(ra + sl.sb * 32);
        const uint4 b1 = *reinterpret_cast<const uint4*>(ra + sl.sb * 32 + 16);
        tc_arrive_warp(tc_smem(&bar_rempty[rr_.slot]), lane);
        pa_lds += tc_clock() - tq0;
        const uint32_t x[8] = {a0.x & b0.x, a0.y & b0.y, a0.z & b0.z, a0.w & b0.w,
                               a1.x & b1.x, a1.y & b1.y, a1.z & b1.z, a1.w & b1.w};
        tc_wait_t(tc_smem(&bar_empty[sr_.slot / cpc]), sr_.phase ^ 1, pa_empty);
        // order the stage's TMEM stores after the MMAs that read it (released by the commit)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + a_col + sr_.slot * 64;
        const long long ts0 = tc_clock();
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          if (dbg & 4) break;
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
        tc_arrive_warp(tc_smem(&bar_full[sr_.slot]), lane);
        pa_st += tc_clock() - ts0;
      }
      rr0 = rr0.plus(u.s1 - u.s0, nr);
      sr0 = sr0.plus(u.s1 - u.s0, nb);
      g += u.s1 - u.s0;
      // epilogue: accumulator lane = pair row, columns 0..ncols-1 = items col0..; the groups
      // split the 16-column chunks
      tc_wait_t(tc_smem(&bar_dfull), uc & 1, pa_dfull);
      const long long te0 = tc_clock();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t td = tmem + ((uint32_t)(quad * 32) << 16);
      for (int j0 = 16 * grp; j0 < u.ncols; j0 += 16 * TC_GA) {
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
      tc_arrive_warp(tc_smem(&bar_dempty), lane);
      pa_epi += tc_clock() - te0;
    }
    if (prof && lane == 0 && warp == 0) {
      atomicAdd((unsigned long long*)&prof[0], (unsigned long long)pa_raw);
      atomicAdd((unsigned long long*)&prof[1], (unsigned long long)pa_empty);
      atomicAdd((unsigned long long*)&prof[2], (unsigned long long)pa_dfull);
      atomicAdd((unsigned long long*)&prof[3], (unsigned long long)pa_epi);
      atomicAdd((unsigned long long*)&prof[13], (unsigned long long)pa_lds);
      atomicAdd((unsigned long long*)&prof[14], (unsigned long long)pa_st);
    }
  } else if (warp < 4 * (TC_GA + TC_GB)) {
    // ---------------- B producers ----------------
    const int grp = (warp - 4 * TC_GA) >> 2, bt = tid - TC_GA * TC_A_THREADS - TC_B_THREADS * grp;
    long long pb_raw = 0, pb_empty = 0;
    TCRing rr0, sr0;
    uint32_t g = 0;
    for (int ui = u_begin; ui < u_end; ++ui) {
      const TCUnit u = units[ui];
      const int N = u.ncols;
      // tasks e = bt + 128 k over (item il = e % N, half h = e / N): 4 words -> 4 x 32 bytes
      int roff[TC_BT], h4[TC_BT];
      uint32_t dst[TC_BT];
#pragma unroll
      for (int k = 0; k < TC_BT; ++k) {
        const int e = bt + TC_B_THREADS * k;
        dst[k] = 0xffffffffu;
        roff[k] = h4[k] = 0;
        if (e < 2 * N) {
          const int il = e % N, h = e / N;
          h4[k] = 4 * h;
          roff[k] = rawa_bytes + il * 32 + 16 * h;
          dst[k] = (uint32_t)((il >> 3) * 2048 + (il & 7) * 16);
        }
      }
      const uint32_t skip = ((uint32_t)grp + TC_GB - g % TC_GB) % TC_GB;
      TCRing rr_ = rr0.plus(skip, nr), sr_ = sr0.plus(skip, nb);
      rr0 = rr0.plus(u.s1 - u.s0, nr);
      sr0 = sr0.plus(u.s1 - u.s0, nb);
      g += u.s1 - u.s0;
      for (int st = u.s0 + (int)skip; st < u.s1; st += TC_GB, rr_.step(TC_GB, nr), sr_.step(TC_GB, nb)) {
        tc_wait_t(tc_smem(&bar_rfull[rr_.slot]), rr_.phase, pb_raw);
        const uint8_t* rb = raw + (size_t)rr_.slot * raw_bytes;
        uint4 cur[TC_BT];
#pragma unroll
        for (int k = 0; k < TC_BT; ++k)
          if (dst[k] != 0xffffffffu) cur[k] = *reinterpret_cast<const uint4*>(rb + roff[k]);
        tc_arrive_warp(tc_smem(&bar_rempty[rr_.slot]), lane);
        tc_wait_t(tc_smem(&bar_empty[sr_.slot / cpc]), sr_.phase ^ 1, pb_empty);
        uint8_t* sp = stages + (size_t)sr_.slot * stage_bytes;
#pragma unroll
        for (int k = 0; k < TC_BT; ++k) {
          if (dst[k] == 0xffffffffu || (dbg & 8)) continue;
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
            *reinterpret_cast<uint4*>(sp + dst[k] + (2 * q) * 128) = lo;
            *reinterpret_cast<uint4*>(sp + dst[k] + (2 * q + 1) * 128) = hi;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_arrive_warp(tc_smem(&bar_full[sr_.slot]), lane);
      }
    }
    if (prof && bt == 0 && grp == 0) {
      atomicAdd((unsigned long long*)&prof[4], (unsigned long long)pb_raw);
      atomicAdd((unsigned long long*)&prof[5], (unsigned long long)pb_empty);
    }
  } else if (warp == 4 * (TC_GA + TC_GB)) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the loop (its operands stay warp-uniform, in uniform registers) and
    // one elected lane issues; a single divergent lane would move every operand through
    // R2UR per instruction (~100 cycles per MMA, measured).
    TCRing sr_;
    int uc = 0, gsub = 0, gidx = 0;  // position inside the current commit group / group index
    long long pm_full = 0, pm_dempty = 0, pm_issue = 0;
    const uint32_t stage0 = tc_smem(stages);
    const uint64_t sdesc0 = tc_sdesc(stage0);
    for (int ui = u_begin; ui < u_end; ++ui, ++uc) {
      const int ncols = __shfl_sync(0xffffffffu, (int)units[ui].ncols, 0);
      const int s0 = __shfl_sync(0xffffffffu, units[ui].s0, 0), s1 = __shfl_sync(0xffffffffu, units[ui].s1, 0);
      // idesc: D s32 (bits 4-5 = 2), A/B u8, K-major, N >> 3 at bit 17, M >> 4 at bit 24
      const uint32_t idesc = (2u << 4) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      tc_wait_t(tc_smem(&bar_dempty), (uc & 1) ^ 1, pm_dempty);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t acc0 = 0;
      for (int st = s0; st < s1; ++st) {
        tc_wait_t(tc_smem(&bar_full[sr_.slot]), sr_.phase, pm_full);
        const long long ti0 = tc_clock();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem + a_col + sr_.slot * 64;
        // descriptor start address advances 256 B (16 in 16-byte units) per K = 32 slice
        const uint64_t db = sdesc0 + (uint64_t)((sr_.slot * (uint32_t)stage_bytes) >> 4);
        if (!(dbg & 2))
          asm volatile(
              "{\n\t.reg .pred e, p;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%5], %6, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%7], %8, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%9], %10, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%11], %12, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%13], %14, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%15], %16, %3, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%17], %18, %3, 1;\n\t}" ::"r"(tmem),
              "r"(ta), "l"(db), "r"(idesc), "r"(acc0), "r"(ta + 8), "l"(db + 16), "r"(ta + 16), "l"(db + 32),
              "r"(ta + 24), "l"(db + 48), "r"(ta + 32), "l"(db + 64), "r"(ta + 40), "l"(db + 80), "r"(ta + 48),
              "l"(db + 96), "r"(ta + 56), "l"(db + 112)
              : "memory");
        // one commit per group of cpc stages (a commit stalls the issue of short MMAs by ~200
        // cycles, tools/microbench6.cu)
        if (++gsub == cpc) {
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                  tc_smem(&bar_empty[gidx]))
              : "memory");
          gsub = 0;
          if (++gidx == nb / cpc) gidx = 0;
        }
        acc0 = 1;
        sr_.next(nb);
        pm_issue += tc_clock() - ti0;
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
              tc_smem(&bar_dfull))
          : "memory");
    }
    if (prof && lane == 0) {
      atomicAdd((unsigned long long*)&prof[6], (unsigned long long)pm_full);
      atomicAdd((unsigned long long*)&prof[7], (unsigned long long)pm_dempty);
      atomicAdd((unsigned long long*)&prof[8], (unsigned long long)pm_issue);
    }
  } else {
    // ---------------- bulk-copy loaders (whole warps, elected issue; loader j takes steps g % L == j) --------
    const int lw = warp - 4 * (TC_GA + TC_GB) - 1;
    TCRing rr0;
    uint32_t g = 0;
    long long pl_empty = 0, pl_issue = 0;
    const uint32_t raw0 = tc_smem(raw);
    for (int ui = u_begin; ui < u_end; ++ui) {
      const int row0 = __shfl_sync(0xffffffffu, units[ui].row0, 0);
      const int col0 = __shfl_sync(0xffffffffu, (int)units[ui].col0, 0);
      const int ncols = __shfl_sync(0xffffffffu, (int)units[ui].ncols, 0);
      const int s0 = __shfl_sync(0xffffffffu, units[ui].s0, 0), s1 = __shfl_sync(0xffffffffu, units[ui].s1, 0);
      const TCSeg& sg = segs[row0 / 128];
      uint32_t soff[TC_MAXSEG], doff[TC_MAXSEG], nby[TC_MAXSEG];
      uint32_t bytes = 0;
#pragma unroll
      for (int k = 0; k < TC_MAXSEG; ++k) {
        const bool on = k < sg.nseg;
        soff[k] = on ? 32u * sg.src[k] : 0u;
        doff[k] = on ? 32u * sg.dst[k] : 0u;
        nby[k] = on ? 32u * sg.len[k] : 0u;
        bytes += nby[k];
      }
      const uint32_t nbb = 32u * (uint32_t)min(ncols, n - col0);
      bytes += nbb;
      const uint32_t skip = ((uint32_t)lw + TC_LOADERS - g % TC_LOADERS) % TC_LOADERS;
      TCRing rr_ = rr0.plus(skip, nr);
      rr0 = rr0.plus(s1 - s0, nr);
      g += s1 - s0;
      for (int st = s0 + (int)skip; st < s1; st += TC_LOADERS, rr_.step(TC_LOADERS, nr)) {
        tc_wait_t(tc_smem(&bar_rempty[rr_.slot]), rr_.phase ^ 1, pl_empty);
        const long long tl0 = tc_clock();
        const uint32_t bar = tc_smem(&bar_rfull[rr_.slot]);
        const char* base = reinterpret_cast<const char*>(pmt) + (int64_t)st * n * 32;
        const uint32_t rdst = raw0 + rr_.slot * raw_bytes;
        if (dbg & 1) {
          if (lane == 0) tc_arrive(bar);
        } else {
          asm volatile(
              "{\n\t.reg .pred e, p;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
              "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %4, [%0];\n\t"
              "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%5], [%6], %7, [%0];\n\t"
              "setp.ne.and.u32 p, %10, 0, e;\n\t"
              "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%8], [%9], %10, [%0];\n\t"
              "setp.ne.and.u32 p, %13, 0, e;\n\t"
              "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%11], [%12], %13, [%0];\n\t"
              "}" ::"r"(bar),
              "r"(bytes), "r"(rdst + (uint32_t)rawa_bytes), "l"(base + 32 * col0), "r"(nbb), "r"(rdst + doff[0]),
              "l"(base + soff[0]), "r"(nby[0]), "r"(rdst + doff[1]), "l"(base + soff[1]), "r"(nby[1]),
              "r"(rdst + doff[2]), "l"(base + soff[2]), "r"(nby[2])
              : "memory");
#pragma unroll
          for (int k = 3; k < TC_MAXSEG; ++k)
            if (nby[k] && lane == 0) tc_bulk(rdst + doff[k], base + soff[k], nby[k], bar);
        }
        pl_issue += tc_clock() - tl0;
      }
    }
    if (prof && lane == 0 && lw == 0) {
      atomicAdd((unsigned long long*)&prof[9], (unsigned long long)pl_empty);
      atomicAdd((unsigned long long*)&prof[10], (unsigned long long)pl_issue);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (prof && tid == 0) {
    atomicAdd((unsigned long long*)&prof[11], (unsigned long long)(tc_clock() - t_start));
    atomicMax((unsigned long long*)&prof[12], (unsigned long long)(tc_clock() - t_start));
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace cs
