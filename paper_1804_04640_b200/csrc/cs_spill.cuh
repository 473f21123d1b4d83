// cs_spill.cuh -- K1sp, the spill class: joint tables up to ~3x one SM's shared memory
// (225K .. ~600K cells), between the narrow-counter SMEM class and the partition class.
//
// The reference's radix strategy partitions ALL rows before it counts any (radix.py:33-79).
// Here one pass counts most rows at once and moves only the rest:
//
//   k_spill_hist<K>   (query, row segment) items, one 1024-thread CTA per SM.  The CTA holds the
//                     first T1 = 220K cells of the table as 8-bit SMEM counters (wrap repair as
//                     in the narrow class, cs_kernels.cuh).  A row whose joint index falls below
//                     T1 is counted on the spot; any other row's index is appended to the warp's
//                     private spill stream: one ballot and two popcounts per 32 rows, the
//                     cursor in a warp-uniform register -- no atomics, no shared memory.  A
//                     stream that would overflow (skewed data; streams hold the uniform
//                     expectation plus slack) sends the rows of that vector to the global table
//                     with one RED each instead, so any distribution counts exactly.
//   k_spill_count     (query, 192K-cell group, row segment) items: streams the segment's 32
//                     warp streams into a table of 8-bit counters (entries of other groups
//                     skipped), adds it to the global table.
//
// HBM per row: K/2 B of 4-bit columns + 4 B written and 4 B x groups read for the fraction of
// rows outside the first T1 cells (the partition class moves 4 B for every row and sorts them
// through SMEM first).
#pragma once
#include "cs_common.cuh"

namespace cs {

#ifndef CS_THREADS_N
#define CS_THREADS_N 1024
#endif
constexpr int SP_THREADS = CS_THREADS_N;
constexpr int SP_WARPS = SP_THREADS / 32;
constexpr uint32_t SP_GROUP_CELLS = 3 * 65536;  // cells per k_spill_count item (192 KB of 8-bit counters)
constexpr int SP_MAXG = 8;                      // groups per query the planner may allow
constexpr int SP_COUNT_SMEM = SP_GROUP_CELLS;

struct __align__(16) SDesc {
  const uint8_t* base;     // 4-bit column block
  int64_t table_off;       // first cell of the query's table
  int64_t reg_off;         // wave scratch byte offset of this query's streams
  int64_t cnt_off;         // wave scratch byte offset of the stream entry counts (uint32 each)
  uint32_t coff[CS_MAXK];  // column of digit v at base + coff[v] * 256
  uint32_t rpair[4];       // joint index from SIMD lanes, as QDesc / RDesc
  uint32_t R0, R2, P01;
  uint32_t cells;          // C
  uint32_t t1;             // cells counted in SMEM by k_spill_hist (multiple of 4)
  uint32_t cap;            // entries per stream (multiple of 4, >= 1024)
  int32_t ng;              // groups = ceil((C - t1) / SP_GROUP_CELLS)
  int32_t nseg;            // row segments
  int32_t q;               // query index in the plan
  int32_t pad[3];
};
static_assert(sizeof(SDesc) % 16 == 0, "SDesc layout");

struct SItem {  // k_spill_hist
  int32_t sq, seg;
  int64_t r0, r1;
};

struct CItem {  // k_spill_count
  int32_t sq, grp, seg, pad;
};

// 8-bit counter of cell c in a table at shared address tab, bumped when `on` (predicated, no
// branch): returns the word before the add, 0 when off
__device__ __forceinline__ uint32_t atoms_byte(uint32_t tab, uint32_t c, uint32_t& inc, bool on) {
  uint32_t old;
  asm("shf.l.wrap.b32 %0, 0, 1, %1;" : "=r"(inc) : "r"(c << 3));
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %3, 0;\n\t"
      "mov.u32 %0, 0;\n\t"
      "@p atom.shared.add.u32 %0, [%1], %2;\n\t}"
      : "=r"(old)
      : "r"(tab + (c & ~3u)), "r"(inc), "r"((uint32_t)on)
      : "memory");
  return old;
}
// the counter held 255 before the add (it wrapped to 0 and carried into its neighbour)
__device__ __forceinline__ bool byte_wrapped(uint32_t old, uint32_t inc) { return (~old & (inc * 255u)) == 0u; }

// red.shared form of atoms_byte (no result): the optimistic pass
__device__ __forceinline__ void reds_byte(uint32_t tab, uint32_t c, bool on) {
  uint32_t inc;
  asm("shf.l.wrap.b32 %0, 0, 1, %1;" : "=r"(inc) : "r"(c << 3));
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %2, 0;\n\t"
      "@p red.shared.add.u32 [%0], %1;\n\t}" ::"r"(tab + (c & ~3u)),
      "r"(inc), "r"((uint32_t)on)
      : "memory");
}

// MODE 0: rows of the SMEM range counted optimistically (red.shared, no wrap test; the caller
//         proves the table by its counter sum afterwards), the others appended to the warp's stream;
// MODE 1: the same, but the stream may be full: the other rows go to the global table one by one
//         (slow += how many);
// MODE 2: the exact recount after a failed proof: only the rows of the SMEM range, returning
//         atomics and wrap repairs, nothing spilled again.
template <int K, int MODE>
__device__ __forceinline__ void spill_rows(const uint32_t (&x)[K][4], const uint32_t (&rp)[4], uint32_t R0,
                                           uint32_t R2, uint32_t P01, uint32_t T1, uint32_t C, uint32_t tab,
                                           uint32_t* gtab, uint32_t* reg, uint32_t& cur, uint32_t lt, bool live,
                                           uint32_t& slow) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t idx[4];
      nib_joint4<K>(x, j, h, rp, R0, R2, P01, idx);
      if constexpr (MODE == 2) {
        // all atomics issued before any wrap test reads a result
        uint32_t old[4], inc[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) old[t] = atoms_byte(tab, idx[t], inc[t], live && idx[t] < T1);
        bool wrap = false;
#pragma unroll
        for (int t = 0; t < 4; ++t) wrap |= byte_wrapped(old[t], inc[t]);
        if (wrap) {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (byte_wrapped(old[t], inc[t])) narrow_fix<8>(old[t], idx[t] & 3u, idx[t] & ~3u, C, gtab);
        }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) reds_byte(tab, idx[t], live && idx[t] < T1);
        // the other rows: appended to the warp's stream (or, MODE 1, sent to the table one by one)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const bool out = live && idx[t] >= T1;
          if (MODE == 1) {
            if (out) {
              atomicAdd(gtab + idx[t], 1u);
              ++slow;
            }
          } else {
            // rank among the warp's spilled rows of this slot, one predicated 4-byte store (no
            // branch), cursor advanced by the slot's count
            uint32_t n;
            asm volatile(
                "{\n\t.reg .pred p;\n\t.reg .b32 m, r;\n\t.reg .b64 a;\n\t"
                "setp.ne.u32 p, %4, 0;\n\t"
                "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
                "and.b32 r, m, %3;\n\t"
                "popc.b32 r, r;\n\t"
                "add.u32 r, r, %2;\n\t"
                "mad.wide.u32 a, r, 4, %1;\n\t"
                "@p st.global.u32 [a], %5;\n\t"
                "popc.b32 %0, m;\n\t}"
                : "=r"(n)
                : "l"(reg), "r"(cur), "r"(lt), "r"((uint32_t)out), "r"(idx[t])
                : "memory");
            cur += n;
          }
        }
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(SP_THREADS, 1)
    k_spill_hist(const SDesc* __restrict__ sd, const SItem* __restrict__ items, int nitems,
                 int* __restrict__ head, uint32_t* tables, char* __restrict__ scratch, int force_exact) {
  extern __shared__ uint32_t sh[];
  __shared__ SDesc s_d;
  __shared__ int s_item, s_redo;
  __shared__ unsigned long long s_red[SP_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t tab = (uint32_t)__cvta_generic_to_shared(sh);
  for (;;) {
    if (tid == 0) s_item = atomicAdd(head, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) return;
    const SItem wi = items[it];
    if (tid < (int)(sizeof(SDesc) / 16))
      reinterpret_cast<int4*>(&s_d)[tid] = reinterpret_cast<const int4*>(sd + wi.sq)[tid];
    __syncthreads();
    const SDesc& d = s_d;
    const uint32_t T1 = d.t1, C = d.cells, cap = d.cap;
    for (uint32_t i = tid; i < T1 / 4; i += SP_THREADS) sh[i] = 0u;
    __syncthreads();
    uint32_t* gtab = tables + d.table_off;
    const int64_t stream = (int64_t)wi.seg * SP_WARPS + warp;
    uint32_t* reg = reinterpret_cast<uint32_t*>(scratch + d.reg_off) + stream * (int64_t)cap;
    const uint8_t* rowp = d.base + (wi.r0 >> 1);
    uint32_t co[K], rp[4];
#pragma unroll
    for (int v = 0; v < K; ++v) co[v] = d.coff[v];
#pragma unroll
    for (int p = 0; p < 4; ++p) rp[p] = d.rpair[p];
    const uint32_t R0 = d.R0, R2 = d.R2, P01 = d.P01;
    const int64_t nrows = wi.r1 - wi.r0;
    const int64_t nvec = (nrows + 31) >> 5;
    // every warp runs the same number of iterations (the spill step is warp-collective); a
    // thread past the end of the segment loads nothing and its rows are skipped
    const int64_t niter = (nvec + SP_THREADS - 1) / SP_THREADS;
    uint32_t cur = 0u;   // entries in this warp's stream (warp-uniform)
    uint32_t slow = 0u;  // this thread's rows that went to the global table instead (stream full)
    auto sweep = [&](auto mode) {
      constexpr int MODE = decltype(mode)::value;
      for (int64_t itn = 0; itn < niter; ++itn) {
        const int64_t vi = itn * SP_THREADS + tid;
        const bool live = vi < nvec;
        uint32_t x[K][4];
        if (live) {
          load_vec16<K>(x, rowp + (vi << 4), co);
        } else {
#pragma unroll
          for (int v = 0; v < K; ++v) x[v][0] = x[v][1] = x[v][2] = x[v][3] = 0u;
        }
        if (MODE == 2) {
          spill_rows<K, 2>(x, rp, R0, R2, P01, T1, C, tab, gtab, reg, cur, lt, live, slow);
        } else {
          // a vector appends at most 1024 entries: when they might not fit, its rows go to the table
          if (cur + 1024u <= cap) spill_rows<K, 0>(x, rp, R0, R2, P01, T1, C, tab, gtab, reg, cur, lt, live, slow);
          else spill_rows<K, 1>(x, rp, R0, R2, P01, T1, C, tab, gtab, reg, cur, lt, live, slow);
        }
      }
    };
    sweep(std::integral_constant<int, 0>{});
    __syncthreads();
    if (lane == 0) reinterpret_cast<uint32_t*>(scratch + d.cnt_off)[stream] = cur;
    {
      // proof of the optimistic pass: no counter of a word wrapped exactly when the word's counter
      // sum equals its increments, so sum(all counters) == rows of the SMEM range == rows of the
      // segment's vectors - rows spilled accepts the table; else count the range again, exactly
      unsigned long long part = 0ull;
      for (uint32_t i = tid; i < T1 / 4; i += SP_THREADS) part += __dp4a(sh[i], 0x01010101u, 0u);
      part += (unsigned long long)slow + (lane == 0 ? cur : 0u);
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
      if (lane == 0) s_red[warp] = part;
      __syncthreads();
      if (tid == 0) {
        unsigned long long tot = 0ull;
        for (int w2 = 0; w2 < SP_WARPS; ++w2) tot += s_red[w2];
        s_redo = force_exact || tot != (unsigned long long)(nvec << 5);
      }
      __syncthreads();
      if (s_redo) {
        for (uint32_t i = tid; i < T1 / 4; i += SP_THREADS) sh[i] = 0u;
        __syncthreads();
        sweep(std::integral_constant<int, 2>{});
        __syncthreads();
      }
    }
    // padding rows (zero nibbles, joint index 0) of the last vector were counted into cell 0
    const int64_t pad = (nvec << 5) - nrows;
    if (pad > 0 && tid == 0) atomicSub(gtab, (uint32_t)pad);
    for (uint32_t c = tid; c < T1; c += SP_THREADS) {
      const uint32_t v = (sh[c >> 2] >> ((c & 3u) * 8u)) & 0xffu;
      if (v) atomicAdd(gtab + c, v);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ uint4 ldg_stream_nc16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__global__ void __launch_bounds__(SP_THREADS, 1)
    k_spill_count(const SDesc* __restrict__ sd, const CItem* __restrict__ items, int nitems,
                  int* __restrict__ head, uint32_t* tables, const char* __restrict__ scratch, int force_exact) {
  extern __shared__ uint32_t tabw[];
  __shared__ SDesc s_d;
  __shared__ int s_item, s_redo;
  __shared__ unsigned long long s_red[SP_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t tab = (uint32_t)__cvta_generic_to_shared(tabw);
  for (;;) {
    if (tid == 0) s_item = atomicAdd(head, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) return;
    const CItem wi = items[it];
    if (tid < (int)(sizeof(SDesc) / 16))
      reinterpret_cast<int4*>(&s_d)[tid] = reinterpret_cast<const int4*>(sd + wi.sq)[tid];
    __syncthreads();
    const SDesc& d = s_d;
    const uint32_t cell0 = d.t1 + (uint32_t)wi.grp * SP_GROUP_CELLS;  // first cell of this item
    const uint32_t ncell = min(SP_GROUP_CELLS, d.cells - cell0);
    for (uint32_t i = tid; i < (ncell + 3u) / 4u; i += SP_THREADS) tabw[i] = 0u;
    __syncthreads();
    uint32_t* gt = tables + d.table_off + cell0;
    // warp w streams what source warp w of this segment spilled
    const int64_t stream = (int64_t)wi.seg * SP_WARPS + warp;
    const uint32_t n = __ldg(reinterpret_cast<const uint32_t*>(scratch + d.cnt_off) + stream);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(scratch + d.reg_off) + stream * (int64_t)d.cap;
    // MODE 0: optimistic (red.shared, no wrap test), every entry of the stream is this group's
    //         (one group); MODE 1: optimistic, entries of this group counted as they are found;
    // MODE 2: exact (returning atomics, wrap repairs).  `mine` = entries this thread counted.
    unsigned long long mine = 0ull;
    auto sweep = [&](auto mode) {
      constexpr int MODE = decltype(mode)::value;
      for (uint32_t i = lane * 4u; i < n; i += 256u) {
        uint4 v[2];
        v[0] = ldg_stream_nc16(src + i);
        v[1] = i + 128u < n ? ldg_stream_nc16(src + i + 128u) : make_uint4(0u, 0u, 0u, 0u);
        uint32_t c[8], old[8], inc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint4& w = v[e >> 2];
          c[e] = ((e & 3) == 0 ? w.x : (e & 3) == 1 ? w.y : (e & 3) == 2 ? w.z : w.w) - cell0;
          // entries past the end of the stream and cells of other groups are skipped
          const bool on = i + (e >> 2) * 128u + (e & 3) < n && c[e] < ncell;
          if (MODE == 2) {
            old[e] = atoms_byte(tab, c[e], inc[e], on);
          } else {
            reds_byte(tab, c[e], on);
            if (MODE == 1) mine += on;
          }
        }
        if constexpr (MODE == 2) {
          bool wrap = false;
#pragma unroll
          for (int e = 0; e < 8; ++e) wrap |= byte_wrapped(old[e], inc[e]);
          if (wrap) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (byte_wrapped(old[e], inc[e])) narrow_fix<8>(old[e], c[e] & 3u, c[e] & ~3u, ncell, gt);
          }
        }
      }
    };
    const bool multi = d.ng > 1;
    if (multi) sweep(std::integral_constant<int, 1>{});
    else sweep(std::integral_constant<int, 0>{});
    __syncthreads();
    {
      // proof (as in k_spill_hist): sum of the counters == entries counted, else recount exactly
      long long part = 0;
      for (uint32_t i = tid; i < (ncell + 3u) / 4u; i += SP_THREADS) part += __dp4a(tabw[i], 0x01010101u, 0u);
      part -= multi ? (long long)mine : (lane == 0 ? (long long)n : 0ll);
#pragma unroll
      for (int o = 16; o; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
      if (lane == 0) s_red[warp] = (unsigned long long)part;
      __syncthreads();
      if (tid == 0) {
        long long tot = 0;
        for (int w2 = 0; w2 < SP_WARPS; ++w2) tot += (long long)s_red[w2];
        s_redo = force_exact || tot != 0;
      }
      __syncthreads();
      if (s_redo) {
        for (uint32_t i = tid; i < (ncell + 3u) / 4u; i += SP_THREADS) tabw[i] = 0u;
        __syncthreads();
        sweep(std::integral_constant<int, 2>{});
      }
    }
    __syncthreads();
    for (uint32_t c = tid; c < ncell; c += SP_THREADS) {
      const uint32_t v = (tabw[c >> 2] >> ((c & 3u) * 8u)) & 0xffu;
      if (v) atomicAdd(gt + c, v);
    }
    __syncthreads();
  }
}

}  // namespace cs
