// cs_radix.cuh -- K1r, the partition class: joint tables above SMEM capacity (C <= 2^24 cells).
//
// The reference's radix strategy counts by successive counting-sort levels over the rows
// (radix.py:33-79 `_partition_level`: per-segment histogram, prefix, scatter of row ids).  On
// the GPU one such level is enough: rows are partitioned by the high bits of their joint index
// so that each partition's cells fit one SM's shared memory, then every partition is counted
// with an SMEM histogram.  This replaces RED.ADD into L2-resident global tables (one L2 atomic
// per row) and the slice class (columns re-read once per slice) for tables of 56K..16M cells.
//
//   k_radix_part<K>   one chunk of RX_CH (4096) rows per CTA iteration: joint index of every row
//                     from the 4-bit columns (16-bit SIMD lanes), SMEM histogram of the bucket
//                     ids (idx >> bb), exclusive scan, counting-sort scatter of the low 15 bits
//                     of idx into an SMEM stage, one coalesced store of the stage (8 KB) plus the
//                     chunk's bucket offsets.  HBM per row: K/2 B read + 2 B written.
//   k_radix_count     (query, 32K-cell group, chunk range) items: each lane streams the run of
//                     one chunk that falls in the group (buckets are sorted inside a chunk, and
//                     a group is 2^(15-bb) consecutive buckets, so the run is contiguous) with
//                     16-B loads into a 128 KB SMEM table, then adds the table into the global
//                     one.  HBM per row: 2 B read.
#pragma once
#include "cs_common.cuh"

namespace cs {

#ifndef CS_RX_THREADS_N
#define CS_RX_THREADS_N 128
#endif
constexpr int RX_THREADS = CS_RX_THREADS_N;  // 1024 / RX_THREADS CTAs per SM (128: 8 CTAs whose barriers
                                             // sync 4 warps each, 252 against 265 us per k = 8 query at 256)
constexpr int RX_CH = RX_THREADS * 32;  // rows per chunk: one 16-B nibble vector per thread and column
constexpr int RX_GROUP_BITS = 15;       // cells per count group (128 KB SMEM table)
constexpr int RX_MAX_NB = 512;          // partition buckets per query
constexpr int RX_NBPT = RX_MAX_NB / RX_THREADS;  // buckets scanned per k_radix_part thread
constexpr int RX_SMEM = RX_CH * 4 + RX_CH * 2 + (RX_MAX_NB + 1) * 4;  // 4 CTAs per SM
constexpr int RC_THREADS = 1024;
constexpr int RC_DUMMY = 1 << RX_GROUP_BITS;          // counter for entries outside a run
constexpr int RC_SMEM = ((1 << RX_GROUP_BITS) + 32) * 4;

// Everything the partition kernels need about one query, precomputed on the host so a CTA
// reloads it only when its item stream crosses into the next query.
struct RDesc {
  const uint8_t* base;  // 4-bit column block
  int64_t buf_off;      // wave scratch byte offset: nchunks x RX_CH staged local indices (idx & 0x7fff)
  int64_t choff_off;    // wave scratch byte offset: nchunks x (nb + 1) bucket offsets per chunk stage
  uint32_t coff[CS_MAXK];  // column of digit v at base + coff[v] * 256
  // joint index of digits d0..d7 (arities r0..r7 <= 16, missing digits 0):
  //   b_p = d_2p + r_2p d_2p+1 (< 256, byte lanes),  lo = b0 + R0 b1,  hi = b2 + R2 b3 (< 65536,
  //   16-bit lanes),  idx = lo + P01 hi   with R0 = r0 r1, R2 = r4 r5, P01 = r0 r1 r2 r3
  uint32_t rpair[4];       // r0, r2, r4, r6
  uint32_t R0, R2, P01;
  uint32_t pad0[CS_MAXK * 3 - 7];
  int32_t q;            // QDesc index
  int32_t bb;           // log2 cells per partition bucket (10..15)
  int32_t nb;           // buckets = ceil(C / 2^bb) <= RX_MAX_NB
  uint32_t plo;         // unused
  int32_t wlog;         // k_radix_count: log2 lanes that stream one chunk's run together (2..5)
  int32_t pad[5];
};
static_assert(sizeof(RDesc) == 192, "RDesc layout");

struct RItem {
  int32_t rq;   // RDesc index
  int32_t grp;  // 32K-cell group
  int32_t c0;   // chunk range [c0, c1)
  int32_t c1;
};

// Joint indices of one thread's 32-row nibble vector.  Digits are paired in byte lanes
// (b_p = d_2p + r_2p d_2p+1 < 256 since arities <= 16), the two pairs of each half combined in
// 16-bit lanes (lo = b0 + R0 b1 < r0 r1 r2 r3 <= 65536, hi = b2 + R2 b3 <= 65535), and
// idx = lo + P01 hi per row: no per-query lane classes, no data-dependent control flow.  Each
// row's index goes to sidx and bumps its bucket counter.  Rows past the end of the database
// (FULL = false only) go to the dummy bucket nb, which sorts after every real bucket and is
// never staged for counting.
template <int K, bool FULL>
__device__ __forceinline__ void radix_rows(const uint32_t (&x)[K][4], const uint32_t (&rp)[4], uint32_t R0,
                                           uint32_t R2, uint32_t P01, int bb, uint32_t dummy, int64_t nvalid,
                                           uint32_t* sidx, uint32_t* cnt) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t w[8];
#pragma unroll
      for (int v = 0; v < 8; ++v)
        w[v] = v < K ? (h ? (x[v < K ? v : 0][j] >> 4) & 0x0f0f0f0fu : x[v < K ? v : 0][j] & 0x0f0f0f0fu) : 0u;
      uint32_t b[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) b[p] = 2 * p + 1 < K ? w[2 * p] + w[2 * p + 1] * rp[p] : w[2 * p];
      uint32_t lo01 = __byte_perm(b[0], 0u, 0x4140), lo23 = __byte_perm(b[0], 0u, 0x4342);
      if (K > 2) {
        lo01 += __byte_perm(b[1], 0u, 0x4140) * R0;
        lo23 += __byte_perm(b[1], 0u, 0x4342) * R0;
      }
      uint32_t idx[4];
      if (K > 4) {
        uint32_t hi01 = __byte_perm(b[2], 0u, 0x4140), hi23 = __byte_perm(b[2], 0u, 0x4342);
        if (K > 6) {
          hi01 += __byte_perm(b[3], 0u, 0x4140) * R2;
          hi23 += __byte_perm(b[3], 0u, 0x4342) * R2;
        }
        idx[0] = (lo01 & 0xffffu) + P01 * (hi01 & 0xffffu);
        idx[1] = (lo01 >> 16) + P01 * (hi01 >> 16);
        idx[2] = (lo23 & 0xffffu) + P01 * (hi23 & 0xffffu);
        idx[3] = (lo23 >> 16) + P01 * (hi23 >> 16);
      } else {
        idx[0] = lo01 & 0xffffu;
        idx[1] = lo01 >> 16;
        idx[2] = lo23 & 0xffffu;
        idx[3] = lo23 >> 16;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = 8 * j + 2 * q + h;  // row inside the 32-row vector
        const uint32_t i = (FULL || rr < nvalid) ? idx[q] : dummy;
        sidx[rr * RX_THREADS + tid] = i;
        atomicAdd(&cnt[i >> bb], 1u);
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(RX_THREADS, 1024 / RX_THREADS)
    k_radix_part(const RDesc* __restrict__ rd, int nrq, int nchunks, int64_t m, char* __restrict__ scratch) {
  extern __shared__ uint32_t rsm[];
  uint32_t* sidx = rsm;                                        // [32][RX_THREADS] joint indices
  uint16_t* stage = reinterpret_cast<uint16_t*>(rsm + RX_CH);  // RX_CH local indices, bucket-sorted
  uint32_t* cnt = rsm + RX_CH + RX_CH / 2;                     // bucket counts, then cursors
  __shared__ uint32_t s_wsum[RX_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if ((int64_t)blockIdx.x >= (int64_t)nrq * nchunks) return;
  // items (query rq, chunk c) in grid-stride order without a division per item
  int rq = (int)(blockIdx.x / nchunks), c = (int)(blockIdx.x % nchunks);
  int cur = -1;
  bool have = false;  // x already holds this item's vectors (prefetched during the last item)
  uint32_t x[K][4];
  auto load_vectors = [&](uint32_t (&xx)[K][4], const uint8_t* b, const uint32_t (&co)[K], int64_t r0) {
    if (r0 < m) {
      const uint8_t* p = b + (r0 >> 1);
#pragma unroll
      for (int v = 0; v < K; ++v) {
        const uint4 t = ldg_stream16(p + ((uint64_t)co[v] << 8));
        xx[v][0] = t.x;
        xx[v][1] = t.y;
        xx[v][2] = t.z;
        xx[v][3] = t.w;
      }
    } else {
#pragma unroll
      for (int v = 0; v < K; ++v) xx[v][0] = xx[v][1] = xx[v][2] = xx[v][3] = 0u;
    }
  };
  const uint8_t* base = nullptr;
  uint32_t coff[K], rp[4], R0 = 0, R2 = 0, P01 = 0;
  int nb = 0, bb = 0;
  char* buf = nullptr;
  int32_t* choff = nullptr;
  for (; rq < nrq;) {
    if (rq != cur) {  // CTA-uniform: reload the query's descriptor
      const RDesc& r = rd[rq];
      base = r.base;
#pragma unroll
      for (int v = 0; v < K; ++v) coff[v] = r.coff[v];
#pragma unroll
      for (int p = 0; p < 4; ++p) rp[p] = r.rpair[p];
      R0 = r.R0;
      R2 = r.R2;
      P01 = r.P01;
      nb = r.nb;
      bb = r.bb;
      buf = scratch + r.buf_off;
      choff = reinterpret_cast<int32_t*>(scratch + r.choff_off);
      cur = rq;
    }
    for (int i = tid; i <= nb; i += RX_THREADS) cnt[i] = 0u;
    const int64_t row0 = (int64_t)c * RX_CH + (int64_t)tid * 32;
    if (!have) load_vectors(x, base, coff, row0);
    const int64_t nvalid = m - row0;  // rows of this thread's vector that exist (may be <= 0)
    const uint32_t dummy = (uint32_t)nb << bb;
    __syncthreads();  // cnt zeroed
    if (nvalid >= 32) radix_rows<K, true>(x, rp, R0, R2, P01, bb, dummy, nvalid, sidx, cnt);
    else radix_rows<K, false>(x, rp, R0, R2, P01, bb, dummy, nvalid, sidx, cnt);
    // next item; its column vectors are fetched now (x is free) and land while this item's
    // scan, scatter and store run.  Only within the same query (the descriptor is loaded).
    int c2 = c + gridDim.x, rq2 = rq;
    while (c2 >= nchunks) {
      c2 -= nchunks;
      ++rq2;
    }
    have = rq2 == rq;
    if (have) load_vectors(x, base, coff, (int64_t)c2 * RX_CH + (int64_t)tid * 32);
    __syncthreads();
    // exclusive scan of the bucket counts, RX_NBPT consecutive buckets per thread; the dummy
    // bucket nb goes last
    uint32_t cv[RX_NBPT];
    uint32_t mine = 0u;
#pragma unroll
    for (int u = 0; u < RX_NBPT; ++u) {
      cv[u] = RX_NBPT * tid + u < nb ? cnt[RX_NBPT * tid + u] : 0u;
      mine += cv[u];
    }
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0u, nstaged = 0u;
#pragma unroll
    for (int w2 = 0; w2 < RX_THREADS / 32; ++w2) {
      const uint32_t t = s_wsum[w2];
      if (w2 < warp) wpre += t;
      nstaged += t;
    }
    uint32_t excl = incl - mine + wpre;
    int32_t* co = choff + (int64_t)c * (nb + 1);
#pragma unroll
    for (int u = 0; u < RX_NBPT; ++u) {
      if (RX_NBPT * tid + u < nb) {
        cnt[RX_NBPT * tid + u] = excl;
        co[RX_NBPT * tid + u] = (int32_t)excl;
      }
      excl += cv[u];
    }
    if (tid == 0) {
      cnt[nb] = nstaged;
      co[nb] = (int32_t)nstaged;
    }
    __syncthreads();
    // counting-sort scatter of the local indices into the stage (dummy rows land past nstaged);
    // all eight ATOMS of a batch are issued before their stores (a stage store may alias a
    // cursor as far as the compiler knows, so interleaving would serialise on each return)
#pragma unroll
    for (int r0 = 0; r0 < 32; r0 += 8) {
      uint32_t pos[8], loc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t i = sidx[(r0 + u) * RX_THREADS + tid];
        pos[u] = atomicAdd(&cnt[i >> bb], 1u);
        loc[u] = i & ((1u << RX_GROUP_BITS) - 1u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) stage[pos[u]] = (uint16_t)loc[u];
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(buf) + (int64_t)c * RX_CH);
    const uint4* src = reinterpret_cast<const uint4*>(stage);
    const uint32_t nv = (nstaged + 7u) >> 3;
    for (uint32_t i = tid; i < nv; i += RX_THREADS) dst[i] = src[i];
    __syncthreads();  // stage, sidx and s_wsum are reused by the next item
    c = c2;
    rq = rq2;
  }
}

__device__ __forceinline__ uint4 ldg_nc16(const void* p) {
  uint4 r;
  asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__global__ void __launch_bounds__(RC_THREADS, 1)
    k_radix_count(const QDesc* __restrict__ qd, const RDesc* __restrict__ rd,
                  const RItem* __restrict__ items, int nitems, int* __restrict__ head, uint32_t* tables,
                  const char* __restrict__ scratch) {
  extern __shared__ uint32_t tab[];
  __shared__ int s_item;
  constexpr uint32_t G = 1u << RX_GROUP_BITS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(head, 1);
    for (uint32_t i = tid; i < G + 32; i += RC_THREADS) tab[i] = 0u;
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) return;
    const RItem wi = items[it];
    const RDesc r = rd[wi.rq];
    const int gs = RX_GROUP_BITS - r.bb;
    const int b0 = wi.grp << gs, b1 = min(r.nb, (wi.grp + 1) << gs);
    const int nb1 = r.nb + 1;
    // lanes work in sub-groups of W = 2^wlog: a sub-group streams one chunk's run with
    // coalesced 16-B loads (W * 16 B per load instruction), 32 / W runs per warp at a time
    const int wl = r.wlog, W = 1 << wl, runs = 32 >> wl;
    const int sub = lane >> wl, sl = lane & (W - 1);
    const char* buf = scratch + r.buf_off;
    const int32_t* choff = reinterpret_cast<const int32_t*>(scratch + r.choff_off);
    // a vector straddling a run boundary: entries outside [s, e) are redirected to the dummy
    // counter (short divergent fix-up; the atomics stay convergent)
    auto clip = [&](uint4& v, int i0, int s, int e) {
      uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = i0 + 2 * t;
        if (i < s || i >= e) wv[t] = (wv[t] & 0xffff0000u) | (uint32_t)RC_DUMMY;
        if (i + 1 < s || i + 1 >= e) wv[t] = (wv[t] & 0xffffu) | ((uint32_t)RC_DUMMY << 16);
      }
      v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    };
    auto bump = [&](const uint4& v) {
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        atomicAdd(&tab[wv[t] & 0xffffu], 1u);
        atomicAdd(&tab[wv[t] >> 16], 1u);
      }
    };
    const int cstride = (RC_THREADS / 32) * runs;
    const int64_t nb1l = nb1;
    int c = wi.c0 + warp * runs + sub;
    int s = 0, e = 0;
    if (c < wi.c1) {
      s = __ldg(choff + c * nb1l + b0);
      e = __ldg(choff + c * nb1l + b1);
    }
    for (; c - sub < wi.c1; c += cstride) {
      // bounds of this sub-group's next run, fetched while the current one streams
      const int cn = c + cstride;
      int sn = 0, en = 0;
      if (cn < wi.c1) {
        sn = __ldg(choff + cn * nb1l + b0);
        en = __ldg(choff + cn * nb1l + b1);
      }
      const uint16_t* src = reinterpret_cast<const uint16_t*>(buf) + (int64_t)c * RX_CH;
      const int step = 8 * W;
      for (int i = (s & ~7) + 8 * sl; i < e; i += 4 * step) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = i + u * step < e ? ldg_nc16(src + i + u * step) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int iu = i + u * step;
          if (iu >= e) break;
          if (iu < s || iu + 8 > e) clip(v[u], iu, s, e);
          bump(v[u]);
        }
      }
      s = sn;
      e = en;
    }
    __syncthreads();
    const uint32_t base = (uint32_t)wi.grp << RX_GROUP_BITS;
    const uint32_t cells = qd[r.q].cells;
    const uint32_t n = min(G, cells - base);
    uint32_t* t = tables + qd[r.q].table_off + base;
    for (uint32_t i = tid; i < n; i += RC_THREADS) {
      const uint32_t v = tab[i];
      if (v) atomicAdd(t + i, v);
    }
    __syncthreads();
  }
}

}  // namespace cs
