// cs_ingest.cuh -- device-side text ingest: delimited integer records -> uint8 variable-major
// columns (survey 8(f) row 2).  Replaces the reference's load_csv tokeniser
// (database.py:160-207: str.splitlines, strip, split on the sniffed / given delimiter or on
// whitespace, int(token), 1-based shift) for files that are too large to parse in Python.
//
// Grammar (the ASCII subset of the reference's): line boundaries are those of str.splitlines
// (\n \v \f \x1c \x1d \x1e, \r, \r\n as one); whitespace is str.isspace (\t..\r, \x1c..\x1f,
// space); a token is int()'s base-10 syntax: optional sign, digits, single underscores between
// digits.  Non-ASCII bytes are never whitespace, boundaries or digits (a token holding one is a
// non-integer token).
//
// Pipeline (all HBM-streaming byte work, one pass each over the text):
//   k_txt_breaks<false>  per 16 KB chunk: count line boundaries
//   scan64               chunk offsets
//   k_txt_breaks<true>   boundary positions (ordered, block scan inside the chunk)
//   k_txt_lines          warp per line: stripped bounds [a, b), non-empty flag
//   scan64 + k_txt_compact   record -> line map (empty lines dropped)
//   k_txt_head           one warp: the first record's ',' presence and token counts (sniff, width)
//   k_txt_parse<DIRECT>  CTA per tile of TR records, warp per record: token starts by ballot,
//                        one lane parses each token; values land in an SMEM tile [W][TR] that
//                        is written out column by column (coalesced); per-column max, global
//                        min, first bad record (ragged / non-integer) by atomics
//   k_txt_shift          1-based files: every state minus one (SIMD bytes)
#pragma once
#include <climits>
#include "cs_common.cuh"

namespace cs {

constexpr int TX_THREADS = 256;
constexpr int TX_PER_THREAD = 64;                     // bytes per thread in k_txt_breaks
constexpr int TX_CHUNK = TX_THREADS * TX_PER_THREAD;  // 16 KB per CTA
constexpr int TX_PAD = 64;                            // zero bytes after the text (vector loads)
constexpr int TX_SAT = 1 << 24;                       // values saturate here (arity check only)
constexpr int TX_SCAN_TILE = 4096;                    // int64 elements per scan CTA (1024 x 4)

__device__ __forceinline__ bool tx_ws(uint32_t c) { return (c - 9u) <= 4u || (c - 28u) <= 4u; }
__device__ __forceinline__ bool tx_brk(uint32_t c, uint32_t next) {
  return c == 10 || c == 11 || c == 12 || (c - 28u) <= 2u || (c == 13 && next != 10);
}

// exclusive scan of one value per thread over the CTA; returns the CTA total in *total
template <int NT>
__device__ __forceinline__ int64_t block_exscan(int64_t v, int64_t* total) {
  __shared__ int64_t s_w[NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < NT / 32 ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) s_w[lane] = w;
  }
  __syncthreads();
  const int64_t before = (warp ? s_w[warp - 1] : 0) + x - v;
  *total = s_w[NT / 32 - 1];
  __syncthreads();
  return before;
}

// In-place exclusive scan of tiles of TX_SCAN_TILE int64; tile totals to sums (if non-null).
__global__ void __launch_bounds__(1024) k_scan64_tiles(int64_t* __restrict__ data, int64_t n,
                                                        int64_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * TX_SCAN_TILE + threadIdx.x * 4;
  int64_t v[4], s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j] = base + j < n ? data[base + j] : 0;
    s += v[j];
  }
  int64_t total;
  int64_t run = block_exscan<1024>(s, &total);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (base + j < n) data[base + j] = run;
    run += v[j];
  }
  if (sums && threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void k_scan64_add(int64_t* __restrict__ data, int64_t n, const int64_t* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) data[i] += sums[i / TX_SCAN_TILE];
}

// Count (WRITE = false) or list (WRITE = true) the line boundaries of the text.  Thread t of
// CTA b owns bytes [b*TX_CHUNK + 64 t, +64); four aligned 16-B loads plus the next byte.
template <bool WRITE>
__global__ void __launch_bounds__(TX_THREADS) k_txt_breaks(const uint8_t* __restrict__ text, int64_t nbytes,
                                                           int64_t* __restrict__ counts,
                                                           const int64_t* __restrict__ offs,
                                                           int64_t* __restrict__ brk) {
  const int64_t base = (int64_t)blockIdx.x * TX_CHUNK + (int64_t)threadIdx.x * TX_PER_THREAD;
  uint32_t w[TX_PER_THREAD / 4 + 1];
  const uint4* p = reinterpret_cast<const uint4*>(text + base);
#pragma unroll
  for (int j = 0; j < TX_PER_THREAD / 16; ++j) {
    const uint4 x = base < nbytes ? p[j] : make_uint4(0, 0, 0, 0);
    w[4 * j] = x.x;
    w[4 * j + 1] = x.y;
    w[4 * j + 2] = x.z;
    w[4 * j + 3] = x.w;
  }
  w[TX_PER_THREAD / 4] = base < nbytes ? text[base + TX_PER_THREAD] : 0;  // padded: always in bounds
  uint64_t bits = 0;  // bit i: byte base + i is a boundary
#pragma unroll
  for (int i = 0; i < TX_PER_THREAD; ++i) {
    const uint32_t c = (w[i >> 2] >> (8 * (i & 3))) & 0xffu;
    const uint32_t nx = (w[(i + 1) >> 2] >> (8 * ((i + 1) & 3))) & 0xffu;
    if (tx_brk(c, nx)) bits |= 1ull << i;
  }
  if (base + TX_PER_THREAD > nbytes) {
    const int64_t keep = nbytes - base;
    bits = keep <= 0 ? 0 : (keep >= 64 ? bits : bits & ((1ull << keep) - 1));
  }
  int64_t total;
  const int64_t before = block_exscan<TX_THREADS>(__popcll(bits), &total);
  if (!WRITE) {
    if (threadIdx.x == 0) counts[blockIdx.x] = total;
    return;
  }
  int64_t o = offs[blockIdx.x] + before;
  while (bits) {
    const int i = __ffsll((long long)bits) - 1;
    bits &= bits - 1;
    brk[o++] = base + i;
  }
}

// 4 bytes -> 4-bit mask of the bytes that are not str.isspace (\t..\r, \x1c..\x20)
__device__ __forceinline__ uint32_t tx_nonws4(uint32_t w) {
  const uint32_t a = __vcmpleu4(__vsub4(w, 0x09090909u), 0x04040404u);
  const uint32_t b = __vcmpleu4(__vsub4(w, 0x1c1c1c1cu), 0x04040404u);
  const uint32_t k = ~(a | b) & 0x01010101u;  // 1 per non-whitespace byte
  return (k * 0x00204081u) >> 21 & 0xfu;       // byte i -> bit i
}

// Warp per line: stripped bounds and the non-empty flag (str.strip, then `if ln`).  Each lane
// takes 16 aligned bytes per step (a 512-B window per warp: one step for typical records);
// SIMD byte compares give a 16-bit non-whitespace mask, clipped to the line, and the first /
// last set byte over the warp are a min / max reduction.
__global__ void k_txt_lines(const uint8_t* __restrict__ text, int64_t nbytes, const int64_t* __restrict__ brk,
                            int64_t nlines, int64_t* __restrict__ la, int64_t* __restrict__ lb,
                            int64_t* __restrict__ nonempty) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t ln = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ln < nlines; ln += nw) {
    const int64_t s = ln == 0 ? 0 : brk[ln - 1] + 1;
    const int64_t e = ln == nlines - 1 ? nbytes : brk[ln];
    int64_t a = INT64_MAX, b = -1;
    for (int64_t q0 = s & ~(int64_t)15; q0 < e; q0 += 512) {
      const int64_t q = q0 + 16 * lane;
      uint32_t mask = 0;  // bit i: byte q + i is in [s, e) and not whitespace
      if (q < e && q + 16 > s) {
        const uint4 v = *reinterpret_cast<const uint4*>(text + q);
        mask = tx_nonws4(v.x) | tx_nonws4(v.y) << 4 | tx_nonws4(v.z) << 8 | tx_nonws4(v.w) << 12;
        const int64_t lo = s - q, hi = e - q;  // keep bits [lo, hi)
        if (lo > 0) mask &= 0xffffu << lo;
        if (hi < 16) mask &= (1u << hi) - 1u;
      }
      int fa = mask ? __ffs(mask) - 1 + 16 * lane : 1 << 30;
      int fb = mask ? 16 * lane + 32 - __clz(mask) : -1;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        fa = min(fa, __shfl_xor_sync(0xffffffffu, fa, o));
        fb = max(fb, __shfl_xor_sync(0xffffffffu, fb, o));
      }
      if (fb >= 0) {
        a = min(a, q0 + fa);
        b = q0 + fb;
      }
    }
    if (lane == 0) {
      const bool ne = b >= 0;
      la[ln] = ne ? a : s;
      lb[ln] = ne ? b : s;
      nonempty[ln] = ne;
    }
  }
}

__global__ void k_txt_compact(const int64_t* __restrict__ flag, const int64_t* __restrict__ rank, int64_t nlines,
                              int64_t* __restrict__ rec_line) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nlines && flag[i]) rec_line[rank[i]] = i;
}

// One warp over the first record: out[0] = 1 if it holds a ',', out[1] = whitespace-split
// token count, out[2] = field count when split on byte dc.
__global__ void k_txt_head(const uint8_t* __restrict__ text, const int64_t* __restrict__ la,
                           const int64_t* __restrict__ lb, const int64_t* __restrict__ rec_line, int32_t dc,
                           int64_t* __restrict__ out) {
  const int lane = threadIdx.x;
  const int64_t ln = rec_line[0], a = la[ln], b = lb[ln];
  int64_t comma = 0, tok = 0, nd = 0;
  for (int64_t p0 = a; p0 < b; p0 += 32) {
    const int64_t p = p0 + lane;
    const uint32_t c = p < b ? text[p] : 32u;
    const uint32_t pv = p > a && p < b ? text[p - 1] : 32u;
    comma += __popc(__ballot_sync(0xffffffffu, p < b && c == ','));
    nd += __popc(__ballot_sync(0xffffffffu, p < b && c == (uint32_t)dc));
    tok += __popc(__ballot_sync(0xffffffffu, p < b && !tx_ws(c) && tx_ws(pv)));
  }
  if (lane == 0) {
    out[0] = comma > 0;
    out[1] = tok;
    out[2] = nd + 1;
  }
}

// int() base 10 on text[s, e) (already stripped): [+-] digit (_? digit)*.  Returns false if the
// token is not an integer; *v saturates at +-TX_SAT.
__device__ __forceinline__ bool tx_int(const uint8_t* __restrict__ text, int64_t s, int64_t e, int* v) {
  if (s >= e) return false;
  int sign = 1;
  uint32_t c = text[s];
  if (c == '+' || c == '-') {
    sign = c == '-' ? -1 : 1;
    if (++s >= e) return false;
  }
  int x = 0;
  bool need_digit = true;
  for (; s < e; ++s) {
    c = text[s];
    if (c - '0' <= 9u) {
      x = min(x * 10 + (int)(c - '0'), TX_SAT);
      need_digit = false;
    } else if (c == '_' && !need_digit) {
      need_digit = true;
    } else {
      return false;
    }
  }
  if (need_digit) return false;
  *v = sign * x;
  return true;
}

// CTA per tile of tr records (dynamic SMEM: W*tr bytes of states + W column maxima), warp per
// record.  DIRECT: no SMEM tile (very wide records), bytes stored straight to the columns.
template <bool DIRECT>
__global__ void __launch_bounds__(TX_THREADS) k_txt_parse(
    const uint8_t* __restrict__ text, const int64_t* __restrict__ la, const int64_t* __restrict__ lb,
    const int64_t* __restrict__ rec_line, int64_t nrec, int32_t width, int32_t delim, int32_t tr,
    uint8_t* __restrict__ cols, int64_t ld, int* __restrict__ colmax, int* __restrict__ gmin,
    unsigned long long* __restrict__ bad) {
  extern __shared__ __align__(16) uint8_t tx_smem[];
  int* s_max = reinterpret_cast<int*>(tx_smem);
  uint8_t* tile = tx_smem + 4 * width;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < width; c += blockDim.x) s_max[c] = INT_MIN;
  const int64_t r0 = (int64_t)blockIdx.x * tr;
  const int nr = (int)(nrec - r0 < tr ? nrec - r0 : tr);
  const uint8_t* src = text;
  __syncthreads();
  int lmin = INT_MAX;
  for (int rr = warp; rr < nr; rr += TX_THREADS / 32) {
    const int64_t rec = r0 + rr, ln = rec_line[rec], a = la[ln], b = lb[ln];
    int ntok = 0;
    bool ok = true;
    for (int64_t p0 = a; p0 <= b; p0 += 32) {
      const int64_t p = p0 + lane;
      bool start;
      if (delim < 0) {
        start = p < b && !tx_ws(src[p]) && (p == a || tx_ws(src[p - 1]));
      } else {
        start = p <= b && (p == a || src[p - 1] == (uint32_t)delim);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, start);
      if (start) {
        const int t = ntok + __popc(m & ((1u << lane) - 1));
        int64_t e = p;
        if (delim < 0) {
          while (e < b && !tx_ws(src[e])) ++e;
        } else {
          while (e < b && src[e] != (uint32_t)delim) ++e;
        }
        int64_t s = p;
        if (delim >= 0) {  // tok.strip()
          while (s < e && tx_ws(src[s])) ++s;
          while (e > s && tx_ws(src[e - 1])) --e;
        }
        int v = 0;
        if (!tx_int(src, s, e, &v)) {
          ok = false;
        } else if (t < width) {
          if (DIRECT) cols[(int64_t)t * ld + rec] = (uint8_t)v;
          else tile[(int64_t)t * tr + rr] = (uint8_t)v;
          atomicMax(&s_max[t], v);
          lmin = min(lmin, v);
        }
      }
      ntok += __popc(m);
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0 && (!ok || ntok != width)) atomicMin(bad, (unsigned long long)rec);
  }
  __syncthreads();
  if (!DIRECT) {
    // tile row t (tr bytes, tr % 32 == 0) -> column t, records r0 .. r0 + nr
    const int wpr = tr >> 2;  // 32-bit words per tile row
    const int nwf = nr >> 2;  // full words of real records
    for (int i = threadIdx.x; i < width * wpr; i += blockDim.x) {
      const int t = i / wpr, j = i - t * wpr;
      uint8_t* dst = cols + (int64_t)t * ld + r0 + 4 * j;
      const uint8_t* src = tile + (int64_t)t * tr + 4 * j;
      if (j < nwf) {
        *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src);
      } else {
        for (int q = 0; q < 4 && 4 * j + q < nr; ++q) dst[q] = src[q];
      }
    }
  }
  for (int c = threadIdx.x; c < width; c += blockDim.x)
    if (s_max[c] != INT_MIN) atomicMax(colmax + c, s_max[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
  if (lane == 0 && lmin != INT_MAX) atomicMin(gmin, lmin);
}

// Thread per record (records of <= ~384 values): one pass over the record's bytes with 16-B
// loads and a branch-free int() state machine per byte, so the 32 lanes of a warp stay
// converged; values go to the SMEM tile [W][tr] (tr = blockDim = 256).  Column maxima are taken
// from the tile bytes at write-out (values > 255 or < 0 also go straight to the global max /
// min, they always end in an error).  Token grammar as tx_int; delim < 0: whitespace runs.
enum : uint32_t { TS_START = 0, TS_SIGN = 1, TS_DIG = 2, TS_UND = 3, TS_TRAIL = 4, TS_BAD = 5 };

__global__ void __launch_bounds__(TX_THREADS) k_txt_parse_thr(
    const uint8_t* __restrict__ text, const int64_t* __restrict__ la, const int64_t* __restrict__ lb,
    const int64_t* __restrict__ rec_line, int64_t nrec, int32_t width, int32_t delim,
    uint8_t* __restrict__ cols, int64_t ld, int* __restrict__ colmax, int* __restrict__ gmin,
    unsigned long long* __restrict__ bad) {
  extern __shared__ __align__(16) uint8_t tx_smem[];
  uint8_t* tile = tx_smem;  // [width][TX_THREADS]
  const int tr = TX_THREADS;
  const int64_t r0 = (int64_t)blockIdx.x * tr;
  const int nr = (int)(nrec - r0 < tr ? nrec - r0 : tr);
  const int rr = threadIdx.x;
  int lmin = INT_MAX;
  if (rr < nr) {
    const int64_t rec = r0 + rr, ln = rec_line[rec], a = la[ln], b = lb[ln];
    const bool wsmode = delim < 0;
    const uint32_t dl = (uint32_t)(wsmode ? 256 : delim);
    uint32_t st = TS_START;
    bool in_tok = false, ok = true;
    int v = 0, neg = 0, t = 0;
    for (int64_t q = a & ~(int64_t)15; q <= b; q += 16) {
      const uint4 x = *reinterpret_cast<const uint4*>(text + q);
      const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int64_t p = q + i;
        if (p < a || p > b) continue;
        const uint32_t c = p == b ? 32u : (w4[i >> 2] >> (8 * (i & 3))) & 0xffu;  // b: virtual end
        const bool end = p == b;
        const bool ws = tx_ws(c);
        const bool sep = end || (wsmode ? ws : c == dl);
        const uint32_t d = c - '0';
        const bool dig = d <= 9u;
        if (!sep) {
          if (wsmode) in_tok = true;
          // next state of the token grammar (delim mode: surrounding whitespace allowed)
          uint32_t ns;
          if (dig) ns = (st == TS_TRAIL || st == TS_BAD) ? TS_BAD : TS_DIG;
          else if (c == '_') ns = st == TS_DIG ? TS_UND : TS_BAD;
          else if (c == '+' || c == '-') ns = st == TS_START ? TS_SIGN : TS_BAD;
          else if (ws) ns = st == TS_START ? TS_START : (st == TS_DIG || st == TS_TRAIL) ? TS_TRAIL : TS_BAD;
          else ns = TS_BAD;
          if (c == '-' && st == TS_START) neg = 1;
          if (dig && ns == TS_DIG) v = min(v * 10 + (int)d, TX_SAT);
          st = ns;
        }
        // a field / token ends here
        if (sep && (!wsmode || in_tok)) {
          const bool good = st == TS_DIG || st == TS_TRAIL;
          ok = ok && good;
          const int val = neg ? -v : v;
          if (good && t < width) {
            tile[t * tr + rr] = (uint8_t)val;
            if (val > 255) atomicMax(colmax + t, val);
            lmin = min(lmin, val);
          }
          ++t;
          st = TS_START;
          v = 0;
          neg = 0;
          in_tok = false;
        }
      }
    }
    if (!ok || t != width) atomicMin(bad, (unsigned long long)rec);
  }
  __syncthreads();
  // write-out: warp per tile row (column), lanes over the row's 64 words; per-column max of the
  // bytes of real records
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = warp; t < width; t += TX_THREADS / 32) {
    uint32_t mx = 0;
    for (int j = lane; j < tr / 4; j += 32) {
      uint32_t wv = *reinterpret_cast<const uint32_t*>(tile + t * tr + 4 * j);
      const int left = nr - 4 * j;
      if (left < 4) wv &= left <= 0 ? 0u : (1u << (8 * left)) - 1u;
      if (left > 0) {
        uint8_t* dst = cols + (int64_t)t * ld + r0 + 4 * j;
        if (left >= 4) *reinterpret_cast<uint32_t*>(dst) = wv;
        else
          for (int q2 = 0; q2 < left; ++q2) dst[q2] = (uint8_t)(wv >> (8 * q2));
      }
      mx = __vmaxu4(mx, wv);
    }
    mx = max(max(mx & 0xffu, (mx >> 8) & 0xffu), max((mx >> 16) & 0xffu, mx >> 24));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) atomicMax(colmax + t, (int)mx);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
  if (lane == 0 && lmin != INT_MAX) atomicMin(gmin, lmin);
}

// 1-based file: every state of rows [0, m) minus one (mod 256: a 256 stored as 0 becomes 255).
__global__ void k_txt_shift(uint8_t* __restrict__ cols, int64_t ld, int64_t m, int n) {
  for (int var = blockIdx.y; var < n; var += gridDim.y) {
    uint32_t* c = reinterpret_cast<uint32_t*>(cols + (int64_t)var * ld);
    const int64_t nw = (m + 3) >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t left = m - 4 * i;
      const uint32_t sub = left >= 4 ? 0x01010101u : (0x01010101u & ((1u << (8 * left)) - 1));
      c[i] = __vsub4(c[i], sub);
    }
  }
}

}  // namespace cs
