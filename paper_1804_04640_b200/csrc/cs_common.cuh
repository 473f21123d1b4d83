// cs_common.cuh -- shared definitions of libcountgpu (B200 / sm_100a counting-query engine).
//
// Layout of the device database:
//   columns : n x ld bytes, variable-major (row i of the reference's int32 (n, m) matrix,
//             database.py:53, narrowed to uint8), ld = round_up(m, 256) so every column
//             starts 256-B aligned and every 16-row vector load is aligned and in bounds.
//             Bytes past m are zero and never counted.
//   nibbles : 4-bit copy of the columns when every arity <= 16 (n x ldn bytes, ldn =
//             round_up(ceil(m/2), 256)); byte j holds row 2j (low nibble) and row 2j+1 (high
//             nibble).  The histogram kernels are L2/HBM-bandwidth bound, so they read this copy:
//             half the bytes per row.
//   planes  : optional bit planes, one per (variable, state), `words` uint32 per plane,
//             bit t%32 of word t/32 = record t (reference bitmap.py:29-31 little-endian).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CS_MAXK 8            // variables per query on the templated fast path
#define CS_MAX_ARITY 256

namespace cs {

// One counting query as the histogram kernels see it (uniform per CTA).
struct __align__(16) QDesc {
  const uint8_t* base;          // database column block
  uint32_t coff[CS_MAXK];       // column of digit v starts at base + coff[v] * 256
  uint32_t stride[CS_MAXK];     // mixed-radix stride of each digit (target digit first)
  int64_t table_off;            // first cell of this query's table in the packed table buffer
  uint32_t cells;               // C = prod of arities
  int32_t k;                    // number of variables (<= CS_MAXK on the fast path)
  int32_t nbyte;                // leading digits whose cumulative product <= 256 (SIMD byte lanes)
  int32_t mode;                 // 0: C <= 256 (byte lanes), 1: C <= 65536 (16-bit lanes), 2: 32-bit
  int32_t rlog;                 // log2 of SMEM replicas (SMEM class)
  int32_t r_target;             // arity of the target digit
  int32_t nseg;                 // row segments this query is split into
  int32_t kind;                 // 0 SMEM class, 1 global-atomic class, 2 generic (k > CS_MAXK)
  int32_t var_base;             // generic class: offset into the plan's var list
  int32_t pack;                 // SMEM class: rows per atomic (1, or 2 / 4 packed tuples)
  int32_t stages;               // SMEM class: cp.async prefetch ring depth (0 = direct loads)
  uint32_t stage_off;           // SMEM class: byte offset of the ring in dynamic SMEM
  int32_t nib;                  // 1: columns read from the 4-bit (nibble) copy, 32 rows / 16 B
  int32_t half;                 // 1: 16-bit counters, two cells per word (hist_smem_half)
  uint32_t scells;              // slice class: cells per slice (C / arity of the last digit)
  int32_t narrow;               // narrow-counter class: counter bits (8 / 16), 0 otherwise
  // joint index from 4-bit digits d0..d7 in SIMD lanes (narrow class, as cs_radix.cuh RDesc):
  //   b_p = d_2p + rpair[p] d_2p+1, lo = b0 + R0 b1, hi = b2 + R2 b3, idx = lo + P01 hi
  uint32_t rpair[4];
  uint32_t R0, R2, P01;
  int32_t npass;                // narrow class: passes over each row segment (cell ranges)
  uint32_t pcells;              // narrow class: cells per pass (multiple of 4)
  // groups of three digits (0-2, 3-5, 6-7), each combined in byte lanes: set when every group's
  // arity product is <= 256 (K >= 4); gstride[v] = product of the arities before v in its group
  int32_t g3;
  uint32_t gstride[CS_MAXK];
};

// One unit of work: rows [r0, r1) of query q.
struct WItem {
  int32_t q;
  int32_t seg;
  int64_t r0;
  int64_t r1;
  int32_t slice;  // slice class: first value of the last (most significant) digit owned
  int32_t nsl;    // slice class: number of consecutive last-digit values owned
};

enum : uint32_t {
  F_TABLES = 0x1u,
  F_LOGLIK = 0x2u,
  F_MI = 0x4u,
  F_NNZ = 0x8u,
  F_PARTIAL = 0x10u,
  F_NLOGN = 0x20u,  // the loglik output receives sum_cells n ln n (joint "entropy numerator")
  F_NARROW_EXACT = 0x100u,  // internal (CS_NARROW_FAST=0): narrow classes skip their optimistic pass
};

// Counter-based generator (twin: oracle/gen_twin.py).  splitmix64 finaliser.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t column_key(uint64_t seed, int32_t var) {
  return mix64(seed ^ mix64(0x632BE59BD9B4E019ull + (uint64_t)(uint32_t)var));
}
__host__ __device__ __forceinline__ uint32_t hash32(uint64_t key, uint64_t row) {
  return (uint32_t)(mix64(key + row) >> 32);
}

}  // namespace cs
