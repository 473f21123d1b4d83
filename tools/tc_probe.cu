// tc_probe.cu -- correctness probe for the tcgen05 int8 binary GEMM used by the itemset
// kernel: D[m, n] = sum_k A[m, k] * B[n, k] with A, B 0/1 bytes expanded from bit planes into
// K-major SWIZZLE_NONE core-matrix SMEM layouts, D (int32) in TMEM.  One CTA, M=128, N=NT,
// K = KSTEPS x 256.  Compares against a CPU popcount reference and prints the mismatch count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tcp tools/tc_probe.cu && /tmp/tcp
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

constexpr int M = 128, NT = 208, KT = 256;  // KT bytes (= data rows) per step

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// core-matrix (g = row / 8, c = k / 16) at ((g * (KT/16) + c) * 128) bytes; row-major 8x16 inside
__device__ __forceinline__ uint32_t cm_off(int row, int kb) {
  return (uint32_t)(((row >> 3) * (KT / 16) + (kb >> 4)) * 128 + (row & 7) * 16 + (kb & 15));
}

__device__ __forceinline__ uint4 expand16(uint32_t bits16) {
  auto e4 = [](uint32_t b) { return ((b & 0xfu) * 0x00204081u) & 0x01010101u; };
  return make_uint4(e4(bits16), e4(bits16 >> 4), e4(bits16 >> 8), e4(bits16 >> 12));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

__global__ void __launch_bounds__(128, 1)
    k_probe(const uint32_t* __restrict__ abits, const uint32_t* __restrict__ bbits, int ksteps, int* out,
            int lbo_sel) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;                 // M x KT bytes
  uint8_t* sb = smem + M * KT;        // NT x KT bytes
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  // idesc: c_format S32 (2) bits[4,6); a,b u8 (0); K-major; n_dim = N>>3 bits[17,23); m_dim = M>>4 bits[24,29)
  const uint32_t idesc = (2u << 4) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  uint32_t phase = 0;
  for (int ks = 0; ks < ksteps; ++ks) {
    // expand: A rows = M items, B rows = NT pairs; each (row, 16-bit group) -> 16 bytes
    if (lbo_sel == 2) {
      // thread tid owns TMEM lane tid = A row tid; columns 256 + c hold K bytes 4c..4c+3
      for (int h = 0; h < KT / 64; ++h) {
        uint32_t v[16];
        for (int q = 0; q < 2; ++q) {
          const uint32_t w = abits[((size_t)tid * ksteps + ks) * (KT / 32) + 2 * h + q];
          for (int i = 0; i < 8; ++i) v[8 * q + i] = (((w >> (4 * i)) & 0xfu) * 0x00204081u) & 0x01010101u;
        }
        tmem_st16(tmem + ((uint32_t)(warp * 32) << 16) + 256u + 16u * h, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("tcgen05.fence::before_thread_sync;");
    } else
    for (int e = tid; e < M * (KT / 16); e += blockDim.x) {
      const int row = e / (KT / 16), g = e % (KT / 16);
      const uint32_t w = abits[((size_t)row * ksteps + ks) * (KT / 32) + g / 2];
      *reinterpret_cast<uint4*>(sa + cm_off(row, g * 16)) = expand16((g & 1) ? (w >> 16) : (w & 0xffffu));
    }
    for (int e = tid; e < NT * (KT / 16); e += blockDim.x) {
      const int row = e / (KT / 16), g = e % (KT / 16);
      const uint32_t w = bbits[((size_t)row * ksteps + ks) * (KT / 32) + g / 2];
      *reinterpret_cast<uint4*>(sb + cm_off(row, g * 16)) = expand16((g & 1) ? (w >> 16) : (w & 0xffffu));
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
      const uint32_t sbo = (KT / 16) * 128;  // row group stride
      const uint32_t lbo = 128;              // K-chunk stride
      for (int j = 0; j < KT / 32; ++j) {
        const uint64_t da = lbo_sel ? sdesc(a0 + j * 256, sbo, lbo) : sdesc(a0 + j * 256, lbo, sbo);
        const uint64_t db = lbo_sel ? sdesc(b0 + j * 256, sbo, lbo) : sdesc(b0 + j * 256, lbo, sbo);
        const uint32_t acc = (ks | j) ? 1u : 0u;
        if (lbo_sel == 2) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 256u + 8u * j), "l"(sdesc(b0 + j * 256, lbo, sbo)), "r"(idesc), "r"(acc));
          continue;
        }
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&s_bar)));
    }
    // wait for the MMAs before the next step overwrites SMEM
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(&s_bar)), "r"(phase));
      }
      phase ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  // D: lane = m (warp w owns lanes 32w..32w+31), column = n
  for (int c0 = 0; c0 < NT; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[tid * NT + c0 + i] = (int)r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  const int ksteps = 8, words = ksteps * KT / 32;
  std::vector<uint32_t> a((size_t)M * words), b((size_t)NT * words);
  srand(7);
  for (auto& x : a) x = (uint32_t)rand() * 2654435761u ^ (uint32_t)rand();
  for (auto& x : b) x = (uint32_t)rand() * 2246822519u ^ (uint32_t)rand();
  uint32_t *da, *db;
  int* dout;
  cudaMalloc(&da, a.size() * 4);
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&dout, M * NT * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (M + NT) * KT + 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int sel = 0; sel < 3; ++sel) {
    cudaMemset(dout, 0, M * NT * 4);
    k_probe<<<1, 128, smem>>>(da, db, ksteps, dout, sel);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> out(M * NT);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0, shown = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < NT; ++n) {
        int ref = 0;
        for (int w = 0; w < words; ++w) ref += __builtin_popcount(a[(size_t)m * words + w] & b[(size_t)n * words + w]);
        if (out[m * NT + n] != ref) {
          if (shown++ < 3) printf("  sel %d m %d n %d got %d want %d\n", sel, m, n, out[m * NT + n], ref);
          ++bad;
        }
      }
    printf("lbo_sel=%d status=%s mismatches=%ld of %d\n", sel, cudaGetErrorString(e), bad, M * NT);
    if (e != cudaSuccess) break;
    if (sel == 0) ++sel;  // skip the wrong-LBO variant
  }
  return 0;
}
