// microbench6.cu -- tcgen05.mma kind::i8 issue cost vs N on sm_100a (M = 128, K = 32 per
// instruction, A from TMEM, B from SMEM): one elected thread per CTA issues back-to-back MMAs
// into one accumulator, committing every 8 (as the itemset kernel does per 256-row step).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb6 tools/microbench6.cu && /tmp/mb6
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) k_mma(int ncols, int steps, int per_commit, int ss, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar, bar_end;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_end)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  auto sdesc = [](uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) |
           ((uint64_t)1 << 46);
  };
  const uint64_t db0 = sdesc(sa(smem));
  const uint64_t da0 = sdesc(sa(smem + 65536));
  long long t0 = clock64();
  if (warp == 1) {
    for (int st = 0; st < steps; ++st) {
      const uint32_t ta = tmem + 256 + (st & 1) * 64;
      const uint64_t db = db0 + (uint64_t)((st & 1) * 2048);
      if (ss) {
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %4, %5, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %6, %7, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %8, %9, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %10, %11, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %12, %13, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %14, %15, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %16, %17, %3, 1;\n\t}" ::"r"(tmem),
            "l"(da0), "l"(db), "r"(idesc), "l"(da0 + 16), "l"(db + 16), "l"(da0 + 32), "l"(db + 32), "l"(da0 + 48),
            "l"(db + 48), "l"(da0 + 64), "l"(db + 64), "l"(da0 + 80), "l"(db + 80), "l"(da0 + 96), "l"(db + 96),
            "l"(da0 + 112), "l"(db + 112)
            : "memory");
      } else {
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%4], %5, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%6], %7, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%8], %9, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%10], %11, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%12], %13, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%14], %15, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%16], %17, %3, 1;\n\t}" ::"r"(tmem),
            "r"(ta), "l"(db), "r"(idesc), "r"(ta + 8), "l"(db + 16), "r"(ta + 16), "l"(db + 32), "r"(ta + 24),
            "l"(db + 48), "r"(ta + 32), "l"(db + 64), "r"(ta + 40), "l"(db + 80), "r"(ta + 48), "l"(db + 96),
            "r"(ta + 56), "l"(db + 112)
            : "memory");
      }
      if (per_commit && (st + 1) % per_commit == 0) {
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(sa(&bar))
            : "memory");
      }
    }
    // per-step commits go to `bar` (never waited: a parity wait cannot tell its phases apart);
    // the final commit goes to bar_end, waited once
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(sa(&bar_end))
        : "memory");
    {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(sa(&bar_end))
            : "memory");
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)(clock64() - t0));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  unsigned long long* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int steps = 2000;
  for (int ss = 0; ss < 2; ++ss)
    for (int per : {1, 0})
      for (int n : {16, 32, 64, 96, 128, 208, 256}) {
        cudaMemset(out, 0, 8);
        k_mma<<<sms, 128, 160 * 1024>>>(n, steps, per, ss, out);
        cudaMemset(out, 0, 8);
        k_mma<<<sms, 128, 160 * 1024>>>(n, steps, per, ss, out);
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
        const double c = (double)cyc / sms / (steps * 8.0);
        printf("%s N %3d commit/%s: %.1f clk per MMA (work at 8192 MAC/clk: %.1f) -> %.0f MAC/clk/SM\n",
               ss ? "SS" : "TS", n, per ? "step" : "end ", c, 128.0 * n * 32 / 8192, 128.0 * n * 32 / c);
      }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
