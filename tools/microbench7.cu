// microbench7.cu -- tcgen05.st (registers -> TMEM) throughput on sm_100a, alone and while one
// warp streams kind::i8 MMAs (A from TMEM) -- the itemset kernel writes its A operand (128 rows x
// 256 bytes per step) this way.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb7 tools/microbench7.cu && /tmp/mb7
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(288, 1) k_st(int iters, int nst_warps, int xw, int with_mma, int ncols,
                                               unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar_end;
  __shared__ int s_stop;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_end)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    s_stop = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (warp < nst_warps) {
    const long long t0 = clock64();
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 16 + i;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 + 64 * (warp >> 2);
    for (int it = 0; it < iters; ++it) {
      // xw x16 stores (xw * 16 columns) then wait, like one A step (64 columns = 4 x16)
      for (int h = 0; h < xw; ++h)
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                base + 16 * (h & 3)),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[it & 15] += 1;
    }
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
    if (threadIdx.x == 0) atomicExch(&s_stop, 1);
  } else if (warp == 8 && with_mma) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t db = (uint64_t)((sa(smem) >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) |
                        ((uint64_t)(2048 >> 4) << 32) | ((uint64_t)1 << 46);
    long long n_mma = 0;
    while (!*(volatile int*)&s_stop) {
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(tmem),
          "r"(tmem + 448), "l"(db), "r"(idesc)
          : "memory");
      n_mma += 4;
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(sa(&bar_end))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
            sa(&bar_end))
        : "memory");
    if ((threadIdx.x & 31) == 0) atomicAdd(out + 1, (unsigned long long)n_mma);
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
  cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k_st, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  struct C {
    int nst, xw, mma, ncols;
  } cs[] = {{4, 4, 0, 0}, {8, 4, 0, 0}, {4, 1, 0, 0}, {4, 16, 0, 0}, {4, 4, 1, 32}, {8, 4, 1, 32}, {4, 4, 1, 128}, {8, 4, 1, 208}};
  for (auto c : cs) {
    cudaMemset(out, 0, 16);
    k_st<<<sms, 288, 100 * 1024>>>(iters, c.nst, c.xw, c.mma, c.ncols, out);
    cudaMemset(out, 0, 16);
    k_st<<<sms, 288, 100 * 1024>>>(iters, c.nst, c.xw, c.mma, c.ncols, out);
    unsigned long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    const double cyc = (double)h[0] / (sms * c.nst);  // per warp
    const double bytes = (double)c.nst * iters * c.xw * 32 * 16 * 4;  // per CTA
    printf("st warps %d x16 per wait %2d mma %d (N %3d): %.0f clk per wait-group per warp, %.0f B/clk/SM TMEM write; "
           "MMAs per SM %.0f (%.1f clk each)\n",
           c.nst, c.xw, c.mma, c.ncols, cyc / iters, bytes / cyc, (double)h[1] / sms,
           h[1] ? cyc / ((double)h[1] / sms) : 0.0);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
