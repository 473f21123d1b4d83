// microbench5.cu -- cp.async.bulk (1D TMA) global->shared throughput per SM on sm_100a, as a
// function of copy size, ring depth, issuing threads and source residency (L2 vs HBM).  Used to
// size the itemset kernel's raw loader (cs_itemsets.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb5 tools/microbench5.cu && /tmp/mb5
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}

__device__ __forceinline__ void spin_bar(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}

// nissuers warps, each with its own ring of R slots of `bytes`; each copy = `pieces` bulk ops
__global__ void k_bulk(const char* __restrict__ src, size_t span, int bytes, int pieces, int R, int iters,
                       unsigned long long* out, int spin) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) uint64_t bars[8][16];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int r = 0; r < R; ++r) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[w][r])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  char* ring = buf + (size_t)w * R * bytes;
  const long long t0 = clock64();
  uint64_t off = ((uint64_t)blockIdx.x * 7919 + w * 104729) * 4096 % span;
  for (int i = 0; i < iters; ++i) {
    const int r = i % R;
    // spin: 0 try_wait per slot, 1 test_wait per slot, 2 no waits in the loop (issue cost only),
    // 3 one expect_tx per R copies + one wait per R copies
    if (i >= R && (spin < 2 || spin == 4)) {
      if (spin) spin_bar(sa(&bars[w][r]), ((i / R) - 1) & 1);
      else wait_bar(sa(&bars[w][r]), ((i / R) - 1) & 1);
    }
    if (spin == 3 && r == 0 && i >= R) wait_bar(sa(&bars[w][0]), ((i / R) - 1) & 1);
    if (lane == 0) {
      if (spin != 3 || r == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[w][spin == 3 ? 0 : r])),
                     "r"(spin == 3 ? bytes * R : bytes)
                     : "memory");
      const int pb = bytes / pieces;
      for (int p = 0; p < pieces; ++p) {
        if (spin == 4)  // .shared::cta destination form
          asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           sa(ring + (size_t)r * bytes + p * pb)),
                       "l"(src + off + p * pb), "r"(pb), "r"(sa(&bars[w][r]))
                       : "memory");
        else
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           sa(ring + (size_t)r * bytes + p * pb)),
                       "l"(src + off + p * pb), "r"(pb), "r"(sa(&bars[w][spin == 3 ? 0 : r]))
                       : "memory");
      }
    }
    __syncwarp();
    off += bytes;
    if (off + bytes > span) off = 0;
  }
  if (spin == 3) wait_bar(sa(&bars[w][0]), ((iters / R) - 1) & 1);
  else if (spin == 2) __nanosleep(100000);
  else
    for (int i = iters; i < iters + R; ++i) {
      const int r = i % R;
      if (i >= R) wait_bar(sa(&bars[w][r]), ((i / R) - 1) & 1);
    }
  const long long t1 = clock64();
  if (lane == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  char* src;
  const size_t big = 2ull << 30;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  unsigned long long* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg {
    int bytes, pieces, R, warps;
    size_t span;
    int spin;
  } cfgs[] = {
      {8192, 1, 8, 1, 16 << 20, 0},  {8192, 1, 8, 1, 16 << 20, 4}, {2048, 1, 8, 1, 16 << 20, 4},
      {8192, 16, 8, 1, 16 << 20, 4}, {8192, 1, 2, 8, 16 << 20, 4},
  };
  for (auto c : cfgs) {
    const int iters = 4000;
    const size_t smem = (size_t)c.warps * c.R * c.bytes;
    if (smem > 200 * 1024) continue;
    cudaMemset(out, 0, 8);
    k_bulk<<<sms, 32 * c.warps, smem>>>(src, c.span, c.bytes, c.pieces, c.R, iters, out, c.spin);
    cudaMemset(out, 0, 8);
    cudaEventRecord(a);
    k_bulk<<<sms, 32 * c.warps, smem>>>(src, c.span, c.bytes, c.pieces, c.R, iters, out, c.spin);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    const double tot = (double)sms * c.warps * iters * c.bytes;
    const double cyc_per_warp = (double)cyc / (sms * c.warps);
    printf("%s bytes %6d pieces %2d R %2d warps %d src %s: %.3f ms  %.2f TB/s  %.1f B/clk/SM  (%.0f clk per copy per issuer)\n",
           c.spin == 0 ? "try_wait " : c.spin == 1 ? "test_wait" : c.spin == 2 ? "no-wait  " : c.spin == 3 ? "batched  " : "cta-dst  ", c.bytes, c.pieces, c.R, c.warps, c.span > (64u << 20) ? "HBM" : "L2 ", ms, tot / (ms * 1e-3) / 1e12,
           (double)c.warps * iters * c.bytes / cyc_per_warp, cyc_per_warp / iters);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
