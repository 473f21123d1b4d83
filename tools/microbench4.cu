// microbench4.cu -- 1-bit tensor-core MMA (mma.sync m16n8k256 .b1 .and.popc) throughput on
// sm_100a vs the CUDA-core AND+POPC / Harley-Seal rate used by k_itemsets.  If the legacy b1
// path is fast, the all-triples itemset kernel could run on bit planes directly.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb4 tools/microbench4.cu && /tmp/mb4
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_b1(int iters, uint32_t seed, int* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + 3 * i + 1);
  for (int i = 0; i < 2; ++i) b[i] = seed ^ (threadIdx.x * 7 + i);
  int c[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
          "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  int s = 0;
  for (int u = 0; u < 4; ++u)
    for (int i = 0; i < 4; ++i) s += c[u][i];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_i8(int iters, uint32_t seed, int* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + 3 * i + 1);
  for (int i = 0; i < 2; ++i) b[i] = seed ^ (threadIdx.x * 7 + i);
  int c[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 "
          "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  int s = 0;
  for (int u = 0; u < 4; ++u)
    for (int i = 0; i < 4; ++i) s += c[u][i];
  if (s == 0x12345678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double clk = khz * 1e3;
  const int sms = p.multiProcessorCount;
  int* out;
  cudaMalloc(&out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int IT = 4096, T = 256, B = sms * 4;
  auto time = [&](auto f) {
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  };
  const double warps = (double)B * T / 32;
  float ms = time([&] { k_b1<<<B, T>>>(IT, 3, out); });
  double macs = warps * IT * 4 * 16.0 * 8 * 256;
  printf("mma.sync b1 m16n8k256 and.popc: %.3f ms  %.1f T bit-MAC/s  (%.0f bit-MAC/clk/SM)\n", ms,
         macs / (ms * 1e-3) / 1e12, macs / (ms * 1e-3) / clk / sms);
  ms = time([&] { k_i8<<<B, T>>>(IT, 3, out); });
  macs = warps * IT * 4 * 16.0 * 8 * 32;
  printf("mma.sync u8 m16n8k32:           %.3f ms  %.1f T MAC/s  (%.0f MAC/clk/SM)\n", ms,
         macs / (ms * 1e-3) / 1e12, macs / (ms * 1e-3) / clk / sms);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
