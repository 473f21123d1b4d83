// microbench.cu -- B200 integer-pipe and SMEM-atomic throughput probes that size the
// counting kernels.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_popc(uint32_t seed, int iters, uint32_t* out) {
  uint32_t a[8], acc[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + 7 * i + 1); acc[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += __popc(a[i]); a[i] = a[i] * 0x9E3779B9u + 1u; }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_popc_only(uint32_t seed, int iters, uint32_t* out) {
  // popc + lop3 chains without the multiply: acc += popc(a & b); a ^= acc
  uint32_t a[8], b[8], acc[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + 7 * i + 1); b[i] = ~a[i] * 3u; acc[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += __popc(a[i] & b[i]); a[i] ^= b[(i + 1) & 7]; b[i] += 1u; }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_lop3(uint32_t seed, int iters, uint32_t* out) {
  uint32_t a[8], b[8], c[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); b[i] = a[i] * 3u; c[i] = a[i] ^ 0x55u; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t s = a[i] ^ b[i] ^ c[i];
      const uint32_t m = (a[i] & b[i]) | (c[i] & (a[i] ^ b[i]));
      a[i] = s; b[i] = m; c[i] = c[i] ^ s;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + b[i] + c[i];
  if (s == 0x12345678) out[0] = s;
}

// SMEM atomics: each thread increments counters; `mode` 0: replica = lane (R=32, conflict
// free), 1: R=1 random cells of a C-cell table, 2: R=8
__global__ void k_atoms(int iters, int C, int mode, uint32_t* out) {
  extern __shared__ uint32_t sh[];
  const int words = (mode == 0 ? 32 : (mode == 2 ? 8 : 1)) * C;
  for (int i = threadIdx.x; i < words; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + 12345u;
  const uint32_t lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const uint32_t c = (x >> 8) % (uint32_t)C;
      uint32_t a;
      if (mode == 0) a = c * 32 + lane;
      else if (mode == 2) a = c * 8 + (lane & 7);
      else a = c;
      atomicAdd(sh + a, 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  uint32_t* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double clk = clk_khz * 1e3;
  auto run = [&](const char* name, auto launch, double ops) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per_clk_sm = ops / (ms * 1e-3) / clk / sms;
    printf("%-34s %8.3f ms  %8.2f ops/clk/SM (at %.0f MHz nominal)\n", name, ms, per_clk_sm, clk / 1e6);
  };
  const int T = 512, B = sms * 4, IT = 4096;
  run("popc (+imad chain)", [&] { k_popc<<<B, T>>>(3, IT, out); }, (double)B * T * IT * 8);
  run("popc(a&b)", [&] { k_popc_only<<<B, T>>>(3, IT, out); }, (double)B * T * IT * 8);
  run("lop3 full-adder (x5 logic ops)", [&] { k_lop3<<<B, T>>>(3, IT, out); }, (double)B * T * IT * 8 * 5);
  for (int mode : {0, 2, 1}) {
    for (int C : {16, 256, 640}) {
      const int words = (mode == 0 ? 32 : (mode == 2 ? 8 : 1)) * C;
      const int smem = words * 4;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(k_atoms, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      char name[64];
      snprintf(name, sizeof name, "atoms mode=%d (R=%d) C=%d", mode, mode == 0 ? 32 : (mode == 2 ? 8 : 1), C);
      run(name, [&] { k_atoms<<<sms * 2, 384, smem>>>(512, C, mode, out); }, (double)sms * 2 * 384 * 512 * 8);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
