// microbench2.cu -- ceilings that bound K1 on B200:
//   (1) SMEM atomic (ATOMS.POPC.INC) issue rate with 16 independent increments per thread,
//       conflict-free (R=32 lane-private replicas) and 32-way-random (R=1, C=2048) addresses;
//   (2) L2 -> SM streaming rate of 16-B ld.global.nc over an L2-resident 96 MB buffer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb2 tools/microbench2.cu && /tmp/mb2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) k_atoms_free(int iters, uint32_t* out) {
  extern __shared__ uint32_t sh[];
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = ((threadIdx.x * 7 + u * 13) & 255) * 32 + lane;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      atomicAdd(sh + a[u], 1u);
      a[u] = (a[u] + 32 * 37) & (256 * 32 - 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[5];
}

__global__ void __launch_bounds__(1024, 1) k_atoms_rand(int iters, uint32_t* out) {
  extern __shared__ uint32_t sh[];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = (threadIdx.x * 2654435761u + u * 40503u) >> 21;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      atomicAdd(sh + a[u], 1u);
      a[u] = (a[u] * 5u + 1u) & 2047u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[5];
}

__global__ void __launch_bounds__(1024, 1) k_stream(const uint4* __restrict__ p, int64_t n16, int reps,
                                                    uint32_t* out) {
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(p + i));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double clk = khz * 1e3;
  uint32_t* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  };
  cudaFuncSetAttribute(k_atoms_free, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int IT = 2048;
  float ms = timeit([&] { k_atoms_free<<<sms, 1024, 256 * 32 * 4>>>(IT, out); });
  double warp_atoms = (double)sms * 32 * IT * 16;
  printf("ATOMS conflict-free : %.3f ms  %.3f warp-instr/clk/SM  (%.1f lane-incs/clk/SM)\n", ms,
         warp_atoms / (ms * 1e-3) / clk / sms, 32 * warp_atoms / (ms * 1e-3) / clk / sms);
  ms = timeit([&] { k_atoms_rand<<<sms, 1024, 2048 * 4>>>(IT, out); });
  printf("ATOMS random (R=1)  : %.3f ms  %.3f warp-instr/clk/SM\n", ms, warp_atoms / (ms * 1e-3) / clk / sms);
  const int64_t bytes = 96ll << 20;
  uint4* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  for (int grid_mult : {1, 2}) {
    const int reps = 20;
    ms = timeit([&] { k_stream<<<sms * grid_mult, 1024 / grid_mult>>>(buf, bytes / 16, reps, out); });
    printf("L2->SM ld.nc.v4 (%d x %d thr): %.3f ms  %.0f GB/s  %.1f B/clk/SM\n", sms * grid_mult,
           1024 / grid_mult, ms, (double)bytes * reps / (ms * 1e-3) / 1e9,
           (double)bytes * reps / (ms * 1e-3) / clk / sms);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
