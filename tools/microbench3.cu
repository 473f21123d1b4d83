// microbench3.cu -- distributed shared memory (DSMEM) atomics across a thread-block cluster
// versus L2 RED.ADD into global memory: the two ways to count into a table larger than one
// SM's shared memory (cfg5).  Random (owner CTA, cell) targets, 16 independent per iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb3 tools/microbench3.cu && /tmp/mb3
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int CL>
__global__ void __launch_bounds__(1024, 1) k_dsmem(int iters, uint32_t cells_per_cta, uint32_t* out) {
  extern __shared__ uint32_t sh[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i < cells_per_cta; i += blockDim.x) sh[i] = 0;
  cl.sync();
  uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 7u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x = x * 1664525u + 1013904223u;
      const uint32_t owner = (x >> 28) & (CL - 1);
      const uint32_t cell = (x >> 8) & (cells_per_cta - 1);
      uint32_t* remote = cl.map_shared_rank(sh + cell, owner);
      atomicAdd(remote, 1u);
    }
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[1];
}

__global__ void __launch_bounds__(1024, 1) k_red(int iters, uint32_t cells, uint32_t* table) {
  uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 7u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x = x * 1664525u + 1013904223u;
      atomicAdd(table + ((x >> 4) & (cells - 1)), 1u);
    }
  }
}

template <int CL>
float run_dsmem(int sms, uint32_t cells_per_cta, uint32_t* out, int iters) {
  auto kern = k_dsmem<CL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((sms / CL) * CL);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = cells_per_cta * 4;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, iters, cells_per_cta, out);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, iters, cells_per_cta, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int nclusters = 0;
  cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
  printf("  (max active clusters of %d: %d)\n", CL, nclusters);
  return ms;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double clk = khz * 1e3;
  uint32_t *out, *table;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&table, 64u << 20);
  cudaMemset(table, 0, 64u << 20);
  const int IT = 256;
  const uint32_t cpc = 32768;  // 128 KB per CTA
  auto report = [&](const char* name, float ms, int grid) {
    const double ops = (double)grid * 1024 * IT * 16;
    printf("%-28s %.3f ms  %.2f lane-atomics/clk/SM  (%.1f G/s)\n", name, ms, ops / (ms * 1e-3) / clk / sms,
           ops / (ms * 1e-3) / 1e9);
  };
  report("DSMEM cluster 2", run_dsmem<2>(sms, cpc, out, IT), (sms / 2) * 2);
  report("DSMEM cluster 4", run_dsmem<4>(sms, cpc, out, IT), (sms / 4) * 4);
  report("DSMEM cluster 8", run_dsmem<8>(sms, cpc, out, IT), (sms / 8) * 8);
  report("DSMEM cluster 16", run_dsmem<16>(sms, cpc, out, IT), (sms / 16) * 16);
  for (uint32_t cells : {1u << 16, 1u << 20, 1u << 24}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_red<<<sms, 1024>>>(IT, cells, table);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k_red<<<sms, 1024>>>(IT, cells, table);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    char name[64];
    snprintf(name, sizeof name, "L2 RED.ADD %u cells", cells);
    report(name, ms, sms);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
