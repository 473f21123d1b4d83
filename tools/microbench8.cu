// microbench8.cu -- the HBM read ceiling K1 can be held to on B200: a read-only stream shaped
// like K1's (persistent 1024-thread CTAs, one per SM, each walking its own 2 MB row segment of
// K columns with 16-B ld.global.nc per thread and column; columns 50 MB apart in a 32 GB
// buffer), K = 1..8, with 1, 2 or 4 vector sets in flight per thread, against the plain
// grid-stride read of one contiguous buffer.  No arithmetic besides an XOR sink.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb8 tools/microbench8.cu && /tmp/mb8
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldnc(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// items: (column set j, segment s); CTA b takes items b, b + grid, ...
template <int K, int U>
__global__ void __launch_bounds__(1024, 1) k_cols(const uint8_t* __restrict__ base, int64_t col_bytes, int ncols,
                                                  int64_t seg_bytes, int nseg, int nitems, uint32_t* out) {
  uint32_t acc = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int q = it / nseg, s = it % nseg;
    const uint8_t* p0 = base + (int64_t)s * seg_bytes;
    int64_t co[K];
#pragma unroll
    for (int v = 0; v < K; ++v) co[v] = (int64_t)((q * 131 + v * 37) % ncols) * col_bytes;
    const int64_t nvec = seg_bytes / 16;
    for (int64_t vi = threadIdx.x; vi < nvec; vi += 1024 * U) {
      uint4 x[U][K];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < K; ++v)
          if (vi + u * 1024 < nvec) x[u][v] = ldnc(p0 + co[v] + ((vi + u * 1024) << 4));
          else x[u][v] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < K; ++v) acc ^= x[u][v].x ^ x[u][v].y ^ x[u][v].z ^ x[u][v].w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __launch_bounds__(1024, 2) k_flat(const uint4* __restrict__ p, int64_t n16, uint32_t* out) {
  uint32_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = i + (int64_t)u * gridDim.x * blockDim.x;
      v[u] = j < n16 ? ldnc(p + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int K, int U>
static void run(const uint8_t* buf, int64_t col_bytes, int ncols, uint32_t* out) {
  const int64_t seg_bytes = 2 << 20;
  const int nseg = (int)(col_bytes / seg_bytes);
  const int nq = 24;
  const int nitems = nq * nseg;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_cols<K, U><<<148, 1024>>>(buf, col_bytes, ncols, seg_bytes, nseg, nitems, out);
  cudaEventRecord(a);
  k_cols<K, U><<<148, 1024>>>(buf, col_bytes, ncols, seg_bytes, nseg, nitems, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)nq * K * nseg * seg_bytes;
  printf("{\"kernel\": \"k_cols\", \"K\": %d, \"in_flight\": %d, \"ms\": %.3f, \"gbs\": %.1f}\n", K, U, ms,
         bytes / ms / 1e6);
}

int main() {
  const int64_t col_bytes = 50 << 20;
  const int ncols = 640;  // 32 GB
  uint8_t* buf;
  uint32_t* out;
  if (cudaMalloc(&buf, col_bytes * ncols) != cudaSuccess) return 1;
  cudaMalloc(&out, 4096);
  cudaMemset(buf, 1, col_bytes * ncols);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int g : {148, 296, 592}) {
    const int64_t n16 = col_bytes * ncols / 16;
    k_flat<<<g, 1024>>>((const uint4*)buf, n16, out);
    cudaEventRecord(a);
    k_flat<<<g, 1024>>>((const uint4*)buf, n16, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"kernel\": \"k_flat\", \"grid\": %d, \"ms\": %.3f, \"gbs\": %.1f}\n", g, ms, (double)n16 * 16 / ms / 1e6);
  }
  run<1, 1>(buf, col_bytes, ncols, out);
  run<1, 4>(buf, col_bytes, ncols, out);
  run<2, 1>(buf, col_bytes, ncols, out);
  run<2, 2>(buf, col_bytes, ncols, out);
  run<2, 4>(buf, col_bytes, ncols, out);
  run<4, 1>(buf, col_bytes, ncols, out);
  run<4, 2>(buf, col_bytes, ncols, out);
  run<4, 4>(buf, col_bytes, ncols, out);
  run<6, 1>(buf, col_bytes, ncols, out);
  run<6, 2>(buf, col_bytes, ncols, out);
  run<8, 1>(buf, col_bytes, ncols, out);
  run<8, 2>(buf, col_bytes, ncols, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
