// ccg_bench.cu -- microbenchmark for the roofline denominator of this path.
//
// The climb kernels are bound by shared-memory table lookups, whose peak
// is not in MEASURED_PEAKS.json.  This kernel measures the achievable LDS crossbar
// bandwidth on the running B200: every warp streams conflict-free 128-bit LDS over a
// 32 KB table (4 wavefronts of 128 B per instruction) and folds the words with XOR so
// nothing is dead code.  Reported as bytes delivered to registers per second.
#include <cuda_runtime.h>

#include "ccg_internal.h"

namespace ccg {
namespace {

constexpr int kBenchThreads = 1024;
constexpr int kBenchWords = 8192;  // 32 KB of uint32

__global__ void __launch_bounds__(kBenchThreads) smem_bw_kernel(int iters, uint32_t* sink) {
  __shared__ __align__(16) uint32_t tab[kBenchWords];
  for (int i = threadIdx.x; i < kBenchWords; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const uint4* t4 = reinterpret_cast<const uint4*>(tab);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t acc = 0;
  int base = (warp * 64) & (kBenchWords / 4 - 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 v = t4[((base + u * 32) & (kBenchWords / 4 - 32)) + lane];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    base += 256;
  }
  if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

}  // namespace

cudaError_t bench_smem_bandwidth(cudaStream_t s, int sm_count, double* bytes_per_s) {
  uint32_t* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, sizeof(uint32_t) * sm_count * 8);
  if (e != cudaSuccess) return e;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sm_count * 2;  // 2 x 1024 threads per SM = full occupancy
  const int iters = 4096;
  smem_bw_kernel<<<grid, kBenchThreads, 0, s>>>(64, sink);  // warm-up
  cudaEventRecord(a, s);
  smem_bw_kernel<<<grid, kBenchThreads, 0, s>>>(iters, sink);
  cudaEventRecord(b, s);
  e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)grid * kBenchThreads * iters * 8 * 16;
  *bytes_per_s = bytes / (ms * 1e-3);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace ccg
