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

// Random 16-bit gathers from a global table (the quadgram table of the n-gram climb: 26^4
// uint16 = 914 KB, L2-resident, larger than L1): every thread walks 8 independent
// xorshift index streams so the L1/L2 request queues stay full.  Reported as gathers/s
// (each touches one 32-byte sector).
__global__ void __launch_bounds__(256) l2_gather_kernel(const uint16_t* __restrict__ tab, uint32_t n,
                                                        int iters, uint32_t* sink) {
  uint32_t x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = (blockIdx.x * blockDim.x + threadIdx.x) * 8u + u + 0x9e3779b9u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x[u] ^= x[u] << 13;
      x[u] ^= x[u] >> 17;
      x[u] ^= x[u] << 5;
      acc += __ldg(tab + __umulhi(x[u], n));
    }
  }
  if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

}  // namespace

cudaError_t bench_l2_gather(cudaStream_t s, int sm_count, int64_t entries, double* gathers_per_s) {
  uint16_t* tab = nullptr;
  uint32_t* sink = nullptr;
  cudaError_t e = cudaMalloc(&tab, (size_t)entries * 2);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&sink, sizeof(uint32_t) * sm_count * 8);
  if (e != cudaSuccess) {
    cudaFree(tab);
    return e;
  }
  cudaMemsetAsync(tab, 1, (size_t)entries * 2, s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = sm_count * 8;  // 8 x 256 threads = full occupancy
  const int iters = 512;
  l2_gather_kernel<<<grid, 256, 0, s>>>(tab, (uint32_t)entries, 16, sink);  // warm-up: table into L2
  cudaEventRecord(a, s);
  l2_gather_kernel<<<grid, 256, 0, s>>>(tab, (uint32_t)entries, iters, sink);
  cudaEventRecord(b, s);
  e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *gathers_per_s = (double)grid * 256 * iters * 8 / (ms * 1e-3);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  cudaFree(tab);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

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
