// gather_bench.cu — HBM microbenchmark for the roofline of the embedding hot path: bandwidth of
// 256-B (D=64 fp32) row gathers from a table of a given size, in random vs sorted index order, and a
// streaming copy for reference. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gb gather_bench.cu
// Run: ./gb <table_GB> [rows_to_gather_M]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

__global__ void gather(const float4 *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n,
                       float4 *__restrict__ out) {
  // 16 lanes per row (256 B), each lane one float4; 8 rows in flight per lane group
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = t >> 4;
  const int c = t & 15;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 4;
  for (int64_t r0 = g * 8; r0 < n; r0 += ng * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = r0 + u;
      if (r < n) v[u] = __ldg(tab + (size_t)idx[r] * 16 + c);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = r0 + u;
      if (r < n) out[(size_t)r * 16 + c] = v[u];
    }
  }
}

__global__ void copyk(const float4 *__restrict__ a, float4 *__restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main(int argc, char **argv) {
  const double tab_gb = argc > 1 ? atof(argv[1]) : 64.0;
  const int64_t n = (int64_t)((argc > 2 ? atof(argv[2]) : 4.0) * 1e6);
  const int64_t rows = (int64_t)(tab_gb * 1e9 / 256.0);
  float4 *tab, *out;
  uint32_t *idx;
  if (cudaMalloc(&tab, (size_t)rows * 256) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMalloc(&out, (size_t)n * 256);
  cudaMalloc(&idx, (size_t)n * 4);
  cudaMemset(tab, 0, (size_t)rows * 256);
  std::mt19937_64 rng(1);
  std::vector<uint32_t> h(n);
  for (auto &x : h) x = (uint32_t)(rng() % (uint64_t)rows);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char *name) {
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    const int blocks = sms * 8;
    for (int w = 0; w < 3; ++w) gather<<<blocks, 256>>>(tab, idx, n, out);
    cudaEventRecord(e0);
    const int it = 10;
    for (int w = 0; w < it; ++w) gather<<<blocks, 256>>>(tab, idx, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)n * 256 * 2 + n * 4;
    printf("table %.1f GB  %-8s gather %ld rows: %.3f ms  %.0f GB/s (read+write)  %.0f GB/s (row reads)\n", tab_gb,
           name, (long)n, ms / it, bytes / (ms / it * 1e-3) / 1e9, n * 256.0 / (ms / it * 1e-3) / 1e9);
  };
  run("random");
  std::sort(h.begin(), h.end());
  run("sorted");
  for (int64_t i = 0; i < n; ++i) h[i] = (uint32_t)(i % rows);
  run("seq");
  {
    const int64_t m = std::min<int64_t>(rows * 16, (int64_t)n * 16);
    cudaEventRecord(e0);
    for (int w = 0; w < 10; ++w) copyk<<<sms * 8, 256>>>(tab, out, m);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("table %.1f GB  copy %ld B: %.0f GB/s (read+write)\n", tab_gb, (long)(m * 16),
           2.0 * m * 16 / (ms / 10 * 1e-3) / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
