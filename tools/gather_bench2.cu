// gather_bench2.cu — what it takes to saturate HBM with random 256-B row gathers on B200.
// Each warp gathers rows (random indices into a 64 GB table) and writes them contiguously, with
// three load mechanisms and a varying amount of data in flight per warp / warps per SM:
//   ldg  : 16 lanes x float4 per row, U rows in flight per 16-lane group (registers)
//   cpa  : per-lane 16-B cp.async into a per-warp smem ring (U rows per warp per stage, 2 stages)
//   tma  : one cp.async.bulk per row into a per-warp smem ring, mbarrier completion (2 stages)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gb2 gather_bench2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U>
__global__ void k_ldg(const float4 *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n,
                      float4 *__restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = t >> 4;
  const int c = t & 15;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 4;
  for (int64_t r0 = g * U; r0 < n; r0 += ng * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < n) v[u] = __ldg(tab + (size_t)idx[r0 + u] * 16 + c);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r0 + u < n) out[(size_t)(r0 + u) * 16 + c] = v[u];
  }
}

// U rows per warp-stage, 2 stages; smem per warp = 2*U*256 B
template <int U>
__global__ void k_cpa(const float4 *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n,
                      float4 *__restrict__ out) {
  extern __shared__ __align__(16) float4 sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 *ring = sm + (size_t)w * 2 * U * 16;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  auto issue = [&](int64_t r0, int s) {
    for (int q = lane; q < U * 16; q += 32) {
      const int u = q >> 4, c = q & 15;
      if (r0 + u < n) {
        const float4 *src = tab + (size_t)idx[r0 + u] * 16 + c;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(ring + (s * U + u) * 16 + c)), "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  int64_t r = gw * U;
  issue(r, 0);
  issue(r + nw * U, 1);
  int s = 0;
  for (; r < n; r += nw * U) {
    asm volatile("cp.async.wait_group 1;");
    __syncwarp();
    for (int q = lane; q < U * 16; q += 32) {
      const int u = q >> 4, c = q & 15;
      if (r + u < n) out[(size_t)(r + u) * 16 + c] = ring[(s * U + u) * 16 + c];
    }
    __syncwarp();
    issue(r + 2 * nw * U, s);
    s ^= 1;
  }
  asm volatile("cp.async.wait_group 0;");
}

template <int U>
__global__ void k_tma(const float4 *__restrict__ tab, const uint32_t *__restrict__ idx, int64_t n,
                      float4 *__restrict__ out) {
  extern __shared__ __align__(128) float4 sm[];
  __shared__ uint64_t bar[32][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 *ring = sm + (size_t)w * 2 * U * 16;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto issue = [&](int64_t r0, int s) {
    int cnt = 0;
    for (int u = 0; u < U; ++u) cnt += (r0 + u < n);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[w][s])), "r"(cnt * 256));
    __syncwarp();
    for (int u = lane; u < U; u += 32)
      if (r0 + u < n)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                         su32(ring + (s * U + u) * 16)),
                     "l"(tab + (size_t)idx[r0 + u] * 16), "r"(su32(&bar[w][s])));
  };
  int64_t r = gw * U;
  issue(r, 0);
  issue(r + nw * U, 1);
  int s = 0;
  uint32_t ph[2] = {0, 0};
  for (; r < n; r += nw * U) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(ok)
                   : "r"(su32(&bar[w][s])), "r"(ph[s]));
    ph[s] ^= 1;
    for (int q = lane; q < U * 16; q += 32) {
      const int u = q >> 4, c = q & 15;
      if (r + u < n) out[(size_t)(r + u) * 16 + c] = ring[(s * U + u) * 16 + c];
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;");
    issue(r + 2 * nw * U, s);
    s ^= 1;
  }
}

int main(int argc, char **argv) {
  const double tab_gb = 64.0;
  const int64_t n = 4000000;
  const int64_t rows = (int64_t)(tab_gb * 1e9 / 256.0);
  float4 *tab, *out;
  uint32_t *idx;
  cudaMalloc(&tab, (size_t)rows * 256);
  cudaMalloc(&out, (size_t)n * 256);
  cudaMalloc(&idx, (size_t)n * 4);
  cudaMemset(tab, 0, (size_t)rows * 256);
  std::mt19937_64 rng(1);
  std::vector<uint32_t> h(n);
  for (auto &x : h) x = (uint32_t)(rng() % (uint64_t)rows);
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](const char *name, int wps, int inflight_rows_per_warp, auto launch) {
    for (int i = 0; i < 2; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const cudaError_t err = cudaGetLastError();
    printf("%-4s warps/SM %3d rows_in_flight/warp %3d KB_in_flight/SM %5.0f : %7.0f GB/s r+w %s\n", name, wps,
           inflight_rows_per_warp, wps * inflight_rows_per_warp * 0.25, 2.0 * n * 256 / (ms * 1e-3) / 1e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
#define LDG(U, WPS)                                                                                              \
  time("ldg", WPS, 2 * U, [&] { k_ldg<U><<<sms * (WPS / 8), 256>>>(tab, idx, n, out); });
  LDG(4, 16) LDG(8, 16) LDG(16, 16) LDG(4, 32) LDG(8, 32) LDG(16, 32) LDG(4, 64) LDG(8, 64)
#define CPA(U, WPS)                                                                                              \
  {                                                                                                              \
    const size_t sm_ = (size_t)8 * 2 * U * 256;                                                                  \
    cudaFuncSetAttribute(k_cpa<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_);                       \
    time("cpa", WPS, U, [&] { k_cpa<U><<<sms * (WPS / 8), 256, sm_>>>(tab, idx, n, out); });                     \
  }
  CPA(8, 16) CPA(16, 16) CPA(8, 32) CPA(16, 32) CPA(24, 16) CPA(32, 16)
#define TMA(U, WPS)                                                                                              \
  {                                                                                                              \
    const size_t sm_ = (size_t)8 * 2 * U * 256;                                                                  \
    cudaFuncSetAttribute(k_tma<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_);                       \
    time("tma", WPS, U, [&] { k_tma<U><<<sms * (WPS / 8), 256, sm_>>>(tab, idx, n, out); });                     \
  }
  TMA(8, 16) TMA(16, 16) TMA(8, 32) TMA(16, 32) TMA(24, 16) TMA(32, 16)
  return 0;
}
