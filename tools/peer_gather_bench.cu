// peer_gather_bench.cu — calibration of random 256-B row gathers across NVLink (2 GPUs, one process,
// cudaDeviceEnablePeerAccess): which access pattern moves rows from a peer's table fastest?
//   pull_nc   : GPU0 threads load float4 from GPU1's table with ld.global.nc, store locally
//   pull_ld   : the same with plain ld.global (L1::no_allocate)
//   pull_cg   : ld.global.cg
//   pull_cpas : cp.async 16 B (LDGSTS) peer -> shared, then store locally
//   push_st   : GPU1 threads load local rows and store them into GPU0's buffer (remote writes)
//   local     : GPU0 gathers from its own table (reference)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/peer_gather_bench tools/peer_gather_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ float4 ld_nc(const float4 *p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_plain(const float4 *p) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_cg(const float4 *p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

template <int MODE, int U>
__global__ void k_gather(const float4 *__restrict__ src, const uint32_t *__restrict__ idx, float4 *__restrict__ dst,
                         int64_t nrows) {
  const int64_t total = nrows * 16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + u * stride;
      if (t < total) {
        const int64_t r = t >> 4;
        const int c = (int)(t & 15);
        const float4 *p = src + (size_t)idx[r] * 16 + c;
        v[u] = MODE == 0 ? ld_nc(p) : (MODE == 1 ? ld_plain(p) : ld_cg(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + u * stride;
      if (t < total) dst[t] = v[u];
    }
  }
}

// cp.async: each warp copies rows (2 per 32 lanes) peer -> smem, then stores them
template <int RPW>
__global__ void k_gather_cpas(const float4 *__restrict__ src, const uint32_t *__restrict__ idx, float4 *__restrict__ dst,
                              int64_t nrows) {
  extern __shared__ float4 sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 *my = sm + (size_t)w * RPW * 16;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = gw * RPW; r0 < nrows; r0 += nw * RPW) {
    for (int q = lane; q < RPW * 16; q += 32) {
      const int64_t r = r0 + q / 16;
      if (r < nrows) {
        const float4 *p = src + (size_t)idx[r] * 16 + (q & 15);
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(my + q);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(p) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    for (int q = lane; q < RPW * 16; q += 32) {
      const int64_t r = r0 + q / 16;
      if (r < nrows) dst[(size_t)r * 16 + (q & 15)] = my[q];
    }
    __syncwarp();
  }
}

int main(int argc, char **argv) {
  const int64_t rows_tab = 50'000'000;    // 12.8 GB table on the owner (C3 at W = 2)
  const int64_t n = 100'000;              // rows gathered
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("needs 2 GPUs\n"); return 0; }
  int ok01 = 0, ok10 = 0;
  CK(cudaDeviceCanAccessPeer(&ok01, 0, 1));
  CK(cudaDeviceCanAccessPeer(&ok10, 1, 0));
  printf("peer access 0->1 %d 1->0 %d\n", ok01, ok10);
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  float4 *tab1, *tab0, *dst0, *dst_remote;
  uint32_t *idx0, *idx1;
  std::vector<uint32_t> hidx(n);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hidx[i] = (uint32_t)(x % rows_tab); }
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&tab1, rows_tab * 256));
  CK(cudaMemset(tab1, 0, rows_tab * 256));
  CK(cudaMalloc(&idx1, n * 4));
  CK(cudaMemcpy(idx1, hidx.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&tab0, rows_tab * 256));
  CK(cudaMemset(tab0, 0, rows_tab * 256));
  CK(cudaMalloc(&dst0, n * 256));
  CK(cudaMalloc(&idx0, n * 4));
  CK(cudaMemcpy(idx0, hidx.data(), n * 4, cudaMemcpyHostToDevice));
  dst_remote = dst0;
  cudaEvent_t e0, e1;
  auto timeit = [&](const char *name, int dev, auto launch) {
    CK(cudaSetDevice(dev));
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    const int reps = 20;
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double us = 1e3 * ms / reps;
    printf("%-28s %8.2f us  %7.1f GB/s (rows moved)\n", name, us, n * 256.0 / (us * 1e-6) / 1e9);
    CK(cudaGetLastError());
  };
  const int B = 256;
  for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
    printf("-- grid %d x %d\n", grid, B);
    timeit("local ld.nc U4", 0, [&] { k_gather<0, 4><<<grid, B>>>(tab0, idx0, dst0, n); });
    timeit("pull ld.nc U4", 0, [&] { k_gather<0, 4><<<grid, B>>>(tab1, idx0, dst0, n); });
    timeit("pull ld U4", 0, [&] { k_gather<1, 4><<<grid, B>>>(tab1, idx0, dst0, n); });
    timeit("pull ld.cg U4", 0, [&] { k_gather<2, 4><<<grid, B>>>(tab1, idx0, dst0, n); });
    timeit("pull ld U8", 0, [&] { k_gather<1, 8><<<grid, B>>>(tab1, idx0, dst0, n); });
    timeit("pull cp.async 8 rows/warp", 0, [&] {
      k_gather_cpas<8><<<grid, B, 8 * 8 * 256>>>(tab1, idx0, dst0, n); });
    timeit("push st U4 (GPU1 -> GPU0)", 1, [&] { k_gather<0, 4><<<grid, B>>>(tab1, idx1, dst_remote, n); });
  }
  return 0;
}
