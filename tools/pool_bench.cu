// pool_bench.cu — calibration only (not part of libemb): which part of the pool's access pattern
// costs bandwidth? 425,984 single-id bags (C2 shape: 26 slots x 16,384), 256-B rows gathered from a
// 133 GB table, written to Y[b][s] (slot-major bags -> rows 26 apart) or contiguously.
// Variants (one warp per 32 bags, 16 rows in flight per lane-row, as k_pool):
//   A  row index from a precomputed u32 array (1 dependent load), contiguous output
//   B  A with the pool's strided Y rows (b*S + s)
//   C  offsets -> id -> row chain (3 dependent loads), strided output  (= the pool's single-id path)
// ids: uniform over 260M rows, or "zipfish" (30% from 1400 hot rows per table).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pool_bench tools/pool_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <random>
#include <vector>

constexpr int S = 26, B = 16384, D = 64;
constexpr int64_t ROWS_T = 10000000, ROWS = ROWS_T * S;

__device__ __forceinline__ float2 ldnc2(const float *p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void stcs2(float *p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256, 3) k_var(const float *__restrict__ tab, const uint32_t *__restrict__ rowidx,
                                                const int64_t *__restrict__ offsets, const int64_t *__restrict__ ids,
                                                float *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nb = (int64_t)S * B;
  const int64_t bag = tile * 32 + lane;
  if (tile * 32 >= nb) return;
  uint32_t row;
  if (MODE == 2) {
    const int64_t off = offsets[bag];
    const int64_t id = ids[off];
    const int s = (int)(bag / B);
    row = (uint32_t)(s * ROWS_T + id);
  } else {
    row = rowidx[bag];
  }
  const uint32_t s = (uint32_t)(bag / B);
  const uint32_t orow = MODE == 0 ? (uint32_t)bag : (uint32_t)((bag - (int64_t)s * B) * S + s);
#pragma unroll
  for (int c0 = 0; c0 < 32; c0 += 16) {
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t ri = __shfl_sync(0xffffffffu, row, c0 + r);
      v[r] = ldnc2(tab + (size_t)ri * D + lane * 2);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t oi = __shfl_sync(0xffffffffu, orow, c0 + r);
      stcs2(out + (size_t)oi * D + lane * 2, v[r]);
    }
  }
}

int main() {
  const int64_t nb = (int64_t)S * B;
  float *tab, *out;
  uint32_t *rowidx;
  int64_t *offsets, *ids;
  if (cudaMalloc(&tab, (size_t)ROWS * D * 4 * 2) != cudaSuccess) {  // 133 GB like C2's table + state
    printf("alloc failed\n");
    return 1;
  }
  cudaMalloc(&out, (size_t)nb * D * 4);
  cudaMalloc(&rowidx, nb * 4);
  cudaMalloc(&offsets, (nb + 1) * 8);
  cudaMalloc(&ids, nb * 8);
  cudaMemset(tab, 0, (size_t)1 << 30);
  std::mt19937_64 rng(7);
  std::vector<int64_t> hoff(nb + 1), hid(nb);
  std::vector<uint32_t> hrow(nb);
  for (int64_t i = 0; i <= nb; ++i) hoff[i] = i;
  for (int dist = 0; dist < 2; ++dist) {
    for (int64_t b = 0; b < nb; ++b) {
      const int s = (int)(b / B);
      uint64_t id = rng() % ROWS_T;
      if (dist == 1 && rng() % 10 < 3) id = (rng() % 1400) * 7919u % ROWS_T;
      hid[b] = (int64_t)id;
      hrow[b] = (uint32_t)(s * ROWS_T + id);
    }
    cudaMemcpy(offsets, hoff.data(), (nb + 1) * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(ids, hid.data(), nb * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(rowidx, hrow.data(), nb * 4, cudaMemcpyHostToDevice);
    const unsigned blocks = (unsigned)((nb / 32 * 32 + 255) / 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
      for (int it = 0; it < 3; ++it) {
        if (mode == 0) k_var<0><<<blocks, 256>>>(tab, rowidx, offsets, ids, out);
        if (mode == 1) k_var<1><<<blocks, 256>>>(tab, rowidx, offsets, ids, out);
        if (mode == 2) k_var<2><<<blocks, 256>>>(tab, rowidx, offsets, ids, out);
      }
      cudaEventRecord(e0);
      const int N = 20;
      for (int it = 0; it < N; ++it) {
        if (mode == 0) k_var<0><<<blocks, 256>>>(tab, rowidx, offsets, ids, out);
        if (mode == 1) k_var<1><<<blocks, 256>>>(tab, rowidx, offsets, ids, out);
        if (mode == 2) k_var<2><<<blocks, 256>>>(tab, rowidx, offsets, ids, out);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms / N * 1000;
      printf("%s ids, variant %c: %.1f us/launch (%.0f GB/s rows read + Y written)\n", dist ? "zipfish" : "uniform",
             'A' + mode, us, 2.0 * nb * D * 4 / (us * 1e3));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
