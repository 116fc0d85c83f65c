// sort_calib.cu — calibration only (not part of libemb): how long does a library radix sort
// (cub::DeviceRadixSort / DeviceSegmentedSort) take on the C2 dedup problem (426k (key, index)
// pairs, 28-bit fused keys; or 26 segments of 16,384 with 24-bit keys)? Sets the bar for segsort.cu.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdio.h>

#include <random>
#include <vector>

int main() {
  const int n = 425984, S = 26, per = 16384;
  std::mt19937_64 rng(7);
  std::vector<uint32_t> hk(n), hv(n);
  for (int s = 0; s < S; ++s)
    for (int i = 0; i < per; ++i) {
      // Zipf-ish: 30% of draws from 1400 hot rows, the rest uniform over 10M
      const uint32_t id = (rng() % 10 < 3) ? (uint32_t)(rng() % 1400) * 7919u % 10000000u : (uint32_t)(rng() % 10000000u);
      hk[s * per + i] = s * 10000000u + id;
      hv[s * per + i] = s * per + i;
    }
  uint32_t *k0, *k1, *v0, *v1;
  cudaMalloc(&k0, n * 4);
  cudaMalloc(&k1, n * 4);
  cudaMalloc(&v0, n * 4);
  cudaMalloc(&v1, n * 4);
  cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n, 0, 28);
  void *dt;
  cudaMalloc(&dt, tmp + (1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) cub::DeviceRadixSort::SortPairs(dt, tmp, k0, k1, v0, v1, n, 0, 28);
  cudaEventRecord(e0);
  for (int i = 0; i < 50; ++i) cub::DeviceRadixSort::SortPairs(dt, tmp, k0, k1, v0, v1, n, 0, 28);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cub::DeviceRadixSort::SortPairs n=%d bits=28: %.1f us\n", n, ms / 50 * 1000);
  // segmented: 26 segments of 16384, sort by full key (cub DeviceSegmentedSort)
  std::vector<int> off(S + 1);
  for (int s = 0; s <= S; ++s) off[s] = s * per;
  int *doff;
  cudaMalloc(&doff, (S + 1) * 4);
  cudaMemcpy(doff, off.data(), (S + 1) * 4, cudaMemcpyHostToDevice);
  size_t tmp2 = 0;
  cub::DeviceSegmentedSort::StableSortPairs(nullptr, tmp2, k0, k1, v0, v1, n, S, doff, doff + 1);
  void *dt2;
  cudaMalloc(&dt2, tmp2 + (1 << 20));
  for (int i = 0; i < 5; ++i) cub::DeviceSegmentedSort::StableSortPairs(dt2, tmp2, k0, k1, v0, v1, n, S, doff, doff + 1);
  cudaEventRecord(e0);
  for (int i = 0; i < 50; ++i) cub::DeviceSegmentedSort::StableSortPairs(dt2, tmp2, k0, k1, v0, v1, n, S, doff, doff + 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cub::DeviceSegmentedSort::StableSortPairs n=%d segs=%d: %.1f us\n", n, S, ms / 50 * 1000);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
