// ipc_gather_bench.cu — like peer_gather_bench.cu but across TWO PROCESSES with CUDA IPC mappings (the
// layout libemb's one-process-per-GPU mode uses): process r on GPU r exports its 12.8 GB table, imports
// the other's, then (a) one direction alone, (b) both directions at the same time: random 256-B row
// pulls (peer loads) and pushes (peer stores) of 100K rows.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ipc_gather_bench tools/ipc_gather_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <unistd.h>
#include <sys/wait.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("[%d] %s: %s\n", getpid(), #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int STORE>
__global__ void k_move(const float4 *__restrict__ src, const uint32_t *__restrict__ idx, float4 *__restrict__ dst,
                       int64_t nrows) {
  const int64_t total = nrows * 16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = t0 + u * stride;
      if (t < total) {
        const int64_t r = t >> 4;
        const int c = (int)(t & 15);
        // STORE = 0: pull (src remote, gathered rows); 1: push (src local gathered, dst remote, gathered)
        v[u] = src[(size_t)idx[r] * 16 + c];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = t0 + u * stride;
      if (t < total) dst[t] = v[u];
    }
  }
}

static void xfer(int wfd, const void *p, size_t n) { if (write(wfd, p, n) != (ssize_t)n) exit(2); }
static void rcv(int rfd, void *p, size_t n) { size_t g = 0; while (g < n) { ssize_t k = read(rfd, (char *)p + g, n - g); if (k <= 0) exit(3); g += k; } }

int run(int me, int rfd, int wfd) {
  const int64_t rows_tab = 50'000'000, n = 100'000;
  CK(cudaSetDevice(me));
  float4 *tab, *dst, *rtab, *rdst;
  uint32_t *idx;
  CK(cudaMalloc(&tab, rows_tab * 256));
  CK(cudaMemset(tab, 0, rows_tab * 256));
  CK(cudaMalloc(&dst, n * 256));
  std::vector<uint32_t> h(n);
  uint64_t x = 88172645463325252ull + me;
  for (int64_t i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)(x % rows_tab); }
  CK(cudaMalloc(&idx, n * 4));
  CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
  cudaIpcMemHandle_t ht, hd, ot, od;
  CK(cudaIpcGetMemHandle(&ht, tab));
  CK(cudaIpcGetMemHandle(&hd, dst));
  xfer(wfd, &ht, sizeof(ht)); xfer(wfd, &hd, sizeof(hd));
  rcv(rfd, &ot, sizeof(ot)); rcv(rfd, &od, sizeof(od));
  CK(cudaIpcOpenMemHandle((void **)&rtab, ot, cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle((void **)&rdst, od, cudaIpcMemLazyEnablePeerAccess));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto sync = [&] { char c = 1; xfer(wfd, &c, 1); rcv(rfd, &c, 1); };
  auto timeit = [&](const char *name, bool active, auto launch) {
    sync();
    if (active) {
      for (int i = 0; i < 3; ++i) launch();
      CK(cudaDeviceSynchronize());
    }
    sync();
    const int reps = 20;
    if (active) {
      CK(cudaEventRecord(e0));
      for (int i = 0; i < reps; ++i) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double us = 1e3 * ms / reps;
      printf("[gpu %d] %-34s %8.2f us  %7.1f GB/s\n", me, name, us, n * 256.0 / (us * 1e-6) / 1e9);
      fflush(stdout);
    }
    sync();
  };
  const int grid = 148 * 8, B = 256;
  timeit("pull ipc, one direction", me == 0, [&] { k_move<0><<<grid, B>>>(rtab, idx, dst, n); });
  timeit("push ipc, one direction", me == 0, [&] { k_move<1><<<grid, B>>>(tab, idx, rdst, n); });
  timeit("pull ipc, both directions", true, [&] { k_move<0><<<grid, B>>>(rtab, idx, dst, n); });
  timeit("push ipc, both directions", true, [&] { k_move<1><<<grid, B>>>(tab, idx, rdst, n); });
  timeit("local gather", true, [&] { k_move<0><<<grid, B>>>(tab, idx, dst, n); });
  CK(cudaIpcCloseMemHandle(rtab));
  CK(cudaIpcCloseMemHandle(rdst));
  return 0;
}

int main() {
  int a[2], b[2];
  if (pipe(a) || pipe(b)) return 1;
  pid_t pid = fork();
  if (pid == 0) return run(1, a[0], b[1]);
  int rc = run(0, b[0], a[1]);
  int st = 0;
  waitpid(pid, &st, 0);
  return rc | WEXITSTATUS(st);
}
