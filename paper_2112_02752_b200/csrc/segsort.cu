// segsort.cu — per-table stable sort of the step's keys (dedup by sorting), the fast
// path of the world == 1 step.
//
// When slot_table is non-decreasing (true for every BASELINE config: C1/C4 share one table, C2/C3/C5
// map slot s -> table s), the slot-major CSR is already grouped by table and the table groups appear
// in fused-key order, so sorting the whole array is the same as sorting each group in place. One
// CTA per group sorts (local id = key - base[t], payload = occurrence index) with a stable LSD radix
// sort on the group's own key bits (ceil(log2(rows[t]+1)): 24 bits = 3 passes for a 10M-row table)
// entirely in shared memory (keys + two index buffers, 12 B per occurrence, up to SEG_CAP = 16,384
// occurrences). Each pass counts digits per warp with shared-memory atomics over the warp's
// contiguous chunk, scans the (digit, warp) counters digit-major across the CTA's 32 warps, then ranks
// stably with a warp-level multisplit (peer masks from 8 ballots per 32-item row) while
// scattering. Larger groups run the same code on global-memory scratch (correct, slower).
// Invalid occurrences (EMB_SENTINEL) get local key rows[t] and sort to the end of their group.
#include "common.cuh"
#include "internal.h"

namespace emb {

namespace {
constexpr int SS_THREADS = 1024;
constexpr int SS_WARPS = SS_THREADS / 32;
}  // namespace

// lanes of the warp holding the same 8-bit digit as this lane (8 ballots; cheaper than match.any)
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid) {
  uint32_t m = __ballot_sync(0xffffffffu, valid);
  if (!valid) m = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return m;
}

size_t segsort_smem_bytes() { return (size_t)SEG_CAP * 12; }

__global__ void __launch_bounds__(SS_THREADS) k_segsort(const __grid_constant__ SegSortArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ uint32_t cnt[SS_WARPS][256];
  __shared__ uint32_t part[SS_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = blockIdx.x;
  const int64_t B = a.batch;
  int64_t lo = a.offsets[(int64_t)a.gslot[g] * B];
  int64_t hi = a.offsets[(int64_t)a.gslot[g + 1] * B];
  lo = lo < 0 ? 0 : (lo > a.nnz ? a.nnz : lo);
  hi = hi < lo ? lo : (hi > a.nnz ? a.nnz : hi);
  const int64_t n = hi - lo;
  if (n == 0) return;
  const uint32_t base = (uint32_t)a.gbase[g];
  const uint32_t rows = a.grows[g];
  const uint32_t bits = a.gbits[g];
  uint32_t *keys, *ia, *ib;
  if (n <= SEG_CAP) {
    keys = sm;
    ia = sm + n;
    ib = sm + 2 * n;
  } else {
    keys = a.scratch_k + lo;
    ia = a.scratch_a + lo;
    ib = a.scratch_b + lo;
  }
#pragma unroll 4
  for (int64_t i = tid; i < n; i += SS_THREADS) {
    const uint32_t k = a.key_csr[lo + i];
    keys[i] = (k == EMB_SENTINEL) ? rows : k - base;
  }
  __syncthreads();
  const int64_t chunk = ((n + SS_WARPS - 1) / SS_WARPS + 31) / 32 * 32;  // rows of 32 per warp
  const int64_t c_lo = (int64_t)w * chunk;
  const int64_t c_hi = (c_lo + chunk < n) ? c_lo + chunk : n;
  const int npass = (int)((bits + 7) / 8);
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = 8 * pass;
    for (int d = lane; d < 256; d += 32) cnt[w][d] = 0;
    __syncwarp();
    // 1. per-warp digit counts over the warp's contiguous chunk (shared-memory atomics)
    for (int64_t p = c_lo + lane; p < c_hi; p += 32) {
      const uint32_t item = pass == 0 ? (uint32_t)p : ia[p];
      atomicAdd(&cnt[w][(keys[item] >> shift) & 0xFFu], 1u);
    }
    __syncthreads();
    // 2. digit-major exclusive scan over (digit, warp): thread t owns digit t/4, warps (t&3)*8 .. +7
    {
      const int d = tid >> 2, w0 = (tid & 3) * 8;
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += cnt[w0 + q][d];
      const uint32_t incl = warp_incl_scan(s);
      if (lane == 31) part[w] = incl;
      __syncthreads();
      if (w == 0) {
        const uint32_t t = lane < SS_THREADS / 32 ? part[lane] : 0;
        const uint32_t ti = warp_incl_scan(t);
        if (lane < SS_THREADS / 32) part[lane] = ti - t;
      }
      __syncthreads();
      uint32_t run = part[w] + incl - s;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t c = cnt[w0 + q][d];
        cnt[w0 + q][d] = run;
        run += c;
      }
    }
    __syncthreads();
    // 3. stable scatter: same walk, running per-warp digit cursors
    for (int64_t r0 = c_lo; r0 < c_hi; r0 += 32) {
      const int64_t p = r0 + lane;
      const bool valid = p < c_hi;
      const uint32_t item = valid ? (pass == 0 ? (uint32_t)p : ia[p]) : 0u;
      const uint32_t d = valid ? (keys[item] >> shift) & 0xFFu : 0u;
      const uint32_t peers = digit_peers(d, valid);
      const int leader = valid ? __ffs(peers) - 1 : 0;
      uint32_t basepos = 0;
      if (valid && lane == leader) {
        basepos = cnt[w][d];
        cnt[w][d] = basepos + __popc(peers);
      }
      basepos = __shfl_sync(0xffffffffu, basepos, leader);
      if (valid) {
        const uint32_t dst = basepos + __popc(peers & lanemask_lt());
        if (dst < (uint64_t)n) ib[dst] = item;
        else atomicOr(a.err, EMB_DEVERR_INTERNAL);
      }
      __syncwarp();
    }
    __syncthreads();
    uint32_t *t = ia;
    ia = ib;
    ib = t;
  }
  for (int64_t i = tid; i < n; i += SS_THREADS) {
    const uint32_t item = ia[i];
    const uint32_t lk = keys[item];
    a.skey[lo + i] = (lk >= rows) ? EMB_SENTINEL : base + lk;
    a.spay[lo + i] = (uint32_t)(lo + item);
  }
}

cudaError_t launch_segsort(const SegSortArgs &a, int32_t groups, cudaStream_t st) {
  if (groups <= 0 || a.nnz <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_segsort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)segsort_smem_bytes());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_segsort<<<groups, SS_THREADS, segsort_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

}  // namespace emb
