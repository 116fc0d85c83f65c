// keys.cu — K1: CSR parse + validation + fused keys g = base[t] + id (readings R4, R5).
//
// One warp per 32 consecutive bags. Lane l holds bag (b0+l)'s [start, end) and its table's base/rows.
// The warp then walks the contiguous id range [start(b0), end(b0+31)) 32 ids at a time (coalesced
// int64 loads); each id finds its bag by a 5-step shuffle binary search over the lanes' starts, so
// skewed bag lengths cost no divergence. Outputs per occurrence j: fused key g (or EMB_SENTINEL for an
// invalid id) and its output row index b*S+s (the row of Y / dY it pools into); per bag: its length
// at that same row index.
#include "common.cuh"
#include "internal.h"

namespace emb {

__global__ void __launch_bounds__(256) k_keys(KeysArgs a) {
  const int64_t nb = (int64_t)a.num_slots * a.batch;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t b0 = warp * 32;
  if (b0 >= nb) return;  // warp-uniform
  const int64_t bag = b0 + lane;
  const bool inb = bag < nb;
  int64_t st = INT64_MAX, en = INT64_MAX;
  uint32_t bad = 0;
  uint64_t base = 0;
  int64_t rows = 0;
  uint32_t orow = 0;
  if (inb) {
    st = a.offsets[bag];
    en = a.offsets[bag + 1];
    if (st < 0 || en < st || en > a.nnz) bad = EMB_DEVERR_INVALID;
    if (bag == 0 && st != 0) bad = EMB_DEVERR_INVALID;
    if (bag == nb - 1 && en != a.nnz) bad = EMB_DEVERR_INVALID;
    st = st < 0 ? 0 : (st > a.nnz ? a.nnz : st);
    en = en < st ? st : (en > a.nnz ? a.nnz : en);
    const uint32_t slot = (uint32_t)bag / (uint32_t)a.batch;
    const uint32_t b = (uint32_t)bag - slot * (uint32_t)a.batch;
    orow = b * (uint32_t)a.num_slots + slot;
    if (a.blen) a.blen[orow] = (int32_t)(en - st);
    const int t = a.slot_table[slot];
    base = a.base[t];
    rows = a.rows[t];
  }
  // id range covered by this warp
  int64_t lo = __shfl_sync(0xffffffffu, st, 0);
  int64_t hi = inb ? en : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    int64_t x = __shfl_xor_sync(0xffffffffu, hi, o);
    hi = x > hi ? x : hi;
  }
  for (int64_t jb = lo; jb < hi; jb += 32) {
    const int64_t j = jb + lane;
    // largest lane l with start(l) <= j
    int l = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1) {
      const int64_t sc = __shfl_sync(0xffffffffu, st, l + step);
      if (sc <= j) l += step;
    }
    const int64_t enl = __shfl_sync(0xffffffffu, en, l);
    const uint64_t basel = __shfl_sync(0xffffffffu, base, l);
    const int64_t rowsl = __shfl_sync(0xffffffffu, rows, l);
    const uint32_t orowl = __shfl_sync(0xffffffffu, orow, l);
    if (j < hi) {
      const int64_t id = a.ids[j];
      uint32_t rk = EMB_SENTINEL;
      if (j >= enl) {
        bad |= EMB_DEVERR_INVALID;  // id not inside any bag (only with broken offsets)
      } else if (id < 0 || id >= rowsl) {
        bad |= EMB_DEVERR_RANGE;
      } else {
        rk = (uint32_t)(basel + (uint64_t)id);  // fused key g (< 2^32 - 1)
      }
      a.key[j] = rk;
      a.drow[j] = orowl;
    }
  }
  // one atomic per warp at most
  uint32_t any = __reduce_or_sync(0xffffffffu, bad);
  if (any && lane == 0) atomicOr(a.err, any);
}

cudaError_t launch_keys(const KeysArgs &a, cudaStream_t st) {
  const int64_t nb = (int64_t)a.num_slots * a.batch;
  if (nb == 0) return cudaSuccess;
  const int64_t warps = (nb + 31) / 32;
  const int threads = 256;
  const int64_t blocks = (warps * 32 + threads - 1) / threads;
  k_keys<<<(unsigned)blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace emb
