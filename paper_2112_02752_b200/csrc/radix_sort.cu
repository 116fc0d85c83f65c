// radix_sort.cu — stable LSD radix sort of (uint32 key, uint32 value) pairs: the sort behind the
// per-rank id dedup and the owner-side merge (A5). Stable, so within one key the
// values keep their input order: that order is what makes the backward's fp64 segment sums
// deterministic (R10).
//
// Design (one-sweep per digit, 8-bit digits, ceil(key_bits/8) passes):
//   k_sort_hist : one read of the keys builds all passes' 256-bin digit histograms (smem atomics,
//                 then one global atomic per non-zero bin and block).
//   k_sort_pass : a tile of 4096 keys per CTA (512 threads x 8 keys, warp-contiguous), tiles claimed
//                 in launch order through an atomic counter (forward progress for the look-back).
//                 Within a warp, keys are ranked stably with __match_any_sync per key row; warps'
//                 digit counts are scanned in smem; the tile's global digit offsets come from a
//                 decoupled look-back over the previous tiles' per-digit (flag|count) words. Then
//                 every key is scattered to its final position.
// All key-dependent work stays on chip except one read and one write of (key, value) per pass; at
// the sizes of the hot path (N <= a few M) the arrays are L2-resident.
#include "common.cuh"
#include "internal.h"

namespace emb {

namespace {
constexpr int RS_THREADS = 512;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096
constexpr int RS_RADIX = 256;
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1u;
}  // namespace

size_t sort_workspace_words(int64_t max_n) {
  const int64_t tiles = (max_n + RS_TILE - 1) / RS_TILE + 1;
  return (size_t)4 * RS_RADIX + 4 + (size_t)4 * tiles * RS_RADIX;
}

// all passes' digit histograms in one read of the keys: warp-private shared-memory histograms (hot-id
// workloads -- C5: 90% of the ids on 1,000 rows per table -- hammer a few bins; a block-wide histogram
// made every block's 512 threads contend on them, a MATCH.ANY per key and pass cost 6x more), then one
// global atomic per non-zero bin and block
constexpr int HIST_THREADS = 256;
__global__ void __launch_bounds__(HIST_THREADS) k_sort_hist(const uint32_t *__restrict__ keys, int64_t n, int npass,
                                                            uint32_t *__restrict__ hist) {
  __shared__ uint32_t h[HIST_THREADS / 32][4][256];
  for (int i = threadIdx.x; i < (HIST_THREADS / 32) * 4 * 256; i += blockDim.x) (&h[0][0][0])[i] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = keys[i];
    for (int p = 0; p < npass; ++p) atomicAdd(&h[w][p][(k >> (8 * p)) & 0xFFu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < HIST_THREADS / 32; ++q) c += h[q][i >> 8][i & 255];
    if (c) atomicAdd(&hist[i], c);
  }
}

__global__ void __launch_bounds__(RS_THREADS) k_sort_pass(const uint32_t *__restrict__ kin,
                                                          const uint32_t *__restrict__ vin,
                                                          uint32_t *__restrict__ kout, uint32_t *__restrict__ vout,
                                                          int64_t n, int shift, const uint32_t *__restrict__ hist,
                                                          uint32_t *status, uint32_t *tile_counter, uint32_t *err) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t warp_cnt[RS_WARPS][RS_RADIX];  // per-warp digit counts -> exclusive warp offsets
  __shared__ uint32_t digit_base[RS_RADIX];           // global start of this tile's digit run
  __shared__ uint32_t hist_scan[RS_RADIX];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&warp_cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t wbase = tile * RS_TILE + (int64_t)w * (RS_ITEMS * 32);

  uint32_t k[RS_ITEMS], v[RS_ITEMS], r[RS_ITEMS];
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    const int64_t pos = wbase + i * 32 + lane;
    k[i] = pos < n ? kin[pos] : 0u;
    v[i] = pos < n ? (vin ? vin[pos] : (uint32_t)pos) : 0u;
  }
  // stable in-warp ranking, row by row (position order = item-major, then lane)
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    const int64_t pos = wbase + i * 32 + lane;
    const bool valid = pos < n;
    const uint32_t d = (k[i] >> shift) & 0xFFu;
    const uint32_t tag = valid ? d : (0x10000u | (uint32_t)lane);
    const uint32_t peers = __match_any_sync(0xffffffffu, tag);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = warp_cnt[w][d];
      warp_cnt[w][d] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    r[i] = old + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan of the global histogram (digit start across the whole array)
  if (tid < RS_RADIX) {
    const uint32_t c = hist[tid];
    // 8 warps x 32 lanes scan
    uint32_t incl = warp_incl_scan(c);
    hist_scan[tid] = incl;  // temporarily inclusive within warp
  }
  __syncthreads();
  uint32_t my_count = 0;
  if (tid < RS_RADIX) {
    uint32_t carry = 0;
    for (int ww = 0; ww < (tid >> 5); ++ww) carry += hist_scan[ww * 32 + 31];
    // scan across warps of this tile per digit
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
      const uint32_t c = warp_cnt[ww][tid];
      warp_cnt[ww][tid] = run;
      run += c;
    }
    my_count = run;
    const uint32_t hist_excl = carry + hist_scan[tid] - hist[tid];
    // decoupled look-back over previous tiles for digit `tid`
    volatile uint32_t *st = status + tile * RS_RADIX + tid;
    uint32_t excl = 0;
    if (tile == 0) {
      *st = FLAG_INC | my_count;
    } else {
      *st = FLAG_AGG | my_count;
      // look back LB predecessors per round trip (independent loads), consuming them in order until
      // an inclusive prefix; a not-yet-published one is re-probed. (One dependent L2 read per
      // predecessor made the look-back chain through every concurrently running tile: 556 us per
      // pass at C5's 27M keys.)
      constexpr int LB = 8;
      int64_t look = tile - 1;
      bool done = false;
      while (!done) {
        uint32_t sv[LB];
#pragma unroll
        for (int q = 0; q < LB; ++q)
          sv[q] = look - q >= 0 ? *(volatile uint32_t *)(status + (look - q) * RS_RADIX + tid) : (FLAG_INC | 0u);
        int used = 0;
#pragma unroll
        for (int q = 0; q < LB; ++q) {
          if (done || used < q) break;  // stop at the first unpublished one (used == q while consuming)
          const uint32_t v = sv[q];
          if ((v & ~VAL_MASK) == 0) break;
          excl += v & VAL_MASK;
          ++used;
          if (v & FLAG_INC) done = true;
        }
        look -= used;
      }
      *st = FLAG_INC | (excl + my_count);
    }
    digit_base[tid] = hist_excl + excl;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    const int64_t pos = wbase + i * 32 + lane;
    if (pos < n) {
      const uint32_t d = (k[i] >> shift) & 0xFFu;
      const uint32_t dst = digit_base[d] + warp_cnt[w][d] + r[i];
      if (dst < (uint64_t)n) {
        kout[dst] = k[i];
        vout[dst] = v[i];
      } else {
        atomicOr(err, EMB_DEVERR_INTERNAL);
      }
    }
  }
}

cudaError_t radix_sort_pairs(const SortWorkspace &ws, const uint32_t *kin, const uint32_t *vin, uint32_t *k0,
                             uint32_t *v0, uint32_t *k1, uint32_t *v1, int64_t n, uint32_t key_bits,
                             cudaStream_t st, uint32_t **keys_out, uint32_t **vals_out, int *launches,
                             ProfHook prof, void *prof_ctx) {
  *keys_out = k0;
  *vals_out = v0;
  if (n <= 0) return cudaSuccess;
  int npass = (int)((key_bits + 7) / 8);
  if (npass < 1) npass = 1;
  if (npass > 4) npass = 4;
  const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  // zero histograms, tile counters and look-back words of the passes we run
  cudaError_t e = cudaMemsetAsync(ws.hist, 0, sizeof(uint32_t) * (4 * RS_RADIX + 4), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ws.status, 0, sizeof(uint32_t) * (size_t)npass * ws.max_tiles * RS_RADIX, st);
  if (e != cudaSuccess) return e;
  int hblocks = (int)((n + 4095) / 4096);
  if (hblocks > 148 * 4) hblocks = 148 * 4;
  if (prof) prof(prof_ctx, KID_SORT_HIST, 0, st);
  k_sort_hist<<<hblocks, HIST_THREADS, 0, st>>>(kin, n, npass, ws.hist);
  if (prof) prof(prof_ctx, KID_SORT_HIST, 1, st);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int nl = 1;
  const uint32_t *ki = kin, *vi = vin;
  uint32_t *ko = k0, *vo = v0, *ka = k1, *va = v1;
  for (int p = 0; p < npass; ++p) {
    if (prof) prof(prof_ctx, KID_SORT_PASS, 0, st);
    k_sort_pass<<<(unsigned)tiles, RS_THREADS, 0, st>>>(ki, vi, ko, vo, n, 8 * p, ws.hist + p * RS_RADIX,
                                                        ws.status + (size_t)p * ws.max_tiles * RS_RADIX,
                                                        ws.counters + p, ws.err);
    if (prof) prof(prof_ctx, KID_SORT_PASS, 1, st);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++nl;
    *keys_out = ko;
    *vals_out = vo;
    ki = ko;
    vi = vo;
    uint32_t *tk = ko, *tv = vo;
    ko = ka;
    vo = va;
    ka = tk;
    va = tv;
  }
  if (launches) *launches += nl;
  return cudaSuccess;
}

}  // namespace emb
