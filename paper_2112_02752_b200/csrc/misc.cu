// misc.cu — dedup compaction (A2; step statistics and emb_last_unique), table init (R15) and row
// export/import kernels.
#include "common.cuh"
#include "internal.h"

namespace emb {

// ------------------------------------------------------------------------------------------------
// k_unique: segment heads of the sorted key array -> unique index per position (useg), unique keys
// (ukey), segment starts (ustart, with ustart[U] = #valid), U. One tile of 4096 positions per CTA,
// 512 threads x 8 consecutive positions; tile prefix by decoupled look-back (tiles claimed in order).
namespace {
constexpr int UQ_THREADS = 512;
constexpr int UQ_ITEMS = 8;
constexpr int UQ_TILE = UQ_THREADS * UQ_ITEMS;
constexpr uint32_t UF_AGG = 1u << 30, UF_INC = 2u << 30, UF_MASK = (1u << 30) - 1u;  // low word; epoch high
}  // namespace

size_t unique_status_words(int64_t max_n) { return (size_t)((max_n + UQ_TILE - 1) / UQ_TILE + 1) + 1; }

__global__ void __launch_bounds__(UQ_THREADS) k_unique(const __grid_constant__ UniqueArgs a) {
  __shared__ uint32_t s_tile, s_excl;
  __shared__ uint32_t warp_tot[UQ_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    s_tile = atomicAdd(a.counter, 1u);
    if (s_tile == gridDim.x - 1) *a.counter = 0;  // last ticket of this launch: ready for the next one
  }
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * UQ_TILE + (int64_t)tid * UQ_ITEMS;
  // the tile's keys (+ one before, one after) staged through shared memory with coalesced loads
  __shared__ uint32_t s_k[UQ_TILE + 2];
  const int64_t t0 = tile * UQ_TILE;
#pragma unroll
  for (int i = 0; i < UQ_ITEMS; ++i) {
    const int64_t p = t0 + i * UQ_THREADS + tid;
    s_k[1 + i * UQ_THREADS + tid] = p < a.n ? a.skey[p] : EMB_SENTINEL;
  }
  if (tid == 0) s_k[0] = (t0 > 0 && t0 - 1 < a.n) ? a.skey[t0 - 1] : EMB_SENTINEL;
  if (tid == 1) s_k[UQ_TILE + 1] = (t0 + UQ_TILE < a.n) ? a.skey[t0 + UQ_TILE] : EMB_SENTINEL;
  __syncthreads();
  uint32_t k[UQ_ITEMS + 1];
  const uint32_t prev = s_k[tid * UQ_ITEMS];
#pragma unroll
  for (int i = 0; i <= UQ_ITEMS; ++i) k[i] = s_k[1 + tid * UQ_ITEMS + i];
  uint32_t flags = 0, cnt = 0;
#pragma unroll
  for (int i = 0; i < UQ_ITEMS; ++i) {
    const uint32_t kp = i == 0 ? prev : k[i - 1];
    const bool h = k[i] != EMB_SENTINEL && k[i] != kp;
    flags |= (uint32_t)h << i;
    cnt += h;
  }
  // block exclusive scan of cnt
  uint32_t incl = warp_incl_scan(cnt);
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < UQ_THREADS / 32 ? warp_tot[lane] : 0;
    uint32_t ti = warp_incl_scan(t);
    if (lane < UQ_THREADS / 32) warp_tot[lane] = ti - t;  // exclusive warp offsets
    const uint32_t total = __shfl_sync(0xffffffffu, ti, UQ_THREADS / 32 - 1);
    if (lane == 0) {
      volatile unsigned long long *st = reinterpret_cast<volatile unsigned long long *>(a.status) + tile;
      const unsigned long long tag = (unsigned long long)a.epoch << 32;
      uint32_t excl = 0;
      if (tile == 0) {
        *st = tag | UF_INC | total;
      } else {
        *st = tag | UF_AGG | total;
        int64_t look = tile - 1;
        while (true) {
          unsigned long long s;
          do {
            s = reinterpret_cast<volatile unsigned long long *>(a.status)[look];
          } while ((s >> 32) != a.epoch || ((uint32_t)s & ~UF_MASK) == 0);
          excl += (uint32_t)s & UF_MASK;
          if ((uint32_t)s & UF_INC) break;
          --look;
        }
        *st = tag | UF_INC | (excl + total);
      }
      s_excl = excl;
      if (tile == (int64_t)gridDim.x - 1) *a.u_count = excl + total;
    }
  }
  __syncthreads();
  uint32_t u = s_excl + warp_tot[w] + (incl - cnt);  // heads before my first position
#pragma unroll
  for (int i = 0; i < UQ_ITEMS; ++i) {
    const int64_t p = base + i;
    if (p >= a.n || k[i] == EMB_SENTINEL) continue;
    if ((flags >> i) & 1u) {
      a.ukey[u] = k[i];
      a.ustart[u] = (uint32_t)p;
      ++u;
    }
    a.useg[p] = u - 1;
    if (k[i + 1] != k[i]) a.uend[u - 1] = (uint32_t)(p + 1);  // last position of the segment
  }
}

cudaError_t launch_unique(const UniqueArgs &a, cudaStream_t st) {
  const int64_t tiles = a.n > 0 ? (a.n + UQ_TILE - 1) / UQ_TILE : 1;
  k_unique<<<(unsigned)tiles, UQ_THREADS, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// table init (R15): w[g][c] = int16(splitmix64(seed ^ (g*D + c)) >> 48) * 2^-19, a = init_accum
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_init(float4 *w, float4 *a, float *a_row, int64_t rows_local, int d4, uint64_t seed,
                       float init_accum, KeySpace ks, int32_t rank) {
  const int64_t total = rows_local * d4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t D = (uint64_t)d4 * 4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t r = t / d4;
    const int c4 = (int)(t - r * d4);
    uint64_t g;
    if (ks.world == 1) g = (uint64_t)r;
    else if (ks.shard == 0) g = (uint64_t)r * (uint64_t)ks.world + (uint64_t)rank;
    else g = (uint64_t)rank * ks.rows_per + (uint64_t)r;
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t h = splitmix64(seed ^ (g * D + (uint64_t)(c4 * 4 + q)));
      v[q] = (float)(int16_t)(uint16_t)(h >> 48) * 0x1p-19f;
    }
    w[t] = make_float4(v[0], v[1], v[2], v[3]);
    if (a) a[t] = make_float4(init_accum, init_accum, init_accum, init_accum);
    if (a_row && c4 == 0) a_row[r] = init_accum;
  }
}
cudaError_t launch_init(float *w, float *a, int32_t a_per_row, int64_t rows_local, int32_t dim, uint64_t seed,
                        float init_accum, const KeySpace &ks, int32_t rank, cudaStream_t st) {
  if (rows_local <= 0) return cudaSuccess;
  k_init<<<148 * 8, 256, 0, st>>>(reinterpret_cast<float4 *>(w), a_per_row ? nullptr : reinterpret_cast<float4 *>(a),
                                  a_per_row ? a : nullptr, rows_local, dim / 4, seed, init_accum, ks, rank);
  return cudaGetLastError();
}

__global__ void k_rows_copy(const float4 *src, float4 *dst, const int64_t *rows, int64_t n, int d4, int gather) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = t / d4;
  const int c = (int)(t - i * d4);
  if (i >= n) return;
  if (gather) dst[t] = src[(size_t)rows[i] * d4 + c];
  else dst[(size_t)rows[i] * d4 + c] = src[t];
}
// one float per row (row-wise Adagrad accumulators)
__global__ void k_rows_copy1(const float *src, float *dst, const int64_t *rows, int64_t n, int gather) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (gather) dst[i] = src[rows[i]];
  else dst[rows[i]] = src[i];
}

cudaError_t launch_rows_gather(const float *src, const int64_t *rows, int64_t n, int32_t dim, float *dst,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (dim == 1) {
    k_rows_copy1<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, rows, n, 1);
    return cudaGetLastError();
  }
  const int d4 = dim / 4;
  k_rows_copy<<<(unsigned)((n * d4 + 255) / 256), 256, 0, st>>>(reinterpret_cast<const float4 *>(src),
                                                                reinterpret_cast<float4 *>(dst), rows, n, d4, 1);
  return cudaGetLastError();
}
cudaError_t launch_rows_scatter(float *dst, const int64_t *rows, int64_t n, int32_t dim, const float *src,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (dim == 1) {
    k_rows_copy1<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, dst, rows, n, 0);
    return cudaGetLastError();
  }
  const int d4 = dim / 4;
  k_rows_copy<<<(unsigned)((n * d4 + 255) / 256), 256, 0, st>>>(reinterpret_cast<const float4 *>(src),
                                                                reinterpret_cast<float4 *>(dst), rows, n, d4, 0);
  return cudaGetLastError();
}

}  // namespace emb
