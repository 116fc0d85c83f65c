// route.cu — shard routing for world > 1 (readings R5-R7).
//
//  * k_part_count / k_part_scatter: stable partition of the rank's sorted distinct keys by owner
//    (cyclic: g mod W; block: g div rows_per). Tiles of 2048 keys: per-(tile, owner) counts, then each
//    CTA scans the tiny count matrix itself for its global offsets and ranks its keys stably with
//    ballots. Output: send buffer of local ids (owner-major, ascending g inside an owner), the send
//    position of every distinct key, and the per-owner counts (X0 payload).
//  * k_outidx: per sorted occurrence: send position of its key (the row it gets back, and the slot of
//    its merged gradient in the X3 send buffer); inverse[occurrence] for the pool.
//  * k_merge_runs: the owner receives W runs (one per source rank), each sorted by local id; a stable
//    W-way merge by ranking (ties keep source-rank order) replaces a full radix sort of the received
//    keys: item i of run r goes to (i - start_r) + sum_{r'<r} upper_bound(r', k) + sum_{r'>r}
//    lower_bound(r', k).
#include "../../include/emb.h"
#include "common.cuh"
#include "internal.h"

namespace emb {

namespace {
constexpr int PT_THREADS = 256;
constexpr int PT_ITEMS = 8;
constexpr int PT_TILE = PT_THREADS * PT_ITEMS;  // 2048
}  // namespace

__device__ __forceinline__ uint32_t owner_of(uint32_t g, const KeySpace &ks) {
  return ks.shard == 0 ? g % (uint32_t)ks.world : (uint32_t)(g / ks.rows_per);
}
__device__ __forceinline__ uint32_t local_of(uint32_t g, const KeySpace &ks) {
  return ks.shard == 0 ? g / (uint32_t)ks.world : (uint32_t)(g % ks.rows_per);
}

__global__ void __launch_bounds__(PT_THREADS) k_part_count(const uint32_t *__restrict__ ukey,
                                                           const uint32_t *__restrict__ u_count, KeySpace ks,
                                                           uint32_t *__restrict__ tcnt) {
  __shared__ uint32_t c[EMB_MAX_WORLD];
  const uint32_t U = *u_count;
  const uint32_t t0 = blockIdx.x * PT_TILE;
  if (threadIdx.x < EMB_MAX_WORLD) c[threadIdx.x] = 0;
  __syncthreads();
  if (t0 < U) {
    for (uint32_t i = t0 + threadIdx.x; i < min(U, t0 + PT_TILE); i += PT_THREADS)
      atomicAdd(&c[owner_of(ukey[i], ks)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < (unsigned)ks.world) tcnt[blockIdx.x * EMB_MAX_WORLD + threadIdx.x] = c[threadIdx.x];
}

__global__ void __launch_bounds__(PT_THREADS) k_part_scatter(const uint32_t *__restrict__ ukey,
                                                             const uint32_t *__restrict__ u_count, KeySpace ks,
                                                             const uint32_t *__restrict__ tcnt, int ntiles,
                                                             uint32_t *__restrict__ send_keys,
                                                             uint32_t *__restrict__ sp,
                                                             int64_t *__restrict__ send_counts) {
  __shared__ uint32_t base[EMB_MAX_WORLD];              // global start of (this tile, owner)
  __shared__ uint32_t wcnt[PT_THREADS / 32][EMB_MAX_WORLD];
  __shared__ uint32_t s_before[EMB_MAX_WORLD], s_total[EMB_MAX_WORLD];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int W = ks.world;
  const uint32_t U = *u_count;
  const int tile = blockIdx.x;
  // per owner: totals over all tiles and the part before this tile; warp d sums column d of the
  // (tile, owner) count matrix with coalesced loads and a warp reduction (not one thread per owner
  // walking every tile: that serial loop was most of this kernel's time)
  for (int d = w; d < W; d += PT_THREADS / 32) {
    uint32_t tot = 0, bef = 0;
    for (int t = lane; t < ntiles; t += 32) {
      const uint32_t v = tcnt[t * EMB_MAX_WORLD + d];
      tot += v;
      bef += t < tile ? v : 0u;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
      bef += __shfl_xor_sync(0xffffffffu, bef, o);
    }
    if (lane == 0) {
      s_total[d] = tot;
      s_before[d] = bef;
    }
  }
  __syncthreads();
  if (tid < W) {
    uint32_t before_owner = 0;
    for (int d = 0; d < tid; ++d) before_owner += s_total[d];
    base[tid] = before_owner + s_before[tid];
    if (tile == 0) send_counts[tid] = s_total[tid];
  }
  const uint32_t t0 = tile * PT_TILE;
  // per-warp counts over the warp's contiguous 256 keys
  const uint32_t w0 = t0 + w * 32 * PT_ITEMS;
  if (lane < EMB_MAX_WORLD) wcnt[w][lane] = 0;
  __syncwarp();
  for (int r = 0; r < PT_ITEMS; ++r) {
    const uint32_t i = w0 + r * 32 + lane;
    const bool v = i < U;
    const uint32_t o = v ? owner_of(ukey[i], ks) : 0;
    const uint32_t peers = __match_any_sync(0xffffffffu, v ? o : 0x100u + lane);
    if (v && lane == __ffs(peers) - 1) wcnt[w][o] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (tid < W) {  // exclusive prefix over warps, per owner, on top of the tile base
    uint32_t run = base[tid];
    for (int q = 0; q < PT_THREADS / 32; ++q) {
      const uint32_t c = wcnt[q][tid];
      wcnt[q][tid] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int r = 0; r < PT_ITEMS; ++r) {
    const uint32_t i = w0 + r * 32 + lane;
    const bool v = i < U;
    const uint32_t g = v ? ukey[i] : 0;
    const uint32_t o = v ? owner_of(g, ks) : 0;
    const uint32_t peers = __match_any_sync(0xffffffffu, v ? o : 0x100u + lane);
    const int leader = v ? __ffs(peers) - 1 : lane;
    uint32_t b = 0;
    if (v && lane == leader) {
      b = wcnt[w][o];
      wcnt[w][o] = b + __popc(peers);
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    if (v) {
      const uint32_t dst = b + __popc(peers & lanemask_lt());
      send_keys[dst] = local_of(g, ks);
      sp[i] = dst;
    }
    __syncwarp();
  }
}

cudaError_t launch_partition(const uint32_t *ukey, const uint32_t *u_count, int64_t cap, const KeySpace &ks,
                             uint32_t *tcnt, uint32_t *send_keys, uint32_t *sp, int64_t *send_counts,
                             cudaStream_t st) {
  const int ntiles = (int)((cap + PT_TILE - 1) / PT_TILE);
  if (ntiles <= 0) return cudaSuccess;
  k_part_count<<<ntiles, PT_THREADS, 0, st>>>(ukey, u_count, ks, tcnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_part_scatter<<<ntiles, PT_THREADS, 0, st>>>(ukey, u_count, ks, tcnt, ntiles, send_keys, sp, send_counts);
  return cudaGetLastError();
}

// per sorted occurrence p: outidx[p] = send position of its distinct key; inverse[occurrence] = same
__global__ void k_outidx(const uint32_t *__restrict__ skey, const uint32_t *__restrict__ spay,
                         const uint32_t *__restrict__ useg, const uint32_t *__restrict__ sp, int64_t n,
                         uint32_t *__restrict__ outidx, uint32_t *__restrict__ inv) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const bool v = skey[p] != EMB_SENTINEL;
  const uint32_t o = v ? sp[useg[p]] : EMB_SENTINEL;
  outidx[p] = o;
  inv[spay[p]] = o;
}
cudaError_t launch_outidx(const uint32_t *skey, const uint32_t *spay, const uint32_t *useg, const uint32_t *sp,
                          int64_t n, uint32_t *outidx, uint32_t *inv, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_outidx<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(skey, spay, useg, sp, n, outidx, inv);
  return cudaGetLastError();
}

// owner side: stable W-way merge of the received runs (counts in recv_counts[0..W))
__global__ void k_merge_runs(const uint32_t *__restrict__ rkeys, const int64_t *__restrict__ recv_counts, int W,
                             int64_t cap, uint32_t *__restrict__ okey, uint32_t *__restrict__ opay,
                             uint32_t *err, uint32_t *fin, uint32_t *err_host) {
  __shared__ int64_t start[EMB_MAX_WORLD + 1];
  if (threadIdx.x == 0) {
    start[0] = 0;
    for (int r = 0; r < W; ++r) start[r + 1] = start[r] + recv_counts[r];
  }
  __syncthreads();
  const int64_t n = start[W];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n && i < cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = 0;
    while (r + 1 < W && i >= start[r + 1]) ++r;
    const uint32_t k = rkeys[i];
    int64_t pos = i - start[r];
    for (int q = 0; q < W; ++q) {
      if (q == r) continue;
      int64_t lo = start[q], len = start[q + 1] - start[q];
      while (len > 0) {  // count of run q's keys <= k (q < r) or < k (q > r)
        const int64_t half = len >> 1;
        const uint32_t x = rkeys[lo + half];
        const bool before = (q < r) ? (x <= k) : (x < k);
        lo = before ? lo + half + 1 : lo;
        len = before ? len - half - 1 : half;
      }
      pos += lo - start[q];
    }
    if (pos < 0 || pos >= n) {
      atomicOr(err, EMB_DEVERR_INTERNAL);
      continue;
    }
    okey[pos] = k;
    opay[pos] = (uint32_t)i;
  }
  if (fin) {  // the later of this merge and the pool publishes the error word (PoolArgs::fin)
    __syncthreads();
    if (threadIdx.x == 0) finish_publish(fin + 1, fin + 2, 2, err, err_host);
  }
}
cudaError_t launch_merge_runs(const uint32_t *rkeys, const int64_t *recv_counts, int W, int64_t n, uint32_t *okey,
                              uint32_t *opay, uint32_t *err, cudaStream_t st, uint32_t *fin, uint32_t *err_host) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  k_merge_runs<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(rkeys, recv_counts, W, n, okey, opay, err,
                                                                          fin, err_host);
  return cudaGetLastError();
}

}  // namespace emb
