// route.cu — shard routing for world > 1 (readings R5-R7).
//
//  * k_part_count / k_part_scatter: stable partition of the rank's sorted distinct keys by owner
//    (cyclic: g mod W; block: g div rows_per). Tiles of 2048 keys: per-(tile, owner) counts, then each
//    CTA scans the tiny count matrix itself for its global offsets and ranks its keys stably with
//    ballots. Output: send buffer of local ids (owner-major, ascending g inside an owner), the send
//    position of every distinct key, and the per-owner counts (X0 payload).
//  * k_outidx: per sorted occurrence: send position of its key (the row it gets back, and the slot of
//    its merged gradient in the X3 send buffer); inverse[occurrence] for the pool.
//  * k_merge_pass: the owner receives W runs (one per source rank), each sorted by local id; a stable
//    merge tree (ceil(log2 W) passes of pairwise merge-path merges, ties keep the lower source rank)
//    replaces a full radix sort of the received keys. Per pass, a CTA owns TILE outputs of one merged
//    run: one merge-path search for its two diagonals, the A / B windows staged in shared memory, then
//    per-thread searches and sequential merges there. (v1, k_merge_runs: every item ranked by binary
//    searches into the W-1 other runs — 60 / 106 us at W = 2 / 4, growing with W.)
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
  // at least one tile: with no ids this step the per-owner send counts must still be written (zeros),
  // or the exchange would announce the previous step's counts
  const int ntiles = cap > 0 ? (int)((cap + PT_TILE - 1) / PT_TILE) : 1;
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

// ---- merge tree (v2)
namespace {
constexpr int MP_THREADS = 256;
constexpr int MP_ITEMS = 8;
constexpr int MP_TILE = MP_THREADS * MP_ITEMS;  // outputs per CTA
}  // namespace

// number of A items among the first d outputs of the stable merge of A (first) and B
__device__ __forceinline__ int64_t merge_path(const uint32_t *A, int64_t m, const uint32_t *B, int64_t n, int64_t d) {
  int64_t lo = d > n ? d - n : 0, hi = d < m ? d : m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// pass r: output run j = stable merge of sources [2j*w, (2j+1)*w) (A) and [(2j+1)*w, (2j+2)*w) (B),
// w = 2^r. ip == nullptr: payload = receive position (first pass).
__global__ void __launch_bounds__(MP_THREADS) k_merge_pass(const uint32_t *__restrict__ ik,
                                                           const uint32_t *__restrict__ ip,
                                                           const int64_t *__restrict__ recv_counts, int W, int w,
                                                           uint32_t *__restrict__ ok, uint32_t *__restrict__ op,
                                                           uint32_t *err, uint32_t *fin, uint32_t *err_host) {
  __shared__ int64_t P[EMB_MAX_WORLD + 1];
  __shared__ uint32_t sk[MP_TILE], sp[MP_TILE];
  __shared__ int64_t s_a0, s_am, s_b0, s_bn, s_i0, s_i1, s_d0, s_d1, s_out;
  const int tid = threadIdx.x;
  if (tid == 0) {
    P[0] = 0;
    for (int r = 0; r < W; ++r) P[r + 1] = P[r] + recv_counts[r];
  }
  __syncthreads();
  const int nruns = (W + 2 * w - 1) / (2 * w);
  // block -> (output run j, tile within the run)
  int j = -1;
  int64_t tile = blockIdx.x;
  for (int q = 0; q < nruns; ++q) {
    const int64_t len = P[min(W, (2 * q + 2) * w)] - P[min(W, 2 * q * w)];
    const int64_t nt = (len + MP_TILE - 1) / MP_TILE;
    if (tile < nt) {
      j = q;
      break;
    }
    tile -= nt;
  }
  if (j >= 0) {
    if (tid == 0) {
      const int64_t a0 = P[min(W, 2 * j * w)], b0 = P[min(W, (2 * j + 1) * w)], e = P[min(W, (2 * j + 2) * w)];
      const int64_t m = b0 - a0, n = e - b0;
      const int64_t d0 = tile * MP_TILE, d1 = min(d0 + MP_TILE, m + n);
      s_a0 = a0;
      s_am = m;
      s_b0 = b0;
      s_bn = n;
      s_d0 = d0;
      s_d1 = d1;
      s_i0 = merge_path(ik + a0, m, ik + b0, n, d0);
      s_i1 = merge_path(ik + a0, m, ik + b0, n, d1);
      s_out = a0 + d0;  // merged run j starts where its A run started
    }
    __syncthreads();
    const int64_t a0 = s_a0, b0 = s_b0, i0 = s_i0, i1 = s_i1, d0 = s_d0, d1 = s_d1;
    const int na = (int)(i1 - i0), nb = (int)((d1 - i1) - (d0 - i0));
    const int64_t bj0 = b0 + (d0 - i0);
    for (int q = tid; q < na; q += MP_THREADS) {
      sk[q] = ik[a0 + i0 + q];
      sp[q] = ip ? ip[a0 + i0 + q] : (uint32_t)(a0 + i0 + q);
    }
    for (int q = tid; q < nb; q += MP_THREADS) {
      sk[na + q] = ik[bj0 + q];
      sp[na + q] = ip ? ip[bj0 + q] : (uint32_t)(bj0 + q);
    }
    __syncthreads();
    // per thread: MP_ITEMS consecutive outputs of the tile
    const int dd = tid * MP_ITEMS;
    const int tot = na + nb;
    if (dd < tot) {
      int lo = dd > nb ? dd - nb : 0, hi = dd < na ? dd : na;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sk[mid] <= sk[na + dd - 1 - mid]) lo = mid + 1;
        else hi = mid;
      }
      int ia = lo, ib = dd - lo;
      const int64_t o = s_out + dd;
      for (int q = 0; q < MP_ITEMS && dd + q < tot; ++q) {
        const bool takeA = ib >= nb || (ia < na && sk[ia] <= sk[na + ib]);
        const int src = takeA ? ia : na + ib;
        ok[o + q] = sk[src];
        op[o + q] = sp[src];
        if (takeA) ++ia;
        else ++ib;
      }
    }
  }
  if (fin) {  // last pass: the later of this merge and the pool publishes the error word
    __syncthreads();
    if (tid == 0) finish_publish(fin + 1, fin + 2, 2, err, err_host);
  }
}

cudaError_t launch_merge_tree(const uint32_t *rkeys, const int64_t *recv_counts, int W, int64_t cap, uint32_t *ok0,
                              uint32_t *op0, uint32_t *ok1, uint32_t *op1, uint32_t *err, cudaStream_t st,
                              uint32_t *fin, uint32_t *err_host) {
  int passes = 0;
  while ((1 << passes) < W) ++passes;
  const int64_t blocks = (cap + MP_TILE - 1) / MP_TILE + W;  // >= sum over runs of their tiles
  const uint32_t *ik = rkeys, *ip = nullptr;
  for (int r = 0; r < passes; ++r) {
    const bool to0 = ((passes - 1 - r) & 1) == 0;  // the last pass lands in (ok0, op0)
    uint32_t *ok = to0 ? ok0 : ok1, *op = to0 ? op0 : op1;
    k_merge_pass<<<(unsigned)blocks, MP_THREADS, 0, st>>>(ik, ip, recv_counts, W, 1 << r, ok, op, err,
                                                          r == passes - 1 ? fin : nullptr, err_host);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ik = ok;
    ip = op;
  }
  return cudaSuccess;
}

// owner side (v1, kept for the NCCL exchange path): stable W-way merge by ranking
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
