// pool.cu — K5 gather + pool (readings R1-R3):
//   Y[b][s][:] = sum_{j in bag(s,b)} row(j)[:]   (mean: / |bag|; empty bag -> 0)
// accumulated in fp64 in occurrence order and rounded once to fp32 (R11), so the result does not
// depend on how the work is split (a one-element bag is copied exactly).
//
// Mapping (v3; the v1/v2 ncu captures showed 131 / 80 warp-instructions per bag and a latency-bound
// pipeline): a warp owns a row (32 lanes x CPL consecutive columns: D=64 -> 8-byte float2 per lane,
// one 256-B coalesced row per instruction) and a tile of 32 consecutive bags (slot-major CSR: one
// slot's consecutive samples), lane l holding bag l's CSR bounds and output row b*S+s (32-bit math).
//  * tiles of single-id bags (the Criteo case): the 32 keys are fetched in one coalesced load and
//    each lane then issues RCH independent row loads (ld.global.nc, L1 no-allocate; RCH = 32 at
//    D <= 64, i.e. the whole tile in flight) and RCH .cs streaming stores per batch;
//  * other tiles: the warp walks the flattened occurrence range of its 32 bags in batches of RCH
//    rows (keys of the next batch prefetched), accumulating in fp64 and flushing each bag at its end.
// One tile per warp (grid-stride loop kept for very large batches). Row loads are unconditional (a
// missing row reads row 0 and is zeroed before use): predicated loads each hold one of the 7
// predicate registers and ptxas then issued them in groups of ~4 instead of RCH at once.
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "vec.cuh"

namespace emb {

namespace {
constexpr int POOL_THREADS = 256;
}  // namespace

// row of occurrence j. Direct mode (per-table sort path): g = base[t] + id validated here (R4) and the
// occurrence's dY row index recorded for the backward; key mode (general sort path): g from the key
// kernel. A row this rank owns is read from the table shard at local(g); at W > 1 a row owned by
// another rank from the rows its owner pushed, at inv[j] (returned with REMOTE_BIT set).
constexpr uint32_t REMOTE_BIT = 0x80000000u;
template <bool REMOTE>
__device__ __forceinline__ uint32_t pool_row_of(const PoolArgs &a, int64_t j, uint32_t slot, uint32_t orow) {
  uint32_t g = EMB_SENTINEL;
  if (a.ids) {
    const int t = a.slot_table[slot];
    const int64_t id = a.ids[j];
    if (id >= 0 && id < a.rows[t]) g = (uint32_t)(a.base[t] + (uint64_t)id);
    else atomicOr(a.err, EMB_DEVERR_RANGE);
    a.drow[j] = orow;
  } else {
    g = a.key[j];
  }
  if (g == EMB_SENTINEL) return EMB_SENTINEL;
  if (REMOTE && owner_of_g(g, a.ks) != (uint32_t)a.ks.rank) {
    const uint32_t r = a.row_idx[j];
    if ((int64_t)r >= a.nrows_remote) {
      atomicOr(a.err, EMB_DEVERR_INTERNAL);
      return EMB_SENTINEL;
    }
    return REMOTE_BIT | r;
  }
  const uint32_t row = REMOTE ? local_of_g(g, a.ks) : g;
  if ((int64_t)row >= a.nrows_src) {
    atomicOr(a.err, EMB_DEVERR_INTERNAL);
    return EMB_SENTINEL;
  }
  return row;
}
// address of a row returned by pool_row_of (EMB_SENTINEL / inactive lanes read row 0 of the shard:
// unconditional loads, zeroed before use)
template <bool REMOTE>
__device__ __forceinline__ const float *pool_row_ptr(const PoolArgs &a, uint32_t ri, bool ok, int D, int col) {
  if (!ok) return a.rows_src;
  if (REMOTE && (ri & REMOTE_BIT)) return a.rows_remote + (size_t)(ri & ~REMOTE_BIT) * D + col;
  return a.rows_src + (size_t)ri * D + col;
}

// general tile: flattened walk over the occurrences [lo, hi) of the tile's bags, fp64 in order
template <int CPL, bool REMOTE>
__device__ __noinline__ void pool_tile_general(const PoolArgs &a, int64_t lo, int64_t hi, int64_t my_end,
                                               uint32_t my_orow, uint32_t my_slot, int nbt) {
  constexpr int RCH = 32 / CPL;
  const int lane = threadIdx.x & 31;
  const int D = a.dim;
  const int col = lane * CPL;
  const bool active = col < D;
  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  int cb = 0;
  int64_t cst = lo;
  int64_t cend = __shfl_sync(0xffffffffu, my_end, 0);
  auto flush = [&]() {
    const uint32_t orow = __shfl_sync(0xffffffffu, my_orow, cb);
    const int64_t len = cend - cst;
    if (active) {
      VecF<CPL> o;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double x = (a.mean && len > 1) ? __ddiv_rn(acc[c], (double)len) : acc[c];
        o.v[c] = (float)x;
      }
      o.store_cs(a.out + (size_t)orow * D + col);
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
    ++cb;
    cst = cend;
    cend = __shfl_sync(0xffffffffu, my_end, cb < 32 ? cb : 31);
  };
  // row of occurrence j (lane-parallel): its bag = the first bag whose end is > j
  auto occ_row = [&](int64_t j) -> uint32_t {
    int l = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1) {
      const int64_t e = __shfl_sync(0xffffffffu, my_end, l + step - 1);
      if (l + step - 1 < nbt && e <= j) l += step;
    }
    const uint32_t sl = __shfl_sync(0xffffffffu, my_slot, l < 32 ? l : 31);
    const uint32_t orw = __shfl_sync(0xffffffffu, my_orow, l < 32 ? l : 31);
    const bool ok = (lane < RCH) && j < hi;
    return ok ? pool_row_of<REMOTE>(a, j, sl, orw) : EMB_SENTINEL;
  };
  // close leading empty bags
  while (cb < nbt && cend <= lo) flush();
  uint32_t nrow = occ_row(lo + lane);
  for (int64_t j0 = lo; j0 < hi; j0 += RCH) {
    const uint32_t row = nrow;
    const int64_t jn = j0 + RCH;
    nrow = occ_row(jn + lane);  // prefetch
    VecF<CPL> v[RCH];
#pragma unroll
    for (int r = 0; r < RCH; ++r) {  // unconditional loads (see the single-id path in k_pool)
      const uint32_t ri = __shfl_sync(0xffffffffu, row, r);
      const bool ok = ri != EMB_SENTINEL && active;
      v[r].load_nc(pool_row_ptr<REMOTE>(a, ri, ok, D, col));
    }
#pragma unroll
    for (int r = 0; r < RCH; ++r) {
      const int64_t j = j0 + r;
      if (j >= hi) break;
      if (__shfl_sync(0xffffffffu, row, r) == EMB_SENTINEL) v[r].zero();
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] += (double)v[r].v[c];
      if (j + 1 == cend) {
        flush();
        while (cb < nbt && cend == cst) flush();  // empty bags right after
      }
    }
  }
  while (cb < nbt) flush();
}

// general tile, lane-group form (D = 16, 32, 64, 128, 256): a group of LPR = D / GC lanes holds one
// row (GC floats each: 128-bit loads) and owns whole bags, G = 32 / LPR of the tile's bags at a time;
// per bag it walks the ids in chunks of RCH (one id per lane, RCH row loads in flight per lane) and
// accumulates in fp64 in occurrence order (R11, same order as pool_tile_general). No per-occurrence
// bag search: the bag's slot, output row and bounds come from the tile header through shared memory.
template <int LPR, int GC, bool REMOTE>
__device__ __noinline__ void pool_tile_groups(const PoolArgs &a, int64_t my_off, int64_t my_end, uint32_t my_orow,
                                              uint32_t my_slot, int nbt) {
  constexpr int G = 32 / LPR;
  constexpr int RCH = LPR < 16 ? LPR : 16;  // ids per chunk (= rows in flight per lane)
  constexpr int D = LPR * GC;
  const int lane = threadIdx.x & 31, grp = lane / LPR, gl = lane % LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << (LPR & 31)) - 1u) << (grp * LPR));
  // (the tile header -- lane l holds bag l's bounds -- is read with warp-uniform shuffles: shared
  // memory for it kept a pool block from sharing an SM with a sort CTA)
  for (int it = 0; it * G < nbt; ++it) {
    const int bi = it * G + grp;
    const int src = bi < 32 ? bi : 31;
    const int64_t off = __shfl_sync(0xffffffffu, my_off, src), end = __shfl_sync(0xffffffffu, my_end, src);
    const uint32_t orow = __shfl_sync(0xffffffffu, my_orow, src), slot = __shfl_sync(0xffffffffu, my_slot, src);
    if (bi >= nbt) continue;
    double acc[GC];
#pragma unroll
    for (int c = 0; c < GC; ++c) acc[c] = 0.0;
    for (int64_t c0 = off; c0 < end; c0 += RCH) {
      const int64_t j = c0 + gl;
      const uint32_t row = (gl < RCH && j < end) ? pool_row_of<REMOTE>(a, j, slot, orow) : EMB_SENTINEL;
      VecF<GC> v[RCH];
#pragma unroll
      for (int r = 0; r < RCH; ++r) {  // unconditional loads (see k_pool), zeroed below
        const uint32_t ri = __shfl_sync(gmask, row, r, LPR);
        v[r].load_nc(pool_row_ptr<REMOTE>(a, ri, ri != EMB_SENTINEL, D, gl * GC));
      }
#pragma unroll
      for (int r = 0; r < RCH; ++r) {
        const uint32_t ri = __shfl_sync(gmask, row, r, LPR);
        if (ri == EMB_SENTINEL) continue;
#pragma unroll
        for (int c = 0; c < GC; ++c) acc[c] += (double)v[r].v[c];
      }
    }
    const int64_t len = end - off;
    VecF<GC> o;
#pragma unroll
    for (int c = 0; c < GC; ++c) o.v[c] = (float)((a.mean && len > 1) ? __ddiv_rn(acc[c], (double)len) : acc[c]);
    o.store_cs(a.out + (size_t)orow * D + gl * GC);
  }
}

template <int CPL, int RCH, int MINB, bool REMOTE, int BPT>
__global__ void __launch_bounds__(POOL_THREADS, MINB) k_pool(const __grid_constant__ PoolArgs a) {
  // RCH rows per batch of the single-id path (RCH * CPL floats in flight per lane)
  const int lane = threadIdx.x & 31;
  const int D = a.dim;
  const int col = lane * CPL;
  const bool active = col < D;
  const uint32_t B = (uint32_t)a.batch, S = (uint32_t)a.num_slots;
  const int64_t nb = (int64_t)a.num_slots * a.batch;
  constexpr int bpt = BPT;  // bags per warp tile
  const int64_t ntiles = (nb + bpt - 1) / bpt;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tile = gw; tile < ntiles; tile += nwarps) {
    const int64_t b0 = tile * bpt;
    const int nbt = (int)((nb - b0) < bpt ? (nb - b0) : bpt);
    const bool inb = lane < nbt;
    const uint32_t bag = (uint32_t)b0 + lane;
    int64_t off = 0, offn = 0;
    if (inb) {
      off = a.offsets[bag];
      offn = a.offsets[bag + 1];
    }
    if (a.ids && inb) {  // direct mode validates the CSR (the key kernel does it in key mode)
      bool bad = off < 0 || offn < off || offn > a.nnz;
      if (bag == 0 && off != 0) bad = true;
      if ((int64_t)bag == nb - 1 && offn != a.nnz) bad = true;
      if (bad) atomicOr(a.err, EMB_DEVERR_INVALID);
    }
    off = off < 0 ? 0 : (off > a.nnz ? a.nnz : off);
    offn = offn < off ? off : (offn > a.nnz ? a.nnz : offn);
    const int len = (int)(offn - off);
    const uint32_t s = bag / B;
    const uint32_t orow = (bag - s * B) * S + s;
    if (a.ids && a.blen && inb) a.blen[orow] = len;
    if (__any_sync(0xffffffffu, len > 1)) {
      const int D_ = a.dim;
      if (D_ == 16 || D_ == 32 || D_ == 64 || D_ == 128 || D_ == 256) {  // lane groups own whole bags
        if (D_ == 16) pool_tile_groups<4, 4, REMOTE>(a, off, offn, orow, s, nbt);
        else if (D_ == 32) pool_tile_groups<8, 4, REMOTE>(a, off, offn, orow, s, nbt);
        else if (D_ == 64) pool_tile_groups<16, 4, REMOTE>(a, off, offn, orow, s, nbt);
        else if (D_ == 128) pool_tile_groups<32, 4, REMOTE>(a, off, offn, orow, s, nbt);
        else pool_tile_groups<32, 8, REMOTE>(a, off, offn, orow, s, nbt);
        continue;
      }
      const int64_t lo = __shfl_sync(0xffffffffu, off, 0);
      const int64_t hi = __shfl_sync(0xffffffffu, offn, nbt - 1);
      pool_tile_general<CPL, REMOTE>(a, lo, hi, offn, orow, s, nbt);
      continue;
    }
    // single-id bags: copy the row (exact)
    const uint32_t row = (len == 1) ? pool_row_of<REMOTE>(a, off, s, orow) : EMB_SENTINEL;
    if (CPL == 2 && D == 64) {
      // D = 64: a half-warp per row (16 lanes x float4: 128-bit loads and stores), the two halves on
      // alternate bags -- half the load / store / shuffle instructions of the 32-lane float2 rows for
      // the same bytes in flight per warp (the north_star's 128-bit row loads)
      const int half = lane >> 4, hl = lane & 15;
#pragma unroll
      for (int c0 = 0; c0 < 32; c0 += 32) {
        float4 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {  // unconditional loads (see below)
          const uint32_t ri = __shfl_sync(0xffffffffu, row, c0 + 2 * r + half);
          v[r] = ld_nc_f4(reinterpret_cast<const float4 *>(pool_row_ptr<REMOTE>(a, ri, ri != EMB_SENTINEL, 64, hl * 4)));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int b = c0 + 2 * r + half;
          const uint32_t ri = __shfl_sync(0xffffffffu, row, b);
          const uint32_t oi = __shfl_sync(0xffffffffu, orow, b);
          if (ri == EMB_SENTINEL) v[r] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (b < nbt) st_cs_f4(reinterpret_cast<float4 *>(a.out + (size_t)oi * 64 + hl * 4), v[r]);
        }
      }
      continue;
    }
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += RCH) {
      if (c0 >= nbt) break;
      VecF<CPL> v[RCH];
#pragma unroll
      for (int r = 0; r < RCH; ++r) {
        // unconditional loads (a missing row reads row 0 and is zeroed at the store): predicated or
        // branched loads need one predicate register each, and with only 7 of them ptxas issued the
        // rows in groups of ~4 between stores instead of RCH in flight
        const uint32_t ri = __shfl_sync(0xffffffffu, row, c0 + r);
        const bool ok = ri != EMB_SENTINEL && active;
        v[r].load_nc(pool_row_ptr<REMOTE>(a, ri, ok, D, col));
      }
#pragma unroll
      for (int r = 0; r < RCH; ++r) {
        const uint32_t ri = __shfl_sync(0xffffffffu, row, c0 + r);
        const uint32_t oi = __shfl_sync(0xffffffffu, orow, c0 + r);
        if (ri == EMB_SENTINEL) v[r].zero();
        if (c0 + r < nbt && active) v[r].store_cs(a.out + (size_t)oi * D + col);
      }
    }
  }
  if (a.fin) {
    __syncthreads();
    if (threadIdx.x == 0) finish_publish(a.fin, a.fin + 2, a.fin_kernels, a.err, a.err_host);
  }
}

template <int CPL, int RCH, int MINB>
static cudaError_t launch_pool_t(const PoolArgs &a, int64_t ntiles, cudaStream_t st) {
  // one tile per warp (not persistent), so the concurrent side-stream sort CTAs get SMs as soon as
  // they are ready and the pool fills the rest
  const int64_t blocks = (ntiles * 32 + POOL_THREADS - 1) / POOL_THREADS;
  const bool remote = a.ks.world > 1;
  if (a.bags_per_tile == 32) {
    if (remote) k_pool<CPL, RCH, MINB, true, 32><<<(unsigned)blocks, POOL_THREADS, 0, st>>>(a);
    else k_pool<CPL, RCH, MINB, false, 32><<<(unsigned)blocks, POOL_THREADS, 0, st>>>(a);
  } else {
    if (remote) k_pool<CPL, RCH, MINB, true, 8><<<(unsigned)blocks, POOL_THREADS, 0, st>>>(a);
    else k_pool<CPL, RCH, MINB, false, 8><<<(unsigned)blocks, POOL_THREADS, 0, st>>>(a);
  }
  return cudaGetLastError();
}

// copy the sticky device error word to the mapped pinned host word (end of every lookup)
__global__ void k_publish_err(const uint32_t *err, uint32_t *err_host) {
  *(volatile uint32_t *)err_host = *(volatile const uint32_t *)err;
}
cudaError_t launch_publish_err(const uint32_t *err, uint32_t *err_host, cudaStream_t st) {
  k_publish_err<<<1, 1, 0, st>>>(err, err_host);
  return cudaGetLastError();
}

cudaError_t launch_pool(const PoolArgs &a0, cudaStream_t st) {
  const int64_t nb = (int64_t)a0.num_slots * a0.batch;
  if (nb == 0) return cudaSuccess;
  PoolArgs a = a0;
  // bags per warp tile: 32 (one per lane) fills the GPU once there are >= ~150K bags; small batches
  // (C1: 4,096 bags, 128 tiles) get 8 per tile so 4x more warps walk their occurrences in parallel
  a.bags_per_tile = nb >= 148 * 8 * 32 * 4 ? 32 : 8;
  const int64_t ntiles = (nb + a.bags_per_tile - 1) / a.bags_per_tile;
  // D <= 64: all 32 rows of a tile in flight per lane (registers allow it because the loads are
  // unconditional): C2 step 136.6 -> 133.5 us against 16 rows (round 1)
  if (a.dim <= 64) return launch_pool_t<2, 32, 3>(a, ntiles, st);
  if (a.dim <= 128) return launch_pool_t<4, 8, 3>(a, ntiles, st);
  return launch_pool_t<8, 4, 3>(a, ntiles, st);
}

}  // namespace emb
