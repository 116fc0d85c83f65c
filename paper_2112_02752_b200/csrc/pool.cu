// pool.cu — K5 gather + pool (readings R1-R3):
//   Y[b][s][:] = sum_{j in bag(s,b)} row(j)[:]   (mean: / |bag|; empty bag -> 0)
// accumulated in fp64 in occurrence order and rounded once to fp32 (R11), so the result is
// independent of how the work is split.
//
// Mapping: one warp per 32 consecutive bags (slot-major CSR, so a warp's bags are one slot's
// consecutive samples). The warp walks the contiguous occurrence range of its bags in pieces of 32
// rows. For each piece every lane issues ONE 1-D TMA bulk copy (cp.async.bulk, SASS UBLKCP) of a
// whole row (D*4 bytes) from HBM into the warp's shared-memory stage; completion is counted on an
// mbarrier (expect_tx). Two stages per warp: piece k+1's rows are in flight while piece k is summed.
// Lanes then own CPL consecutive columns each (D=64: 32 lanes x 2 columns, 256-B coalesced output
// stores with .cs streaming hint). The row source is the table itself at W=1 (row = routing key) or
// the rows received from the owners at W>1 (row = inverse[j]).
#include "common.cuh"
#include "internal.h"

namespace emb {

namespace {
constexpr int POOL_WARPS = 4;   // max warps per CTA (D <= 64; 2 for D <= 128, 1 above)
constexpr int PIECE = 32;       // rows per stage (one per lane)
constexpr int STAGES = 2;
}  // namespace

template <int CPL>
__global__ void __launch_bounds__(POOL_WARPS * 32) k_pool(PoolArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[POOL_WARPS][STAGES];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int D = a.dim;
  const uint32_t RB = (uint32_t)D * 4u;
  float *stage_buf = reinterpret_cast<float *>(smem) + (size_t)wib * STAGES * PIECE * D;
  const int64_t nb = (int64_t)a.num_slots * a.batch;
  const int64_t b0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * 32;

  if (blockIdx.x == 0 && threadIdx.x == 0 && a.err_host) {
    // publish the sticky error word of this step's key kernel (ran before us on the stream)
    *(volatile uint32_t *)a.err_host = *(volatile const uint32_t *)a.err;
  }
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[wib][s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (b0 >= nb) return;

  const int64_t bag = b0 + lane;
  const bool inb = bag < nb;
  const int nbags = (int)((nb - b0) < 32 ? (nb - b0) : 32);
  int64_t en = inb ? a.offsets[bag + 1] : 0;
  int64_t lo = a.offsets[b0];
  int64_t hi = __shfl_sync(0xffffffffu, en, nbags - 1);
  // clamp (offsets were validated by the key kernel; stay memory-safe if they are broken)
  lo = lo < 0 ? 0 : (lo > a.nnz ? a.nnz : lo);
  hi = hi < lo ? lo : (hi > a.nnz ? a.nnz : hi);
  const int64_t npieces = (hi - lo + PIECE - 1) / PIECE;

  // issue piece p into stage p % STAGES; returns the valid-row mask of the piece
  auto issue = [&](int64_t p) -> uint32_t {
    const int s = (int)(p % STAGES);
    const int64_t j = lo + p * PIECE + lane;
    uint32_t row = EMB_SENTINEL;
    if (j < hi) {
      const uint32_t k = a.key[j];
      if (k != EMB_SENTINEL) row = a.row_idx ? a.row_idx[j] : k;
      if (row != EMB_SENTINEL && (int64_t)row >= a.nrows_src) {
        atomicOr(a.err, EMB_DEVERR_INTERNAL);
        row = EMB_SENTINEL;
      }
    }
    const uint32_t vmask = __ballot_sync(0xffffffffu, row != EMB_SENTINEL);
    if (lane == 0) mbar_arrive_expect_tx(&bars[wib][s], (uint32_t)__popc(vmask) * RB);
    __syncwarp();
    if (row != EMB_SENTINEL)
      bulk_g2s(stage_buf + ((size_t)s * PIECE + lane) * D, a.rows_src + (size_t)row * D, RB, &bars[wib][s]);
    return vmask;
  };

  uint32_t vm[STAGES];
  for (int64_t p = 0; p < STAGES && p < npieces; ++p) vm[p] = issue(p);

  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  const int col = lane * CPL;
  const bool active = col < D;
  int cb = 0;  // current bag (relative)
  int64_t cend = __shfl_sync(0xffffffffu, en, 0);
  int64_t cst = lo;

  auto flush = [&](int rb, int64_t len) {
    const int64_t gbag = b0 + rb;
    const int s = (int)(gbag / a.batch), b = (int)(gbag % a.batch);
    float *dst = a.out + ((size_t)b * a.num_slots + s) * D + col;
    if (active) {
      if (a.mean && len > 0) {  // R1: divide the fp64 sum by |bag| (IEEE division, as the oracle)
        const double dl = (double)len;
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = __ddiv_rn(acc[c], dl);
      }
      if (CPL == 2) {
        st_cs_f2(reinterpret_cast<float2 *>(dst), make_float2((float)acc[0], (float)acc[1]));
      } else {
#pragma unroll
        for (int c = 0; c < CPL; c += 4)
          st_cs_f4(reinterpret_cast<float4 *>(dst + c),
                   make_float4((float)acc[c], (float)acc[c + 1], (float)acc[c + 2], (float)acc[c + 3]));
      }
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  };

  for (int64_t p = 0; p < npieces; ++p) {
    const int s = (int)(p % STAGES);
    mbar_wait(&bars[wib][s], (uint32_t)((p / STAGES) & 1));
    const uint32_t vmask = vm[s];
    const int64_t pj0 = lo + p * PIECE;
    const int cnt = (int)((hi - pj0) < PIECE ? (hi - pj0) : PIECE);
    const float *buf = stage_buf + (size_t)s * PIECE * D;
    for (int i = 0; i < cnt; ++i) {
      const int64_t j = pj0 + i;
      while (cb < nbags && j >= cend) {  // close finished (and empty) bags
        flush(cb, cend - cst);
        ++cb;
        cst = cend;
        cend = __shfl_sync(0xffffffffu, en, cb < 32 ? cb : 31);
      }
      if ((vmask >> i) & 1u) {
        if (active) {
          const float *r = buf + (size_t)i * D + col;
          if (CPL == 2) {
            const float2 v = *reinterpret_cast<const float2 *>(r);
            acc[0] += (double)v.x;
            acc[1] += (double)v.y;
          } else {
#pragma unroll
            for (int c = 0; c < CPL; c += 4) {
              const float4 v = *reinterpret_cast<const float4 *>(r + c);
              acc[c] += (double)v.x;
              acc[c + 1] += (double)v.y;
              acc[c + 2] += (double)v.z;
              acc[c + 3] += (double)v.w;
            }
          }
        }
      }
    }
    __syncwarp();
    if (p + STAGES < npieces) {
      fence_proxy_async_smem();  // generic-proxy reads of this stage before the async-proxy refill
      vm[s] = issue(p + STAGES);
    }
  }
  while (cb < nbags) {
    flush(cb, cend - cst);
    ++cb;
    cst = cend;
    cend = __shfl_sync(0xffffffffu, en, cb < 32 ? cb : 31);
  }
}

static int pool_warps(int D) { return D <= 64 ? 4 : (D <= 128 ? 2 : 1); }

template <int CPL>
static cudaError_t launch_pool_t(const PoolArgs &a, int64_t blocks, int wpc, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_pool<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_pool<CPL><<<(unsigned)blocks, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pool(const PoolArgs &a, cudaStream_t st) {
  const int64_t nb = (int64_t)a.num_slots * a.batch;
  if (nb == 0) return cudaSuccess;
  const int wpc = pool_warps(a.dim);
  const int64_t warps = (nb + 31) / 32;
  const int64_t blocks = (warps + wpc - 1) / wpc;
  const size_t smem = (size_t)wpc * STAGES * PIECE * a.dim * sizeof(float);
  if (a.dim <= 64) return launch_pool_t<2>(a, blocks, wpc, smem, st);
  if (a.dim <= 128) return launch_pool_t<4>(a, blocks, wpc, smem, st);
  return launch_pool_t<8>(a, blocks, wpc, smem, st);
}

}  // namespace emb
