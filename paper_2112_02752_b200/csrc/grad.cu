// grad.cu — K6+K7 fused: deterministic segment reduce of duplicate-id gradients + sparse optimizer
// apply (readings R8-R14, R16).
//
// Input is the stably sorted (routing key, payload) array of the step, so every distinct key is a
// contiguous SEGMENT whose contributions appear in occurrence order. Work is split into fixed chunks
// of 32 sorted positions, one warp per chunk (balanced whatever the Zipf skew):
//  1. lane i loads position c*32+i: key, payload -> the contribution row address (dY[b][s][:] via the
//     occurrence's bag, or a received gradient row) and, at every segment head (and at the chunk's
//     first position), the table row w (and Adagrad row a) of that key;
//  2. all those rows (up to 32 + 2*32 per chunk) are fetched by 1-D TMA bulk copies into the warp's
//     shared memory, completion on one mbarrier — deep memory-level parallelism with no registers;
//  3. the warp walks the 32 positions in order, lanes owning CPL columns each, accumulating in fp64
//     (mean: c = dY / |bag|). A segment that starts and ends inside the chunk is complete: apply.
//  4. A segment crossing chunk boundaries leaves one fp64 partial per chunk (slot 2c for the piece
//     that continues from chunk c-1, slot 2c+1 for the piece that starts in c and continues), then
//     takes a ticket on the segment's start chunk; the LAST arriving warp sums the partials in chunk
//     order and applies. The sum order is fixed by the chunk grid, so results are bitwise
//     reproducible run to run (R10) although warps finish in any order.
// Sinks: mode 0 applies SGD (w -= lr*G) or element-wise Adagrad (a += G^2; w -= lr*G/(sqrt(a)+eps))
// in fp64 from the fp32 state with IEEE _rn intrinsics (no FMA contraction), rounding once, as the
// oracle; mode 1 writes the fp32 per-unique-key gradient (requester side of the W>1 exchange).
#include "common.cuh"
#include "internal.h"

namespace emb {

namespace {
constexpr int GW_MAX = 4;  // warps per CTA for D <= 64 (2 for D <= 128, 1 above)
constexpr int CH = 32;     // sorted positions per chunk
}  // namespace

static __device__ int64_t seg_first(const uint32_t *skey, int64_t p, uint32_t k) {
  // first position q <= p with skey[q] == k (exponential then binary search; segments are sorted)
  int64_t step = 1, hi = p, lo;
  while (true) {
    const int64_t q = p - step;
    if (q < 0 || ld_cg_u32(skey + q) != k) {
      lo = q;  // skey[lo] != k (or lo = -1)
      break;
    }
    hi = q;
    step <<= 1;
  }
  while (hi - lo > 1) {
    const int64_t m = lo + (hi - lo) / 2;
    if (ld_cg_u32(skey + m) == k) hi = m; else lo = m;
  }
  return hi;
}
static __device__ int64_t seg_last(const uint32_t *skey, int64_t n, int64_t p, uint32_t k) {
  int64_t step = 1, lo = p, hi;
  while (true) {
    const int64_t q = p + step;
    if (q >= n || ld_cg_u32(skey + q) != k) {
      hi = q;
      break;
    }
    lo = q;
    step <<= 1;
  }
  while (hi - lo > 1) {
    const int64_t m = lo + (hi - lo) / 2;
    if (ld_cg_u32(skey + m) == k) lo = m; else hi = m;
  }
  return lo;
}

template <int CPL>
__global__ void __launch_bounds__(GW_MAX * 32) k_grad(GradArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[GW_MAX];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int D = a.dim;
  const uint32_t RB = (uint32_t)D * 4u;
  const bool adagrad = a.sink_mode == 0 && a.opt == 1;
  float *dybuf = reinterpret_cast<float *>(smem) + (size_t)wib * 3 * CH * D;
  float *wbuf = dybuf + (size_t)CH * D;
  float *abuf = wbuf + (size_t)CH * D;
  const int64_t c = (int64_t)blockIdx.x * nw + wib;
  const int64_t p0 = c * CH;
  if (lane == 0) {
    mbar_init(&bars[wib], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (p0 >= a.n) return;

  // ---- 1. keys, segment structure, row addresses
  const int64_t p = p0 + lane;
  uint32_t k = p < a.n ? a.skey[p] : EMB_SENTINEL;
  const bool valid = k != EMB_SENTINEL;
  uint32_t kprev = __shfl_up_sync(0xffffffffu, k, 1);
  if (lane == 0) kprev = p0 > 0 ? a.skey[p0 - 1] : ~k;
  uint32_t knext = __shfl_down_sync(0xffffffffu, k, 1);
  if (lane == 31) knext = (p0 + CH < a.n) ? a.skey[p0 + CH] : EMB_SENTINEL;
  const bool head = valid && k != kprev;
  const bool tail = valid && k != knext;
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  const uint32_t hmask = __ballot_sync(0xffffffffu, head);
  const uint32_t tmask = __ballot_sync(0xffffffffu, tail);
  const bool wantw = a.sink_mode == 0 && valid && (head || lane == 0);

  const float *src_row = nullptr;
  int32_t len = 1;
  const uint32_t local = k & a.lmask;
  bool guard_ok = true;
  if (valid) {
    const uint32_t pay = a.spay[p];
    if (a.src_mode == 0) {
      const uint32_t bag = pay < (uint64_t)a.nsrc_occ ? a.bag_of[pay] : 0xFFFFFFFFu;
      guard_ok = (int64_t)bag < a.nsrc;
      const uint32_t s = bag / (uint32_t)a.batch, b = bag % (uint32_t)a.batch;
      src_row = a.dy + ((size_t)b * a.num_slots + s) * D;
      if (a.blen && guard_ok) len = a.blen[bag];
    } else {
      guard_ok = (int64_t)pay < a.nsrc;
      src_row = a.src + (size_t)pay * D;
    }
    if (a.sink_mode == 0 && (int64_t)local >= a.nrows) guard_ok = false;
  }
  if (__any_sync(0xffffffffu, valid && !guard_ok)) {
    // a broken invariant (bug): report and skip the whole chunk (never issue an unchecked copy)
    if (lane == 0) atomicOr(a.err, EMB_DEVERR_INTERNAL);
    return;
  }
  const uint32_t nwant = __popc(__ballot_sync(0xffffffffu, wantw));
  if (lane == 0)
    mbar_arrive_expect_tx(&bars[wib], (__popc(vmask) + nwant * (adagrad ? 2u : 1u)) * RB);
  __syncwarp();
  if (valid) bulk_g2s(dybuf + (size_t)lane * D, src_row, RB, &bars[wib]);
  if (wantw) {
    bulk_g2s(wbuf + (size_t)lane * D, a.w + (size_t)local * D, RB, &bars[wib]);
    if (adagrad) bulk_g2s(abuf + (size_t)lane * D, a.a + (size_t)local * D, RB, &bars[wib]);
  }
  mbar_wait(&bars[wib], 0);

  // ---- 2. walk the chunk in order
  const int col = lane * CPL;
  const bool active = col < D;
  double acc[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) acc[q] = 0.0;
  const double lr = (double)a.lr, eps = (double)a.eps;

  // sink for a complete segment whose w/a rows sit at smem slot `ws`
  auto sink = [&](int ws, uint32_t key, int64_t pos_any) {
    if (!active) return;
    if (a.sink_mode == 1) {
      const uint32_t u = a.useg[pos_any];
      if ((int64_t)u >= a.nout) {
        if (lane == 0) atomicOr(a.err, EMB_DEVERR_INTERNAL);
        return;
      }
      float *dst = a.out_rows + (size_t)u * D + col;
#pragma unroll
      for (int q = 0; q < CPL; q += 2)
        *reinterpret_cast<float2 *>(dst + q) = make_float2((float)acc[q], (float)acc[q + 1]);
      return;
    }
    const uint32_t lrow = key & a.lmask;
    const float *wr = wbuf + (size_t)ws * D + col;
    float *wg = a.w + (size_t)lrow * D + col;
    if (!adagrad) {
#pragma unroll
      for (int q = 0; q < CPL; q += 2) {
        const float2 w2 = *reinterpret_cast<const float2 *>(wr + q);
        float2 o;
        o.x = (float)__dsub_rn((double)w2.x, __dmul_rn(lr, acc[q]));
        o.y = (float)__dsub_rn((double)w2.y, __dmul_rn(lr, acc[q + 1]));
        *reinterpret_cast<float2 *>(wg + q) = o;
      }
    } else {
      const float *ar = abuf + (size_t)ws * D + col;
      float *ag = a.a + (size_t)lrow * D + col;
#pragma unroll
      for (int q = 0; q < CPL; q += 2) {
        const float2 w2 = *reinterpret_cast<const float2 *>(wr + q);
        const float2 a2 = *reinterpret_cast<const float2 *>(ar + q);
        const double g0 = acc[q], g1 = acc[q + 1];
        const double a0 = __dadd_rn((double)a2.x, __dmul_rn(g0, g0));
        const double a1 = __dadd_rn((double)a2.y, __dmul_rn(g1, g1));
        const double w0 = __dsub_rn((double)w2.x, __ddiv_rn(__dmul_rn(lr, g0), __dadd_rn(__dsqrt_rn(a0), eps)));
        const double w1 = __dsub_rn((double)w2.y, __ddiv_rn(__dmul_rn(lr, g1), __dadd_rn(__dsqrt_rn(a1), eps)));
        *reinterpret_cast<float2 *>(wg + q) = make_float2((float)w0, (float)w1);
        *reinterpret_cast<float2 *>(ag + q) = make_float2((float)a0, (float)a1);
      }
    }
  };

  // piece crossing a chunk boundary: store partial, ticket, last arriver combines + sinks
  auto span = [&](int64_t slot, int ws, uint32_t key, int64_t pos) {
    double *dstp = a.partials + (size_t)slot * D + col;
    if (active) {
#pragma unroll
      for (int q = 0; q < CPL; q += 2) __stcg(reinterpret_cast<double2 *>(dstp + q), make_double2(acc[q], acc[q + 1]));
    }
    __threadfence();
    __syncwarp();
    int64_t c0 = 0, c1 = 0;
    int last = 0;
    if (lane == 0) {
      c0 = seg_first(a.skey, pos, key) / CH;
      c1 = seg_last(a.skey, a.n, pos, key) / CH;
      const uint32_t t = atomicAdd(&a.tickets[c0], 1u);
      last = (t == (uint32_t)(c1 - c0));
      if (last) {
        a.tickets[c0] = 0;  // ready for the next step
        __threadfence();
      }
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    c1 = __shfl_sync(0xffffffffu, c1, 0);
    if (active) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[q] = 0.0;
      for (int64_t cc = c0; cc <= c1; ++cc) {
        const double *src = a.partials + (size_t)(cc == c0 ? 2 * cc + 1 : 2 * cc) * D + col;
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
          const double2 v = ld_cg_d2(reinterpret_cast<const double2 *>(src + q));
          acc[q] = __dadd_rn(acc[q], v.x);
          acc[q + 1] = __dadd_rn(acc[q + 1], v.y);
        }
      }
    }
    sink(ws, key, pos);
  };

  int pstart = 0;
  const int nvalid = __popc(vmask);  // valid positions are a prefix of the chunk
  for (int i = 0; i < nvalid; ++i) {
    if ((hmask >> i) & 1u) {
      pstart = i;
#pragma unroll
      for (int q = 0; q < CPL; ++q) acc[q] = 0.0;
    }
    const int32_t li = __shfl_sync(0xffffffffu, len, i);
    if (active) {
      const float *r = dybuf + (size_t)i * D + col;
      if (a.blen && li > 0) {
        const double dl = (double)li;
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
          const float2 v = *reinterpret_cast<const float2 *>(r + q);
          acc[q] = __dadd_rn(acc[q], __ddiv_rn((double)v.x, dl));
          acc[q + 1] = __dadd_rn(acc[q + 1], __ddiv_rn((double)v.y, dl));
        }
      } else {
#pragma unroll
        for (int q = 0; q < CPL; q += 2) {
          const float2 v = *reinterpret_cast<const float2 *>(r + q);
          acc[q] = __dadd_rn(acc[q], (double)v.x);
          acc[q + 1] = __dadd_rn(acc[q + 1], (double)v.y);
        }
      }
    }
    if ((tmask >> i) & 1u) {
      const uint32_t ki = __shfl_sync(0xffffffffu, k, i);
      if ((hmask >> pstart) & 1u) sink(pstart, ki, p0 + i);   // complete inside the chunk
      else span(2 * c, 0, ki, p0 + i);                         // continuation piece ending here
    }
  }
  if (nvalid > 0 && !((tmask >> (nvalid - 1)) & 1u)) {
    // the last piece continues into the next chunk
    const uint32_t ki = __shfl_sync(0xffffffffu, k, nvalid - 1);
    if ((hmask >> pstart) & 1u) span(2 * c + 1, pstart, ki, p0 + nvalid - 1);
    else span(2 * c, 0, ki, p0 + nvalid - 1);  // the whole chunk lies inside one segment
  }
}

static int grad_warps(int D) { return D <= 64 ? 4 : (D <= 128 ? 2 : 1); }

template <int CPL>
static cudaError_t launch_grad_t(const GradArgs &a, int64_t blocks, int wpc, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_grad<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_grad<CPL><<<(unsigned)blocks, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_grad(const GradArgs &a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  const int wpc = grad_warps(a.dim);
  const int64_t chunks = (a.n + CH - 1) / CH;
  const int64_t blocks = (chunks + wpc - 1) / wpc;
  const size_t smem = (size_t)wpc * 3 * CH * a.dim * sizeof(float);
  if (a.dim <= 64) return launch_grad_t<2>(a, blocks, wpc, smem, st);
  if (a.dim <= 128) return launch_grad_t<4>(a, blocks, wpc, smem, st);
  return launch_grad_t<8>(a, blocks, wpc, smem, st);
}

}  // namespace emb
