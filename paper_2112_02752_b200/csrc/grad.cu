// grad.cu — K6+K7 fused: deterministic segment reduce of duplicate-id gradients + sparse optimizer
// apply (readings R8-R14, R16).
//
// Input: the stably sorted (routing key, payload) array of the step. Every distinct key is a
// contiguous SEGMENT whose contributions appear in occurrence order (stable sort); invalid
// occurrences (EMB_SENTINEL keys) are skipped wherever they sit.
//
// Mapping (v4; ncu history: v1 IPC 0.72 at 10% occupancy; v2/v3 ~100 instructions per position and
// spill stores of in-flight row registers serialising the loads):
//  * persistent warps; warp w owns the contiguous position range [w*R, (w+1)*R) of the sorted array
//    (R = ceil(n / #warps), fixed by n and the grid, so the summation order is fixed);
//  * the range is cut into tiles of T positions (lane i < T owns position i's metadata: key, source
//    row, segment flags). Each tile's rows — the T contribution rows (dY[b][s] or a received gradient
//    row) and the table + Adagrad rows of the segments that END in the tile and began in the range —
//    are fetched by 1-D TMA bulk copies (cp.async.bulk, one row per lane-issued copy) into a
//    shared-memory stage, completion counted on that stage's mbarrier. Two stages per warp: tile k+1
//    is in flight while tile k is reduced, and no row ever sits in registers waiting for memory;
//  * the reduce walks the tile in position order, lanes owning CPL columns, accumulating in fp64
//    (mean: c = dY / |bag|); a segment that starts and ends in the warp's range is applied at its last
//    position (table rows read from the stage, written back with plain stores);
//  * a segment crossing range boundaries leaves one fp64 partial per warp (slot 2w: the piece that
//    continues from warp w-1; slot 2w+1: the piece that starts in w and continues) and takes a ticket
//    on tickets[first position of the segment] (segment bounds by a warp-parallel gallop search); the
//    LAST arriving warp sums the partials in warp order and applies. Warp order is fixed, so the
//    results are bitwise reproducible run to run (R10).
// Sinks: mode 0 = optimizer. SGD: w <- w - lr*G in fp64, rounded once (as the oracle). Adagrad
// (element-wise, eps outside the sqrt, R12): a <- a + G^2 in fp64 rounded to fp32; the update
// lr*G/(sqrt(a)+eps) in fp32 with MUFU sqrt/rcp (|update| <= lr, so its relative error of a few
// 1e-7 is <= 1e-8 absolute, far inside the 1e-6 + 1e-5|w| tolerance; DESIGN.md §3 R16').
// Mode 1 = write the fp32 per-unique-key gradient (requester side of the W>1 exchange).
#include "common.cuh"
#include "internal.h"
#include "vec.cuh"

namespace emb {

namespace {
constexpr int NS = 2;  // stages per warp
}  // namespace

template <int CPL>
struct DAcc {
  double v[CPL];
};

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// smem row fragment of a lane (generic pointer: works for smem stages and global rows)
template <int CPL>
__device__ __forceinline__ void ld_frag(VecF<CPL> &v, const float *p) {
  if constexpr (CPL == 2) {
    const float2 t = *reinterpret_cast<const float2 *>(p);
    v.v[0] = t.x;
    v.v[1] = t.y;
  } else {
#pragma unroll
    for (int c = 0; c < CPL; c += 4) {
      const float4 t = *reinterpret_cast<const float4 *>(p + c);
      v.v[c] = t.x; v.v[c + 1] = t.y; v.v[c + 2] = t.z; v.v[c + 3] = t.w;
    }
  }
}

// shared-memory fragment load at a 32-bit shared address
template <int CPL>
__device__ __forceinline__ void lds_frag(VecF<CPL> &v, uint32_t saddr) {
#pragma unroll
  for (int c = 0; c < CPL; c += 2)
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.v[c]), "=f"(v.v[c + 1]) : "r"(saddr + 4u * c));
}
template <int CPL>
__device__ __forceinline__ void stg_frag(float *p, const VecF<CPL> &v) {
#pragma unroll
  for (int c = 0; c < CPL; c += 2)
    asm volatile("st.global.v2.f32 [%0], {%1,%2};" ::"l"(p + c), "f"(v.v[c]), "f"(v.v[c + 1]) : "memory");
}

// optimizer update of one row fragment; w / a fragments already in registers
template <int CPL>
__device__ __forceinline__ void apply_frag(const GradArgs &a, const double (&acc)[CPL], const VecF<CPL> &wv,
                                           const VecF<CPL> &av, uint32_t lrow, int col) {
  float *wg = a.w + (size_t)lrow * a.dim + col;
  VecF<CPL> wo;
  if (a.opt == 0) {
    const double lr = a.lr;
#pragma unroll
    for (int c = 0; c < CPL; ++c) wo.v[c] = (float)__dsub_rn((double)wv.v[c], __dmul_rn(lr, acc[c]));
    stg_frag<CPL>(wg, wo);
  } else {
    VecF<CPL> ao;
    const float lrf = (float)a.lr, epsf = (float)a.eps;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const double a64 = __dadd_rn((double)av.v[c], __dmul_rn(acc[c], acc[c]));
      const float af = (float)a64;
      const float g = (float)acc[c];
      const float r = rcp_approx(sqrt_approx(af) + epsf);
      ao.v[c] = af;
      wo.v[c] = wv.v[c] - (lrf * g) * r;
    }
    stg_frag<CPL>(wg, wo);
    stg_frag<CPL>(a.a + (size_t)lrow * a.dim + col, ao);
  }
}

// row update reading w / a from (generic) memory
template <int CPL>
__device__ __forceinline__ void apply_row(const GradArgs &a, const double (&acc)[CPL], const float *wsrc,
                                          const float *asrc, uint32_t lrow, int col) {
  VecF<CPL> wv, av;
  ld_frag<CPL>(wv, wsrc);
  if (a.opt != 0) ld_frag<CPL>(av, asrc);
  apply_frag<CPL>(a, acc, wv, av, lrow, col);
}

// warp-parallel gallop: first (dir = -1) or last (dir = +1) position of the segment of key k that
// contains position p (all lanes call; one L2 round trip per 32x of distance)
__device__ int64_t seg_bound_warp(const uint32_t *skey, int64_t n, int64_t p, uint32_t k, int dir) {
  const int lane = threadIdx.x & 31;
  int64_t in = p;  // known inside the segment
  int64_t stride = 1;
  // gallop outwards until a probe leaves the segment
  while (true) {
    const int64_t q = in + dir * (int64_t)(lane + 1) * stride;
    const bool out = q < 0 || q >= n || ld_cg_u32(skey + q) != k;
    const uint32_t m = __ballot_sync(0xffffffffu, out);
    if (m) {
      const int f = __ffs(m) - 1;  // probes 0..f-1 are inside
      in = in + dir * (int64_t)f * stride;
      if (stride == 1) return in;
      stride >>= 5;  // refine inside (in, in + dir*32*stride_old]
      break;
    }
    in = in + dir * 32 * stride;
    stride <<= 5;
  }
  while (true) {
    const int64_t q = in + dir * (int64_t)(lane + 1) * stride;
    const bool out = q < 0 || q >= n || ld_cg_u32(skey + q) != k;
    const uint32_t m = __ballot_sync(0xffffffffu, out);
    const int f = m ? __ffs(m) - 1 : 32;
    in = in + dir * (int64_t)f * stride;
    if (stride == 1) return in;
    stride >>= 5;
  }
}

// piece crossing a range boundary: store the partial, take a ticket on the segment; the last arriving
// warp sums the partials in warp order and sinks the total. (Rare path: <= 2 per warp; not inlined.)
template <int CPL>
__device__ __noinline__ void span_piece(const GradArgs &a, const DAcc<CPL> acc, int64_t slot, int64_t pos,
                                        uint32_t key, int64_t R) {
  const int lane = threadIdx.x & 31;
  const int D = a.dim;
  const int col = lane * CPL;
  const bool active = col < D;
  double *dst = a.partials + (size_t)slot * D + col;
  if (active) {
#pragma unroll
    for (int c = 0; c < CPL; c += 2)
      __stcg(reinterpret_cast<double2 *>(dst + c), make_double2(acc.v[c], acc.v[c + 1]));
  }
  const int64_t first = seg_bound_warp(a.skey, a.n, pos, key, -1);
  const int64_t lastp = seg_bound_warp(a.skey, a.n, pos, key, +1);
  __threadfence();
  __syncwarp();
  int last = 0;
  const int64_t w0 = first / R, w1 = lastp / R;
  if (lane == 0) {
    const uint32_t t = atomicAdd(&a.tickets[first], 1u);
    last = (t == (uint32_t)(w1 - w0));
    if (last) {
      a.tickets[first] = 0;  // ready for the next step
      __threadfence();
    }
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last || !active) return;
  double tot[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) tot[c] = 0.0;
  for (int64_t ww = w0; ww <= w1; ++ww) {
    const double *src = a.partials + (size_t)(ww == w0 ? 2 * ww + 1 : 2 * ww) * D + col;
#pragma unroll
    for (int c = 0; c < CPL; c += 2) {
      const double2 v = ld_cg_d2(reinterpret_cast<const double2 *>(src + c));
      tot[c] = __dadd_rn(tot[c], v.x);
      tot[c + 1] = __dadd_rn(tot[c + 1], v.y);
    }
  }
  if (a.sink_mode == 0) {
    const uint32_t lrow = key & a.lmask;
    apply_row<CPL>(a, tot, a.w + (size_t)lrow * D + col, a.opt == 1 ? a.a + (size_t)lrow * D + col : nullptr,
                   lrow, col);
  } else {
    VecF<CPL> o;
#pragma unroll
    for (int c = 0; c < CPL; ++c) o.v[c] = (float)tot[c];
    o.store(a.out_rows + (size_t)a.useg[pos] * D + col);
  }
}

// per-lane metadata of one tile (lane i < T describes position t0 + i)
struct TileMeta {
  uint32_t key;   // routing key (EMB_SENTINEL = invalid / beyond the range)
  uint32_t srow;  // row of dY (mode 0) or of the received gradients (mode 1)
  int32_t len;    // bag length (mean pooling)
  uint32_t vmask, hmask, tmask, amask;  // warp-uniform: valid / head / tail / applies-here
  int cnt;
};

template <int CPL, int T>
__global__ void __launch_bounds__(256) k_grad(const __grid_constant__ GradArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[8][NS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int D = a.dim;
  const uint32_t RB = (uint32_t)D * 4u;
  const int col = lane * CPL;
  const bool active = col < D;
  const bool sink_opt = a.sink_mode == 0;
  const bool adagrad = sink_opt && a.opt == 1;
  // per-warp stages: [NS][3][T][D] floats (contribution rows, w rows, a rows)
  float *stage0 = reinterpret_cast<float *>(smem) + (size_t)wib * NS * 3 * T * D;
  const int64_t gw = ((int64_t)blockIdx.x * (blockDim.x >> 5)) + wib;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n = a.n;
  const int64_t R = (n + nwarps - 1) / nwarps;
  const int64_t p_lo = gw * R;
  const int64_t p_hi = (p_lo + R < n) ? p_lo + R : n;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[wib][s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (p_lo >= p_hi) return;
  const float *src_base = a.src_mode == 0 ? a.dy : a.src;

  bool seen_head = false;  // a head was issued earlier in this range (=> open pieces began here)
  uint32_t kprev_carry = p_lo > 0 ? a.skey[p_lo - 1] : EMB_SENTINEL;
  bool bad = false;

  // load metadata of the tile at t0 and issue its bulk copies into stage s
  auto issue = [&](int64_t t0, int s, TileMeta &m) {
    const int cnt = (int)((p_hi - t0) < T ? (p_hi - t0) : T);
    m.cnt = cnt;
    const int64_t p = t0 + lane;
    uint32_t k = EMB_SENTINEL, kn = EMB_SENTINEL, srow = 0;
    int32_t len = 1;
    if (lane < cnt) {
      k = a.skey[p];
      if (k != EMB_SENTINEL) {
        const uint32_t pay = a.spay[p];
        if (a.src_mode == 0) {
          srow = pay < (uint64_t)a.nsrc_occ ? a.drow[pay] : 0xFFFFFFFEu;
        } else {
          srow = pay;
        }
        if ((int64_t)srow >= a.nsrc) bad = true;
        else if (a.blen) len = a.blen[srow];
        if (sink_opt && (int64_t)(k & a.lmask) >= a.nrows) bad = true;
      }
    }
    if (lane == cnt - 1) kn = (p + 1 < n) ? a.skey[p + 1] : EMB_SENTINEL;
    uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    if (lane == 0) kp = kprev_carry;
    const uint32_t kd = __shfl_down_sync(0xffffffffu, k, 1);
    if (lane < cnt - 1) kn = kd;
    const bool valid = lane < cnt && k != EMB_SENTINEL && !bad;
    const bool head = valid && k != kp;
    const bool tail = valid && k != kn;
    m.vmask = __ballot_sync(0xffffffffu, valid);
    m.hmask = __ballot_sync(0xffffffffu, head);
    m.tmask = __ballot_sync(0xffffffffu, tail);
    const uint32_t le_mask = (lane < 31) ? ((2u << lane) - 1u) : 0xFFFFFFFFu;
    const bool applies = tail && (((m.hmask & le_mask) != 0) || seen_head);
    m.amask = __ballot_sync(0xffffffffu, applies);
    seen_head = seen_head || m.hmask != 0;
    kprev_carry = __shfl_sync(0xffffffffu, k, cnt - 1);
    m.key = k;
    m.srow = srow;
    m.len = len;
    // bulk copies of the tile's rows
    float *st = stage0 + (size_t)s * 3 * T * D;
    const bool wantw = sink_opt && applies;
    const uint32_t bytes =
        (__popc(m.vmask) + __popc(m.amask & (sink_opt ? 0xFFFFFFFFu : 0u)) * (adagrad ? 2u : 1u)) * RB;
    if (lane == 0) mbar_arrive_expect_tx(&bars[wib][s], bytes);
    __syncwarp();
    if (valid) bulk_g2s(st + (size_t)lane * D, src_base + (size_t)srow * D, RB, &bars[wib][s]);
    if (wantw) {
      const size_t off = (size_t)(k & a.lmask) * D;
      bulk_g2s(st + (size_t)(T + lane) * D, a.w + off, RB, &bars[wib][s]);
      if (adagrad) bulk_g2s(st + (size_t)(2 * T + lane) * D, a.a + off, RB, &bars[wib][s]);
    }
  };

  TileMeta meta[NS];
  const int64_t ntile = (p_hi - p_lo + T - 1) / T;
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (s < ntile) issue(p_lo + (int64_t)s * T, s, meta[s]);
  if (__any_sync(0xffffffffu, bad)) {  // broken invariant (bug): report, never apply garbage
    if (lane == 0) atomicOr(a.err, EMB_DEVERR_INTERNAL);
  }

  DAcc<CPL> acc;
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc.v[c] = 0.0;
  bool begins = false;  // the open piece began inside this warp's range
  bool open = false;
  int64_t open_pos = p_lo;
  uint32_t open_key = 0;

  for (int64_t tb = 0; tb < ntile; tb += NS) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {  // static stage index: the tile metadata stays in registers
      const int64_t ti = tb + s;
      if (ti >= ntile) break;
      const int64_t t0 = p_lo + ti * T;
      TileMeta &m = meta[s];
      mbar_wait(&bars[wib][s], (uint32_t)((ti / NS) & 1));
      const uint32_t sbase = smem_u32(stage0 + (size_t)s * 3 * T * D) + 4u * (uint32_t)col;
      const uint32_t vmask = m.vmask, hmask = m.hmask, tmask = m.tmask;
#pragma unroll
      for (int i = 0; i < T; ++i) {  // compile-time positions: constant shared offsets
        if (!((vmask >> i) & 1u)) continue;
        if ((hmask >> i) & 1u) {
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc.v[c] = 0.0;
          begins = true;
        }
        VecF<CPL> v;
        if (active) lds_frag<CPL>(v, sbase + 4u * (uint32_t)(i * D));
        else v.zero();
        if (a.blen) {
          const int32_t li = __shfl_sync(0xffffffffu, m.len, i);
          const double dl = (double)li;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            acc.v[c] = __dadd_rn(acc.v[c], li > 1 ? __ddiv_rn((double)v.v[c], dl) : (double)v.v[c]);
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc.v[c] = __dadd_rn(acc.v[c], (double)v.v[c]);
        }
        if ((tmask >> i) & 1u) {
          const uint32_t ki = __shfl_sync(0xffffffffu, m.key, i);
          if (begins) {  // complete inside the range
            if (active) {
              if (sink_opt) {
                VecF<CPL> wv, av;
                lds_frag<CPL>(wv, sbase + 4u * (uint32_t)((T + i) * D));
                if (adagrad) lds_frag<CPL>(av, sbase + 4u * (uint32_t)((2 * T + i) * D));
                apply_frag<CPL>(a, acc.v, wv, av, ki & a.lmask, col);
              } else {
                VecF<CPL> o;
#pragma unroll
                for (int c = 0; c < CPL; ++c) o.v[c] = (float)acc.v[c];
                stg_frag<CPL>(a.out_rows + (size_t)a.useg[t0 + i] * D + col, o);
              }
            }
          } else {
            span_piece<CPL>(a, acc, 2 * gw, t0 + i, ki, R);  // continuation piece that ends here
          }
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc.v[c] = 0.0;
          begins = false;
        }
      }
      // an open piece at the end of the tile: remember where it stands (used after the last tile)
      const uint32_t after_last_tail = tmask ? (vmask & ~((2u << (31 - __clz(tmask))) - 1u)) : vmask;
      if (after_last_tail) {
        const int lv = 31 - __clz(vmask);
        open = true;
        open_pos = t0 + lv;
        open_key = __shfl_sync(0xffffffffu, m.key, lv);
      } else if (tmask) {
        open = false;
      }
      __syncwarp();
      if (ti + NS < ntile) {
        fence_proxy_async_smem();  // our generic reads of the stage precede the async refill
        issue(p_lo + (ti + NS) * T, s, m);
        if (__any_sync(0xffffffffu, bad)) {
          if (lane == 0) atomicOr(a.err, EMB_DEVERR_INTERNAL);
        }
      }
    }
  }
  if (open) span_piece<CPL>(a, acc, begins ? 2 * gw + 1 : 2 * gw, open_pos, open_key, R);  // continues past the range
}

static int g_sms = 0;

template <int CPL, int T>
static cudaError_t launch_grad_t(const GradArgs &a, cudaStream_t st) {
  const size_t per_warp = (size_t)NS * 3 * T * a.dim * sizeof(float);
  int wpc = (int)(112 * 1024 / per_warp);  // warps per CTA: ~112 KB of stages, 2 CTAs per SM
  if (wpc > 8) wpc = 8;
  if (wpc < 1) wpc = 1;
  const size_t smem = per_warp * wpc;
  static size_t attr = 0;
  if (attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(k_grad<CPL, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grad<CPL, T>, wpc * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)g_sms * per_sm;
  const int64_t max_blocks = ((a.n + 4 * T - 1) / (4 * T) + wpc - 1) / wpc;  // >= 4 tiles per warp
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  k_grad<CPL, T><<<(unsigned)blocks, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

int64_t grad_max_warps(int dev) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int64_t)sms * 64;  // upper bound on resident warps (partials are sized from it)
}

cudaError_t launch_grad(const GradArgs &a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (a.dim <= 64) return launch_grad_t<2, 8>(a, st);
  if (a.dim <= 128) return launch_grad_t<4, 8>(a, st);
  return launch_grad_t<8, 8>(a, st);
}

}  // namespace emb
