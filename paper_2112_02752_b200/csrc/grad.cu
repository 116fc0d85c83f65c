// grad.cu — K6+K7 fused: deterministic segment reduce of duplicate-id gradients + sparse optimizer
// apply (readings R8-R14, R16).
//
// Input: the stably sorted (fused key, payload) array of the step. Every distinct key is a
// contiguous SEGMENT whose contributions appear in occurrence order (stable sort); invalid
// occurrences (EMB_SENTINEL keys) are skipped wherever they sit.
//
// Mapping (v5; ncu history: v1 IPC 0.72 at 10% occupancy; v2/v3 spill stores of in-flight row
// registers; v4 per-lane TMA bulk copies compile to a serialised uniform-register loop, ~8
// instructions per row, and deeper TMA pipelines lost warps => the walk is issue-bound):
//  * persistent warps; warp w owns the contiguous position range [w*R, (w+1)*R) of the sorted array
//    (R = ceil(n / #warps), fixed by n and the grid, so the summation order is fixed);
//  * the range is cut into tiles of T positions; lane i < T owns position i's metadata. Metadata is
//    a rolling software pipeline (key/payload NS+2 tiles ahead, source row index NS+1 ahead);
//  * each tile's rows — the T contribution rows (dY[b][s] or a received gradient row) and the table
//    + Adagrad rows of the segments that END in the tile and began in the range — are copied into
//    the warp's shared-memory stage with per-lane 16-byte cp.async (LDGSTS: a whole 256-B row per 16
//    lanes, no register staging), one commit group per tile, NS stages in flight;
//  * the walk is unrolled over the T positions at compile time: fp64 accumulation in position order
//    (mean: c = dY / |bag|); a segment that starts and ends in the warp's range is applied at its
//    last position straight from the stage;
//  * a segment crossing range boundaries leaves one fp64 partial per warp (slot 2w: the piece that
//    continues from warp w-1; slot 2w+1: the piece that starts in w and continues) and takes a ticket
//    on tickets[first position of the segment] (segment bounds by a warp-parallel gallop search); the
//    LAST arriving warp sums the partials in warp order and applies. Warp order is fixed, so the
//    results are bitwise reproducible run to run (R10).
// Sinks (template MODE): 0 = SGD: w <- w - lr*G in fp64, rounded once (as the oracle). 1 = Adagrad
// (element-wise, eps outside the sqrt, R12): a <- fma(g, g, a) in fp32 with g = fp32(G) (relative
// error <= ~2e-7 against the oracle's fp64 a + G^2 rounded once; the fp64 form cost 4 us per step in
// conversions); the update lr*g/(sqrt(a)+eps) in fp32 with MUFU sqrt/rcp (|update| <= lr, so its
// relative error of a few 1e-7 is <= 1e-8 absolute, far inside the 1e-6 + 1e-5|w| tolerance;
// DESIGN.md §2 R16').
// 3 = the merged fp32 per-key row stored into the owner's gradient region through peer memory
// (requester side of the W > 1 exchange; host sink_mode 2). 4 = row-wise Adagrad (SURVEY §8(f) f1, R14'): one
// accumulator per row, a <- a + (1/D) sum_c g[c]^2 with g = fp32(G) (fp32 FMAs + an xor-butterfly
// warp reduction: every lane ends with the same total); w as in mode 1 with the row's a.
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "vec.cuh"
#include "p2p_dev.cuh"

namespace emb {

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

template <int CPL>
__device__ __forceinline__ void lds_frag(VecF<CPL> &v, uint32_t saddr) {
#pragma unroll
  for (int c = 0; c < CPL; c += 2)
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.v[c]), "=f"(v.v[c + 1]) : "r"(saddr + 4u * c));
}
template <int CPL>
__device__ __forceinline__ void ldg_frag(VecF<CPL> &v, const float *p) {
#pragma unroll
  for (int c = 0; c < CPL; c += 2)
    asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(v.v[c]), "=f"(v.v[c + 1]) : "l"(p + c));
}
template <int CPL>
__device__ __forceinline__ void stg_frag(float *p, const VecF<CPL> &v) {
#pragma unroll
  for (int c = 0; c < CPL; c += 2)
    asm volatile("st.global.v2.f32 [%0], {%1,%2};" ::"l"(p + c), "f"(v.v[c]), "f"(v.v[c + 1]) : "memory");
}

// optimizer constants, converted once per kernel
// PRECISE (template parameter of the Adagrad sinks, chosen on the host for lr > 1): fp64 from the fp32
// state, the oracle's formula with one rounding each, instead of R16' (fp32 FMA accumulator +
// approximate sqrt / reciprocal, whose absolute error ~lr * 3e-7 exceeds the 1e-6 absolute tolerance
// once lr > ~3). A separate instantiation: a runtime branch, even out of line, cost the fast path
// 79 -> 125 us at C2 (register pressure around the call), DESIGN.md §2 R16'.
struct OptConst {
  double lr, eps;
  float lrf, epsf;
};
__device__ __forceinline__ OptConst opt_const(const GradArgs &a) { return {a.lr, a.eps, (float)a.lr, (float)a.eps}; }

// the fp64 Adagrad sink of one lane's fragment (PRECISE instantiations only)
template <int CPL>
__device__ __forceinline__ void adagrad_precise(const double (&acc)[CPL], const VecF<CPL> &wv, const VecF<CPL> &av,
                                             VecF<CPL> &wo, VecF<CPL> &ao, double lr, double eps) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const double an = __dadd_rn((double)av.v[c], __dmul_rn(acc[c], acc[c]));
    ao.v[c] = (float)an;
    wo.v[c] = (float)__dsub_rn((double)wv.v[c], __ddiv_rn(__dmul_rn(lr, acc[c]), __dadd_rn(__dsqrt_rn(an), eps)));
  }
}

// optimizer update (MODE 0/1) of one lane's row fragment, w / a already in registers; D = row width
// (compile-time when DC != 0)
template <int CPL, int MODE, bool PRECISE = false>
__device__ __forceinline__ void apply_frag(const GradArgs &a, const OptConst &oc, const double (&acc)[CPL],
                                           const VecF<CPL> &wv, const VecF<CPL> &av, size_t row_off) {
  VecF<CPL> wo;
  if constexpr (MODE == 0) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) wo.v[c] = (float)__dsub_rn((double)wv.v[c], __dmul_rn(oc.lr, acc[c]));
    stg_frag<CPL>(a.w + row_off, wo);
  } else {
    VecF<CPL> ao;
    if constexpr (PRECISE) {
      adagrad_precise<CPL>(acc, wv, av, wo, ao, oc.lr, oc.eps);
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const float g = (float)acc[c];
        const float af = __fmaf_rn(g, g, av.v[c]);  // a + G^2: one fp32 FMA from the rounded G (R16')
        const float r = rcp_approx(sqrt_approx(af) + oc.epsf);
        ao.v[c] = af;
        wo.v[c] = wv.v[c] - (oc.lrf * g) * r;
      }
    }
    stg_frag<CPL>(a.w + row_off, wo);
    stg_frag<CPL>(a.a + row_off, ao);
  }
}

// fp64 row-wise Adagrad sink (PRECISE instantiations only): warp-collective
template <int CPL>
__device__ __forceinline__ void rowwise_precise(const GradArgs &a, const OptConst &oc, const double (&acc)[CPL],
                                             const VecF<CPL> &wv, float a_old, size_t row_off, uint32_t lrow,
                                             bool active, int D) {
  double sd = 0.0;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (active) sd = __dadd_rn(sd, __dmul_rn(acc[c], acc[c]));
#pragma unroll
  for (int o = 16; o; o >>= 1) sd = __dadd_rn(sd, __shfl_xor_sync(0xffffffffu, sd, o));
  const double an = __dadd_rn((double)a_old, __ddiv_rn(sd, (double)D));
  const double den = __dadd_rn(__dsqrt_rn(an), oc.eps);
  if (active) {
    VecF<CPL> wo;
#pragma unroll
    for (int c = 0; c < CPL; ++c) wo.v[c] = (float)__dsub_rn((double)wv.v[c], __ddiv_rn(__dmul_rn(oc.lr, acc[c]), den));
    stg_frag<CPL>(a.w + row_off, wo);
  }
  if ((threadIdx.x & 31) == 0) a.a[lrow] = (float)an;
}

// row-wise Adagrad (MODE 4) of one row: warp-collective (every lane calls it; inactive lanes hold no
// columns). a_old is the row's accumulator (the same value in every lane).
template <int CPL, bool PRECISE = false>
__device__ __forceinline__ void apply_rowwise(const GradArgs &a, const OptConst &oc, const double (&acc)[CPL],
                                              const VecF<CPL> &wv, float a_old, size_t row_off, uint32_t lrow,
                                              bool active, int D) {
  // the row's sum of squares in fp32 from the rounded gradient g = fp32(G) (the g the update uses):
  // FMAs per lane, then an xor butterfly -- at every level the two partners add the same two operands
  // (commutative), so all lanes end with the bitwise identical total. Relative error <= ~4e-7 against
  // the oracle's fp64 mean of G^2 (reading R14'); the fp64 chain cost ~20 us of the C2 step.
  VecF<CPL> g;
  if constexpr (PRECISE) {  // fp64 from the fp32 state (see OptConst)
    rowwise_precise<CPL>(a, oc, acc, wv, a_old, row_off, lrow, active, D);
    return;
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    g.v[c] = (float)acc[c];
    if (active) s = __fmaf_rn(g.v[c], g.v[c], s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  // s / D: a multiply by the exact reciprocal when D is a power of two (every configured D)
  const float mean = (D & (D - 1)) == 0 ? __fmul_rn(s, 1.0f / (float)D) : __fdiv_rn(s, (float)D);
  const float af = __fadd_rn(a_old, mean);
  const float r = rcp_approx(sqrt_approx(af) + oc.epsf);
  if (active) {
    VecF<CPL> wo;
#pragma unroll
    for (int c = 0; c < CPL; ++c) wo.v[c] = wv.v[c] - (oc.lrf * g.v[c]) * r;
    stg_frag<CPL>(a.w + row_off, wo);
  }
  if ((threadIdx.x & 31) == 0) a.a[lrow] = af;
}

// destination row of a merged per-key gradient (MODE 3, requester side at W > 1): the owner o of key g
// holds a region of cap rows per source; this rank's key of rank ui in o's list goes to row
// rank*cap + ui there (peer memory over NVLink, or this rank's own buffer when o == rank)
__device__ __forceinline__ float *out_row3(const GradArgs &a, uint32_t ui, int D) {
  // ui = owner << OUT_OWNER_SHIFT | rank in the owner's list (written by the route); the hi row
  return a.p2p.peer_grecv[ui >> OUT_OWNER_SHIFT] + (size_t)((int64_t)a.p2p.rank * a.p2p.cap + (ui & OUT_POS_MASK)) * D;
}
// does the owner need the lo half of this key's partial (more than one rank sent the key)? The owner
// wrote the byte after its merge (p2p.cu k_lo_flags, LOF flag)
__device__ __forceinline__ bool need_lo(const GradArgs &a, uint32_t ui) {
  return a.lof[(int64_t)(ui >> OUT_OWNER_SHIFT) * a.p2p.cap + (ui & OUT_POS_MASK)] != 0;
}

// a merged per-key partial crosses the exchange as a double-float pair: hi = fp32(G) into the owner's
// hi region, lo = fp32(G - hi) into its lo region (lo_stride floats further) -- only when the owner
// receives the key from more than one rank: hi + lo carries ~48 bits, so partials of different ranks
// that cancel keep the fp64 result (an fp32 partial alone failed the tolerance on hot keys, reading
// R11''); a key with one source is applied from g = fp32(G) = hi anyway. ~80% of the keys at W = 2.
template <int CPL>
__device__ __forceinline__ void store_hilo(const GradArgs &a, float *dst_hi, const double (&g)[CPL], bool lo_too) {
  VecF<CPL> hi, lo;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    hi.v[c] = (float)g[c];
    lo.v[c] = (float)__dsub_rn(g[c], (double)hi.v[c]);
  }
  stg_frag<CPL>(dst_hi, hi);
  if (lo_too) stg_frag<CPL>(dst_hi + a.lo_stride, lo);
}

// the last CTA of the grid to finish raises the exchange flag: one system-scope fence per CTA, by the
// thread that counts the CTA in, after the barrier (the CTA's stores happen before it). A fence in
// every thread, then in every warp, made membar / ERRBAR the top stall of the requester pass (ncu,
// profiles/r02_ncu_w2_group*.txt).
__device__ __forceinline__ void grad_signal_last_cta(const GradArgs &a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t t = atomicAdd(a.p2p.done + a.signal_kind, 1u);
    if (t == gridDim.x - 1) {
      a.p2p.done[a.signal_kind] = 0;
      p2p_raise(a.p2p, a.signal_kind);
    }
  }
}

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// warp-parallel gallop: first (dir = -1) or last (dir = +1) position of the segment of key k that
// contains position p (all lanes call; one L2 round trip per 32x of distance)
__device__ int64_t seg_bound_warp(const uint32_t *skey, int64_t n, int64_t p, uint32_t k, int dir) {
  const int lane = threadIdx.x & 31;
  int64_t in = p;  // known inside the segment
  int64_t stride = 1;
  while (true) {  // gallop outwards until a probe leaves the segment
    const int64_t q = in + dir * (int64_t)(lane + 1) * stride;
    const bool out = q < 0 || q >= n || ld_cg_u32(skey + q) != k;
    const uint32_t m = __ballot_sync(0xffffffffu, out);
    if (m) {
      const int f = __ffs(m) - 1;  // probes 0..f-1 are inside
      in = in + dir * (int64_t)f * stride;
      if (stride == 1) return in;
      stride >>= 5;
      break;
    }
    in = in + dir * 32 * stride;
    stride <<= 5;
  }
  while (true) {  // refine inside (in, in + dir*32*stride]
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
template <int CPL, int MODE, bool PRECISE>
__device__ __noinline__ void span_piece(const GradArgs &a, const DAcc<CPL> acc, int64_t slot, int64_t pos,
                                        uint32_t key, int64_t R, int64_t n) {
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
  const int64_t first = seg_bound_warp(a.skey, n, pos, key, -1);
  const int64_t lastp = seg_bound_warp(a.skey, n, pos, key, +1);
  // the warp's partial stores happen before lane 0's release (syncwarp); the last arriver's acquire
  // happens before its lanes' partial loads (syncwarp after the broadcast). acq_rel atomics instead of
  // two gpu-scope fences per piece (ERRBAR stalls, profiles/r02_ncu_w2_group_b.txt).
  __syncwarp();
  int last = 0;
  const int64_t w0 = first / R, w1 = lastp / R;
  if (lane == 0) {
    const uint32_t t = atom_add_acq_rel(&a.tickets[first], 1u);
    last = (t == (uint32_t)(w1 - w0));
    if (last) a.tickets[first] = 0;  // ready for the next step (kernel boundary orders it)
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  __syncwarp();
  if (!last) return;
  if (MODE != 4 && !active) return;  // (row-wise Adagrad reduces over the whole warp)
  double tot[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) tot[c] = 0.0;
  for (int64_t ww = w0; ww <= w1 && active; ++ww) {
    const double *src = a.partials + (size_t)(ww == w0 ? 2 * ww + 1 : 2 * ww) * D + col;
#pragma unroll
    for (int c = 0; c < CPL; c += 2) {
      const double2 v = ld_cg_d2(reinterpret_cast<const double2 *>(src + c));
      tot[c] = __dadd_rn(tot[c], v.x);
      tot[c + 1] = __dadd_rn(tot[c + 1], v.y);
    }
  }
  if constexpr (MODE == 3) {
    const uint32_t ui = a.useg[pos];
    store_hilo<CPL>(a, out_row3(a, ui, D) + col, tot, need_lo(a, ui));
  } else if constexpr (MODE == 4) {
    const uint32_t lrow = key & a.lmask;
    const size_t off = (size_t)lrow * D + col;
    VecF<CPL> wv;
    if (active) ldg_frag<CPL>(wv, a.w + off);
    else wv.zero();
    const float a_old = __ldcg(a.a + lrow);
    apply_rowwise<CPL, PRECISE>(a, opt_const(a), tot, wv, a_old, off, lrow, active, D);
  } else {
    const size_t off = (size_t)(key & a.lmask) * D + col;
    VecF<CPL> wv, av;
    ldg_frag<CPL>(wv, a.w + off);
    if (MODE == 1) ldg_frag<CPL>(av, a.a + off);
    apply_frag<CPL, MODE, PRECISE>(a, opt_const(a), tot, wv, av, off);
  }
}

// per-lane metadata of one tile (lane i < T describes position t0 + i)
struct TileMeta {
  uint32_t key;   // sorted key (EMB_SENTINEL = invalid / beyond the range)
  int32_t len;    // bag length (mean pooling)
  uint32_t uo;    // MODE 3: rank of the key in its owner's list
  uint32_t lo;    // MODE 3: the owner needs the lo half (k_lo_flags)
  uint32_t vmask, hmask, tmask;  // warp-uniform: valid / head / tail
};

template <int CPL, int T, int NS, bool MEAN, int MODE, int DC, int MINB = 2, bool LO = false, bool PRECISE = false>
__global__ void __launch_bounds__(256, MINB) k_grad(const __grid_constant__ GradArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  // row arrays per stage: contribution (+ its low part, LO: owner side at W > 1), w, a
  constexpr int NA = ((MODE == 1) ? 3 : ((MODE == 0 || MODE == 4) ? 2 : 1)) + (LO ? 1 : 0);
  constexpr int OFF_W = (1 + (LO ? 1 : 0)) * T;  // stage offsets in rows of D floats
  constexpr int OFF_A = OFF_W + T;
  constexpr bool SINK_OPT = MODE < 2 || MODE == 4;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int D = DC ? DC : a.dim;  // compile-time row width for D = 64 / 128 / 256
  const int col = lane * CPL;
  const bool active = DC ? true : col < D;
  const int C16 = D >> 2;  // 16-byte chunks per row (a constant when DC != 0)
  const size_t stage_floats = (size_t)NA * T * D + (MODE == 4 ? T : 0);  // (+ T row accumulators)
  const uint32_t wbase = smem_u32(smem) + (uint32_t)(wib * NS * stage_floats * 4);
  const int64_t gw = ((int64_t)blockIdx.x * (blockDim.x >> 5)) + wib;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  // a step with an input error (any rank), a peer timeout or a tripped guard applies nothing; every
  // warp reads the same words, so the decision is grid-uniform and the last-warp signal still fires
  bool skip = a.skip_mask && (ld_cg_u32(a.err) & a.skip_mask);
  if (a.abort_bits)
    for (int s = 0; s < a.p2p.world; ++s) skip = skip || a.abort_bits[s] != 0;
  const int64_t n = skip ? 0 : (a.n_dev ? *a.n_dev : a.n);
  const int64_t R = (n + nwarps - 1) / nwarps;
  const int64_t p_lo = gw * R;
  const int64_t p_hi = (p_lo + R < n) ? p_lo + R : n;
  if (p_lo < p_hi) {  // (no early return: the end-of-grid signal below is CTA-collective)
  const float *src_base = a.src_mode == 0 ? a.dy : a.src;
  const OptConst oc = opt_const(a);

  bool seen_head = false;  // a head was issued earlier in this range (=> open pieces began here)
  uint32_t kprev_carry = p_lo > 0 ? a.skey[p_lo - 1] : EMB_SENTINEL;
  const uint32_t k_after = p_hi < n ? a.skey[p_hi] : EMB_SENTINEL;
  bool bad = false;
  const int64_t ntile = (p_hi - p_lo + T - 1) / T;

  auto load_kp = [&](int64_t j, uint32_t &k, uint32_t &pay) {
    const int64_t p = p_lo + j * T + lane;
    k = EMB_SENTINEL;
    pay = 0;
    if (j < ntile && lane < T && p < p_hi) {
      k = a.skey[p];
      pay = a.spay[p];
    }
  };
  auto load_row = [&](uint32_t k, uint32_t pay) -> uint32_t {
    if (k == EMB_SENTINEL) return 0;
    if (a.src_mode != 0) return pay;
    return pay < (uint64_t)a.nsrc_occ ? a.drow[pay] : 0xFFFFFFFEu;
  };
  // MODE 3: the key's rank in its owner's list, loaded with the source row (NS+1 tiles ahead: a load
  // consumed in the same tile stalled the warp for a full memory latency per tile)
  auto load_uo = [&](int64_t j) -> uint32_t {
    if (MODE != 3) return 0;
    const int64_t p = p_lo + j * T + lane;
    return (j < ntile && lane < T && p < p_hi) ? a.useg[p] : 0u;
  };
  // flags + async copies of tile j into stage s (keys k, source rows srow; knext_tile = first key of tile j+1)
  auto issue = [&](int64_t j, int s, TileMeta &m, uint32_t k, uint32_t srow, uint32_t uo_in, uint32_t knext_tile) {
    const int64_t t0 = p_lo + j * T;
    const int cnt = (int)((p_hi - t0) < T ? (p_hi - t0) : T);
    int32_t len = 1;
    uint32_t uo = 0, lo_flag = 0;
    if (k != EMB_SENTINEL) {
      if ((int64_t)srow >= a.nsrc) bad = true;
      else if (MEAN) len = a.blen[srow];
      if (SINK_OPT && (int64_t)(k & a.lmask) >= a.nrows) bad = true;
      if (!SINK_OPT) {
        uo = uo_in;
        if ((int64_t)(uo & OUT_POS_MASK) >= a.nout || (uo >> OUT_OWNER_SHIFT) >= (uint32_t)a.p2p.world) bad = true;
        else lo_flag = need_lo(a, uo);  // (consumed NS tiles later: the load is off the critical path)
      }
    }
    uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    if (lane == 0) kp = kprev_carry;
    uint32_t kn = __shfl_down_sync(0xffffffffu, k, 1);
    if (lane == cnt - 1) kn = (j + 1 < ntile) ? knext_tile : k_after;
    const bool valid = lane < cnt && k != EMB_SENTINEL && !bad;
    const bool head = valid && k != kp;
    const bool tail = valid && k != kn;
    m.vmask = __ballot_sync(0xffffffffu, valid);
    m.hmask = __ballot_sync(0xffffffffu, head);
    m.tmask = __ballot_sync(0xffffffffu, tail);
    const uint32_t le_mask = (lane < 31) ? ((2u << lane) - 1u) : 0xFFFFFFFFu;
    const bool applies = SINK_OPT && tail && (((m.hmask & le_mask) != 0) || seen_head);
    const uint32_t amask = __ballot_sync(0xffffffffu, applies);
    seen_head = seen_head || m.hmask != 0;
    kprev_carry = __shfl_sync(0xffffffffu, k, cnt - 1);
    m.key = k;
    m.len = len;
    m.uo = uo;
    m.lo = lo_flag;
    // async copies: chunk q = it*32 + lane of the tile's rows, row i = q / C16, 16-B chunk c = q % C16
    // (LO: the hi row, and the lo row only where the segment has more than one contribution)
    const uint32_t sb = wbase + (uint32_t)(s * stage_floats * 4);
    const uint32_t lomask = m.vmask & ~(m.hmask & m.tmask);
    for (int q0 = 0; q0 < T * C16; q0 += 32) {
      const int q = q0 + lane;
      const int i = q / C16, c = q - i * C16;
      const uint32_t ri = __shfl_sync(0xffffffffu, srow, i < T ? i : 0);
      const uint32_t off = (uint32_t)((i * D + c * 4) * 4);
      if (i < T && ((m.vmask >> i) & 1u)) cp_async16(sb + off, src_base + (size_t)ri * D + c * 4);
      if (LO && i < T && ((lomask >> i) & 1u))
        cp_async16(sb + (uint32_t)(T * D * 4) + off, src_base + a.lo_stride + (size_t)ri * D + c * 4);
    }
    if (SINK_OPT) {
      const unsigned long long wrow = (unsigned long long)(k & a.lmask) * D;
      for (int q0 = 0; q0 < T * C16; q0 += 32) {
        const int q = q0 + lane;
        const int i = q / C16, c = q - i * C16;
        const unsigned long long wri = __shfl_sync(0xffffffffu, wrow, i < T ? i : 0);
        const uint32_t off = (uint32_t)((i * D + c * 4) * 4);
        if (i < T && ((amask >> i) & 1u)) {
          cp_async16(sb + (uint32_t)(OFF_W * D * 4) + off, a.w + wri + c * 4);
          if (MODE == 1) cp_async16(sb + (uint32_t)(OFF_A * D * 4) + off, a.a + wri + c * 4);
        }
      }
    }
    if (MODE == 4 && lane < T && ((amask >> lane) & 1u))  // the row's accumulator (4 bytes)
      cp_async4(sb + (uint32_t)(OFF_A * D * 4) + 4u * (uint32_t)lane, a.a + (k & a.lmask));
  };

  TileMeta meta[NS];
  // prologue: keys of tiles 0..NS+1, rows of tiles 0..NS, copies of tiles 0..NS-1 (one group each)
  uint32_t kk[NS + 2], pp[NS + 2], rr[NS + 1], uu[NS + 1];
#pragma unroll
  for (int j = 0; j < NS + 2; ++j) load_kp(j, kk[j], pp[j]);
#pragma unroll
  for (int j = 0; j < NS + 1; ++j) {
    rr[j] = load_row(kk[j], pp[j]);
    uu[j] = load_uo(j);
  }
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    if (j < ntile) issue(j, j, meta[j], kk[j], rr[j], uu[j], __shfl_sync(0xffffffffu, kk[j + 1], 0));
    cp_async_commit();
  }
  // metadata slots by tile parity (NS even, tb a multiple of NS: the slot of tiles ti + NS and
  // ti + NS + 2 is s & 1, that of ti + NS + 1 the other one -- compile-time indices). A rotation
  // k2 = k3, k3 = k4 after the loads instead compiled to register moves that waited on the loads just
  // issued: 24% of k_grad's stall samples sat on two such moves (profiles/r02_ncu_w1_c2.txt).
  static_assert(NS % 2 == 0, "metadata slots assume an even stage count");
  uint32_t KS[2], PS[2], RS[2], US[2];
  KS[0] = kk[NS];
  RS[0] = rr[NS];
  US[0] = uu[NS];
  PS[0] = 0;
  KS[1] = kk[NS + 1];
  PS[1] = pp[NS + 1];
  RS[1] = 0;
  US[1] = 0;

  DAcc<CPL> acc;
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc.v[c] = 0.0;
  bool begins = false;  // the open piece began inside this warp's range
  bool open = false;
  int64_t open_pos = p_lo;
  uint32_t open_key = 0;

  bool broken = false;  // (the signal below must still fire: peers wait for it)
  for (int64_t tb = 0; tb < ntile && !broken; tb += NS) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {  // static stage index: the tile metadata stays in registers
      const int64_t ti = tb + s;
      if (ti >= ntile) break;
      const int64_t t0 = p_lo + ti * T;
      TileMeta &m = meta[s];
      cp_async_wait<NS - 1>();  // this lane's copies of tile ti have landed
      __syncwarp();             // ... and every other lane's
      if (__any_sync(0xffffffffu, bad)) {  // broken invariant (bug): report and stop, never apply garbage
        if (lane == 0) atomicOr(a.err, EMB_DEVERR_INTERNAL);
        broken = true;
        break;
      }
      const uint32_t sbase = wbase + (uint32_t)(s * stage_floats * 4) + 4u * (uint32_t)col;
      const uint32_t vmask = m.vmask, hmask = m.hmask, tmask = m.tmask;
      // a full tile inside one segment (no head, no tail: long hot-key segments, C5) only accumulates
      // -- without the per-position mask bookkeeping of the general walk below
      const bool plain = !MEAN && !LO && (hmask | tmask) == 0 && vmask == ((1u << T) - 1u);
      if (plain) {
#pragma unroll
        for (int i = 0; i < T; ++i) {
          VecF<CPL> v;
          if (active) lds_frag<CPL>(v, sbase + 4u * (uint32_t)(i * D));
          else v.zero();
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc.v[c] = __dadd_rn(acc.v[c], (double)v.v[c]);
        }
      }
#pragma unroll
      for (int i = 0; i < T && !plain; ++i) {  // compile-time positions: constant shared offsets
        if (!((vmask >> i) & 1u)) continue;
        const bool hd = (hmask >> i) & 1u;
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc.v[c] = hd ? 0.0 : acc.v[c];
        begins = begins || hd;
        VecF<CPL> v;
        if constexpr (LO) {  // a received per-key partial = hi (+ lo where the key has several sources)
          if (active) lds_frag<CPL>(v, sbase + 4u * (uint32_t)(i * D));
          else v.zero();
          if (!((hmask >> i) & (tmask >> i) & 1u)) {
            VecF<CPL> vl;
            if (active) lds_frag<CPL>(vl, sbase + 4u * (uint32_t)((T + i) * D));
            else vl.zero();
#pragma unroll
            for (int c = 0; c < CPL; ++c) acc.v[c] = __dadd_rn(__dadd_rn(acc.v[c], (double)v.v[c]), (double)vl.v[c]);
          } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c) acc.v[c] = __dadd_rn(acc.v[c], (double)v.v[c]);
          }
        } else if constexpr (MEAN) {
          if (active) lds_frag<CPL>(v, sbase + 4u * (uint32_t)(i * D));
          else v.zero();
          const int32_t li = __shfl_sync(0xffffffffu, m.len, i);
          const double dl = (double)li;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            acc.v[c] = __dadd_rn(acc.v[c], li > 1 ? __ddiv_rn((double)v.v[c], dl) : (double)v.v[c]);
        } else {
          if (active) lds_frag<CPL>(v, sbase + 4u * (uint32_t)(i * D));
          else v.zero();
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc.v[c] = __dadd_rn(acc.v[c], (double)v.v[c]);
        }
        if ((tmask >> i) & 1u) {
          const uint32_t ki = __shfl_sync(0xffffffffu, m.key, i);
          if (begins) {  // complete inside the range
            if constexpr (!SINK_OPT) {
              const uint32_t ui = __shfl_sync(0xffffffffu, m.uo, i);
              const bool lo_i = __shfl_sync(0xffffffffu, m.lo, i);
              if (active) store_hilo<CPL>(a, out_row3(a, ui, D) + col, acc.v, lo_i);
            } else if constexpr (MODE == 4) {
              VecF<CPL> wv;
              if (active) lds_frag<CPL>(wv, sbase + 4u * (uint32_t)((OFF_W + i) * D));
              else wv.zero();
              float a_old;
              const uint32_t sa_ = wbase + (uint32_t)(s * stage_floats * 4) + 4u * (uint32_t)(OFF_A * D + i);
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(a_old) : "r"(sa_));
              const uint32_t lrow = ki & a.lmask;
              apply_rowwise<CPL, PRECISE>(a, oc, acc.v, wv, a_old, (size_t)lrow * D + col, lrow, active, D);
            } else {
              if (active) {
                VecF<CPL> wv, av;
                lds_frag<CPL>(wv, sbase + 4u * (uint32_t)((OFF_W + i) * D));
                if (MODE == 1) lds_frag<CPL>(av, sbase + 4u * (uint32_t)((OFF_A + i) * D));
                apply_frag<CPL, MODE, PRECISE>(a, oc, acc.v, wv, av, (size_t)(ki & a.lmask) * D + col);
              }
            }
          } else {
            span_piece<CPL, MODE, PRECISE>(a, acc, 2 * gw, t0 + i, ki, R, n);  // continuation piece that ends here
          }
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc.v[c] = 0.0;
          begins = false;
        }
      }
      // a piece still open at the end of the tile: remember where it stands (used after the last tile)
      const uint32_t after_last_tail = tmask ? (vmask & ~((2u << (31 - __clz(tmask))) - 1u)) : vmask;
      if (after_last_tail) {
        const int lv = 31 - __clz(vmask);
        open = true;
        open_pos = t0 + lv;
        open_key = __shfl_sync(0xffffffffu, m.key, lv);
      } else if (tmask) {
        open = false;
      }
      __syncwarp();  // every lane is done reading the stage before it is refilled
      const int c = s & 1, o = c ^ 1;  // (s is the unrolled stage index: compile-time after unrolling)
      if (ti + NS < ntile) issue(ti + NS, s, m, KS[c], RS[c], US[c], __shfl_sync(0xffffffffu, KS[o], 0));
      cp_async_commit();  // (possibly empty) group keeps the wait_group accounting uniform
      // advance the metadata pipeline: rows of tile ti+NS+1, keys of tile ti+NS+2
      RS[o] = load_row(KS[o], PS[o]);
      US[o] = load_uo(ti + NS + 1);
      load_kp(ti + NS + 2, KS[c], PS[c]);
    }
  }
  cp_async_wait<0>();
  if (open && !broken) span_piece<CPL, MODE, PRECISE>(a, acc, begins ? 2 * gw + 1 : 2 * gw, open_pos, open_key, R, n);  // continues past the range
  }  // p_lo < p_hi
  if (a.signal_kind >= 0) grad_signal_last_cta(a);
}

static int g_sms = 0;

template <int CPL, int T, int NS, bool MEAN, int MODE, int DC, int MINB = 2, bool LO = false, bool PRECISE = false>
static cudaError_t launch_grad_t(const GradArgs &a, cudaStream_t st) {
  constexpr int NA = ((MODE == 1) ? 3 : ((MODE == 0 || MODE == 4) ? 2 : 1)) + (LO ? 1 : 0);
  const size_t per_warp = (size_t)NS * ((size_t)NA * T * a.dim + (MODE == 4 ? T : 0)) * sizeof(float);
  int wpc = (int)(110 * 1024 / per_warp);  // warps per CTA: ~110 KB of stages, 2 CTAs per SM
  if (wpc > 8) wpc = 8;
  if (wpc < 1) wpc = 1;
  const size_t smem = per_warp * wpc;
  static size_t attr[EMB_MAX_DEVICES] = {};  // per device: the attribute is a per-context setting
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= EMB_MAX_DEVICES) return cudaErrorInvalidDevice;
  if (attr[dev] < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(k_grad<CPL, T, NS, MEAN, MODE, DC, MINB, LO, PRECISE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[dev] = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_grad<CPL, T, NS, MEAN, MODE, DC, MINB, LO, PRECISE>, wpc * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)g_sms * per_sm;
  // >= 1 tile per warp: small inputs (C1: 18K positions) spread over more warps instead of walking
  // 4+ tiles' latency chains each; large ones fill the resident grid anyway
  const int64_t max_blocks = ((a.n + T - 1) / T + wpc - 1) / wpc;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  k_grad<CPL, T, NS, MEAN, MODE, DC, MINB, LO, PRECISE><<<(unsigned)blocks, wpc * 32, smem, st>>>(a);
  return cudaGetLastError();
}

template <int CPL, int T, int DC>
static cudaError_t launch_grad_d(const GradArgs &a, cudaStream_t st) {
  const bool mean = a.blen != nullptr;
  const int mode = a.sink_mode == 2 ? 3 : (a.opt == 1 ? 1 : (a.opt == 2 ? 4 : 0));
  if (mean) {
    if (mode == 0) return launch_grad_t<CPL, T, 2, true, 0, DC>(a, st);
    if (mode == 1) return launch_grad_t<CPL, T, 2, true, 1, DC>(a, st);
    if (mode == 4) return launch_grad_t<CPL, T, 2, true, 4, DC>(a, st);
    return launch_grad_t<CPL, T, 2, true, 3, DC>(a, st);
  }
  if (a.src_lo) {  // owner side at W > 1: double-float received partials
    if (mode == 0) return launch_grad_t<CPL, T, 2, false, 0, DC, 2, true>(a, st);
    if (mode == 1) return launch_grad_t<CPL, T, 2, false, 1, DC, 2, true>(a, st);
    if (mode == 4) return launch_grad_t<CPL, T, 2, false, 4, DC, 2, true>(a, st);
    return cudaErrorInvalidValue;
  }
  if (mode == 0) return launch_grad_t<CPL, T, 2, false, 0, DC>(a, st);
  if (mode == 1) return launch_grad_t<CPL, T, 2, false, 1, DC>(a, st);
  if (mode == 4) return launch_grad_t<CPL, T, 2, false, 4, DC>(a, st);
  return launch_grad_t<CPL, T, 2, false, 3, DC>(a, st);
}

template <int CPL, int T>
static cudaError_t launch_grad_precise(const GradArgs &a, int mode, cudaStream_t st) {
  const bool mean = a.blen != nullptr;
  if (a.src_lo) {
    if (mode == 1) return launch_grad_t<CPL, T, 2, false, 1, 0, 2, true, true>(a, st);
    return launch_grad_t<CPL, T, 2, false, 4, 0, 2, true, true>(a, st);
  }
  if (mean) {
    if (mode == 1) return launch_grad_t<CPL, T, 2, true, 1, 0, 2, false, true>(a, st);
    return launch_grad_t<CPL, T, 2, true, 4, 0, 2, false, true>(a, st);
  }
  if (mode == 1) return launch_grad_t<CPL, T, 2, false, 1, 0, 2, false, true>(a, st);
  return launch_grad_t<CPL, T, 2, false, 4, 0, 2, false, true>(a, st);
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
  const int mode = a.sink_mode == 2 ? 3 : (a.opt == 1 ? 1 : (a.opt == 2 ? 4 : 0));
  if ((mode == 1 || mode == 4) && a.lr > 1.0) {  // fp64 Adagrad sinks (OptConst): generic-D kernels
    if (a.dim <= 64) return launch_grad_precise<2, 8>(a, mode, st);
    if (a.dim <= 128) return launch_grad_precise<4, 8>(a, mode, st);
    return launch_grad_precise<8, 8>(a, mode, st);
  }
  if (a.dim == 64) return launch_grad_d<2, 8, 64>(a, st);
  if (a.dim == 128) return launch_grad_d<4, 8, 128>(a, st);
  if (a.dim == 256) return launch_grad_d<8, 8, 256>(a, st);
  if (a.dim <= 64) return launch_grad_d<2, 8, 0>(a, st);
  if (a.dim <= 128) return launch_grad_d<4, 8, 0>(a, st);
  return launch_grad_d<8, 8, 0>(a, st);
}

}  // namespace emb
