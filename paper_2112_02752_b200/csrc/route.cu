// route.cu — shard routing for world > 1 (readings R5-R7).
//
//  * k_route (A3 + A4 fused): one pass over the rank's sorted fused keys (segments = distinct keys).
//    Tiles of 4096 positions, claimed in launch order through a ticket (forward progress for the
//    look-back); a warp walks 8 rows of 32 consecutive positions. Per row, MATCH.ANY groups the lanes
//    by owner and a ballot marks the segment heads, so each lane knows how many heads of its owner
//    precede it in the row; per-warp and per-tile counts of heads per owner give the exclusive base
//    (warp prefix in shared memory, tile prefix by a decoupled look-back over W counters, one lane per
//    owner). A position's key then has rank `sendpos` among this rank's distinct keys of that owner
//    (ascending g). Outputs: outidx per sorted position (the row of the merged gradient in the owner's
//    region), inv per occurrence (the row the owner pushes back), the head's local id into the owner's
//    receive region (peer store). The last block publishes the per-owner
//    counts and this rank's input-error bits into every owner's xmat and raises KEYS.
//  * k_merge_pass (A5): the owner receives W runs (source s at region s*cap), each sorted by local id;
//    a stable merge tree (ceil(log2 W) passes of pairwise merge-path merges, ties keep the lower
//    source rank) gives the owner's merged order. Per pass a CTA owns TILE outputs of one merged run:
//    two merge-path diagonals found by warp-parallel 32-ary searches (4 dependent L2 round trips
//    instead of ~17 for a serial binary search), the A / B windows staged in shared memory, then
//    per-thread searches and sequential merges there.
#include "../../include/emb.h"
#include "common.cuh"
#include "internal.h"
#include "p2p_dev.cuh"

namespace emb {

namespace {
constexpr int RT_THREADS = 512;
constexpr int RT_WARPS = RT_THREADS / 32;
constexpr int RT_ROWS = 8;                      // rows of 32 positions per warp
constexpr int RT_TILE = RT_THREADS * RT_ROWS;   // 4096 positions per CTA
constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_VAL = (1u << 30) - 1u;
}  // namespace

size_t route_status_words(int64_t max_n) { return (size_t)((max_n + RT_TILE - 1) / RT_TILE + 1) * P2P_MAXW; }

__device__ __forceinline__ unsigned lanemask_le() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

__global__ void __launch_bounds__(RT_THREADS) k_route(const __grid_constant__ RouteArgs a) {
  __shared__ uint32_t s_tile, s_last;
  __shared__ uint32_t wcnt[RT_WARPS][P2P_MAXW];  // per (warp, owner) head counts -> running bases
  __shared__ uint32_t s_excl[P2P_MAXW];          // heads of each owner in earlier tiles
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int W = a.p2p.world;
  const int64_t cap = a.p2p.cap;
  if (tid == 0) {
    s_tile = atomicAdd(a.counter, 1u);
    if (s_tile == gridDim.x - 1) *a.counter = 0;  // last ticket: ready for the next launch
  }
  if (tid < RT_WARPS * P2P_MAXW) (&wcnt[0][0])[tid] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t w0 = tile * RT_TILE + (int64_t)w * 32 * RT_ROWS;
  uint32_t key[RT_ROWS], pay[RT_ROWS];  // (payloads loaded up front: pass 2's scattered stores need them)
#pragma unroll
  for (int r = 0; r < RT_ROWS; ++r) {
    const int64_t p = w0 + r * 32 + lane;
    key[r] = p < a.n ? a.skey[p] : EMB_SENTINEL;
    pay[r] = p < a.n ? a.spay[p] : 0u;
  }
  const uint32_t k_before = (lane == 0 && w0 > 0 && w0 - 1 < a.n) ? a.skey[w0 - 1] : EMB_SENTINEL;
  // head / owner of the lane's position in row r (warp-collective)
  auto row_info = [&](int r, bool &valid, bool &head, uint32_t &o, uint32_t &peers, uint32_t &hb) {
    uint32_t prev = __shfl_up_sync(0xffffffffu, key[r], 1);
    const uint32_t prev_row_last = __shfl_sync(0xffffffffu, r > 0 ? key[r > 0 ? r - 1 : 0] : 0u, 31);
    if (lane == 0) prev = r == 0 ? k_before : prev_row_last;
    valid = key[r] != EMB_SENTINEL;
    head = valid && key[r] != prev;
    o = valid ? owner_of_g(key[r], a.ks) : 0u;
    peers = __match_any_sync(0xffffffffu, valid ? o : 0x100u + lane);
    hb = __ballot_sync(0xffffffffu, head);
  };
  // ---- pass 1: heads per owner for this warp
#pragma unroll
  for (int r = 0; r < RT_ROWS; ++r) {
    bool valid, head;
    uint32_t o, peers, hb;
    row_info(r, valid, head, o, peers, hb);
    if (valid && lane == __ffs(peers) - 1) wcnt[w][o] += __popc(peers & hb);
    __syncwarp();
  }
  __syncthreads();
  // ---- per owner (warp o): exclusive prefix over the warps, tile aggregate, decoupled look-back over
  // earlier tiles, 32 predecessors per probe (tiles finish pass 1 at about the same time, so a
  // one-tile-at-a-time walk would chain ~#tiles dependent L2 reads)
  if (w < W) {
    const int o = w;
    const uint32_t c = lane < RT_WARPS ? wcnt[lane][o] : 0u;
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
    if (lane < RT_WARPS) wcnt[lane][o] = incl - c;
    const unsigned long long tag = (unsigned long long)a.tag << 32;
    volatile unsigned long long *st = reinterpret_cast<volatile unsigned long long *>(a.status);
    if (lane == 0) st[tile * P2P_MAXW + o] = tag | (tile == 0 ? LB_INC : LB_AGG) | agg;
    uint32_t excl = 0;
    if (tile > 0) {
      int64_t look = tile - 1;
      while (true) {
        const int64_t t = look - lane;  // lane l probes tile look - l
        unsigned long long sv = 0;
        if (t >= 0) {
          do {
            sv = st[t * P2P_MAXW + o];
          } while ((sv >> 32) != a.tag || ((uint32_t)sv & ~LB_VAL) == 0);
        }
        const bool inc = t < 0 || ((uint32_t)sv & LB_INC);
        const uint32_t m = __ballot_sync(0xffffffffu, inc);
        const int last = m ? __ffs(m) - 1 : 31;  // nearest inclusive predecessor ends the walk
        uint32_t v = (lane <= last && t >= 0) ? ((uint32_t)sv & LB_VAL) : 0u;
#pragma unroll
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        excl += v;
        if (m) break;
        look -= 32;
      }
      if (lane == 0) st[tile * P2P_MAXW + o] = tag | LB_INC | (excl + agg);
    }
    if (lane == 0) {
      s_excl[o] = excl;
      if (agg) atomicAdd(a.tot + o, agg);
    }
  }
  __syncthreads();
  // ---- pass 2: ranks, outputs, peer stores of the heads' local ids
  const int parity_off = (int)(a.p2p.epoch & 1u);
  bool bad = false;
#pragma unroll
  for (int r = 0; r < RT_ROWS; ++r) {
    bool valid, head;
    uint32_t o, peers, hb;
    row_info(r, valid, head, o, peers, hb);
    const int64_t p = w0 + r * 32 + lane;
    const uint32_t same = peers & hb;
    if (p < a.n) {
      uint32_t sp = EMB_SENTINEL;
      if (valid) {
        const uint32_t incl = __popc(same & lanemask_le());
        const int64_t pos = (int64_t)s_excl[o] + wcnt[w][o] + incl - 1;  // the segment head's rank
        if (pos < 0 || pos >= cap) {
          bad = true;
        } else {
          sp = (o << OUT_OWNER_SHIFT) | (uint32_t)pos;  // owner in the top bits (no division downstream)
          a.inv[pay[r]] = (uint32_t)(o * cap + pos);
          if (head)
            a.p2p.peer_recv_keys[o][(int64_t)parity_off * W * cap + (int64_t)a.p2p.rank * cap + pos] =
                local_of_g(key[r], a.ks);
        }
      }
      a.outidx[p] = sp;
    }
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[w][o] += __popc(same);
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err, EMB_DEVERR_INTERNAL);
  // ---- the last block publishes the counts + error bits and raises KEYS (one system fence per block,
  // after the barrier: per-thread fences made membar the top stall, profiles/r02_ncu_w2_group.txt)
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    s_last = atomicAdd(a.blk_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (tid == 0) *a.blk_done = 0;
  if (tid < W) {
    const int o = tid;
    const int64_t c = atomicExch(a.tot + o, 0u);
    a.scnt[o] = c;
    uint32_t eb = ld_cg_u32(a.err) & (EMB_DEVERR_RANGE | EMB_DEVERR_INVALID);
    if (a.extra_err) {
      eb |= a.extra_err;
      if (o == 0) atomicOr(a.err, a.extra_err);
    }
    a.p2p.peer_xmat[o][xmat_idx(a.p2p.epoch, 0, a.p2p.rank)] = c;
    a.p2p.peer_xmat[o][xmat_idx(a.p2p.epoch, 1, a.p2p.rank)] = eb;
  }
  __syncthreads();
  if (tid == 0) p2p_raise(a.p2p, P2P_KEYS);
}

cudaError_t launch_route(const RouteArgs &a, cudaStream_t st) {
  // at least one block: with no ids the per-owner counts must still be published (zeros) and KEYS raised
  const int64_t tiles = a.n > 0 ? (a.n + RT_TILE - 1) / RT_TILE : 1;
  k_route<<<(unsigned)tiles, RT_THREADS, 0, st>>>(a);
  return cudaGetLastError();
}

// ---- merge tree
namespace {
constexpr int MP_THREADS = 256;
constexpr int MP_ITEMS = 8;
constexpr int MP_TILE = MP_THREADS * MP_ITEMS;  // outputs per CTA
}  // namespace

// number of A items among the first d outputs of the stable merge of A (first) and B: the first i in
// [max(0, d-n), min(d, m)] with A[i] > B[d-1-i] (or the upper end). Warp-collective 32-ary search.
__device__ int64_t merge_path_warp(const uint32_t *A, int64_t m, const uint32_t *B, int64_t n, int64_t d) {
  const int lane = threadIdx.x & 31;
  int64_t lo = d > n ? d - n : 0, hi = d < m ? d : m;
  while (lo < hi) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t i = lo + (int64_t)lane * step;
    const bool f = i < hi && A[i] > B[d - 1 - i];  // predicate "A[i] <= B[d-1-i]" is false at i
    const uint32_t m_ = __ballot_sync(0xffffffffu, f);
    if (m_ == 0) {
      const int last = (int)((hi - 1 - lo) / step);  // last probed lane
      lo = lo + (int64_t)last * step + 1;
    } else {
      const int fl = __ffs(m_) - 1;
      const int64_t ifl = lo + (int64_t)fl * step;
      if (fl == 0) return ifl;
      hi = ifl;
      lo = lo + (int64_t)(fl - 1) * step + 1;
    }
  }
  return lo;
}

// pass with width w (= 2^r): input run q covers sources [q*w, (q+1)*w); pass 0 reads source q's region
// at q*cap (payload = receive position q*cap + i), later passes the compact previous output at P[q*w].
// Output run j = stable merge of input runs 2j (A) and 2j+1 (B), written compactly at P[2j*w].
__global__ void __launch_bounds__(MP_THREADS) k_merge_pass(const uint32_t *__restrict__ ik,
                                                           const uint32_t *__restrict__ ip,
                                                           const int64_t *__restrict__ counts, int W, int64_t cap,
                                                           int w, uint32_t *__restrict__ ok, uint32_t *__restrict__ op,
                                                           int64_t *n_merged) {
  __shared__ int64_t P[P2P_MAXW + 1];
  __shared__ uint32_t sk[MP_TILE], sp[MP_TILE];
  __shared__ int64_t s_i0, s_i1;
  const int tid = threadIdx.x;
  if (tid == 0) {
    P[0] = 0;
    for (int r = 0; r < W; ++r) P[r + 1] = P[r] + counts[r];
    if (n_merged && blockIdx.x == 0) *n_merged = P[W];
  }
  __syncthreads();
  const int nruns = (W + 2 * w - 1) / (2 * w);
  // grid-stride over the (output run, tile) pairs of all runs
  for (int64_t gt = blockIdx.x;; gt += gridDim.x) {
    int j = -1;
    int64_t tile = gt;
    for (int q = 0; q < nruns; ++q) {
      const int64_t len = P[min(W, (2 * q + 2) * w)] - P[min(W, 2 * q * w)];
      const int64_t nt = (len + MP_TILE - 1) / MP_TILE;
      if (tile < nt) {
        j = q;
        break;
      }
      tile -= nt;
    }
    if (j < 0) return;  // block-uniform
    const int qa = 2 * j, qb = 2 * j + 1;
    const int64_t m = P[min(W, (qa + 1) * w)] - P[min(W, qa * w)];
    const int64_t n = P[min(W, (qb + 1) * w)] - P[min(W, qb * w)];
    const int64_t a0 = w == 1 ? (int64_t)qa * cap : P[min(W, qa * w)];
    const int64_t b0 = w == 1 ? (int64_t)min(qb, W - 1) * cap : P[min(W, qb * w)];
    const int64_t d0 = tile * MP_TILE, d1 = min(d0 + MP_TILE, m + n);
    const int wid = tid >> 5;
    if (wid == 0) {
      const int64_t i0 = merge_path_warp(ik + a0, m, ik + b0, n, d0);
      if ((tid & 31) == 0) s_i0 = i0;
    } else if (wid == 1) {
      const int64_t i1 = merge_path_warp(ik + a0, m, ik + b0, n, d1);
      if ((tid & 31) == 0) s_i1 = i1;
    }
    __syncthreads();
    const int64_t i0 = s_i0, i1 = s_i1;
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
      const int64_t o = P[min(W, qa * w)] + d0 + dd;  // merged run j starts where its A run starts
      for (int q = 0; q < MP_ITEMS && dd + q < tot; ++q) {
        const bool takeA = ib >= nb || (ia < na && sk[ia] <= sk[na + ib]);
        const int src = takeA ? ia : na + ib;
        ok[o + q] = sk[src];
        op[o + q] = sp[src];
        if (takeA) ++ia;
        else ++ib;
      }
    }
    __syncthreads();  // the windows are refilled by the next tile
  }
}

cudaError_t launch_merge_tree(const uint32_t *rkeys, const int64_t *counts, int W, int64_t cap, uint32_t *ok0,
                              uint32_t *op0, uint32_t *ok1, uint32_t *op1, int64_t *n_merged, cudaStream_t st) {
  int passes = 0;
  while ((1 << passes) < W) ++passes;
  int64_t blocks = (W * cap + MP_TILE - 1) / MP_TILE + W;  // >= sum over runs of their tiles
  if (blocks > 148 * 4) blocks = 148 * 4;                      // (grid-stride beyond that)
  const uint32_t *ik = rkeys, *ip = nullptr;
  for (int r = 0; r < passes; ++r) {
    const bool to0 = ((passes - 1 - r) & 1) == 0;  // the last pass lands in (ok0, op0)
    uint32_t *ok = to0 ? ok0 : ok1, *op = to0 ? op0 : op1;
    k_merge_pass<<<(unsigned)blocks, MP_THREADS, 0, st>>>(ik, ip, counts, W, cap, 1 << r, ok, op,
                                                          r == 0 ? n_merged : nullptr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ik = ok;
    ip = op;
  }
  return cudaSuccess;
}

}  // namespace emb
