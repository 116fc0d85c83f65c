// segsort.cu — per-table stable sort of the step's keys (dedup by sorting), the fast
// path of the world == 1 step.
//
// When slot_table is non-decreasing (true for every BASELINE config: C1/C4 share one table, C2/C3/C5
// map slot s -> table s), the slot-major CSR is already grouped by table and the table groups appear
// in fused-key order, so sorting the whole array is the same as sorting each group in place.
//
// One kernel, K CTAs per table group (v3; v1 = one CTA per group, issue-bound on 26 of 148 SMs; v2 =
// chunk sorts + a K-way merge by ranking, search-bound; v4 = one 1024-thread CTA per group with
// per-thread 4-bit digit counters, 98 vs 57 us, dropped):
//  * CTA (g, b) owns the b-th of K equal ranges of the table's local-id space (bucket(local) =
//    (local * mul) >> 32, monotone, mul = floor(2^32 K / (rows + 1))). Each warp scans a contiguous
//    1/16 of the group's keys twice: once to count its items below / inside the range (ballots), then
//    -- after a block scan of the per-warp counts -- to compact the range's items into shared memory
//    in occurrence order. The range's output offset is the number of group items in lower ranges.
//  * the compacted items (local id, occurrence index) are sorted with a stable LSD radix sort on the
//    group's key bits (24 bits = 3 passes of 8 for a 10M-row table): per pass, per-warp digit counts
//    (shared-memory atomics over the warp's contiguous sub-chunk), a digit-major scan of the
//    (digit, warp) counters, then a stable scatter ranked by a warp multisplit (peer masks from one
//    MATCH.ANY per 32-item row; 8 ballots before: sort alone 40 -> 37 us, step time unchanged because
//    the concurrent pool then takes the freed issue slots);
//  * items are written straight to their final sorted positions: no merge.
// Ranges above SEG_CHUNK_CAP items run the same code on global scratch (correct, slower). Invalid
// occurrences (EMB_SENTINEL) get local key rows[t] and sort to the end of their group.
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"
#include "p2p_dev.cuh"

#ifndef EMB_SEG_MATCH
#define EMB_SEG_MATCH 1
#endif

namespace emb {

namespace {
constexpr int SS_THREADS = 512;
constexpr int SS_WARPS = SS_THREADS / 32;
constexpr uint32_t SEG_CHUNK_CAP = 8192;  // items per range sorted in shared memory (128 KB)
}  // namespace

// lanes of the warp holding the same 8-bit digit as this lane (8 ballots)
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool valid) {
#if EMB_SEG_MATCH
  // one MATCH.ANY instead of 8 ballots (invalid lanes get a value no valid lane has)
  const uint32_t m = __match_any_sync(0xffffffffu, valid ? d : 0x100u + (threadIdx.x & 31));
  return valid ? m : 0u;
#else
  uint32_t m = __ballot_sync(0xffffffffu, valid);
  if (!valid) m = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return m;
#endif
}

// bits needed for values 0..x
__device__ __forceinline__ uint32_t bits_span(uint32_t x) { return x ? 32u - __clz(x) : 0u; }

__device__ __forceinline__ void group_bounds(const SegSortArgs &a, int g, int64_t &lo, int64_t &hi) {
  const int64_t B = a.batch;
  lo = a.offsets[(int64_t)a.gslot[g] * B];
  hi = a.offsets[(int64_t)a.gslot[g + 1] * B];
  lo = lo < 0 ? 0 : (lo > a.nnz ? a.nnz : lo);
  hi = hi < lo ? lo : (hi > a.nnz ? a.nnz : hi);
}
// the sorted key range of one CTA: items in sorted order are keys[pa[i]] (table-local ids; `rows` =
// invalid) with occurrence glo + ia[pa[i]], at sorted positions pos0 + i, i < n
struct SortedRange {
  bool redo = false;  // SMEM pass only: the range exceeds the shared-memory buffers (run the global one)
  uint32_t n = 0;
  int64_t pos0 = 0, glo = 0;
  const uint32_t *keys = nullptr, *pa = nullptr, *ia = nullptr;
  uint32_t base = 0, rows = 0;
};

// SMEM: the range's buffers are in shared memory (n <= SEG_CHUNK_CAP, else it returns redo), so every
// access compiles to LDS / STS; a runtime choice between shared and global buffers made them all
// generic LD / ST. !SMEM: global scratch (oversized ranges, rare).
// the body's static shared memory, one copy for both instantiations
struct SortShared {
  uint32_t cnt[SS_WARPS][256];
  uint32_t part[SS_THREADS / 32];
  uint32_t wbelow[SS_WARPS], wmine[SS_WARPS];
  uint32_t kmin, kmax;  // key span of the range (the radix passes sort key - min)
};
__device__ __forceinline__ SortShared &sort_shared() {
  __shared__ SortShared ss;
  return ss;
}

template <bool SMEM>
__device__ __forceinline__ SortedRange segsort_range_body(const SegSortArgs &a, int work) {
  extern __shared__ __align__(16) uint32_t sm[];
  SortShared &ss = sort_shared();
  auto &cnt = ss.cnt;
  auto &part = ss.part;
  auto &wbelow = ss.wbelow;
  auto &wmine = ss.wmine;
  uint32_t &s_kmin = ss.kmin;
  uint32_t &s_kmax = ss.kmax;
  SortedRange out;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int K = a.K;
  const int g = work / K, bkt = work % K;
  // CSR validation (R4; before any early return; W > 1 only -- at W = 1 the concurrent pool validates):
  // CTA (g, bkt) checks the bkt-th 1/K slice of its group's bags, so every input error is known before
  // the route publishes it. CTA (0, 0) also checks both ends and marks sorted positions no group covers
  // (only with broken offsets) as invalid, so nothing stale from an earlier step is ever routed.
  if (a.validate) {
    const int64_t B = a.batch;
    const int64_t nb_all = (int64_t)a.gslot[a.ngroups] * B;
    const int64_t b_lo = (int64_t)a.gslot[g] * B, b_hi = (int64_t)a.gslot[g + 1] * B;
    const int64_t per = (b_hi - b_lo + K - 1) / K;
    const int64_t s0 = b_lo + per * bkt, s1 = min(b_hi, s0 + per);
    bool bad = false;
    for (int64_t i = s0 + tid; i < s1; i += SS_THREADS) {
      const int64_t o0 = a.offsets[i], o1 = a.offsets[i + 1];
      bad |= o0 < 0 || o1 < o0 || o1 > a.nnz;
    }
    if (work == 0) {
      const int64_t first = a.offsets[0], last = a.offsets[nb_all];
      if (tid == 0) bad |= first != 0 || last != a.nnz;
      const int64_t f = first < 0 ? 0 : (first > a.nnz ? a.nnz : first);
      int64_t l = last < f ? f : (last > a.nnz ? a.nnz : last);
      for (int64_t i = tid; i < f; i += SS_THREADS) a.skey[i] = EMB_SENTINEL;
      for (int64_t i = l + tid; i < a.nnz; i += SS_THREADS) a.skey[i] = EMB_SENTINEL;
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(a.err, EMB_DEVERR_INVALID);
  }
  int64_t glo, ghi;
  group_bounds(a, g, glo, ghi);
  const uint32_t ng = (uint32_t)(ghi - glo);
  if (ng == 0) return out;
  const uint32_t base = (uint32_t)a.gbase[g];
  const uint32_t rows = a.grows[g];
  const uint32_t bits = a.gbits[g];
  // bucket(lk) = floor(lk * mul / 2^32), mul = floor(2^32 K / (rows + 1)) < 2^32: one IMAD.HI, monotone
  const uint32_t mul = (uint32_t)((((uint64_t)K) << 32) / ((uint64_t)rows + 1u));
  // table-local id; invalid ids (R4) become `rows` and sort to the end of the group
  auto local_of = [&](int64_t id) { return (id >= 0 && id < (int64_t)rows) ? (uint32_t)id : rows; };
  auto bucket_of = [&](uint32_t lk) {
    const uint32_t b = __umulhi(lk, mul);
    return b < (uint32_t)K ? b : (uint32_t)K - 1u;
  };
  // stage the whole group's local ids in shared memory once (both scans below read them twice)
  const bool staged = ng <= (uint32_t)SEG_CAP;
  uint32_t *gk = sm + 4 * SEG_CHUNK_CAP;  // [SEG_CAP] after the range buffers
  if (staged) {
    // 16-byte loads (two ids each), all of a thread's loads in flight before the first store: 8-byte
    // loads four deep made this staging ~12% of the kernel's stall samples (profiles/r02_ncu_sort_*.txt).
    // Clamped (unpredicated) loads, as in k_pool.
    const int64_t *src = a.ids + glo;
    const uint32_t h = min((uint32_t)(((uintptr_t)src >> 3) & 1u), ng);  // a leading id to reach 16-B alignment
    const uint32_t npair = (ng - h) / 2;
    if (tid == 0) {
      if (h) gk[0] = local_of(src[0]);
      if ((ng - h) & 1u) gk[ng - 1] = local_of(src[ng - 1]);
    }
    if (npair > 0) {
      const longlong2 *src2 = reinterpret_cast<const longlong2 *>(src + h);
      constexpr int U = 16;
      for (uint32_t p0 = tid; p0 < npair; p0 += SS_THREADS * U) {
        longlong2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(src2 + min(p0 + (uint32_t)u * SS_THREADS, npair - 1u));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t p = p0 + (uint32_t)u * SS_THREADS;
          if (p < npair) {
            gk[h + 2 * p] = local_of(v[u].x);
            gk[h + 2 * p + 1] = local_of(v[u].y);
          }
        }
      }
    }
    __syncthreads();
  }
  auto key_at = [&](uint32_t i) -> uint32_t { return staged ? gk[i] : local_of(a.ids[glo + i]); };
  // ---- 1. count: items below / inside this range, per warp over a contiguous 1/16 of the group
  const uint32_t span = ((ng + SS_WARPS - 1) / SS_WARPS + 31) / 32 * 32;
  const uint32_t s_lo = w * span, s_hi = min(ng, s_lo + span);
  uint32_t below = 0, mine = 0;
  bool badid = false;
  for (uint32_t r0 = s_lo; r0 < s_hi; r0 += 32) {
    const uint32_t i = r0 + lane;
    uint32_t bb = 0xFFFFFFFFu;
    if (i < s_hi) {
      const uint32_t lk = key_at(i);
      badid |= lk == rows;
      bb = bucket_of(lk);
    }
    below += __popc(__ballot_sync(0xffffffffu, bb < (uint32_t)bkt));
    mine += __popc(__ballot_sync(0xffffffffu, bb == (uint32_t)bkt));
  }
  if (bkt == 0 && __any_sync(0xffffffffu, badid) && lane == 0) atomicOr(a.err, EMB_DEVERR_RANGE);  // (R4)
  if (lane == 0) {
    wbelow[w] = below;
    wmine[w] = mine;
  }
  if (tid == 0) {
    s_kmin = 0xFFFFFFFFu;
    s_kmax = 0u;
  }
  __syncthreads();
  uint32_t out_lo = 0, my_start = 0, n = 0;
  for (int q = 0; q < SS_WARPS; ++q) {
    out_lo += wbelow[q];
    if (q < w) my_start += wmine[q];
    n += wmine[q];
  }
  if (n == 0) return out;
  uint32_t *keys, *ia, *ib;
  if (SMEM) {
    if (n > SEG_CHUNK_CAP) {
      out.redo = true;
      return out;
    }
    keys = sm;
    ia = sm + n;
    ib = sm + 2 * n;
  } else {  // oversized range: global scratch at the range's own output slice
    keys = a.scratch_k + glo + out_lo;
    ia = a.scratch_a + glo + out_lo;
    ib = a.scratch_b + glo + out_lo;
  }
  // ---- 2. compact the range's items in occurrence order: keys[] = local id, ia[] = group index
  uint32_t kmin_l = 0xFFFFFFFFu, kmax_l = 0u;
  {
    uint32_t cur = my_start;
    for (uint32_t r0 = s_lo; r0 < s_hi; r0 += 32) {
      const uint32_t i = r0 + lane;
      uint32_t lk = 0;
      bool in = false;
      if (i < s_hi) {
        lk = key_at(i);
        in = bucket_of(lk) == (uint32_t)bkt;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      if (in) {
        const uint32_t d = cur + __popc(m & lanemask_lt());
        keys[d] = lk;
        ia[d] = i;
        kmin_l = min(kmin_l, lk);
        kmax_l = max(kmax_l, lk);
      }
      cur += __popc(m);
    }
    kmin_l = __reduce_min_sync(0xffffffffu, kmin_l);
    kmax_l = __reduce_max_sync(0xffffffffu, kmax_l);
    if (lane == 0) {
      atomicMin(&s_kmin, kmin_l);
      atomicMax(&s_kmax, kmax_l);
    }
  }
  __syncthreads();
  // ---- 3. stable LSD radix sort of the n compacted items (ia holds the payload, permuted by value)
  const uint32_t chunk = ((n + SS_WARPS - 1) / SS_WARPS + 31) / 32 * 32;  // rows of 32 per warp
  const uint32_t c_lo = w * chunk;
  const uint32_t c_hi = min(n, c_lo + chunk);
  // passes over the range's actual key span (a few thousand values per range at C1: 2 passes instead
  // of the table's 3)
  const uint32_t kmin = s_kmin;
  const int npass = (int)((min(bits, bits_span(s_kmax - kmin)) + 7) / 8);
  // sort item ordinals 0..n-1 (ping-pong pa/pb); keys[] and ia[] stay in place
  uint32_t *pa = ib;
  uint32_t *pb = SMEM ? sm + 3 * n : a.run_k + glo + out_lo;
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = 8 * pass;
    for (int d = lane; d < 256; d += 32) cnt[w][d] = 0;
    __syncwarp();
    for (uint32_t p = c_lo + lane; p < c_hi; p += 32) {
      const uint32_t item = pass == 0 ? p : pa[p];
      atomicAdd(&cnt[w][((keys[item] - kmin) >> shift) & 0xFFu], 1u);
    }
    __syncthreads();
    {
      const int d = tid >> 1, w0 = (tid & 1) * 8;
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += cnt[w0 + q][d];
      const uint32_t incl = warp_incl_scan(s);
      if (lane == 31) part[w] = incl;
      __syncthreads();
      if (w == 0) {
        const uint32_t t = lane < SS_THREADS / 32 ? part[lane] : 0;
        const uint32_t ti = warp_incl_scan(t);
        if (lane < SS_THREADS / 32) part[lane] = ti - t;
      }
      __syncthreads();
      uint32_t run = part[w] + incl - s;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t cc = cnt[w0 + q][d];
        cnt[w0 + q][d] = run;
        run += cc;
      }
    }
    __syncthreads();
    for (uint32_t r0 = c_lo; r0 < c_hi; r0 += 32) {
      const uint32_t p = r0 + lane;
      const bool valid = p < c_hi;
      const uint32_t item = valid ? (pass == 0 ? p : pa[p]) : 0u;
      const uint32_t d = valid ? ((keys[item] - kmin) >> shift) & 0xFFu : 0u;
      const uint32_t peers = digit_peers(d, valid);
      const int leader = valid ? __ffs(peers) - 1 : 0;
      uint32_t basepos = 0;
      if (valid && lane == leader) {
        basepos = cnt[w][d];
        cnt[w][d] = basepos + __popc(peers);
      }
      basepos = __shfl_sync(0xffffffffu, basepos, leader);
      if (valid) {
        const uint32_t dst = basepos + __popc(peers & lanemask_lt());
        if (dst < n) pb[dst] = item;
        else atomicOr(a.err, EMB_DEVERR_INTERNAL);
      }
      __syncwarp();
    }
    __syncthreads();
    uint32_t *t = pa;
    pa = pb;
    pb = t;
  }
  if (npass == 0) {  // (a 0-bit group -- rows = 1 -- keeps the identity order)
    for (uint32_t i = tid; i < n; i += SS_THREADS) pa[i] = i;
    __syncthreads();
  }
  out.n = n;
  out.pos0 = glo + out_lo;
  out.glo = glo;
  out.keys = keys;
  out.pa = pa;
  out.ia = ia;
  out.base = base;
  out.rows = rows;
  return out;
}

// ---- 4. final positions: group offset of the range + rank
__device__ __forceinline__ void segsort_write(const SegSortArgs &a, const SortedRange &r) {
  for (uint32_t i = threadIdx.x; i < r.n; i += SS_THREADS) {
    const uint32_t item = r.pa[i];
    const uint32_t lk = r.keys[item];
    a.skey[r.pos0 + i] = (lk >= r.rows) ? EMB_SENTINEL : r.base + lk;
    a.spay[r.pos0 + i] = (uint32_t)(r.glo + r.ia[item]);
  }
}

// ---- 4' (W > 1): the final write fused with the route (route.cu k_route, same outputs): the CTAs
// take their (group, range) in ticket order, which is sorted-position order, so each CTA's per-owner
// head counts get their exclusive prefix by a decoupled look-back over the earlier CTAs. A range's
// first item is always a segment head (ranges partition a table's key space).
__device__ __forceinline__ void segsort_route(const SegSortArgs &a, const SortedRange &r, int work) {
  const RouteArgs &ra = a.rt;
  __shared__ uint32_t wcnt[SS_WARPS][P2P_MAXW];
  __shared__ uint32_t s_excl[P2P_MAXW];
  __shared__ uint32_t s_last;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int W = ra.p2p.world;
  const int64_t cap = ra.p2p.cap;
  if (tid < SS_WARPS * P2P_MAXW) (&wcnt[0][0])[tid] = 0;
  __syncthreads();
  // warp w: items [w*per, (w+1)*per) in rows of 32, per a multiple of 32
  const uint32_t per = ((r.n + SS_WARPS - 1) / SS_WARPS + 31) / 32 * 32;
  const uint32_t i_lo = w * per, i_hi = min(r.n, i_lo + per);
  auto info = [&](uint32_t i, uint32_t &lk, bool &valid, bool &head, uint32_t &o) {
    lk = i < i_hi ? r.keys[r.pa[i]] : r.rows;
    valid = i < i_hi && lk < r.rows;
    const uint32_t prev = (i > 0 && i < i_hi) ? r.keys[r.pa[i - 1]] : 0xFFFFFFFFu;
    head = valid && (i == 0 || lk != prev);
    o = valid ? owner_of_g(r.base + lk, ra.ks) : 0u;
  };
  // pass 1: heads per owner for this warp
  for (uint32_t r0 = i_lo; r0 < i_hi; r0 += 32) {
    uint32_t lk, o;
    bool valid, head;
    info(r0 + lane, lk, valid, head, o);
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? o : 0x100u + lane);
    const uint32_t hb = __ballot_sync(0xffffffffu, head);
    if (valid && lane == __ffs(peers) - 1) wcnt[w][o] += __popc(peers & hb);
    __syncwarp();
  }
  __syncthreads();
  // per owner (warp o): prefix over warps, aggregate, look-back over the earlier CTAs (32 per probe)
  if (w < W) {
    const int o = w;
    const uint32_t c = lane < SS_WARPS ? wcnt[lane][o] : 0u;
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
    if (lane < SS_WARPS) wcnt[lane][o] = incl - c;
    const unsigned long long tag = (unsigned long long)ra.tag << 32;
    constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_VAL = (1u << 30) - 1u;
    volatile unsigned long long *st = reinterpret_cast<volatile unsigned long long *>(ra.status);
    if (lane == 0) st[(int64_t)work * P2P_MAXW + o] = tag | (work == 0 ? LB_INC : LB_AGG) | agg;
    uint32_t excl = 0;
    if (work > 0) {
      int64_t look = work - 1;
      while (true) {
        const int64_t t = look - lane;
        unsigned long long sv = 0;
        if (t >= 0) {
          do {
            sv = st[t * P2P_MAXW + o];
          } while ((sv >> 32) != ra.tag || ((uint32_t)sv & ~LB_VAL) == 0);
        }
        const bool inc = t < 0 || ((uint32_t)sv & LB_INC);
        const uint32_t m = __ballot_sync(0xffffffffu, inc);
        const int last = m ? __ffs(m) - 1 : 31;
        uint32_t v = (lane <= last && t >= 0) ? ((uint32_t)sv & LB_VAL) : 0u;
#pragma unroll
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        excl += v;
        if (m) break;
        look -= 32;
      }
      if (lane == 0) st[(int64_t)work * P2P_MAXW + o] = tag | LB_INC | (excl + agg);
    }
    if (lane == 0) {
      s_excl[o] = excl;
      if (agg) atomicAdd(ra.tot + o, agg);
    }
  }
  __syncthreads();
  // pass 2: sorted keys / payloads, ranks, peer stores of the heads' local ids
  const int64_t parity_off = (int64_t)(ra.p2p.epoch & 1u) * W * cap;
  bool bad = false;
  for (uint32_t r0 = i_lo; r0 < i_hi; r0 += 32) {
    const uint32_t i = r0 + lane;
    uint32_t lk, o;
    bool valid, head;
    info(i, lk, valid, head, o);
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? o : 0x100u + lane);
    const uint32_t same = peers & __ballot_sync(0xffffffffu, head);
    if (i < i_hi) {
      const int64_t p = r.pos0 + i;
      const uint32_t occ = (uint32_t)(r.glo + r.ia[r.pa[i]]);
      a.skey[p] = valid ? r.base + lk : EMB_SENTINEL;
      a.spay[p] = occ;
      uint32_t sp = EMB_SENTINEL;
      if (valid) {
        const uint32_t incl = __popc(same & ((2u << lane) - 1u));
        const int64_t pos = (int64_t)s_excl[o] + wcnt[w][o] + incl - 1;
        if (pos < 0 || pos >= cap) {
          bad = true;
        } else {
          sp = (o << OUT_OWNER_SHIFT) | (uint32_t)pos;
          ra.inv[occ] = (uint32_t)(o * cap + pos);
          if (head)
            ra.p2p.peer_recv_keys[o][parity_off + (int64_t)ra.p2p.rank * cap + pos] = local_of_g(r.base + lk, ra.ks);
        }
      }
      ra.outidx[p] = sp;
    }
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[w][o] += __popc(same);
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(ra.err, EMB_DEVERR_INTERNAL);
  // the last CTA publishes the counts + error bits and raises KEYS (one system fence per CTA)
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    s_last = atomicAdd(ra.blk_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (tid == 0) *ra.blk_done = 0;
  if (tid < W) {
    const int o = tid;
    const int64_t c = atomicExch(ra.tot + o, 0u);
    ra.scnt[o] = c;
    uint32_t eb = ld_cg_u32(ra.err) & (EMB_DEVERR_RANGE | EMB_DEVERR_INVALID);
    if (ra.extra_err) {
      eb |= ra.extra_err;
      if (o == 0) atomicOr(ra.err, ra.extra_err);
    }
    ra.p2p.peer_xmat[o][xmat_idx(ra.p2p.epoch, 0, ra.p2p.rank)] = c;
    ra.p2p.peer_xmat[o][xmat_idx(ra.p2p.epoch, 1, ra.p2p.rank)] = eb;
  }
  __syncthreads();
  if (tid == 0) p2p_raise(ra.p2p, P2P_KEYS);
}

__global__ void __launch_bounds__(SS_THREADS) k_segsort_range(const __grid_constant__ SegSortArgs a) {
  int work = blockIdx.x;
  if (a.route) {  // ticket order = sorted-position order (forward progress of the look-back)
    __shared__ uint32_t s_work;
    if (threadIdx.x == 0) {
      s_work = atomicAdd(a.rt.counter, 1u);
      if (s_work == gridDim.x - 1) *a.rt.counter = 0;
    }
    __syncthreads();
    work = (int)s_work;
  }
  const SortedRange r = segsort_range_body<true>(a, work);  // (block-uniform)
  if (!r.redo) {
    if (a.route) {
      __syncthreads();
      segsort_route(a, r, work);
    } else {
      segsort_write(a, r);
    }
  } else {  // (validation and staging repeat: idempotent)
    __syncthreads();
    const SortedRange rg = segsort_range_body<false>(a, work);
    if (a.route) {
      __syncthreads();
      segsort_route(a, rg, work);
    } else {
      segsort_write(a, rg);
    }
  }
  if (a.fin) {
    __syncthreads();
    if (threadIdx.x == 0) finish_publish(a.fin + 1, a.fin + 2, 2, a.err, a.err_host);
  }
}

size_t segsort_smem_bytes() { return (size_t)SEG_CHUNK_CAP * 16 + (size_t)SEG_CAP * 4; }

cudaError_t launch_segsort(const SegSortArgs &a, int32_t groups, cudaStream_t st) {
  if (groups <= 0 || a.nnz <= 0 || a.batch <= 0) return cudaSuccess;
  static bool attr[EMB_MAX_DEVICES] = {};  // per device: the attribute is a per-context setting
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= EMB_MAX_DEVICES) return cudaErrorInvalidDevice;
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_segsort_range, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)segsort_smem_bytes());
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  k_segsort_range<<<groups * a.K, SS_THREADS, segsort_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

}  // namespace emb
