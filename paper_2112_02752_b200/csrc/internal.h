// internal.h — host-side declarations shared by the libemb translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int EMB_MAX_DEVICES = 64;  // per-device launch-attribute caches

namespace emb {

// Sharding / key-space parameters (R7). Every sorted key is the FUSED row g = base[t] + id (< 2^32):
//   owner(g) = g mod W, local(g) = g div W          (cyclic, the default)
//   owner(g) = g div rows_per, local(g) = g mod rows_per   (block)
// At W == 1 owner = 0 and local = g.
struct KeySpace {
  int32_t world;
  int32_t rank;
  int32_t shard;       // 0 cyclic, 1 block
  uint32_t rows_per;   // block sharding: ceil(R_total / W)
  uint32_t key_bits;   // bits the general radix sort must look at (sentinel strictly above every valid key)
};

__host__ __device__ __forceinline__ uint32_t owner_of_g(uint32_t g, const KeySpace &ks) {
  if (ks.world == 1) return 0;
  return ks.shard == 0 ? g % (uint32_t)ks.world : g / ks.rows_per;
}
__host__ __device__ __forceinline__ uint32_t local_of_g(uint32_t g, const KeySpace &ks) {
  if (ks.world == 1) return g;
  return ks.shard == 0 ? g / (uint32_t)ks.world : g % ks.rows_per;
}

// kernel ids for the per-kernel event profiler (order = emb_profile_name)
enum KernelId {
  KID_KEYS = 0,
  KID_SORT_HIST,
  KID_SORT_PASS,
  KID_POOL,
  KID_GRAD_APPLY,
  KID_UNIQUE,
  KID_ROUTE,
  KID_GATHER_PUSH,
  KID_GRAD_PUSH,
  KID_SIGNAL,
  KID_INIT,
  KID_MERGE,
  KID_WAIT,
  KID_LOFLAGS,
  KID_COUNT
};

// ---- world > 1 exchange over peer memory (p2p.cu, route.cu) ----------------------------------------
// Every rank owns fixed per-source regions of `cap` entries (cap = max over ranks of max_ids) in its
// receive buffers, so a source writes its keys / gradients without first learning where the other
// sources' runs end. Flags are per-(kind, source) epoch words raised in every peer; a wait requires
// EXACTLY the expected epoch (a rank that fell behind times out instead of reading stale buffers).
constexpr int P2P_MAXW = 16;  // == EMB_MAX_WORLD
enum { P2P_KEYS = 0, P2P_ROWS = 1, P2P_GRADS = 2, P2P_LOF = 3, P2P_NKIND = 4 };
// xmat layout (int64): [parity][0][s] = keys received from source s, [parity][1][s] = input-error
// bits of source s in this step (parity = epoch & 1: double-buffered, a fast peer may already write
// step e+1 while this rank still reads step e)
__host__ __device__ __forceinline__ int xmat_idx(uint64_t epoch, int which, int s) {
  return (int)(epoch & 1u) * 2 * P2P_MAXW + which * P2P_MAXW + s;
}
struct P2PArgs {
  int32_t world, rank;
  uint64_t epoch;
  int64_t cap;                          // entries per source region
  uint64_t *flags;                      // own [P2P_NKIND][P2P_MAXW]
  uint32_t *done;                       // own [P2P_NKIND] finished-block counters (last block raises)
  int64_t *xmat;                        // own [2][2][P2P_MAXW]
  uint64_t *peer_flags[P2P_MAXW];
  int64_t *peer_xmat[P2P_MAXW];
  uint32_t *peer_recv_keys[P2P_MAXW];   // [2][W * cap] owner-local ids, region s = source s
  float *peer_grecv[P2P_MAXW];          // [2][W * cap][D] merged per-key gradients as double-float:
                                        // hi rows, then lo rows; region s = source s
  uint8_t *peer_lof[P2P_MAXW];          // [W * cap] requester side: does owner o need the lo half of
                                        // my key of rank i (region o, written by owner o)
  float *peer_uniq_rows[P2P_MAXW];      // [W * cap][D] rows received by the requester, region o = owner o
};
// wait (one thread, bounded) until every source raised `kind` with exactly `epoch`
cudaError_t launch_wait(const P2PArgs &a, int kind, uint64_t epoch, uint32_t *err, cudaStream_t st);
// raise `kind` in every peer (a producer with nothing to do); err_bits != 0 are first OR-ed into every
// owner's error slot of this step (xmat[parity][1][rank]): the owners then skip the update
cudaError_t launch_signal(const P2PArgs &a, int kind, uint32_t err_bits, cudaStream_t st);
// OR `bits` into the sticky device error word
cudaError_t launch_mark_err(uint32_t *err, uint32_t bits, cudaStream_t st);
// owner (A6 + X2 fused): for every source s != rank and i < xmat[s] (keys received from s this step),
// the table row of local id recv_keys[s*cap + i] is stored straight into requester s's row region for
// this owner, peer_uniq_rows[s][rank*cap + i] (peer stores over NVLink); the last block raises ROWS.
// (Peer LOADS through CUDA-IPC mappings measured 19 GB/s against 600 GB/s for peer stores,
// profiles/r02_ipc_gather_bench.log, so rows are pushed by the owner, not pulled by the requester.)
cudaError_t launch_gather_push(const P2PArgs &a, const float *w, const uint32_t *recv_keys, const int64_t *counts,
                               int dim, int64_t rows_local, uint32_t *err, cudaStream_t st);
// owner, after its merge: for every received key, whether another rank sent the same key (its merged
// neighbours): that byte into the requester's lof region for this owner; the last block raises LOF
// fin != nullptr: the later of this kernel and the pool publishes the error word (PoolArgs::fin)
cudaError_t launch_lo_flags(const P2PArgs &a, const uint32_t *okey, const uint32_t *opay, const int64_t *n_merged,
                            int64_t max_n, uint32_t *fin, uint32_t *err, uint32_t *err_host, cudaStream_t st);

// A3+A4 fused (route.cu): over the sorted fused keys, per distinct key (segment head) its owner o and
// its rank `sendpos` among this rank's distinct keys owned by o (ascending g); the head's local id is
// stored straight into owner o's receive region; per sorted position outidx = sendpos; per
// occurrence inv = o*cap + sendpos (the row owner o pushes back). The last block publishes the
// per-owner counts and this rank's input-error bits into every owner's xmat and raises KEYS.
// outidx of a sorted position: owner << OUT_OWNER_SHIFT | rank in that owner's list (cap < 2^28)
constexpr uint32_t OUT_OWNER_SHIFT = 28;
constexpr uint32_t OUT_POS_MASK = (1u << OUT_OWNER_SHIFT) - 1u;
struct RouteArgs {
  const uint32_t *skey, *spay;
  int64_t n;
  KeySpace ks;
  P2PArgs p2p;
  uint32_t *outidx;       // [n] owner << OUT_OWNER_SHIFT | sendpos
  uint32_t *inv;          // [max_ids] by occurrence
  int64_t *scnt;          // [P2P_MAXW] out
  uint32_t *tot;          // [P2P_MAXW] zero on entry, left zero
  uint64_t *status;       // [tiles][P2P_MAXW] look-back words (epoch-tagged: no per-launch memset)
  uint32_t *counter;      // tile ticket, self-resetting
  uint32_t *blk_done;     // finished-block counter, self-resetting
  uint32_t tag;           // distinct per launch, never 0
  uint32_t *err;          // device sticky error word
  uint32_t extra_err;     // host-detected argument error bits of this call (published + made sticky)
};
size_t route_status_words(int64_t max_n);
cudaError_t launch_route(const RouteArgs &a, cudaStream_t st);

// ---- launchers (each returns cudaGetLastError()) ------------------------------------------------
struct KeysArgs {
  const int64_t *ids;
  const int64_t *offsets;
  int64_t nnz;
  int32_t batch;
  int32_t num_slots;
  const int32_t *slot_table;  // device [S]
  const uint64_t *base;       // device [T]
  const int64_t *rows;        // device [T]
  uint32_t *key;     // out [nnz] fused key g = base[t] + id, or EMB_SENTINEL
  uint32_t *drow;    // out [nnz] output row index b*S+s of the occurrence's bag (row of Y and dY)
  int32_t *blen;     // out [B*S] bag length, indexed by output row b*S+s
  uint32_t *err;     // sticky device error word
};
cudaError_t launch_keys(const KeysArgs &a, cudaStream_t st);

// stable LSD radix sort of (key, value) pairs on the low `key_bits` bits. Input (kin, vin) is left
// untouched; vin == nullptr means value = index. Result lands in (*keys_out, *vals_out), one of the
// two scratch pairs (k0, v0) / (k1, v1).
struct SortWorkspace {
  uint32_t *hist;      // [4][256]
  uint32_t *counters;  // [4]
  uint32_t *status;    // [4][max_tiles][256]
  int64_t max_tiles;
  uint32_t *err;       // sticky device error word (internal bounds guard)
};
size_t sort_workspace_words(int64_t max_n);
typedef void (*ProfHook)(void *ctx, int kid, int end, cudaStream_t st);
cudaError_t radix_sort_pairs(const SortWorkspace &ws, const uint32_t *kin, const uint32_t *vin, uint32_t *k0,
                             uint32_t *v0, uint32_t *k1, uint32_t *v1, int64_t n, uint32_t key_bits,
                             cudaStream_t st, uint32_t **keys_out, uint32_t **vals_out, int *launches,
                             ProfHook prof, void *prof_ctx);

// forward pool: Y[b][s][:] = sum (mean) over the bag's rows. A row g owned by this rank is read from
// the table shard at local(g); at W > 1 a row owned by another rank from the rows its owner pushed.
struct PoolArgs {
  // direct mode (ids != nullptr, monotone slot -> table map): the pool validates the CSR and ids
  // itself, computes g = base[t] + id, and writes the per-occurrence dY row index (drow) and bag
  // lengths (blen). Key mode (general sort path): g from `key` (the key kernel did all that).
  const int64_t *ids;      // [nnz] (direct mode) or nullptr
  const int32_t *slot_table;
  const uint64_t *base;
  const int64_t *rows;
  uint32_t *drow;          // out (direct mode) [nnz]
  int32_t *blen;           // out (direct mode) [B*S] or nullptr
  const uint32_t *key;     // [nnz] fused keys in CSR order (EMB_SENTINEL = skip), key mode
  const int64_t *offsets;  // [S*B+1]
  int64_t nnz;
  int32_t batch, num_slots, dim;
  int32_t mean;
  KeySpace ks;
  const float *rows_src;   // the table shard
  int64_t nrows_src;       // rows_local (bounds guard)
  const float *rows_remote;  // W > 1: rows pushed by their owners [W*cap][D]
  int64_t nrows_remote;      // W * cap (bounds guard)
  const uint32_t *row_idx; // W > 1: inv (occurrence -> o*cap + sendpos) for rows owned elsewhere
  int32_t bags_per_tile;   // 32 or 8 bags per warp tile (launch_pool sets it)
  float *out;
  uint32_t *err;           // device error word
  uint32_t *err_host;      // mapped pinned host word
  uint32_t *fin;           // [3] finish counters (pool blocks, other kernel's blocks, kernels) or nullptr:
                           // when set, the last of the fin_kernels concurrently running kernels (pool +
                           // segsort at W = 1) publishes err to err_host
  uint32_t fin_kernels;
};
cudaError_t launch_pool(const PoolArgs &a, cudaStream_t st);
cudaError_t launch_publish_err(const uint32_t *err, uint32_t *err_host, cudaStream_t st);

// backward: segment reduce over sorted (key, pay) + sink
struct GradArgs {
  const uint32_t *skey;    // [n] sorted keys (EMB_SENTINEL = invalid, skipped anywhere)
  const uint32_t *spay;    // [n] payload (occurrence index j, or receive position)
  int64_t n;               // positions (upper bound when n_dev is set: sizes the grid)
  int32_t dim;
  // contribution source: mode 0 = dY rows via drow/blen; mode 1 = rows of `src` at index spay
  int32_t src_mode;
  const float *dy;         // [B][S][D]
  const uint32_t *drow;    // [nnz] dY row index b*S+s per occurrence
  int64_t nsrc_occ;        // entries of drow (bounds guard)
  const int32_t *blen;     // [B*S] bag length by dY row (mean) or nullptr
  int32_t batch, num_slots;
  const float *src;        // mode 1
  const float *src_lo;     // non-null (W > 1 owner side): src rows are double-float partials, the lo
                           // rows lo_stride floats after the hi rows (grad.cu store_hilo)
  int64_t lo_stride;       // floats from a hi row to its lo row (W * cap * D)
  const uint8_t *lof;      // sink 2: per (owner, rank) "the owner needs the lo half" bytes
  // sink: 0 = optimizer apply on table rows (row = key & lmask); 2 = the merged fp32 row stored
  // straight into the owner's gradient region through peer memory (requester side at W > 1)
  int32_t sink_mode;
  const int64_t *n_dev;    // if set, the number of sorted positions is read from the device
  int32_t signal_kind;     // >= 0: the last warp to finish raises this p2p flag in every peer
  P2PArgs p2p;             // sink mode 2 / signal
  KeySpace ks;             // sink mode 2: owner of the key
  // skip the whole pass (still signalling) when (*err & skip_mask) != 0 or any abort_bits[s] != 0,
  // s < W: a step with an input error on any rank updates nothing (errors)
  uint32_t skip_mask;
  const int64_t *abort_bits;
  uint32_t lmask;
  int32_t opt;             // 0 sgd 1 adagrad 2 row-wise adagrad (a: one float per row)
  double lr, eps;
  float *w, *a;
  int64_t nrows;           // rows of w/a (bounds guard)
  int64_t nsrc;            // rows of dy (S*B) or src (bounds guard)
  int64_t nout;            // sink 2: entries of a region (cap, bounds guard)
  uint32_t *err;
  const uint32_t *useg;    // sink 2: per sorted position, the key's rank in its owner's list (outidx)
  double *partials;        // [2 * max resident warps][D]
  uint32_t *tickets;       // [>= n], zero on entry, left zero
};
cudaError_t launch_grad(const GradArgs &a, cudaStream_t st);
int64_t grad_max_warps(int dev);

// dedup of sorted keys: useg[p] = unique index of valid sorted position p, ukey[u], segment
// [ustart[u], uend[u]) (multiplicity = uend - ustart), *u_count = U (device). Sentinel positions
// (anywhere) are skipped.
struct UniqueArgs {
  const uint32_t *skey;
  int64_t n;
  uint32_t *useg, *ukey, *ustart, *uend, *u_count;
  uint64_t *status;  // [tiles] look-back words tagged with `epoch` (stale words of earlier launches
                     // read as "not ready": no per-launch memset)
  uint32_t *counter; // tile ticket; zero before the first launch, reset by the last tile
  uint32_t epoch;    // distinct per launch on the same status buffer (caller increments, never 0)
};
size_t unique_status_words(int64_t max_n);
cudaError_t launch_unique(const UniqueArgs &a, cudaStream_t st);

// table init (R15) and row helpers
cudaError_t launch_init(float *w, float *a, int32_t a_per_row, int64_t rows_local, int32_t dim, uint64_t seed,
                        float init_accum, const KeySpace &ks, int32_t rank, cudaStream_t st);
cudaError_t launch_rows_gather(const float *src, const int64_t *rows, int64_t n, int32_t dim, float *dst,
                               cudaStream_t st);
cudaError_t launch_rows_scatter(float *dst, const int64_t *rows, int64_t n, int32_t dim, const float *src,
                                cudaStream_t st);

// per-table stable sort (world == 1 fast path), see segsort.cu
// ids of one table group staged in shared memory by every sort CTA of the group (above: read from
// global memory in both scans). 20,480 covers C1's single group (~18.4K ids: 16,384 left it unstaged,
// 36 us per sort); 8,192 x 16 B of range buffers + 80 KB + 17 KB static = 225 KB of the 227 KB per CTA
constexpr int64_t SEG_CAP = 20480;
constexpr int64_t SEG_BIG = 65536;  // average ids per table group above which the general sort path runs
struct SegSortArgs {
  const int64_t *ids;       // [nnz] table-local ids in CSR order (validated here: out of range = invalid)
  const int64_t *offsets;   // [S*B+1]
  int64_t nnz;
  int32_t batch;
  const int32_t *gslot;     // [G+1] slot boundaries of the table groups
  int32_t ngroups;          // G
  const uint64_t *gbase;    // [G] first fused key of the group's table
  const uint32_t *grows;    // [G] rows of the group's table
  const uint32_t *gbits;    // [G] bits covering [0, rows] (rows = the invalid marker)
  uint32_t *skey, *spay;    // out [nnz]
  uint32_t *scratch_k, *scratch_a, *scratch_b;  // [nnz] global buffers for chunks above the smem cap
  uint32_t *run_k, *run_i;  // [nnz] sorted runs (local key, chunk-relative index)
  int32_t K;                // chunks (CTAs) per group
  int32_t validate;         // check the CSR offsets + fill uncovered positions (W > 1; the pool does it at W = 1)
  int32_t route;            // W > 1: the final write fused with k_route's work (rt; CTAs in ticket order)
  RouteArgs rt;
  uint32_t *err;
  uint32_t *err_host;       // with fin: see PoolArgs::fin
  uint32_t *fin;
};
cudaError_t launch_segsort(const SegSortArgs &a, int32_t groups, cudaStream_t st);
// owner side: stable merge of the W received runs (source s's run at s*cap, length counts[s], each
// sorted by local id) into (ok0, op0): keys and receive positions s*cap + i, ties in source-rank order
// (ceil(log2 W) merge-path passes); writes the merged length to *n_merged
cudaError_t launch_merge_tree(const uint32_t *rkeys, const int64_t *counts, int W, int64_t cap, uint32_t *ok0,
                              uint32_t *op0, uint32_t *ok1, uint32_t *op1, int64_t *n_merged, cudaStream_t st);

}  // namespace emb
