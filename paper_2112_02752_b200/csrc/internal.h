// internal.h — host-side declarations shared by the libemb translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int EMB_MAX_DEVICES = 64;  // per-device launch-attribute caches

namespace emb {

// Sharding / key-space parameters (R7). The ROUTING KEY of a fused row g is
//   W == 1 : rk = g
//   W  > 1 : rk = owner(g) << lbits | local(g)
// so sorting routing keys groups the unique keys by owner, ascending local id within an owner.
struct KeySpace {
  int32_t world;
  int32_t rank;
  int32_t shard;       // 0 cyclic, 1 block
  uint32_t lbits;      // bits of the local row id (W > 1)
  uint64_t rows_per;   // block sharding: ceil(R_total / W)
  uint32_t key_bits;   // bits the radix sort must look at (sentinel strictly above every valid key)
};

__host__ __device__ inline uint32_t route_key(uint64_t g, const KeySpace &ks) {
  if (ks.world == 1) return (uint32_t)g;
  uint64_t owner, local;
  if (ks.shard == 0) {
    owner = g % (uint64_t)ks.world;
    local = g / (uint64_t)ks.world;
  } else {
    owner = g / ks.rows_per;
    local = g % ks.rows_per;
  }
  return (uint32_t)((owner << ks.lbits) | local);
}
__host__ __device__ inline uint64_t key_to_global(uint32_t rk, const KeySpace &ks) {
  if (ks.world == 1) return rk;
  uint64_t owner = rk >> ks.lbits, local = rk & ((1u << ks.lbits) - 1u);
  return ks.shard == 0 ? local * (uint64_t)ks.world + owner : owner * ks.rows_per + local;
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
  KID_OWNER_GATHER,
  KID_GRAD_LOCAL,
  KID_NCCL,
  KID_INIT,
  KID_MERGE,
  KID_WAIT,
  KID_COUNT
};

// ---- world > 1 peer-memory exchange (p2p.cu) ------------------------------------------------------
constexpr int P2P_MAXW = 16;  // == EMB_MAX_WORLD
enum { P2P_COUNTS = 0, P2P_KEYS = 1, P2P_ROWS = 2, P2P_GRADS = 3, P2P_NKIND = 4 };
struct RouteTable {               // device-resident, rebuilt every step from the count matrix
  int64_t soff[P2P_MAXW + 1];     // my send buffer: start of owner d's keys
  int64_t roff[P2P_MAXW + 1];     // my receive buffer: start of source s's run
  int64_t dst_off[P2P_MAXW];      // where my keys / gradients start in owner d's receive buffer
  int64_t src_off[P2P_MAXW];      // where my rows start in requester s's row buffer
  int64_t recv_counts[P2P_MAXW];
  int64_t n_recv, n_send;
};
struct P2PArgs {
  int32_t world, rank;
  uint64_t epoch;
  uint64_t *flags;                 // own [P2P_NKIND][P2P_MAXW]
  int64_t *xmat;                   // own [W][W]
  RouteTable *rt;
  uint32_t *done;                  // own [P2P_NKIND] finished-block counters (last block raises the flag)
  int64_t *peer_xmat[P2P_MAXW];
  uint64_t *peer_flags[P2P_MAXW];
  uint32_t *peer_recv_keys[P2P_MAXW];
  float *peer_uniq_rows[P2P_MAXW];
  float *peer_grecv[P2P_MAXW];
};
cudaError_t launch_push_rows(const P2PArgs &a, const float *rows, int dim, int64_t cap, cudaStream_t st);
cudaError_t launch_xcounts(const P2PArgs &a, const int64_t *send_counts, uint32_t *err, cudaStream_t st);
// device helpers (p2p_dev.cuh): the producing kernels (push_keys, gather_push, grad MODE 3) raise
// their exchange flag from their last block / warp
cudaError_t launch_signal(const P2PArgs &a, int kind, cudaStream_t st);
cudaError_t launch_wait(const P2PArgs &a, int kind, uint32_t *err, cudaStream_t st);
cudaError_t launch_push_keys(const P2PArgs &a, const uint32_t *send_keys, int64_t cap, cudaStream_t st);
cudaError_t launch_gather_push(const P2PArgs &a, const float *w, const uint32_t *recv_keys, int dim, int64_t cap,
                               int64_t rows_local, uint32_t *err, cudaStream_t st);

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
  KeySpace ks;
  uint32_t *key;     // out [nnz] routing key or EMB_SENTINEL
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

// W == 1 forward: Y[b][s][:] = pool over bag of table rows, straight from the table.
struct PoolArgs {
  // W == 1 ("direct"): ids != nullptr; the pool validates the CSR and ids itself, computes the row
  // g = base[t] + id, and writes the per-occurrence dY row index (drow) and bag lengths (blen).
  const int64_t *ids;      // [nnz] (direct mode) or nullptr
  const int32_t *slot_table;
  const uint64_t *base;
  const int64_t *rows;
  uint32_t *drow;          // out (direct mode) [nnz]
  int32_t *blen;           // out (direct mode) [B*S] or nullptr
  const uint32_t *key;     // [nnz] routing keys in CSR order (EMB_SENTINEL = skip), key mode
  const int64_t *offsets;  // [S*B+1]
  int64_t nnz;
  int32_t batch, num_slots, dim;
  int32_t mean;
  const float *rows_src;   // table (W==1) or received unique rows (W>1)
  int64_t nrows_src;       // rows in rows_src (bounds guard)
  const uint32_t *row_idx; // nullptr: row = key (W==1); else row = row_idx[j] (inverse -> unique index)
  float *out;
  uint32_t *err;           // device error word
  uint32_t *err_host;      // mapped pinned host word
  uint32_t *fin;           // [3] finish counters (pool blocks, other kernel's blocks, kernels) or nullptr:
                           // when set, the last of the fin_kernels concurrently running kernels (pool +
                           // segsort at W = 1, pool + owner merge at W > 1) publishes err to err_host
  uint32_t fin_kernels;
};
cudaError_t launch_pool(const PoolArgs &a, cudaStream_t st);
cudaError_t launch_publish_err(const uint32_t *err, uint32_t *err_host, cudaStream_t st);

// backward: segment reduce over sorted (key, pay) + sink
struct GradArgs {
  const uint32_t *skey;    // [n] sorted routing keys (sentinel last)
  const uint32_t *spay;    // [n] payload (occurrence index j, or receive slot)
  int64_t n;
  int32_t dim;
  // contribution source: mode 0 = dY rows via bag_of/blen; mode 1 = rows of `src` at index spay
  int32_t src_mode;
  const float *dy;         // [B][S][D]
  const uint32_t *drow;    // [nnz] dY row index b*S+s per occurrence
  int64_t nsrc_occ;        // entries of drow (bounds guard)
  const int32_t *blen;     // [B*S] bag length by dY row (mean) or nullptr
  int32_t batch, num_slots;
  const float *src;        // mode 1
  // sink: mode 0 = optimizer apply on table rows (local row = key & lmask); mode 1 = write fp32 row
  // to out_rows[useg[p]] (requester-side local grad); mode 2 = the same row stored straight into the
  // owner's gradient buffer through peer memory (p2p exchange)
  int32_t sink_mode;
  const int64_t *n_dev;    // if set, the number of sorted positions is read from the device
  int32_t signal_kind;     // >= 0: the last warp to finish raises this p2p flag in every peer
  P2PArgs p2p;             // sink mode 2 / signal
  uint32_t lmask;
  int32_t opt;             // 0 sgd 1 adagrad 2 row-wise adagrad (a: one float per row)
  double lr, eps;
  float *w, *a;
  int64_t nrows;           // rows of w/a (bounds guard)
  int64_t nsrc;            // rows of dy (S*B) or src (bounds guard)
  int64_t nout;            // rows of out_rows (bounds guard)
  uint32_t *err;
  const uint32_t *useg;    // unique index per sorted position (dedup of skey)
  const uint32_t *ustart;  // segment starts [U+1] (ustart[U] = number of valid positions)
  const uint32_t *u_count; // device U
  float *out_rows;
  double *partials;        // [2 * max resident warps][D]
  uint32_t *tickets;       // [>= U], zero on entry, left zero
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

// W > 1 helpers
cudaError_t launch_owner_counts(const uint32_t *ukey, const uint32_t *u_count, int32_t world, uint32_t lbits,
                                int64_t *send_counts, cudaStream_t st);
cudaError_t launch_scatter_inverse(const uint32_t *skey, const uint32_t *spay, const uint32_t *useg, int64_t n,
                                   uint32_t *inv, cudaStream_t st);

// per-table stable sort (world == 1 fast path), see segsort.cu
constexpr int64_t SEG_CAP = 16384;
struct SegSortArgs {
  const int64_t *ids;       // [nnz] table-local ids in CSR order (validated here: out of range = invalid)
  const int64_t *offsets;   // [S*B+1]
  int64_t nnz;
  int32_t batch;
  const int32_t *gslot;     // [G+1] slot boundaries of the table groups
  const uint64_t *gbase;    // [G] first fused key of the group's table
  const uint32_t *grows;    // [G] rows of the group's table
  const uint32_t *gbits;    // [G] bits covering [0, rows] (rows = the invalid marker)
  uint32_t *skey, *spay;    // out [nnz]
  uint32_t *scratch_k, *scratch_a, *scratch_b;  // [nnz] global buffers for chunks above the smem cap
  uint32_t *run_k, *run_i;  // [nnz] sorted runs (local key, chunk-relative index)
  int32_t K;                // chunks (CTAs) per group
  uint32_t *err;
  uint32_t *err_host;       // with fin: see PoolArgs::fin
  uint32_t *fin;
};
cudaError_t launch_segsort(const SegSortArgs &a, int32_t groups, cudaStream_t st);
cudaError_t launch_local_of_unique(const uint32_t *ukey, const uint32_t *u_count, int64_t cap, uint32_t lmask,
                                   uint32_t *out, cudaStream_t st);
cudaError_t launch_partition(const uint32_t *ukey, const uint32_t *u_count, int64_t cap, const KeySpace &ks,
                             uint32_t *tcnt, uint32_t *send_keys, uint32_t *sp, int64_t *send_counts,
                             cudaStream_t st);
cudaError_t launch_outidx(const uint32_t *skey, const uint32_t *spay, const uint32_t *useg, const uint32_t *sp,
                          int64_t n, uint32_t *outidx, uint32_t *inv, cudaStream_t st);
cudaError_t launch_merge_tree(const uint32_t *rkeys, const int64_t *recv_counts, int W, int64_t cap, uint32_t *ok0,
                              uint32_t *op0, uint32_t *ok1, uint32_t *op1, uint32_t *err, cudaStream_t st,
                              uint32_t *fin, uint32_t *err_host);
cudaError_t launch_merge_runs(const uint32_t *rkeys, const int64_t *recv_counts, int W, int64_t n, uint32_t *okey,
                              uint32_t *opay, uint32_t *err, cudaStream_t st, uint32_t *fin = nullptr,
                              uint32_t *err_host = nullptr);
cudaError_t launch_owner_gather(const float *w, const uint32_t *local, int64_t n, int32_t dim, float *out,
                                cudaStream_t st);

}  // namespace emb
