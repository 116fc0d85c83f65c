/*
 * emb.h — C ABI of the B200-native sparse distributed embedding layer (libemb.so).
 *
 * The operation (§1, §3.3): the "large sparse distributed embedding
 * lookup layer" of a recommender that converts "massive high-dimensional sparse data into dense
 * features". The paper gives no algorithm; the semantics implemented here are BASELINE.json
 * north_star (BJ:5: slot-wise id dedup, shard routing, gather + sum/mean pool per bag; backward =
 * scatter-merge of per-id gradients + sparse SGD/Adagrad row update) with the readings R1-R22 of
 * SURVEY.md §8(c) restated in DESIGN.md §3. The row-sharded synchronous model-parallel mode is the
 * synchronous analogue of the paper's push-pull PS executor.
 *
 * Conventions (all calls):
 *  - Pointers documented "device" are CUDA device pointers OWNED BY THE CALLER that must stay valid
 *    until the work enqueued on `cuda_stream` completes. Pointers documented "host" are read or
 *    written before the call returns (unless stated otherwise).
 *  - The library owns the table shard, the optimizer state and all workspace; everything is
 *    allocated in emb_create, nothing is allocated in the step path.
 *  - CSR input (slot-major, FBGEMM style): bag (s, b) = ids[offsets[s*B+b] .. offsets[s*B+b+1]),
 *    offsets[0] = 0, non-decreasing, offsets[S*B] = nnz. ids are TABLE-LOCAL row ids of table
 *    slot_table[s]. Output/gradient layout: out[b][s][0..D) fp32, row-major (per-sample contiguous
 *    dense feature vector of S*D floats, the input of the dense stage).
 *  - Error behaviour: argument errors are returned synchronously and nothing is enqueued. Errors the
 *    device detects (id < 0 or id >= rows[t]: EMB_ERR_RANGE; non-monotone offsets or offsets[S*B] !=
 *    nnz: EMB_ERR_INVALID) set a sticky flag; an offending id contributes nothing and updates
 *    nothing; the flag is returned by the next API call after the device work completed, and stays
 *    set until emb_clear_error(). The update of a step whose input had an error is skipped entirely
 *    (decided on the device, so it does not depend on host timing). emb_last_error() gives a text.
 *    No call ever aborts the process.
 *  - Step protocol: emb_lookup, then exactly one emb_backward_update (else EMB_ERR_STATE); one host
 *    thread per handle. With world > 1 every rank makes the same sequence of lookup/backward calls
 *    (they are collective); per-rank batch sizes may differ.
 *  - Errors at world > 1: a lookup / backward call always takes part in the collective step, even
 *    with bad arguments (the rank then contributes an empty batch and returns EMB_ERR_INVALID). A step
 *    in which ANY rank had an input error (bad arguments, an id out of range, bad offsets, or a sticky
 *    error not yet cleared) updates no row on any rank; forward outputs of valid bags are still
 *    computed. A rank that skips a collective call makes its peers' waits time out after ~4 s: they
 *    report EMB_ERR_NCCL (sticky) and skip the work; the handles must then be recreated.
 *  - Sharding (R7): fused row space g = base[t] + id, base[t] = sum_{t'<t} rows[t']. CYCLIC: owner(g)
 *    = g mod W, local(g) = g div W. BLOCK: rows_per = ceil(R_total/W), owner = g div rows_per, local =
 *    g mod rows_per. Requires R_total < 2^32 and (for W > 1) the routing key owner*2^b + local < 2^32.
 */
#ifndef EMB_H_
#define EMB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMB_MAX_WORLD 16
#define EMB_MAX_TABLES 1024
#define EMB_MAX_SLOTS 1024

typedef struct emb_ctx *emb_handle_t;

typedef enum {
  EMB_OK = 0,
  EMB_ERR_INVALID = 1, /* bad config / argument / shape / CSR offsets                          */
  EMB_ERR_RANGE = 2,   /* an id < 0 or >= rows[t] (device-detected, sticky)                      */
  EMB_ERR_STATE = 3,   /* backward without lookup, double lookup, unsupported call in this state */
  EMB_ERR_NOMEM = 4,   /* device or pinned-host allocation failed in emb_create                   */
  EMB_ERR_CUDA = 5,    /* a CUDA runtime call failed                                              */
  EMB_ERR_NCCL = 6     /* NCCL bootstrap failed, or a peer never arrived at an exchange (timeout) */
} emb_status_t;

typedef enum { EMB_POOL_SUM = 0, EMB_POOL_MEAN = 1 } emb_pool_t;          /* R1 */
/* R12; EMB_OPT_ROWWISE_ADAGRAD (reading R14'): one fp32 accumulator per row,
   a <- a + (1/D) sum_c G[c]^2, w <- w - lr*G/(sqrt(a)+eps) -- 4 bytes of state per row instead of 4D */
typedef enum { EMB_OPT_SGD = 0, EMB_OPT_ADAGRAD = 1, EMB_OPT_ROWWISE_ADAGRAD = 2 } emb_opt_t;
typedef enum { EMB_SHARD_CYCLIC = 0, EMB_SHARD_BLOCK = 1 } emb_shard_t;   /* R7 */

typedef struct {
  int32_t num_tables;       /* T >= 1                                                        */
  const int64_t *rows;      /* host [T], rows[t] >= 1; sum < 2^32                            */
  int32_t dim;              /* D: 4 <= D <= 256, D % 4 == 0 (same for all tables)           */
  int32_t num_slots;        /* S >= 1                                                        */
  const int32_t *slot_table;/* host [S] -> table id; slots may share a table (R5)            */
  int32_t pool;             /* emb_pool_t                                                    */
  int32_t opt;              /* emb_opt_t                                                     */
  double eps;               /* Adagrad epsilon, > 0 (R13)                                    */
  float init_accum;         /* initial Adagrad accumulator, >= 0 (R13)                       */
  uint64_t init_seed;       /* table init: w[g,c] = int16(splitmix64(seed ^ (g*D+c)) >> 48) * 2^-19 (R15) */
  int32_t max_batch;        /* per-rank per-step capacity B_max >= 1 (sizes the workspace)   */
  int64_t max_ids;          /* per-rank per-step capacity nnz_max >= 1                       */
  int32_t rank;             /* 0 <= rank < world                                             */
  int32_t world;            /* 1 <= world <= EMB_MAX_WORLD                                   */
  const void *nccl_id;      /* host, 128-byte ncclUniqueId from emb_get_unique_id on rank 0; required iff
                               world > 1 and the handle is created with emb_create (one rank per
                               process; NCCL only bootstraps the peer mappings); ignored by
                               emb_create_group */
  int32_t device;           /* CUDA device ordinal used by this handle                       */
  int32_t shard;            /* emb_shard_t                                                   */
} emb_config_t;

/* Per-step statistics of the last lookup (requester side and owner side). */
typedef struct {
  int64_t nnz;                           /* occurrences in the last batch                           */
  int64_t num_bags;                      /* S*B                                                     */
  int64_t unique_local;                  /* U_l: distinct keys of this rank's batch                 */
  int64_t unique_owner;                  /* U_o: distinct rows this rank owns that were requested (W>1; = U_l at W=1) */
  int64_t recv_keys;                     /* keys received from all ranks (W>1; = U_l at W=1)       */
  int32_t world;
  int32_t launches;                      /* kernels enqueued by the last lookup+backward            */
  int64_t send_counts[EMB_MAX_WORLD];    /* keys sent to each owner                                 */
  int64_t recv_counts[EMB_MAX_WORLD];    /* keys received from each requester                       */
} emb_step_info_t;

/* ---- lifecycle ------------------------------------------------------------------------------ */

/* Create a handle: validates cfg, selects cfg->device, allocates the fp32 shard [rows_local][D]
 * (+ the Adagrad accumulator), initialises it with the R15 hash, sizes the workspace from
 * max_batch / max_ids / world. world > 1 (one rank per process, all on one host): collective across
 * ranks -- ncclCommInitRank, an all-gather of max_ids and the GPUs' PCI ids (every rank must have peer
 * access to every other rank's GPU, else EMB_ERR_INVALID), then an all-gather of CUDA IPC handles of
 * the exchange buffers and table shards. Synchronous. On failure *out is NULL. */
emb_status_t emb_create(const emb_config_t *cfg, emb_handle_t *out);

/* Create ALL n = world ranks of a row-sharded layer in this process (group mode): cfgs[r] has
 * world == n and rank == r; devices may differ (peer access is enabled between them) or coincide
 * (several ranks emulated on one GPU). out: host array [n] of handles. The ranks step together
 * through emb_lookup_group / emb_backward_update_group only (emb_lookup on a group handle returns
 * EMB_ERR_STATE). Every kernel of the exchange is the one a multi-process rank runs; the group calls
 * order the ranks' phases with cross-stream events, so no kernel waits on a kernel that is not
 * already complete. Destroy each handle with emb_destroy. */
emb_status_t emb_create_group(const emb_config_t *cfgs, int32_t n, emb_handle_t *out);

/* Free everything the handle owns (synchronises its streams). NULL is a no-op. */
emb_status_t emb_destroy(emb_handle_t h);

/* Write a fresh 128-byte ncclUniqueId to out128 (host). Call on rank 0 and broadcast. */
emb_status_t emb_get_unique_id(void *out128);

/* ---- the step (enqueued on cuda_stream; no host synchronisation) ---------------------------- */

/* Forward: out[b][s][:] = sum (or mean) over bag (s,b) of W_t[id][:]  (R1-R5).
 * ids: device int64 [nnz]; offsets: device int64 [S*batch+1]; out: device fp32 [batch][S][D],
 * 16-byte aligned. 0 <= batch <= max_batch, 0 <= nnz <= max_ids. Also dedups the ids per rank and,
 * when world > 1, routes the distinct keys to their owners and pulls the remote distinct rows from
 * the owners' shards (collective; device-side exchange over NVLink peer memory, no host
 * synchronisation). Saves what backward needs in the workspace, so ids and offsets may be reused once
 * the stream work completes. */
emb_status_t emb_lookup(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch,
                        int64_t nnz, float *out, void *cuda_stream);

/* Optional pipelining (per-table sort path, i.e. a monotone slot -> table map; a no-op returning
 * EMB_OK otherwise or for an empty batch): declare the NEXT emb_lookup's inputs, ready on cuda_stream
 * at this call. Called between emb_lookup(k) and emb_backward_update(k), the first part of lookup k+1
 * is launched by emb_backward_update(k) right after its gradient kernel (on a lowest-priority library
 * stream) and overlaps the gradient pass. Results are identical with or without it.
 *  - world == 1: the per-table dedup sort. The next emb_lookup consumes it when called with the same
 *    ids / offsets pointers and batch / nnz; any other call discards it.
 *  - world > 1: the dedup sort AND the route (the step's distinct keys are stored into their owners'
 *    receive regions: the first phase of the next collective step, which cannot be withdrawn once
 *    launched). The next emb_lookup must then pass the same ids / offsets pointers and batch / nnz;
 *    if it does not, it returns EMB_ERR_INVALID after taking part with an empty batch and the step
 *    updates nothing on any rank. A second prefetch before that lookup returns EMB_ERR_STATE. Ranks
 *    may mix prefetching and plain lookups freely. Group handles use emb_lookup_prefetch_group.
 * A request followed by emb_lookup without a backward in between launched nothing and is dropped.
 * ids and offsets must stay valid and unmodified until the consuming emb_lookup. */
emb_status_t emb_lookup_prefetch(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch,
                                 int64_t nnz, void *cuda_stream);

/* Backward + update for the last lookup: c_j = d_out[b][s][:] (mean: / |bag|), G[g] = sum of c_j over
 * all occurrences of all ranks (fp64 accumulation, deterministic order), then one SGD or element-wise
 * Adagrad (or row-wise Adagrad) update per touched row (R8-R14'). d_out: device fp32 [batch][S][D], 16-byte aligned.
 * Collective when world > 1: the merged per-key gradients go to the rows' owners, which merge the
 * ranks' contributions in source-rank order and apply. */
emb_status_t emb_backward_update(emb_handle_t h, const float *d_out, double lr, void *cuda_stream);

/* Group-mode step over all n ranks (handles from emb_create_group, in rank order). Per rank r the
 * arguments mean what they mean for emb_lookup / emb_backward_update; ids, offsets, batch, nnz, out,
 * d_out are host arrays [n] of per-rank values; streams: host array [n] of cudaStream_t on each rank's
 * device (NULL = the legacy default stream for every rank). Returns the first error of any rank (the
 * other ranks' calls still took part, see "Errors at world > 1"). */
emb_status_t emb_lookup_group(emb_handle_t *hs, int32_t n, const int64_t *const *ids, const int64_t *const *offsets,
                              const int32_t *batch, const int64_t *nnz, float *const *out, void *const *streams);
emb_status_t emb_backward_update_group(emb_handle_t *hs, int32_t n, const float *const *d_out, double lr,
                                       void *const *streams);
/* Group form of emb_lookup_prefetch: per rank r, emb_lookup_prefetch(hs[r], ids[r], offsets[r],
 * batch[r], nnz[r], streams[r]) (streams may be NULL: default streams). The next emb_lookup_group
 * consumes the prefetched first phases. Returns the first rank's error, if any. */
emb_status_t emb_lookup_prefetch_group(emb_handle_t *hs, int32_t n, const int64_t *const *ids,
                                       const int64_t *const *offsets, const int32_t *batch, const int64_t *nnz,
                                       void *const *streams);

/* End-to-end variants over HOST buffers (pinned memory, else the copies serialise): ASYNCHRONOUS --
 * each call returns after enqueueing. emb_lookup_host copies ids/offsets host->device on the
 * library's H2D copy stream into one of two staging sets, runs emb_lookup on cuda_stream after them,
 * and copies out[] device->host on the library's D2H copy stream; emb_backward_update_host copies
 * d_out host->device (H2D stream) and runs emb_backward_update on cuda_stream. With two staging sets
 * the D2H of step k's output overlaps the H2D copies of step k's gradient and of step k+1's ids (the
 * two PCIe directions). Host buffers must stay valid and unmodified, and out[] must not be read, until
 * emb_host_sync(h) returns. Layouts as for the device calls. Argument / state errors are returned
 * synchronously; device-detected errors as for the device calls. Not for group handles. */
emb_status_t emb_lookup_host(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch,
                             int64_t nnz, float *out, void *cuda_stream);
emb_status_t emb_backward_update_host(emb_handle_t h, const float *d_out, double lr, void *cuda_stream);
/* Wait until every host-buffer call of h completed (copies included); returns the sticky status. */
emb_status_t emb_host_sync(emb_handle_t h);

/* ---- host-synchronous helpers (tests, checkpoint, accounting; call between steps) ------------- */

/* Read / overwrite rows of table `table` that THIS rank owns (owner(base[table]+row) == rank, else
 * EMB_ERR_INVALID). rows_host: host int64 [n] table-local ids; w_host: host fp32 [n][D]; a_host: host
 * fp32 [n][D] (element-wise Adagrad) or [n] (row-wise Adagrad); a_host may be NULL (ignored for SGD).
 * Synchronises the handle's last stream. */
emb_status_t emb_read_rows(emb_handle_t h, int32_t table, const int64_t *rows_host, int64_t n,
                           float *w_host, float *a_host);
emb_status_t emb_write_rows(emb_handle_t h, int32_t table, const int64_t *rows_host, int64_t n,
                            const float *w_host, const float *a_host);

/* Statistics of the last lookup (synchronises the last stream). */
emb_status_t emb_last_step_info(emb_handle_t h, emb_step_info_t *info);

/* The GPU's dedup result of the last lookup, copied to host: the sorted distinct fused keys g of this
 * rank's batch (keys_host, uint64 [U_l]) and their multiplicities (counts_host, int64 [U_l]).
 * cap = capacity of both arrays; *n_out = U_l (EMB_ERR_INVALID if cap < U_l). Either array may be NULL. */
emb_status_t emb_last_unique(emb_handle_t h, uint64_t *keys_host, int64_t *counts_host, int64_t cap,
                             int64_t *n_out);

/* Owner side (world > 1): the sorted distinct fused keys this rank owns that the last step touched
 * (U_o) and, per key, the number of requesting ranks that sent it (fan-in; the
 * global multiplicity is the sum of the requesters' emb_last_unique counts). At world == 1 equals
 * emb_last_unique. */
emb_status_t emb_last_owner_unique(emb_handle_t h, uint64_t *keys_host, int64_t *counts_host,
                                   int64_t cap, int64_t *n_out);

/* Rows held by this rank (rows_local of the sharding rule R7). */
int64_t emb_rows_local(emb_handle_t h);

/* Per-kernel device-time accounting with CUDA events (off by default). When enabled, every kernel
 * the library launches is bracketed by an event pair on the stream it runs on; emb_profile_read
 * synchronises and returns, for kernel index k < *n (names via emb_profile_name), the summed device
 * milliseconds and the number of launches since the last reset. */
emb_status_t emb_profile_enable(emb_handle_t h, int32_t on);
emb_status_t emb_profile_reset(emb_handle_t h);
emb_status_t emb_profile_read(emb_handle_t h, double *ms, int64_t *launches, int32_t cap, int32_t *n);
const char *emb_profile_name(int32_t k);

/* Clear the sticky device error flag. */
emb_status_t emb_clear_error(emb_handle_t h);

/* Text of the last error on h (or of the last failed emb_create when h == NULL). Never NULL. */
const char *emb_last_error(emb_handle_t h);

#ifdef __cplusplus
}
#endif
#endif /* EMB_H_ */
