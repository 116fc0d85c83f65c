// emb_api.cu — EmbContext runtime + the C ABI of include/emb.h.
//
// Owns: the fp32 row shard [rows_local][D] (+ Adagrad accumulator), all step workspace (sized once
// in emb_create from max_batch / max_ids / world), a side stream for the sort (overlapped with the
// forward pool), the NCCL communicator for world > 1, and the step state machine.
//
// Step at world == 1 (no host sync):
//   lookup   : K1 keys -> fork{ side: radix sort (key, j) } ; main: K5 pool straight from the table
//              -> join
//   backward : K6+K7 fused segment-reduce + optimizer apply over the sorted keys
// Step at world > 1 (v1 exchange: grouped ncclSend/ncclRecv all-to-allv, one host sync for counts):
//   lookup   : K1 keys (owner-major routing keys) -> sort -> unique -> per-owner counts
//              -> X0 counts all-to-all -> host reads counts -> X1 local ids all-to-allv
//              -> owner gather -> X2 rows all-to-allv -> K5 pool from the received unique rows;
//              side stream: owner-side sort of the received keys (for the backward merge)
//   backward : K6 segment reduce -> per-unique-key fp32 grads -> X3 all-to-allv to the owners
//              -> K6+K7 owner merge (source-rank order) + optimizer apply
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/emb.h"
#include "common.cuh"
#include "internal.h"

using namespace emb;

namespace {

std::mutex g_err_mu;
std::string g_create_error = "no error";

const char *kKernelNames[KID_COUNT] = {"keys",        "sort_hist",  "sort_pass", "pool",
                                       "grad_apply",  "unique",     "route",     "owner_gather",
                                       "grad_local",  "nccl",       "init",      "owner_merge",
                                       "p2p_wait"};

uint32_t bits_for(uint64_t x) {  // smallest b with x < 2^b (x >= 0)
  uint32_t b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

}  // namespace

struct emb_ctx {
  // ---- config
  int32_t T = 0, D = 0, S = 0;
  std::vector<int64_t> rows;
  std::vector<uint64_t> base;
  std::vector<int32_t> slot_table;
  int32_t pool = 0, opt = 0;
  double eps = 1e-6;
  float init_accum = 0.f;
  uint64_t seed = 0;
  int32_t max_batch = 0;
  int64_t max_ids = 0;
  int32_t rank = 0, world = 1, device = 0, shard = 0;
  uint64_t R_total = 0;
  KeySpace ks{};
  int64_t rows_local = 0, rows_local_max = 0;
  uint32_t lmask = 0xFFFFFFFFu;
  uint32_t owner_key_bits = 0;

  // ---- device state
  float *w = nullptr, *a = nullptr;
  int32_t *d_slot_table = nullptr;
  uint64_t *d_base = nullptr;
  int64_t *d_rows = nullptr;

  // ---- workspace
  std::vector<void *> allocs;
  uint32_t *key_csr = nullptr, *drow = nullptr, *k0 = nullptr, *v0 = nullptr, *k1 = nullptr, *v1 = nullptr;
  // W = 1 sort output, two sets: a prefetched sort of the next step (emb_lookup_prefetch) writes the
  // set the pending backward does not read
  uint32_t *sk_set[2] = {nullptr, nullptr}, *sp_set[2] = {nullptr, nullptr}, *sort_scratch = nullptr;
  int cur_set = 0;
  struct {
    bool valid = false;
    const int64_t *ids = nullptr, *offsets = nullptr;
    int32_t batch = 0;
    int64_t nnz = 0;
    int set = 0;
  } pf;
  int32_t *blen = nullptr;
  SortWorkspace sws{};
  double *partials = nullptr;
  uint32_t *tickets = nullptr;
  uint32_t *useg = nullptr, *ukey = nullptr, *ustart = nullptr, *uend = nullptr, *u_count = nullptr,
           *uniq_counter = nullptr, *fin = nullptr;
  uint64_t *uniq_status = nullptr, *ouniq_status = nullptr;
  uint32_t uniq_epoch = 0, ouniq_epoch = 0;
  // world == 1 per-table sort (segsort.cu): table groups of the slot-major CSR
  bool segsort_ok = false;
  int32_t G = 0, segK = 1;
  uint32_t *run_k = nullptr, *run_i = nullptr;
  int32_t *d_gslot = nullptr;
  uint64_t *d_gbase = nullptr;
  uint32_t *d_grows = nullptr, *d_gbits = nullptr;
  uint32_t *err_dev = nullptr;
  uint32_t *err_host = nullptr;      // pinned, mapped
  uint32_t *err_host_dev = nullptr;  // device alias of err_host
  // world > 1
  uint32_t *inv = nullptr;           // [max_ids] occurrence -> unique index
  uint32_t *send_keys = nullptr;     // [max_ids] local ids grouped by owner
  uint32_t *recv_keys = nullptr;     // [recv_cap]
  float *owner_rows = nullptr;       // [recv_cap][D]
  float *uniq_rows = nullptr;        // [max_ids][D]
  float *gloc = nullptr;             // [max_ids][D]
  float *grecv = nullptr;            // [recv_cap][D]
  uint32_t *ok0 = nullptr, *ov0 = nullptr, *ok1 = nullptr, *ov1 = nullptr;  // owner sort buffers
  uint32_t *sp = nullptr, *outidx = nullptr, *tcnt = nullptr;  // owner partition (segsort path)
  bool ukey_is_g = false;        // requester unique keys are fused keys g (segsort path) or routing keys
  bool owner_unique_done = false;
  uint32_t *ouseg = nullptr, *oukey = nullptr, *oustart = nullptr, *ouend = nullptr, *ou_count = nullptr,
           *ouniq_counter = nullptr;  // owner-side dedup of the received keys
  int64_t *d_counts = nullptr;       // [2][EMB_MAX_WORLD] send, recv
  int64_t *h_counts = nullptr;       // pinned [2*EMB_MAX_WORLD + 1]
  int64_t recv_cap = 0;
  ncclComm_t comm = nullptr;
  // peer-memory exchange (p2p.cu): IPC-mapped peer buffers, epoch flags, device route table
  bool use_p2p = false;
  P2PArgs p2p{};
  uint64_t epoch = 0;
  int64_t *xmat = nullptr;
  uint64_t *flags = nullptr;
  RouteTable *rt = nullptr;
  uint32_t *p2p_done = nullptr;
  std::vector<void *> ipc_opened;
  bool counts_synced = true;

  // ---- streams / step state
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_pf = nullptr;
  int state = 0;  // 0 idle, 1 looked up
  int32_t batch = 0;
  int64_t nnz = 0;
  uint32_t *skey = nullptr, *spay = nullptr;   // requester-side sorted keys / payload of the last lookup
  uint32_t *okey = nullptr, *opay = nullptr;   // owner-side sorted received keys / payload
  int64_t U_l = 0, n_recv = 0;
  int64_t send_counts[EMB_MAX_WORLD] = {0}, recv_counts[EMB_MAX_WORLD] = {0};
  int64_t soff[EMB_MAX_WORLD + 1] = {0}, roff[EMB_MAX_WORLD + 1] = {0};
  cudaStream_t last_stream = nullptr;
  int launches = 0;

  // ---- host-buffer (e2e) staging, allocated on first use
  int64_t *st_ids = nullptr, *st_offsets = nullptr;
  float *st_out = nullptr, *st_dout = nullptr;

  // ---- profiler
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  std::vector<int> prof_kid;
  size_t prof_used = 0;
  int prof_open_kid = -1;
  double prof_ms[KID_COUNT] = {0};
  int64_t prof_cnt[KID_COUNT] = {0};

  std::string last_error = "no error";
};

namespace {

emb_status_t fail(emb_ctx *h, emb_status_t s, const std::string &msg) {
  if (h) h->last_error = msg;
  return s;
}
#define CUDA_TRY(h, call)                                                                          \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail(h, EMB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)
#define NCCL_TRY(h, call)                                                                          \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess)                                                                         \
      return fail(h, EMB_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));            \
  } while (0)

template <typename T>
cudaError_t dalloc(emb_ctx *h, T **p, size_t count) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e == cudaSuccess) h->allocs.push_back(q);
  *p = static_cast<T *>(q);
  return e;
}

// profiler hook: kid, end=0 before the launch, 1 after
void prof_hook(void *vctx, int kid, int end, cudaStream_t st) {
  emb_ctx *h = static_cast<emb_ctx *>(vctx);
  if (!h->prof_on) return;
  if (!end) {
    if (h->prof_used + 2 > h->prof_ev.size()) {
      h->prof_open_kid = -1;
      return;
    }
    cudaEventRecord(h->prof_ev[h->prof_used], st);
    h->prof_open_kid = kid;
  } else {
    if (h->prof_open_kid != kid) return;
    cudaEventRecord(h->prof_ev[h->prof_used + 1], st);
    h->prof_kid.push_back(kid);
    h->prof_used += 2;
    h->prof_open_kid = -1;
  }
}

emb_status_t check_sticky(emb_ctx *h) {
  const uint32_t e = *(volatile uint32_t *)h->err_host;
  if (e & EMB_DEVERR_TIMEOUT)
    return fail(h, EMB_ERR_NCCL, "device: a peer never raised its exchange flag (sticky)");
  if (e & EMB_DEVERR_INTERNAL)
    return fail(h, EMB_ERR_CUDA, "device: an internal bounds guard tripped (library bug; work was skipped)");
  if (e & EMB_DEVERR_RANGE) return fail(h, EMB_ERR_RANGE, "device: an id was < 0 or >= rows[t] (sticky)");
  if (e & EMB_DEVERR_INVALID)
    return fail(h, EMB_ERR_INVALID, "device: CSR offsets not monotone or offsets[S*B] != nnz (sticky)");
  return EMB_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int64_t owner_of_global(const emb_ctx *h, uint64_t g) {
  if (h->world == 1) return 0;
  return h->shard == 0 ? (int64_t)(g % (uint64_t)h->world) : (int64_t)(g / h->ks.rows_per);
}
int64_t local_of_global(const emb_ctx *h, uint64_t g) {
  if (h->world == 1) return (int64_t)g;
  return h->shard == 0 ? (int64_t)(g / (uint64_t)h->world) : (int64_t)(g % h->ks.rows_per);
}

// ------------------------------------------------------------------------------------------------
// optimizer-state floats per row: D (element-wise Adagrad) or 1 (row-wise)
int32_t accum_width(const emb_ctx *h) { return h->opt == EMB_OPT_ROWWISE_ADAGRAD ? 1 : h->D; }

// world > 1: map every peer's exchange buffers (CUDA IPC handles all-gathered over NCCL)
emb_status_t setup_p2p(emb_ctx *h) {
  const int W = h->world;
  if (dalloc(h, &h->xmat, (size_t)P2P_MAXW * P2P_MAXW) || dalloc(h, &h->flags, (size_t)P2P_NKIND * P2P_MAXW) ||
      dalloc(h, &h->rt, 1) || dalloc(h, &h->p2p_done, (size_t)P2P_NKIND))
    return fail(h, EMB_ERR_NOMEM, "alloc p2p state");
  CUDA_TRY(h, cudaMemset(h->p2p_done, 0, sizeof(uint32_t) * P2P_NKIND));
  CUDA_TRY(h, cudaMemset(h->xmat, 0, sizeof(int64_t) * P2P_MAXW * P2P_MAXW));
  CUDA_TRY(h, cudaMemset(h->flags, 0, sizeof(uint64_t) * P2P_NKIND * P2P_MAXW));
  CUDA_TRY(h, cudaMemset(h->rt, 0, sizeof(RouteTable)));
  constexpr int NB = 5;
  void *mine[NB] = {h->xmat, h->flags, h->recv_keys, h->uniq_rows, h->grecv};
  std::vector<cudaIpcMemHandle_t> hs(NB);
  for (int b = 0; b < NB; ++b) CUDA_TRY(h, cudaIpcGetMemHandle(&hs[b], mine[b]));
  const size_t bytes = sizeof(cudaIpcMemHandle_t) * NB;
  char *dsend = nullptr, *drecv = nullptr;
  CUDA_TRY(h, cudaMalloc(&dsend, bytes));
  CUDA_TRY(h, cudaMalloc(&drecv, bytes * W));
  CUDA_TRY(h, cudaMemcpy(dsend, hs.data(), bytes, cudaMemcpyHostToDevice));
  NCCL_TRY(h, ncclAllGather(dsend, drecv, bytes, ncclUint8, h->comm, 0));
  CUDA_TRY(h, cudaDeviceSynchronize());
  std::vector<cudaIpcMemHandle_t> all((size_t)NB * W);
  CUDA_TRY(h, cudaMemcpy(all.data(), drecv, bytes * W, cudaMemcpyDeviceToHost));
  cudaFree(dsend);
  cudaFree(drecv);
  P2PArgs &p = h->p2p;
  p.world = W;
  p.rank = h->rank;
  p.flags = h->flags;
  p.xmat = h->xmat;
  p.rt = h->rt;
  p.done = h->p2p_done;
  for (int r = 0; r < W; ++r) {
    void *ptr[NB];
    for (int b = 0; b < NB; ++b) {
      if (r == h->rank) {
        ptr[b] = mine[b];
      } else {
        void *q = nullptr;
        CUDA_TRY(h, cudaIpcOpenMemHandle(&q, all[(size_t)r * NB + b], cudaIpcMemLazyEnablePeerAccess));
        h->ipc_opened.push_back(q);
        ptr[b] = q;
      }
    }
    p.peer_xmat[r] = static_cast<int64_t *>(ptr[0]);
    p.peer_flags[r] = static_cast<uint64_t *>(ptr[1]);
    p.peer_recv_keys[r] = static_cast<uint32_t *>(ptr[2]);
    p.peer_uniq_rows[r] = static_cast<float *>(ptr[3]);
    p.peer_grecv[r] = static_cast<float *>(ptr[4]);
  }
  return EMB_OK;
}

// p2p mode: bring the step's counts (device route table) to the host, for statistics only
emb_status_t sync_counts(emb_ctx *h) {
  if (h->counts_synced) return EMB_OK;
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  RouteTable rt;
  CUDA_TRY(h, cudaMemcpy(&rt, h->rt, sizeof(rt), cudaMemcpyDeviceToHost));
  const int W = h->world;
  for (int p = 0; p <= W; ++p) {
    h->soff[p] = rt.soff[p];
    h->roff[p] = rt.roff[p];
  }
  for (int p = 0; p < W; ++p) {
    h->send_counts[p] = rt.soff[p + 1] - rt.soff[p];
    h->recv_counts[p] = rt.recv_counts[p];
  }
  h->U_l = rt.n_send;
  h->n_recv = rt.n_recv;
  h->counts_synced = true;
  return EMB_OK;
}

emb_status_t create_impl(const emb_config_t *cfg, emb_ctx *h) {
  if (!cfg) return fail(h, EMB_ERR_INVALID, "cfg is NULL");
  if (cfg->num_tables < 1 || cfg->num_tables > EMB_MAX_TABLES || !cfg->rows)
    return fail(h, EMB_ERR_INVALID, "num_tables must be in [1, EMB_MAX_TABLES] and rows non-NULL");
  if (cfg->num_slots < 1 || cfg->num_slots > EMB_MAX_SLOTS || !cfg->slot_table)
    return fail(h, EMB_ERR_INVALID, "num_slots must be in [1, EMB_MAX_SLOTS] and slot_table non-NULL");
  if (cfg->dim < 4 || cfg->dim > 256 || cfg->dim % 4 != 0 || (cfg->dim > 128 && cfg->dim % 8 != 0))
    return fail(h, EMB_ERR_INVALID, "dim must be a multiple of 4 in [4, 256] (multiple of 8 above 128)");
  if (cfg->pool != EMB_POOL_SUM && cfg->pool != EMB_POOL_MEAN) return fail(h, EMB_ERR_INVALID, "bad pool");
  if (cfg->opt != EMB_OPT_SGD && cfg->opt != EMB_OPT_ADAGRAD && cfg->opt != EMB_OPT_ROWWISE_ADAGRAD)
    return fail(h, EMB_ERR_INVALID, "bad opt");
  if (!(cfg->eps > 0)) return fail(h, EMB_ERR_INVALID, "eps must be > 0");
  if (!(cfg->init_accum >= 0)) return fail(h, EMB_ERR_INVALID, "init_accum must be >= 0");
  if (cfg->max_batch < 1 || cfg->max_ids < 1 || cfg->max_ids >= (1ll << 30))
    return fail(h, EMB_ERR_INVALID, "max_batch >= 1 and 1 <= max_ids < 2^30 required");
  if (cfg->world < 1 || cfg->world > EMB_MAX_WORLD || cfg->rank < 0 || cfg->rank >= cfg->world)
    return fail(h, EMB_ERR_INVALID, "need 1 <= world <= EMB_MAX_WORLD and 0 <= rank < world");
  if (cfg->world > 1 && !cfg->nccl_id) return fail(h, EMB_ERR_INVALID, "world > 1 needs nccl_id");
  if (cfg->shard != EMB_SHARD_CYCLIC && cfg->shard != EMB_SHARD_BLOCK) return fail(h, EMB_ERR_INVALID, "bad shard");
  if ((int64_t)cfg->num_slots * cfg->max_batch >= (1ll << 31))
    return fail(h, EMB_ERR_INVALID, "num_slots * max_batch must be < 2^31");

  h->T = cfg->num_tables;
  h->D = cfg->dim;
  h->S = cfg->num_slots;
  h->rows.assign(cfg->rows, cfg->rows + h->T);
  h->slot_table.assign(cfg->slot_table, cfg->slot_table + h->S);
  h->base.resize(h->T);
  uint64_t acc = 0;
  for (int t = 0; t < h->T; ++t) {
    if (h->rows[t] < 1) return fail(h, EMB_ERR_INVALID, "rows[t] must be >= 1");
    h->base[t] = acc;
    acc += (uint64_t)h->rows[t];
    if (acc >= (1ull << 32) - 1) return fail(h, EMB_ERR_INVALID, "total rows must be < 2^32 - 1");
  }
  for (int s = 0; s < h->S; ++s)
    if (h->slot_table[s] < 0 || h->slot_table[s] >= h->T) return fail(h, EMB_ERR_INVALID, "slot_table out of range");
  h->R_total = acc;
  h->pool = cfg->pool;
  h->opt = cfg->opt;
  h->eps = cfg->eps;
  h->init_accum = cfg->init_accum;
  h->seed = cfg->init_seed;
  h->max_batch = cfg->max_batch;
  h->max_ids = cfg->max_ids;
  h->rank = cfg->rank;
  h->world = cfg->world;
  h->device = cfg->device;
  h->shard = cfg->shard;

  // key space
  KeySpace &ks = h->ks;
  ks.world = h->world;
  ks.rank = h->rank;
  ks.shard = h->shard;
  ks.rows_per = (h->R_total + h->world - 1) / h->world;
  if (h->world == 1) {
    h->rows_local = h->rows_local_max = (int64_t)h->R_total;
    ks.lbits = 32;
    ks.key_bits = bits_for(h->R_total);  // max valid key R-1 < sentinel-mask 2^b - 1
    if (ks.key_bits == 0) ks.key_bits = 1;
    h->lmask = 0xFFFFFFFFu;
  } else {
    const uint64_t W = h->world;
    if (h->shard == 0) {
      h->rows_local = (int64_t)((h->R_total - h->rank + W - 1) / W);
      h->rows_local_max = (int64_t)((h->R_total + W - 1) / W);
    } else {
      const int64_t lo = std::min<int64_t>((int64_t)h->R_total, (int64_t)ks.rows_per * h->rank);
      const int64_t hi = std::min<int64_t>((int64_t)h->R_total, (int64_t)ks.rows_per * (h->rank + 1));
      h->rows_local = hi - lo;
      h->rows_local_max = (int64_t)ks.rows_per;
    }
    ks.lbits = bits_for((uint64_t)h->rows_local_max - 1);
    if (ks.lbits == 0) ks.lbits = 1;
    const uint64_t max_valid = ((uint64_t)(h->world - 1) << ks.lbits) + (uint64_t)h->rows_local_max - 1;
    if (max_valid + 1 >= 0xFFFFFFFFull) return fail(h, EMB_ERR_INVALID, "routing key space exceeds 32 bits");
    ks.key_bits = bits_for(max_valid + 1);
    h->lmask = (1u << ks.lbits) - 1u;
    h->owner_key_bits = ks.lbits;
  }

  CUDA_TRY(h, cudaSetDevice(h->device));
  // table shard + state
  const size_t row_elems = (size_t)std::max<int64_t>(h->rows_local, 1) * h->D;
  if (dalloc(h, &h->w, row_elems) != cudaSuccess) return fail(h, EMB_ERR_NOMEM, "cannot allocate the table shard");
  if (h->opt == EMB_OPT_ADAGRAD && dalloc(h, &h->a, row_elems) != cudaSuccess)
    return fail(h, EMB_ERR_NOMEM, "cannot allocate the Adagrad state");
  if (h->opt == EMB_OPT_ROWWISE_ADAGRAD && dalloc(h, &h->a, (size_t)std::max<int64_t>(h->rows_local, 1)) != cudaSuccess)
    return fail(h, EMB_ERR_NOMEM, "cannot allocate the row-wise Adagrad state");
  {
    // the side stream carries the latency-critical sort: highest priority, so its CTAs are scheduled
    // ahead of the bandwidth-bound pool CTAs as SMs free up
    int lo_prio = 0, hi_prio = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi_prio));
  }
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_pf, cudaEventDisableTiming));
  CUDA_TRY(h, launch_init(h->w, h->a, h->opt == EMB_OPT_ROWWISE_ADAGRAD, h->rows_local, h->D, h->seed,
                          h->init_accum, ks, h->rank, h->side));

  // small config arrays
  if (dalloc(h, &h->d_slot_table, h->S) || dalloc(h, &h->d_base, h->T) || dalloc(h, &h->d_rows, h->T))
    return fail(h, EMB_ERR_NOMEM, "alloc config");
  CUDA_TRY(h, cudaMemcpy(h->d_slot_table, h->slot_table.data(), sizeof(int32_t) * h->S, cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->d_base, h->base.data(), sizeof(uint64_t) * h->T, cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->d_rows, h->rows.data(), sizeof(int64_t) * h->T, cudaMemcpyHostToDevice));

  // workspace
  const int64_t N = h->max_ids, SB = (int64_t)h->S * h->max_batch;
  const int W = h->world;
  h->recv_cap = W > 1 ? (int64_t)W * N : N;
  const int64_t grad_n = std::max<int64_t>(N, h->recv_cap);
  const int64_t nticket = grad_n + 1;
  const int64_t nwarps_max = grad_max_warps(h->device);
  bool bad = false;
  bad |= dalloc(h, &h->key_csr, N) != cudaSuccess;
  bad |= dalloc(h, &h->drow, N) != cudaSuccess;
  bad |= dalloc(h, &h->k0, N) != cudaSuccess;
  bad |= dalloc(h, &h->v0, N) != cudaSuccess;
  if (h->world == 1) {
    bad |= dalloc(h, &h->sk_set[1], N) != cudaSuccess;
    bad |= dalloc(h, &h->sp_set[1], N) != cudaSuccess;
    bad |= dalloc(h, &h->sort_scratch, N) != cudaSuccess;
  }
  bad |= dalloc(h, &h->k1, N) != cudaSuccess;
  bad |= dalloc(h, &h->v1, N) != cudaSuccess;
  bad |= dalloc(h, &h->blen, SB) != cudaSuccess;
  const int64_t sort_n = std::max<int64_t>(N, h->recv_cap);
  uint32_t *sort_words = nullptr;
  const size_t sww = sort_workspace_words(sort_n);
  bad |= dalloc(h, &sort_words, sww) != cudaSuccess;
  bad |= dalloc(h, &h->partials, (size_t)2 * nwarps_max * h->D) != cudaSuccess;
  bad |= dalloc(h, &h->tickets, nticket) != cudaSuccess;
  bad |= dalloc(h, &h->useg, sort_n) != cudaSuccess;
  bad |= dalloc(h, &h->ukey, sort_n) != cudaSuccess;
  bad |= dalloc(h, &h->ustart, sort_n + 1) != cudaSuccess;
  bad |= dalloc(h, &h->uend, sort_n + 1) != cudaSuccess;
  bad |= dalloc(h, &h->u_count, 2) != cudaSuccess;
  bad |= dalloc(h, &h->uniq_status, unique_status_words(sort_n)) != cudaSuccess;
  bad |= dalloc(h, &h->uniq_counter, 1) != cudaSuccess;
  bad |= dalloc(h, &h->fin, 3) != cudaSuccess;
  bad |= dalloc(h, &h->err_dev, 1) != cudaSuccess;
  if (W > 1) {
    bad |= dalloc(h, &h->inv, N) != cudaSuccess;
    bad |= dalloc(h, &h->send_keys, N) != cudaSuccess;
    bad |= dalloc(h, &h->recv_keys, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->owner_rows, (size_t)h->recv_cap * h->D) != cudaSuccess;
    bad |= dalloc(h, &h->uniq_rows, (size_t)N * h->D) != cudaSuccess;
    bad |= dalloc(h, &h->gloc, (size_t)N * h->D) != cudaSuccess;
    bad |= dalloc(h, &h->grecv, (size_t)h->recv_cap * h->D) != cudaSuccess;
    bad |= dalloc(h, &h->ok0, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->ov0, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->ok1, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->ov1, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->d_counts, 2 * EMB_MAX_WORLD) != cudaSuccess;
    bad |= dalloc(h, &h->ouseg, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->oukey, h->recv_cap) != cudaSuccess;
    bad |= dalloc(h, &h->oustart, h->recv_cap + 1) != cudaSuccess;
    bad |= dalloc(h, &h->ouend, h->recv_cap + 1) != cudaSuccess;
    bad |= dalloc(h, &h->ou_count, 2) != cudaSuccess;
    bad |= dalloc(h, &h->ouniq_status, unique_status_words(h->recv_cap)) != cudaSuccess;
    bad |= dalloc(h, &h->ouniq_counter, 1) != cudaSuccess;
    bad |= dalloc(h, &h->sp, N) != cudaSuccess;
    bad |= dalloc(h, &h->outidx, N) != cudaSuccess;
    bad |= dalloc(h, &h->tcnt, (size_t)((N + 2047) / 2048 + 1) * EMB_MAX_WORLD) != cudaSuccess;
  }
  if (bad) return fail(h, EMB_ERR_NOMEM, "cannot allocate the step workspace");
  h->sk_set[0] = h->k0;
  h->sp_set[0] = h->v0;
  h->sws.hist = sort_words;
  h->sws.counters = sort_words + 4 * 256;
  h->sws.status = sort_words + 4 * 256 + 4;
  h->sws.max_tiles = (sort_n + 4095) / 4096 + 1;
  h->sws.err = h->err_dev;
  CUDA_TRY(h, cudaMemset(h->tickets, 0, sizeof(uint32_t) * nticket));
  // table groups of the slot-major CSR (segsort fast path needs a non-decreasing slot_table)
  {
    h->segsort_ok = true;
    for (int s = 1; s < h->S; ++s)
      if (h->slot_table[s] < h->slot_table[s - 1]) h->segsort_ok = false;
    if (h->segsort_ok) {
      std::vector<int32_t> gslot;
      std::vector<uint64_t> gbase;
      std::vector<uint32_t> grows, gbits;
      for (int s = 0; s < h->S; ++s) {
        if (s == 0 || h->slot_table[s] != h->slot_table[s - 1]) {
          const int t = h->slot_table[s];
          gslot.push_back(s);
          gbase.push_back(h->base[t]);
          grows.push_back((uint32_t)h->rows[t]);
          gbits.push_back(bits_for((uint64_t)h->rows[t]));
        }
      }
      gslot.push_back(h->S);
      h->G = (int32_t)gbase.size();
      // key ranges (CTAs) per group: ~4K occurrences per CTA at the capacity bound (K sweep on C2:
      // K=2/4/8/16 -> 206/157/176/201 us per step); every CTA scans
      // its whole group, so K stays small
      const int64_t per = (h->max_ids + h->G - 1) / h->G;
      h->segK = (int32_t)std::min<int64_t>(16, std::max<int64_t>(1, (per + 4095) / 4096));
      if (const char *ek = getenv("EMB_SEGK")) h->segK = std::max(1, std::min(32, atoi(ek)));  // experiment knob
      if (dalloc(h, &h->run_k, h->max_ids) || dalloc(h, &h->run_i, h->max_ids))
        return fail(h, EMB_ERR_NOMEM, "alloc sort runs");
      if (dalloc(h, &h->d_gslot, gslot.size()) || dalloc(h, &h->d_gbase, h->G) || dalloc(h, &h->d_grows, h->G) ||
          dalloc(h, &h->d_gbits, h->G))
        return fail(h, EMB_ERR_NOMEM, "alloc groups");
      CUDA_TRY(h, cudaMemcpy(h->d_gslot, gslot.data(), sizeof(int32_t) * gslot.size(), cudaMemcpyHostToDevice));
      CUDA_TRY(h, cudaMemcpy(h->d_gbase, gbase.data(), sizeof(uint64_t) * h->G, cudaMemcpyHostToDevice));
      CUDA_TRY(h, cudaMemcpy(h->d_grows, grows.data(), sizeof(uint32_t) * h->G, cudaMemcpyHostToDevice));
      CUDA_TRY(h, cudaMemcpy(h->d_gbits, gbits.data(), sizeof(uint32_t) * h->G, cudaMemcpyHostToDevice));
    }
  }
  CUDA_TRY(h, cudaMemset(h->err_dev, 0, sizeof(uint32_t)));
  CUDA_TRY(h, cudaMemset(h->fin, 0, 3 * sizeof(uint32_t)));
  CUDA_TRY(h, cudaMemset(h->uniq_counter, 0, sizeof(uint32_t)));
  CUDA_TRY(h, cudaMemset(h->uniq_status, 0, sizeof(uint64_t) * unique_status_words(sort_n)));
  if (h->ouniq_status) {
    CUDA_TRY(h, cudaMemset(h->ouniq_counter, 0, sizeof(uint32_t)));
    CUDA_TRY(h, cudaMemset(h->ouniq_status, 0, sizeof(uint64_t) * unique_status_words(h->recv_cap)));
  }
  CUDA_TRY(h, cudaMemset(h->u_count, 0, 2 * sizeof(uint32_t)));
  void *hp = nullptr;
  if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) != cudaSuccess)
    return fail(h, EMB_ERR_NOMEM, "cannot allocate pinned error word");
  h->err_host = static_cast<uint32_t *>(hp);
  *h->err_host = 0;
  CUDA_TRY(h, cudaHostGetDevicePointer(reinterpret_cast<void **>(&h->err_host_dev), hp, 0));
  if (W > 1) {
    void *hc = nullptr;
    if (cudaHostAlloc(&hc, sizeof(int64_t) * (2 * EMB_MAX_WORLD + 2), cudaHostAllocDefault) != cudaSuccess)
      return fail(h, EMB_ERR_NOMEM, "cannot allocate pinned counts");
    h->h_counts = static_cast<int64_t *>(hc);
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    NCCL_TRY(h, ncclCommInitRank(&h->comm, W, id, h->rank));
    const char *ex = getenv("EMB_EXCHANGE");  // "nccl" selects the v1 grouped send/recv exchange
    h->use_p2p = h->segsort_ok && !(ex && std::strcmp(ex, "nccl") == 0);
    if (h->use_p2p) {
      emb_status_t ps = setup_p2p(h);
      if (ps != EMB_OK) return ps;
    }
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->side));
  CUDA_TRY(h, cudaDeviceSynchronize());
  return EMB_OK;
}

void destroy_impl(emb_ctx *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (void *p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  if (h->comm) ncclCommDestroy(h->comm);
  for (void *p : h->allocs) cudaFree(p);
  if (h->err_host) cudaFreeHost(h->err_host);
  if (h->h_counts) cudaFreeHost(h->h_counts);
  for (cudaEvent_t e : h->prof_ev) cudaEventDestroy(e);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_pf) cudaEventDestroy(h->ev_pf);
  if (h->side) cudaStreamDestroy(h->side);
  delete h;
}

// ------------------------------------------------------------------------------------------------
#define LAUNCH(h, kid, st, expr)                                   \
  do {                                                             \
    prof_hook(h, kid, 0, st);                                      \
    cudaError_t e__ = (expr);                                      \
    prof_hook(h, kid, 1, st);                                      \
    if (e__ != cudaSuccess)                                        \
      return fail(h, EMB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
    ++h->launches;                                                 \
  } while (0)

emb_status_t exchange(emb_ctx *h, const void *sendbuf, const int64_t *scnt, const int64_t *soff, void *recvbuf,
                      const int64_t *rcnt, const int64_t *roff, size_t elem_bytes, ncclDataType_t dt,
                      int64_t elems_per_item, cudaStream_t st) {
  prof_hook(h, KID_NCCL, 0, st);
  NCCL_TRY(h, ncclGroupStart());
  for (int p = 0; p < h->world; ++p) {
    if (scnt[p] > 0)
      NCCL_TRY(h, ncclSend(static_cast<const char *>(sendbuf) + (size_t)soff[p] * elems_per_item * elem_bytes,
                           (size_t)scnt[p] * elems_per_item, dt, p, h->comm, st));
    if (rcnt[p] > 0)
      NCCL_TRY(h, ncclRecv(static_cast<char *>(recvbuf) + (size_t)roff[p] * elems_per_item * elem_bytes,
                           (size_t)rcnt[p] * elems_per_item, dt, p, h->comm, st));
  }
  NCCL_TRY(h, ncclGroupEnd());
  prof_hook(h, KID_NCCL, 1, st);
  ++h->launches;
  return EMB_OK;
}

// per-table sort arguments (W = 1 path) writing sort-output set `set`
SegSortArgs segsort_args(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz, int set) {
  SegSortArgs sa{};
  sa.ids = ids;
  sa.offsets = offsets;
  sa.nnz = nnz;
  sa.batch = batch;
  sa.gslot = h->d_gslot;
  sa.gbase = h->d_gbase;
  sa.grows = h->d_grows;
  sa.gbits = h->d_gbits;
  sa.skey = h->sk_set[set];
  sa.spay = h->sp_set[set];
  sa.scratch_k = h->k1;
  sa.scratch_a = h->v1;
  sa.scratch_b = h->sort_scratch;
  sa.run_k = h->run_k;
  sa.run_i = h->run_i;
  sa.K = h->segK;
  sa.err = h->err_dev;
  sa.err_host = h->err_host_dev;
  sa.fin = nullptr;
  return sa;
}

emb_status_t lookup_prefetch_impl(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch,
                                  int64_t nnz, cudaStream_t st) {
  if (batch < 0 || batch > h->max_batch || nnz < 0 || nnz > h->max_ids || (batch == 0 && nnz != 0))
    return fail(h, EMB_ERR_INVALID, "prefetch: batch / nnz out of range");
  if ((batch > 0 && !offsets) || (nnz > 0 && !ids)) return fail(h, EMB_ERR_INVALID, "prefetch: NULL ids/offsets");
  h->pf.valid = false;
  if (h->world != 1 || !h->segsort_ok || batch == 0 || nnz == 0) return EMB_OK;  // nothing to overlap
  CUDA_TRY(h, cudaSetDevice(h->device));
  // ordered after everything already on the caller stream (the inputs, the current lookup), not after
  // the backward the caller enqueues next: the sort of step k+1 overlaps the gradient pass of step k.
  // It writes the sort-output set the pending backward does not read.
  CUDA_TRY(h, cudaEventRecord(h->ev_pf, st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_pf, 0));
  const int set = h->cur_set ^ 1;
  SegSortArgs sa = segsort_args(h, ids, offsets, batch, nnz, set);
  LAUNCH(h, KID_SORT_PASS, h->side, launch_segsort(sa, h->G, h->side));
  h->pf.valid = true;
  h->pf.ids = ids;
  h->pf.offsets = offsets;
  h->pf.batch = batch;
  h->pf.nnz = nnz;
  h->pf.set = set;
  return EMB_OK;
}

emb_status_t lookup_impl(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                         float *out, cudaStream_t st) {
  if (h->state != 0) return fail(h, EMB_ERR_STATE, "emb_lookup called twice without emb_backward_update");
  if (batch < 0 || batch > h->max_batch) return fail(h, EMB_ERR_INVALID, "batch out of [0, max_batch]");
  if (nnz < 0 || nnz > h->max_ids) return fail(h, EMB_ERR_INVALID, "nnz out of [0, max_ids]");
  if (batch == 0 && nnz != 0) return fail(h, EMB_ERR_INVALID, "nnz must be 0 when batch == 0");
  if ((batch > 0 && (!offsets || !out)) || (nnz > 0 && !ids))
    return fail(h, EMB_ERR_INVALID, "NULL ids/offsets/out");
  if (batch > 0 && !aligned16(out)) return fail(h, EMB_ERR_INVALID, "out must be 16-byte aligned");
  emb_status_t s = check_sticky(h);
  if (s != EMB_OK) return s;
  CUDA_TRY(h, cudaSetDevice(h->device));
  h->launches = 0;
  h->batch = batch;
  h->nnz = nnz;
  h->last_stream = st;
  const bool mean = h->pool == EMB_POOL_MEAN;

  KeysArgs ka{};
  ka.ids = ids;
  ka.offsets = offsets;
  ka.nnz = nnz;
  ka.batch = batch;
  ka.num_slots = h->S;
  ka.slot_table = h->d_slot_table;
  ka.base = h->d_base;
  ka.rows = h->d_rows;
  ka.ks = h->ks;
  ka.key = h->key_csr;
  ka.drow = h->drow;
  ka.blen = h->blen;
  ka.err = h->err_dev;
  // with the per-table sort, the pool and the sort read the ids themselves (no key kernel); at W > 1
  // the pool then takes each occurrence's received row through row_idx
  const bool direct = h->segsort_ok;
  if (batch > 0 && !direct) LAUNCH(h, KID_KEYS, st, launch_keys(ka, st));

  PoolArgs pa{};
  pa.key = h->key_csr;
  pa.offsets = offsets;
  pa.nnz = nnz;
  pa.batch = batch;
  pa.num_slots = h->S;
  pa.dim = h->D;
  pa.mean = mean;
  pa.out = out;
  pa.err = h->err_dev;
  pa.err_host = h->err_host_dev;
  if (direct) {
    pa.ids = ids;
    pa.slot_table = h->d_slot_table;
    pa.base = h->d_base;
    pa.rows = h->d_rows;
    pa.drow = h->drow;
    pa.blen = mean ? h->blen : nullptr;
  }

  if (h->world == 1) {
    // fork: the sort runs on the side stream while the pool streams rows on the caller stream
    CUDA_TRY(h, cudaEventRecord(h->ev_fork, st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    // a sort prefetched for exactly these inputs (emb_lookup_prefetch) is already queued on the side
    // stream: consume it (the join below waits for it)
    const bool use_pf = h->pf.valid && h->pf.ids == ids && h->pf.offsets == offsets && h->pf.batch == batch &&
                        h->pf.nnz == nnz;
    h->pf.valid = false;
    if (use_pf) {
      h->cur_set = h->pf.set;
      h->skey = h->sk_set[h->cur_set];
      h->spay = h->sp_set[h->cur_set];
    } else if (h->segsort_ok) {
      h->cur_set ^= 1;  // (stream-ordered after the previous backward: either set is free)
      SegSortArgs sa = segsort_args(h, ids, offsets, batch, nnz, h->cur_set);
      sa.fin = (batch > 0 && nnz > 0) ? h->fin : nullptr;  // the later of sort / pool publishes the error word
      h->skey = sa.skey;
      h->spay = sa.spay;
      static int serial = -1;  // experiment knob: EMB_SERIAL=1 runs the sort before the pool (no overlap)
      if (serial < 0) serial = getenv("EMB_SERIAL") ? atoi(getenv("EMB_SERIAL")) : 0;
      cudaStream_t ss = serial ? st : h->side;
      if (batch > 0) LAUNCH(h, KID_SORT_PASS, ss, launch_segsort(sa, h->G, ss));
    } else {
      int nl = 0;
      cudaError_t e = radix_sort_pairs(h->sws, h->key_csr, nullptr, h->k0, h->v0, h->k1, h->v1, nnz,
                                       h->ks.key_bits, h->side, &h->skey, &h->spay, &nl, prof_hook, h);
      if (e != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("radix sort: ") + cudaGetErrorString(e));
      h->launches += nl;
    }
    pa.rows_src = h->w;
    pa.nrows_src = h->rows_local;
    pa.row_idx = nullptr;
    const bool fused_pub = h->segsort_ok && batch > 0 && nnz > 0;
    pa.fin = fused_pub ? h->fin : nullptr;
    pa.fin_kernels = use_pf ? 1 : 2;  // a prefetched sort does not take part in the publish
    if (batch > 0) LAUNCH(h, KID_POOL, st, launch_pool(pa, st));
    CUDA_TRY(h, cudaEventRecord(h->ev_join, h->side));
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_join, 0));
    if (batch > 0 && !fused_pub) LAUNCH(h, KID_KEYS, st, launch_publish_err(h->err_dev, h->err_host_dev, st));
    h->U_l = -1;  // computed on demand
    h->state = 1;
    return EMB_OK;
  }

  // ---------------- world > 1
  const int W = h->world;
  int nl = 0;
  cudaError_t e = cudaSuccess;
  if (h->segsort_ok) {
    // per-table sort by fused key g, dedup, then a stable partition of the distinct keys by owner
    SegSortArgs sa{};
    sa.ids = ids;
    sa.offsets = offsets;
    sa.nnz = nnz;
    sa.batch = batch;
    sa.gslot = h->d_gslot;
    sa.gbase = h->d_gbase;
    sa.grows = h->d_grows;
    sa.gbits = h->d_gbits;
    sa.skey = h->k0;
    sa.spay = h->v0;
    sa.scratch_k = h->k1;
    sa.scratch_a = h->v1;
    sa.scratch_b = h->outidx;  // overwritten later in this step
    sa.run_k = h->run_k;
    sa.run_i = h->run_i;
    sa.K = h->segK;
    sa.err = h->err_dev;
    h->skey = h->k0;
    h->spay = h->v0;
    if (batch > 0) LAUNCH(h, KID_SORT_PASS, st, launch_segsort(sa, h->G, st));
    UniqueArgs ua{h->skey, nnz, h->useg, h->ukey, h->ustart, h->uend, h->u_count, h->uniq_status, h->uniq_counter, ++h->uniq_epoch};
    LAUNCH(h, KID_UNIQUE, st, launch_unique(ua, st));
    LAUNCH(h, KID_ROUTE, st,
           launch_partition(h->ukey, h->u_count, nnz, h->ks, h->tcnt, h->send_keys, h->sp, h->d_counts, st));
    LAUNCH(h, KID_ROUTE, st, launch_outidx(h->skey, h->spay, h->useg, h->sp, nnz, h->outidx, h->inv, st));
    h->ukey_is_g = true;
  } else {
    e = radix_sort_pairs(h->sws, h->key_csr, nullptr, h->k0, h->v0, h->k1, h->v1, nnz, h->ks.key_bits, st,
                         &h->skey, &h->spay, &nl, prof_hook, h);
    if (e != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("radix sort: ") + cudaGetErrorString(e));
    h->launches += nl;
    UniqueArgs ua{h->skey, nnz, h->useg, h->ukey, h->ustart, h->uend, h->u_count, h->uniq_status, h->uniq_counter, ++h->uniq_epoch};
    LAUNCH(h, KID_UNIQUE, st, launch_unique(ua, st));
    LAUNCH(h, KID_ROUTE, st, launch_owner_counts(h->ukey, h->u_count, W, h->ks.lbits, h->d_counts, st));
    LAUNCH(h, KID_ROUTE, st, launch_scatter_inverse(h->skey, h->spay, h->useg, nnz, h->inv, st));
    LAUNCH(h, KID_ROUTE, st, launch_local_of_unique(h->ukey, h->u_count, nnz, h->lmask, h->send_keys, st));
    h->ukey_is_g = false;
  }
  if (h->use_p2p) {
    // ---- peer-memory exchange: no host synchronisation
    P2PArgs px = h->p2p;
    px.epoch = ++h->epoch;
    const int64_t cap = h->recv_cap;
    // X0 (counts + wait + route table), X1 (keys; its last block raises KEYS)
    LAUNCH(h, KID_NCCL, st, launch_xcounts(px, h->d_counts, h->err_dev, st));
    LAUNCH(h, KID_ROUTE, st, launch_push_keys(px, h->send_keys, nnz, st));
    // consumers wait in a one-thread kernel, not in their own prologue: a spinning grid would hold
    // SMs the concurrent side-stream merge and the gather need (measured slower at W = 4)
    LAUNCH(h, KID_WAIT, st, launch_wait(px, P2P_KEYS, h->err_dev, st));
    // owner side: stable W-way merge of the received runs, overlapped with the gather-push
    CUDA_TRY(h, cudaEventRecord(h->ev_fork, st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    h->okey = h->ok0;
    h->opay = h->ov0;
    const bool fused_pub = batch > 0 && direct;  // the later of merge / pool publishes the error word
    LAUNCH(h, KID_MERGE, h->side,
           launch_merge_tree(h->recv_keys, h->rt->recv_counts, W, cap, h->ok0, h->ov0, h->ok1, h->ov1, h->err_dev,
                             h->side, fused_pub ? h->fin : nullptr, h->err_host_dev));
    // X2 fused with the gather (its last block raises ROWS)
    LAUNCH(h, KID_OWNER_GATHER, st,
           launch_gather_push(px, h->w, h->recv_keys, h->D, cap, h->rows_local, h->err_dev, st));
    LAUNCH(h, KID_WAIT, st, launch_wait(px, P2P_ROWS, h->err_dev, st));
    pa.rows_src = h->uniq_rows;
    pa.nrows_src = h->max_ids;
    pa.row_idx = h->inv;
    pa.fin = fused_pub ? h->fin : nullptr;
    pa.fin_kernels = 2;
    if (batch > 0) LAUNCH(h, KID_POOL, st, launch_pool(pa, st));
    CUDA_TRY(h, cudaEventRecord(h->ev_join, h->side));
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_join, 0));
    if (batch > 0 && !fused_pub) LAUNCH(h, KID_KEYS, st, launch_publish_err(h->err_dev, h->err_host_dev, st));
    h->counts_synced = false;
    h->U_l = -1;
    h->n_recv = -1;
    h->owner_unique_done = false;
    h->state = 1;
    return EMB_OK;
  }
  // X0: per-peer counts
  {
    int64_t ones[EMB_MAX_WORLD], offs[EMB_MAX_WORLD];
    for (int p = 0; p < W; ++p) {
      ones[p] = 1;
      offs[p] = p;
    }
    emb_status_t es = exchange(h, h->d_counts, ones, offs, h->d_counts + EMB_MAX_WORLD, ones, offs, sizeof(int64_t),
                               ncclInt64, 1, st);
    if (es != EMB_OK) return es;
  }
  CUDA_TRY(h, cudaMemcpyAsync(h->h_counts, h->d_counts, sizeof(int64_t) * 2 * EMB_MAX_WORLD, cudaMemcpyDeviceToHost,
                              st));
  CUDA_TRY(h, cudaStreamSynchronize(st));  // v1: the host sizes the all-to-allv from the counts
  h->soff[0] = h->roff[0] = 0;
  for (int p = 0; p < W; ++p) {
    h->send_counts[p] = h->h_counts[p];
    h->recv_counts[p] = h->h_counts[EMB_MAX_WORLD + p];
    h->soff[p + 1] = h->soff[p] + h->send_counts[p];
    h->roff[p + 1] = h->roff[p] + h->recv_counts[p];
  }
  h->U_l = h->soff[W];
  h->n_recv = h->roff[W];
  if (h->n_recv > h->recv_cap) return fail(h, EMB_ERR_INVALID, "received keys exceed the receive capacity");
  // X1: local ids to their owners
  emb_status_t es = exchange(h, h->send_keys, h->send_counts, h->soff, h->recv_keys, h->recv_counts, h->roff,
                             sizeof(uint32_t), ncclUint32, 1, st);
  if (es != EMB_OK) return es;
  // owner side: the W received runs are each sorted by local id -> stable W-way merge (source-rank
  // order inside a row) on the side stream, overlapped with the gather and X2
  CUDA_TRY(h, cudaEventRecord(h->ev_fork, st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  if (h->ukey_is_g || h->shard == 1) {
    h->okey = h->ok0;
    h->opay = h->ov0;
    LAUNCH(h, KID_SORT_PASS, h->side,
           launch_merge_runs(h->recv_keys, h->d_counts + EMB_MAX_WORLD, W, h->n_recv, h->okey, h->opay, h->err_dev,
                             h->side));
  } else {
    e = radix_sort_pairs(h->sws, h->recv_keys, nullptr, h->ok0, h->ov0, h->ok1, h->ov1, h->n_recv, h->owner_key_bits,
                         h->side, &h->okey, &h->opay, &nl, prof_hook, h);
    if (e != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("owner sort: ") + cudaGetErrorString(e));
    h->launches += nl;
  }
  h->owner_unique_done = false;  // the owner-side dedup is only built on demand (step statistics)
  // gather requested rows and send them back
  LAUNCH(h, KID_OWNER_GATHER, st, launch_owner_gather(h->w, h->recv_keys, h->n_recv, h->D, h->owner_rows, st));
  es = exchange(h, h->owner_rows, h->recv_counts, h->roff, h->uniq_rows, h->send_counts, h->soff, sizeof(float),
                ncclFloat32, h->D, st);
  if (es != EMB_OK) return es;
  pa.rows_src = h->uniq_rows;
  pa.nrows_src = h->U_l;
  pa.row_idx = h->inv;
  if (batch > 0) LAUNCH(h, KID_POOL, st, launch_pool(pa, st));
  CUDA_TRY(h, cudaEventRecord(h->ev_join, h->side));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_join, 0));
  if (batch > 0) LAUNCH(h, KID_KEYS, st, launch_publish_err(h->err_dev, h->err_host_dev, st));
  h->state = 1;
  return EMB_OK;
}

emb_status_t backward_impl(emb_ctx *h, const float *d_out, double lr, cudaStream_t st) {
  if (h->state != 1) return fail(h, EMB_ERR_STATE, "emb_backward_update without a preceding emb_lookup");
  if (h->batch > 0 && (!d_out || !aligned16(d_out)))
    return fail(h, EMB_ERR_INVALID, "d_out must be a non-NULL 16-byte aligned device pointer");
  CUDA_TRY(h, cudaSetDevice(h->device));
  h->last_stream = st;
  const bool mean = h->pool == EMB_POOL_MEAN;
  GradArgs g{};
  g.signal_kind = -1;
  g.dim = h->D;
  g.dy = d_out;
  g.drow = h->drow;
  g.blen = mean ? h->blen : nullptr;
  g.batch = h->batch;
  g.num_slots = h->S;
  g.opt = h->opt;
  g.lr = lr;
  g.eps = h->eps;
  g.w = h->w;
  g.a = h->a;
  g.partials = h->partials;
  g.tickets = h->tickets;
  g.nrows = h->rows_local;
  g.nsrc = (int64_t)h->S * h->batch;
  g.nsrc_occ = h->nnz;
  g.nout = h->U_l;
  g.err = h->err_dev;
  g.useg = h->useg;
  g.ustart = h->ustart;
  g.u_count = h->u_count;
  if (h->world == 1) {
    g.skey = h->skey;
    g.spay = h->spay;
    g.n = h->nnz;
    g.src_mode = 0;
    g.sink_mode = 0;
    g.lmask = 0xFFFFFFFFu;
    LAUNCH(h, KID_GRAD_APPLY, st, launch_grad(g, st));
    h->state = 0;
    return EMB_OK;
  }
  if (h->use_p2p) {
    // requester: merged per-key gradients stored straight into the owners' receive buffers (fused X3)
    P2PArgs px = h->p2p;
    px.epoch = h->epoch;
    g.skey = h->skey;
    g.spay = h->spay;
    g.n = h->nnz;
    g.src_mode = 0;
    g.sink_mode = 2;
    g.useg = h->outidx;
    g.nout = h->max_ids;
    g.p2p = px;
    static int push = -1;  // experiment knob: EMB_GRAD_PUSH=1 -> local merge (MODE 2) + streaming push
    if (push < 0) push = getenv("EMB_GRAD_PUSH") ? atoi(getenv("EMB_GRAD_PUSH")) : 0;
    if (push && g.n > 0) {
      g.sink_mode = 1;
      g.out_rows = h->gloc;
      LAUNCH(h, KID_GRAD_LOCAL, st, launch_grad(g, st));
      LAUNCH(h, KID_NCCL, st, launch_push_rows(px, h->gloc, h->D, h->max_ids, st));
    } else {
    g.signal_kind = P2P_GRADS;  // the last warp of the requester grad raises GRADS
    if (g.n > 0)
      LAUNCH(h, KID_GRAD_LOCAL, st, launch_grad(g, st));
    else
      LAUNCH(h, KID_NCCL, st, launch_signal(px, P2P_GRADS, st));
    }
    // owner: merge the W sources' gradients per row (source-rank order) and apply
    GradArgs o = g;
    o.skey = h->okey;
    o.spay = h->opay;
    o.n = h->recv_cap;
    o.n_dev = &h->rt->n_recv;
    o.src_mode = 1;
    o.src = h->grecv;
    o.nsrc = h->recv_cap;
    o.blen = nullptr;
    o.sink_mode = 0;
    o.lmask = 0xFFFFFFFFu;
    o.signal_kind = -1;
    LAUNCH(h, KID_WAIT, st, launch_wait(px, P2P_GRADS, h->err_dev, st));
    LAUNCH(h, KID_GRAD_APPLY, st, launch_grad(o, st));
    h->state = 0;
    return EMB_OK;
  }
  // requester: per-unique-key local gradient (fp32 rows in unique order = owner-grouped send order)
  g.skey = h->skey;
  g.spay = h->spay;
  g.n = h->nnz;
  g.src_mode = 0;
  g.sink_mode = 1;
  g.out_rows = h->gloc;
  if (h->ukey_is_g) g.useg = h->outidx;  // merged gradient of a key goes to its send position
  LAUNCH(h, KID_GRAD_LOCAL, st, launch_grad(g, st));
  emb_status_t es = exchange(h, h->gloc, h->send_counts, h->soff, h->grecv, h->recv_counts, h->roff, sizeof(float),
                             ncclFloat32, h->D, st);
  if (es != EMB_OK) return es;
  // owner: merge the W sources' gradients per row (source-rank order) and apply
  GradArgs o = g;
  o.skey = h->okey;
  o.spay = h->opay;
  o.n = h->n_recv;
  o.src_mode = 1;
  o.src = h->grecv;
  o.nsrc = h->n_recv;
  o.useg = h->ouseg;
  o.ustart = h->oustart;
  o.u_count = h->ou_count;
  o.blen = nullptr;
  o.sink_mode = 0;
  o.lmask = 0xFFFFFFFFu;
  LAUNCH(h, KID_GRAD_APPLY, st, launch_grad(o, st));
  h->state = 0;
  return EMB_OK;
}

// host-side unique of the last step (runs the GPU dedup kernel if the step did not)
emb_status_t ensure_unique(emb_ctx *h) {
  if (h->world > 1) return sync_counts(h);
  if (h->U_l >= 0) return EMB_OK;
  // world == 1: the step itself never needs the compacted unique list; build it on demand
  cudaStream_t st = h->last_stream;
  UniqueArgs ua{h->skey, h->nnz, h->useg, h->ukey, h->ustart, h->uend, h->u_count, h->uniq_status, h->uniq_counter, ++h->uniq_epoch};
  CUDA_TRY(h, launch_unique(ua, st));
  uint32_t u = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&u, h->u_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  h->U_l = u;
  return EMB_OK;
}

// owner-side dedup of the merged received keys, built on demand (not part of the step)
emb_status_t ensure_owner_unique(emb_ctx *h) {
  if (h->world > 1) {
    emb_status_t s = sync_counts(h);
    if (s != EMB_OK) return s;
  }
  if (h->world == 1 || h->owner_unique_done || h->n_recv <= 0) return EMB_OK;
  cudaStream_t st = h->last_stream;
  UniqueArgs ua{h->okey, h->n_recv, h->ouseg, h->oukey, h->oustart, h->ouend, h->ou_count, h->ouniq_status,
                h->ouniq_counter, ++h->ouniq_epoch};
  CUDA_TRY(h, launch_unique(ua, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  h->owner_unique_done = true;
  return EMB_OK;
}

emb_status_t copy_unique(emb_ctx *h, const uint32_t *uend_dev, const uint32_t *ukey_dev, const uint32_t *ustart_dev,
                         int64_t U, bool routing_keys, bool owner_local_keys, uint64_t *keys_host,
                         int64_t *counts_host, int64_t cap, int64_t *n_out) {
  if (n_out) *n_out = U;
  if (cap < U) return fail(h, EMB_ERR_INVALID, "capacity smaller than the number of unique keys");
  std::vector<uint32_t> k(U), s(U), e(U);
  if (U > 0) {
    CUDA_TRY(h, cudaMemcpy(k.data(), ukey_dev, sizeof(uint32_t) * U, cudaMemcpyDeviceToHost));
    CUDA_TRY(h, cudaMemcpy(s.data(), ustart_dev, sizeof(uint32_t) * U, cudaMemcpyDeviceToHost));
    CUDA_TRY(h, cudaMemcpy(e.data(), uend_dev, sizeof(uint32_t) * U, cudaMemcpyDeviceToHost));
  }
  for (int64_t u = 0; u < U; ++u) {
    if (keys_host) {
      uint64_t g;
      if (owner_local_keys) {
        // owner-side local id -> global
        const uint64_t local = k[u];
        g = h->shard == 0 ? local * (uint64_t)h->world + (uint64_t)h->rank : (uint64_t)h->rank * h->ks.rows_per + local;
      } else {
        g = routing_keys ? key_to_global(k[u], h->ks) : k[u];
      }
      keys_host[u] = g;
    }
    if (counts_host) counts_host[u] = (int64_t)e[u] - (int64_t)s[u];
  }
  if (keys_host && !owner_local_keys && h->world > 1) {
    // requester keys are owner-major; report them sorted by global key like the oracle's U
    std::vector<std::pair<uint64_t, int64_t>> v(U);
    for (int64_t u = 0; u < U; ++u) v[u] = {keys_host[u], counts_host ? counts_host[u] : 0};
    std::sort(v.begin(), v.end());
    for (int64_t u = 0; u < U; ++u) {
      keys_host[u] = v[u].first;
      if (counts_host) counts_host[u] = v[u].second;
    }
  }
  return EMB_OK;
}

}  // namespace

// =================================================================================================
extern "C" {

emb_status_t emb_create(const emb_config_t *cfg, emb_handle_t *out) {
  if (!out) return EMB_ERR_INVALID;
  *out = nullptr;
  emb_ctx *h = new (std::nothrow) emb_ctx();
  if (!h) return EMB_ERR_NOMEM;
  emb_status_t s = create_impl(cfg, h);
  if (s != EMB_OK) {
    {
      std::lock_guard<std::mutex> lk(g_err_mu);
      g_create_error = h->last_error;
    }
    destroy_impl(h);
    return s;
  }
  *out = h;
  return EMB_OK;
}

emb_status_t emb_destroy(emb_handle_t h) {
  destroy_impl(h);
  return EMB_OK;
}

emb_status_t emb_get_unique_id(void *out128) {
  if (!out128) return EMB_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return EMB_ERR_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return EMB_OK;
}

emb_status_t emb_lookup(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                        float *out, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  return lookup_impl(h, ids, offsets, batch, nnz, out, static_cast<cudaStream_t>(cuda_stream));
}

emb_status_t emb_lookup_prefetch(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch,
                                 int64_t nnz, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  return lookup_prefetch_impl(h, ids, offsets, batch, nnz, static_cast<cudaStream_t>(cuda_stream));
}

emb_status_t emb_backward_update(emb_handle_t h, const float *d_out, double lr, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  emb_status_t s = check_sticky(h);
  if (s != EMB_OK) {
    h->state = 0;
    return s;
  }
  return backward_impl(h, d_out, lr, static_cast<cudaStream_t>(cuda_stream));
}

static emb_status_t ensure_staging(emb_ctx *h) {
  if (h->st_ids) return EMB_OK;
  const size_t SB = (size_t)h->S * h->max_batch;
  if (dalloc(h, &h->st_ids, h->max_ids) || dalloc(h, &h->st_offsets, SB + 1) ||
      dalloc(h, &h->st_out, SB * h->D) || dalloc(h, &h->st_dout, SB * h->D))
    return fail(h, EMB_ERR_NOMEM, "cannot allocate host-path staging");
  return EMB_OK;
}

emb_status_t emb_lookup_host(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                             float *out, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  if (batch < 0 || batch > h->max_batch || nnz < 0 || nnz > h->max_ids)
    return fail(h, EMB_ERR_INVALID, "batch/nnz out of range");
  if ((batch > 0 && (!offsets || !out)) || (nnz > 0 && !ids)) return fail(h, EMB_ERR_INVALID, "NULL host buffer");
  CUDA_TRY(h, cudaSetDevice(h->device));
  emb_status_t s = ensure_staging(h);
  if (s != EMB_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const size_t SB = (size_t)h->S * batch;
  if (nnz > 0) CUDA_TRY(h, cudaMemcpyAsync(h->st_ids, ids, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
  if (batch > 0)
    CUDA_TRY(h, cudaMemcpyAsync(h->st_offsets, offsets, sizeof(int64_t) * (SB + 1), cudaMemcpyHostToDevice, st));
  s = lookup_impl(h, h->st_ids, h->st_offsets, batch, nnz, h->st_out, st);
  if (s != EMB_OK) return s;
  if (batch > 0)
    CUDA_TRY(h, cudaMemcpyAsync(out, h->st_out, sizeof(float) * SB * h->D, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return check_sticky(h);
}

emb_status_t emb_backward_update_host(emb_handle_t h, const float *d_out, double lr, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  emb_status_t s = ensure_staging(h);
  if (s != EMB_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const size_t SB = (size_t)h->S * h->batch;
  if (h->state == 1 && h->batch > 0) {
    if (!d_out) return fail(h, EMB_ERR_INVALID, "NULL d_out");
    CUDA_TRY(h, cudaMemcpyAsync(h->st_dout, d_out, sizeof(float) * SB * h->D, cudaMemcpyHostToDevice, st));
  }
  s = emb_backward_update(h, h->st_dout, lr, st);
  if (s != EMB_OK) return s;
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return check_sticky(h);
}

emb_status_t emb_read_rows(emb_handle_t h, int32_t table, const int64_t *rows_host, int64_t n, float *w_host,
                           float *a_host) {
  if (!h) return EMB_ERR_INVALID;
  if (table < 0 || table >= h->T || n < 0 || (n > 0 && (!rows_host || !w_host)))
    return fail(h, EMB_ERR_INVALID, "bad table / rows / buffers");
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  CUDA_TRY(h, cudaDeviceSynchronize());
  if (n == 0) return EMB_OK;
  std::vector<int64_t> loc(n);
  for (int64_t i = 0; i < n; ++i) {
    if (rows_host[i] < 0 || rows_host[i] >= h->rows[table]) return fail(h, EMB_ERR_INVALID, "row out of range");
    const uint64_t g = h->base[table] + (uint64_t)rows_host[i];
    if (owner_of_global(h, g) != h->rank) return fail(h, EMB_ERR_INVALID, "row not owned by this rank");
    loc[i] = local_of_global(h, g);
  }
  int64_t *d_loc = nullptr;
  float *d_buf = nullptr;
  CUDA_TRY(h, cudaMalloc(&d_loc, sizeof(int64_t) * n));
  CUDA_TRY(h, cudaMalloc(&d_buf, sizeof(float) * n * h->D));
  cudaError_t e = cudaMemcpy(d_loc, loc.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_rows_gather(h->w, d_loc, n, h->D, d_buf, 0);
  if (e == cudaSuccess) e = cudaMemcpy(w_host, d_buf, sizeof(float) * n * h->D, cudaMemcpyDeviceToHost);
  const int32_t aw = accum_width(h);
  if (e == cudaSuccess && a_host) {
    if (h->a) {
      e = launch_rows_gather(h->a, d_loc, n, aw, d_buf, 0);
      if (e == cudaSuccess) e = cudaMemcpy(a_host, d_buf, sizeof(float) * n * aw, cudaMemcpyDeviceToHost);
    } else {
      std::fill(a_host, a_host + n * aw, 0.f);
    }
  }
  cudaFree(d_loc);
  cudaFree(d_buf);
  if (e != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("read_rows: ") + cudaGetErrorString(e));
  return EMB_OK;
}

emb_status_t emb_write_rows(emb_handle_t h, int32_t table, const int64_t *rows_host, int64_t n, const float *w_host,
                            const float *a_host) {
  if (!h) return EMB_ERR_INVALID;
  if (table < 0 || table >= h->T || n < 0 || (n > 0 && (!rows_host || !w_host)))
    return fail(h, EMB_ERR_INVALID, "bad table / rows / buffers");
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  CUDA_TRY(h, cudaDeviceSynchronize());
  if (n == 0) return EMB_OK;
  std::vector<int64_t> loc(n);
  for (int64_t i = 0; i < n; ++i) {
    if (rows_host[i] < 0 || rows_host[i] >= h->rows[table]) return fail(h, EMB_ERR_INVALID, "row out of range");
    const uint64_t g = h->base[table] + (uint64_t)rows_host[i];
    if (owner_of_global(h, g) != h->rank) return fail(h, EMB_ERR_INVALID, "row not owned by this rank");
    loc[i] = local_of_global(h, g);
  }
  int64_t *d_loc = nullptr;
  float *d_buf = nullptr;
  CUDA_TRY(h, cudaMalloc(&d_loc, sizeof(int64_t) * n));
  CUDA_TRY(h, cudaMalloc(&d_buf, sizeof(float) * n * h->D));
  cudaError_t e = cudaMemcpy(d_loc, loc.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_buf, w_host, sizeof(float) * n * h->D, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_rows_scatter(h->w, d_loc, n, h->D, d_buf, 0);
  if (e == cudaSuccess && a_host && h->a) {
    const int32_t aw = accum_width(h);
    e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(d_buf, a_host, sizeof(float) * n * aw, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_rows_scatter(h->a, d_loc, n, aw, d_buf, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(d_loc);
  cudaFree(d_buf);
  if (e != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("write_rows: ") + cudaGetErrorString(e));
  return EMB_OK;
}

emb_status_t emb_last_step_info(emb_handle_t h, emb_step_info_t *info) {
  if (!h || !info) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  emb_status_t s = ensure_unique(h);
  if (s != EMB_OK) return s;
  std::memset(info, 0, sizeof(*info));
  info->nnz = h->nnz;
  info->num_bags = (int64_t)h->S * h->batch;
  info->unique_local = h->U_l;
  info->world = h->world;
  info->launches = h->launches;
  if (h->world == 1) {
    info->unique_owner = h->U_l;
    info->recv_keys = h->U_l;
    info->send_counts[0] = h->U_l;
    info->recv_counts[0] = h->U_l;
  } else {
    info->recv_keys = h->n_recv;
    for (int p = 0; p < h->world; ++p) {
      info->send_counts[p] = h->send_counts[p];
      info->recv_counts[p] = h->recv_counts[p];
    }
    emb_status_t s2 = ensure_owner_unique(h);
    if (s2 != EMB_OK) return s2;
    uint32_t u = 0;
    CUDA_TRY(h, cudaMemcpy(&u, h->ou_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    info->unique_owner = h->n_recv > 0 ? u : 0;
  }
  return EMB_OK;
}

emb_status_t emb_last_unique(emb_handle_t h, uint64_t *keys_host, int64_t *counts_host, int64_t cap, int64_t *n_out) {
  if (!h) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  emb_status_t s = ensure_unique(h);
  if (s != EMB_OK) return s;
  uint32_t U = 0;
  CUDA_TRY(h, cudaMemcpy(&U, h->u_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return copy_unique(h, h->uend, h->ukey, h->ustart, U, !h->ukey_is_g, false, keys_host, counts_host, cap, n_out);
}

emb_status_t emb_last_owner_unique(emb_handle_t h, uint64_t *keys_host, int64_t *counts_host, int64_t cap,
                                   int64_t *n_out) {
  if (!h) return EMB_ERR_INVALID;
  if (h->world == 1) return emb_last_unique(h, keys_host, counts_host, cap, n_out);
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  uint32_t U = 0;
  if (h->n_recv > 0) CUDA_TRY(h, cudaMemcpy(&U, h->ou_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return copy_unique(h, h->ouend, h->oukey, h->oustart, U, false, true, keys_host, counts_host, cap, n_out);
}

int64_t emb_rows_local(emb_handle_t h) { return h ? h->rows_local : -1; }

emb_status_t emb_profile_enable(emb_handle_t h, int32_t on) {
  if (!h) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (on && h->prof_ev.empty()) {
    h->prof_ev.resize(2 * 16384);
    for (auto &e : h->prof_ev) CUDA_TRY(h, cudaEventCreate(&e));
  }
  h->prof_on = on != 0;
  return EMB_OK;
}

emb_status_t emb_profile_reset(emb_handle_t h) {
  if (!h) return EMB_ERR_INVALID;
  if (h->last_stream) cudaStreamSynchronize(h->last_stream);
  h->prof_used = 0;
  h->prof_kid.clear();
  for (int k = 0; k < KID_COUNT; ++k) {
    h->prof_ms[k] = 0;
    h->prof_cnt[k] = 0;
  }
  return EMB_OK;
}

emb_status_t emb_profile_read(emb_handle_t h, double *ms, int64_t *launches, int32_t cap, int32_t *n) {
  if (!h) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  CUDA_TRY(h, cudaDeviceSynchronize());
  for (size_t i = 0; i < h->prof_kid.size(); ++i) {
    float t = 0;
    CUDA_TRY(h, cudaEventElapsedTime(&t, h->prof_ev[2 * i], h->prof_ev[2 * i + 1]));
    h->prof_ms[h->prof_kid[i]] += t;
    h->prof_cnt[h->prof_kid[i]] += 1;
  }
  h->prof_kid.clear();
  h->prof_used = 0;
  if (n) *n = KID_COUNT;
  for (int k = 0; k < KID_COUNT && k < cap; ++k) {
    if (ms) ms[k] = h->prof_ms[k];
    if (launches) launches[k] = h->prof_cnt[k];
  }
  return EMB_OK;
}

const char *emb_profile_name(int32_t k) { return (k >= 0 && k < KID_COUNT) ? kKernelNames[k] : "?"; }

emb_status_t emb_clear_error(emb_handle_t h) {
  if (!h) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  CUDA_TRY(h, cudaDeviceSynchronize());
  CUDA_TRY(h, cudaMemset(h->err_dev, 0, sizeof(uint32_t)));
  *(volatile uint32_t *)h->err_host = 0;
  h->state = 0;
  h->last_error = "no error";
  return EMB_OK;
}

const char *emb_last_error(emb_handle_t h) {
  if (!h) {
    std::lock_guard<std::mutex> lk(g_err_mu);
    return g_create_error.c_str();
  }
  return h->last_error.c_str();
}

}  // extern "C"
