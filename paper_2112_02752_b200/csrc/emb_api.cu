// emb_api.cu — EmbContext runtime + the C ABI of include/emb.h.
//
// Owns: the fp32 row shard [rows_local][D] (+ Adagrad accumulator), all step workspace (sized once
// in emb_create from max_batch / max_ids / world), a side stream, the peer mappings for world > 1,
// and the step state machine.
//
// Step at world == 1 (no host sync):
//   lookup   : fork{ side: per-table dedup sort (key, occurrence) } ; main: pool straight from the
//              table -> join
//   backward : fused segment-reduce + optimizer apply over the sorted keys
// Step at world > 1 (no host sync; e = the step's epoch, exchanges over peer memory, p2p.cu):
//   lookup   : L0 sort -> k_route (keys into the owners' regions, counts + error bits, KEYS(e))
//              L1 wait KEYS(e) -> side: owner merge of the W received runs
//                                 main: gather the rows the others asked for, store them into their
//                                       row regions (ROWS(e))
//              L2 wait ROWS(e) -> pool -> join
//   backward : B0 requester merge of duplicate-id gradients, rows stored into the owners' regions
//                 (GRADS(e))
//              B1 wait GRADS(e) -> owner merge over sources (source-rank order) + apply
// Multi-process (one rank per process): a rank runs its phases back to back and the in-kernel flag
// waits order it against its peers. Group mode (emb_create_group: all ranks in this process, any
// devices, possibly one): emb_lookup_group / emb_backward_update_group run phase by phase over the
// ranks with cross-stream events between phases, so every flag a wait looks at was raised by a
// kernel that already completed -- no kernel ever waits on a kernel that may not be running.
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
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

const char *kKernelNames[KID_COUNT] = {"keys",      "sort_hist", "sort_pass", "pool",        "grad_apply",
                                       "unique",    "route",     "gather_push", "grad_push",   "signal",
                                       "init",      "owner_merge", "p2p_wait",  "lo_flags"};

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
  int64_t rows_local = 0;

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
    uint64_t epoch = 0;  // W > 1: the step whose first phase (sort + route) the prefetch ran
    bool requested = false;  // recorded by emb_lookup_prefetch, launched by the next backward
  } pf;
  bool pf_mismatch = false;   // W > 1: the lookup consumed a prefetched step with other arguments
  uint32_t late_err_bits = 0; // W > 1: error bits the step's gradient signal must still carry
  int32_t *blen = nullptr;
  SortWorkspace sws{};
  double *partials = nullptr;
  uint32_t *tickets = nullptr;
  int64_t nticket = 0;
  uint32_t *useg = nullptr, *ukey = nullptr, *ustart = nullptr, *uend = nullptr, *u_count = nullptr,
           *uniq_counter = nullptr, *fin = nullptr;
  uint64_t *uniq_status = nullptr, *ouniq_status = nullptr;
  uint32_t uniq_epoch = 0, ouniq_epoch = 0;
  // per-table sort (segsort.cu): table groups of the slot-major CSR
  bool segsort_ok = false;
  int32_t G = 0, segK = 1;
  uint32_t *run_k = nullptr, *run_i = nullptr;
  int32_t *d_gslot = nullptr;
  uint64_t *d_gbase = nullptr;
  uint32_t *d_grows = nullptr, *d_gbits = nullptr;
  uint32_t *err_dev = nullptr;
  uint32_t *err_host = nullptr;      // pinned, mapped
  uint32_t *err_host_dev = nullptr;  // device alias of err_host

  // ---- world > 1 (p2p.cu / route.cu)
  int64_t cap = 0;                   // entries per source region: max over ranks of max_ids
  uint32_t *inv = nullptr;           // [max_ids] occurrence -> o*cap + sendpos
  uint32_t *outidx = nullptr;        // [max_ids] sorted position -> sendpos
  int64_t *scnt = nullptr;           // [P2P_MAXW] my per-owner counts (device)
  // (the three above point into set epoch & 1 of these, like skey / spay into sk_set / sp_set: a
  // prefetched first phase of step e + 1 writes the set step e's backward does not read)
  uint32_t *inv_set[2] = {nullptr, nullptr}, *outidx_set[2] = {nullptr, nullptr};
  int64_t *scnt_set[2] = {nullptr, nullptr};
  uint32_t *route_tot = nullptr, *route_counter = nullptr, *route_done = nullptr;
  uint64_t *route_status = nullptr;
  uint32_t route_tag = 0;
  uint32_t *recv_keys = nullptr;     // [2][W*cap] (peer-written)
  float *uniq_rows = nullptr;        // [W*cap][D] rows pushed by their owners (peer-written)
  float *grecv = nullptr;            // [2][W*cap][D] hi rows, then lo rows (peer-written)
  uint8_t *lof = nullptr;            // [W*cap] "owner o needs the lo half of my key i" (peer-written)
  uint32_t *ok0 = nullptr, *ov0 = nullptr, *ok1 = nullptr, *ov1 = nullptr;  // owner merge
  int64_t *n_merged = nullptr;       // device: keys received this step
  int64_t *xmat = nullptr;           // [2][2][P2P_MAXW] (peer-written)
  uint64_t *flags = nullptr;         // [P2P_NKIND][P2P_MAXW] (peer-written)
  uint32_t *p2p_done = nullptr;
  P2PArgs p2p{};
  uint64_t epoch = 0;
  ncclComm_t comm = nullptr;
  std::vector<void *> ipc_opened;
  bool group = false;                // created by emb_create_group (all ranks in this process)
  bool counts_synced = true;
  bool owner_unique_done = false;
  uint32_t *ouseg = nullptr, *oukey = nullptr, *oustart = nullptr, *ouend = nullptr, *ou_count = nullptr,
           *ouniq_counter = nullptr;  // owner-side dedup of the merged keys (statistics, on demand)
  uint32_t step_err_bits = 0;        // host-detected argument errors of the pending collective step

  // ---- streams / step state
  cudaStream_t side = nullptr;
  cudaStream_t side_lo = nullptr;  // lowest priority: prefetched work (launch_prefetch)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_pf = nullptr, ev_phase = nullptr, ev_pfdone = nullptr,
              ev_pre = nullptr;  // ev_pre: on the caller stream right before the backward's gradient kernel
  int state = 0;  // 0 idle, 1 looked up
  int32_t batch = 0;
  int64_t nnz = 0;
  const int64_t *cur_ids = nullptr, *cur_offsets = nullptr;
  float *cur_out = nullptr;
  uint32_t *skey = nullptr, *spay = nullptr;   // requester-side sorted keys / payload of the last lookup
  int64_t U_l = 0, n_recv = 0;
  int64_t send_counts[EMB_MAX_WORLD] = {0}, recv_counts[EMB_MAX_WORLD] = {0};
  cudaStream_t last_stream = nullptr;
  int launches = 0;

  // ---- host-buffer (e2e) path, allocated on first use: two staging sets (step k uses set k & 1), H2D
  // copies on h2d_stream, D2H on d2h_stream (opposite PCIe directions overlap), events between them
  int64_t *st_ids[2] = {nullptr, nullptr}, *st_offsets[2] = {nullptr, nullptr};
  float *st_out[2] = {nullptr, nullptr}, *st_dout[2] = {nullptr, nullptr};
  int st_set = 0, host_set = 0;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr, host_stream = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_h2d2[2] = {}, ev_looked[2] = {}, ev_d2h[2] = {}, ev_free[2] = {};

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
    return fail(h, EMB_ERR_NCCL,
                "device: a peer never raised its exchange flag (sticky; a rank skipped a collective call: "
                "recreate the handles)");
  if (e & EMB_DEVERR_INTERNAL)
    return fail(h, EMB_ERR_CUDA, "device: an internal bounds guard tripped (library bug; work was skipped)");
  if (e & EMB_DEVERR_RANGE) return fail(h, EMB_ERR_RANGE, "device: an id was < 0 or >= rows[t] (sticky)");
  if (e & EMB_DEVERR_INVALID)
    return fail(h, EMB_ERR_INVALID, "device: CSR offsets not monotone or offsets[S*B] != nnz (sticky)");
  return EMB_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int64_t owner_of_global(const emb_ctx *h, uint64_t g) { return owner_of_g((uint32_t)g, h->ks); }
int64_t local_of_global(const emb_ctx *h, uint64_t g) { return local_of_g((uint32_t)g, h->ks); }

// optimizer-state floats per row: D (element-wise Adagrad) or 1 (row-wise)
int32_t accum_width(const emb_ctx *h) { return h->opt == EMB_OPT_ROWWISE_ADAGRAD ? 1 : h->D; }

// world > 1: the buffers peers write into / read from, in P2PArgs order
constexpr int NB_PEER = 6;
void peer_buffers(emb_ctx *h, void *out[NB_PEER]) {
  out[5] = h->lof;
  out[0] = h->xmat;
  out[1] = h->flags;
  out[2] = h->recv_keys;
  out[3] = h->grecv;
  out[4] = h->uniq_rows;
}
void set_peer(emb_ctx *h, int r, void *const ptr[NB_PEER]) {
  P2PArgs &p = h->p2p;
  p.peer_xmat[r] = static_cast<int64_t *>(ptr[0]);
  p.peer_flags[r] = static_cast<uint64_t *>(ptr[1]);
  p.peer_recv_keys[r] = static_cast<uint32_t *>(ptr[2]);
  p.peer_grecv[r] = static_cast<float *>(ptr[3]);
  p.peer_lof[r] = static_cast<uint8_t *>(ptr[5]);
  p.peer_uniq_rows[r] = static_cast<float *>(ptr[4]);
}
void init_p2p_args(emb_ctx *h) {
  P2PArgs &p = h->p2p;
  p.world = h->world;
  p.rank = h->rank;
  p.cap = h->cap;
  p.flags = h->flags;
  p.done = h->p2p_done;
  p.xmat = h->xmat;
}

// multi-process: before allocating, agree on the region size (max of max_ids) and check that every
// peer GPU is reachable with peer access from this one (same host, NVLink / PCIe P2P)
struct RankInfo {
  int64_t max_ids;
  uint64_t host;
  char busid[32];
};
emb_status_t mp_handshake(emb_ctx *h, int64_t *cap_out) {
  const int W = h->world;
  RankInfo mine{};
  mine.max_ids = h->max_ids;
  {
    char hn[256] = {0};
    gethostname(hn, sizeof(hn) - 1);
    uint64_t x = 1469598103934665603ull;  // FNV-1a of the host name
    for (const char *c = hn; *c; ++c) x = (x ^ (unsigned char)*c) * 1099511628211ull;
    mine.host = x;
  }
  CUDA_TRY(h, cudaDeviceGetPCIBusId(mine.busid, sizeof(mine.busid), h->device));
  char *dsend = nullptr, *drecv = nullptr;
  CUDA_TRY(h, cudaMalloc(&dsend, sizeof(RankInfo)));
  CUDA_TRY(h, cudaMalloc(&drecv, sizeof(RankInfo) * W));
  CUDA_TRY(h, cudaMemcpy(dsend, &mine, sizeof(RankInfo), cudaMemcpyHostToDevice));
  NCCL_TRY(h, ncclAllGather(dsend, drecv, sizeof(RankInfo), ncclUint8, h->comm, 0));
  CUDA_TRY(h, cudaDeviceSynchronize());
  std::vector<RankInfo> all(W);
  CUDA_TRY(h, cudaMemcpy(all.data(), drecv, sizeof(RankInfo) * W, cudaMemcpyDeviceToHost));
  cudaFree(dsend);
  cudaFree(drecv);
  int64_t cap = 0;
  for (int r = 0; r < W; ++r) {
    cap = std::max(cap, all[r].max_ids);
    if (all[r].host != mine.host)
      return fail(h, EMB_ERR_INVALID, "world > 1 needs every rank on one host (peer-memory exchange)");
    if (r == h->rank) continue;
    int dev = -1, ok = 0;
    if (cudaDeviceGetByPCIBusId(&dev, all[r].busid) != cudaSuccess || dev < 0 ||
        cudaDeviceCanAccessPeer(&ok, h->device, dev) != cudaSuccess || !ok)
      return fail(h, EMB_ERR_INVALID,
                  std::string("world > 1 needs peer access to every rank's GPU; no access to ") + all[r].busid);
  }
  *cap_out = cap;
  return EMB_OK;
}

// multi-process: map every peer's exchange buffers and table shard (CUDA IPC handles all-gathered
// over NCCL once)
emb_status_t setup_ipc(emb_ctx *h) {
  const int W = h->world;
  void *mine[NB_PEER];
  peer_buffers(h, mine);
  std::vector<cudaIpcMemHandle_t> hs(NB_PEER);
  for (int b = 0; b < NB_PEER; ++b) CUDA_TRY(h, cudaIpcGetMemHandle(&hs[b], mine[b]));
  const size_t bytes = sizeof(cudaIpcMemHandle_t) * NB_PEER;
  char *dsend = nullptr, *drecv = nullptr;
  CUDA_TRY(h, cudaMalloc(&dsend, bytes));
  CUDA_TRY(h, cudaMalloc(&drecv, bytes * W));
  CUDA_TRY(h, cudaMemcpy(dsend, hs.data(), bytes, cudaMemcpyHostToDevice));
  NCCL_TRY(h, ncclAllGather(dsend, drecv, bytes, ncclUint8, h->comm, 0));
  CUDA_TRY(h, cudaDeviceSynchronize());
  std::vector<cudaIpcMemHandle_t> all((size_t)NB_PEER * W);
  CUDA_TRY(h, cudaMemcpy(all.data(), drecv, bytes * W, cudaMemcpyDeviceToHost));
  cudaFree(dsend);
  cudaFree(drecv);
  init_p2p_args(h);
  for (int r = 0; r < W; ++r) {
    void *ptr[NB_PEER];
    for (int b = 0; b < NB_PEER; ++b) {
      if (r == h->rank) {
        ptr[b] = mine[b];
      } else {
        void *q = nullptr;
        CUDA_TRY(h, cudaIpcOpenMemHandle(&q, all[(size_t)r * NB_PEER + b], cudaIpcMemLazyEnablePeerAccess));
        h->ipc_opened.push_back(q);
        ptr[b] = q;
      }
    }
    set_peer(h, r, ptr);
  }
  return EMB_OK;
}

// group mode: every rank is a handle of this process; peers' buffers are plain pointers (peer access
// enabled between distinct devices)
emb_status_t setup_group(std::vector<emb_ctx *> &hs) {
  const int W = (int)hs.size();
  for (int r = 0; r < W; ++r) {
    emb_ctx *h = hs[r];
    CUDA_TRY(h, cudaSetDevice(h->device));
    for (int p = 0; p < W; ++p) {
      if (hs[p]->device == h->device) continue;
      int ok = 0;
      CUDA_TRY(h, cudaDeviceCanAccessPeer(&ok, h->device, hs[p]->device));
      if (!ok) return fail(h, EMB_ERR_INVALID, "emb_create_group: no peer access between the ranks' devices");
      cudaError_t e = cudaDeviceEnablePeerAccess(hs[p]->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
    }
    init_p2p_args(h);
    for (int p = 0; p < W; ++p) {
      void *ptr[NB_PEER];
      peer_buffers(hs[p], ptr);
      set_peer(h, p, ptr);
    }
  }
  return EMB_OK;
}

// bring the last step's counts to the host (statistics only)
emb_status_t sync_counts(emb_ctx *h) {
  if (h->counts_synced) return EMB_OK;
  if (h->last_stream) CUDA_TRY(h, cudaStreamSynchronize(h->last_stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->side));
  const int W = h->world;
  int64_t sc[P2P_MAXW], xm[4 * P2P_MAXW], nm = 0;
  CUDA_TRY(h, cudaMemcpy(sc, h->scnt, sizeof(int64_t) * P2P_MAXW, cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaMemcpy(xm, h->xmat, sizeof(int64_t) * 4 * P2P_MAXW, cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaMemcpy(&nm, h->n_merged, sizeof(int64_t), cudaMemcpyDeviceToHost));
  int64_t ul = 0;
  for (int p = 0; p < W; ++p) {
    h->send_counts[p] = sc[p];
    h->recv_counts[p] = xm[xmat_idx(h->epoch, 0, p)];
    ul += sc[p];
  }
  h->U_l = ul;
  h->n_recv = nm;
  h->counts_synced = true;
  return EMB_OK;
}

// group_cap > 0: group mode (every rank in this process; the caller computed the region size)
emb_status_t create_impl(const emb_config_t *cfg, emb_ctx *h, int64_t group_cap) {
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
  if (cfg->world > 1 && !group_cap && !cfg->nccl_id)
    return fail(h, EMB_ERR_INVALID, "world > 1 needs nccl_id (or emb_create_group)");
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
  h->group = group_cap > 0;

  // key space: sorted keys are the fused rows g at every W
  KeySpace &ks = h->ks;
  ks.world = h->world;
  ks.rank = h->rank;
  ks.shard = h->shard;
  ks.rows_per = (uint32_t)((h->R_total + h->world - 1) / h->world);
  ks.key_bits = std::max<uint32_t>(1, bits_for(h->R_total));  // max valid key R-1 < sentinel-mask 2^b - 1
  if (h->world == 1) {
    h->rows_local = (int64_t)h->R_total;
  } else if (h->shard == 0) {
    h->rows_local = (int64_t)((h->R_total - h->rank + h->world - 1) / h->world);
  } else {
    const int64_t lo = std::min<int64_t>((int64_t)h->R_total, (int64_t)ks.rows_per * h->rank);
    const int64_t hi = std::min<int64_t>((int64_t)h->R_total, (int64_t)ks.rows_per * (h->rank + 1));
    h->rows_local = hi - lo;
  }

  CUDA_TRY(h, cudaSetDevice(h->device));
  const int W = h->world;
  if (W > 1 && !h->group) {
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    NCCL_TRY(h, ncclCommInitRank(&h->comm, W, id, h->rank));
    emb_status_t hs = mp_handshake(h, &h->cap);
    if (hs != EMB_OK) return hs;
  } else if (W > 1) {
    h->cap = group_cap;
  }
  if (W > 1 && ((int64_t)W * h->cap >= (1ll << 31) - 1 || h->cap > (int64_t)OUT_POS_MASK))
    return fail(h, EMB_ERR_INVALID, "world > 1 needs world * max_ids < 2^31 - 1 and max_ids < 2^28");

  // table shard + state
  const size_t row_elems = (size_t)std::max<int64_t>(h->rows_local, 1) * h->D;
  if (dalloc(h, &h->w, row_elems) != cudaSuccess) return fail(h, EMB_ERR_NOMEM, "cannot allocate the table shard");
  if (h->opt == EMB_OPT_ADAGRAD && dalloc(h, &h->a, row_elems) != cudaSuccess)
    return fail(h, EMB_ERR_NOMEM, "cannot allocate the Adagrad state");
  if (h->opt == EMB_OPT_ROWWISE_ADAGRAD && dalloc(h, &h->a, (size_t)std::max<int64_t>(h->rows_local, 1)) != cudaSuccess)
    return fail(h, EMB_ERR_NOMEM, "cannot allocate the row-wise Adagrad state");
  {
    // the side stream carries the latency-critical sort (W = 1) / owner merge (W > 1): highest
    // priority, so its CTAs are scheduled ahead of the bandwidth-bound pool CTAs as SMs free up
    int lo_prio = 0, hi_prio = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi_prio));
  }
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_pf, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_phase, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_pfdone, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_pre, cudaEventDisableTiming));
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
  const int64_t WC = W > 1 ? (int64_t)W * h->cap : 0;
  h->nticket = std::max<int64_t>(N, WC) + 1;
  const int64_t nwarps_max = grad_max_warps(h->device);
  bool bad = false;
  bad |= dalloc(h, &h->key_csr, N) != cudaSuccess;
  bad |= dalloc(h, &h->drow, N) != cudaSuccess;
  bad |= dalloc(h, &h->k0, N) != cudaSuccess;
  bad |= dalloc(h, &h->v0, N) != cudaSuccess;
  bad |= dalloc(h, &h->sort_scratch, N) != cudaSuccess;
  bad |= dalloc(h, &h->sk_set[1], N) != cudaSuccess;
  bad |= dalloc(h, &h->sp_set[1], N) != cudaSuccess;
  bad |= dalloc(h, &h->k1, N) != cudaSuccess;
  bad |= dalloc(h, &h->v1, N) != cudaSuccess;
  bad |= dalloc(h, &h->blen, SB) != cudaSuccess;
  uint32_t *sort_words = nullptr;
  bad |= dalloc(h, &sort_words, sort_workspace_words(N)) != cudaSuccess;
  bad |= dalloc(h, &h->partials, (size_t)2 * nwarps_max * h->D) != cudaSuccess;
  bad |= dalloc(h, &h->tickets, h->nticket) != cudaSuccess;
  bad |= dalloc(h, &h->useg, N) != cudaSuccess;
  bad |= dalloc(h, &h->ukey, N) != cudaSuccess;
  bad |= dalloc(h, &h->ustart, N + 1) != cudaSuccess;
  bad |= dalloc(h, &h->uend, N + 1) != cudaSuccess;
  bad |= dalloc(h, &h->u_count, 2) != cudaSuccess;
  bad |= dalloc(h, &h->uniq_status, unique_status_words(N)) != cudaSuccess;
  bad |= dalloc(h, &h->uniq_counter, 1) != cudaSuccess;
  bad |= dalloc(h, &h->fin, 3) != cudaSuccess;
  bad |= dalloc(h, &h->err_dev, 1) != cudaSuccess;
  if (W > 1) {
    for (int k = 0; k < 2; ++k) {
      bad |= dalloc(h, &h->inv_set[k], N) != cudaSuccess;
      bad |= dalloc(h, &h->outidx_set[k], N) != cudaSuccess;
      bad |= dalloc(h, &h->scnt_set[k], P2P_MAXW) != cudaSuccess;
    }
    h->inv = h->inv_set[0];
    h->outidx = h->outidx_set[0];
    h->scnt = h->scnt_set[0];
    bad |= dalloc(h, &h->route_tot, P2P_MAXW) != cudaSuccess;
    bad |= dalloc(h, &h->route_counter, 1) != cudaSuccess;
    bad |= dalloc(h, &h->route_done, 1) != cudaSuccess;
    // look-back words: one set per route tile, or per sort CTA when the route is fused into the
    // per-table sort (groups x ranges <= EMB_MAX_SLOTS x 32)
    bad |= dalloc(h, &h->route_status, std::max<size_t>(route_status_words(N), (size_t)(EMB_MAX_SLOTS * 32 + 1) * P2P_MAXW)) !=
           cudaSuccess;
    bad |= dalloc(h, &h->recv_keys, 2 * WC) != cudaSuccess;
    bad |= dalloc(h, &h->uniq_rows, (size_t)WC * h->D) != cudaSuccess;
    bad |= dalloc(h, &h->grecv, (size_t)2 * WC * h->D) != cudaSuccess;  // hi and lo parts
    bad |= dalloc(h, &h->lof, WC) != cudaSuccess;
    bad |= dalloc(h, &h->ok0, WC) != cudaSuccess;
    bad |= dalloc(h, &h->ov0, WC) != cudaSuccess;
    bad |= dalloc(h, &h->ok1, WC) != cudaSuccess;
    bad |= dalloc(h, &h->ov1, WC) != cudaSuccess;
    bad |= dalloc(h, &h->n_merged, 1) != cudaSuccess;
    bad |= dalloc(h, &h->xmat, 4 * P2P_MAXW) != cudaSuccess;
    bad |= dalloc(h, &h->flags, (size_t)P2P_NKIND * P2P_MAXW) != cudaSuccess;
    bad |= dalloc(h, &h->p2p_done, P2P_NKIND) != cudaSuccess;
    bad |= dalloc(h, &h->ouseg, WC) != cudaSuccess;
    bad |= dalloc(h, &h->oukey, WC) != cudaSuccess;
    bad |= dalloc(h, &h->oustart, WC + 1) != cudaSuccess;
    bad |= dalloc(h, &h->ouend, WC + 1) != cudaSuccess;
    bad |= dalloc(h, &h->ou_count, 2) != cudaSuccess;
    bad |= dalloc(h, &h->ouniq_status, unique_status_words(WC)) != cudaSuccess;
    bad |= dalloc(h, &h->ouniq_counter, 1) != cudaSuccess;
  }
  if (bad) return fail(h, EMB_ERR_NOMEM, "cannot allocate the step workspace");
  h->sk_set[0] = h->k0;
  h->sp_set[0] = h->v0;
  h->sws.hist = sort_words;
  h->sws.counters = sort_words + 4 * 256;
  h->sws.status = sort_words + 4 * 256 + 4;
  h->sws.max_tiles = (N + 4095) / 4096 + 1;
  h->sws.err = h->err_dev;
  CUDA_TRY(h, cudaMemset(h->tickets, 0, sizeof(uint32_t) * h->nticket));
  // table groups of the slot-major CSR (the per-table sort needs a non-decreasing slot_table)
  {
    h->segsort_ok = true;
    for (int s = 1; s < h->S; ++s)
      if (h->slot_table[s] < h->slot_table[s - 1]) h->segsort_ok = false;
    int32_t ngroups = 0;
    for (int s = 0; s < h->S; ++s) ngroups += (s == 0 || h->slot_table[s] != h->slot_table[s - 1]);
    // the per-table sort keeps a group's key ranges in shared memory: K <= 16 CTAs per group, each
    // scanning the whole group. Groups much larger than that (C4: 1.7M ids on one table; C5: 1M ids
    // per table) take the general path instead -- key kernel + onesweep LSD radix sort over all keys
    // (round 1 measured 7.6 ms of per-table sort at C5 against a few hundred us for the radix passes)
    if (h->segsort_ok && (h->max_ids + ngroups - 1) / ngroups > (int64_t)SEG_BIG) h->segsort_ok = false;
    if (const char *ef = getenv("EMB_FORCE_GENERAL")) if (atoi(ef)) h->segsort_ok = false;  // experiment knob
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
      // K=2/4/8/16 -> 206/157/176/201 us per step); every CTA scans its whole group, so K stays small.
      // With few groups (C1: one table) the CTAs would not fill the GPU: ~1K occurrences per CTA then
      const int64_t per = (h->max_ids + h->G - 1) / h->G;
      const int64_t per_cta = h->G >= 8 ? 4096 : 1024;
      h->segK = (int32_t)std::min<int64_t>(16, std::max<int64_t>(1, (per + per_cta - 1) / per_cta));
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
  CUDA_TRY(h, cudaMemset(h->uniq_status, 0, sizeof(uint64_t) * unique_status_words(N)));
  CUDA_TRY(h, cudaMemset(h->u_count, 0, 2 * sizeof(uint32_t)));
  if (W > 1) {
    CUDA_TRY(h, cudaMemset(h->ouniq_counter, 0, sizeof(uint32_t)));
    CUDA_TRY(h, cudaMemset(h->ouniq_status, 0, sizeof(uint64_t) * unique_status_words(WC)));
    CUDA_TRY(h, cudaMemset(h->route_tot, 0, sizeof(uint32_t) * P2P_MAXW));
    CUDA_TRY(h, cudaMemset(h->route_counter, 0, sizeof(uint32_t)));
    CUDA_TRY(h, cudaMemset(h->route_done, 0, sizeof(uint32_t)));
    CUDA_TRY(h, cudaMemset(h->route_status, 0,
                           sizeof(uint64_t) * std::max<size_t>(route_status_words(N), (size_t)(EMB_MAX_SLOTS * 32 + 1) * P2P_MAXW)));
    for (int k = 0; k < 2; ++k) CUDA_TRY(h, cudaMemset(h->scnt_set[k], 0, sizeof(int64_t) * P2P_MAXW));
    CUDA_TRY(h, cudaMemset(h->n_merged, 0, sizeof(int64_t)));
    CUDA_TRY(h, cudaMemset(h->xmat, 0, sizeof(int64_t) * 4 * P2P_MAXW));
    CUDA_TRY(h, cudaMemset(h->flags, 0, sizeof(uint64_t) * P2P_NKIND * P2P_MAXW));
    CUDA_TRY(h, cudaMemset(h->p2p_done, 0, sizeof(uint32_t) * P2P_NKIND));
  }
  void *hp = nullptr;
  if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) != cudaSuccess)
    return fail(h, EMB_ERR_NOMEM, "cannot allocate pinned error word");
  h->err_host = static_cast<uint32_t *>(hp);
  *h->err_host = 0;
  CUDA_TRY(h, cudaHostGetDevicePointer(reinterpret_cast<void **>(&h->err_host_dev), hp, 0));
  CUDA_TRY(h, cudaStreamSynchronize(h->side));
  CUDA_TRY(h, cudaDeviceSynchronize());
  if (W > 1 && !h->group) {
    emb_status_t ps = setup_ipc(h);
    if (ps != EMB_OK) return ps;
  }
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
  for (cudaEvent_t e : h->prof_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : {h->ev_fork, h->ev_join, h->ev_pf, h->ev_phase, h->ev_pfdone, h->ev_pre})
    if (e) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k)
    for (cudaEvent_t e : {h->ev_h2d[k], h->ev_h2d2[k], h->ev_looked[k], h->ev_d2h[k], h->ev_free[k]})
      if (e) cudaEventDestroy(e);
  for (cudaStream_t q : {h->side, h->side_lo, h->h2d_stream, h->d2h_stream})
    if (q) cudaStreamDestroy(q);
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

// per-table sort arguments writing sort-output set `set`
SegSortArgs segsort_args(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz, int set) {
  SegSortArgs sa{};
  sa.ids = ids;
  sa.offsets = offsets;
  sa.nnz = nnz;
  sa.batch = batch;
  sa.gslot = h->d_gslot;
  sa.ngroups = h->G;
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

emb_status_t launch_l0(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                       uint64_t e, uint32_t extra_err, cudaStream_t st);

emb_status_t launch_l0(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                       uint64_t e, uint32_t extra_err, cudaStream_t st);

// emb_lookup_prefetch only RECORDS the request (the inputs are ready at ev_pf on the caller stream);
// the next backward launches it (launch_prefetch) right after its own gradient kernel, on the
// lowest-priority stream, so the persistent gradient pass's CTAs are resident first and the prefetched
// work takes SMs as they free up. (Launched at the prefetch call, the per-table sort's CTAs -- one per
// SM, 192 KB of shared memory each -- were resident first and the static-range gradient pass waited
// for them: the W = 2 requester pass stretched 75 -> 122 us, and C2 swung between 129 and 146 us/step
// with the race.) What it launches:
//  - W = 1: the per-table sort into the sort-output set the pending backward does not read;
//  - W > 1: the first phase of the NEXT step (sort + route into buffer set (epoch + 1) & 1, raises
//    KEYS); the next lookup consumes it (lookup_phase0). Once launched it cannot be withdrawn (its
//    keys are on their way to the owners): a lookup with other arguments then takes part with an
//    empty batch and fails the step everywhere.
// A request with no backward before the next lookup is dropped (nothing was launched).
emb_status_t lookup_prefetch_impl(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch,
                                  int64_t nnz, cudaStream_t st) {
  if (batch < 0 || batch > h->max_batch || nnz < 0 || nnz > h->max_ids || (batch == 0 && nnz != 0))
    return fail(h, EMB_ERR_INVALID, "prefetch: batch / nnz out of range");
  if ((batch > 0 && !offsets) || (nnz > 0 && !ids)) return fail(h, EMB_ERR_INVALID, "prefetch: NULL ids/offsets");
  if (h->world > 1 && (h->pf.valid || h->pf.requested))
    return fail(h, EMB_ERR_STATE, "prefetch: a prefetched step is already pending (world > 1: the next emb_lookup "
                                  "consumes it)");
  h->pf.valid = false;  // (W = 1: a new request replaces an older one)
  h->pf.requested = false;
  if (!h->segsort_ok || batch == 0 || nnz == 0) return EMB_OK;  // the lookup runs its own first phase
  CUDA_TRY(h, cudaSetDevice(h->device));
  CUDA_TRY(h, cudaEventRecord(h->ev_pf, st));
  h->pf.requested = true;
  h->pf.ids = ids;
  h->pf.offsets = offsets;
  h->pf.batch = batch;
  h->pf.nnz = nnz;
  return EMB_OK;
}

// called by the backward right after its gradient kernel: launch a recorded prefetch request
emb_status_t launch_prefetch(emb_ctx *h) {
  if (!h->pf.requested) return EMB_OK;
  h->pf.requested = false;
  if (!h->side_lo) {
    int lo_prio = 0, hi_prio = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->side_lo, cudaStreamNonBlocking, lo_prio));
  }
  CUDA_TRY(h, cudaStreamWaitEvent(h->side_lo, h->ev_pf, 0));
  // ... and not before the gradient kernel is ready (at W > 1 it sits behind a flag wait): ready
  // together, the gradient kernel (enqueued first, no lower priority) is resident first
  CUDA_TRY(h, cudaStreamWaitEvent(h->side_lo, h->ev_pre, 0));
  if (h->world > 1) {
    const uint64_t e = h->epoch + 1;
    emb_status_t s = launch_l0(h, h->pf.ids, h->pf.offsets, h->pf.batch, h->pf.nnz, e, 0u, h->side_lo);
    if (s != EMB_OK) return s;
    h->pf.set = (int)(e & 1u);
    h->pf.epoch = e;
  } else {
    const int set = h->cur_set ^ 1;
    SegSortArgs sa = segsort_args(h, h->pf.ids, h->pf.offsets, h->pf.batch, h->pf.nnz, set);
    LAUNCH(h, KID_SORT_PASS, h->side_lo, launch_segsort(sa, h->G, h->side_lo));
    h->pf.set = set;
  }
  CUDA_TRY(h, cudaEventRecord(h->ev_pfdone, h->side_lo));
  h->pf.valid = true;
  return EMB_OK;
}

// argument checks shared by every lookup entry point ("" = fine)
const char *lookup_arg_error(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                             const float *out) {
  if (batch < 0 || batch > h->max_batch) return "batch out of [0, max_batch]";
  if (nnz < 0 || nnz > h->max_ids) return "nnz out of [0, max_ids]";
  if (batch == 0 && nnz != 0) return "nnz must be 0 when batch == 0";
  if ((batch > 0 && (!offsets || !out)) || (nnz > 0 && !ids)) return "NULL ids/offsets/out";
  if (batch > 0 && !aligned16(out)) return "out must be 16-byte aligned";
  return "";
}

KeysArgs keys_args(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz) {
  KeysArgs ka{};
  ka.ids = ids;
  ka.offsets = offsets;
  ka.nnz = nnz;
  ka.batch = batch;
  ka.num_slots = h->S;
  ka.slot_table = h->d_slot_table;
  ka.base = h->d_base;
  ka.rows = h->d_rows;
  ka.key = h->key_csr;
  ka.drow = h->drow;
  ka.blen = h->blen;
  ka.err = h->err_dev;
  return ka;
}

PoolArgs pool_args(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz, float *out) {
  const bool mean = h->pool == EMB_POOL_MEAN;
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
  pa.ks = h->ks;
  pa.rows_src = h->w;
  pa.nrows_src = h->rows_local;
  pa.rows_remote = h->uniq_rows;
  pa.nrows_remote = h->world > 1 ? (int64_t)h->world * h->cap : 0;
  pa.row_idx = h->inv;
  if (h->segsort_ok) {  // direct mode: the pool reads the ids itself (no key kernel)
    pa.ids = ids;
    pa.slot_table = h->d_slot_table;
    pa.base = h->d_base;
    pa.rows = h->d_rows;
    pa.drow = h->drow;
    pa.blen = mean ? h->blen : nullptr;
  }
  return pa;
}

emb_status_t lookup_w1(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz, float *out,
                       cudaStream_t st) {
  // key mode (general sort path): the key kernel feeds both the sort and the pool
  if (batch > 0 && !h->segsort_ok) LAUNCH(h, KID_KEYS, st, launch_keys(keys_args(h, ids, offsets, batch, nnz), st));
  // fork: the sort runs on the side stream while the pool streams rows on the caller stream
  CUDA_TRY(h, cudaEventRecord(h->ev_fork, st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  // a sort prefetched for exactly these inputs (emb_lookup_prefetch) is already queued on the side
  // stream: consume it (the join below waits for it)
  const bool use_pf = h->pf.valid && h->pf.ids == ids && h->pf.offsets == offsets && h->pf.batch == batch &&
                      h->pf.nnz == nnz;
  h->pf.valid = false;
  h->pf.requested = false;  // (a request no backward launched is dropped)
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
  PoolArgs pa = pool_args(h, ids, offsets, batch, nnz, out);
  const bool fused_pub = h->segsort_ok && batch > 0 && nnz > 0;
  pa.fin = fused_pub ? h->fin : nullptr;
  pa.fin_kernels = use_pf ? 1 : 2;  // a prefetched sort does not take part in the publish
  if (batch > 0) LAUNCH(h, KID_POOL, st, launch_pool(pa, st));
  CUDA_TRY(h, cudaEventRecord(h->ev_join, h->side));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_join, 0));
  if (use_pf) CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_pfdone, 0));  // the prefetched sort (side_lo)
  if (batch > 0 && !fused_pub) LAUNCH(h, KID_KEYS, st, launch_publish_err(h->err_dev, h->err_host_dev, st));
  return EMB_OK;
}

// ---- world > 1 phases (see the file header). The step's arguments are in h (cur_*, batch, nnz).
constexpr const char *PF_MISMATCH_MSG =
    "emb_lookup arguments differ from the pending emb_lookup_prefetch (the rank took part with an empty batch; the "
    "step updates nothing on any rank)";

// make step e current: its epoch and its buffer set (e & 1)
void begin_step(emb_ctx *h, uint64_t e) {
  const int set = (int)(e & 1u);
  h->epoch = e;
  h->p2p.epoch = e;
  h->skey = h->sk_set[set];
  h->spay = h->sp_set[set];
  h->inv = h->inv_set[set];
  h->outidx = h->outidx_set[set];
  h->scnt = h->scnt_set[set];
}

// L0 of the step with epoch e: dedup sort + route into buffer set e & 1 (raises KEYS(e)). Only the
// per-table sort path writes the set buffers; the general radix path (never prefetched) leaves its
// sorted keys in h->skey / h->spay.
emb_status_t launch_l0(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                       uint64_t e, uint32_t extra_err, cudaStream_t st) {
  const int set = (int)(e & 1u);
  RouteArgs ra{};
  ra.skey = h->sk_set[set];
  ra.spay = h->sp_set[set];
  ra.n = (batch > 0) ? nnz : 0;
  ra.ks = h->ks;
  ra.p2p = h->p2p;
  ra.p2p.epoch = e;
  ra.outidx = h->outidx_set[set];
  ra.inv = h->inv_set[set];
  ra.scnt = h->scnt_set[set];
  ra.tot = h->route_tot;
  ra.status = h->route_status;
  ra.counter = h->route_counter;
  ra.blk_done = h->route_done;
  if (++h->route_tag == 0) h->route_tag = 1;
  ra.tag = h->route_tag;
  ra.err = h->err_dev;
  ra.extra_err = extra_err;
  static int fuse = -1;  // experiment knob EMB_FUSED_ROUTE=0: separate k_route after the per-table sort
  if (fuse < 0) fuse = getenv("EMB_FUSED_ROUTE") ? atoi(getenv("EMB_FUSED_ROUTE")) : 1;
  if (batch > 0 && nnz > 0) {
    if (h->segsort_ok) {
      SegSortArgs sa = segsort_args(h, ids, offsets, batch, nnz, set);
      sa.validate = 1;
      if (fuse) {  // the route runs in the sort's epilogue (no separate launch)
        sa.route = 1;
        sa.rt = ra;
        LAUNCH(h, KID_SORT_PASS, st, launch_segsort(sa, h->G, st));
        return EMB_OK;
      }
      LAUNCH(h, KID_SORT_PASS, st, launch_segsort(sa, h->G, st));
    } else {
      LAUNCH(h, KID_KEYS, st, launch_keys(keys_args(h, ids, offsets, batch, nnz), st));
      int nl = 0;
      cudaError_t r = radix_sort_pairs(h->sws, h->key_csr, nullptr, h->k0, h->v0, h->k1, h->v1, nnz, h->ks.key_bits,
                                       st, &h->skey, &h->spay, &nl, prof_hook, h);
      if (r != cudaSuccess) return fail(h, EMB_ERR_CUDA, std::string("radix sort: ") + cudaGetErrorString(r));
      h->launches += nl;
      ra.skey = h->skey;
      ra.spay = h->spay;
    }
  } else if (batch > 0 && !h->segsort_ok) {
    LAUNCH(h, KID_KEYS, st, launch_keys(keys_args(h, ids, offsets, batch, nnz), st));  // validates the CSR
  }
  LAUNCH(h, KID_ROUTE, st, launch_route(ra, st));
  return EMB_OK;
}

// L0: dedup sort + route (raises KEYS), or consume the first phase a prefetch already ran
emb_status_t lookup_phase0(emb_ctx *h, cudaStream_t st) {
  h->pf_mismatch = false;
  h->pf.requested = false;  // (a request no backward launched is dropped: nothing was sent)
  if (h->pf.valid) {
    h->pf.valid = false;
    const bool match = h->step_err_bits == 0 && h->pf.ids == h->cur_ids && h->pf.offsets == h->cur_offsets &&
                       h->pf.batch == h->batch && h->pf.nnz == h->nnz;
    begin_step(h, h->pf.epoch);
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_pfdone, 0));
    if (!match) {  // the owners already hold the prefetched keys: take part empty, fail the step everywhere
      h->pf_mismatch = true;
      h->late_err_bits = EMB_DEVERR_INVALID;
      h->batch = 0;
      h->nnz = 0;
      h->cur_out = nullptr;
      LAUNCH(h, KID_SIGNAL, st, launch_mark_err(h->err_dev, EMB_DEVERR_INVALID, st));  // sticky, as a lookup argument error
    }
    return EMB_OK;
  }
  begin_step(h, h->epoch + 1);
  return launch_l0(h, h->cur_ids, h->cur_offsets, h->batch, h->nnz, h->epoch, h->step_err_bits, st);
}

// L1: wait KEYS -> owner merge (side stream) | gather + push the requested rows (raises ROWS)
emb_status_t lookup_phase1(emb_ctx *h, cudaStream_t st) {
  const P2PArgs &px = h->p2p;
  const int W = h->world;
  const uint32_t *rk = h->recv_keys + (size_t)(h->epoch & 1u) * W * h->cap;
  const int64_t *cnt = h->xmat + xmat_idx(h->epoch, 0, 0);
  LAUNCH(h, KID_WAIT, st, launch_wait(px, P2P_KEYS, h->epoch, h->err_dev, st));
  CUDA_TRY(h, cudaEventRecord(h->ev_fork, st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  LAUNCH(h, KID_MERGE, h->side,
         launch_merge_tree(rk, cnt, W, h->cap, h->ok0, h->ov0, h->ok1, h->ov1, h->n_merged, h->side));
  // (no fused error publish here: the per-block barrier + atomic it adds to the 1,664 short pool blocks
  // cost more than the separate publish kernel, W = 2 297.6 -> 304-307 us/step)
  LAUNCH(h, KID_LOFLAGS, h->side,
         launch_lo_flags(px, h->ok0, h->ov0, h->n_merged, (int64_t)W * h->cap, nullptr, h->err_dev, h->err_host_dev,
                         h->side));
  LAUNCH(h, KID_GATHER_PUSH, st, launch_gather_push(px, h->w, rk, cnt, h->D, h->rows_local, h->err_dev, st));
  return EMB_OK;
}

// L2: wait ROWS -> pool; join the merge
emb_status_t lookup_phase2(emb_ctx *h, cudaStream_t st) {
  LAUNCH(h, KID_WAIT, st, launch_wait(h->p2p, P2P_ROWS, h->epoch, h->err_dev, st));
  if (h->batch > 0 && h->cur_out) {
    PoolArgs pa = pool_args(h, h->cur_ids, h->cur_offsets, h->batch, h->nnz, h->cur_out);
    LAUNCH(h, KID_POOL, st, launch_pool(pa, st));
  }
  CUDA_TRY(h, cudaEventRecord(h->ev_join, h->side));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_join, 0));
  LAUNCH(h, KID_KEYS, st, launch_publish_err(h->err_dev, h->err_host_dev, st));
  h->counts_synced = false;
  h->owner_unique_done = false;
  h->U_l = -1;
  h->n_recv = -1;
  return EMB_OK;
}

GradArgs grad_args(emb_ctx *h, const float *d_out, double lr) {
  GradArgs g{};
  g.signal_kind = -1;
  g.dim = h->D;
  g.dy = d_out;
  g.drow = h->drow;
  g.blen = h->pool == EMB_POOL_MEAN ? h->blen : nullptr;
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
  g.err = h->err_dev;
  g.lmask = 0xFFFFFFFFu;
  g.ks = h->ks;
  g.p2p = h->p2p;
  return g;
}

// B0: requester merge, rows stored into the owners' regions (raises GRADS). d_out == nullptr (an
// argument error at W > 1): no contribution, the step is marked failed at every owner.
emb_status_t backward_phase0(emb_ctx *h, const float *d_out, double lr, cudaStream_t st) {
  GradArgs g = grad_args(h, d_out, lr);
  g.skey = h->skey;
  g.spay = h->spay;
  g.n = h->nnz;
  g.src_mode = 0;
  g.sink_mode = 2;
  g.useg = h->outidx;
  g.nout = h->cap;
  g.lof = h->lof;
  g.lo_stride = (int64_t)h->world * h->cap * h->D;
  g.signal_kind = P2P_GRADS;
  // the owners' "needs lo" bytes (written after their merges, long done by now)
  LAUNCH(h, KID_WAIT, st, launch_wait(h->p2p, P2P_LOF, h->epoch, h->err_dev, st));
  if (h->pf.requested) CUDA_TRY(h, cudaEventRecord(h->ev_pre, st));
  if (h->batch > 0 && h->nnz > 0 && d_out)
    LAUNCH(h, KID_GRAD_PUSH, st, launch_grad(g, st));
  else
    LAUNCH(h, KID_SIGNAL, st, launch_signal(h->p2p, P2P_GRADS, (d_out || h->batch == 0 ? 0u : EMB_DEVERR_INVALID) |
                                                                  h->late_err_bits, st));
  h->late_err_bits = 0;
  return launch_prefetch(h);
}

// B1: wait GRADS, owner merge over sources + apply
emb_status_t backward_phase1(emb_ctx *h, double lr, cudaStream_t st) {
  const int W = h->world;
  GradArgs o = grad_args(h, nullptr, lr);
  o.skey = h->ok0;
  o.spay = h->ov0;
  o.n = (int64_t)W * h->cap;
  o.n_dev = h->n_merged;
  o.src_mode = 1;
  o.src = h->grecv;
  o.src_lo = h->grecv + (size_t)W * h->cap * h->D;  // lo rows (read only for keys with several sources)
  o.lo_stride = (int64_t)W * h->cap * h->D;
  o.nsrc = (int64_t)W * h->cap;
  o.blen = nullptr;
  o.sink_mode = 0;
  o.signal_kind = -1;
  o.skip_mask = EMB_DEVERR_TIMEOUT | EMB_DEVERR_INTERNAL;
  o.abort_bits = h->xmat + xmat_idx(h->epoch, 1, 0);
  LAUNCH(h, KID_WAIT, st, launch_wait(h->p2p, P2P_GRADS, h->epoch, h->err_dev, st));
  LAUNCH(h, KID_GRAD_APPLY, st, launch_grad(o, st));
  return EMB_OK;
}

// one rank's lookup; at W > 1 a multi-process rank runs both phases back to back
emb_status_t lookup_impl(emb_ctx *h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                         float *out, cudaStream_t st) {
  if (h->state != 0) return fail(h, EMB_ERR_STATE, "emb_lookup called twice without emb_backward_update");
  if (h->group) return fail(h, EMB_ERR_STATE, "a group handle steps through emb_lookup_group");
  const char *ae = lookup_arg_error(h, ids, offsets, batch, nnz, out);
  CUDA_TRY(h, cudaSetDevice(h->device));
  h->launches = 0;
  h->last_stream = st;
  if (h->world == 1) {
    if (*ae) return fail(h, EMB_ERR_INVALID, ae);
    emb_status_t s = check_sticky(h);
    if (s != EMB_OK) return s;
    h->batch = batch;
    h->nnz = nnz;
    emb_status_t r = lookup_w1(h, ids, offsets, batch, nnz, out, st);
    if (r != EMB_OK) return r;
    h->U_l = -1;
    h->state = 1;
    return EMB_OK;
  }
  // W > 1: the call is collective -- a rank with bad arguments still takes part (empty batch) and
  // marks the step failed at every owner, so no peer waits for it and no rank applies the step
  h->step_err_bits = *ae ? EMB_DEVERR_INVALID : 0u;
  h->batch = *ae ? 0 : batch;
  h->nnz = *ae ? 0 : nnz;
  h->cur_ids = ids;
  h->cur_offsets = offsets;
  h->cur_out = *ae ? nullptr : out;
  emb_status_t r = lookup_phase0(h, st);
  if (r == EMB_OK) r = lookup_phase1(h, st);
  if (r == EMB_OK) r = lookup_phase2(h, st);
  if (r != EMB_OK) return r;
  h->state = 1;
  if (*ae) return fail(h, EMB_ERR_INVALID, std::string(ae) + " (the rank took part with an empty batch; the step "
                                                              "updates nothing on any rank)");
  if (h->pf_mismatch) return fail(h, EMB_ERR_INVALID, PF_MISMATCH_MSG);
  return check_sticky(h);
}

emb_status_t backward_impl(emb_ctx *h, const float *d_out, double lr, cudaStream_t st) {
  if (h->state != 1) return fail(h, EMB_ERR_STATE, "emb_backward_update without a preceding emb_lookup");
  if (h->group) return fail(h, EMB_ERR_STATE, "a group handle steps through emb_backward_update_group");
  const bool bad_dout = h->batch > 0 && (!d_out || !aligned16(d_out));
  CUDA_TRY(h, cudaSetDevice(h->device));
  h->last_stream = st;
  if (h->world == 1) {
    if (bad_dout) return fail(h, EMB_ERR_INVALID, "d_out must be a non-NULL 16-byte aligned device pointer");
    GradArgs g = grad_args(h, d_out, lr);
    g.skey = h->skey;
    g.spay = h->spay;
    g.n = h->nnz;
    g.src_mode = 0;
    g.sink_mode = 0;
    // a step whose input had an error updates nothing (decided on the device: deterministic)
    g.skip_mask = EMB_DEVERR_RANGE | EMB_DEVERR_INVALID | EMB_DEVERR_INTERNAL;
    if (h->pf.requested) CUDA_TRY(h, cudaEventRecord(h->ev_pre, st));
    LAUNCH(h, KID_GRAD_APPLY, st, launch_grad(g, st));
    h->state = 0;
    return launch_prefetch(h);
  }
  emb_status_t r = backward_phase0(h, bad_dout ? nullptr : d_out, lr, st);
  if (r == EMB_OK) r = backward_phase1(h, lr, st);
  h->state = 0;
  if (r != EMB_OK) return r;
  if (bad_dout)
    return fail(h, EMB_ERR_INVALID, "d_out must be a non-NULL 16-byte aligned device pointer (the rank took part; "
                                    "the step updates nothing on any rank)");
  return check_sticky(h);
}

// group mode: run phase `ph` of every rank, each after every rank's previous phase (cross-stream
// events), so the flag waits inside a phase always find their flags raised
template <typename F>
emb_status_t group_phase(emb_ctx *const *hs, int n, void *const *streams, F &&phase) {
  for (int r = 0; r < n; ++r) {
    emb_ctx *h = hs[r];
    cudaStream_t st = static_cast<cudaStream_t>(streams ? streams[r] : nullptr);
    CUDA_TRY(h, cudaSetDevice(h->device));
    for (int p = 0; p < n; ++p)
      if (p != r) CUDA_TRY(h, cudaStreamWaitEvent(st, hs[p]->ev_phase, 0));
  }
  for (int r = 0; r < n; ++r) {
    emb_ctx *h = hs[r];
    cudaStream_t st = static_cast<cudaStream_t>(streams ? streams[r] : nullptr);
    CUDA_TRY(h, cudaSetDevice(h->device));
    h->last_stream = st;
    emb_status_t s = phase(h, r, st);
    if (s != EMB_OK) return s;
    CUDA_TRY(h, cudaEventRecord(h->ev_phase, st));
  }
  return EMB_OK;
}

emb_status_t check_group(emb_ctx *const *hs, int n) {
  if (!hs || n < 1) return EMB_ERR_INVALID;
  for (int r = 0; r < n; ++r)
    if (!hs[r] || !hs[r]->group || hs[r]->world != n || hs[r]->rank != r) return EMB_ERR_INVALID;
  return EMB_OK;
}

// host-side unique of the last step (runs the GPU dedup kernel on demand)
emb_status_t ensure_unique(emb_ctx *h) {
  if (h->U_l >= 0) return EMB_OK;
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
  if (h->world == 1 || h->owner_unique_done) return EMB_OK;
  emb_status_t s = sync_counts(h);
  if (s != EMB_OK) return s;
  if (h->n_recv > 0) {
    cudaStream_t st = h->last_stream;
    UniqueArgs ua{h->ok0, h->n_recv, h->ouseg, h->oukey, h->oustart, h->ouend, h->ou_count, h->ouniq_status,
                  h->ouniq_counter, ++h->ouniq_epoch};
    CUDA_TRY(h, launch_unique(ua, st));
    CUDA_TRY(h, cudaStreamSynchronize(st));
  }
  h->owner_unique_done = true;
  return EMB_OK;
}

emb_status_t copy_unique(emb_ctx *h, const uint32_t *uend_dev, const uint32_t *ukey_dev, const uint32_t *ustart_dev,
                         int64_t U, bool owner_local_keys, uint64_t *keys_host, int64_t *counts_host, int64_t cap,
                         int64_t *n_out) {
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
      uint64_t g = k[u];
      if (owner_local_keys) {  // owner-side local id -> global
        const uint64_t local = k[u];
        g = h->shard == 0 ? local * (uint64_t)h->world + (uint64_t)h->rank
                          : (uint64_t)h->rank * h->ks.rows_per + local;
      }
      keys_host[u] = g;
    }
    if (counts_host) counts_host[u] = (int64_t)e[u] - (int64_t)s[u];
  }
  return EMB_OK;
}

// ---- host-buffer (e2e) path: double-buffered staging, asynchronous. A call returns after enqueueing:
// the H2D copies of step k run on h2d_stream as soon as staging set k & 1 is free (its step k-2 backward
// completed), the device work on the caller stream after them, the D2H of Y on d2h_stream after the
// lookup -- so the D2H of Y_k overlaps the H2D of dY_k and of the ids of step k+1 (the two PCIe
// directions). emb_host_sync waits for all of it.
emb_status_t ensure_staging(emb_ctx *h) {
  if (h->st_ids[0]) return EMB_OK;
  const size_t SB = (size_t)h->S * h->max_batch;
  for (int k = 0; k < 2; ++k)
    if (dalloc(h, &h->st_ids[k], h->max_ids) || dalloc(h, &h->st_offsets[k], SB + 1) ||
        dalloc(h, &h->st_out[k], SB * h->D) || dalloc(h, &h->st_dout[k], SB * h->D))
      return fail(h, EMB_ERR_NOMEM, "cannot allocate host-path staging");
  CUDA_TRY(h, cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking));
  CUDA_TRY(h, cudaStreamCreateWithFlags(&h->d2h_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k)
    for (cudaEvent_t *e : {&h->ev_h2d[k], &h->ev_h2d2[k], &h->ev_looked[k], &h->ev_d2h[k], &h->ev_free[k]})
      CUDA_TRY(h, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
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
  emb_status_t s = create_impl(cfg, h, 0);
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

emb_status_t emb_create_group(const emb_config_t *cfgs, int32_t n, emb_handle_t *out) {
  if (!out || !cfgs || n < 1 || n > EMB_MAX_WORLD) return EMB_ERR_INVALID;
  for (int r = 0; r < n; ++r) out[r] = nullptr;
  int64_t cap = 0;
  for (int r = 0; r < n; ++r) {
    if (cfgs[r].world != n || cfgs[r].rank != r) {
      std::lock_guard<std::mutex> lk(g_err_mu);
      g_create_error = "emb_create_group: cfgs[r] must have world == n and rank == r";
      return EMB_ERR_INVALID;
    }
    cap = std::max<int64_t>(cap, cfgs[r].max_ids);
  }
  std::vector<emb_ctx *> hs(n, nullptr);
  emb_status_t s = EMB_OK;
  std::string msg;
  for (int r = 0; r < n && s == EMB_OK; ++r) {
    hs[r] = new (std::nothrow) emb_ctx();
    if (!hs[r]) {
      s = EMB_ERR_NOMEM;
      msg = "out of host memory";
      break;
    }
    s = create_impl(&cfgs[r], hs[r], std::max<int64_t>(cap, 1));
    if (s != EMB_OK) msg = hs[r]->last_error;
  }
  if (s == EMB_OK && n > 1) {
    s = setup_group(hs);
    if (s != EMB_OK)
      for (auto *h : hs)
        if (h && h->last_error != "no error") msg = h->last_error;
  }
  if (s != EMB_OK) {
    {
      std::lock_guard<std::mutex> lk(g_err_mu);
      g_create_error = msg;
    }
    for (auto *h : hs) destroy_impl(h);
    return s;
  }
  for (int r = 0; r < n; ++r) out[r] = hs[r];
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
  if (h->group && h->world > 1) return fail(h, EMB_ERR_STATE, "a group handle prefetches through emb_lookup_prefetch_group");
  return lookup_prefetch_impl(h, ids, offsets, batch, nnz, static_cast<cudaStream_t>(cuda_stream));
}

emb_status_t emb_lookup_prefetch_group(emb_handle_t *hs, int32_t n, const int64_t *const *ids,
                                       const int64_t *const *offsets, const int32_t *batch, const int64_t *nnz,
                                       void *const *streams) {
  if (check_group(hs, n) != EMB_OK || !ids || !offsets || !batch || !nnz) return EMB_ERR_INVALID;
  // every rank's first phase only raises flags (no waits), so the ranks' prefetches need no ordering
  // among themselves; the next emb_lookup_group orders its second phase after all of them
  emb_status_t first_err = EMB_OK;
  for (int r = 0; r < n; ++r) {
    emb_status_t s = lookup_prefetch_impl(hs[r], ids[r], offsets[r], batch[r], nnz[r],
                                          static_cast<cudaStream_t>(streams ? streams[r] : nullptr));
    if (s != EMB_OK && first_err == EMB_OK) first_err = s;
  }
  return first_err;
}

emb_status_t emb_backward_update(emb_handle_t h, const float *d_out, double lr, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  if (h->world == 1 && h->state == 1) {
    emb_status_t s = check_sticky(h);  // fail fast (the device skips the update anyway)
    if (s != EMB_OK) {
      h->state = 0;
      return s;
    }
  }
  return backward_impl(h, d_out, lr, static_cast<cudaStream_t>(cuda_stream));
}

emb_status_t emb_lookup_group(emb_handle_t *hs, int32_t n, const int64_t *const *ids, const int64_t *const *offsets,
                              const int32_t *batch, const int64_t *nnz, float *const *out, void *const *streams) {
  if (check_group(hs, n) != EMB_OK || !ids || !offsets || !batch || !nnz || !out) return EMB_ERR_INVALID;
  for (int r = 0; r < n; ++r)
    if (hs[r]->state != 0) return fail(hs[r], EMB_ERR_STATE, "emb_lookup_group called twice without a backward");
  emb_status_t first_err = EMB_OK;
  for (int r = 0; r < n; ++r) {
    emb_ctx *h = hs[r];
    const char *ae = lookup_arg_error(h, ids[r], offsets[r], batch[r], nnz[r], out[r]);
    h->launches = 0;
    h->step_err_bits = *ae ? EMB_DEVERR_INVALID : 0u;
    h->batch = *ae ? 0 : batch[r];
    h->nnz = *ae ? 0 : nnz[r];
    h->cur_ids = ids[r];
    h->cur_offsets = offsets[r];
    h->cur_out = *ae ? nullptr : out[r];
    if (*ae && first_err == EMB_OK) first_err = fail(h, EMB_ERR_INVALID, std::string("rank ") + std::to_string(r) + ": " + ae);
  }
  if (n == 1) {  // a group of one is a W = 1 layer
    emb_ctx *h = hs[0];
    if (first_err != EMB_OK) return first_err;
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(streams ? streams[0] : nullptr);
    h->last_stream = st;
    emb_status_t s = check_sticky(h);
    if (s != EMB_OK) return s;
    s = lookup_w1(h, ids[0], offsets[0], batch[0], nnz[0], out[0], st);
    if (s != EMB_OK) return s;
    h->U_l = -1;
    h->state = 1;
    return EMB_OK;
  }
  emb_status_t s = group_phase(hs, n, streams, [](emb_ctx *h, int, cudaStream_t st) { return lookup_phase0(h, st); });
  if (s == EMB_OK)
    s = group_phase(hs, n, streams, [](emb_ctx *h, int, cudaStream_t st) { return lookup_phase1(h, st); });
  if (s == EMB_OK)
    s = group_phase(hs, n, streams, [](emb_ctx *h, int, cudaStream_t st) { return lookup_phase2(h, st); });
  if (s != EMB_OK) return s;
  for (int r = 0; r < n; ++r) hs[r]->state = 1;
  if (first_err != EMB_OK) return first_err;
  for (int r = 0; r < n; ++r)
    if (hs[r]->pf_mismatch) return fail(hs[r], EMB_ERR_INVALID, std::string("rank ") + std::to_string(r) + ": " + PF_MISMATCH_MSG);
  for (int r = 0; r < n; ++r) {
    emb_status_t e = check_sticky(hs[r]);
    if (e != EMB_OK) return e;
  }
  return EMB_OK;
}

emb_status_t emb_backward_update_group(emb_handle_t *hs, int32_t n, const float *const *d_out, double lr,
                                       void *const *streams) {
  if (check_group(hs, n) != EMB_OK || !d_out) return EMB_ERR_INVALID;
  for (int r = 0; r < n; ++r)
    if (hs[r]->state != 1) return fail(hs[r], EMB_ERR_STATE, "emb_backward_update_group without a lookup");
  if (n == 1) {
    emb_ctx *h = hs[0];
    h->group = false;  // (the W = 1 path of backward_impl)
    emb_status_t s = emb_backward_update(h, d_out[0], lr, streams ? streams[0] : nullptr);
    h->group = true;
    return s;
  }
  emb_status_t first_err = EMB_OK;
  std::vector<const float *> dd(n);
  for (int r = 0; r < n; ++r) {
    const bool bad = hs[r]->batch > 0 && (!d_out[r] || !aligned16(d_out[r]));
    dd[r] = bad ? nullptr : d_out[r];
    if (bad && first_err == EMB_OK) first_err = fail(hs[r], EMB_ERR_INVALID, "d_out must be a non-NULL 16-byte aligned device pointer");
  }
  emb_status_t s = group_phase(hs, n, streams,
                               [&](emb_ctx *h, int r, cudaStream_t st) { return backward_phase0(h, dd[r], lr, st); });
  if (s == EMB_OK)
    s = group_phase(hs, n, streams, [&](emb_ctx *h, int, cudaStream_t st) { return backward_phase1(h, lr, st); });
  for (int r = 0; r < n; ++r) hs[r]->state = 0;
  if (s != EMB_OK) return s;
  if (first_err != EMB_OK) return first_err;
  for (int r = 0; r < n; ++r) {
    emb_status_t e = check_sticky(hs[r]);
    if (e != EMB_OK) return e;
  }
  return EMB_OK;
}

emb_status_t emb_lookup_host(emb_handle_t h, const int64_t *ids, const int64_t *offsets, int32_t batch, int64_t nnz,
                             float *out, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  if (batch < 0 || batch > h->max_batch || nnz < 0 || nnz > h->max_ids)
    return fail(h, EMB_ERR_INVALID, "batch/nnz out of range");
  if ((batch > 0 && (!offsets || !out)) || (nnz > 0 && !ids)) return fail(h, EMB_ERR_INVALID, "NULL host buffer");
  if (h->state != 0) return fail(h, EMB_ERR_STATE, "emb_lookup_host called twice without a backward");
  CUDA_TRY(h, cudaSetDevice(h->device));
  emb_status_t s = ensure_staging(h);
  if (s != EMB_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const size_t SB = (size_t)h->S * batch;
  const int k = h->st_set;
  h->host_set = k;
  h->st_set ^= 1;
  h->host_stream = st;
  // inputs into set k once its previous user (step k-2's backward) is done
  CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_free[k], 0));
  if (nnz > 0) CUDA_TRY(h, cudaMemcpyAsync(h->st_ids[k], ids, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, h->h2d_stream));
  if (batch > 0)
    CUDA_TRY(h, cudaMemcpyAsync(h->st_offsets[k], offsets, sizeof(int64_t) * (SB + 1), cudaMemcpyHostToDevice,
                                h->h2d_stream));
  CUDA_TRY(h, cudaEventRecord(h->ev_h2d[k], h->h2d_stream));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_h2d[k], 0));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_d2h[k], 0));  // step k-2's Y left st_out[k]
  s = lookup_impl(h, h->st_ids[k], h->st_offsets[k], batch, nnz, h->st_out[k], st);
  if (s != EMB_OK && h->state != 1) return s;  // (at W > 1 a failed call still took part: copy what there is)
  CUDA_TRY(h, cudaEventRecord(h->ev_looked[k], st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->d2h_stream, h->ev_looked[k], 0));
  if (batch > 0 && h->batch > 0)
    CUDA_TRY(h, cudaMemcpyAsync(out, h->st_out[k], sizeof(float) * SB * h->D, cudaMemcpyDeviceToHost, h->d2h_stream));
  CUDA_TRY(h, cudaEventRecord(h->ev_d2h[k], h->d2h_stream));
  return s;
}

emb_status_t emb_backward_update_host(emb_handle_t h, const float *d_out, double lr, void *cuda_stream) {
  if (!h) return EMB_ERR_INVALID;
  if (!h->st_ids[0] || h->state != 1)
    return fail(h, EMB_ERR_STATE, "emb_backward_update_host without a preceding emb_lookup_host");
  CUDA_TRY(h, cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const size_t SB = (size_t)h->S * h->batch;
  const int k = h->host_set;
  if (h->batch > 0) {
    if (!d_out) return fail(h, EMB_ERR_INVALID, "NULL d_out");
    CUDA_TRY(h, cudaMemcpyAsync(h->st_dout[k], d_out, sizeof(float) * SB * h->D, cudaMemcpyHostToDevice, h->h2d_stream));
  }
  CUDA_TRY(h, cudaEventRecord(h->ev_h2d2[k], h->h2d_stream));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_h2d2[k], 0));
  emb_status_t s = emb_backward_update(h, h->st_dout[k], lr, st);
  CUDA_TRY(h, cudaEventRecord(h->ev_free[k], st));
  return s;
}

emb_status_t emb_host_sync(emb_handle_t h) {
  if (!h) return EMB_ERR_INVALID;
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (h->h2d_stream) CUDA_TRY(h, cudaStreamSynchronize(h->h2d_stream));
  if (h->host_stream) CUDA_TRY(h, cudaStreamSynchronize(h->host_stream));
  if (h->d2h_stream) CUDA_TRY(h, cudaStreamSynchronize(h->d2h_stream));
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
    s = ensure_owner_unique(h);
    if (s != EMB_OK) return s;
    info->recv_keys = h->n_recv;
    for (int p = 0; p < h->world; ++p) {
      info->send_counts[p] = h->send_counts[p];
      info->recv_counts[p] = h->recv_counts[p];
    }
    uint32_t u = 0;
    if (h->n_recv > 0) CUDA_TRY(h, cudaMemcpy(&u, h->ou_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    info->unique_owner = u;
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
  return copy_unique(h, h->uend, h->ukey, h->ustart, U, false, keys_host, counts_host, cap, n_out);
}

emb_status_t emb_last_owner_unique(emb_handle_t h, uint64_t *keys_host, int64_t *counts_host, int64_t cap,
                                   int64_t *n_out) {
  if (!h) return EMB_ERR_INVALID;
  if (h->world == 1) return emb_last_unique(h, keys_host, counts_host, cap, n_out);
  CUDA_TRY(h, cudaSetDevice(h->device));
  emb_status_t s = ensure_owner_unique(h);  // (syncs the counts and builds the owner dedup on demand)
  if (s != EMB_OK) return s;
  uint32_t U = 0;
  if (h->n_recv > 0) CUDA_TRY(h, cudaMemcpy(&U, h->ou_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return copy_unique(h, h->ouend, h->oukey, h->oustart, U, true, keys_host, counts_host, cap, n_out);
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
  // diagnostics: EMB_PROFILE_TIMELINE=<path prefix> writes every profiled launch (kernel, start, end in
  // ms from the first profiled launch) to <prefix>.rank<r>.txt
  if (const char *tl = getenv("EMB_PROFILE_TIMELINE")) {
    std::string path = std::string(tl) + ".rank" + std::to_string(h->rank) + ".txt";
    if (FILE *f = fopen(path.c_str(), "w")) {
      for (size_t i = 0; i < h->prof_kid.size(); ++i) {
        float t0 = 0, t1 = 0;
        cudaEventElapsedTime(&t0, h->prof_ev[0], h->prof_ev[2 * i]);
        cudaEventElapsedTime(&t1, h->prof_ev[0], h->prof_ev[2 * i + 1]);
        fprintf(f, "%s %.4f %.4f\n", kKernelNames[h->prof_kid[i]], t0, t1);
      }
      fclose(f);
    }
  }
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
  // a pass stopped by a tripped guard can leave segment tickets taken: start clean
  CUDA_TRY(h, cudaMemset(h->tickets, 0, sizeof(uint32_t) * h->nticket));
  CUDA_TRY(h, cudaDeviceSynchronize());
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
