// p2p.cu — the world > 1 exchange over NVLink peer memory (the synchronous analogue of
// the paper's push-pull PS executor).
//
// Every rank maps its peers' receive buffers (CUDA IPC, handles all-gathered once over NCCL at
// create). One step, no host synchronisation:
//   X0  k_xcounts    : my per-owner key counts -> row `rank` of EVERY rank's W x W count matrix;
//                      spin (bounded) until all W rows arrived, then build the route table (send /
//                      receive offsets, where my keys land in each owner, where rows land in each
//                      requester);
//   X1  k_push_keys  : my distinct keys (local ids) stored straight into each owner's key buffer;
//   X2  k_gather_push: the owner gathers its table rows and stores them straight into the requesting
//                      rank's row buffer, in that rank's send order (gather fused with the exchange);
//   X3  (grad.cu MODE 3): the requester's merged per-key gradient rows are stored straight into the
//                      owner's gradient buffer.
// Ordering: writers fence at system scope (__threadfence_system); the last block (or warp) of the
// producing kernel then raises the per-(kind, source) epoch flag in every peer (p2p_dev.cuh); a
// one-thread k_wait spins on the flags (bounded: a timeout sets EMB_DEVERR_TIMEOUT instead of
// hanging) before the consuming kernel runs on the same stream. Waiting inside the consumers'
// prologues instead was measured slower at W = 4 (spinning grids hold SMs the side-stream merge and
// the gather need).
#include "../../include/emb.h"
#include "common.cuh"
#include "internal.h"
#include "p2p_dev.cuh"

namespace emb {

// X0: write my per-owner counts into row `rank` of every rank's matrix, raise the COUNTS flag, wait
// for every peer's row, then build the route table (one block; everything after reads it)
__global__ void k_xcounts(P2PArgs a, const int64_t *send_counts, uint32_t *err) {
  const int t = threadIdx.x;  // t = p * W + d
  const int W = a.world;
  if (t < W * W) {
    const int p = t / W, d = t % W;
    a.peer_xmat[p][a.rank * W + d] = send_counts[d];
  }
  __syncthreads();
  if (t == 0) {
    p2p_raise(a, P2P_COUNTS);
    p2p_spin(a, P2P_COUNTS, err);
    RouteTable *rt = a.rt;
    const int64_t *m = a.xmat;  // own replica, [src][dst]
    const int r = a.rank;
    int64_t s = 0;
    for (int d = 0; d < W; ++d) {
      rt->soff[d] = s;
      s += m[r * W + d];
    }
    rt->soff[W] = s;
    s = 0;
    for (int q = 0; q < W; ++q) {
      rt->roff[q] = s;
      s += m[q * W + r];
    }
    rt->roff[W] = s;
    for (int d = 0; d < W; ++d) {  // where my keys start in owner d's buffer
      int64_t o = 0;
      for (int q = 0; q < r; ++q) o += m[q * W + d];
      rt->dst_off[d] = o;
    }
    for (int q = 0; q < W; ++q) {  // where requester q expects my rows (its send offset for owner r)
      int64_t o = 0;
      for (int d = 0; d < r; ++d) o += m[q * W + d];
      rt->src_off[q] = o;
    }
    for (int q = 0; q < W; ++q) rt->recv_counts[q] = m[q * W + r];
    rt->n_recv = rt->roff[W];
    rt->n_send = rt->soff[W];
  }
}
cudaError_t launch_xcounts(const P2PArgs &a, const int64_t *send_counts, uint32_t *err, cudaStream_t st) {
  k_xcounts<<<1, 256, 0, st>>>(a, send_counts, err);
  return cudaGetLastError();
}

// raise flag `kind` for this rank in every peer (after the previous kernels' peer stores)
__global__ void k_signal(P2PArgs a, int kind) { p2p_raise(a, kind); }
cudaError_t launch_signal(const P2PArgs &a, int kind, cudaStream_t st) {
  k_signal<<<1, 1, 0, st>>>(a, kind);
  return cudaGetLastError();
}

// wait for flag `kind` from every source
__global__ void k_wait(P2PArgs a, int kind, uint32_t *err) {
  if (threadIdx.x == 0) p2p_spin(a, kind, err);
}
cudaError_t launch_wait(const P2PArgs &a, int kind, uint32_t *err, cudaStream_t st) {
  k_wait<<<1, 32, 0, st>>>(a, kind, err);
  return cudaGetLastError();
}

__device__ __forceinline__ int seg_of(const int64_t *off, int W, int64_t i) {
  int s = 0;
  while (s + 1 < W && i >= off[s + 1]) ++s;
  return s;
}

// X1: my send buffer (owner-major local ids) -> each owner's key buffer
__global__ void k_push_keys(P2PArgs a, const uint32_t *__restrict__ send_keys) {
  const RouteTable *rt = a.rt;
  const int W = a.world;
  const int64_t n = rt->n_send;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int d = seg_of(rt->soff, W, q);
    a.peer_recv_keys[d][rt->dst_off[d] + (q - rt->soff[d])] = send_keys[q];
  }
  p2p_signal_last_block(a, P2P_KEYS);
}
cudaError_t launch_push_keys(const P2PArgs &a, const uint32_t *send_keys, int64_t cap, cudaStream_t st) {
  int64_t blocks = (cap + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  k_push_keys<<<(unsigned)blocks, 256, 0, st>>>(a, send_keys);
  return cudaGetLastError();
}

// X2 fused with the gather: received key i (source s, index q in s's run) -> table row -> requester s's
// row buffer at s's send position (src_off[s] + q). One float4 per thread, a row per D/4 threads.
__global__ void k_gather_push(P2PArgs a, const float4 *__restrict__ w, const uint32_t *__restrict__ recv_keys,
                              int d4, int64_t rows_local, uint32_t *err) {
  const RouteTable *rt = a.rt;
  const int W = a.world;
  const int64_t n = rt->n_recv * d4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / d4;
    const int c = (int)(t - i * d4);
    const int s = seg_of(rt->roff, W, i);
    const uint32_t lr = recv_keys[i];
    if ((int64_t)lr >= rows_local) {
      atomicOr(err, EMB_DEVERR_INTERNAL);
      continue;
    }
    const float4 v = ld_nc_f4(w + (size_t)lr * d4 + c);
    float4 *dst = reinterpret_cast<float4 *>(a.peer_uniq_rows[s]) + (size_t)(rt->src_off[s] + (i - rt->roff[s])) * d4 + c;
    *dst = v;
  }
  p2p_signal_last_block(a, P2P_ROWS);
}
// X3 as a separate stream (experiment knob EMB_GRAD_PUSH=1): the requester's merged gradient rows,
// written locally in send order (grad MODE 2), streamed to each owner's receive buffer with
// contiguous float4 stores; the last block raises GRADS
__global__ void k_push_rows(P2PArgs a, const float4 *__restrict__ rows, int d4) {
  const RouteTable *rt = a.rt;
  const int W = a.world;
  const int64_t n = rt->n_send * d4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = t / d4;
    const int c = (int)(t - q * d4);
    const int d = seg_of(rt->soff, W, q);
    float4 *dst = reinterpret_cast<float4 *>(a.peer_grecv[d]) + (size_t)(rt->dst_off[d] + (q - rt->soff[d])) * d4 + c;
    *dst = rows[t];
  }
  p2p_signal_last_block(a, P2P_GRADS);
}
cudaError_t launch_push_rows(const P2PArgs &a, const float *rows, int dim, int64_t cap, cudaStream_t st) {
  const int d4 = dim / 4;
  int64_t blocks = (cap * d4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_push_rows<<<(unsigned)blocks, 256, 0, st>>>(a, reinterpret_cast<const float4 *>(rows), d4);
  return cudaGetLastError();
}

cudaError_t launch_gather_push(const P2PArgs &a, const float *w, const uint32_t *recv_keys, int dim, int64_t cap,
                               int64_t rows_local, uint32_t *err, cudaStream_t st) {
  const int d4 = dim / 4;
  int64_t blocks = (cap * d4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_gather_push<<<(unsigned)blocks, 256, 0, st>>>(a, reinterpret_cast<const float4 *>(w), recv_keys, d4, rows_local,
                                                   err);
  return cudaGetLastError();
}

}  // namespace emb
