// p2p.cu — the world > 1 exchange over NVLink peer memory (the synchronous analogue of
// the paper's push-pull PS executor: a worker receives the rows it needs and
// pushes its gradients to the rows' owner).
//
// Every rank maps its peers' exchange buffers once at create (CUDA IPC handles all-gathered over NCCL,
// or plain pointers when all ranks live in one process). Every transfer is a peer STORE: peer loads
// through CUDA-IPC mappings measured 19 GB/s against 600 GB/s for stores (profiles/r02_ipc_gather_bench.log).
// One step, no host synchronisation (e = the step's epoch):
//   A3+A4 k_route (route.cu): my distinct keys -> each owner's receive region for me; per-owner
//                counts + my input-error bits -> every owner's xmat; raises KEYS(e).
//   A5    owner: wait KEYS(e), stable merge of the W received runs (side stream).
//   A6    k_gather_push: owner gathers the rows every other rank asked for and stores them into that
//                rank's row region for me; raises ROWS(e). The requester waits ROWS(e), then pools
//                (rows it owns straight from its shard).
//   B2    k_grad MODE 3 (grad.cu): my merged per-key gradients -> each owner's gradient region for
//                me; raises GRADS(e).
//   B3+B4 owner: wait GRADS(e), merge the W sources per row in source-rank order + apply.
// Ordering: writers fence at system scope; the last block (or warp) of the producing kernel raises the
// per-(kind, source) epoch flag in every peer (p2p_dev.cuh); a one-thread k_wait spins (bounded) on the
// flags before the consuming kernel runs on the same stream.
#include "../../include/emb.h"
#include "common.cuh"
#include "internal.h"
#include "p2p_dev.cuh"

namespace emb {

// raise flag `kind` for this rank in every peer (after the previous kernels' peer stores); with
// err_bits, first mark this step as failed at every owner (they skip the update)
__global__ void k_signal(P2PArgs a, int kind, uint32_t err_bits) {
  if (err_bits)
    for (int p = 0; p < a.world; ++p) atomicOr(reinterpret_cast<unsigned long long *>(a.peer_xmat[p] + xmat_idx(a.epoch, 1, a.rank)),
                                               (unsigned long long)err_bits);
  p2p_raise(a, kind);
}
cudaError_t launch_signal(const P2PArgs &a, int kind, uint32_t err_bits, cudaStream_t st) {
  k_signal<<<1, 1, 0, st>>>(a, kind, err_bits);
  return cudaGetLastError();
}

// OR bits into the sticky device error word (a host-detected error of an already routed step)
__global__ void k_mark_err(uint32_t *err, uint32_t bits) { atomicOr(err, bits); }
cudaError_t launch_mark_err(uint32_t *err, uint32_t bits, cudaStream_t st) {
  k_mark_err<<<1, 1, 0, st>>>(err, bits);
  return cudaGetLastError();
}

// wait for flag `kind` == epoch from every source
__global__ void k_wait(P2PArgs a, int kind, uint64_t epoch, uint32_t *err) {
  if (threadIdx.x == 0) p2p_spin(a, kind, epoch, err);
}
cudaError_t launch_wait(const P2PArgs &a, int kind, uint64_t epoch, uint32_t *err, cudaStream_t st) {
  k_wait<<<1, 32, 0, st>>>(a, kind, epoch, err);
  return cudaGetLastError();
}

// A6 + X2: the owner gathers its rows for every other source's received keys and stores them straight
// into that requester's row region for this owner. A row is D/4 float4 chunks; the flattened (row,
// chunk) space of all sources != rank is walked grid-stride with GP_UNROLL independent table loads in
// flight per thread before the peer stores. The last block raises ROWS.
namespace {
constexpr int GP_THREADS = 256;
constexpr int GP_UNROLL = 4;
}  // namespace

__global__ void __launch_bounds__(GP_THREADS) k_gather_push(P2PArgs a, const float4 *__restrict__ w,
                                                            const uint32_t *__restrict__ recv_keys,
                                                            const int64_t *__restrict__ counts, int d4,
                                                            int64_t rows_local, uint32_t *err) {
  __shared__ int64_t pre[P2P_MAXW + 1];
  __shared__ int32_t src[P2P_MAXW];
  const int W = a.world;
  if (threadIdx.x == 0) {  // compact prefix over the other sources
    int64_t s = 0;
    int q = 0;
    for (int o = 0; o < W; ++o) {
      if (o == a.rank) continue;
      pre[q] = s;
      src[q] = o;
      s += counts[o];
      ++q;
    }
    pre[q] = s;
  }
  __syncthreads();
  const int nq = W - 1;
  const int64_t total = pre[nq] * d4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * GP_UNROLL) {
    float4 v[GP_UNROLL];
    float4 *dst[GP_UNROLL];
#pragma unroll
    for (int u = 0; u < GP_UNROLL; ++u) {
      const int64_t t = t0 + u * stride;
      dst[u] = nullptr;
      if (t < total) {
        const int64_t r = t / d4;
        const int c = (int)(t - r * d4);
        int q = 0;
        while (q + 1 < nq && r >= pre[q + 1]) ++q;
        const int s = src[q];
        const int64_t i = r - pre[q];
        const uint32_t lr = recv_keys[(int64_t)s * a.cap + i];
        if ((int64_t)lr >= rows_local) {
          bad = true;
          continue;
        }
        v[u] = ld_nc_f4(w + (size_t)lr * d4 + c);
        dst[u] = reinterpret_cast<float4 *>(a.peer_uniq_rows[s]) + (size_t)((int64_t)a.rank * a.cap + i) * d4 + c;
      }
    }
#pragma unroll
    for (int u = 0; u < GP_UNROLL; ++u)
      if (dst[u]) *dst[u] = v[u];
  }
  if (bad) atomicOr(err, EMB_DEVERR_INTERNAL);
  p2p_signal_last_block(a, P2P_ROWS);
}

cudaError_t launch_gather_push(const P2PArgs &a, const float *w, const uint32_t *recv_keys, const int64_t *counts,
                               int dim, int64_t rows_local, uint32_t *err, cudaStream_t st) {
  const int d4 = dim / 4;
  int64_t blocks = ((int64_t)a.world * a.cap * d4 + GP_THREADS * GP_UNROLL - 1) / (GP_THREADS * GP_UNROLL);
  // 4 blocks per SM keep ~64 KB of row loads in flight per SM (enough for the NVLink stores:
  // profiles/r02_peer_gather_bench.log) and leave warp slots for the concurrent owner merge
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  k_gather_push<<<(unsigned)blocks, GP_THREADS, 0, st>>>(a, reinterpret_cast<const float4 *>(w), recv_keys, counts,
                                                         d4, rows_local, err);
  return cudaGetLastError();
}

// owner: per merged received key, "another rank sent it too" -> the requester's lof byte
__global__ void k_lo_flags(P2PArgs a, const uint32_t *__restrict__ okey, const uint32_t *__restrict__ opay,
                           const int64_t *__restrict__ n_merged, uint32_t *fin, uint32_t *err, uint32_t *err_host) {
  const int64_t n = *n_merged;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = okey[p];
    const bool multi = (p > 0 && okey[p - 1] == k) || (p + 1 < n && okey[p + 1] == k);
    const uint32_t rp = opay[p];  // receive position s * cap + i
    const int64_t s = rp / a.cap, i = rp - s * a.cap;
    a.peer_lof[s][(int64_t)a.rank * a.cap + i] = multi ? 1 : 0;
  }
  p2p_signal_last_block(a, P2P_LOF);
  if (fin && threadIdx.x == 0) finish_publish(fin + 1, fin + 2, 2, err, err_host);  // (the later of this and the pool)
}
cudaError_t launch_lo_flags(const P2PArgs &a, const uint32_t *okey, const uint32_t *opay, const int64_t *n_merged,
                            int64_t max_n, uint32_t *fin, uint32_t *err, uint32_t *err_host, cudaStream_t st) {
  int64_t blocks = (max_n + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks < 1) blocks = 1;
  k_lo_flags<<<(unsigned)blocks, 256, 0, st>>>(a, okey, opay, n_merged, fin, err, err_host);
  return cudaGetLastError();
}

}  // namespace emb
