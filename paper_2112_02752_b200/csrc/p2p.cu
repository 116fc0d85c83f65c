// p2p.cu — the world > 1 exchange over NVLink peer memory (the synchronous analogue of
// the paper's push-pull PS executor: a worker pulls the rows it needs and
// pushes its gradients to the rows' owner).
//
// Every rank maps its peers' exchange buffers and table shard once at create (CUDA IPC handles
// all-gathered over NCCL, or plain pointers when all ranks live in one process). One step, no host
// synchronisation (e = the step's epoch):
//   A3+A4 k_route (route.cu): my distinct keys -> each owner's receive region for me; per-owner
//                counts + my input-error bits -> every owner's xmat; raises KEYS(e).
//   A5    owner: wait KEYS(e), stable merge of the W received runs (side stream).
//   A6    k_pull: wait APPLIED(e-1) (every owner finished the previous update), then read my remote
//                distinct rows straight from the owners' shards over NVLink.
//   B2    k_grad MODE 3 (grad.cu): my merged per-key gradients -> each owner's gradient region for
//                me; raises GRADS(e).
//   B3+B4 owner: wait GRADS(e), merge the W sources per row in source-rank order + apply; raises
//                APPLIED(e).
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

// wait for flag `kind` == epoch from every source
__global__ void k_wait(P2PArgs a, int kind, uint64_t epoch, uint32_t *err) {
  if (threadIdx.x == 0) p2p_spin(a, kind, epoch, err);
}
cudaError_t launch_wait(const P2PArgs &a, int kind, uint64_t epoch, uint32_t *err, cudaStream_t st) {
  k_wait<<<1, 32, 0, st>>>(a, kind, epoch, err);
  return cudaGetLastError();
}

// A6 pull: uniq_rows[o*cap + i][:] = peer_w[o][send_local[o*cap + i]][:] for every remote owner o,
// i < scnt[o]. A row is D/4 float4 chunks; the flattened (row, chunk) index space of all remote
// owners is walked grid-stride with PULL_UNROLL independent peer loads in flight per thread before
// the stores (NVLink round trips are long; the loads of a thread are independent).
namespace {
constexpr int PULL_THREADS = 256;
constexpr int PULL_UNROLL = 4;
}  // namespace

__global__ void __launch_bounds__(PULL_THREADS) k_pull(P2PArgs a, const int64_t *__restrict__ scnt,
                                                       const uint32_t *__restrict__ send_local,
                                                       float4 *__restrict__ uniq_rows, int d4) {
  __shared__ int64_t pre[P2P_MAXW + 1];
  __shared__ int32_t own[P2P_MAXW];
  const int W = a.world;
  if (threadIdx.x == 0) {  // compact prefix over the remote owners
    int64_t s = 0;
    int q = 0;
    for (int o = 0; o < W; ++o) {
      if (o == a.rank) continue;
      pre[q] = s;
      own[q] = o;
      s += scnt[o];
      ++q;
    }
    pre[q] = s;
    for (int r = q + 1; r <= P2P_MAXW; ++r) pre[r] = s;
  }
  __syncthreads();
  const int nq = W - 1;
  const int64_t total = pre[nq] * d4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * PULL_UNROLL) {
    float4 v[PULL_UNROLL];
    float4 *dst[PULL_UNROLL];
#pragma unroll
    for (int u = 0; u < PULL_UNROLL; ++u) {
      const int64_t t = t0 + u * stride;
      dst[u] = nullptr;
      if (t < total) {
        const int64_t r = t / d4;
        const int c = (int)(t - r * d4);
        int q = 0;
        while (q + 1 < nq && r >= pre[q + 1]) ++q;
        const int o = own[q];
        const int64_t slot = (int64_t)o * a.cap + (r - pre[q]);
        const uint32_t lr = send_local[slot];
        v[u] = ld_nc_f4(reinterpret_cast<const float4 *>(a.peer_w[o]) + (size_t)lr * d4 + c);
        dst[u] = uniq_rows + (size_t)slot * d4 + c;
      }
    }
#pragma unroll
    for (int u = 0; u < PULL_UNROLL; ++u)
      if (dst[u]) *dst[u] = v[u];
  }
}

cudaError_t launch_pull(const P2PArgs &a, const int64_t *scnt, const uint32_t *send_local, float *uniq_rows,
                        int dim, int64_t max_rows, cudaStream_t st) {
  if (a.world <= 1) return cudaSuccess;
  const int d4 = dim / 4;
  int64_t blocks = (max_rows * d4 + PULL_THREADS * PULL_UNROLL - 1) / (PULL_THREADS * PULL_UNROLL);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_pull<<<(unsigned)blocks, PULL_THREADS, 0, st>>>(a, scnt, send_local, reinterpret_cast<float4 *>(uniq_rows),
                                                    d4);
  return cudaGetLastError();
}

}  // namespace emb
