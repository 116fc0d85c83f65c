// p2p_dev.cuh — in-kernel wait / signal of the world > 1 peer-memory exchange (see p2p.cu).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace emb {

__device__ __forceinline__ void st_sys_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acq_sys_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// one thread: spin (bounded) until every source raised flag `kind` with exactly `epoch`. Exact match:
// under the step protocol a flag never runs more than the awaited step ahead, so a
// value other than `epoch` means a rank skipped a collective call; the wait then times out and sets
// EMB_DEVERR_TIMEOUT (sticky; the consumers skip their work) instead of reading stale buffers. After a
// timeout, later waits return at once (the handles must be recreated).
__device__ __forceinline__ void p2p_spin(const P2PArgs &a, int kind, uint64_t epoch, uint32_t *err) {
  if (ld_cg_u32(err) & EMB_DEVERR_TIMEOUT) return;
  for (int s = 0; s < a.world; ++s) {
    const uint64_t *f = a.flags + kind * P2P_MAXW + s;
    uint64_t spins = 0;
    while (ld_acq_sys_u64(f) != epoch) {
      __nanosleep(64);
      if (++spins > (1ull << 26)) {  // ~4 s: a peer never arrived; report instead of hanging the GPU
        atomicOr(err, EMB_DEVERR_TIMEOUT);
        return;
      }
    }
  }
  __threadfence_system();
}

// one thread: raise flag `kind` for this rank in every peer (after this thread's fence)
__device__ __forceinline__ void p2p_raise(const P2PArgs &a, int kind) {
  __threadfence_system();
  for (int p = 0; p < a.world; ++p) st_sys_u64(a.peer_flags[p] + kind * P2P_MAXW + a.rank, a.epoch);
}

// block epilogue: after the block's peer stores, the last block to finish raises flag `kind`. The
// barrier orders the block's stores before thread 0's system fence (the cooperative-groups grid-sync
// pattern); a fence in every thread made membar the top stall (profiles/r02_ncu_w2_group.txt).
__device__ __forceinline__ void p2p_signal_last_block(const P2PArgs &a, int kind) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t t = atomicAdd(a.done + kind, 1u);
    if (t == gridDim.x - 1) {
      a.done[kind] = 0;
      p2p_raise(a, kind);
    }
  }
}

}  // namespace emb
