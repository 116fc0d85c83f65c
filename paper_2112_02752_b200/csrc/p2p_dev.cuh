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

// one thread: spin (bounded) until every peer raised flag `kind` for this epoch
__device__ __forceinline__ void p2p_spin(const P2PArgs &a, int kind, uint32_t *err) {
  for (int s = 0; s < a.world; ++s) {
    const uint64_t *f = a.flags + kind * P2P_MAXW + s;
    uint64_t spins = 0;
    while (ld_acq_sys_u64(f) < a.epoch) {
      __nanosleep(64);
      if (++spins > (1ull << 26)) {  // a peer never arrived: report instead of hanging the GPU
        atomicOr(err, EMB_DEVERR_TIMEOUT);
        break;
      }
    }
  }
  __threadfence_system();
}

// one thread: raise flag `kind` for this rank in every peer
__device__ __forceinline__ void p2p_raise(const P2PArgs &a, int kind) {
  __threadfence_system();
  for (int p = 0; p < a.world; ++p) st_sys_u64(a.peer_flags[p] + kind * P2P_MAXW + a.rank, a.epoch);
}

// block epilogue: after the block's peer stores, the last block to finish raises flag `kind`
__device__ __forceinline__ void p2p_signal_last_block(const P2PArgs &a, int kind) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(a.done + kind, 1u);
    if (t == gridDim.x - 1) {
      a.done[kind] = 0;
      p2p_raise(a, kind);
    }
  }
}

}  // namespace emb
