// common.cuh — device helpers shared by the sm_100a kernels of libemb (no torch, no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define EMB_SENTINEL 0xFFFFFFFFu  // routing key of an invalid occurrence: sorts last, never applied

// sticky device error bits (emb_status_t values as bit positions)
#define EMB_DEVERR_INVALID 0x2u
#define EMB_DEVERR_RANGE 0x4u
#define EMB_DEVERR_INTERNAL 0x8u  // a data-dependent address failed its bounds guard (bug)
#define EMB_DEVERR_TIMEOUT 0x10u  // a peer never raised an exchange flag (world > 1)

namespace emb {

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- streaming / read-only global access -----------------------------------------------------
__device__ __forceinline__ float4 ld_nc_f4(const float4 *p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_cs_f2(float2 *p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_cs_f4(float4 *p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_cg_d2(const double2 *p) {
  double2 r;
  asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// ---- mbarrier + bulk async copy (TMA engine, 1-D: cp.async.bulk) -------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned),
// completion signalled as tx bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- per-thread async copies (cp.async, SASS LDGSTS): 16 B global -> shared, L2 only ------------
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void *src_gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src_gmem) : "memory");
}
// end-of-kernel hand-off (thread 0 of every block, after the block's work): the last block of the
// kernel bumps kern_ctr; the last of `nkern` concurrently running kernels copies the sticky device
// error word to the mapped host word (replaces a separate publish launch after the stream join)
__device__ __forceinline__ void finish_publish(uint32_t *blk_ctr, uint32_t *kern_ctr, uint32_t nkern,
                                               uint32_t *err, uint32_t *err_host) {
  __threadfence();
  if (atomicAdd(blk_ctr, 1u) != gridDim.x - 1) return;
  *blk_ctr = 0;
  __threadfence();
  if (atomicAdd(kern_ctr, 1u) != nkern - 1) return;
  *kern_ctr = 0;
  __threadfence();
  *(volatile uint32_t *)err_host = atomicOr(err, 0u);
  __threadfence_system();
}

__device__ __forceinline__ void cp_async4(uint32_t dst_smem, const void *src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst_smem), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- warp helpers -----------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

}  // namespace emb
