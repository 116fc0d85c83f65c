// vec.cuh — per-lane row fragments: a lane owns CPL consecutive fp32 columns of a row (CPL = 2, 4
// or 8), so one warp-wide access moves a whole 256-B (D=64), 512-B (D=128) or 1-KB (D=256) row.
#pragma once
#include "common.cuh"

namespace emb {

template <int CPL>
struct VecF {
  float v[CPL];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = 0.f;
  }
  // read-only, streaming (table rows, dY rows)
  __device__ __forceinline__ void load_nc(const float *p) {
    if constexpr (CPL == 2) {
      asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v[0]), "=f"(v[1]) : "l"(p));
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 4) {
        const float4 t = ld_nc_f4(reinterpret_cast<const float4 *>(p + c));
        v[c] = t.x; v[c + 1] = t.y; v[c + 2] = t.z; v[c + 3] = t.w;
      }
    }
  }
  // coherent load (rows that this kernel also writes: table / optimizer state)
  __device__ __forceinline__ void load(const float *p) {
    if constexpr (CPL == 2) {
      const float2 t = *reinterpret_cast<const float2 *>(p);
      v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 4) {
        const float4 t = *reinterpret_cast<const float4 *>(p + c);
        v[c] = t.x; v[c + 1] = t.y; v[c + 2] = t.z; v[c + 3] = t.w;
      }
    }
  }
  __device__ __forceinline__ void store(float *p) const {
    if constexpr (CPL == 2) {
      *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 4)
        *reinterpret_cast<float4 *>(p + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    }
  }
  __device__ __forceinline__ void store_cs(float *p) const {
    if constexpr (CPL == 2) {
      st_cs_f2(reinterpret_cast<float2 *>(p), make_float2(v[0], v[1]));
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 4)
        st_cs_f4(reinterpret_cast<float4 *>(p + c), make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]));
    }
  }
};

}  // namespace emb
