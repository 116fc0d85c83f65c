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
  // read-only streaming load if `pred`, else zeros: a single predicated instruction per 16 / 8 bytes
  __device__ __forceinline__ void load_nc_pred(const float *p, bool pred) {
    const uint32_t q = pred;
    if constexpr (CPL == 2) {
      asm volatile(
          "{\n .reg .pred pp;\n setp.ne.u32 pp, %3, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n"
          " @pp ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];\n}"
          : "=f"(v[0]), "=f"(v[1])
          : "l"(p), "r"(q));
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 4)
        asm volatile(
            "{\n .reg .pred pp;\n setp.ne.u32 pp, %5, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n mov.b32 %2, 0;\n"
            " mov.b32 %3, 0;\n @pp ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n}"
            : "=f"(v[c]), "=f"(v[c + 1]), "=f"(v[c + 2]), "=f"(v[c + 3])
            : "l"(p + c), "r"(q));
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
