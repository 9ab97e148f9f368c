// common.cuh — shared device helpers for the spmk sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace spmk_dev {

// Modes of the row currently swept by a work unit (seq_sweep / par_ws):
//   NORMAL     row owned by this unit, finished by it (possibly past the tile
//              end, "owner extends" into the next tile only).
//   ENTER_LONG long row that started before this tile: emit one partial per
//              chunk into the H slots (reference head slots, kernels.hpp:419-424
//              / :303-307) so the fix-up can add them in ascending order.
//   OWNER_LONG long row that starts here and runs >= 2 tiles further: emit the
//              prefix (reference order) into this tile's T slot and stop.
enum : int { MODE_NORMAL = 0, MODE_ENTER_LONG = 1, MODE_OWNER_LONG = 2 };

// Exact reference arithmetic: the reference is compiled without -march (no FMA
// contraction), so `acc += v * x` is two roundings.
__device__ __forceinline__ float mul_add_rn(float acc, float v, float x) {
  return __fadd_rn(acc, __fmul_rn(v, x));
}

// Packed fp32 pairs (sm_100 FMUL2 / FFMA2).  Both lanes round to nearest like
// the scalar ops, so results are bit-identical to __fmul_rn / __fadd_rn.
// ptxas contracts mul.rn.f32x2 followed by add.rn.f32x2 into ONE FFMA2 (one
// rounding — not the reference's two, tools/probes/f32x2_fusion.cu), even
// with -fmad=false, so the exact add is issued as fma(p, one, acc) with
// `one` = {1.0f, 1.0f} passed in by the host: ptxas cannot see it is 1 and
// cannot fold the product in, and p*1 + acc rounds once = add.rn(acc, p).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2_pack(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(f32x2 r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
// {v*x.lo, v*x.hi}, each rounded (FMUL2 with a broadcast scalar operand)
__device__ __forceinline__ f32x2 f2_mul(float v, f32x2 x) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(v, v)), "l"(x));
  return d;
}
// {acc.lo + p.lo, acc.hi + p.hi}, each rounded once (FFMA2 by `one`)
__device__ __forceinline__ f32x2 f2_add(f32x2 acc, f32x2 p, f32x2 one) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(p), "l"(one), "l"(acc));
  return d;
}
constexpr f32x2 kOnePair = 0x3f8000003f800000ull;

// Streaming loads for the A arrays (read once): bypass L1 allocation and mark
// evict-first in L2 so they do not push X out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ld_stream(const int* ptr, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* ptr, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ int4 ld_stream4(const int* ptr, uint64_t pol) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_stream4(const float* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(ptr), "l"(pol));
  return v;
}
// X gathers: read-only path, normal L1 allocation (hub columns repeat), and
// an L2 evict-last priority against the evict-first A stream, so the dense
// operand keeps its L2 lines when it does not fit (measured on B200: cfg5
// par-ws 2.73 -> 2.57 ms, par-rs 3.11 -> 3.05 ms).
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float ld_x(const float* p) {
  float v;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(evict_last_policy()));
  return v;
}
__device__ __forceinline__ float2 ld_x2(const float* p) {
  float2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(evict_last_policy()));
  return v;
}
__device__ __forceinline__ float4 ld_x4(const float* p) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(evict_last_policy()));
  return v;
}
// Y is written once: streaming store.
__device__ __forceinline__ void st_y(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_y2(float* p, float a, float b) {
  __stcs(reinterpret_cast<float2*>(p), make_float2(a, b));
}
__device__ __forceinline__ void st_y4(float* p, float a, float b, float c, float d) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}

// Lane-group (LPU lanes, LPU | 32) helpers.
template <int LPU>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (LPU == 32) {
    return 0xffffffffu;
  } else {
    return ((1u << LPU) - 1u) << ((threadIdx.x & 31) & ~(LPU - 1));
  }
}
// Group broadcast.  Callers keep the whole warp converged (warp-uniform loop
// trip counts), so the shuffle uses the full mask: a runtime group mask makes
// nvcc wrap every shuffle in a MATCH/REDUX convergence sequence.
template <int LPU, typename T>
__device__ __forceinline__ T gshfl(T v, int src) {
  if constexpr (LPU == 1) {
    return v;
  } else {
    return __shfl_sync(0xffffffffu, v, src, LPU);
  }
}

// Column mapping of a lane inside its group for one column tile of Nt columns.
//   VEC:    lane gl owns [CPL*gl, CPL*gl+CPL)  (float2/float4 loads)
//   scalar: lane gl owns {gl + LPU*k : k < CPL}
template <int LPU, int CPL, bool VEC>
struct ColMap {
  int gl, nt;
  __device__ __forceinline__ bool valid(int k) const {
    return VEC ? (CPL * gl < nt) : (gl + LPU * k < nt);
  }
  __device__ __forceinline__ int off(int k) const {
    return VEC ? CPL * gl + k : gl + LPU * k;
  }
  __device__ __forceinline__ void load(const float* __restrict__ row,
                                       float (&x)[CPL]) const {
    if constexpr (VEC && CPL == 4) {
      if (CPL * gl < nt) {
        float4 t = ld_x4(row + 4 * gl);
        x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
      } else {
#pragma unroll
        for (int k = 0; k < CPL; ++k) x[k] = 0.f;
      }
    } else if constexpr (VEC && CPL == 2) {
      if (CPL * gl < nt) {
        float2 t = ld_x2(row + 2 * gl);
        x[0] = t.x; x[1] = t.y;
      } else {
        x[0] = 0.f; x[1] = 0.f;
      }
    } else {
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[k] = valid(k) ? ld_x(row + off(k)) : 0.f;
    }
  }
  __device__ __forceinline__ void store(float* __restrict__ row,
                                        const float (&v)[CPL]) const {
    if constexpr (VEC && CPL == 4) {
      if (CPL * gl < nt) st_y4(row + 4 * gl, v[0], v[1], v[2], v[3]);
    } else if constexpr (VEC && CPL == 2) {
      if (CPL * gl < nt) st_y2(row + 2 * gl, v[0], v[1]);
    } else {
#pragma unroll
      for (int k = 0; k < CPL; ++k)
        if (valid(k)) st_y(row + off(k), v[k]);
    }
  }
  // plain (cacheable) store for partial slots that are re-read by the fix-up
  __device__ __forceinline__ void store_slot(float* __restrict__ row,
                                             const float (&v)[CPL]) const {
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      if (valid(k)) row[off(k)] = v[k];
  }
};

}  // namespace spmk_dev
