// fmv_common.cuh -- shared types for the B200 FFTMatvec kernels.
//
// Precision tags follow the reference's 5-slot config (config.hpp:14-33):
// 'd' fp64, 's' fp32, plus this project's 'h' fp16 extension. Complex values
// are interleaved pairs (double2 / float2 / __half2), matching the
// reference's std::complex storage (SPEC.md "Complex elements are stored
// interleaved").
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fmv {

enum Prec : int { PD = 0, PS = 1, PH = 2 };

template <int P>
struct PT;
template <>
struct PT<PD> {
  using real = double;
  using cplx = double2;
  using acc = double;
  using cacc = double2;
};
template <>
struct PT<PS> {
  using real = float;
  using cplx = float2;
  using acc = float;
  using cacc = float2;
};
template <>
struct PT<PH> {
  using real = __half;
  using cplx = __half2;
  using acc = float;
  using cacc = float2;
};

// ---- value rounding: "cast to precision P" (precision.hpp:44-61, RNE) ----
template <int P>
__device__ __forceinline__ double rnd(double v) {
  if constexpr (P == PD) return v;
  else if constexpr (P == PS) return (double)__double2float_rn(v);
  else return (double)__half2float(__double2half(v));
}

// ---- conversions between element types (all RNE, single rounding) ----
__device__ __forceinline__ double to_d(double v) { return v; }
__device__ __forceinline__ double to_d(float v) { return (double)v; }
__device__ __forceinline__ double to_d(__half v) { return (double)__half2float(v); }

template <class T>
__device__ __forceinline__ T from_d(double v);
template <>
__device__ __forceinline__ double from_d<double>(double v) { return v; }
template <>
__device__ __forceinline__ float from_d<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ __half from_d<__half>(double v) { return __double2half(v); }

__device__ __forceinline__ double2 to_cd(double2 v) { return v; }
__device__ __forceinline__ double2 to_cd(float2 v) { return make_double2(v.x, v.y); }
__device__ __forceinline__ double2 to_cd(__half2 v) {
  const float2 f = __half22float2(v);
  return make_double2(f.x, f.y);
}

template <class C>
__device__ __forceinline__ C cfrom_d(double2 v);
template <>
__device__ __forceinline__ double2 cfrom_d<double2>(double2 v) { return v; }
template <>
__device__ __forceinline__ float2 cfrom_d<float2>(double2 v) {
  return make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
}
template <>
__device__ __forceinline__ __half2 cfrom_d<__half2>(double2 v) {
  return __halves2half2(__double2half(v.x), __double2half(v.y));
}

// float2 -> narrower/wider complex without a double round trip where exact
template <class C>
__device__ __forceinline__ C cfrom_f(float2 v);
template <>
__device__ __forceinline__ double2 cfrom_f<double2>(float2 v) { return make_double2(v.x, v.y); }
template <>
__device__ __forceinline__ float2 cfrom_f<float2>(float2 v) { return v; }
template <>
__device__ __forceinline__ __half2 cfrom_f<__half2>(float2 v) { return __floats2half2_rn(v.x, v.y); }

// ---- complex helpers in arithmetic type R ----
template <class R>
struct CT;
template <>
struct CT<double> {
  using c = double2;
  static __device__ __forceinline__ c mk(double a, double b) { return make_double2(a, b); }
};
template <>
struct CT<float> {
  using c = float2;
  static __device__ __forceinline__ c mk(float a, float b) { return make_float2(a, b); }
};

template <class C>
__device__ __forceinline__ C cadd(C a, C b) {
  return {a.x + b.x, a.y + b.y};
}
template <class C>
__device__ __forceinline__ C csub(C a, C b) {
  return {a.x - b.x, a.y - b.y};
}
template <class C>
__device__ __forceinline__ C cmul(C a, C b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <class C>
__device__ __forceinline__ C cconj(C a) {
  return {a.x, -a.y};
}
// multiply by +i (s=+1) or -i (s=-1)
template <int S, class C>
__device__ __forceinline__ C cmuli(C a) {
  if constexpr (S > 0) return {-a.y, a.x};
  else return {a.y, -a.x};
}

// Programmatic dependent launch: the hot kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so their CTAs may start
// while the previous kernel drains; griddepcontrol.wait (a no-op for a normal
// launch) blocks until that kernel's memory operations are visible. Every
// kernel calls it before its first global access.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace fmv
