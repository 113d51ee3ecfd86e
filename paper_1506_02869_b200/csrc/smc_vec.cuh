// smc_vec.cuh -- candidate vectors for K2 (sm_100a packed FP32).
//
// A K2 lane carries NC in {1, 2} MH candidates of one aircraft through the same
// arithmetic (common random numbers).  With NC = 2 the two
// candidates' values live in one float2 and every add / mul / fma is a single
// packed FADD2 / FMUL2 / FFMA2 instruction (sm_100: same FMA throughput as the
// scalar forms, half the issue slots -- tools/micro/ffma2.cu); the SASS forms
// take a broadcast scalar (R.F32) or immediate operand and |abs| / negation
// modifiers, so scalar coefficients cost nothing extra.  MUFU functions,
// comparisons and selects stay per candidate (vmap / cget).
#pragma once
#include <cuda_runtime.h>

namespace smc {

template <int NC> struct VecOf { using type = float; };
template <> struct VecOf<2> { using type = float2; };
template <int NC> using vec_t = typename VecOf<NC>::type;

__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 operator-(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 operator-(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 operator*(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 operator+(float2 a, float b) { return __fadd2_rn(a, make_float2(b, b)); }
__device__ __forceinline__ float2 operator-(float2 a, float b) { return __fadd2_rn(a, make_float2(-b, -b)); }
__device__ __forceinline__ float2 operator-(float b, float2 a) { return __fadd2_rn(make_float2(b, b), make_float2(-a.x, -a.y)); }
__device__ __forceinline__ float2 operator*(float2 a, float b) { return __fmul2_rn(a, make_float2(b, b)); }
__device__ __forceinline__ float2 operator*(float b, float2 a) { return __fmul2_rn(make_float2(b, b), a); }

// a * b + c, one rounding
__device__ __forceinline__ float vfma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float b, float2 c) { return __ffma2_rn(a, make_float2(b, b), c); }
__device__ __forceinline__ float2 vfma(float a, float2 b, float2 c) { return __ffma2_rn(make_float2(a, a), b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float c) { return __ffma2_rn(a, b, make_float2(c, c)); }
__device__ __forceinline__ float2 vfma(float2 a, float b, float c) { return __ffma2_rn(a, make_float2(b, b), make_float2(c, c)); }

__device__ __forceinline__ float vabs(float a) { return fabsf(a); }
__device__ __forceinline__ float2 vabs(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }

// component access
__device__ __forceinline__ float cget(float a, int) { return a; }
__device__ __forceinline__ float cget(float2 a, int c) { return c ? a.y : a.x; }
__device__ __forceinline__ void cset(float &a, int, float v) { a = v; }
__device__ __forceinline__ void cset(float2 &a, int c, float v) { if (c) a.y = v; else a.x = v; }

template <class V> __device__ __forceinline__ V vsplat(float s);
template <> __device__ __forceinline__ float vsplat<float>(float s) { return s; }
template <> __device__ __forceinline__ float2 vsplat<float2>(float s) { return make_float2(s, s); }

// per-component scalar function
template <class F> __device__ __forceinline__ float vmap(float a, F f) { return f(a); }
template <class F> __device__ __forceinline__ float2 vmap(float2 a, F f) { return make_float2(f(a.x), f(a.y)); }

}  // namespace smc
