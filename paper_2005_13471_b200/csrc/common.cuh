// common.cuh -- shared device helpers of the bsct library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bsct {

template <typename T> struct cplx_of;
template <> struct cplx_of<float> { using type = float2; };
template <> struct cplx_of<double> { using type = double2; };
template <typename T> using cplx = typename cplx_of<T>::type;

template <typename V> __host__ __device__ __forceinline__ V cadd(V a, V b) { return {a.x + b.x, a.y + b.y}; }
template <typename V> __host__ __device__ __forceinline__ V csub(V a, V b) { return {a.x - b.x, a.y - b.y}; }
template <typename V> __host__ __device__ __forceinline__ V cmul(V a, V b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// a * conj(b)
template <typename V> __host__ __device__ __forceinline__ V cmulc(V a, V b) {
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
template <typename V> __host__ __device__ __forceinline__ V cconj(V a) { return {a.x, -a.y}; }
template <typename V, typename S> __host__ __device__ __forceinline__ V cscale(V a, S s) { return {a.x * s, a.y * s}; }

// FP32 complex arithmetic on the packed FP32x2 pipe of sm_100 (add/sub/mul/fma.rn.f32x2:
// FADD2 / FMUL2 / FFMA2, whose operands take swap, broadcast and per-half negation
// modifiers): a complex add is one instruction instead of two, a complex multiply two
// (FMUL2 + FFMA2) instead of four.  Every lane is IEEE round-to-nearest like the scalar
// instructions; the multiply is the usual FMA-contracted form
// (a.x b.x - a.y b.y, a.y b.x + a.x b.y) with the a.? b.x products rounded first.
// BSCT_NO_F32X2 selects the scalar forms (A/B timing).
#if defined(__CUDA_ARCH__) && !defined(BSCT_NO_F32X2)
#define BSCT_F32X2 1
__device__ __forceinline__ unsigned long long x2pack(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 x2unpack(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 x2add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x2pack(a.x, a.y)), "l"(x2pack(b.x, b.y)));
  return x2unpack(d);
}
__device__ __forceinline__ float2 x2sub(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x2pack(a.x, a.y)), "l"(x2pack(b.x, b.y)));
  return x2unpack(d);
}
__device__ __forceinline__ float2 x2mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x2pack(a.x, a.y)), "l"(x2pack(b.x, b.y)));
  return x2unpack(d);
}
__device__ __forceinline__ float2 x2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x2pack(a.x, a.y)), "l"(x2pack(b.x, b.y)), "l"(x2pack(c.x, c.y)));
  return x2unpack(d);
}
#endif

__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#ifdef BSCT_F32X2
  return x2add(a, b);
#else
  return {a.x + b.x, a.y + b.y};
#endif
}
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) {
#ifdef BSCT_F32X2
  return x2sub(a, b);
#else
  return {a.x - b.x, a.y - b.y};
#endif
}
// a * (c + i s) for real c, s (twiddles)
__host__ __device__ __forceinline__ float2 crot(float2 a, float c, float s) {
#ifdef BSCT_F32X2
  return x2fma(float2{a.y, a.x}, float2{-s, s}, x2mul(a, float2{c, c}));
#else
  return {a.x * c - a.y * s, a.x * s + a.y * c};
#endif
}
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) { return crot(a, b.x, b.y); }
__host__ __device__ __forceinline__ float2 cmulc(float2 a, float2 b) { return crot(a, b.x, -b.y); }
// componentwise a * b + c (not a complex product)
__host__ __device__ __forceinline__ float2 cfma2(float2 a, float2 b, float2 c) {
#ifdef BSCT_F32X2
  return x2fma(a, b, c);
#else
  return {fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y)};
#endif
}
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) {
#ifdef BSCT_F32X2
  return x2mul(a, float2{s, s});
#else
  return {a.x * s, a.y * s};
#endif
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

// Per-angle piecewise-polynomial table of a centred univariate box spline M_W
// restricted to its right half [0, W/2] (M_W is even).  Built on the device in FP64
// (tables.cu) from the truncated-power subset sum; evaluated with Horner in local
// coordinates t = |x| - knot_j (no catastrophic cancellation).
constexpr int PP_MAXW = 6;        // widths per kernel (Gram: 6, BP: <= 6, forward: <= 3)
constexpr int PP_MAXP = 34;       // right-half pieces (<= 2^(PP_MAXW-1) + 1)
constexpr int PP_NC = 8;          // coefficients per piece (degree <= PP_MAXW - 1), padded



}  // namespace bsct
