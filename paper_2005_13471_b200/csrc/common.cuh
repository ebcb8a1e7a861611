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

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

// Per-angle piecewise-polynomial table of a centred univariate box spline M_W
// restricted to its right half [0, W/2] (M_W is even).  Built on the device in FP64
// (tables.cu) from the truncated-power subset sum; evaluated with Horner in local
// coordinates t = |x| - knot_j (no catastrophic cancellation).
constexpr int PP_MAXW = 6;        // widths per kernel (Gram: 6, BP: <= 6, forward: <= 3)
constexpr int PP_MAXP = 34;       // right-half pieces (<= 2^(PP_MAXW-1) + 1)
constexpr int PP_NC = 8;          // coefficients per piece (degree <= PP_MAXW - 1), padded



}  // namespace bsct
