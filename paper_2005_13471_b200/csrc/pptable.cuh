// pptable.cuh -- evaluation of the per-angle box-spline tables (see tables.cu).
#pragma once

#include "common.cuh"

namespace bsct {

enum PPKind : int {
  PP_GRAM = 0,  // [l|c|, l|c|, l|s|, l|s|, zeta, zeta]
  PP_BP = 1,    // [l|c|, l|s|, zeta] U [lambda_y]^(d+1), d = #nonzero(first 3) - 1
  PP_FWD = 2    // [l|c|, l|s|, zeta]                                         (Eq.(3), Eq.(4))
};

// Device-side view with typed coefficients.
template <typename T>
struct PPView {
  const int *__restrict__ npieces;
  const int *__restrict__ nwidths;
  const double *__restrict__ half;
  const double *__restrict__ knots;  // [n][PP_MAXP+1]
  const T *__restrict__ coef;        // [n][PP_MAXP][PP_NC]
};

// Horner in local coordinate t on piece j of angle a (degree <= 5, zero padded).
template <typename T>
__device__ __forceinline__ T pp_horner(const T *__restrict__ c, T t) {
  T r = c[5];
  r = fma(r, t, c[4]);
  r = fma(r, t, c[3]);
  r = fma(r, t, c[2]);
  r = fma(r, t, c[1]);
  r = fma(r, t, c[0]);
  return r;
}

// M_W(x) for angle a; x in FP64 (the argument must be accurate, SURVEY.md 7 "Gram
// argument"), polynomial in T.  n = 1 widths: half-open box [-w/2, w/2) (R6).
template <typename T>
__device__ __forceinline__ T pp_eval(const PPView<T> &tb, int a, double x) {
  const double H = tb.half[a];
  if (tb.nwidths[a] == 1) return (x >= -H && x < H) ? (T)(0.5 / H) : (T)0;
  const double ax = fabs(x);
  if (!(ax < H)) return (T)0;
  const double *kn = tb.knots + (size_t)a * (PP_MAXP + 1);
  int lo = 0, hi = tb.npieces[a] - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (kn[mid] <= ax) lo = mid; else hi = mid - 1;
  }
  const T t = (T)(ax - kn[lo]);
  return pp_horner<T>(tb.coef + ((size_t)a * PP_MAXP + lo) * PP_NC, t);
}

}  // namespace bsct
