// gram.cu -- K1: exact Gram filter taps.
//
//   G[dk] = lambda_x^4 sum_t M_[l|c|, l|c|, l|s|, l|s|, zeta, zeta](lambda_x (-s dk1 + c dk2))
//
// One thread per tap; angles are staged in shared memory in chunks and summed in
// ascending index order (deterministic).  The argument is formed in FP64 (an FP32
// argument costs 1e-5 relative L2 at N = 1024); terms outside the
// support |u| >= W/2 are exactly zero and skipped.
#include "kernels.cuh"
#include "pptable.cuh"

namespace bsct {

constexpr int GRAM_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(GRAM_THREADS) gram_taps_kernel(int N, double lx, int n, const double *__restrict__ cs,
                                                                 PPView<T> tb, T *__restrict__ taps) {
  const int D = 2 * N - 1;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = idx < (long)D * D;
  const double a = valid ? (double)(idx / D - (N - 1)) : 0.0;  // dk1
  const double b = valid ? (double)(idx % D - (N - 1)) : 0.0;  // dk2
  __shared__ double sc[GRAM_THREADS], ss[GRAM_THREADS], sh[GRAM_THREADS];
  T acc = (T)0;
  for (int a0 = 0; a0 < n; a0 += GRAM_THREADS) {
    const int cnt = min(GRAM_THREADS, n - a0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      sc[threadIdx.x] = lx * cs[2 * (a0 + threadIdx.x)];
      ss[threadIdx.x] = lx * cs[2 * (a0 + threadIdx.x) + 1];
      sh[threadIdx.x] = tb.half[a0 + threadIdx.x];
    }
    __syncthreads();
    if (valid) {
      for (int i = 0; i < cnt; ++i) {
        const double u = fma(-ss[i], a, sc[i] * b);
        if (fabs(u) < sh[i]) acc += pp_eval<T>(tb, a0 + i, u);
      }
    }
  }
  if (valid) {
    const double l2 = lx * lx;
    taps[idx] = (T)(l2 * l2) * acc;
  }
}

template <typename T>
cudaError_t gram_taps(int N, double lx, int n, const double *cs, PPView<T> tb, T *taps, cudaStream_t s) {
  const long D = 2L * N - 1;
  const long total = D * D;
  const int blocks = (int)((total + GRAM_THREADS - 1) / GRAM_THREADS);
  gram_taps_kernel<T><<<blocks, GRAM_THREADS, 0, s>>>(N, lx, n, cs, tb, taps);
  return cudaGetLastError();
}

// Windowed variant: with (dk1, dk2) = r (cos phi, sin phi) the argument is
// u = lx r sin(phi - t), so only angles with |sin(phi - t)| < Hmax / (lx r) contribute.
// Angles are pre-sorted mod pi (theta_s[]); each tap binary-searches its window
// (phi -+ asin(Hmax/(lx r)), wrapping at pi) and sums it in sorted order.  Taps with
// lx r <= Hmax sum every angle.  Exactly the terms the dense loop keeps (it skips
// |u| >= W_t/2 too); only the order of the FP additions differs.
template <typename T>
__global__ void __launch_bounds__(GRAM_THREADS) gram_taps_window_kernel(int N, double lx, int n,
                                                                        const double *__restrict__ theta_s,
                                                                        const double *__restrict__ cs,
                                                                        PPView<T> tb, double Hmax,
                                                                        T *__restrict__ taps) {
  const int D = 2 * N - 1;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)D * D) return;
  const double a = (double)(idx / D - (N - 1));
  const double b = (double)(idx % D - (N - 1));
  const double r = lx * sqrt(a * a + b * b);
  T acc = (T)0;
  auto term = [&](int i) {
    const double u = lx * fma(-cs[2 * i + 1], a, cs[2 * i] * b);
    if (fabs(u) < tb.half[i]) acc += pp_eval<T>(tb, i, u);
  };
  if (r <= Hmax * (1.0 + 1e-9)) {
    for (int i = 0; i < n; ++i) term(i);
  } else {
    const double pi = 3.141592653589793238462643383279502884;
    const double om = asin(fmin(1.0, Hmax / r)) + 1e-9;
    double phi = atan2(b, a);
    phi -= pi * floor(phi / pi);  // [0, pi)
    double lo = phi - om;
    if (lo < 0) lo += pi;
    // first sorted index with theta >= lo
    int l = 0, h = n;
    while (l < h) {
      const int m = (l + h) >> 1;
      if (theta_s[m] < lo) l = m + 1; else h = m;
    }
    const double span = 2.0 * om;
    for (int c = 0, i = l; c < n; ++c, ++i) {
      if (i == n) i = 0;
      double d = theta_s[i] - lo;
      if (d < 0) d += pi;
      if (d > span) break;
      term(i);
    }
  }
  const double l2 = lx * lx;
  taps[idx] = (T)(l2 * l2) * acc;
}

template <typename T>
cudaError_t gram_taps_window(int N, double lx, int n, const double *theta_sorted, const double *cs, PPView<T> tb,
                             double Hmax, T *taps, cudaStream_t s) {
  const long D = 2L * N - 1;
  const int blocks = (int)((D * D + GRAM_THREADS - 1) / GRAM_THREADS);
  gram_taps_window_kernel<T><<<blocks, GRAM_THREADS, 0, s>>>(N, lx, n, theta_sorted, cs, tb, Hmax, taps);
  return cudaGetLastError();
}

template cudaError_t gram_taps_window<float>(int, double, int, const double *, const double *, PPView<float>, double,
                                             float *, cudaStream_t);
template cudaError_t gram_taps_window<double>(int, double, int, const double *, const double *, PPView<double>,
                                              double, double *, cudaStream_t);
template cudaError_t gram_taps<float>(int, double, int, const double *, PPView<float>, float *, cudaStream_t);
template cudaError_t gram_taps<double>(int, double, int, const double *, PPView<double>, double *, cudaStream_t);

}  // namespace bsct
