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

template cudaError_t gram_taps<float>(int, double, int, const double *, PPView<float>, float *, cudaStream_t);
template cudaError_t gram_taps<double>(int, double, int, const double *, PPView<double>, double *, cudaStream_t);

}  // namespace bsct
