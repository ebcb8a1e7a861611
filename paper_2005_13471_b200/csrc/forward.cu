// forward.cu -- K7 forward projection g = H c (Eq.(3), Eq.(4)).
//
//   g[t][m] = lambda_x^2 sum_k c_k M_[l|c|, l|s|, zeta](y_m - k_t)
//
// Ray driven (one thread per detector sample, deterministic, no atomics): the pixels
// whose footprint covers y_m lie in a strip; iterate over the axis along which the
// ray advances fastest and, per line of pixels, over the <= 2H/max(|c|,|s|) + 1
// pixels inside the support.  A support op of the hot path (data synthesis, the
// paper's exactness property); NEXT-1 in SURVEY.md 8(f).
#include "kernels.cuh"
#include "pptable.cuh"

namespace bsct {

template <typename T>
__global__ void __launch_bounds__(256) forward_kernel(int N, double lx, double ly, int n_angles, int M,
                                                      const double *__restrict__ cs, PPView<T> tb,
                                                      const T *__restrict__ c, T *__restrict__ sino) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = blockIdx.y;
  const int b = blockIdx.z;
  if (m >= M) return;
  const double co = cs[2 * a], si = cs[2 * a + 1];
  const double H = tb.half[a];
  const double y = ly * (double)(m - M / 2);
  const T *img = c + (size_t)b * N * N;
  const int h = N / 2;
  T acc = 0;
  // k_t = -si * x1 + co * x2, x = lx (k - h)
  if (fabs(co) >= fabs(si)) {
    for (int k1 = 0; k1 < N; ++k1) {
      const double x1 = lx * (double)(k1 - h);
      // co * x2 in (y + si*x1 - H, y + si*x1 + H)
      const double lo = (y + si * x1 - H) / co, hi = (y + si * x1 + H) / co;
      const double xa = fmin(lo, hi), xb = fmax(lo, hi);
      int k2lo = max(0, (int)floor(xa / lx) + h);
      int k2hi = min(N - 1, (int)ceil(xb / lx) + h);
      for (int k2 = k2lo; k2 <= k2hi; ++k2) {
        const double kt = fma(-si, x1, co * lx * (double)(k2 - h));
        const T v = pp_eval<T>(tb, a, y - kt);
        if (v != (T)0) acc = fma(img[(size_t)k1 * N + k2], v, acc);
      }
    }
  } else {
    for (int k2 = 0; k2 < N; ++k2) {
      const double x2 = lx * (double)(k2 - h);
      // -si * x1 in (y - co*x2 - H, y - co*x2 + H)
      const double lo = (co * x2 - y - H) / si, hi = (co * x2 - y + H) / si;
      const double xa = fmin(lo, hi), xb = fmax(lo, hi);
      int k1lo = max(0, (int)floor(xa / lx) + h);
      int k1hi = min(N - 1, (int)ceil(xb / lx) + h);
      for (int k1 = k1lo; k1 <= k1hi; ++k1) {
        const double kt = fma(-si, lx * (double)(k1 - h), co * x2);
        const T v = pp_eval<T>(tb, a, y - kt);
        if (v != (T)0) acc = fma(img[(size_t)k1 * N + k2], v, acc);
      }
    }
  }
  sino[((size_t)b * n_angles + a) * M + m] = (T)(lx * lx) * acc;
}

template <typename T>
cudaError_t forward_project(int N, double lx, double ly, int n_angles, int M, int B, const double *cs,
                            PPView<T> tb, const T *c, T *sino, cudaStream_t s) {
  dim3 grid((M + 255) / 256, n_angles, B);
  forward_kernel<T><<<grid, 256, 0, s>>>(N, lx, ly, n_angles, M, cs, tb, c, sino);
  return cudaGetLastError();
}

template cudaError_t forward_project<float>(int, double, double, int, int, int, const double *, PPView<float>,
                                            const float *, float *, cudaStream_t);
template cudaError_t forward_project<double>(int, double, double, int, int, int, const double *, PPView<double>,
                                             const double *, double *, cudaStream_t);

}  // namespace bsct
