// forward.cu -- K7 forward projection g = H c (Eq.(3), Eq.(4)).
//
//   g[t][m] = lambda_x^2 sum_k c_k M_[l|c|, l|s|, zeta](y_m - k_t)
//
// Ray driven (one thread per detector sample, deterministic, no atomics): the pixels
// whose footprint covers y_m lie in a strip; iterate over the axis along which the
// ray advances fastest and, per line of pixels, over the <= 2H/max(|c|,|s|) + 1
// pixels inside the support.  A support op of the hot path (data synthesis, the
// paper's exactness property); NEXT-1 in SURVEY.md 8(f).
#include <cstdlib>

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

// K7 v2.  Same sums as forward_kernel, same order (ascending line, then ascending pixel
// within the strip), but: one CTA per (angle, slice) with the angle's right-half table
// (<= FWD_MAXP pieces of degree <= 2: the box spline of <= 3 widths) in shared memory;
// FP64 only once per line of pixels (the strip bounds and the argument at its first
// pixel); along the strip the argument steps by the per-pixel advance in T (<= ~8 steps
// from an FP64 anchor, so the argument error stays ~1e-6 of a detector cell); piece
// selection by register compares; no binary search in global memory.
constexpr int FWD_MAXP = 8;

template <typename T>
__global__ void __launch_bounds__(256) forward_v2_kernel(int N, double lx, double ly, int n_angles, int M,
                                                         const double *__restrict__ cs, PPView<T> tb,
                                                         const T *__restrict__ c, T *__restrict__ sino) {
  const int a = blockIdx.x, b = blockIdx.y;
  __shared__ T kn_s[FWD_MAXP + 1], cf_s[FWD_MAXP][3];
  __shared__ int np_s, nw_s;
  const int np = tb.npieces[a];
  if (threadIdx.x <= FWD_MAXP) kn_s[threadIdx.x] = threadIdx.x <= np ? (T)tb.knots[(size_t)a * (PP_MAXP + 1) + threadIdx.x] : (T)3e38;
  if (threadIdx.x < FWD_MAXP * 3) {
    const int j = threadIdx.x / 3, k = threadIdx.x % 3;
    cf_s[j][k] = j < np ? tb.coef[((size_t)a * PP_MAXP + j) * PP_NC + k] : (T)0;
  }
  if (threadIdx.x == 0) { np_s = np; nw_s = tb.nwidths[a]; }
  __syncthreads();
  const double co = cs[2 * a], si = cs[2 * a + 1];
  const double H = tb.half[a];
  const T Ht = (T)H;
  const int nw = nw_s;
  T kn[FWD_MAXP];
#pragma unroll
  for (int j = 1; j < FWD_MAXP; ++j) kn[j] = kn_s[j];
  auto eval = [&](T x) -> T {  // M(x), x within ~1e-6 of the exact argument
    if (nw == 1) return (x >= -Ht && x < Ht) ? (T)(0.5 / H) : (T)0;  // half-open box (R6)
    const T ax = x < 0 ? -x : x;
    if (!(ax < Ht)) return (T)0;
    int j = 0;
#pragma unroll
    for (int q = 1; q < FWD_MAXP; ++q) j += (ax >= kn[q]) ? 1 : 0;
    const T t = ax - kn_s[j];
    return fma(fma(cf_s[j][2], t, cf_s[j][1]), t, cf_s[j][0]);
  };
  const T *img = c + (size_t)b * N * N;
  const int h = N / 2;
  const bool rows = fabs(co) >= fabs(si);
  // lines: rows k1 (pixels k2 along the row) or columns k2 (pixels k1 along the column);
  // arg(line, j) = A(line) - st * j with A(line) = y - kt(line, 0), st = d kt / d j
  const double st = rows ? co * lx : -si * lx;
  const double inv = 1.0 / st;
  const T stT = (T)st;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const double y = ly * (double)(m - M / 2);
    T acc = 0;
    for (int l = 0; l < N; ++l) {
      const double xl = lx * (double)(l - h);
      // kt(l, j) = rows ? (-si xl + co lx (j - h)) : (-si lx (j - h) + co xl)
      const double A = rows ? y + si * xl + co * lx * h : y - co * xl - si * lx * h;
      // |A - st j| < H  <=>  j in ((A - H)/st, (A + H)/st) (interval ends swap for st < 0)
      const double e0 = (A - H) * inv, e1 = (A + H) * inv;
      int j0 = (int)floor(fmin(e0, e1)), j1 = (int)ceil(fmax(e0, e1));
      j0 = max(0, j0);
      j1 = min(N - 1, j1);
      if (j0 > j1) continue;
      T arg = (T)(A - st * (double)j0);
      const T *line = rows ? img + (size_t)l * N : img + l;
      const size_t step = rows ? 1 : (size_t)N;
      for (int j = j0; j <= j1; ++j, arg -= stT) {
        const T v = eval(arg);
        if (v != (T)0) acc = fma(line[(size_t)j * step], v, acc);
      }
    }
    sino[((size_t)b * n_angles + a) * M + m] = (T)(lx * lx) * acc;
  }
}

template <typename T>
cudaError_t forward_project(int N, double lx, double ly, int n_angles, int M, int B, const double *cs,
                            PPView<T> tb, const T *c, T *sino, cudaStream_t s) {
  const char *v1 = getenv("BSCT_FWD_V1");
  if (v1 && v1[0] == '1') {
    dim3 grid((M + 255) / 256, n_angles, B);
    forward_kernel<T><<<grid, 256, 0, s>>>(N, lx, ly, n_angles, M, cs, tb, c, sino);
  } else {
    forward_v2_kernel<T><<<dim3(n_angles, B), 256, 0, s>>>(N, lx, ly, n_angles, M, cs, tb, c, sino);
  }
  return cudaGetLastError();
}

template cudaError_t forward_project<float>(int, double, double, int, int, int, const double *, PPView<float>,
                                            const float *, float *, cudaStream_t);
template cudaError_t forward_project<double>(int, double, double, int, int, int, const double *, PPView<double>,
                                             const double *, double *, cudaStream_t);

}  // namespace bsct
