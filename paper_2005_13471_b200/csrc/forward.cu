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

// K7 v3.  Same sums as forward_kernel, same order (ascending line, then ascending pixel
// within the strip).  One CTA per (angle, slice) with the angle's right-half table (<= FWD_MAXP
// pieces of degree <= 2: the box spline of <= 3 widths) in shared memory.  Lines are image rows
// when |cos t| >= |sin t| and rows of the transposed image otherwise, so the lanes of a warp
// (consecutive detector samples) always read neighbouring pixels of one row.  Per line the strip
// bounds advance by a constant in FP64 and are rounded with the 1.5 * 2^52 trick (no conversion
// instructions); the argument at the strip's first pixel, H + st (e - j0) with e - j0 exact, is
// the one FP64 -> T conversion; along the strip the argument steps by st in T (<= ~8 steps).
constexpr int FWD_MAXP = 8;
constexpr double FWD_MAGIC = 6755399441055744.0;  // 1.5 * 2^52

template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(int N, const T *__restrict__ c, T *__restrict__ ct) {
  __shared__ T t[32][33];
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const T *src = c + (size_t)b * N * N;
  T *dst = ct + (size_t)b * N * N;
  for (int r = threadIdx.y; r < 32; r += 8)
    if (y0 + r < N && x0 + threadIdx.x < N) t[r][threadIdx.x] = src[(size_t)(y0 + r) * N + x0 + threadIdx.x];
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8)
    if (x0 + r < N && y0 + threadIdx.x < N) dst[(size_t)(x0 + r) * N + y0 + threadIdx.x] = t[threadIdx.x][r];
}

// SB slices per CTA: the weight M(arg) of a (sample, pixel) pair is the same for every slice,
// so each evaluation serves SB pixel loads and FMAs.
template <typename T, int PC, int SB>
__global__ void __launch_bounds__(256) forward_v3_kernel(int N, int B, double lx, double ly, int n_angles, int M,
                                                         const double *__restrict__ cs, PPView<T> tb,
                                                         const T *__restrict__ c, const T *__restrict__ ct,
                                                         T *__restrict__ sino) {
  const int a = blockIdx.x, b0 = blockIdx.y * SB;
  const int nb = min(SB, B - b0);
  __shared__ T kn_s[FWD_MAXP + 1], cf_s[FWD_MAXP][3];
  __shared__ int nw_s;
  const int np = tb.npieces[a];
  if (threadIdx.x <= FWD_MAXP) kn_s[threadIdx.x] = threadIdx.x <= np ? (T)tb.knots[(size_t)a * (PP_MAXP + 1) + threadIdx.x] : (T)3e38;
  if (threadIdx.x < FWD_MAXP * 3) {
    const int j = threadIdx.x / 3, k = threadIdx.x % 3;
    cf_s[j][k] = j < np ? tb.coef[((size_t)a * PP_MAXP + j) * PP_NC + k] : (T)0;
  }
  if (threadIdx.x == 0) nw_s = tb.nwidths[a];
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
  const bool rows = fabs(co) >= fabs(si);
  const T *img = (rows ? c : ct) + (size_t)b0 * N * N;  // line l = row l of img, pixels j along it
  const size_t NN = (size_t)N * N;
  const int h = N / 2;
  // arg(l, j) = A(l) - st j;  A(l) = A0 + l dA  (rows: kt = -si x1 + co x2 with x1 = lx (l - h),
  // x2 = lx (j - h); columns: x2 = lx (l - h), x1 = lx (j - h))
  const double st = rows ? co * lx : -si * lx;
  const double dA = rows ? si * lx : -co * lx;
  const double A0c = rows ? -si * lx * h + co * lx * h : co * lx * h - si * lx * h;  // A0 = y + A0c
  const double inv = 1.0 / st;
  const double sH = st > 0 ? H : -H;  // e_lo = (A - sH)/st is the lower strip end
  const T stT = (T)st;
  const T box = (T)(0.5 / H);  // one width: M = 1/w on [-w/2, w/2) (R6)
  const double de = dA * inv;
  // pixels per line in the strip: j in (e_lo, e_lo + 2H/|st|) -> at most KS = floor(2H/|st|) + 2
  // candidates from j0 = floor(e_lo) (uniform across the CTA: no divergent inner loops)
  const int KS = (int)(2.0 * H / fabs(st)) + 2;
  // the strip is non-empty in line l iff e_lo(l) < N and e_lo(l) + 2H/|st| > -1: a contiguous
  // range of l (e_lo is linear in l), computed per sample
  const double w = 2.0 * H * fabs(inv);
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    const double y = ly * (double)(m - M / 2);
    const double e00 = (y + A0c - sH) * inv;  // e_lo at l = 0
    int l0 = 0, l1 = N - 1;
    if (de != 0.0) {
      // e_lo(l) = e00 + l de; need -1 - w < e_lo(l) < N
      double la = (-1.0 - w - e00) / de, lb = ((double)N - e00) / de;
      if (la > lb) { const double tt = la; la = lb; lb = tt; }
      l0 = max(0, (int)floor(la));
      l1 = min(N - 1, (int)ceil(lb));
    } else if (!(e00 < N && e00 + w > -1.0)) {
      l1 = -1;
    }
    T acc[SB];
#pragma unroll
    for (int sl = 0; sl < SB; ++sl) acc[sl] = 0;
    double elo = e00 + (double)l0 * de;
    for (int l = l0; l <= l1; ++l, elo += de) {
      const double t0 = (elo - 0.5) + FWD_MAGIC;
      const int j0 = __double2loint(t0);             // ~floor(e_lo)
      const double f0 = elo - (t0 - FWD_MAGIC);      // e_lo - j0, exact
      T arg = (T)(sH + st * f0);                      // arg at j = j0
      const T *line = img + (size_t)l * N;
      for (int k = 0; k < KS; ++k, arg -= stT) {
        const int j = j0 + k;
        // branch-free M(arg): piece by compares, zero outside [-H, H) and outside the image
        const T ax = fabs(arg);
        int q = 0;
#pragma unroll
        for (int qq = 1; qq <= PC; ++qq) q += (ax >= kn[qq]) ? 1 : 0;
        const T tq = ax - kn_s[q];
        const T v = nw == 1 ? box : fma(fma(cf_s[q][2], tq, cf_s[q][1]), tq, cf_s[q][0]);
        const bool sup = nw == 1 ? (arg >= -Ht && arg < Ht) : (ax < Ht);
        const bool in = sup && (unsigned)j < (unsigned)N;
        if (in)
#pragma unroll
          for (int sl = 0; sl < SB; ++sl)
            if (sl < nb) acc[sl] = fma(line[sl * NN + j], v, acc[sl]);
      }
    }
#pragma unroll
    for (int sl = 0; sl < SB; ++sl)
      if (sl < nb) sino[((size_t)(b0 + sl) * n_angles + a) * M + m] = (T)(lx * lx) * acc[sl];
  }
}

template <typename T>
cudaError_t forward_project(int N, double lx, double ly, int n_angles, int M, int B, const double *cs,
                            PPView<T> tb, const T *c, T *sino, cudaStream_t s, T *work) {
  const char *v1 = getenv("BSCT_FWD_V1");
  if (v1 && v1[0] == '1') {
    dim3 grid((M + 255) / 256, n_angles, B);
    forward_kernel<T><<<grid, 256, 0, s>>>(N, lx, ly, n_angles, M, cs, tb, c, sino);
  } else {
    if (!work) return cudaErrorInvalidValue;  // [B][N][N] scratch for the transposed image
    transpose_kernel<T><<<dim3((N + 31) / 32, (N + 31) / 32, B), dim3(32, 8), 0, s>>>(N, c, work);
    // the forward model's box spline has <= 3 widths: <= 5 right-half pieces, 4 knot compares
    constexpr int FSB = 8;  // slices per CTA (measured: 4 -> 339, 8 -> 356 Gvox-angle/s at config 5)
    forward_v3_kernel<T, 4, FSB><<<dim3(n_angles, (B + FSB - 1) / FSB), 256, 0, s>>>(N, B, lx, ly, n_angles, M, cs,
                                                                                  tb, c, work, sino);
  }
  return cudaGetLastError();
}

template cudaError_t forward_project<float>(int, double, double, int, int, int, const double *, PPView<float>,
                                            const float *, float *, cudaStream_t, float *);
template cudaError_t forward_project<double>(int, double, double, int, int, int, const double *, PPView<double>,
                                             const double *, double *, cudaStream_t, double *);

}  // namespace bsct
