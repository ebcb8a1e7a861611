// tables.cu -- K0: per-angle box-spline tables, built on the device in FP64.
//
// For each angle the univariate box spline M_W (Eq.(1); projected widths of
// Eq.(2), P:61 / P:80 / P:107 / P:128) is written as a piecewise polynomial on the
// right half [0, W/2] of its support (M_W is even).  Knots are the distinct subset
// sums of W minus W/2; on piece j starting at rho_j the local Taylor coefficients are
//   a_k = [(n-1)! prod W]^-1 C(n-1, k) sum_{S active} (-1)^|S| (rho_j + W/2 - sum S)^(n-1-k)
// (binomial expansion of the truncated powers active on the piece).  Evaluating
// these in local coordinates (pptable.cuh) avoids the catastrophic cancellation of the
// global truncated-power sum in FP32 ("FP32 box-spline evaluation").
#include "kernels.cuh"
#include "pptable.cuh"

namespace bsct {

__device__ __forceinline__ double ipow(double x, int e) {
  double r = 1.0;
  for (int i = 0; i < e; ++i) r *= x;
  return r;
}

template <typename T>
__global__ void __launch_bounds__(64) build_pp_tables_kernel(const double *__restrict__ angles, int n, int kind,
                                                             double lx, double ly, double zeta, PPTables<T> out) {
  const int a = blockIdx.x;
  const int tid = threadIdx.x;
  __shared__ double w[8];
  __shared__ int nw;
  __shared__ double sig[64];
  __shared__ int sgn[64];
  __shared__ double sorted[64];
  __shared__ double kn[PP_MAXP + 1];
  __shared__ int K;
  if (a >= n) return;
  if (tid == 0) {
    double s, c;
    sincos(angles[a], &s, &c);
    out.cs[2 * a] = c;
    out.cs[2 * a + 1] = s;
    const double ac = lx * fabs(c), as = lx * fabs(s);
    double raw[8];
    int nr = 0;
    if (kind == PP_GRAM) {
      raw[nr++] = ac; raw[nr++] = ac; raw[nr++] = as; raw[nr++] = as;
      if (zeta > 0) { raw[nr++] = zeta; raw[nr++] = zeta; }
    } else {
      raw[nr++] = ac; raw[nr++] = as;
      if (zeta > 0) raw[nr++] = zeta;
      if (kind == PP_BP) {
        // interpolation degree d = #nonzero{l|c|, l|s|, zeta} - 1 (R9)
        double s3 = 0;
        for (int i = 0; i < nr; ++i) s3 += raw[i];
        const double thr3 = 1e-12 * fmax(1.0, s3);
        int nz = 0;
        for (int i = 0; i < nr; ++i) nz += raw[i] > thr3;
        const int d = nz - 1;
        out.degree[a] = d;
        for (int i = 0; i <= d; ++i) raw[nr++] = ly;
      }
    }
    double ssum = 0;
    for (int i = 0; i < nr; ++i) ssum += raw[i];
    const double thr = 1e-12 * fmax(1.0, ssum);  // drop degenerate widths (R9)
    int k = 0;
    for (int i = 0; i < nr; ++i)
      if (raw[i] > thr) w[k++] = raw[i];
    nw = k;
    out.nwidths[a] = k;
  }
  __syncthreads();
  const int n_w = nw;
  const int ns = 1 << n_w;
  if (tid < ns) {
    double sm = 0;
    int pc = 0;
    for (int i = 0; i < n_w; ++i)
      if ((tid >> i) & 1) { sm += w[i]; ++pc; }
    sig[tid] = sm;
    sgn[tid] = (pc & 1) ? -1 : 1;
  }
  __syncthreads();
  if (tid < ns) {
    int r = 0;
    const double me = sig[tid];
    for (int j = 0; j < ns; ++j) r += (sig[j] < me) || (sig[j] == me && j < tid);
    sorted[r] = me;
  }
  __syncthreads();
  double W = 0;
  for (int i = 0; i < n_w; ++i) W += w[i];
  const double H = 0.5 * W;
  const double tol = 1e-12 * fmax(1.0, W);
  if (tid == 0) {
    int KK = 0;
    kn[0] = 0.0;
    for (int i = 0; i < ns; ++i) {
      const double x = sorted[i] - H;
      if (x > kn[KK] + tol && KK < PP_MAXP) kn[++KK] = x;
    }
    kn[KK] = H;  // the full-set sum closes the support
    K = KK;
    out.npieces[a] = KK;
    out.half[a] = H;
  }
  __syncthreads();
  for (int i = tid; i <= PP_MAXP; i += blockDim.x) out.knots[(size_t)a * (PP_MAXP + 1) + i] = i <= K ? kn[i] : H;
  double prodw = 1.0;
  for (int i = 0; i < n_w; ++i) prodw *= w[i];
  double fact = 1.0;
  for (int i = 2; i < n_w; ++i) fact *= i;
  const double norm = 1.0 / (fact * prodw);
  const int deg = n_w - 1;
  for (int j = tid; j < PP_MAXP; j += blockDim.x) {
    T *cj = out.coef + ((size_t)a * PP_MAXP + j) * PP_NC;
    if (j >= K) {
      for (int k = 0; k < PP_NC; ++k) cj[k] = (T)0;
      continue;
    }
    if (n_w == 1) {  // plain box: constant 1/w (evaluated half-open in pptable.cuh)
      cj[0] = (T)(1.0 / w[0]);
      for (int k = 1; k < PP_NC; ++k) cj[k] = (T)0;
      continue;
    }
    const double u0 = kn[j] + H;
    double acc[PP_MAXW] = {0, 0, 0, 0, 0, 0};
    for (int S = 0; S < ns; ++S) {
      if (sig[S] > u0 + tol) continue;  // inactive on this piece
      const double dl = fmax(0.0, u0 - sig[S]);
      for (int k = 0; k <= deg; ++k) acc[k] += sgn[S] * ipow(dl, deg - k);
    }
    double binom = 1.0;  // C(deg, k)
    for (int k = 0; k < PP_NC; ++k) {
      if (k <= deg) {
        cj[k] = (T)(norm * binom * acc[k]);
        binom = binom * (deg - k) / (k + 1);
      } else {
        cj[k] = (T)0;
      }
    }
  }
}

template <typename T>
cudaError_t build_pp_tables(const double *angles_dev, int n, int kind, double lx, double ly, double zeta,
                            PPTables<T> out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  build_pp_tables_kernel<T><<<n, 64, 0, s>>>(angles_dev, n, kind, lx, ly, zeta, out);
  return cudaGetLastError();
}

template cudaError_t build_pp_tables<float>(const double *, int, int, double, double, double, PPTables<float>,
                                            cudaStream_t);
template cudaError_t build_pp_tables<double>(const double *, int, int, double, double, double, PPTables<double>,
                                             cudaStream_t);

}  // namespace bsct
