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


template <typename T>
__global__ void __launch_bounds__(128) build_pp_tables_kernel(const double *__restrict__ angles, int n, int kind,
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
  __shared__ double csh[2];
  __shared__ unsigned kmask[2];
  // let a programmatic dependent (K1 of gram_build) launch now: its prologue does not read the tables
  asm volatile("griddepcontrol.launch_dependents;");
  if (a >= n) return;
  if (tid == 0) {
    double s, c;
    sincos(angles[a], &s, &c);
    out.cs[2 * a] = c;
    out.cs[2 * a + 1] = s;
    csh[0] = c;
    csh[1] = s;
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
  // Knots of the right half: the sorted subset sums minus H, a new knot wherever a value exceeds
  // its predecessor (or 0) by more than tol (clusters of equal sums within tol merge into their
  // first member); each flagged value's knot index is the prefix count of the flags.
  {
    const int lane = tid & 31, wp = tid >> 5;
    bool flag = false;
    double x = 0.0;
    if (tid < ns) {
      x = sorted[tid] - H;
      const double prev = tid > 0 ? fmax(sorted[tid - 1] - H, 0.0) : 0.0;
      flag = x > prev + tol;
    }
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    if (lane == 0 && wp < 2) kmask[wp] = m;
    __syncthreads();
    if (flag) {
      const int idx = 1 + __popc(m & ((1u << lane) - 1u)) + (wp == 1 ? __popc(kmask[0]) : 0);
      if (idx <= PP_MAXP) kn[idx] = x;
    }
    if (tid == 0) {
      int KK = __popc(kmask[0]) + __popc(kmask[1]);
      KK = KK < PP_MAXP ? KK : PP_MAXP;
      kn[0] = 0.0;
      K = KK;
    }
    __syncthreads();
    if (tid == 0) {
      kn[K] = H;  // the full-set sum closes the support
      out.npieces[a] = K;
      out.half[a] = H;
    }
    __syncthreads();
  }
  for (int i = tid; i <= PP_MAXP; i += blockDim.x) out.knots[(size_t)a * (PP_MAXP + 1) + i] = i <= K ? kn[i] : H;
  T *rg = (kind == PP_GRAM && out.grec) ? out.grec + (size_t)a * GR_WORDS : nullptr;
  if (rg && tid < GR_MAXP) rg[GR_KN + tid] = tid <= K ? (T)kn[tid] : (T)INFINITY;
  if (rg && tid == 0) {  // argument coefficients (gram.cu header: hi/lo split for FP32) and H
    const double C = lx * csh[0], S = lx * csh[1];
    if (sizeof(T) == 4) {
      int e;
      frexp(lx, &e);                         // lx <= 2^e
      const double q0 = ldexp(1.0, e - 11);  // |hi| / q0 <= 2^11
      const double ch = rint(C / q0) * q0, sh = rint(S / q0) * q0;
      rg[0] = (T)ch;
      rg[1] = (T)(C - ch);
      rg[2] = (T)sh;
      rg[3] = (T)(S - sh);
    } else {
      rg[0] = (T)C;
      rg[1] = (T)0;
      rg[2] = (T)S;
      rg[3] = (T)0;
    }
    rg[GR_H] = (T)H;
    rg[5] = rg[6] = rg[7] = (T)0;
  }
  double prodw = 1.0;
  for (int i = 0; i < n_w; ++i) prodw *= w[i];
  double fact = 1.0;
  for (int i = 2; i < n_w; ++i) fact *= i;
  const double norm = 1.0 / (fact * prodw);
  const int deg = n_w - 1;
  // Local Taylor coefficients: 4 threads per piece, each summing every 4th subset; the four
  // partial sums are combined by a fixed xor-shuffle tree.
  const int part = tid & 3;
  for (int jb = 0; jb < PP_MAXP; jb += (int)blockDim.x / 4) {
    const int j = jb + tid / 4;
    // ae[e] = sum over active subsets of sgn dl^e (powers as left-to-right products 1 * dl * dl ...)
    double ae[PP_MAXW] = {0, 0, 0, 0, 0, 0};
    if (j < K && n_w > 1) {
      const double u0 = kn[j] + H;
      for (int S = part; S < ns; S += 4) {
        if (sig[S] > u0 + tol) continue;  // inactive on this piece
        const double dl = fmax(0.0, u0 - sig[S]);
        const double sg = (double)sgn[S];
        double pw = 1.0;
#pragma unroll
        for (int e = 0; e < PP_MAXW; ++e) {
          ae[e] += sg * pw;
          pw *= dl;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < PP_MAXW; ++e) {
      ae[e] += __shfl_xor_sync(0xffffffffu, ae[e], 1);
      ae[e] += __shfl_xor_sync(0xffffffffu, ae[e], 2);
    }
    if (part != 0 || j >= PP_MAXP) continue;
    T *cj = out.coef + ((size_t)a * PP_MAXP + j) * PP_NC;
    T *gj = (rg && j < GR_MAXP) ? rg + GR_CO + j * GR_NC : nullptr;
    if (j >= K) {
      for (int k = 0; k < PP_NC; ++k) cj[k] = (T)0;
      if (gj)
        for (int k = 0; k < GR_NC; ++k) gj[k] = (T)0;
      continue;
    }
    if (n_w == 1) {  // plain box: constant 1/w (evaluated half-open in pptable.cuh)
      cj[0] = (T)(1.0 / w[0]);
      for (int k = 1; k < PP_NC; ++k) cj[k] = (T)0;
      continue;
    }
    // coefficient of t^k, k = deg - e: norm C(deg, k) ae[e] with C(deg, k) = C(deg, e) (exact integer
    // recursion over e, compile-time divisors after unrolling); ae stays in registers
    int binom = 1;
#pragma unroll
    for (int e = 0; e < PP_MAXW; ++e) {
      if (e <= deg) {
        const int k = deg - e;
        const T v = (T)(norm * (double)binom * ae[e]);
        cj[k] = v;
        if (gj && k < GR_NC) gj[k] = v;
        binom = binom * (deg - e) / (e + 1);
      }
    }
    for (int k = deg + 1; k < PP_NC; ++k) {
      cj[k] = (T)0;
      if (gj && k < GR_NC) gj[k] = (T)0;
    }
  }
}

template <typename T>
cudaError_t build_pp_tables(const double *angles_dev, int n, int kind, double lx, double ly, double zeta,
                            PPTables<T> out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  build_pp_tables_kernel<T><<<n, 128, 0, s>>>(angles_dev, n, kind, lx, ly, zeta, out);
  return cudaGetLastError();
}

template cudaError_t build_pp_tables<float>(const double *, int, int, double, double, double, PPTables<float>,
                                            cudaStream_t);
template cudaError_t build_pp_tables<double>(const double *, int, int, double, double, double, PPTables<double>,
                                             cudaStream_t);

}  // namespace bsct
