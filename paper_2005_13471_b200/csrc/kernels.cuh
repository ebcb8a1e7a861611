// kernels.cuh -- host-side launchers of the bsct kernels (internal C++ interface).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "pptable.cuh"

namespace bsct {

// Gram record of one angle (K0 -> K1), GR_WORDS elements of the table type T:
//   [0] C_hi [1] C_lo [2] S_hi [3] S_lo   lambda_x cos t, lambda_x sin t (FP32: hi/lo split, gram.cu;
//                                         FP64: hi = value, lo = 0)
//   [GR_H] H = W/2                        half support
//   [GR_KN .. +16) knots of the right half, knot 0 = 0, +inf beyond the last piece
//   [GR_CO .. +16*GR_NC) local Taylor coefficients of each piece (degree <= 5)
constexpr int GR_H = 4, GR_KN = 8, GR_MAXP = 16, GR_NC = 6, GR_CO = GR_KN + GR_MAXP, GR_WORDS = GR_CO + GR_MAXP * GR_NC;

// Mutable device storage of per-angle tables (tables.cu).
template <typename T>
struct PPTables {
  int *npieces = nullptr;   // [n]
  int *nwidths = nullptr;   // [n]
  int *degree = nullptr;    // [n]   (PP_BP: interpolation degree d)
  double *half = nullptr;   // [n]
  double *knots = nullptr;  // [n][PP_MAXP+1]
  T *coef = nullptr;        // [n][PP_MAXP][PP_NC]
  double *cs = nullptr;     // [n][2]  cos t, sin t
  T *grec = nullptr;        // [n][GR_WORDS] Gram records (PP_GRAM only; not carved, set by the caller)
  PPView<T> view() const { return PPView<T>{npieces, nwidths, half, knots, coef}; }
  static size_t bytes(int n) {
    return (size_t)n * (3 * sizeof(int) + sizeof(double) * (1 + (PP_MAXP + 1) + 2) + sizeof(T) * PP_MAXP * PP_NC) +
           8 * 256;
  }
  // carve from one allocation
  void carve(void *base, int n) {
    char *p = (char *)base;
    auto take = [&](size_t sz) { char *r = p; p += (sz + 255) & ~(size_t)255; return (void *)r; };
    coef = (T *)take(sizeof(T) * (size_t)n * PP_MAXP * PP_NC);
    knots = (double *)take(sizeof(double) * (size_t)n * (PP_MAXP + 1));
    half = (double *)take(sizeof(double) * n);
    cs = (double *)take(sizeof(double) * 2 * n);
    npieces = (int *)take(sizeof(int) * n);
    nwidths = (int *)take(sizeof(int) * n);
    degree = (int *)take(sizeof(int) * n);
  }
};

// K0 (tables.cu)
template <typename T>
cudaError_t build_pp_tables(const double *angles_dev, int n, int kind, double lx, double ly, double zeta,
                            PPTables<T> out, cudaStream_t s);

// K1 (gram.cu): taps[(2N-1)^2] = lx^4 sum_{a < n} M_a(lx <(-s_a, c_a), dk>) from the per-angle
// Gram records (GramRec layout, written by K0 when PPTables::grec is set) of angles sorted by
// t mod pi; bucket[k] (k = 0..nb) = number of sorted angles with (t mod pi) < k pi / nb;
// Hmax >= max_t W_t / 2.  dense: every (tap, angle) pair (measurement mode).  n_dens: angles per pi
// where the set is densest (n for a set spread over [0, pi); sizes the central tile levels).
template <typename T>
cudaError_t gram_build_tiles(int N, double lx, int n, double n_dens, const T *rec, const int *bucket, int nb,
                             double Hmax, bool dense, T *taps, cudaStream_t s);

// K2 (normal.cu): S[q][p] = Re DFT2(E)[p][q] / L^2, work >= (L/2+1)*L complex
template <typename T>
cudaError_t filter_spectrum(int N, int L, const T *taps, T *S, cplx<T> *work, const cplx<T> *tw, cudaStream_t s);

// K5 (normal.cu): the three FFT passes of y = G x.
//   A: x[B][N][N] -> T1[B][L/2+1][N] (row DFTs, column-major)
//   B: T1 -> T1 (column DFT, * S, inverse column DFT, first N rows); gpart[b][blk] +=
//      sum_q w_q S |P~|^2 partials (= <x, G x> by Parseval), may be null
//   C: T1 -> y[B][N][N] (inverse row DFTs, first N columns)
template <typename T>
cudaError_t pass_a(int N, int L, int B, const T *x, cplx<T> *T1, const cplx<T> *tw, cudaStream_t s);
template <typename T>
cudaError_t pass_b(int N, int L, int B, cplx<T> *T1, const T *S, const cplx<T> *tw, double *gpart, cudaStream_t s);
template <typename T>
cudaError_t pass_c(int N, int L, int B, const cplx<T> *T1, T *y, const cplx<T> *tw, cudaStream_t s);
int pass_b_blocks(int L, bool fp32);  // CTAs per slice of pass B (gpart row length)
bool pass_b_warp_enabled();           // FP32 L = 512 / 1024 / 2048 warp-level pass B (BSCT_PASSB_V1=1: off)
bool pass_c_warp_enabled();           // FP32 L = 512 / 1024 / 2048 warp-FFT passes A and C (BSCT_PASSC_V1=1: off)
const float2 *tw1024_table();         // W_1024^{jt} [32][32] on the current device (lazily uploaded)
const float2 *tw2048_table();         // W_2048^{(2m+e)t} [4][32][32] (pass B, L = 2048; lazily uploaded)
bool bulk_stage_enabled();            // pass C T1 staging by bulk (TMA) copies (BSCT_BULK=1)

// K3/K4 (backproject.cu)
template <typename T>
cudaError_t correction_filter(int n_angles, int M, int B, const int *degree, const T *sino, T *gt, cudaStream_t s,
                              T *split = nullptr, int ldt = 0);
template <typename T>
cudaError_t backproject(int N, double lx, double ly, int n_angles, int M, int B, const double *cs, PPView<T> tb,
                        const T *gt, T *b, cudaStream_t s);

// K4 v2: per-angle sub-interval basis (bp_tables) + per-tile piecewise polynomial of
// F_t(u) = sum_m g~[m] C_t(y_m - k_t) in shared memory (backproject.cu).
constexpr int BP_PMAX = 16;   // sub-intervals of the unit detector cell (<= 9 used: 8 subset sums + wrap)
constexpr int BP_SMAX = 12;   // detector samples touching one cell's pixels
struct BPAngle {
  double u0;        // (k_t(pixel 0,0) - y_0) / lambda_y
  double du1, du2;  // d u / d k1, d u / d k2
  double bp[BP_PMAX];  // sub-interval starts in [0,1), bp[0] = 0, unused = +huge
  int P, S, imin, pad;
  unsigned char ilo[BP_PMAX], ihi[BP_PMAX];  // per sub-interval: first / last nonzero basis row
  float bpf[BP_PMAX];                         // bp as FP32 (K4 v4's sub-interval search)
};
// K4 v4 (bp_tc.cu): tensor-core back projection of g~ = gt + gt_lo (TF32 split by K3; row stride ldt,
// a multiple of 4 floats for TMA); bp_tc_supported: every 8 x 16 pixel tile fits the 32-sample window
bool bp_tc_supported(int n, const double *angles, double lx, double ly, double zeta);
size_t bp_tc_smem();
cudaError_t backproject_tc(int N, int n_angles, int M, int B, const BPAngle *ang, const float *Btab, const float *gt,
                           const float *gt_lo, int ldt, float *out, double scale, int maxP, cudaStream_t s);
size_t bp_table_floats(int n);  // size of the basis table B[n][BP_PMAX][BP_SMAX][8]
int bp_v2_max_cells(double lx, double ly, double zeta);  // 0: geometry not supported by v2
int bp_v2_max_p(int n, const double *angles, double lx, double ly, double zeta);  // host, sub-intervals per cell
template <typename T>
cudaError_t build_bp_tables(int N, int M, double lx, double ly, double zeta, int n, const PPTables<T> &tb,
                            BPAngle *ang, T *Btab, cudaStream_t s, int interp = 1);
// gt = pad(w * (g - h)) in K4's [B][n_angles][M + 2 HC] layout (w, h nullable)
template <typename T>
cudaError_t pad_rows(int n_angles, int M, int B, const T *g, const T *h, const T *w, T *gt, cudaStream_t s);
// SIRT helpers (solver.cu): x += C * d (elementwise, C [N*N] broadcast over slices); v -> v > 0 ? 1/v : 0
template <typename T>
cudaError_t sirt_update(long n, int B, const T *C, const T *d, T *x, cudaStream_t s);
template <typename T>
cudaError_t safe_reciprocal(long n, T *v, cudaStream_t s);
// Chebyshev semi-iteration (solver.cu): x = 0, r = b, d = b / theta; x += d, r -= y, d = c1 d + c2 r
template <typename T>
cudaError_t cheb_init(int N, int B, const T *b, T *x, T *r, T *d, double inv_theta, cudaStream_t s);
template <typename T>
cudaError_t cheb_update(int N, int B, double c1, double c2, T *x, T *r, T *d, const T *y, double *rpart,
                        double *resid, int iters, int k, cudaStream_t s);
template <typename T>
cudaError_t backproject_v2(int N, int n_angles, int M, int B, const BPAngle *ang, const T *Btab, const T *gt, T *b,
                           int max_cells, int maxP, double scale, cudaStream_t s);

// K4 v3 (FP32): SB in {1, 2, 4} slices per CTA share each pixel's locate
int bp_v3_slices(int B, int maxP, int max_cells);
// ncoef: 6 (back projection, degree 5) or 3 (plain adjoint, degree <= 2)
cudaError_t backproject_v3(int N, int n_angles, int M, int B, const BPAngle *ang, const float *Btab, const float *gt,
                           float *b, int max_cells, int maxP, double scale, int SB, cudaStream_t s, int ncoef = 6);

// K7 (forward.cu)
// work: [B][N][N] scratch (transposed image); not read by the caller afterwards
template <typename T>
cudaError_t forward_project(int N, double lx, double ly, int n_angles, int M, int B, const double *cs,
                            PPView<T> tb, const T *c, T *sino, cudaStream_t s, T *work);

// K6 (solver.cu)
struct SolverWork {
  double *rho;      // [B][iters+1]  <r_k, r_k>
  double *alpha;    // [B]
  double *gpart;    // [B][gstride] <d, G d> partials from pass B
  int gstride;
  double *rpart;    // [B][rstride] <r, r> partials
  int rstride;
  int *flags;       // [B] or null
  double *resid;    // [B][iters] or null
  double *tau;      // device scalar (Landweber)
};
int vec_blocks(int N);

// fused solver iteration (cg.cu): pass A(CG) / pass C with the vector updates folded in
struct FusedWork {
  double *rho;     // [B][rho_stride]
  int rho_stride;
  double *alpha;   // [B]
  double *gpart;   // [B][gparts] from pass B
  double *rpart;   // [2][B][nparts] <r,r> partials, by iteration parity
  int nparts;      // pass A / pass C CTAs per slice
  int B;
  int *flags;      // [B] or null
  double *resid;   // [B][iters] or null
  int iters;
  double *tau;     // Landweber step (device)
};
int fused_parts(int N, int L, bool fp32);  // pass A / C CTAs per slice
// NEXT-2 (onchip.cu): cluster-resident solver loop for small N (L <= 512); mode 0 CG, 1 SD, 2 Landweber
bool onchip_enabled();                               // opt-in: BSCT_ONCHIP=1
int onchip_cluster_size(int N, int L, bool fp32);    // 0: not supported
template <typename T>
cudaError_t onchip_solve(int N, int L, int B, int iters, int mode, const T *b, T *x, T *r, T *p, const T *S,
                         const cplx<T> *tw, const double *tau, double *resid, int *flags, cudaStream_t s);
// y = G x with the FP32 L = 1024 warp-FFT passes A and C (cudaErrorNotSupported otherwise)
cudaError_t warp_apply_a(int N, int L, int B, const float *x, float2 *T1, cudaStream_t s);
cudaError_t warp_apply_c(int N, int L, int B, const float2 *T1, float *y, cudaStream_t s);
template <typename T>
cudaError_t fused_init(int N, int B, const T *b, T *x, T *r, T *p, FusedWork w, cudaStream_t s);
template <typename T>
cudaError_t fused_pass_a(int N, int L, int B, int k, T *x, const T *r, T *p, cplx<T> *T1, const cplx<T> *tw,
                         FusedWork w, cudaStream_t s);
template <typename T>
cudaError_t fused_pass_c(int N, int L, int B, int k, int mode, int gparts, const cplx<T> *T1, T *x, T *r,
                         const cplx<T> *tw, FusedWork w, cudaStream_t s);
// persistent single-launch CG iterations (FP32, L = 2048, small B; cg.cu)
bool persist_enabled(int L, bool fp32, int B, int solver_cg);
cudaError_t persist_cg_2048(int N, int B, int iters, float *x, float *r, float *p, float2 *T1, const float *S,
                            FusedWork w, int gparts, cudaStream_t s);
template <typename T>
cudaError_t fused_final(int N, int B, int K, int cg, T *x, const T *p, FusedWork w, cudaStream_t s);
// resume from a saved state (x_j, r_j, p_j): r = r_in, p = q = p_in, partials of <r_j, r_j>
template <typename T>
cudaError_t fused_resume(int N, int B, const T *r_in, const T *p_in, T *r, T *p, T *q, FusedWork w, cudaStream_t s);
// export r_K and (p_out != null) p_K = r_K + beta_K p_{K-1}
template <typename T>
cudaError_t fused_export(int N, int B, int K, const T *r, const T *p, T *r_out, T *p_out, FusedWork w,
                         cudaStream_t s);
template <typename T>
cudaError_t solver_init(int N, int B, const T *b, T *x, T *r, T *p, SolverWork w, int iters, cudaStream_t s);
template <typename T>
cudaError_t solver_update(int N, int B, int solver, int it, int iters, T *x, T *r, T *p, const T *q, SolverWork w,
                          cudaStream_t s);
template <typename T>
cudaError_t solver_finish(int N, int B, int solver, int it, int iters, const T *r, T *p, SolverWork w, cudaStream_t s);
template <typename T>
cudaError_t spectrum_max(int L, const T *S, double *out, cudaStream_t s);

}  // namespace bsct
