/*
 * bsct.h -- C ABI of the B200-native box-spline parallel-beam CT hot path
 *           (arXiv 2005.13471, "PAPER.md"; citations P:<line>).
 *
 * The library computes, on an NVIDIA B200 (sm_100a), the three parts of the
 * paper's iterative reconstruction ("a single back projection ... at the
 * beginning and apply the filter in every iteration"):
 *   (a) the exact (2N-1)x(2N-1) Gram filter              bsct_gram_build
 *   (b) the interpolated back projection b = H^T g^      bsct_backproject
 *   (c) the normal operator y = G x as a zero-padded
 *       L x L FFT convolution, and the solver loop        bsct_normal_apply / bsct_cg_solve
 *
 *
 * Conventions:
 *  - Image c[k1][k2], row-major, N x N; pixel centre x_k = lambda_x (k - floor(N/2))
 *    per axis; k1 is the first coordinate (reading R5).
 *  - Projection angle t: ray direction (cos t, sin t), detector axis
 *    (-sin t, cos t) (R4); sinogram g[angle][m], detector sample
 *    y_m = lambda_y (m - floor(n_det/2)) ("delta(y - lambda_y m)", R5).
 *  - Forward model H = (1/zeta) box(./zeta) * P_t, unit-integral box
 *    splines throughout (R1), continuous detector coordinate (R2).
 *  - Gram taps G[dk1 + N-1][dk2 + N-1], dk = k_i - k_j.
 *  - FFT size L = smallest power of two >= max(2, 2N-1) (bsct_fft_size).
 *  - Every data pointer is caller-owned DEVICE memory unless marked HOST;
 *    element type = the plan's dtype (float for BSCT_F32, double for BSCT_F64).
 *  - Every call is ordered on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and returns without synchronising, except bsct_plan_create
 *    (small table upload) and bsct_reconstruct_host (host buffers).
 *  - Errors: a negative bsct_status; bsct_last_error() returns a thread-local
 *    message.  Inputs are validated before any work is enqueued, so an error
 *    return leaves outputs untouched (BSCT_ECUDA excepted).
 *  - Limits: 1 <= N <= 2048 (L <= 4096), 1 <= n_angles <= 65536,
 *    1 <= n_det <= 1<<20, lambda_x, lambda_y > 0, zeta >= 0, finite angles.
 */
#ifndef BSCT_H
#define BSCT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *bsct_stream; /* == cudaStream_t */

typedef enum {
  BSCT_OK = 0,
  BSCT_EINVAL = -1,     /* invalid geometry / argument (N<1, lambda<=0, zeta<0, bad angle range...) */
  BSCT_ECUDA = -2,      /* a CUDA runtime error (message in bsct_last_error)                    */
  BSCT_ENOMEM = -3,     /* device allocation failed                                             */
  BSCT_EBREAKDOWN = -4, /* solver breakdown <p,Gp> <= 0 (reported per slice through flags)      */
  BSCT_ESHAPE = -5      /* batch larger than the plan's max_batch, or dtype mismatch            */
} bsct_status;

typedef enum { BSCT_F32 = 0, BSCT_F64 = 1 } bsct_dtype;

typedef enum { BSCT_CG = 0, BSCT_SD = 1, BSCT_LANDWEBER = 2 } bsct_solver;

/* The paper's problem statement. */
typedef struct {
  int32_t N;             /* image is N x N coefficients c_k                          */
  double lambda_x;       /* isotropic pixel step, Lambda_x = lambda_x I */
  int32_t n_angles;      /* number of projection angles                             */
  const double *angles;  /* HOST [n_angles], radians; summed in the order given      */
  double lambda_y;       /* detector sampling step                            */
  int32_t n_det;         /* detector samples M per angle                             */
  double zeta_blur;      /* detector cell width; 0 disables the blur          */
} bsct_geometry;

typedef struct bsct_plan_s *bsct_plan;

/* Library version (major*10000 + minor*100 + patch). */
int32_t bsct_version(void);

/* Thread-local message of the last failing call ("" if none). */
const char *bsct_last_error(void);

/* FFT size L used by the normal operator for an N x N image (>= 2N-1, power of 2). */
int32_t bsct_fft_size(int32_t N);

/*
 * (a) Gram filter, P:96-100 (no blur) and P:122-129 (blur):
 *     G[dk] = lambda_x^4 sum_{angles a in [angle_begin, angle_end)}
 *             M_[l|c|, l|c|, l|s|, l|s|, zeta, zeta](lambda_x <(-sin t, cos t), dk>)
 *     written to taps[(2N-1)*(2N-1)] (dtype dt; OVERWRITTEN, not accumulated).
 *     The angle range selects a shard: the full filter is the sum of the shards
 *     (BASELINE.json config 4 sums them with an NCCL allreduce).
 *     Errors: BSCT_EINVAL for an invalid geometry or 0 <= begin <= end <= n_angles violated.
 */
bsct_status bsct_gram_build(const bsct_geometry *g, bsct_dtype dt, int32_t angle_begin, int32_t angle_end,
                            void *taps, bsct_stream stream);

/*
 * Plan: per-geometry device state -- per-angle box-spline tables, the filter
 * spectrum of the L x L circulant embedding of `taps` (DEVICE, full filter,
 * dtype dt; read during this call only), FFT twiddles and workspaces for up to
 * max_batch slices (0 <= max_batch <= 65535, else BSCT_EINVAL).  Synchronises `stream`
 * once (table upload).  The plan owns all of its memory; destroy with bsct_plan_destroy.
 * A plan may be used from one host thread at a time.
 */
bsct_status bsct_plan_create(const bsct_geometry *g, bsct_dtype dt, const void *taps, int32_t max_batch,
                             bsct_plan *out, bsct_stream stream);
bsct_status bsct_plan_destroy(bsct_plan plan);

/*
 * Re-derive a plan's per-geometry filter state from (new) taps without reallocating:
 * per-angle tables (K0) and the filter spectrum (K2).  Stream-ordered, no host sync.
 * This is the per-geometry part of a reconstruction step (gram_build -> set_filter).
 */
bsct_status bsct_plan_set_filter(bsct_plan plan, const void *taps, bsct_stream stream);

/* Copy of the filter spectrum S[q][p] = Re DFT2(E)[p][q] / L^2, q in [0, L/2], p in [0, L)
 * (layout [L/2+1][L], plan dtype) into `out` (DEVICE). */
bsct_status bsct_plan_spectrum(bsct_plan plan, void *out, bsct_stream stream);

/*
 * (b) step 1: correction filter, Eq.(5) P:145-150.  For each angle of B slices:
 *     degree d = #nonzero{l|cos t|, l|sin t|, zeta} - 1;
 *     d = 2: g~ = g_s * q, q[m] = sqrt(2)(2sqrt(2)-3)^|m|, |m| <= 25 (reading R7/R8,
 *     zero-extended full linear convolution); d <= 1: g~ = g_s (q = delta).
 *     sino [B][n_angles][n_det] -> g_tilde [B][n_angles][n_det + 50] (sample j <-> m = j - 25).
 */
bsct_status bsct_correction_filter(bsct_plan plan, const void *sino, void *g_tilde, int32_t B,
                                   bsct_stream stream);

/*
 * (b) Back projection b = H^T g^_psi of B sinograms:
 *     b[k] = lambda_x^2 lambda_y sum_t sum_m g~[t][m] M_[l|c|, l|s|, zeta] U [lambda_y]^(d+1)(y_m - k_t)
 *     sino [B][n_angles][n_det] -> b [B][N][N].  Uses plan workspace (g~).
 */
bsct_status bsct_backproject(bsct_plan plan, const void *sino, void *b, int32_t B, bsct_stream stream);

/*
 * (c) Normal operator y = G x for B slices: y[i] = sum_j G[i - j] x[j],
 *     computed as crop(IFFT_L(S * FFT_L(pad x))).  x, y [B][N][N]; x == y allowed.
 */
bsct_status bsct_normal_apply(bsct_plan plan, const void *x, void *y, int32_t B, bsct_stream stream);

/*
 * Solver for G x = b on B independent slices, `iters` iterations from x = 0:
 *   BSCT_CG         conjugate gradients (north_star)
 *   BSCT_SD         steepest descent with exact line search
 *   BSCT_LANDWEBER  x += tau (b - G x), tau = 1 / max(spectrum * L^2)
 * b, x [B][N][N] (x is output).  resid_hist: DEVICE double [B][iters] receiving ||r_k||
 * after each iteration, or NULL.  flags: DEVICE int32 [B] (0 ok, 1 breakdown
 * <p,Gp> <= 0 -- that slice stops updating), or NULL.  Scalars are accumulated in FP64.
 */
bsct_status bsct_cg_solve(bsct_plan plan, const void *b, void *x, int32_t B, int32_t iters, int32_t solver,
                          double *resid_hist, int32_t *flags, bsct_stream stream);

/*
 * Resume (checkpoint / restart) of a solve on G x = b from a saved state after some iteration j
 * (textbook recurrences, oracle/solvers.py):
 *   x [B][N][N]  IN x_j, OUT x_{j+iters}
 *   r [B][N][N]  IN r_j = b - G x_j, OUT r_{j+iters}
 *   p [B][N][N]  (CG only; may be NULL for SD / Landweber) IN the search direction p_j,
 *                OUT p_{j+iters} = r_{j+iters} + beta p_{j+iters-1}
 * and runs `iters` iterations on the same fused kernels as bsct_cg_solve (the CG step from
 * (x_j, r_j, p_j) is alpha = <r,r>/<p,Gp>, x += alpha p, r -= alpha G p, beta = <r',r'>/<r,r>).
 * alpha_last: DEVICE double [B] receiving the step length of the last iteration, or NULL.
 * resid_hist / flags as in bsct_cg_solve.  Used for R12 check (ii) (one step from the oracle's
 * state) and to continue a solve in pieces.  All buffers caller-owned DEVICE memory.
 */
bsct_status bsct_cg_resume(bsct_plan plan, void *x, void *r, void *p, int32_t B, int32_t iters, int32_t solver,
                           double *alpha_last, double *resid_hist, int32_t *flags, bsct_stream stream);

/*
 * Forward projection g = H c (Eq.(3), Eq.(4)):
 *     g[t][m] = lambda_x^2 sum_k c_k M_[l|c|, l|s|, zeta](y_m - k_t)
 *     c [B][N][N] -> sino [B][n_angles][n_det].  (Support op: data synthesis, exactness checks.)
 */
bsct_status bsct_forward_project(bsct_plan plan, const void *c, void *sino, int32_t B, bsct_stream stream);

/*
 * Chebyshev semi-iteration for G x = b (NEXT-4; Saad, Alg. 12.1), spectrum assumed in
 * [lambda_min, lambda_max]: no inner products, so x_k is a fixed polynomial in G applied to b
 * (linear in b; FP32 iterates keep parity with FP64).  lambda_max <= 0 takes the plan's bound
 * max(DFT of the L x L embedding) >= lambda_max(G) (interlacing).  Requires
 * 0 < lambda_min < lambda_max (BSCT_EINVAL).  Per iteration: the three FFT passes of
 * bsct_normal_apply + one update kernel.  resid_hist: DEVICE [B][iters] ||r_k|| or NULL.
 */
bsct_status bsct_chebyshev_solve(bsct_plan plan, const void *b, void *x, int32_t B, int32_t iters,
                                 double lambda_min, double lambda_max, double *resid_hist, bsct_stream stream);

/*
 * Plain adjoint of the sampled forward model (SIRT's back projection; NEXT-1):
 *     img[k] = lambda_x^2 sum_t sum_m sino[t][m] M_[l|c|, l|s|, zeta](y_m - k_t)
 * i.e. the transpose of bsct_forward_project (no correction filter, no interpolant --
 * contrast bsct_backproject).  sino [B][n_angles][n_det] -> img [B][N][N].
 * Runs on the K4 kernels with the forward model's box-spline tables (built on first use).
 * BSCT_EINVAL if the geometry is outside K4 v2/v3's support (detector step much finer
 * than the pixel: more than 12 samples per cell).
 */
bsct_status bsct_adjoint_project(bsct_plan plan, const void *sino, void *img, int32_t B, bsct_stream stream);

/*
 * SIRT (simultaneous iterative reconstruction technique) on the forward model, the
 * projection-based iteration the paper's filter method avoids (P:4):
 *     x_0 = 0,  x_{k+1} = x_k + C H^T R (sino - H x_k),
 *     R = 1 / (H 1) per detector sample, C = 1 / (H^T 1) per pixel (0 where the sum is 0),
 * H = bsct_forward_project, H^T = bsct_adjoint_project.  sino [B][n_angles][n_det] ->
 * x [B][N][N].  Weights are computed on first use and kept by the plan.
 */
bsct_status bsct_sirt_solve(bsct_plan plan, const void *sino, void *x, int32_t B, int32_t iters,
                            bsct_stream stream);

/*
 * Reconstruction from DEVICE buffers: x = solver^iters(G, H^T g^) per slice (one back
 * projection, then the filter in every iteration), i.e. bsct_backproject followed by
 * bsct_cg_solve with the same arguments, results identical to that sequence (slices may be
 * processed in chunks of BSCT_PIPE_CHUNK slices; BSCT_PIPE_OVERLAP=1 runs the back projection
 * of chunk c+1 on a plan-owned stream while chunk c iterates -- measured no faster on B200).
 * sino [B][n_angles][n_det] -> x [B][N][N], stream-ordered on `stream`;
 * resid_hist / flags as in bsct_cg_solve (may be NULL).  Uses plan workspace for b.
 */
bsct_status bsct_reconstruct(bsct_plan plan, const void *sino, void *x, int32_t B, int32_t iters, int32_t solver,
                             double *resid_hist, int32_t *flags, bsct_stream stream);

/*
 * End-to-end reconstruction from HOST buffers (the e2e path): copies sino_host
 * [B][n_angles][n_det] to the device, back projects, runs `iters` iterations of
 * `solver`, copies x to x_host [B][N][N], and synchronises `stream`.  Host
 * buffers should be pinned for full PCIe bandwidth.  B <= max_batch.  Pipelined by slice
 * chunks (BSCT_PIPE_CHUNK, default 512, first and last chunk a quarter of that): each chunk's H2D copy runs on a plan-owned stream
 * ahead of its back projection and its D2H copy after its solve, overlapping the kernels.
 */
bsct_status bsct_reconstruct_host(bsct_plan plan, const void *sino_host, void *x_host, int32_t B, int32_t iters,
                                  int32_t solver, bsct_stream stream);

/* Number of kernel launches the last call on this plan enqueued (graph nodes counted). */
int64_t bsct_plan_launch_count(bsct_plan plan);

/* Kernel classes of the profiler (index into bsct_plan_profile_read's arrays). */
typedef enum {
  BSCT_K_TABLES = 0,         /* K0 per-angle box-spline tables            */
  BSCT_K_SPECTRUM = 1,       /* K2 filter spectrum (+ max for Landweber)  */
  BSCT_K_CORRECTION = 2,     /* K3 correction filter                      */
  BSCT_K_BACKPROJECT = 3,    /* K4 back projection                        */
  BSCT_K_PASS_A = 4,         /* K5 row FFTs                               */
  BSCT_K_PASS_B = 5,         /* K5 column FFT * spectrum * inverse        */
  BSCT_K_PASS_C = 6,         /* K5 inverse row FFTs                       */
  BSCT_K_SOLVER_INIT = 7,    /* K6 x = 0, r = p = b, <b,b>                */
  BSCT_K_SOLVER_UPDATE = 8,  /* K6 x += a d, r -= a G d, <r,r>            */
  BSCT_K_SOLVER_FINISH = 9,  /* K6 scalars, p = r + beta p                */
  BSCT_K_FORWARD = 10,       /* K7 forward projection                     */
  BSCT_K_FUSED_CG = 11,      /* fused CG iteration kernels (if used)      */
  BSCT_K_COUNT = 12
} bsct_kernel_class;

/*
 * Profiler: when enabled, every launch enqueued by calls on this plan is bracketed by
 * CUDA events recorded on the caller's stream (device time, no extra sync).
 * bsct_plan_profile_read synchronises on the last recorded event and returns, per
 * kernel class, the accumulated milliseconds and bracket counts since the previous
 * read (ms/count: HOST arrays of length n, either may be NULL), then resets them.
 */
bsct_status bsct_plan_profile(bsct_plan plan, int32_t enable);
bsct_status bsct_plan_profile_read(bsct_plan plan, double *ms, int64_t *count, int32_t n);

#ifdef __cplusplus
}
#endif

#endif /* BSCT_H */
