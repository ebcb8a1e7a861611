// backproject.cu -- K3 correction filter (Eq.(5)) and K4 back projection
// b = H^T g^_psi.
//
// K3: for angles whose interpolation degree is 2 (blur, non-axis angle) the
//     sinogram row is convolved with q[m] = sqrt(2)(2 sqrt(2) - 3)^|m|, |m| <= 25
//     (readings R7, R8: zero-extended full linear convolution, M + 50 outputs);
//     otherwise q = delta and the row is copied into the middle.
// K4: b[k] = lambda_x^2 lambda_y sum_t sum_m g~[t][m] C_t(y_m - k_t), C_t the box spline
//     with widths [l|c|, l|s|, zeta] U [lambda_y]^(d+1) (the pixel footprint convolved with
//     the degree-d B-spline interpolant, Eq.(1)); only the <= floor(W/lambda_y)+1 samples
//     inside C_t's support contribute.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "pptable.cuh"

namespace bsct {

constexpr int HC = 25;  // correction filter half-width ("truncated", R8)

__constant__ double c_q64[2 * HC + 1];
__constant__ float c_q32[2 * HC + 1];

template <typename T> __device__ __forceinline__ T qtap(int i);
template <> __device__ __forceinline__ float qtap<float>(int i) { return c_q32[i]; }
template <> __device__ __forceinline__ double qtap<double>(int i) { return c_q64[i]; }

// q lives in __constant__ memory, which exists per device: uploaded once per device (the
// flags are per device and guarded by a mutex, so a second GPU of the same process gets its
// own copy instead of convolving with q = 0).
static cudaError_t upload_q() {
  static std::mutex mu;
  static std::vector<int> ready;  // devices whose c_q32 / c_q64 hold q
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(ready.begin(), ready.end(), dev) != ready.end()) return cudaSuccess;
  double q[2 * HC + 1];
  float qf[2 * HC + 1];
  const long double z = 2.0L * sqrtl(2.0L) - 3.0L;
  for (int m = -HC; m <= HC; ++m) {
    long double v = sqrtl(2.0L);
    for (int k = 0; k < (m < 0 ? -m : m); ++k) v *= z;
    q[m + HC] = (double)v;
    qf[m + HC] = (float)v;
  }
  e = cudaMemcpyToSymbol(c_q64, q, sizeof(q));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_q32, qf, sizeof(qf));
  if (e == cudaSuccess) ready.push_back(dev);
  return e;
}

// One CTA per (angle, slice-group): CR_ROWS sinogram rows of the same angle (one per slice)
// staged in shared memory, zero-extended.  Each thread computes CJ consecutive outputs of one row
// from a register window of CJ + 2 HC inputs (vector shared-memory loads), the 51 taps as
// constant-bank operands: 51 CJ FMAs per (CJ + 2 HC) / 4 shared loads instead of two shared loads
// per FMA (the round-1 form was bound by shared-memory bandwidth: 5.4 ms per config-5 step against
// ~1 ms of HBM traffic; this form 1.95 ms, tools/time_k3.py).  Per output the taps are summed in the same order as before (t = 0..2 HC),
// so the result is bitwise unchanged.  The degree test is per angle, hence uniform per CTA.
#ifndef BSCT_CR_ROWS
#define BSCT_CR_ROWS 4
#define BSCT_CR_THREADS 128
#define BSCT_CJ 4
#endif
constexpr int CR_ROWS = BSCT_CR_ROWS;  // rows (slices) per CTA
constexpr int CR_THREADS = BSCT_CR_THREADS;
constexpr int CJ = BSCT_CJ;            // outputs per thread

// split != nullptr (FP32, K4 v4): gt receives the TF32-rounded value (cvt.rna) and split the exact
// FP32 residual, both with row stride ldt (the 3xTF32 operands of the tensor-core back projection)
__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// shared-memory row stride: the groups of CJ outputs plus the window overhang, a multiple of 4
__host__ __device__ inline int correction_row_stride(int M) {
  const int G = (M + 2 * HC + CJ - 1) / CJ;
  return (G * CJ + 2 * HC + 4 + 3) & ~3;
}

template <typename T>
__device__ __forceinline__ void correction_store(T v, size_t o, T *__restrict__ gt, T *__restrict__ split) {
  if (split) {
    if constexpr (sizeof(T) == 4) {
      const T hi = tf32_round(v);
      gt[o] = hi;
      split[o] = v - hi;
    }
  } else {
    gt[o] = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(CR_THREADS) correction_kernel(int n_angles, int M, int B, const int *__restrict__ degree,
                                                         const T *__restrict__ sino, T *__restrict__ gt,
                                                         T *__restrict__ split, int ldt, int vec_ok) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *rows = reinterpret_cast<T *>(smem_raw);  // [CR_ROWS][Mp]: rows[rr Mp + u] = g[u - 2 HC], zero outside [0, M)
  const int a = blockIdx.x, b0 = blockIdx.y * CR_ROWS;
  const int nb = min(CR_ROWS, B - b0);
  const int Mt = M + 2 * HC, Mp = correction_row_stride(M);
  const int d = degree[a];
  // every global load of the CTA is issued at once as cp.async (rows start at 4-byte alignment
  // only: M is odd in the paper's geometries); the zero extension by plain stores
  for (int rr = 0; rr < nb; ++rr) {
    const T *src = sino + ((size_t)(b0 + rr) * n_angles + a) * M;
    T *dst = rows + rr * Mp;
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + 2 * HC + m);
      if constexpr (sizeof(T) == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(src + m) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src + m) : "memory");
    }
    for (int u = threadIdx.x; u < Mp - M; u += blockDim.x) dst[u < 2 * HC ? u : u + M] = (T)0;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (d != 2) {  // no correction at this angle: g~[m] = g[m], output j <-> detector index m = j - HC
    for (int i = threadIdx.x; i < nb * Mt; i += blockDim.x) {
      const int rr = i / Mt, j = i - rr * Mt;
      correction_store<T>(rows[rr * Mp + j + HC], ((size_t)(b0 + rr) * n_angles + a) * ldt + j, gt, split);
    }
    return;
  }
  constexpr int VE = 16 / (int)sizeof(T);                      // elements per 16-byte shared load
  constexpr int NW = ((CJ + 2 * HC + VE - 1) / VE) * VE;       // window registers
  const int G = (Mt + CJ - 1) / CJ;
  for (int it = threadIdx.x; it < nb * G; it += blockDim.x) {
    const int rr = it / G, j0 = (it - rr * G) * CJ;            // outputs j0 .. j0 + CJ - 1 of row rr
    const T *row = rows + rr * Mp + j0;                        // row[u] = g[j0 - 2 HC + u], 16-byte aligned
    T w[NW];
#pragma unroll
    for (int k = 0; k < NW / VE; ++k) {
      if constexpr (sizeof(T) == 4) {
        const float4 t4 = reinterpret_cast<const float4 *>(row)[k];
        w[4 * k] = t4.x, w[4 * k + 1] = t4.y, w[4 * k + 2] = t4.z, w[4 * k + 3] = t4.w;
      } else {
        const double2 t2 = reinterpret_cast<const double2 *>(row)[k];
        w[2 * k] = t2.x, w[2 * k + 1] = t2.y;
      }
    }
    // g~[m] = sum_{t=0}^{2 HC} q[t - HC] g[m - (t - HC)]: v[k] = sum_t q[t] row[k + 2 HC - t]
    T v[CJ];
#pragma unroll
    for (int k = 0; k < CJ; ++k) v[k] = (T)0;
#pragma unroll
    for (int t = 0; t <= 2 * HC; ++t) {
      const T q = qtap<T>(t);
#pragma unroll
      for (int k = 0; k < CJ; ++k) v[k] = fma(q, w[k + 2 * HC - t], v[k]);
    }
    const size_t o = ((size_t)(b0 + rr) * n_angles + a) * ldt + j0;
    if (sizeof(T) == 4 && vec_ok && j0 + CJ <= Mt) {
      if constexpr (sizeof(T) == 4) {
        float hi[CJ], lo[CJ];
#pragma unroll
        for (int k = 0; k < CJ; ++k) {
          hi[k] = split ? tf32_round(v[k]) : v[k];
          lo[k] = v[k] - hi[k];
        }
#pragma unroll
        for (int k = 0; k < CJ; k += 4) {
          *reinterpret_cast<float4 *>(gt + o + k) = float4{hi[k], hi[k + 1], hi[k + 2], hi[k + 3]};
          if (split) *reinterpret_cast<float4 *>(split + o + k) = float4{lo[k], lo[k + 1], lo[k + 2], lo[k + 3]};
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < CJ; ++k)
        if (j0 + k < Mt) correction_store<T>(v[k], o + k, gt, split);
    }
  }
}

template <typename T>
cudaError_t correction_filter(int n_angles, int M, int B, const int *degree, const T *sino, T *gt, cudaStream_t s,
                              T *split, int ldt) {
  cudaError_t e = upload_q();
  if (e != cudaSuccess) return e;
  const size_t sm = sizeof(T) * (size_t)CR_ROWS * correction_row_stride(M);
  if (sm > 48 * 1024) {
    e = cudaFuncSetAttribute(correction_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  if (ldt <= 0) ldt = M + 2 * HC;
  // 16-byte output stores where every row start is aligned (the K4 v4 operand layout: ldt % 4 == 0)
  const int vec_ok = sizeof(T) == 4 && ldt % 4 == 0 && ((uintptr_t)gt & 15) == 0 && ((uintptr_t)split & 15) == 0;
  correction_kernel<T><<<dim3(n_angles, (B + CR_ROWS - 1) / CR_ROWS), CR_THREADS, sm, s>>>(n_angles, M, B, degree, sino, gt,
                                                                                     split, ldt, vec_ok);
  return cudaGetLastError();
}

// K4 v1: one thread per pixel, 16 x 16 pixel tiles, all angles in order.
template <typename T>
__global__ void __launch_bounds__(256) backproject_kernel(int N, double lx, double ly, int n_angles, int M,
                                                          const double *__restrict__ cs, PPView<T> tb,
                                                          const T *__restrict__ gt, T *__restrict__ out) {
  const int k2 = blockIdx.x * 16 + threadIdx.x;
  const int k1 = blockIdx.y * 16 + threadIdx.y;
  const int b = blockIdx.z;
  const double x1 = lx * (double)(k1 - N / 2);
  const double x2 = lx * (double)(k2 - N / 2);
  const int Mt = M + 2 * HC;
  const T *g = gt + (size_t)b * n_angles * Mt;
  const double m_off = (double)(M / 2);
  T acc = 0;
  for (int a = 0; a < n_angles; ++a) {
    const double c = cs[2 * a], s = cs[2 * a + 1];
    const double kt = fma(-s, x1, c * x2);
    const double H = tb.half[a];
    // samples with |y_m - k_t| < H, y_m = ly (m - floor(M/2))
    int m = (int)floor((kt - H) / ly + m_off) + 1;
    const T *ga = g + (size_t)a * Mt + HC;
    for (;; ++m) {
      const double arg = ly * ((double)m - m_off) - kt;
      if (arg >= H) break;
      const int j = m + HC;
      if (j < 0 || j >= Mt) continue;
      acc = fma(ga[m], pp_eval<T>(tb, a, arg), acc);
    }
  }
  if (k1 < N && k2 < N) out[((size_t)b * N + k1) * N + k2] = (T)(lx * lx * ly) * acc;
}

template <typename T>
cudaError_t backproject(int N, double lx, double ly, int n_angles, int M, int B, const double *cs, PPView<T> tb,
                        const T *gt, T *b, cudaStream_t s) {
  dim3 grid((N + 15) / 16, (N + 15) / 16, B);
  backproject_kernel<T><<<grid, dim3(16, 16), 0, s>>>(N, lx, ly, n_angles, M, cs, tb, gt, b);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// K4 v2.  With u = (k_t - y_0)/lambda_y = c + phi (cell c = floor(u), phi in [0,1)):
//   F_t(u) = sum_m g~[m] C_t(y_m - k_t) = sum_{i} g~[c + i + imin] C_t(lambda_y (i + imin - phi)).
// The knots of C_t map to phi-breakpoints frac((W/2 - sigma)/lambda_y) where sigma runs over
// subset sums of the non-lambda_y widths {l|c|, l|s|, zeta} (the lambda_y widths shift knots by
// whole cells), so the unit cell splits into P <= 9 sub-intervals on which every
// C_t(lambda_y(i + imin - phi)) is one polynomial Q_{p,i}(tau), tau = phi - bp[p].
// build_bp_tables: B[a][p][i][k] = coefficients of Q_{p,i} (FP64, subset sums, left half).
// backproject_v2: per 64x64 pixel tile and angle, F[c][p][k] = sum_i g~[c+i+imin] B[p][i][k]
// in shared memory for the tile's cells, then per pixel one sub-interval search and one
// degree-5 Horner.  Same closed form as K4 v1 (and the oracle), different evaluation order.
// ----------------------------------------------------------------------------------------

size_t bp_table_floats(int n) { return (size_t)n * BP_PMAX * BP_SMAX * 8; }

// interp = 1: the back projection's kernel C_t = [l|c|, l|s|, zeta] U [lambda_y]^(d+1) (degree-d
// B-spline interpolant of g); interp = 0: the plain adjoint of the sampled forward
// model, C_t = M_[l|c|, l|s|, zeta] (H^T, used by SIRT).  Same breakpoint structure.
template <typename T>
__global__ void __launch_bounds__(128) bp_tables_kernel(int N, int M, double lx, double ly, double zeta, int n,
                                                        const double *__restrict__ cs, const int *__restrict__ degree,
                                                        BPAngle *__restrict__ ang, T *__restrict__ Btab, int interp) {
  const int a = blockIdx.x;
  const int tid = threadIdx.x;
  __shared__ double w[8], sig[64], bp[16], wb[4];
  __shared__ int sgn[64], nw, nbase, P, S, imin;
  __shared__ bool rownz[BP_PMAX * BP_SMAX];
  __shared__ double H;
  if (a >= n) return;
  const double c = cs[2 * a], s = cs[2 * a + 1];
  if (tid == 0) {
    double raw[8];
    int nr = 0;
    raw[nr++] = lx * fabs(c);
    raw[nr++] = lx * fabs(s);
    if (zeta > 0) raw[nr++] = zeta;
    const int d = degree[a];
    const int nbr = nr;
    if (interp)
      for (int i = 0; i <= d; ++i) raw[nr++] = ly;
    double ssum = 0;
    for (int i = 0; i < nr; ++i) ssum += raw[i];
    const double thr = 1e-12 * fmax(1.0, ssum);
    int k = 0, kb = 0;
    for (int i = 0; i < nr; ++i)
      if (raw[i] > thr) {
        w[k++] = raw[i];
        if (i < nbr) wb[kb++] = raw[i];
      }
    nw = k;
    nbase = kb;
    double W = 0;
    for (int i = 0; i < k; ++i) W += w[i];
    H = 0.5 * W;
    const int cw = (int)ceil(H / ly - 1e-12);
    imin = -cw;
    S = 2 * cw + 1;
    // phi breakpoints
    double f[9];
    int nf = 0;
    f[nf++] = 0.0;
    for (int m = 0; m < (1 << kb); ++m) {
      double sg = 0;
      for (int i = 0; i < kb; ++i)
        if ((m >> i) & 1) sg += wb[i];
      double v = (H - sg) / ly;
      v -= floor(v);
      if (v > 1.0 - 1e-12) v = 0.0;
      f[nf++] = v;
    }
    for (int i = 1; i < nf; ++i)  // insertion sort
      for (int j = i; j > 0 && f[j] < f[j - 1]; --j) { double t = f[j]; f[j] = f[j - 1]; f[j - 1] = t; }
    int np = 0;
    for (int i = 0; i < nf; ++i)
      if (np == 0 || f[i] > bp[np - 1] + 1e-12) bp[np++] = f[i];
    P = np;
    BPAngle A;
    const double x0 = lx * (double)(0 - N / 2), y0 = ly * (double)(0 - M / 2);
    A.u0 = (fma(-s, x0, c * x0) - y0) / ly;
    A.du1 = -s * lx / ly;
    A.du2 = c * lx / ly;
    for (int i = 0; i < BP_PMAX; ++i) A.bp[i] = i < np ? bp[i] : 3.0e38;
    for (int i = 0; i < BP_PMAX; ++i) A.bpf[i] = i < np ? (float)bp[i] : 3.0e38f;
    A.P = np;
    A.S = S;
    A.imin = -cw;
    A.pad = 0;
    ang[a] = A;
  }
  __syncthreads();
  const int n_w = nw, ns = 1 << n_w;
  if (tid < ns) {
    double sm = 0;
    int pc = 0;
    for (int i = 0; i < n_w; ++i)
      if ((tid >> i) & 1) { sm += w[i]; ++pc; }
    sig[tid] = sm;
    sgn[tid] = (pc & 1) ? -1 : 1;
  }
  __syncthreads();
  double prodw = 1.0, fact = 1.0;
  for (int i = 0; i < n_w; ++i) prodw *= w[i];
  for (int i = 2; i < n_w; ++i) fact *= i;
  const double norm = 1.0 / (fact * prodw);
  const int deg = n_w - 1;
  const double Hh = H;
  T *Ba = Btab + (size_t)a * BP_PMAX * BP_SMAX * 8;
  for (int item = tid; item < BP_PMAX * BP_SMAX; item += blockDim.x) {
    const int p = item / BP_SMAX, i = item % BP_SMAX;
    double coef[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (p < P && i < S) {
      const double ph = bp[p], phn = (p + 1 < P) ? bp[p + 1] : 1.0;
      const double x0 = ly * ((double)(i + imin) - ph);  // argument at tau = 0; x(tau) = x0 - ly tau
      const double e = x0 - 0.5 * ly * (phn - ph);        // interior point of the range
      if (fabs(e) < Hh) {
        // even symmetry: evaluate on the left half, y(tau) = y0 + g tau
        const bool fl = e > 0;
        const double y0v = fl ? -x0 : x0, g = fl ? ly : -ly, ye = fl ? -e : e;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int S2 = 0; S2 < ns; ++S2) {
          if (!(sig[S2] - Hh < ye)) continue;  // knot right of the range: inactive
          const double dl = fmax(0.0, y0v + Hh - sig[S2]);
          double pw = 1.0;  // dl^(deg-k) for k = deg..0
          for (int k = deg; k >= 0; --k) {
            acc[k] += sgn[S2] * pw;
            pw *= dl;
          }
        }
        double binom = 1.0, gk = 1.0;
        for (int k = 0; k <= deg; ++k) {
          coef[k] = norm * binom * gk * acc[k];
          binom = binom * (deg - k) / (k + 1);
          gk *= g;
        }
      }
    }
    for (int k = 0; k < 8; ++k) Ba[(size_t)item * 8 + k] = (T)coef[k];
    bool nz = false;
    for (int k = 0; k < 8; ++k) nz = nz || (T)coef[k] != (T)0;
    rownz[item] = nz;
  }
  __syncthreads();
  // nonzero row range per sub-interval: rows outside the kernel's support on that sub-interval
  // are all-zero, and K4 skips them when it builds its tables (identical sums: exact zeros)
  if (tid < BP_PMAX) {
    int lo = BP_SMAX, hi = -1;
    for (int i = 0; i < BP_SMAX; ++i)
      if (rownz[tid * BP_SMAX + i]) {
        lo = i < lo ? i : lo;
        hi = i;
      }
    if (hi < 0) lo = 1, hi = 0;  // empty range
    ang[a].ilo[tid] = (unsigned char)lo;
    ang[a].ihi[tid] = (unsigned char)hi;
  }
}

template <typename T>
cudaError_t build_bp_tables(int N, int M, double lx, double ly, double zeta, int n, const PPTables<T> &tb,
                            BPAngle *ang, T *Btab, cudaStream_t s, int interp) {
  bp_tables_kernel<T><<<n, 128, 0, s>>>(N, M, lx, ly, zeta, n, tb.cs, tb.degree, ang, Btab, interp);
  return cudaGetLastError();
}

// gt[b][a][j] = w[a][m] (g[b][a][m] - h[b][a][m]) for m = j - HC in [0, M), zero in the HC-wide
// ends (the layout K4 reads); w and h may be null (factor 1, nothing subtracted).
template <typename T>
__global__ void __launch_bounds__(256) pad_rows_kernel(int n_angles, int M, int B, const T *__restrict__ g,
                                                       const T *__restrict__ h, const T *__restrict__ w,
                                                       T *__restrict__ gt) {
  const int Mt = M + 2 * HC;
  const size_t total = (size_t)B * n_angles * Mt;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i / Mt;
    const int m = (int)(i - row * Mt) - HC;
    T v = 0;
    if (m >= 0 && m < M) {
      const size_t e = row * M + m;
      v = g[e];
      if (h) v -= h[e];
      if (w) v *= w[(row % n_angles) * M + m];
    }
    gt[i] = v;
  }
}

template <typename T>
cudaError_t pad_rows(int n_angles, int M, int B, const T *g, const T *h, const T *w, T *gt, cudaStream_t s) {
  const size_t total = (size_t)B * n_angles * (M + 2 * HC);
  const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
  pad_rows_kernel<T><<<blocks, 256, 0, s>>>(n_angles, M, B, g, h, w, gt);
  return cudaGetLastError();
}
template cudaError_t pad_rows<float>(int, int, int, const float *, const float *, const float *, float *, cudaStream_t);
template cudaError_t pad_rows<double>(int, int, int, const double *, const double *, const double *, double *,
                                      cudaStream_t);

constexpr int BPT = 64;          // tile edge (pixels)
constexpr int BP_ROWS = 16;      // rows per thread
constexpr int BP_THREADS = 256;  // 8 warps = 4 (rows of 16) x 2 (32 columns)

template <typename T>
__device__ __forceinline__ T horner6(const T *e, T t) {
  T r = e[5];
  r = fma(r, t, e[4]);
  r = fma(r, t, e[3]);
  r = fma(r, t, e[2]);
  r = fma(r, t, e[1]);
  r = fma(r, t, e[0]);
  return r;
}

// 16-byte shared-memory vector of T (float4 / double2x2 halves)
template <typename T> struct Vec8;
template <> struct Vec8<float> {
  __device__ static void load(const float *p, float *v) {
    const float4 a = reinterpret_cast<const float4 *>(p)[0], b = reinterpret_cast<const float4 *>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ static void store(float *p, const float *v) {
    reinterpret_cast<float4 *>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4 *>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <> struct Vec8<double> {
  __device__ static void load(const double *p, double *v) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 a = reinterpret_cast<const double2 *>(p)[i];
      v[2 * i] = a.x; v[2 * i + 1] = a.y;
    }
  }
  __device__ static void store(double *p, const double *v) {
#pragma unroll
    for (int i = 0; i < 4; ++i) reinterpret_cast<double2 *>(p)[i] = make_double2(v[2 * i], v[2 * i + 1]);
  }
};

struct BPTileAngle {  // per (tile, angle) parameters
  int c_lo, ncell;
};
__device__ __forceinline__ BPTileAngle bp_tile_angle(const BPAngle &A, int tk1, int tk2, int max_cells) {
  const double ua = fma(A.du1, (double)tk1, fma(A.du2, (double)tk2, A.u0));
  const double e1 = A.du1 * (BPT - 1), e2 = A.du2 * (BPT - 1);
  const double umin = ua + fmin(0.0, e1) + fmin(0.0, e2), umax = ua + fmax(0.0, e1) + fmax(0.0, e2);
  BPTileAngle r;
  r.c_lo = (int)floor(umin) - 1;
  r.ncell = min((int)floor(umax) - r.c_lo + 2, max_cells);
  return r;
}

// Shared memory per buffer (double-buffered by angle parity):
//   table [max_cells][maxP*8+4]  entries {c0..c5, bp_p, 0}; the odd number of 16-byte units per
//                                 cell row keeps consecutive cells in distinct bank groups
//   Bst   [maxP][BP_SMAX][8]     this angle's basis B[p][i][k]
//   gst   [max_cells + BP_SMAX]  this tile's segment of g~
// PC = compile-time number of breakpoint compares (>= maxP - 1; unused breakpoints are +huge).
template <typename T, int PC>
__global__ void __launch_bounds__(BP_THREADS) bp_v2_kernel(int N, int n_angles, int M, const BPAngle *__restrict__ ang,
                                                           const T *__restrict__ Btab, const T *__restrict__ gt,
                                                           T *__restrict__ out, int max_cells, int maxP, T scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *sm = reinterpret_cast<T *>(smem_raw);
  const int tab_sz = max_cells * (maxP * 8 + 4);
  const int bst_sz = maxP * BP_SMAX * 8;
  const int buf_sz = tab_sz + bst_sz + ((max_cells + BP_SMAX + 7) & ~7);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tk1 = blockIdx.y * BPT, tk2 = blockIdx.x * BPT;
  const int k1_0 = tk1 + (warp >> 1) * BP_ROWS;
  const int k2 = tk2 + (warp & 1) * 32 + lane;
  const int b = blockIdx.z;
  const int Mt = M + 2 * HC;
  const T *g = gt + (size_t)b * n_angles * Mt;

  // stage angle a's basis and g~ segment into buffer a & 1
  auto stage = [&](int a) {
    const BPAngle &A = ang[a];
    const BPTileAngle ta = bp_tile_angle(A, tk1, tk2, max_cells);
    T *base = sm + (a & 1) * buf_sz;
    T *Bst = base + tab_sz;
    T *gst = Bst + bst_sz;
    const T *Ba = Btab + (size_t)a * BP_PMAX * BP_SMAX * 8;
    const int nb = A.P * BP_SMAX * 8;
    for (int i = threadIdx.x * 4; i < nb; i += BP_THREADS * 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) Bst[i + u] = Ba[i + u];
    }
    const T *ga = g + (size_t)a * Mt + HC;  // ga[m]: g~ at detector index m in [-HC, M+HC)
    const int m0 = ta.c_lo + A.imin;
    for (int j = threadIdx.x; j < ta.ncell + A.S; j += BP_THREADS) {
      const int m = m0 + j;
      gst[j] = (m >= -HC && m < M + HC) ? ga[m] : (T)0;
    }
  };

  T acc[BP_ROWS];
#pragma unroll
  for (int j = 0; j < BP_ROWS; ++j) acc[j] = 0;
  stage(0);
  __syncthreads();
  for (int a = 0; a < n_angles; ++a) {
    const BPAngle &A = ang[a];
    const int P = A.P, S = A.S;
    const BPTileAngle ta = bp_tile_angle(A, tk1, tk2, max_cells);
    const int stride = P * 8 + 4;
    T *buf = sm + (a & 1) * buf_sz;
    const T *Bst = buf + tab_sz;
    const T *gst = Bst + bst_sz;
    // build F[c][p][k] = sum_i g~[c + i + imin] B[p][i][k] for the tile's cells
    for (int item = threadIdx.x; item < P * ta.ncell; item += BP_THREADS) {
      const int p = item / ta.ncell, cc = item - p * ta.ncell;
      T f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const T *Bp = Bst + p * BP_SMAX * 8;
      for (int i = 0; i < S; ++i) {
        const T gv = gst[cc + i];
        T bb[8];
        Vec8<T>::load(Bp + i * 8, bb);
#pragma unroll
        for (int k = 0; k < 6; ++k) f[k] = fma(gv, bb[k], f[k]);
      }
      f[6] = (T)A.bp[p];
      Vec8<T>::store(buf + cc * stride + p * 8, f);
    }
    if (a + 1 < n_angles) stage(a + 1);  // the other buffer: last read before the previous barrier
    __syncthreads();
    // evaluate: cell, sub-interval (uniform breakpoints in registers), one Horner
    T bk[BP_PMAX];
#pragma unroll
    for (int k = 1; k <= PC; ++k) bk[k] = (T)A.bp[k];
    const double ub = fma(A.du1, (double)k1_0, fma(A.du2, (double)k2, A.u0));
    const double cb = floor(ub);
    const T fb = (T)(ub - cb);
    const int cbi = (int)cb - ta.c_lo;
    const T d1 = (T)A.du1;
#pragma unroll
    for (int j = 0; j < BP_ROWS; ++j) {
      const T v = fma(d1, (T)j, fb);
      const T cf = floor(v);
      const T ph = v - cf;
      const int cc = cbi + (int)cf;
      int p = 0;
#pragma unroll
      for (int k = 1; k <= PC; ++k) p += (ph >= bk[k]) ? 1 : 0;
      T e[8];
      Vec8<T>::load(buf + cc * stride + p * 8, e);
      const T tau = ph - e[6];
      T rr = e[5];
      rr = fma(rr, tau, e[4]);
      rr = fma(rr, tau, e[3]);
      rr = fma(rr, tau, e[2]);
      rr = fma(rr, tau, e[1]);
      rr = fma(rr, tau, e[0]);
      acc[j] += rr;
    }
  }
  if (k2 < N) {
    T *o = out + (size_t)b * N * N;
#pragma unroll
    for (int j = 0; j < BP_ROWS; ++j)
      if (k1_0 + j < N) o[(size_t)(k1_0 + j) * N + k2] = scale * acc[j];
  }
}

template <typename T>
cudaError_t backproject_v2(int N, int n_angles, int M, int B, const BPAngle *ang, const T *Btab, const T *gt, T *b,
                           int max_cells, int maxP, double scale, cudaStream_t s) {
  const int tab_sz = max_cells * (maxP * 8 + 4);
  const int buf_sz = tab_sz + maxP * BP_SMAX * 8 + ((max_cells + BP_SMAX + 7) & ~7);
  const size_t sm = sizeof(T) * 2 * (size_t)buf_sz;
  dim3 grid((N + BPT - 1) / BPT, (N + BPT - 1) / BPT, B);
  cudaError_t e;
  if (maxP <= 5) {
    e = cudaFuncSetAttribute(bp_v2_kernel<T, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    bp_v2_kernel<T, 4><<<grid, BP_THREADS, sm, s>>>(N, n_angles, M, ang, Btab, gt, b, max_cells, maxP, (T)scale);
  } else {
    e = cudaFuncSetAttribute(bp_v2_kernel<T, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    bp_v2_kernel<T, 8><<<grid, BP_THREADS, sm, s>>>(N, n_angles, M, ang, Btab, gt, b, max_cells, maxP, (T)scale);
  }
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
// K4 v3 (FP32): SB slices per CTA.  The per-(tile, angle) geometry -- which cell and which
// sub-interval each pixel falls in, and tau -- depends only on the angle, so one locate per
// pixel-angle serves SB slices; each slice then costs two 16-byte table loads and one
// degree-5 Horner.  Table entries are interleaved by slice, [cell][p][s][8] = {c0..c5,
// bp_p - 1/2, 0}, so the SB loads of one pixel use immediate offsets from one address.
// The cell index uses round-to-nearest through the FP32 magic constant 1.5 * 2^23 on
// u - 1/2 (no conversion instructions): ph - 1/2 = (u - 1/2) - round(u - 1/2), exact.
// At ph = 1 (a tie rounded to even) the last sub-interval of the previous cell is
// evaluated at its right end, which equals F at the cell start (F_t is continuous: the
// box spline has >= 2 nonzero widths).  Same closed form as K4 v1/v2.
// ----------------------------------------------------------------------------------------
constexpr float BP_MAGIC = 12582912.0f;  // 1.5 * 2^23

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
// 4-byte copy; src_bytes = 0 writes a zero (src must still be a valid address)
__device__ __forceinline__ void cp_async4(void *dst, const void *src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND)); }

// Shared memory: table double buffer [2][SB][6][PL] FP32 coefficient planes (entry
// idx = cell * P + p, one float per plane) + a 3-slot staging ring [3][stg_sz] (basis of
// the angle + the SB g~ segments) filled by cp.async two angles ahead, so that the
// global-load latency overlaps a whole angle of work.  Each warp evaluates 4 x 8 pixel
// blocks: with one 4-byte load per coefficient plane, a block's lanes hit ~1.4
// wavefronts per load on average over the config-5 angles (vs ~7.4 per 16-byte load for
// 32-pixel rows with 32-byte entries; bank model checked against ncu).  The sub-interval
// start bp_p is selected from registers alongside the sub-interval search.
// NC: polynomial coefficients per entry -- 6 for the back projection's degree-5 kernel, 3 for
// the plain adjoint's (forward model, <= 3 widths: degree <= 2; half the table traffic)
template <int SB, int PC, int PL, int NC>
__global__ void __launch_bounds__(BP_THREADS, 2) bp_v3_kernel(int N, int B, int n_angles, int M,
                                                              const BPAngle *__restrict__ ang,
                                                              const float *__restrict__ Btab,
                                                              const float *__restrict__ gt, float *__restrict__ out,
                                                              int max_cells, int maxP, float scale) {
  constexpr int TAB = SB * NC * PL;  // floats per table buffer
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *sm = reinterpret_cast<float *>(smem_raw);
  const int bst_sz = maxP * BP_SMAX * 8;
  const int gseg = (max_cells + BP_SMAX + 3) & ~3;
  const int stg_sz = bst_sz + SB * gseg;
  float *stg0 = sm + 2 * TAB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tk1 = blockIdx.y * BPT, tk2 = blockIdx.x * BPT;
  // warp w: columns 8w..8w+7 of the tile; lane: row (lane >> 3) of each 4-row block
  const int k1_0 = tk1 + (lane >> 3);
  const int k2 = tk2 + warp * 8 + (lane & 7);
  const int b0 = blockIdx.z * SB;
  const int Mt = M + 2 * HC;

  auto stage = [&](int a) {  // asynchronous: basis + g~ segments of angle a into ring slot a % 3
    if (a < n_angles) {
      const BPAngle &A = ang[a];
      const BPTileAngle ta = bp_tile_angle(A, tk1, tk2, max_cells);
      float *Bst = stg0 + (a % 3) * stg_sz;
      float *gst = Bst + bst_sz;
      const float *Ba = Btab + (size_t)a * BP_PMAX * BP_SMAX * 8;
      const int nb4 = A.P * BP_SMAX * 2;
      for (int i = threadIdx.x; i < nb4; i += BP_THREADS) cp_async16(Bst + 4 * i, Ba + 4 * i);
      const int m0 = ta.c_lo + A.imin;
      const int len = ta.ncell + A.S;
      for (int j = threadIdx.x; j < SB * len; j += BP_THREADS) {
        const int sl = j / len, jj = j - sl * len;
        const int m = m0 + jj;
        const bool ok = b0 + sl < B && m >= -HC && m < M + HC;
        const float *src = ok ? gt + ((size_t)(b0 + sl) * n_angles + a) * Mt + HC + m : gt;
        cp_async4(gst + sl * gseg + jj, src, ok ? 4 : 0);
      }
    }
    cp_async_commit();  // (possibly empty) group per angle keeps the wait count uniform
  };

  float acc[SB][BP_ROWS];
#pragma unroll
  for (int sl = 0; sl < SB; ++sl)
#pragma unroll
    for (int j = 0; j < BP_ROWS; ++j) acc[sl][j] = 0.f;
  stage(0);
  stage(1);
  cp_async_wait<1>();
  __syncthreads();
  for (int a = 0; a < n_angles; ++a) {
    const BPAngle &A = ang[a];
    const int P = A.P, S = A.S;
    const BPTileAngle ta = bp_tile_angle(A, tk1, tk2, max_cells);
    float *tab = sm + (a & 1) * TAB;
    const float *Bst = stg0 + (a % 3) * stg_sz;
    const float *gst = Bst + bst_sz;
    // build F_s[c][p][k] = sum_i g~_s[c + i + imin] B[p][i][k] for the tile's cells, all SB slices
    for (int item = threadIdx.x; item < P * ta.ncell; item += BP_THREADS) {
      const int p = item / ta.ncell, cc = item - p * ta.ncell;
      float f[SB][NC];
#pragma unroll
      for (int sl = 0; sl < SB; ++sl)
#pragma unroll
        for (int k = 0; k < NC; ++k) f[sl][k] = 0.f;
      const float *Bp = Bst + p * BP_SMAX * 8;
      const int ilo = A.ilo[p], ihi = A.ihi[p];  // basis rows outside [ilo, ihi] are zero
      for (int i = ilo; i <= ihi; ++i) {
        float bb[8];
        Vec8<float>::load(Bp + i * 8, bb);
#pragma unroll
        for (int sl = 0; sl < SB; ++sl) {
          const float gv = gst[sl * gseg + cc + i];
          if constexpr (NC % 2 == 0) {  // coefficient pairs on the packed FP32x2 pipe
#pragma unroll
            for (int k = 0; k < NC; k += 2) {
              const float2 r = cfma2(float2{gv, gv}, float2{bb[k], bb[k + 1]}, float2{f[sl][k], f[sl][k + 1]});
              f[sl][k] = r.x;
              f[sl][k + 1] = r.y;
            }
          } else {
#pragma unroll
            for (int k = 0; k < NC; ++k) f[sl][k] = fmaf(gv, bb[k], f[sl][k]);
          }
        }
      }
      float *dst = tab + cc * P + p;
#pragma unroll
      for (int sl = 0; sl < SB; ++sl)
#pragma unroll
        for (int k = 0; k < NC; ++k) dst[(sl * NC + k) * PL] = f[sl][k];
    }
    // slot (a + 2) % 3 was last read by build(a - 1), before the previous barrier
    stage(a + 2);
    cp_async_wait<1>();  // this thread's copies of angle a + 1 have landed
    __syncthreads();     // table(a) and staged(a + 1) visible to the CTA
    // evaluate: one locate per pixel, 6 plane loads + one Horner per slice
    float bkm[PC + 1];
#pragma unroll
    for (int k = 1; k <= PC; ++k) bkm[k] = (float)(A.bp[k] - 0.5);
    const double ub = fma(A.du1, (double)k1_0, fma(A.du2, (double)k2, A.u0));
    const double cb = floor(ub);
    const float fbm = (float)(ub - cb) - 0.5f;
    const float *tb = tab + ((int)cb - ta.c_lo) * P;
    const float d4 = (float)(4.0 * A.du1);  // u step between the 4-row blocks
#pragma unroll
    for (int j = 0; j < BP_ROWS; ++j) {
      const float w = fmaf(d4, (float)j, fbm);
      const float t = w + BP_MAGIC;
      const int ci = __float_as_int(t) - __float_as_int(BP_MAGIC);
      const float phm = w - (t - BP_MAGIC);
      int po = 0;
      float bsel = -0.5f;  // bp_0 - 1/2
#pragma unroll
      for (int k = 1; k <= PC; ++k) {
        const bool ge = phm >= bkm[k];
        po += ge ? 1 : 0;
        bsel = ge ? bkm[k] : bsel;
      }
      const float tau = phm - bsel;
      const float *e = tb + ci * P + po;
      if constexpr (SB % 2 == 0) {  // slice pairs on the packed FP32x2 pipe (same tau)
#pragma unroll
        for (int sl = 0; sl < SB; sl += 2) {
          float2 rr{e[(sl * NC + NC - 1) * PL], e[((sl + 1) * NC + NC - 1) * PL]};
#pragma unroll
          for (int k = NC - 2; k >= 0; --k)
            rr = cfma2(rr, float2{tau, tau}, float2{e[(sl * NC + k) * PL], e[((sl + 1) * NC + k) * PL]});
          const float2 sum = cadd(float2{acc[sl][j], acc[sl + 1][j]}, rr);
          acc[sl][j] = sum.x;
          acc[sl + 1][j] = sum.y;
        }
      } else {
#pragma unroll
        for (int sl = 0; sl < SB; ++sl) {
          float rr = e[(sl * NC + NC - 1) * PL];
#pragma unroll
          for (int k = NC - 2; k >= 0; --k) rr = fmaf(rr, tau, e[(sl * NC + k) * PL]);
          acc[sl][j] += rr;
        }
      }
    }
  }
  if (k2 < N) {
#pragma unroll
    for (int sl = 0; sl < SB; ++sl) {
      if (b0 + sl >= B) break;
      float *o = out + (size_t)(b0 + sl) * N * N;
#pragma unroll
      for (int j = 0; j < BP_ROWS; ++j)
        if (k1_0 + 4 * j < N) o[(size_t)(k1_0 + 4 * j) * N + k2] = scale * acc[sl][j];
    }
  }
}

static int bp_v3_plane(int max_cells, int maxP) {
  const int need = max_cells * maxP;
  return need <= 512 ? 512 : need <= 1024 ? 1024 : need <= 2048 ? 2048 : 0;
}

static size_t bp_v3_smem(int SB, int max_cells, int maxP, int NC = 6) {
  const size_t PL = (size_t)bp_v3_plane(max_cells, maxP);
  const size_t stg = (size_t)maxP * BP_SMAX * 8 + SB * (size_t)((max_cells + BP_SMAX + 3) & ~3);
  return sizeof(float) * (2 * (size_t)SB * NC * PL + 3 * stg);
}

template <int SB, int PC, int PL, int NC>
static cudaError_t launch_bp_v3(int N, int n_angles, int M, int B, const BPAngle *ang, const float *Btab,
                                const float *gt, float *b, int max_cells, int maxP, float scale, cudaStream_t s) {
  const size_t sm = bp_v3_smem(SB, max_cells, maxP, NC);
  if (sm > 227 * 1024 || max_cells * maxP > PL) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(bp_v3_kernel<SB, PC, PL, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dim3 grid((N + BPT - 1) / BPT, (N + BPT - 1) / BPT, (B + SB - 1) / SB);
  bp_v3_kernel<SB, PC, PL, NC><<<grid, BP_THREADS, sm, s>>>(N, B, n_angles, M, ang, Btab, gt, b, max_cells, maxP, scale);
  return cudaGetLastError();
}

int bp_v3_slices(int B, int maxP, int max_cells) {
  // slices per CTA (BSCT_BP_SB overrides; default 4, measured best on config 5: 285 ms vs
  // 354 (SB = 2) and 495 (SB = 1)); 0 when no plane size fits (use K4 v2)
  if (bp_v3_plane(max_cells, maxP) == 0) return 0;
  int sb = B >= 4 ? 4 : B >= 2 ? 2 : 1;
  if (const char *e = getenv("BSCT_BP_SB")) sb = atoi(e);
  if (sb != 1 && sb != 2 && sb != 4) sb = 1;
  while (sb > 1 && bp_v3_smem(sb, max_cells, maxP) > 227 * 1024) sb /= 2;
  return bp_v3_smem(sb, max_cells, maxP) > 227 * 1024 ? 0 : sb;
}

cudaError_t backproject_v3(int N, int n_angles, int M, int B, const BPAngle *ang, const float *Btab, const float *gt,
                           float *b, int max_cells, int maxP, double scale, int SB, cudaStream_t s, int ncoef) {
  const float sc = (float)scale;
  const int PL = bp_v3_plane(max_cells, maxP);
#define BP3N(SBV, PLV, NCV)                                                                                     \
  return maxP <= 5 ? launch_bp_v3<SBV, 4, PLV, NCV>(N, n_angles, M, B, ang, Btab, gt, b, max_cells, maxP, sc, s) \
                   : launch_bp_v3<SBV, 8, PLV, NCV>(N, n_angles, M, B, ang, Btab, gt, b, max_cells, maxP, sc, s)
#define BP3(SBV, PLV)                 \
  if (ncoef == 3) { BP3N(SBV, PLV, 3); } \
  BP3N(SBV, PLV, 6)
#define BP3P(SBV)                        \
  switch (PL) {                          \
    case 512: BP3(SBV, 512);             \
    case 1024: BP3(SBV, 1024);           \
    case 2048: BP3(SBV, 2048);           \
    default: return cudaErrorInvalidValue; \
  }
  if (SB == 4) { BP3P(4); }
  if (SB == 2) { BP3P(2); }
  BP3P(1);
#undef BP3P
#undef BP3
#undef BP3N
}

// Host replica of the breakpoint count of bp_tables_kernel (sizes the shared memory; merges
// with a tighter tolerance than the device, so it never under-counts).
int bp_v2_max_p(int n, const double *angles, double lx, double ly, double zeta) {
  int best = 1;
  for (int a = 0; a < n; ++a) {
    const double c = std::cos(angles[a]), s = std::sin(angles[a]);
    double raw[8];
    int nr = 0;
    raw[nr++] = lx * std::fabs(c);
    raw[nr++] = lx * std::fabs(s);
    if (zeta > 0) raw[nr++] = zeta;
    const int nbr = nr;
    double s3 = 0;
    for (int i = 0; i < nr; ++i) s3 += raw[i];
    const double thr3 = 1e-12 * std::fmax(1.0, s3);
    int nz = 0;
    for (int i = 0; i < nr; ++i) nz += raw[i] > thr3;
    for (int i = 0; i < nz; ++i) raw[nr++] = ly;
    double ssum = 0;
    for (int i = 0; i < nr; ++i) ssum += raw[i];
    const double thr = 1e-12 * std::fmax(1.0, ssum);
    double wb[3], W = 0;
    int kb = 0;
    for (int i = 0; i < nr; ++i)
      if (raw[i] > thr) {
        W += raw[i];
        if (i < nbr) wb[kb++] = raw[i];
      }
    const double H = 0.5 * W;
    double f[9];
    int nf = 0;
    f[nf++] = 0.0;
    for (int m = 0; m < (1 << kb); ++m) {
      double sg = 0;
      for (int i = 0; i < kb; ++i)
        if ((m >> i) & 1) sg += wb[i];
      double v = (H - sg) / ly;
      v -= std::floor(v);
      if (v > 1.0 - 1e-13) v = 0.0;
      f[nf++] = v;
    }
    std::sort(f, f + nf);
    int np = 0;
    double last = -1;
    for (int i = 0; i < nf; ++i)
      if (np == 0 || f[i] > last + 1e-13) { last = f[i]; ++np; }
    best = np > best ? np : best;
  }
  return best > 9 ? 9 : best;
}

int bp_v2_max_cells(double lx, double ly, double zeta) {
  const double H = 0.5 * (lx * 1.4142135623730951 + zeta + 3.0 * ly);
  const int S = 2 * (int)ceil(H / ly) + 1;
  if (S > BP_SMAX) return 0;  // too many samples per cell: use K4 v1
  return (int)ceil((BPT - 1) * lx * 1.4142135623730951 / ly) + 5;
}

template cudaError_t build_bp_tables<float>(int, int, double, double, double, int, const PPTables<float> &, BPAngle *,
                                            float *, cudaStream_t, int);
template cudaError_t build_bp_tables<double>(int, int, double, double, double, int, const PPTables<double> &,
                                             BPAngle *, double *, cudaStream_t, int);
template cudaError_t backproject_v2<float>(int, int, int, int, const BPAngle *, const float *, const float *, float *,
                                           int, int, double, cudaStream_t);
template cudaError_t backproject_v2<double>(int, int, int, int, const BPAngle *, const double *, const double *,
                                            double *, int, int, double, cudaStream_t);
template cudaError_t correction_filter<float>(int, int, int, const int *, const float *, float *, cudaStream_t, float *,
                                              int);
template cudaError_t correction_filter<double>(int, int, int, const int *, const double *, double *, cudaStream_t,
                                               double *, int);
template cudaError_t backproject<float>(int, double, double, int, int, int, const double *, PPView<float>,
                                        const float *, float *, cudaStream_t);
template cudaError_t backproject<double>(int, double, double, int, int, int, const double *, PPView<double>,
                                         const double *, double *, cudaStream_t);

}  // namespace bsct
