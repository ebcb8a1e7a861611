// solver.cu -- K6: vector updates and FP64 scalar reductions of the solvers
// (CG: north_star; steepest descent: P:210; Landweber), batched over slices.
//
// Per slice b the scalars live on the device: rho[b][k] = <r_k, r_k>, the pass-B
// partials of <d, G d> and the <r, r> partials.  Every CTA that needs a scalar
// re-reduces the partials of its slice in a fixed order (no atomics, no extra launch),
// so results are bitwise reproducible.
#include "kernels.cuh"

namespace bsct {

constexpr int VT = 256;  // threads per vector CTA

int vec_blocks(int N) {
  const long n = (long)N * N;
  long vb = (n + VT * 8 - 1) / (VT * 8);
  if (vb < 1) vb = 1;
  if (vb > 128) vb = 128;
  return (int)vb;
}

// Deterministic block sum of `v` (all threads get the result).
__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0;
  const int nw = (blockDim.x + 31) >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

// sum of parts[0..n) by the whole CTA in a fixed order
__device__ __forceinline__ double reduce_parts(const double *__restrict__ parts, int n, double *red) {
  double v = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += parts[i];
  return block_sum(v, red);
}

template <typename T>
__global__ void __launch_bounds__(VT) init_kernel(long n, const T *__restrict__ b, T *__restrict__ x, T *__restrict__ r,
                                                  T *__restrict__ p, double *__restrict__ rpart, int rstride) {
  __shared__ double red[32];
  const size_t off = (size_t)blockIdx.y * n;
  double acc = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const T v = b[off + i];
    x[off + i] = 0;
    r[off + i] = v;
    if (p) p[off + i] = v;
    acc += (double)v * v;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) rpart[(size_t)blockIdx.y * rstride + blockIdx.x] = s;
}

__global__ void __launch_bounds__(VT) rho0_kernel(SolverWork w, int iters, int nparts) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  const double s = reduce_parts(w.rpart + (size_t)b * w.rstride, nparts, red);
  if (threadIdx.x == 0) {
    w.rho[(size_t)b * (iters + 1)] = s;
    if (w.flags) w.flags[b] = 0;
  }
}

// x += alpha d; r -= alpha q; rpart <- <r, r>.  d = p (CG) or r (SD, Landweber).
template <typename T>
__global__ void __launch_bounds__(VT) update_kernel(long n, int solver, int it, int iters, T *__restrict__ x,
                                                    T *__restrict__ r, const T *__restrict__ p,
                                                    const T *__restrict__ q, SolverWork w, int gparts) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  const double rho = w.rho[(size_t)b * (iters + 1) + it];
  double alpha;
  if (solver == 2) {
    alpha = *w.tau;
  } else {
    const double gam = reduce_parts(w.gpart + (size_t)b * w.gstride, gparts, red);
    const bool broken = (w.flags && w.flags[b]) || (rho > 0 && !(gam > 0));
    alpha = (rho > 0 && !broken) ? rho / gam : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && rho > 0 && !(gam > 0) && w.flags) w.flags[b] = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) w.alpha[b] = alpha;
  const T al = (T)alpha;
  const size_t off = (size_t)b * n;
  const T *d = solver == 0 ? p : r;
  double acc = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const T di = d[off + i];
    const T ri = fma(-al, q[off + i], r[off + i]);
    x[off + i] = fma(al, di, x[off + i]);
    r[off + i] = ri;
    acc += (double)ri * ri;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) w.rpart[(size_t)b * w.rstride + blockIdx.x] = s;
}

// rho[it+1] = sum rpart; resid; CG: p = r + beta p.
template <typename T>
__global__ void __launch_bounds__(VT) finish_kernel(long n, int solver, int it, int iters, const T *__restrict__ r,
                                                    T *__restrict__ p, SolverWork w, int rparts) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  const double rho_new = reduce_parts(w.rpart + (size_t)b * w.rstride, rparts, red);
  const double rho = w.rho[(size_t)b * (iters + 1) + it];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    w.rho[(size_t)b * (iters + 1) + it + 1] = rho_new;
    if (w.resid) w.resid[(size_t)b * iters + it] = sqrt(rho_new);
  }
  if (solver != 0) return;
  const T beta = (T)(rho > 0 ? rho_new / rho : 0.0);
  const size_t off = (size_t)b * n;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[off + i] = fma(beta, p[off + i], r[off + i]);
}

template <typename T>
cudaError_t solver_init(int N, int B, const T *b, T *x, T *r, T *p, SolverWork w, int iters, cudaStream_t s) {
  const long n = (long)N * N;
  const int vb = vec_blocks(N);
  init_kernel<T><<<dim3(vb, B), VT, 0, s>>>(n, b, x, r, p, w.rpart, w.rstride);
  rho0_kernel<<<dim3(1, B), VT, 0, s>>>(w, iters, vb);
  return cudaGetLastError();
}

template <typename T>
cudaError_t solver_update(int N, int B, int solver, int it, int iters, T *x, T *r, T *p, const T *q, SolverWork w,
                          cudaStream_t s) {
  const long n = (long)N * N;
  update_kernel<T><<<dim3(vec_blocks(N), B), VT, 0, s>>>(n, solver, it, iters, x, r, p, q, w, w.gstride);
  return cudaGetLastError();
}

template <typename T>
cudaError_t solver_finish(int N, int B, int solver, int it, int iters, const T *r, T *p, SolverWork w,
                          cudaStream_t s) {
  const long n = (long)N * N;
  const int vb = vec_blocks(N);
  finish_kernel<T><<<dim3(solver == 0 ? vb : 1, B), VT, 0, s>>>(n, solver, it, iters, r, p, w, vb);
  return cudaGetLastError();
}

constexpr int SPEC_MAX_CTAS = 148;  // one CTA per SM; out[1 .. SPEC_MAX_CTAS] hold the partial maxima

template <typename T>
__global__ void __launch_bounds__(VT) spectrum_max_kernel(long n, const T *__restrict__ S, double *out) {
  __shared__ double red[32];
  double m = -1e300;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    m = fmax(m, (double)S[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mm = fmax(mm, red[i]);
    out[1 + blockIdx.x] = mm;
  }
}

// out[0] = 1 / (L^2 max S) = 1 / max(DFT of the embedding): the Landweber step (max of the
// partial maxima: exact, so independent of the partition)
__global__ void __launch_bounds__(32) tau_kernel(int L, int parts, double *out) {
  double m = -1e300;
  for (int i = threadIdx.x; i < parts; i += 32) m = fmax(m, out[1 + i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) out[0] = 1.0 / ((double)L * (double)L * m);
}

template <typename T>
cudaError_t spectrum_max(int L, const T *S, double *out, cudaStream_t s) {
  spectrum_max_kernel<T><<<SPEC_MAX_CTAS, VT, 0, s>>>((long)(L / 2 + 1) * L, S, out);
  tau_kernel<<<1, 32, 0, s>>>(L, SPEC_MAX_CTAS, out);
  return cudaGetLastError();
}

// SIRT update x[b] += C * d[b] (C: per-pixel weights shared by the slices)
template <typename T>
__global__ void __launch_bounds__(256) sirt_update_kernel(long n, int B, const T *__restrict__ C,
                                                          const T *__restrict__ d, T *__restrict__ x) {
  const size_t total = (size_t)n * B;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
    x[i] = fma(C[i % n], d[i], x[i]);
}

template <typename T>
cudaError_t sirt_update(long n, int B, const T *C, const T *d, T *x, cudaStream_t s) {
  const size_t total = (size_t)n * B;
  const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  sirt_update_kernel<T><<<blocks, 256, 0, s>>>(n, B, C, d, x);
  return cudaGetLastError();
}

template <typename T>
__global__ void __launch_bounds__(256) safe_reciprocal_kernel(long n, T *__restrict__ v) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    v[i] = v[i] > (T)0 ? (T)1 / v[i] : (T)0;
}

template <typename T>
cudaError_t safe_reciprocal(long n, T *v, cudaStream_t s) {
  const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  safe_reciprocal_kernel<T><<<blocks, 256, 0, s>>>(n, v);
  return cudaGetLastError();
}

// ---- Chebyshev semi-iteration (NEXT-4, oracle/solvers.py chebyshev): coefficients are a fixed
// host-computed sequence; per iteration y = G d (normal apply), then this update.
// init: x = 0, r = b, d = b / theta
template <typename T>
__global__ void __launch_bounds__(VT) cheb_init_kernel(long n, const T *__restrict__ b, T *__restrict__ x,
                                                       T *__restrict__ r, T *__restrict__ d, double inv_theta) {
  const size_t off = (size_t)blockIdx.y * n;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const T v = b[off + i];
    x[off + i] = 0;
    r[off + i] = v;
    d[off + i] = (T)((double)v * inv_theta);
  }
}

// x += d; r -= y; d = c1 d + c2 r; partials of <r, r> per (slice, CTA) when rpart != null
template <typename T>
__global__ void __launch_bounds__(VT) cheb_update_kernel(long n, T c1, T c2, T *__restrict__ x, T *__restrict__ r,
                                                         T *__restrict__ d, const T *__restrict__ y,
                                                         double *__restrict__ rpart) {
  __shared__ double red[32];
  const size_t off = (size_t)blockIdx.y * n;
  double acc = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const size_t e = off + i;
    const T dv = d[e];
    x[e] += dv;
    const T rv = r[e] - y[e];
    r[e] = rv;
    d[e] = fma(c1, dv, c2 * rv);
    acc += (double)rv * rv;
  }
  if (rpart) {
    const double sm = block_sum(acc, red);
    if (threadIdx.x == 0) rpart[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = sm;
  }
}

__global__ void __launch_bounds__(VT) cheb_resid_kernel(const double *__restrict__ rpart, int nparts, double *resid,
                                                        int iters, int k) {
  __shared__ double red[32];
  const double s = reduce_parts(rpart + (size_t)blockIdx.x * nparts, nparts, red);
  if (threadIdx.x == 0) resid[(size_t)blockIdx.x * iters + k] = sqrt(s);
}

template <typename T>
cudaError_t cheb_init(int N, int B, const T *b, T *x, T *r, T *d, double inv_theta, cudaStream_t s) {
  cheb_init_kernel<T><<<dim3(vec_blocks(N), B), VT, 0, s>>>((long)N * N, b, x, r, d, inv_theta);
  return cudaGetLastError();
}

template <typename T>
cudaError_t cheb_update(int N, int B, double c1, double c2, T *x, T *r, T *d, const T *y, double *rpart,
                        double *resid, int iters, int k, cudaStream_t s) {
  const int vb = vec_blocks(N);
  cheb_update_kernel<T><<<dim3(vb, B), VT, 0, s>>>((long)N * N, (T)c1, (T)c2, x, r, d, y, resid ? rpart : nullptr);
  if (resid) cheb_resid_kernel<<<B, VT, 0, s>>>(rpart, vb, resid, iters, k);
  return cudaGetLastError();
}

#define BSCT_SOLVER_INST(T)                                                                                        \
  template cudaError_t solver_init<T>(int, int, const T *, T *, T *, T *, SolverWork, int, cudaStream_t);          \
  template cudaError_t solver_update<T>(int, int, int, int, int, T *, T *, T *, const T *, SolverWork,             \
                                        cudaStream_t);                                                             \
  template cudaError_t solver_finish<T>(int, int, int, int, int, const T *, T *, SolverWork, cudaStream_t);        \
  template cudaError_t spectrum_max<T>(int, const T *, double *, cudaStream_t);                                 \
  template cudaError_t sirt_update<T>(long, int, const T *, const T *, T *, cudaStream_t);                       \
  template cudaError_t safe_reciprocal<T>(long, T *, cudaStream_t);                                             \
  template cudaError_t cheb_init<T>(int, int, const T *, T *, T *, T *, double, cudaStream_t);                  \
  template cudaError_t cheb_update<T>(int, int, double, double, T *, T *, T *, const T *, double *, double *,    \
                                      int, int, cudaStream_t);
BSCT_SOLVER_INST(float)
BSCT_SOLVER_INST(double)

}  // namespace bsct
