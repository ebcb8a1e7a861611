// cg.cu -- K5+K6 fused solver iteration: three launches per iteration (north_star "CG loop",
// P:34 "apply the filter in every iteration", P:210 steepest descent).
//
// CG (textbook recurrences, FP64 per-slice scalars):
//   pass A(k):  rho_k = <r_k, r_k> (reduced from pass C(k-1) partials), beta = rho_k / rho_{k-1},
//               x_k = x_{k-1} + alpha_{k-1} p_{k-1},  p_k = r_k + beta p_{k-1},  row DFTs of pad(p_k)
//   pass B(k):  column DFT, * spectrum, inverse column DFT; gamma_k = <p_k, G p_k> by Parseval
//   pass C(k):  alpha_k = rho_k / gamma_k; inverse row DFTs -> (G p_k) rows;
//               r_{k+1} = r_k - alpha_k G p_k; partials of <r_{k+1}, r_{k+1}>
//   final:      x_K = x_{K-1} + alpha_{K-1} p_{K-1}; rho_K
// G p_k never touches HBM.  Steepest descent / Landweber use pass A of normal.cu on r and
// update x in pass C (x += alpha r_k before r is overwritten).
// Partials of <r,r> are double-buffered by iteration parity so that a kernel may read the
// previous partials while writing the next ones.
#include "fft.cuh"
#include "fft32.cuh"
#include "pass_b2048.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include "kernels.cuh"

namespace bsct {

const float2 *tw1024_table();  // normal.cu: W_1024^{jt}, [32][32]
const float2 *tw2048_table();  // normal.cu: W_2048^{(2m+e)t}, [4][32][32]
bool pass_c_warp_enabled();
bool bulk_stage_enabled();  // BSCT_BULK=1: bulk (TMA) copies instead of cp.async staging

__device__ __forceinline__ double cta_sum(double v, double *red) {
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

__device__ __forceinline__ double cta_reduce_parts(const double *__restrict__ parts, int n, double *red) {
  double v = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += parts[i];
  return cta_sum(v, red);
}

// ---------------------------------------------------------------- init: x = 0, r = p = b, partials of <b,b>
template <typename T>
__global__ void __launch_bounds__(256) cg_init_kernel(long n, const T *__restrict__ b, T *__restrict__ x,
                                                      T *__restrict__ r, T *__restrict__ p, FusedWork w) {
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
  const double s = cta_sum(acc, red);
  if (threadIdx.x == 0) w.rpart[(size_t)blockIdx.y * w.nparts + blockIdx.x] = s;  // parity 0
  if (blockIdx.x == 0 && threadIdx.x == 0 && w.flags) w.flags[blockIdx.y] = 0;
}

// ---------------------------------------------------------------- resume: a saved CG/SD/LW state (x_j, r_j, p_j)
// r = r_in, p = q = p_in (q feeds pass A's "r" operand at the first resumed iteration, where
// beta = alpha_prev = 0, so pass A leaves x unchanged and forms p = q + 0 p = p_in exactly);
// partials of <r_j, r_j> (parity 0).  x is the caller's buffer, updated in place.
template <typename T>
__global__ void __launch_bounds__(256) cg_resume_kernel(long n, const T *__restrict__ r_in,
                                                        const T *__restrict__ p_in, T *__restrict__ r,
                                                        T *__restrict__ p, T *__restrict__ q, FusedWork w) {
  __shared__ double red[32];
  const size_t off = (size_t)blockIdx.y * n;
  double acc = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const T v = r_in[off + i];
    r[off + i] = v;
    if (p) {
      const T u = p_in[off + i];
      p[off + i] = u;
      q[off + i] = u;
    }
    acc += (double)v * v;
  }
  const double s = cta_sum(acc, red);
  if (threadIdx.x == 0) w.rpart[(size_t)blockIdx.y * w.nparts + blockIdx.x] = s;  // parity 0
  if (blockIdx.x == 0 && threadIdx.x == 0 && w.flags) w.flags[blockIdx.y] = 0;
}

// export the state after iteration K for a later resume: r_out = r_K and (CG)
// p_out = r_K + beta_K p_{K-1}, beta_K = rho_K / rho_{K-1} -- the same fma as pass A's p update
template <typename T>
__global__ void __launch_bounds__(256) cg_export_kernel(long n, int K, const T *__restrict__ r,
                                                        const T *__restrict__ p, T *__restrict__ r_out,
                                                        T *__restrict__ p_out, FusedWork w) {
  const int b = blockIdx.y;
  double beta = 0.0;
  if (p_out && K > 0) {
    const double rho = w.rho[(size_t)b * w.rho_stride + K], rho_prev = w.rho[(size_t)b * w.rho_stride + K - 1];
    beta = rho_prev > 0 ? rho / rho_prev : 0.0;
  }
  const T be = (T)beta;
  const size_t off = (size_t)b * n;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const T rv = r[off + i];
    r_out[off + i] = rv;
    if (p_out) p_out[off + i] = (K > 0) ? fma(be, p[off + i], rv) : p[off + i];
  }
}

// VW-wide (16-byte when VW = 16/sizeof(T)) global loads / stores
template <typename T, int VW>
__device__ __forceinline__ void vload(T *dst, const T *__restrict__ src) {
  if constexpr (VW * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      const float4 v = *reinterpret_cast<const float4 *>(src);
      dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
    } else {
      const double2 v = *reinterpret_cast<const double2 *>(src);
      dst[0] = v.x; dst[1] = v.y;
    }
  } else {
#pragma unroll
    for (int u = 0; u < VW; ++u) dst[u] = src[u];
  }
}
template <typename T, int VW>
__device__ __forceinline__ void vstore(T *dst, const T *src) {
  if constexpr (VW * sizeof(T) == 16) {
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4 *>(dst) = make_float4(src[0], src[1], src[2], src[3]);
    } else {
      *reinterpret_cast<double2 *>(dst) = make_double2(src[0], src[1]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < VW; ++u) dst[u] = src[u];
  }
}

// ---------------------------------------------------------------- pass A (CG): p-update fused with row DFTs
template <typename T, int L, int VW>
__global__ void __launch_bounds__(FftLaunch<L>::THREADS) cg_pass_a_kernel(int N, int k, T *__restrict__ x,
                                                                          const T *__restrict__ r,
                                                                          T *__restrict__ p,
                                                                          cplx<T> *__restrict__ T1,
                                                                          const cplx<T> *__restrict__ tw,
                                                                          FusedWork w) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunch<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  __shared__ double red[32];
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int b = blockIdx.y;
  // scalars of slice b
  const double rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
  double beta = 0.0, alpha_prev = 0.0;
  if (k > 0) {
    const double rho_prev = w.rho[(size_t)b * w.rho_stride + k - 1];
    beta = rho_prev > 0 ? rho / rho_prev : 0.0;
    alpha_prev = w.alpha[b];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    w.rho[(size_t)b * w.rho_stride + k] = rho;
    if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
  }
  const T be = (T)beta, al = (T)alpha_prev;
  const int row0 = blockIdx.x * 2 * G;
  const size_t so = (size_t)b * N * N;
  // streaming phase: x += a p_old, p = r + b p_old over the CTA's 2G rows, VW-wide accesses,
  // p written into the groups' FFT buffers (row 2gg -> real part, 2gg+1 -> imaginary part)
  T *smT = reinterpret_cast<T *>(smem);
  for (int i = threadIdx.x; i < G * (L - N); i += blockDim.x) {  // zero padding columns [N, L)
    const int gg = i / (L - N), j = N + i % (L - N);
    smem[gg * Cf::SMEM + pidx(j)] = V{0, 0};
  }
  const int rows = min(2 * G, N - row0);
  if (rows < 2 * G)
    for (int i = threadIdx.x; i < (2 * G - rows) * N; i += blockDim.x) {  // rows beyond N
      const int rr = rows + i / N, j = i % N;
      smT[2 * ((rr >> 1) * Cf::SMEM + pidx(j)) + (rr & 1)] = 0;
    }
  const int nv = N / VW;
  for (int i = threadIdx.x; i < rows * nv; i += blockDim.x) {
    const int rr = i / nv, j = (i - rr * nv) * VW;
    const size_t e = so + (size_t)(row0 + rr) * N + j;
    T pv[VW], rv[VW], xv[VW];
    vload<T, VW>(pv, p + e);
    vload<T, VW>(rv, r + e);
    vload<T, VW>(xv, x + e);
#pragma unroll
    for (int u = 0; u < VW; ++u) {
      xv[u] = fma(al, pv[u], xv[u]);
      pv[u] = fma(be, pv[u], rv[u]);
      smT[2 * ((rr >> 1) * Cf::SMEM + pidx(j + u)) + (rr & 1)] = pv[u];
    }
    vstore<T, VW>(x + e, xv);
    vstore<T, VW>(p + e, pv);
  }
  __syncthreads();
  V *sm = smem + g * Cf::SMEM;
  V v[E];
#pragma unroll
  for (int rr = 0; rr < E; ++rr) v[rr] = sm[pidx(t + rr * P)];
  __syncthreads();
  fft_group<T, L, false>(v, sm, tw, t);
  V *T1s = T1 + (size_t)b * Q * N;
  for (int idx = threadIdx.x; idx < Q * G; idx += blockDim.x) {
    const int q = idx / G, gg = idx % G;
    const int ra2 = row0 + 2 * gg;
    if (ra2 >= N) continue;
    const V *s2 = smem + gg * Cf::SMEM;
    const V z = s2[pidx(q)];
    const V zc = s2[pidx((L - q) & (L - 1))];
    T1s[(size_t)q * N + ra2] = V{(T)0.5 * (z.x + zc.x), (T)0.5 * (z.y - zc.y)};
    if (ra2 + 1 < N) T1s[(size_t)q * N + ra2 + 1] = V{(T)0.5 * (z.y + zc.y), (T)0.5 * (zc.x - z.x)};
  }
}

// 16-byte cp.async global -> shared, zero-filling the bytes past src_bytes (0 or 16)
__device__ __forceinline__ void cp_async16z(void *dst, const void *src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}

// ---------------------------------------------------------------- pass A (CG), L = 1024 (FP32 warp FFTs)
// Same contract as cg_pass_a_kernel (16 rows per CTA).  Streaming phase: x += alpha p,
// p = r + beta p with 16-byte accesses, the new p rows kept in shared memory; each warp
// then transforms one row pair (z = p_a + i p_b) with the pruned four-step FFT, splits
// Z into the two rows' half spectra with lane shuffles (Z[L - q] sits in lane (32 - j) mod
// 32, register 31 - k), and the CTA writes T1[q][row0 .. row0 + 16) through a [q][9]
// float4 staging tile (128 contiguous bytes per q).
template <int VW, bool PLAIN, int ROWS>
__global__ void __launch_bounds__(ROWS * 16, 32 / ROWS) cg_pass_a_1024_kernel(int N, int k, float *__restrict__ x,
                                                                const float *__restrict__ r,
                                                                float *__restrict__ p, float2 *__restrict__ T1,
                                                                const float2 *__restrict__ tw1024, FusedWork w) {
  constexpr int L = 1024, Q = L / 2 + 1, NW = ROWS / 2, RS = NW + 1, PW = 512, NT = 32 * NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *ps = reinterpret_cast<float *>(smem_raw);    // [ROWS][PW] new p rows
  float4 *st = reinterpret_cast<float4 *>(smem_raw);  // [Q][RS] output staging (after the FFTs)
  float2 *trb = reinterpret_cast<float2 *>(smem_raw); // [NW][32][33] transposes
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  // PLAIN (y = G x): p is the input x, nothing is updated.  The scalars (rho_k from the <r, r>
  // partials, beta, alpha_{k-1}) are formed after the first batch of row loads is in flight.
  float be = 0.f, al = 0.f;
  auto scalars = [&]() {
    if (PLAIN) return;
    const double rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    double beta = 0.0, alpha_prev = 0.0;
    if (k > 0) {
      const double rho_prev = w.rho[(size_t)b * w.rho_stride + k - 1];
      beta = rho_prev > 0 ? rho / rho_prev : 0.0;
      alpha_prev = w.alpha[b];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
    be = (float)beta;
    al = (float)alpha_prev;
  };
  const int row0 = blockIdx.x * ROWS;
  const int rows = min(ROWS, N - row0);
  const size_t so = (size_t)b * N * N + (size_t)row0 * N;
  if constexpr (VW == 4) {
    // streaming phase, 16-byte rows: the CTA's p (and r, x) rows are copied into shared memory by
    // cp.async (columns >= N and rows >= N zero-filled), so that all of its loads are in flight at
    // once while the scalars are reduced; then x += a p_old, p = r + b p_old in place, written back
    float *sp = ps, *sr = ps + ROWS * PW, *sx = ps + 2 * ROWS * PW;
    constexpr int CH = ROWS * (PW / 4);  // 16-byte chunks per array
    for (int i = threadIdx.x; i < CH; i += NT) {
      const int rr = i / (PW / 4), j = (i - rr * (PW / 4)) * 4;
      const bool ok = rr < rows && j < N;
      const size_t e = ok ? so + (size_t)rr * N + j : so;
      const int o = rr * PW + j, nb = ok ? 16 : 0;
      cp_async16z(sp + o, p + e, nb);
      if (!PLAIN) {
        cp_async16z(sr + o, r + e, nb);
        cp_async16z(sx + o, x + e, nb);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    scalars();
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (!PLAIN) {
      for (int i = threadIdx.x; i < CH; i += NT) {
        const int rr = i / (PW / 4), j = (i - rr * (PW / 4)) * 4;
        if (rr < rows && j < N) {
          const int o = rr * PW + j;
          const float4 pv = *reinterpret_cast<const float4 *>(sp + o), rv = *reinterpret_cast<const float4 *>(sr + o),
                       xv = *reinterpret_cast<const float4 *>(sx + o);
          const float4 xn = make_float4(fmaf(al, pv.x, xv.x), fmaf(al, pv.y, xv.y), fmaf(al, pv.z, xv.z),
                                        fmaf(al, pv.w, xv.w));
          const float4 pn = make_float4(fmaf(be, pv.x, rv.x), fmaf(be, pv.y, rv.y), fmaf(be, pv.z, rv.z),
                                        fmaf(be, pv.w, rv.w));
          const size_t e = so + (size_t)rr * N + j;
          *reinterpret_cast<float4 *>(x + e) = xn;
          *reinterpret_cast<float4 *>(p + e) = pn;
          *reinterpret_cast<float4 *>(sp + o) = pn;
        }
      }
    }
  } else {
    // streaming phase (VW-wide): x += a p_old, p = r + b p_old; p rows -> ps, zero-padded to PW
    // batches of UB items per thread: all 3 UB loads are issued before the first use
    constexpr int ITEMS = ROWS * (PW / VW), UB = 4;
    static_assert(ITEMS % (UB * NT) == 0, "every thread runs the same number of batches (the first one reduces)");
    for (int i0 = threadIdx.x; i0 < ITEMS; i0 += UB * NT) {
      float pv[UB][VW], rv[UB][VW], xv[UB][VW];
      bool ok[UB];
  #pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int i = i0 + u * NT;
        const int rr = i / (PW / VW), j = (i - rr * (PW / VW)) * VW;
        ok[u] = i < ITEMS && rr < rows && j < N;
        if (ok[u]) {
          const size_t e = so + (size_t)rr * N + j;
          vload<float, VW>(pv[u], p + e);
          if (!PLAIN) {
            vload<float, VW>(rv[u], r + e);
            vload<float, VW>(xv[u], x + e);
          }
        }
      }
      if (i0 == (int)threadIdx.x) scalars();  // first batch: uniform across the CTA
  #pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int i = i0 + u * NT;
        if (i >= ITEMS) break;
        const int rr = i / (PW / VW), j = (i - rr * (PW / VW)) * VW;
        if (ok[u]) {
          if (!PLAIN) {
            const size_t e = so + (size_t)rr * N + j;
  #pragma unroll
            for (int c = 0; c < VW; ++c) {
              xv[u][c] = fmaf(al, pv[u][c], xv[u][c]);
              pv[u][c] = fmaf(be, pv[u][c], rv[u][c]);
            }
            vstore<float, VW>(x + e, xv[u]);
            vstore<float, VW>(p + e, pv[u]);
          }
        } else {
  #pragma unroll
          for (int c = 0; c < VW; ++c) pv[u][c] = 0.f;
        }
        vstore<float, VW>(ps + rr * PW + j, pv[u]);
      }
    }
  }
  __syncthreads();
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = float2{ps[(2 * warp) * PW + lane + 32 * m], ps[(2 * warp + 1) * PW + lane + 32 * m]};
  __syncthreads();  // ps becomes the transpose buffers
  dft32<false, true>(v);  // over m (v[16..31] = 0): v[j] = sum_m z[lane + 32 m] W_32^{m j}
  twiddle1024<false>(v, tw1024, lane);  // W_1024^{j t}
  float2 *tr = trb + warp * (32 * 33);
  warp_transpose32(v, tr, lane);  // lane j: v[t]
  dft32<false>(v);                // v[kk] = Z[lane + 32 kk]
  __syncthreads();  // transposes done CTA-wide: the area becomes the output staging tile
  const int src = (32 - lane) & 31;
#pragma unroll
  for (int kk = 0; kk <= 16; ++kk) {
    // Z[L - q] for q = lane + 32 kk: lane (32 - lane) mod 32, register 31 - kk (lane 0: (32 - kk) mod 32)
    float2 zc;
    zc.x = __shfl_sync(0xffffffffu, v[kk < 16 ? 31 - kk : 15].x, src);  // kk = 16: lane 0 only
    zc.y = __shfl_sync(0xffffffffu, v[kk < 16 ? 31 - kk : 15].y, src);
    if (lane == 0) zc = v[(32 - kk) & 31];
    if (kk == 16 && lane != 0) break;
    const float2 z = v[kk];
    const int q = lane + 32 * kk;
    st[q * RS + warp] = make_float4(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y), 0.5f * (z.y + zc.y), 0.5f * (zc.x - z.x));
  }
  __syncthreads();
  float2 *T1s = T1 + (size_t)b * Q * N + row0;
  for (int i = threadIdx.x; i < Q * NW; i += blockDim.x) {
    const int q = i / NW, pr = i % NW, rp = 2 * pr;
    if (rp >= rows) continue;
    const float4 e = st[q * RS + pr];
    float2 *dst = T1s + (size_t)q * N + rp;
    if (rp + 1 < rows) {
      if (!(N & 1)) {
        *reinterpret_cast<float4 *>(dst) = e;
      } else {
        dst[0] = float2{e.x, e.y};
        dst[1] = float2{e.z, e.w};
      }
    } else {
      dst[0] = float2{e.x, e.y};
    }
  }
}

// ---------------------------------------------------------------- pass A (CG), L = 512 (FP32 half-warp FFTs)
// Same contract as cg_pass_a_kernel<float, 512> (32 rows per CTA).  Streaming phase as in
// cg_pass_a_1024_kernel (p rows kept in shared memory, row stride 264 floats so that the two
// half-warps of a warp read different banks); each half-warp transforms one row pair
// (z = p_a + i p_b) with the 16 x 32 four-step FFT of pass_b_512_kernel, which leaves
// Z[t + 32 k] and Z[t + 16 + 32 k] in lane t; Z[L - q] sits in lane 16 - t, registers 15 - k
// of the other set (lane 0: its own registers), fetched with one shuffle per register.
template <int VW, bool PLAIN>
__global__ void __launch_bounds__(256, 2) cg_pass_a_512_kernel(int N, int k, float *__restrict__ x,
                                                               const float *__restrict__ r, float *__restrict__ p,
                                                               float2 *__restrict__ T1,
                                                               const float2 *__restrict__ tw1024, FusedWork w) {
  constexpr int L = 512, Q = L / 2 + 1, ROWS = 32, NP = ROWS / 2, RS = NP + 1, PW = 256, PWS = 264, NT = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *ps = reinterpret_cast<float *>(smem_raw);    // [ROWS][PWS] new p rows
  float4 *st = reinterpret_cast<float4 *>(smem_raw);  // [Q][RS] output staging (after the FFTs)
  float2 *trb = reinterpret_cast<float2 *>(smem_raw); // [NP][32][17] transposes
  __shared__ float2 twl[32 * 32];
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = lane & 15, h = lane >> 4;
  const int pair = 2 * warp + h;
  const int b = blockIdx.y;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {  // layout of pass_b_512_kernel
    const int rr = i >> 5, c = i & 31;
    twl[rr * 32 + (c >> 1) + 16 * (c & 1)] = tw1024[i];
  }
  // PLAIN (y = G x): p is the input x, nothing is updated
  float be = 0.f, al = 0.f;
  auto scalars = [&]() {
    if (PLAIN) return;
    const double rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    double beta = 0.0, alpha_prev = 0.0;
    if (k > 0) {
      const double rho_prev = w.rho[(size_t)b * w.rho_stride + k - 1];
      beta = rho_prev > 0 ? rho / rho_prev : 0.0;
      alpha_prev = w.alpha[b];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
    be = (float)beta;
    al = (float)alpha_prev;
  };
  const int row0 = blockIdx.x * ROWS;
  const int rows = min(ROWS, N - row0);
  const size_t so = (size_t)b * N * N + (size_t)row0 * N;
  constexpr int ITEMS = ROWS * (PW / VW), UB = 4;
  static_assert(ITEMS % (UB * NT) == 0, "every thread runs the same number of batches (the first one reduces)");
  for (int i0 = threadIdx.x; i0 < ITEMS; i0 += UB * NT) {
    float pv[UB][VW], rv[UB][VW], xv[UB][VW];
    bool ok[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int i = i0 + u * NT;
      const int rr = i / (PW / VW), j = (i - rr * (PW / VW)) * VW;
      ok[u] = rr < rows && j < N;
      if (ok[u]) {
        const size_t e = so + (size_t)rr * N + j;
        vload<float, VW>(pv[u], p + e);
        if (!PLAIN) {
          vload<float, VW>(rv[u], r + e);
          vload<float, VW>(xv[u], x + e);
        }
      }
    }
    if (i0 == (int)threadIdx.x) scalars();  // first batch: uniform across the CTA
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int i = i0 + u * NT;
      const int rr = i / (PW / VW), j = (i - rr * (PW / VW)) * VW;
      if (ok[u]) {
        if (!PLAIN) {
          const size_t e = so + (size_t)rr * N + j;
#pragma unroll
          for (int c = 0; c < VW; ++c) {
            xv[u][c] = fmaf(al, pv[u][c], xv[u][c]);
            pv[u][c] = fmaf(be, pv[u][c], rv[u][c]);
          }
          vstore<float, VW>(x + e, xv[u]);
          vstore<float, VW>(p + e, pv[u]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < VW; ++c) pv[u][c] = 0.f;
      }
      vstore<float, VW>(ps + rr * PWS + j, pv[u]);
    }
  }
  __syncthreads();
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = float2{ps[(2 * pair) * PWS + t + 16 * m], ps[(2 * pair + 1) * PWS + t + 16 * m]};
  __syncthreads();  // ps becomes the transpose buffers
  dft32<false, true>(v);  // over m (v[16..31] = 0): v[j] = sum_m z[t + 16 m] W_32^{m j}
#pragma unroll
  for (int j = 1; j < 32; ++j) v[j] = cmul(v[j], twl[j * 32 + t]);  // W_512^{t j}
  float2 *tr = trb + pair * (32 * 17);
#pragma unroll
  for (int j = 0; j < 32; ++j) tr[j * 17 + t] = v[j];
  __syncwarp();
  float2 a0[16], a1[16];
#pragma unroll
  for (int tt = 0; tt < 16; ++tt) {
    a0[tt] = tr[t * 17 + tt];
    a1[tt] = tr[(t + 16) * 17 + tt];
  }
  dft_reg<16, false>(a0);  // a0[kk] = Z[t + 32 kk]
  dft_reg<16, false>(a1);  // a1[kk] = Z[t + 16 + 32 kk]
  __syncthreads();  // transposes done CTA-wide: the area becomes the output staging tile
  const int src = (h << 4) | ((16 - t) & 15);
#pragma unroll
  for (int kk = 0; kk <= 8; ++kk) {
    // partner of Z[t + 32 kk] is Z[L - q] = a1[15 - kk] of lane 16 - t (lane 0: its own a0[16 - kk])
    float2 zc0, zc1;
    const float2 s0 = a1[(15 - kk) & 15], s1 = a0[(15 - kk) & 15];
    zc0.x = __shfl_sync(0xffffffffu, s0.x, src);
    zc0.y = __shfl_sync(0xffffffffu, s0.y, src);
    zc1.x = __shfl_sync(0xffffffffu, s1.x, src);
    zc1.y = __shfl_sync(0xffffffffu, s1.y, src);
    if (t == 0) {
      zc0 = a0[(16 - kk) & 15];
      zc1 = a1[(15 - kk) & 15];
    }
    if (kk < 8 || t == 0) {
      const float2 z = a0[kk & 15];
      const int q = t + 32 * kk;
      st[q * RS + pair] = make_float4(0.5f * (z.x + zc0.x), 0.5f * (z.y - zc0.y), 0.5f * (z.y + zc0.y), 0.5f * (zc0.x - z.x));
    }
    if (kk < 8) {
      const float2 z = a1[kk];
      const int q = t + 16 + 32 * kk;
      st[q * RS + pair] = make_float4(0.5f * (z.x + zc1.x), 0.5f * (z.y - zc1.y), 0.5f * (z.y + zc1.y), 0.5f * (zc1.x - z.x));
    }
  }
  __syncthreads();
  float2 *T1s = T1 + (size_t)b * Q * N + row0;
  for (int i = threadIdx.x; i < Q * NP; i += blockDim.x) {
    const int q = i / NP, pr = i % NP, rp = 2 * pr;
    if (rp >= rows) continue;
    const float4 e = st[q * RS + pr];
    float2 *dst = T1s + (size_t)q * N + rp;
    if (rp + 1 < rows) {
      if (!(N & 1)) {
        *reinterpret_cast<float4 *>(dst) = e;
      } else {
        dst[0] = float2{e.x, e.y};
        dst[1] = float2{e.z, e.w};
      }
    } else {
      dst[0] = float2{e.x, e.y};
    }
  }
}

// ---------------------------------------------------------------- pass A (CG), L = 2048 (FP32 warp FFTs)
// Same contract as cg_pass_a_kernel<float, 2048> (8 rows per CTA).  Streaming phase as in
// cg_pass_a_1024_kernel (new p rows in shared memory, stride 1032 floats); two warps per row
// pair run pass_b_2048_kernel's parity-split forward FFT of z = p_a + i p_b: warp e ends with
// Z[2m + e + 64 k] in lane m, register k, whose Hermitian partner Z[L - q] has the same parity:
// lane (32 - m) mod 32, register 31 - k for e = 0 (lane 0: its own register (32 - k) mod 32) and
// lane 31 - m, register 31 - k for e = 1 -- one shuffle per register.  T1[q][row0 .. row0 + 8)
// is written through a [q parity][q / 2][5] float4 staging tile (64 contiguous bytes per q).
// Tile bx (rows 8 bx .. 8 bx + 7) of slice b; 256 threads; smem: the dynamic shared memory.
// The caller synchronises the CTA before reusing smem for another tile.
template <int VW, bool PLAIN, int UB = 4>
__device__ __forceinline__ void cg_pass_a_2048_tile(int bx, int b, int N, int k, float *__restrict__ x,
                                                    const float *__restrict__ r, float *__restrict__ p,
                                                    float2 *__restrict__ T1, const float2 *__restrict__ tw2,
                                                    FusedWork w, unsigned char *smem_raw) {
  constexpr int L = 2048, Q = L / 2 + 1, ROWS = 8, NP = ROWS / 2, RS = NP + 1, HALF = L / 4 + 1;
  constexpr int PW = 1024, PWS = 1032, NT = 256;
  float *ps = reinterpret_cast<float *>(smem_raw);    // [ROWS][PWS] new p rows
  float4 *st = reinterpret_cast<float4 *>(smem_raw);  // [2][HALF][RS] output staging (after the FFTs)
  float2 *trb = reinterpret_cast<float2 *>(smem_raw); // [8][32][33] transposes
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, e = warp & 1;
  float be = 0.f, al = 0.f;
  auto scalars = [&]() {
    if (PLAIN) return;
    const double rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    double beta = 0.0, alpha_prev = 0.0;
    if (k > 0) {
      const double rho_prev = w.rho[(size_t)b * w.rho_stride + k - 1];
      beta = rho_prev > 0 ? rho / rho_prev : 0.0;
      alpha_prev = w.alpha[b];
    }
    if (bx == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
    be = (float)beta;
    al = (float)alpha_prev;
  };
  const int row0 = bx * ROWS;
  const int rows = min(ROWS, N - row0);
  const size_t so = (size_t)b * N * N + (size_t)row0 * N;
  constexpr int ITEMS = ROWS * (PW / VW);  // UB: row batches in flight per thread
  static_assert(ITEMS % (UB * NT) == 0, "every thread runs the same number of batches (the first one reduces)");
  for (int i0 = threadIdx.x; i0 < ITEMS; i0 += UB * NT) {
    float pv[UB][VW], rv[UB][VW], xv[UB][VW];
    bool ok[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int i = i0 + u * NT;
      const int rr = i / (PW / VW), j = (i - rr * (PW / VW)) * VW;
      ok[u] = rr < rows && j < N;
      if (ok[u]) {
        const size_t e2 = so + (size_t)rr * N + j;
        vload<float, VW>(pv[u], p + e2);
        if (!PLAIN) {
          vload<float, VW>(rv[u], r + e2);
          vload<float, VW>(xv[u], x + e2);
        }
      }
    }
    if (i0 == (int)threadIdx.x) scalars();  // first batch: uniform across the CTA
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int i = i0 + u * NT;
      const int rr = i / (PW / VW), j = (i - rr * (PW / VW)) * VW;
      if (ok[u]) {
        if (!PLAIN) {
          const size_t e2 = so + (size_t)rr * N + j;
#pragma unroll
          for (int c = 0; c < VW; ++c) {
            xv[u][c] = fmaf(al, pv[u][c], xv[u][c]);
            pv[u][c] = fmaf(be, pv[u][c], rv[u][c]);
          }
          vstore<float, VW>(x + e2, xv[u]);
          vstore<float, VW>(p + e2, pv[u]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < VW; ++c) pv[u][c] = 0.f;
      }
      vstore<float, VW>(ps + rr * PWS + j, pv[u]);
    }
  }
  __syncthreads();
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const float2 z{ps[(2 * pair) * PWS + lane + 32 * m], ps[(2 * pair + 1) * PWS + lane + 32 * m]};
    v[m] = e ? twiddle64<false>(z, m) : z;  // z_r W_64^{r e}
  }
  __syncthreads();  // ps becomes the transpose buffers
  dft32<false>(v);  // v[m] = Y[2m + e]
twiddle2048_fwd(v, tw2, e, lane);  // W_2048^{(2m + e) t}
  float2 *tr = trb + warp * (32 * 33);
  warp_transpose32(v, tr, lane);  // lane m: v[t]
  dft32<false>(v);                // v[kk] = Z[2 lane + e + 64 kk]
  __syncthreads();  // transposes done CTA-wide: the area becomes the output staging tile
  const int src = e ? 31 - lane : (32 - lane) & 31;
  auto slot = [&](int q) { return st + ((q & 1) * HALF + (q >> 1)) * RS; };
#pragma unroll
  for (int kk = 0; kk <= 16; ++kk) {
    float2 zc;
    zc.x = __shfl_sync(0xffffffffu, v[(31 - kk) & 31].x, src);
    zc.y = __shfl_sync(0xffffffffu, v[(31 - kk) & 31].y, src);
    if (!e && lane == 0) zc = v[(32 - kk) & 31];
    const int q = 2 * lane + e + 64 * kk;
    if (kk < 16 || q == L / 2) {
      const float2 z = v[kk];
      slot(q)[pair] = make_float4(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y), 0.5f * (z.y + zc.y), 0.5f * (zc.x - z.x));
    }
  }
  __syncthreads();
  float2 *T1s = T1 + (size_t)b * Q * N + row0;
  for (int i = threadIdx.x; i < Q * NP; i += blockDim.x) {
    const int q = i / NP, pr = i % NP, rp = 2 * pr;
    if (rp >= rows) continue;
    const float4 c = slot(q)[pr];
    float2 *dst = T1s + (size_t)q * N + rp;
    if (rp + 1 < rows) {
      if (!(N & 1)) {
        *reinterpret_cast<float4 *>(dst) = c;
      } else {
        dst[0] = float2{c.x, c.y};
        dst[1] = float2{c.z, c.w};
      }
    } else {
      dst[0] = float2{c.x, c.y};
    }
  }
}

template <int VW, bool PLAIN>
__global__ void __launch_bounds__(256, 2) cg_pass_a_2048_kernel(int N, int k, float *__restrict__ x,
                                                                const float *__restrict__ r, float *__restrict__ p,
                                                                float2 *__restrict__ T1,
                                                                const float2 *__restrict__ tw2, FusedWork w) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg_pass_a_2048_tile<VW, PLAIN>(blockIdx.x, blockIdx.y, N, k, x, r, p, T1, tw2, w, smem_raw);
}

// ---------------------------------------------------------------- pass C: inverse row DFTs fused with the r update
// MODE 0: CG (x deferred to pass A); 1: steepest descent; 2: Landweber (alpha = tau)
template <typename T, int L, int MODE, int VW>
__global__ void __launch_bounds__(FftLaunch<L>::THREADS) cg_pass_c_kernel(int N, int k, int gparts,
                                                                          const cplx<T> *__restrict__ T1,
                                                                          T *__restrict__ x, T *__restrict__ r,
                                                                          const cplx<T> *__restrict__ tw,
                                                                          FusedWork w) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunch<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  __shared__ double red[32];
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int b = blockIdx.y;
  double rho;
  if (MODE == 0) {
    rho = w.rho[(size_t)b * w.rho_stride + k];
  } else {
    rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
  }
  double alpha;
  if (MODE == 2) {
    alpha = *w.tau;
  } else {
    const double gam = cta_reduce_parts(w.gpart + (size_t)b * gparts, gparts, red);
    const bool bad = rho > 0 && !(gam > 0);
    const bool frozen = bad || (w.flags && w.flags[b]);
    alpha = (rho > 0 && !frozen) ? rho / gam : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && bad && w.flags) w.flags[b] = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) w.alpha[b] = alpha;
  const T al = (T)alpha;
  const int row0 = blockIdx.x * 2 * G;
  const V *T1s = T1 + (size_t)b * Q * N;
  for (int idx = threadIdx.x; idx < Q * G; idx += blockDim.x) {
    const int q = idx / G, gg = idx % G;
    const int ra2 = row0 + 2 * gg;
    V xa = V{0, 0}, xb = V{0, 0};
    if (ra2 < N) {
      xa = T1s[(size_t)q * N + ra2];
      if (ra2 + 1 < N) xb = T1s[(size_t)q * N + ra2 + 1];
    }
    if (q == 0 || q == L / 2) { xa.y = 0; xb.y = 0; }
    V *s2 = smem + gg * Cf::SMEM;
    s2[pidx(q)] = V{xa.x - xb.y, xa.y + xb.x};
    if (q != 0 && q != L / 2) s2[pidx(L - q)] = V{xa.x + xb.y, xb.x - xa.y};
  }
  __syncthreads();
  V *sm = smem + g * Cf::SMEM;
  V v[E];
#pragma unroll
  for (int rr = 0; rr < E; ++rr) v[rr] = sm[pidx(t + rr * P)];
  __syncthreads();
  fft_group<T, L, true>(v, sm, tw, t);
  // streaming phase: r -= alpha (G d) (and x += alpha r for SD / Landweber), VW-wide accesses
  const size_t so = (size_t)b * N * N;
  const T *smT = reinterpret_cast<const T *>(smem);
  const int rows = min(2 * G, N - row0);
  const int nv = N / VW;
  double acc = 0;
  for (int i = threadIdx.x; i < rows * nv; i += blockDim.x) {
    const int rr = i / nv, j = (i - rr * nv) * VW;
    const size_t e = so + (size_t)(row0 + rr) * N + j;
    T rv[VW], xv[VW];
    vload<T, VW>(rv, r + e);
    if (MODE != 0) vload<T, VW>(xv, x + e);
#pragma unroll
    for (int u = 0; u < VW; ++u) {
      const T z = smT[2 * ((rr >> 1) * Cf::SMEM + pidx(j + u)) + (rr & 1)];
      if (MODE != 0) xv[u] = fma(al, rv[u], xv[u]);
      rv[u] = fma(-al, z, rv[u]);
      acc += (double)rv[u] * rv[u];
    }
    vstore<T, VW>(r + e, rv);
    if (MODE != 0) vstore<T, VW>(x + e, xv);
  }
  const double s = cta_sum(acc, red);
  if (threadIdx.x == 0) w.rpart[((size_t)((k + 1) & 1) * w.B + b) * w.nparts + blockIdx.x] = s;
}

// ---------------------------------------------------------------- pass C, L = 1024 (FP32 warp FFTs)
// Same contract as cg_pass_c_kernel (16 rows per CTA, the same rpart layout).  The 16 rows'
// T1 entries are staged by cp.async into shared memory as [q][9] row-pair float4 slots
// (9: the eight lanes of a quarter warp reading consecutive q hit distinct bank groups),
// each warp inverts one row pair with a 32 x 32 four-step FFT (fft32.cuh) forming only the
// first N <= 512 outputs, and updates r (and x) in place; its r (x) rows are loaded into
// registers before the FFT so that their latency overlaps the arithmetic.
__device__ __forceinline__ void cp_async16_g(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async8_g(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}

template <int MODE, int ROWS>
__global__ void __launch_bounds__(ROWS * 16, 32 / ROWS) cg_pass_c_1024_kernel(int N, int k, int gparts,
                                                                const float2 *__restrict__ T1,
                                                                float *__restrict__ x, float *__restrict__ r,
                                                                const float2 *__restrict__ tw1024, FusedWork w,
                                                                int use_bulk) {
  constexpr int L = 1024, Q = L / 2 + 1, NW = ROWS / 2, RS = NW + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4 *st = reinterpret_cast<float4 *>(smem_raw);  // [Q][RS] row pairs, later [NW][32][33] float2
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * ROWS;
  const int rows = min(ROWS, N - row0);
  // stage T1[q][row0 .. row0 + ROWS) asynchronously; rows beyond N are zero.  N even: one bulk
  // (TMA) copy per q of the rows' contiguous 8 * rows bytes, completion counted on an mbarrier;
  // N odd: 8-byte cp.async per entry
  const float2 *T1s = T1 + (size_t)b * Q * N + row0;
  __shared__ __align__(8) unsigned long long stage_bar;
  const bool bulk = !(N & 1) && use_bulk;
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&stage_bar);
  if (bulk) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(Q * rows * 8));
    }
    __syncthreads();
    for (int q = threadIdx.x; q < Q; q += blockDim.x) {
      float4 *dst = st + q * RS;
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
          "l"(T1s + (size_t)q * N), "r"(rows * 8), "r"(bar)
          : "memory");
      for (int pr = rows / 2; pr < NW; ++pr) dst[pr] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  for (int i = threadIdx.x; i < (bulk ? 0 : Q * NW); i += blockDim.x) {
    const int q = i / NW, pr = i % NW, rp = 2 * pr;
    float4 *dst = st + q * RS + pr;
    const float2 *src = T1s + (size_t)q * N + rp;
    if (rp + 1 < rows) {
      if (!(N & 1)) {
        cp_async16_g(dst, src);  // N even: (q, even row) pairs are 16-byte aligned
      } else {
        cp_async8_g(dst, src);
        cp_async8_g(reinterpret_cast<float2 *>(dst) + 1, src + 1);
      }
    } else if (rp < rows) {
      cp_async8_g(dst, src);
      reinterpret_cast<float2 *>(dst)[1] = float2{0.f, 0.f};
    } else {
      *dst = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  // scalars of slice b (overlap the staging); MODE 3 (y = G x) has none
  double rho = 0.0;
  if (MODE == 3) {
  } else if (MODE == 0) {
    rho = w.rho[(size_t)b * w.rho_stride + k];
  } else {
    rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
  }
  double alpha = 0.0;
  if (MODE == 3) {
  } else if (MODE == 2) {
    alpha = *w.tau;
  } else {
    const double gam = cta_reduce_parts(w.gpart + (size_t)b * gparts, gparts, red);
    const bool bad = rho > 0 && !(gam > 0);
    const bool frozen = bad || (w.flags && w.flags[b]);
    alpha = (rho > 0 && !frozen) ? rho / gam : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && bad && w.flags) w.flags[b] = 1;
  }
  if (MODE != 3 && blockIdx.x == 0 && threadIdx.x == 0) w.alpha[b] = alpha;
  const float al = (float)alpha;
  asm volatile("cp.async.wait_group 0;\n" ::);
  if (bulk) {  // phase 0 of the staging barrier: every byte of the tile has landed
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar)
          : "memory");
  }
  __syncthreads();
  // row pair (2 warp, 2 warp + 1): Z[q] = X_a[q] + i X_b[q], Z[L - q] = conj X_a[q] + i conj X_b[q]
  float2 v[32];
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    const int q = lane + 32 * rr;
    if (rr < 16 || (rr == 16 && lane == 0)) {  // q <= 512: direct
      float4 e = st[q * RS + warp];
      if (q == 0 || q == L / 2) { e.y = 0.f; e.w = 0.f; }  // DC / Nyquist of real rows
      v[rr] = float2{e.x - e.w, e.y + e.z};
    } else {
      const float4 e = st[(L - q) * RS + warp];
      v[rr] = float2{e.x + e.w, e.z - e.y};
    }
  }
  // this warp's r (x) rows into registers: latency overlaps the FFT below
  const int ra = row0 + 2 * warp;
  const bool ha = ra < N, hb = ra + 1 < N;
  float *r0 = r + ((size_t)b * N + ra) * N, *x0 = x + ((size_t)b * N + ra) * N;
  float rv[2][16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int n = lane + 32 * m;
    rv[0][m] = (MODE != 3 && ha && n < N) ? r0[n] : 0.f;
    rv[1][m] = (MODE != 3 && hb && n < N) ? r0[N + n] : 0.f;
  }
  __syncthreads();  // staging area becomes the transpose buffers
  float2 *tr = reinterpret_cast<float2 *>(smem_raw) + warp * (32 * 33);
  dft32<true>(v);  // over rr: v[a] = U[lane][a]
  twiddle1024<true>(v, tw1024, lane);  // conj W_1024^{a t}
  warp_transpose32(v, tr, lane);  // lane a: v[j] = U[j][a]
  dft32<true>(v);                 // v[m] = z[lane + 32 m] = y_a + i y_b
  // streaming phase: r -= alpha (G d) (and x += alpha r for SD / Landweber)
  float ac = 0.f;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int n = lane + 32 * m;
    if (n < N) {
      if (MODE == 3) {  // y = G x into the r pointer
        if (ha) r0[n] = v[m].x;
        if (hb) r0[N + n] = v[m].y;
        continue;
      }
      if (ha) {
        if (MODE != 0) x0[n] = fmaf(al, rv[0][m], x0[n]);
        const float t = fmaf(-al, v[m].x, rv[0][m]);
        r0[n] = t;
        ac = fmaf(t, t, ac);
      }
      if (hb) {
        if (MODE != 0) x0[N + n] = fmaf(al, rv[1][m], x0[N + n]);
        const float t = fmaf(-al, v[m].y, rv[1][m]);
        r0[N + n] = t;
        ac = fmaf(t, t, ac);
      }
    }
  }
  if (MODE == 3) return;  // y = G x: no partials
  const double s = cta_sum((double)ac, red);
  if (threadIdx.x == 0) w.rpart[((size_t)((k + 1) & 1) * w.B + b) * w.nparts + blockIdx.x] = s;
}

// ---------------------------------------------------------------- pass C, L = 512 (FP32 half-warp FFTs)
// Same contract as cg_pass_c_kernel<float, 512> (32 rows per CTA = the generic pass A's
// partition, so the rpart layout is shared).  T1 staged as in cg_pass_c_1024_kernel ([q][17]
// row-pair float4 slots); each half-warp inverts one row pair with the 16 x 32 four-step FFT of
// pass_b_512_kernel run backwards: lane t takes Z[t + 32 k] and Z[t + 16 + 32 k] (k < 16),
// two inverse DFT_16, conj W_512 twiddles (even-columns-first table), a padded 32 x 17
// transpose, and one inverse DFT_32 forming only z[t + 16 r], r < 16 (N <= 256).
template <int MODE>
__global__ void __launch_bounds__(256, 2) cg_pass_c_512_kernel(int N, int k, int gparts, const float2 *__restrict__ T1,
                                                               float *__restrict__ x, float *__restrict__ r,
                                                               const float2 *__restrict__ tw1024, FusedWork w) {
  constexpr int L = 512, Q = L / 2 + 1, ROWS = 32, NP = ROWS / 2, RS = NP + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float4 *st = reinterpret_cast<float4 *>(smem_raw);  // [Q][RS] row pairs, later [NP][32][17] float2
  __shared__ float2 twl[32 * 32];
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = lane & 15;
  const int pair = 2 * warp + (lane >> 4);
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * ROWS;
  const int rows = min(ROWS, N - row0);
  const float2 *T1s = T1 + (size_t)b * Q * N + row0;
  for (int i = threadIdx.x; i < Q * NP; i += blockDim.x) {
    const int q = i / NP, pr = i % NP, rp = 2 * pr;
    float4 *dst = st + q * RS + pr;
    const float2 *src = T1s + (size_t)q * N + rp;
    if (rp + 1 < rows) {
      if (!(N & 1)) {
        cp_async16_g(dst, src);
      } else {
        cp_async8_g(dst, src);
        cp_async8_g(reinterpret_cast<float2 *>(dst) + 1, src + 1);
      }
    } else if (rp < rows) {
      cp_async8_g(dst, src);
      reinterpret_cast<float2 *>(dst)[1] = float2{0.f, 0.f};
    } else {
      *dst = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {  // layout of pass_b_512_kernel
    const int rr = i >> 5, c = i & 31;
    twl[rr * 32 + (c >> 1) + 16 * (c & 1)] = tw1024[i];
  }
  double rho = 0.0;
  if (MODE == 3) {
  } else if (MODE == 0) {
    rho = w.rho[(size_t)b * w.rho_stride + k];
  } else {
    rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
  }
  double alpha = 0.0;
  if (MODE == 3) {
  } else if (MODE == 2) {
    alpha = *w.tau;
  } else {
    const double gam = cta_reduce_parts(w.gpart + (size_t)b * gparts, gparts, red);
    const bool bad = rho > 0 && !(gam > 0);
    const bool frozen = bad || (w.flags && w.flags[b]);
    alpha = (rho > 0 && !frozen) ? rho / gam : 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && bad && w.flags) w.flags[b] = 1;
  }
  if (MODE != 3 && blockIdx.x == 0 && threadIdx.x == 0) w.alpha[b] = alpha;
  const float al = (float)alpha;
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // Z[q] = X_a[q] + i X_b[q] (q <= 256), Z[L - q] = conj X_a[q] + i conj X_b[q]
  auto zdir = [&](int q) {
    float4 e = st[q * RS + pair];
    if (q == 0 || q == L / 2) { e.y = 0.f; e.w = 0.f; }  // DC / Nyquist of real rows
    return float2{e.x - e.w, e.y + e.z};
  };
  auto zmir = [&](int q) {
    const float4 e = st[(L - q) * RS + pair];
    return float2{e.x + e.w, e.z - e.y};
  };
  float2 a0[16], a1[16];
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    const int q0 = t + 32 * kk, q1 = q0 + 16;
    a0[kk] = (kk < 8 || (kk == 8 && t == 0)) ? zdir(q0) : zmir(q0);
    a1[kk] = kk < 8 ? zdir(q1) : zmir(q1);
  }
  // this half-warp's r (x) rows into registers: latency overlaps the FFT below
  const int ra = row0 + 2 * pair;
  const bool ha = ra < N, hb = ra + 1 < N;
  float *r0 = r + ((size_t)b * N + ra) * N, *x0 = x + ((size_t)b * N + ra) * N;
  float rv[2][16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int n = t + 16 * m;
    rv[0][m] = (MODE != 3 && ha && n < N) ? r0[n] : 0.f;
    rv[1][m] = (MODE != 3 && hb && n < N) ? r0[N + n] : 0.f;
  }
  dft_reg<16, true>(a0);  // over k: a0[tt] = U[j = t][tt]
  dft_reg<16, true>(a1);  // a1[tt] = U[j = t + 16][tt]
#pragma unroll
  for (int tt = 1; tt < 16; ++tt) {
    a0[tt] = cmulc(a0[tt], twl[tt * 64 + (t >> 1) + 16 * (t & 1)]);      // W_512^{t tt}
    a1[tt] = cmulc(a1[tt], twl[tt * 64 + 8 + (t >> 1) + 16 * (t & 1)]);  // W_512^{(t + 16) tt}
  }
  __syncthreads();  // staging area becomes the transpose buffers
  float2 *tr = reinterpret_cast<float2 *>(smem_raw) + pair * (32 * 17);
#pragma unroll
  for (int tt = 0; tt < 16; ++tt) {
    tr[t * 17 + tt] = a0[tt];
    tr[(t + 16) * 17 + tt] = a1[tt];
  }
  __syncwarp();
  float2 v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = tr[j * 17 + t];  // lane t: U[j][t]
  dft32<true>(v);                                       // v[m] = z[t + 16 m] = y_a + i y_b
  float ac = 0.f;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int n = t + 16 * m;
    if (n < N) {
      if (MODE == 3) {  // y = G x into the r pointer
        if (ha) r0[n] = v[m].x;
        if (hb) r0[N + n] = v[m].y;
        continue;
      }
      if (ha) {
        if (MODE != 0) x0[n] = fmaf(al, rv[0][m], x0[n]);
        const float tv = fmaf(-al, v[m].x, rv[0][m]);
        r0[n] = tv;
        ac = fmaf(tv, tv, ac);
      }
      if (hb) {
        if (MODE != 0) x0[N + n] = fmaf(al, rv[1][m], x0[N + n]);
        const float tv = fmaf(-al, v[m].y, rv[1][m]);
        r0[N + n] = tv;
        ac = fmaf(tv, tv, ac);
      }
    }
  }
  if (MODE == 3) return;
  const double s = cta_sum((double)ac, red);
  if (threadIdx.x == 0) w.rpart[((size_t)((k + 1) & 1) * w.B + b) * w.nparts + blockIdx.x] = s;
}

// ---------------------------------------------------------------- pass C, L = 2048 (FP32 warp FFTs)
// Same contract as cg_pass_c_kernel<float, 2048> (8 rows per CTA = the generic pass A's
// partition).  T1[q][row0 .. row0 + 8) staged by cp.async as [q parity][q / 2][5] row-pair
// float4 slots (a warp only reads one parity of q, so consecutive lanes hit consecutive slots);
// two warps per row pair run the inverse of pass_b_2048_kernel's parity split: warp e takes
// Z[2m + e + 64 k] (lane m), IDFT_32 over k, conj W_2048^{(2m + e) t}, transpose, IDFT_32 over
// m, * W_64^{-r e}; the two warps swap halves through their transpose buffers and warp e
// updates r (and x) of row a (e = 0) or b (e = 1) of the pair (z = y_a + i y_b, outputs r < 32
// only: N <= 1024), its r row prefetched into registers before the FFT.
// Tile bx (rows 8 bx .. 8 bx + 7) of slice b; 256 threads; the caller synchronises the CTA
// before reusing smem for another tile.
template <int MODE>
__device__ __forceinline__ void cg_pass_c_2048_tile(int bx, int b, int N, int k, int gparts,
                                                    const float2 *__restrict__ T1, float *__restrict__ x,
                                                    float *__restrict__ r, const float2 *__restrict__ tw2,
                                                    FusedWork w, unsigned char *smem_raw) {
  constexpr int L = 2048, Q = L / 2 + 1, ROWS = 8, NP = ROWS / 2, RS = NP + 1, HALF = L / 4 + 1;
  float4 *st = reinterpret_cast<float4 *>(smem_raw);  // [2][HALF][RS], later [8][32][33] float2
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, e = warp & 1;
  const int row0 = bx * ROWS;
  const int rows = min(ROWS, N - row0);
  const float2 *T1s = T1 + (size_t)b * Q * N + row0;
  auto slot = [&](int q) { return st + ((q & 1) * HALF + (q >> 1)) * RS; };
  for (int i = threadIdx.x; i < Q * NP; i += blockDim.x) {
    const int q = i / NP, pr = i % NP, rp = 2 * pr;
    float4 *dst = slot(q) + pr;
    const float2 *src = T1s + (size_t)q * N + rp;
    if (rp + 1 < rows) {
      if (!(N & 1)) {
        cp_async16_g(dst, src);
      } else {
        cp_async8_g(dst, src);
        cp_async8_g(reinterpret_cast<float2 *>(dst) + 1, src + 1);
      }
    } else if (rp < rows) {
      cp_async8_g(dst, src);
      reinterpret_cast<float2 *>(dst)[1] = float2{0.f, 0.f};
    } else {
      *dst = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  double rho = 0.0;
  if (MODE == 3) {
  } else if (MODE == 0) {
    rho = w.rho[(size_t)b * w.rho_stride + k];
  } else {
    rho = cta_reduce_parts(w.rpart + ((size_t)(k & 1) * w.B + b) * w.nparts, w.nparts, red);
    if (bx == 0 && threadIdx.x == 0) {
      w.rho[(size_t)b * w.rho_stride + k] = rho;
      if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
    }
  }
  double alpha = 0.0;
  if (MODE == 3) {
  } else if (MODE == 2) {
    alpha = *w.tau;
  } else {
    const double gam = cta_reduce_parts(w.gpart + (size_t)b * gparts, gparts, red);
    const bool bad = rho > 0 && !(gam > 0);
    const bool frozen = bad || (w.flags && w.flags[b]);
    alpha = (rho > 0 && !frozen) ? rho / gam : 0.0;
    if (bx == 0 && threadIdx.x == 0 && bad && w.flags) w.flags[b] = 1;
  }
  if (MODE != 3 && bx == 0 && threadIdx.x == 0) w.alpha[b] = alpha;
  const float al = (float)alpha;
  // this warp's row (a for e = 0, b for e = 1) of r into registers: latency overlaps the FFT
  const int row = row0 + 2 * pair + e;
  const bool hr = row < N;
  float *rw = r + ((size_t)b * N + row) * N, *xw = x + ((size_t)b * N + row) * N;
  float rv[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int n = lane + 32 * m;
    rv[m] = (MODE != 3 && hr && n < N) ? rw[n] : 0.f;
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // Z[q] = X_a[q] + i X_b[q] (q <= 1024), Z[L - q] = conj X_a[q] + i conj X_b[q]
  float2 v[32];
#pragma unroll
  for (int kk = 0; kk < 32; ++kk) {
    const int qq = 2 * lane + e + 64 * kk;
    if (kk < 16 || (kk == 16 && qq == L / 2)) {
      float4 c = slot(qq)[pair];
      if (qq == 0 || qq == L / 2) { c.y = 0.f; c.w = 0.f; }  // DC / Nyquist of real rows
      v[kk] = float2{c.x - c.w, c.y + c.z};
    } else {
      const float4 c = slot(L - qq)[pair];
      v[kk] = float2{c.x + c.w, c.z - c.y};
    }
  }
  dft32<true>(v);  // over k: v[t] = U[2 lane + e][t]
twiddle2048_inv(v, tw2, e, lane);  // conj W_2048^{(2 lane + e) t}
  __syncthreads();  // staging area becomes the transpose buffers
  float2 *tr = reinterpret_cast<float2 *>(smem_raw) + warp * (32 * 33);
  warp_transpose32(v, tr, lane);  // lane t: v[m] = U[2m + e][t]
  dft32<true>(v);                 // v[rr] = sum_m U[2m + e][t] W_32^{-rr m}
  if (e) {
#pragma unroll
    for (int rr = 1; rr < 32; ++rr) v[rr] = twiddle64<true>(v[rr], rr);  // W_64^{-rr}
  }
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) tr[rr * 32 + lane] = v[rr];  // hand this half to the other warp
  __syncthreads();
  const float2 *zo = reinterpret_cast<float2 *>(smem_raw) + (warp ^ 1) * (32 * 33);
  float ac = 0.f;
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int n = lane + 32 * m;
    if (hr && n < N) {
      const float2 z = cadd(v[m], zo[m * 32 + lane]);  // z_0 + z_1 = y_a + i y_b at n
      const float zv = e ? z.y : z.x;
      if (MODE == 3) {  // y = G x into the r pointer
        rw[n] = zv;
        continue;
      }
      if (MODE != 0) xw[n] = fmaf(al, rv[m], xw[n]);
      const float tv = fmaf(-al, zv, rv[m]);
      rw[n] = tv;
      ac = fmaf(tv, tv, ac);
    }
  }
  if (MODE == 3) return;
  const double s = cta_sum((double)ac, red);
  if (threadIdx.x == 0) w.rpart[((size_t)((k + 1) & 1) * w.B + b) * w.nparts + bx] = s;
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) cg_pass_c_2048_kernel(int N, int k, int gparts, const float2 *__restrict__ T1,
                                                                float *__restrict__ x, float *__restrict__ r,
                                                                const float2 *__restrict__ tw2, FusedWork w) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg_pass_c_2048_tile<MODE>(blockIdx.x, blockIdx.y, N, k, gparts, T1, x, r, tw2, w, smem_raw);
}

// ---------------------------------------------------------------- final: rho_K, resid, CG x update
template <typename T>
__global__ void __launch_bounds__(256) cg_final_kernel(long n, int K, int cg, T *__restrict__ x,
                                                       const T *__restrict__ p, FusedWork w) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  const double rho = cta_reduce_parts(w.rpart + ((size_t)(K & 1) * w.B + b) * w.nparts, w.nparts, red);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    w.rho[(size_t)b * w.rho_stride + K] = rho;
    if (K > 0 && w.resid) w.resid[(size_t)b * w.iters + K - 1] = sqrt(rho);
  }
  if (!cg || K == 0) return;
  const T al = (T)w.alpha[b];
  const size_t off = (size_t)b * n;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    x[off + i] = fma(al, p[off + i], x[off + i]);
}

// ---------------------------------------------------------------- persistent CG, FP32 L = 2048
// Small batches of large slices (config 4: one 1024^2 slice, 128 pass-A/C tiles and 257
// four-column pass-B tiles per iteration) leave most of the GPU idle between three dependent
// launches.  Opt-in (BSCT_PERSIST=1, measured slower: persist_enabled below): one cooperative
// launch runs all K iterations instead: each CTA loops over the
// tiles of a pass (the same tile functions as the per-pass kernels, so every value, partial
// and scalar is formed exactly as there), and a grid barrier separates the passes.  The whole
// working set (T1 8.4 MB + x, r, p 12.6 MB per slice) stays in L2 across iterations.
constexpr int PERSIST_BCOLS = 4;  // pass-B columns per tile (256 threads)
#ifndef BSCT_PERSIST_UB
#define BSCT_PERSIST_UB 2
#endif
constexpr int PERSIST_UB = BSCT_PERSIST_UB;  // pass-A row batches in flight (4 spills in the persistent kernel)

#ifndef BSCT_PERSIST_MINB
#define BSCT_PERSIST_MINB 2
#endif
template <int VW, bool FULL>
__global__ void __launch_bounds__(256, BSCT_PERSIST_MINB) cg_persist_2048_kernel(int N, int B, int iters, float *__restrict__ x,
                                                                 float *__restrict__ r, float *__restrict__ p,
                                                                 float2 *__restrict__ T1, const float *__restrict__ S,
                                                                 const float2 *__restrict__ tw2, FusedWork w,
                                                                 int gparts, int skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  constexpr int TB = (2048 / 2 + 1 + PERSIST_BCOLS - 1) / PERSIST_BCOLS;  // pass-B tiles per slice
  const int na = w.nparts * B, nb = TB * B;
  for (int k = 0; k < iters; ++k) {
    for (int t = blockIdx.x; t < ((skip & 1) ? 0 : na); t += gridDim.x) {
      cg_pass_a_2048_tile<VW, false, PERSIST_UB>(t % w.nparts, t / w.nparts, N, k, x, r, p, T1, tw2, w, smem_raw);
      __syncthreads();
    }
    grid.sync();
    for (int t = blockIdx.x; t < ((skip & 2) ? 0 : nb); t += gridDim.x) {
      pass_b_2048_tile<FULL, PERSIST_BCOLS>(t % TB, t / TB, gparts, N, T1, S, tw2, w.gpart,
                                            reinterpret_cast<float2 *>(smem_raw));
      __syncthreads();
    }
    grid.sync();
    for (int t = blockIdx.x; t < ((skip & 4) ? 0 : na); t += gridDim.x) {
      cg_pass_c_2048_tile<0>(t % w.nparts, t / w.nparts, N, k, gparts, T1, x, r, tw2, w, smem_raw);
      __syncthreads();
    }
    grid.sync();
  }
}

// ---------------------------------------------------------------- launchers
template <int L>
static int fused_parts_L(int N) {
  constexpr int G = FftLaunch<L>::G;
  return (N + 2 * G - 1) / (2 * G);
}

// rows per CTA of the FP32 L = 1024 warp-FFT passes A and C (2 rows per warp).  Round 1 (whole-
// batch launches, HBM-resident): 16 rows (2 CTAs/SM) 3% faster than 8; round 2 (L2-resident solver
// chunks, api.cu): 8 rows (4 CTAs/SM, more independent tiles per SM) 3% faster (config 5 CG 325 ->
// 315 ms per 2048 x 50, profiles/r02/wrows_ab.txt)
#ifndef BSCT_WROWS
#define BSCT_WROWS 8
#endif
constexpr int WROWS = BSCT_WROWS;

int fused_parts(int N, int L, bool fp32) {
  if (fp32 && L == 1024 && pass_c_warp_enabled()) return (N + WROWS - 1) / WROWS;
  switch (L) {
    case 2: return fused_parts_L<2>(N);
    case 4: return fused_parts_L<4>(N);
    case 8: return fused_parts_L<8>(N);
    case 16: return fused_parts_L<16>(N);
    case 32: return fused_parts_L<32>(N);
    case 64: return fused_parts_L<64>(N);
    case 128: return fused_parts_L<128>(N);
    case 256: return fused_parts_L<256>(N);
    case 512: return fused_parts_L<512>(N);
    case 1024: return fused_parts_L<1024>(N);
    case 2048: return fused_parts_L<2048>(N);
    case 4096: return fused_parts_L<4096>(N);
  }
  return 0;
}

template <int L>
constexpr size_t cg_smem(size_t elem) { return (size_t)FftLaunch<L>::G * FftCfg<L>::SMEM * elem; }

template <typename K>
static cudaError_t cg_set_smem(K kernel, size_t bytes) {
  // dynamic + static shared memory above 48 KB needs the opt-in (the kernels' static parts are ~1-2 KB)
  if (bytes > 40 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

// 16-byte vector accesses need N divisible by the vector width and 16-byte aligned bases
template <typename T>
static bool can_vec(int N, const void *a, const void *b, const void *c) {
  constexpr int VW = 16 / sizeof(T);
  auto al = [](const void *q) { return q == nullptr || ((uintptr_t)q & 15) == 0; };
  return N % VW == 0 && al(a) && al(b) && al(c);
}

// Bulk (TMA, cp.async.bulk) staging of pass C's T1 tile: opt-in (BSCT_BULK=1).  Measured on B200,
// config 5: 117 ms per step vs 97 ms with 16-byte cp.async -- one 128-byte bulk copy per q is too
// small for the bulk-copy path to pay off.
bool bulk_stage_enabled() {
  const char *e = getenv("BSCT_BULK");
  return e && e[0] == '1';
}

bool pass_c_warp_enabled() {
  const char *e = getenv("BSCT_PASSC_V1");  // read per call: tests switch it within one process
  return !(e && e[0] == '1');
}

template <typename T, int L, int VW>
static cudaError_t cg_pass_a_LV(int N, int B, int k, T *x, const T *r, T *p, cplx<T> *T1, const cplx<T> *tw,
                                FusedWork w, cudaStream_t s) {
  const size_t sm = cg_smem<L>(sizeof(cplx<T>));
  cudaError_t e = cg_set_smem(cg_pass_a_kernel<T, L, VW>, sm);
  if (e != cudaSuccess) return e;
  cg_pass_a_kernel<T, L, VW><<<dim3(w.nparts, B), FftLaunch<L>::THREADS, sm, s>>>(N, k, x, r, p, T1, tw, w);
  return cudaGetLastError();
}
template <typename T, int L>
static cudaError_t cg_pass_a_L(int N, int B, int k, T *x, const T *r, T *p, cplx<T> *T1, const cplx<T> *tw,
                               FusedWork w, cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value && L == 1024) {
    if (pass_c_warp_enabled()) {
      const float2 *twl = tw1024_table();
      if (!twl) return cudaErrorMemoryAllocation;
      constexpr size_t sm = sizeof(float4) * (L / 2 + 1) * (WROWS / 2 + 1);
      constexpr size_t sm4 = std::max(sm, sizeof(float) * 3 * WROWS * 512);  // + the cp.async row staging
      if (can_vec<T>(N, x, r, p)) {
        cudaError_t e = cg_set_smem(cg_pass_a_1024_kernel<4, false, WROWS>, sm4);
        if (e != cudaSuccess) return e;
        cg_pass_a_1024_kernel<4, false, WROWS><<<dim3(w.nparts, B), WROWS * 16, sm4, s>>>(N, k, x, r, p, T1, twl, w);
      } else {
        cudaError_t e = cg_set_smem(cg_pass_a_1024_kernel<1, false, WROWS>, sm);
        if (e != cudaSuccess) return e;
        cg_pass_a_1024_kernel<1, false, WROWS><<<dim3(w.nparts, B), WROWS * 16, sm, s>>>(N, k, x, r, p, T1, twl, w);
      }
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value && L == 2048) {
    if (pass_c_warp_enabled()) {
      const float2 *tw2 = tw2048_table();
      if (!tw2) return cudaErrorMemoryAllocation;
      constexpr size_t sm = sizeof(float4) * 2 * (L / 4 + 1) * 5;
      static_assert(sm >= sizeof(float) * 8 * 1032 && sm >= sizeof(float2) * 8 * 32 * 33, "pass A 2048 smem");
      if (can_vec<T>(N, x, r, p)) {
        cudaError_t e = cg_set_smem(cg_pass_a_2048_kernel<4, false>, sm);
        if (e != cudaSuccess) return e;
        cg_pass_a_2048_kernel<4, false><<<dim3(w.nparts, B), 256, sm, s>>>(N, k, x, r, p, T1, tw2, w);
      } else {
        cudaError_t e = cg_set_smem(cg_pass_a_2048_kernel<1, false>, sm);
        if (e != cudaSuccess) return e;
        cg_pass_a_2048_kernel<1, false><<<dim3(w.nparts, B), 256, sm, s>>>(N, k, x, r, p, T1, tw2, w);
      }
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value && L == 512) {
    if (pass_c_warp_enabled()) {
      const float2 *twl = tw1024_table();
      if (!twl) return cudaErrorMemoryAllocation;
      constexpr size_t sm = sizeof(float4) * (L / 2 + 1) * 17;
      static_assert(sm >= sizeof(float) * 32 * 264 && sm >= sizeof(float2) * 16 * 32 * 17, "pass A 512 smem");
      if (can_vec<T>(N, x, r, p)) {
        cudaError_t e = cg_set_smem(cg_pass_a_512_kernel<4, false>, sm);
        if (e != cudaSuccess) return e;
        cg_pass_a_512_kernel<4, false><<<dim3(w.nparts, B), 256, sm, s>>>(N, k, x, r, p, T1, twl, w);
      } else {
        cudaError_t e = cg_set_smem(cg_pass_a_512_kernel<1, false>, sm);
        if (e != cudaSuccess) return e;
        cg_pass_a_512_kernel<1, false><<<dim3(w.nparts, B), 256, sm, s>>>(N, k, x, r, p, T1, twl, w);
      }
      return cudaGetLastError();
    }
  }
  if (can_vec<T>(N, x, r, p)) return cg_pass_a_LV<T, L, 16 / sizeof(T)>(N, B, k, x, r, p, T1, tw, w, s);
  return cg_pass_a_LV<T, L, 1>(N, B, k, x, r, p, T1, tw, w, s);
}

template <typename T, int L, int MODE, int VW>
static cudaError_t cg_pass_c_LMV(int N, int B, int k, int gparts, const cplx<T> *T1, T *x, T *r, const cplx<T> *tw,
                                 FusedWork w, cudaStream_t s) {
  const size_t sm = cg_smem<L>(sizeof(cplx<T>));
  cudaError_t e = cg_set_smem(cg_pass_c_kernel<T, L, MODE, VW>, sm);
  if (e != cudaSuccess) return e;
  cg_pass_c_kernel<T, L, MODE, VW><<<dim3(w.nparts, B), FftLaunch<L>::THREADS, sm, s>>>(N, k, gparts, T1, x, r,
                                                                                         tw, w);
  return cudaGetLastError();
}
template <typename T, int L, int MODE>
static cudaError_t cg_pass_c_LM(int N, int B, int k, int gparts, const cplx<T> *T1, T *x, T *r, const cplx<T> *tw,
                                FusedWork w, cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value && L == 1024) {
    if (pass_c_warp_enabled()) {
      const float2 *twl = tw1024_table();
      if (!twl) return cudaErrorMemoryAllocation;
      constexpr size_t sm = sizeof(float4) * (L / 2 + 1) * (WROWS / 2 + 1);
      cudaError_t e = cg_set_smem(cg_pass_c_1024_kernel<MODE, WROWS>, sm);
      if (e != cudaSuccess) return e;
      cg_pass_c_1024_kernel<MODE, WROWS><<<dim3(w.nparts, B), WROWS * 16, sm, s>>>(N, k, gparts, T1, x, r, twl, w,
                                                                                   bulk_stage_enabled());
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value && L == 2048) {
    static_assert(2 * FftLaunch<2048>::G == 8, "cg_pass_c_2048_kernel covers the generic pass A's 8-row partition");
    if (pass_c_warp_enabled()) {
      const float2 *tw2 = tw2048_table();
      if (!tw2) return cudaErrorMemoryAllocation;
      constexpr size_t sm = sizeof(float4) * 2 * (L / 4 + 1) * 5;
      static_assert(sm >= sizeof(float2) * 8 * 32 * 33, "pass C 2048 smem");
      cudaError_t e = cg_set_smem(cg_pass_c_2048_kernel<MODE>, sm);
      if (e != cudaSuccess) return e;
      cg_pass_c_2048_kernel<MODE><<<dim3(w.nparts, B), 256, sm, s>>>(N, k, gparts, T1, x, r, tw2, w);
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value && L == 512) {
    static_assert(2 * FftLaunch<512>::G == 32, "cg_pass_c_512_kernel covers the generic pass A's 32-row partition");
    if (pass_c_warp_enabled()) {
      const float2 *twl = tw1024_table();
      if (!twl) return cudaErrorMemoryAllocation;
      constexpr size_t sm = sizeof(float4) * (L / 2 + 1) * 17;
      cudaError_t e = cg_set_smem(cg_pass_c_512_kernel<MODE>, sm);
      if (e != cudaSuccess) return e;
      cg_pass_c_512_kernel<MODE><<<dim3(w.nparts, B), 256, sm, s>>>(N, k, gparts, T1, x, r, twl, w);
      return cudaGetLastError();
    }
  }
  if (can_vec<T>(N, x, r, nullptr)) return cg_pass_c_LMV<T, L, MODE, 16 / sizeof(T)>(N, B, k, gparts, T1, x, r, tw, w, s);
  return cg_pass_c_LMV<T, L, MODE, 1>(N, B, k, gparts, T1, x, r, tw, w, s);
}
template <typename T, int L>
static cudaError_t cg_pass_c_L(int N, int B, int k, int mode, int gparts, const cplx<T> *T1, T *x, T *r,
                               const cplx<T> *tw, FusedWork w, cudaStream_t s) {
  switch (mode) {
    case 0: return cg_pass_c_LM<T, L, 0>(N, B, k, gparts, T1, x, r, tw, w, s);
    case 1: return cg_pass_c_LM<T, L, 1>(N, B, k, gparts, T1, x, r, tw, w, s);
    default: return cg_pass_c_LM<T, L, 2>(N, B, k, gparts, T1, x, r, tw, w, s);
  }
}

#define CG_L_SWITCH(L, CALL)                             \
  switch (L) {                                           \
    case 2: { constexpr int LL = 2; CALL; } break;       \
    case 4: { constexpr int LL = 4; CALL; } break;       \
    case 8: { constexpr int LL = 8; CALL; } break;       \
    case 16: { constexpr int LL = 16; CALL; } break;     \
    case 32: { constexpr int LL = 32; CALL; } break;     \
    case 64: { constexpr int LL = 64; CALL; } break;     \
    case 128: { constexpr int LL = 128; CALL; } break;   \
    case 256: { constexpr int LL = 256; CALL; } break;   \
    case 512: { constexpr int LL = 512; CALL; } break;   \
    case 1024: { constexpr int LL = 1024; CALL; } break; \
    case 2048: { constexpr int LL = 2048; CALL; } break; \
    case 4096: { constexpr int LL = 4096; CALL; } break; \
    default: return cudaErrorInvalidValue;               \
  }

template <typename T>
cudaError_t fused_init(int N, int B, const T *b, T *x, T *r, T *p, FusedWork w, cudaStream_t s) {
  cg_init_kernel<T><<<dim3(w.nparts, B), 256, 0, s>>>((long)N * N, b, x, r, p, w);
  return cudaGetLastError();
}
template <typename T>
cudaError_t fused_resume(int N, int B, const T *r_in, const T *p_in, T *r, T *p, T *q, FusedWork w, cudaStream_t s) {
  cg_resume_kernel<T><<<dim3(w.nparts, B), 256, 0, s>>>((long)N * N, r_in, p_in, r, p, q, w);
  return cudaGetLastError();
}
template <typename T>
cudaError_t fused_export(int N, int B, int K, const T *r, const T *p, T *r_out, T *p_out, FusedWork w,
                         cudaStream_t s) {
  const long n = (long)N * N;
  int vb = (int)((n + 2047) / 2048);
  vb = vb < 1 ? 1 : (vb > 128 ? 128 : vb);
  cg_export_kernel<T><<<dim3(vb, B), 256, 0, s>>>(n, K, r, p, r_out, p_out, w);
  return cudaGetLastError();
}
template <typename T>
cudaError_t fused_pass_a(int N, int L, int B, int k, T *x, const T *r, T *p, cplx<T> *T1, const cplx<T> *tw,
                         FusedWork w, cudaStream_t s) {
  CG_L_SWITCH(L, return (cg_pass_a_L<T, LL>(N, B, k, x, r, p, T1, tw, w, s)));
}
template <typename T>
cudaError_t fused_pass_c(int N, int L, int B, int k, int mode, int gparts, const cplx<T> *T1, T *x, T *r,
                         const cplx<T> *tw, FusedWork w, cudaStream_t s) {
  CG_L_SWITCH(L, return (cg_pass_c_L<T, LL>(N, B, k, mode, gparts, T1, x, r, tw, w, s)));
}
template <typename T>
cudaError_t fused_final(int N, int B, int K, int cg, T *x, const T *p, FusedWork w, cudaStream_t s) {
  const long n = (long)N * N;
  int vb = (int)((n + 2047) / 2048);
  vb = vb < 1 ? 1 : (vb > 128 ? 128 : vb);
  cg_final_kernel<T><<<dim3(cg ? vb : 1, B), 256, 0, s>>>(n, K, cg, x, p, w);
  return cudaGetLastError();
}

// y = G x with the warp-FFT passes (FP32, L = 512 or 1024): pass A in PLAIN mode (x -> T1), pass B
// (normal.cu), pass C in MODE 3 (T1 -> y).  Returns cudaErrorNotSupported otherwise.
cudaError_t warp_apply_a(int N, int L, int B, const float *x, float2 *T1, cudaStream_t s) {
  if ((L != 1024 && L != 512 && L != 2048) || !pass_c_warp_enabled()) return cudaErrorNotSupported;
  if (L == 2048) {
    const float2 *tw2 = tw2048_table();
    if (!tw2) return cudaErrorMemoryAllocation;
    constexpr size_t sm2 = sizeof(float4) * 2 * (2048 / 4 + 1) * 5;
    FusedWork w{};
    w.nparts = fused_parts(N, L, true);
    w.B = B;
    float *xp = const_cast<float *>(x);
    if (can_vec<float>(N, x, nullptr, nullptr)) {
      cudaError_t e = cg_set_smem(cg_pass_a_2048_kernel<4, true>, sm2);
      if (e != cudaSuccess) return e;
      cg_pass_a_2048_kernel<4, true><<<dim3(w.nparts, B), 256, sm2, s>>>(N, 0, nullptr, nullptr, xp, T1, tw2, w);
    } else {
      cudaError_t e = cg_set_smem(cg_pass_a_2048_kernel<1, true>, sm2);
      if (e != cudaSuccess) return e;
      cg_pass_a_2048_kernel<1, true><<<dim3(w.nparts, B), 256, sm2, s>>>(N, 0, nullptr, nullptr, xp, T1, tw2, w);
    }
    return cudaGetLastError();
  }
  const float2 *twl = tw1024_table();
  if (!twl) return cudaErrorMemoryAllocation;
  if (L == 512) {
    constexpr size_t sm5 = sizeof(float4) * (512 / 2 + 1) * 17;
    FusedWork w{};
    w.nparts = fused_parts(N, L, true);
    w.B = B;
    float *xp = const_cast<float *>(x);
    if (can_vec<float>(N, x, nullptr, nullptr)) {
      cudaError_t e = cg_set_smem(cg_pass_a_512_kernel<4, true>, sm5);
      if (e != cudaSuccess) return e;
      cg_pass_a_512_kernel<4, true><<<dim3(w.nparts, B), 256, sm5, s>>>(N, 0, nullptr, nullptr, xp, T1, twl, w);
    } else {
      cudaError_t e = cg_set_smem(cg_pass_a_512_kernel<1, true>, sm5);
      if (e != cudaSuccess) return e;
      cg_pass_a_512_kernel<1, true><<<dim3(w.nparts, B), 256, sm5, s>>>(N, 0, nullptr, nullptr, xp, T1, twl, w);
    }
    return cudaGetLastError();
  }
  constexpr size_t sm = sizeof(float4) * (1024 / 2 + 1) * (WROWS / 2 + 1);
  FusedWork w{};
  w.nparts = fused_parts(N, L, true);
  w.B = B;
  float *xp = const_cast<float *>(x);
  if (can_vec<float>(N, x, nullptr, nullptr)) {
    cudaError_t e = cg_set_smem(cg_pass_a_1024_kernel<4, true, WROWS>, sm);
    if (e != cudaSuccess) return e;
    cg_pass_a_1024_kernel<4, true, WROWS><<<dim3(w.nparts, B), WROWS * 16, sm, s>>>(N, 0, nullptr, nullptr, xp, T1, twl, w);
  } else {
    cudaError_t e = cg_set_smem(cg_pass_a_1024_kernel<1, true, WROWS>, sm);
    if (e != cudaSuccess) return e;
    cg_pass_a_1024_kernel<1, true, WROWS><<<dim3(w.nparts, B), WROWS * 16, sm, s>>>(N, 0, nullptr, nullptr, xp, T1, twl, w);
  }
  return cudaGetLastError();
}
cudaError_t warp_apply_c(int N, int L, int B, const float2 *T1, float *y, cudaStream_t s) {
  if ((L != 1024 && L != 512 && L != 2048) || !pass_c_warp_enabled()) return cudaErrorNotSupported;
  if (L == 2048) {
    const float2 *tw2 = tw2048_table();
    if (!tw2) return cudaErrorMemoryAllocation;
    constexpr size_t sm2 = sizeof(float4) * 2 * (2048 / 4 + 1) * 5;
    FusedWork w{};
    w.nparts = fused_parts(N, L, true);
    w.B = B;
    cudaError_t e = cg_set_smem(cg_pass_c_2048_kernel<3>, sm2);
    if (e != cudaSuccess) return e;
    cg_pass_c_2048_kernel<3><<<dim3(w.nparts, B), 256, sm2, s>>>(N, 0, 0, T1, nullptr, y, tw2, w);
    return cudaGetLastError();
  }
  const float2 *twl = tw1024_table();
  if (!twl) return cudaErrorMemoryAllocation;
  if (L == 512) {
    constexpr size_t sm5 = sizeof(float4) * (512 / 2 + 1) * 17;
    FusedWork w{};
    w.nparts = fused_parts(N, L, true);
    w.B = B;
    cudaError_t e = cg_set_smem(cg_pass_c_512_kernel<3>, sm5);
    if (e != cudaSuccess) return e;
    cg_pass_c_512_kernel<3><<<dim3(w.nparts, B), 256, sm5, s>>>(N, 0, 0, T1, nullptr, y, twl, w);
    return cudaGetLastError();
  }
  constexpr size_t sm = sizeof(float4) * (1024 / 2 + 1) * (WROWS / 2 + 1);
  FusedWork w{};
  w.nparts = fused_parts(N, L, true);
  w.B = B;
  cudaError_t e = cg_set_smem(cg_pass_c_1024_kernel<3, WROWS>, sm);
  if (e != cudaSuccess) return e;
  cg_pass_c_1024_kernel<3, WROWS><<<dim3(w.nparts, B), WROWS * 16, sm, s>>>(N, 0, 0, T1, nullptr, y, twl, w,
                                                                             bulk_stage_enabled());
  return cudaGetLastError();
}

#define CG_INST(T)                                                                                               \
  template cudaError_t fused_init<T>(int, int, const T *, T *, T *, T *, FusedWork, cudaStream_t);               \
  template cudaError_t fused_pass_a<T>(int, int, int, int, T *, const T *, T *, cplx<T> *, const cplx<T> *,     \
                                       FusedWork, cudaStream_t);                                               \
  template cudaError_t fused_pass_c<T>(int, int, int, int, int, int, const cplx<T> *, T *, T *, const cplx<T> *, \
                                       FusedWork, cudaStream_t);                                               \
  template cudaError_t fused_final<T>(int, int, int, int, T *, const T *, FusedWork, cudaStream_t);             \
  template cudaError_t fused_resume<T>(int, int, const T *, const T *, T *, T *, T *, FusedWork, cudaStream_t); \
  template cudaError_t fused_export<T>(int, int, int, const T *, const T *, T *, T *, FusedWork, cudaStream_t);
CG_INST(float)
CG_INST(double)

// BSCT_PERSIST=1: run the persistent solver for FP32 L = 2048 CG (opt-in).  Measured slower than
// the per-pass launches replayed from a CUDA graph (config 4, B = 1: 51 vs 24 us per iteration;
// B = 16: 24 vs 17.5 us per slice-iteration; profiles/r02/persist_probe.txt): the three grid
// barriers cost ~4 us per iteration, and the tiles run slower in the fused kernel (one register
// budget for all three passes: spills at 2 CTAs/SM, half the pass-B warps at 1 CTA/SM) than as
// separate kernels, whose own launch gaps the graph already hides.  Single-slice iterations are
// bound by the per-warp latency of the tiles, not by launches.
bool persist_enabled(int L, bool fp32, int B, int solver_cg) {
  (void)B;
  if (!(fp32 && L == 2048 && solver_cg && pass_c_warp_enabled() && pass_b_warp_enabled())) return false;
  const char *e = getenv("BSCT_PERSIST");
  return e && e[0] == '1';
}

cudaError_t persist_cg_2048(int N, int B, int iters, float *x, float *r, float *p, float2 *T1, const float *S,
                            FusedWork w, int gparts, cudaStream_t s) {
  if (N > 1024 || iters <= 0) return iters <= 0 ? cudaSuccess : cudaErrorInvalidValue;
  const float2 *tw2 = tw2048_table();
  if (!tw2) return cudaErrorMemoryAllocation;
  constexpr size_t sm_ac = sizeof(float4) * 2 * (2048 / 4 + 1) * 5;
  constexpr size_t sm = std::max(sm_ac, pass_b_2048_smem<PERSIST_BCOLS>());
  const bool vec = can_vec<float>(N, x, r, p), full = N == 1024;
  void (*kern)(int, int, int, float *, float *, float *, float2 *, const float *, const float2 *, FusedWork, int,
               int) =
      vec ? (full ? cg_persist_2048_kernel<4, true> : cg_persist_2048_kernel<4, false>)
          : (full ? cg_persist_2048_kernel<1, true> : cg_persist_2048_kernel<1, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, sm)) != cudaSuccess) return e;
  if (per < 1) return cudaErrorLaunchOutOfResources;
  constexpr int TB = (2048 / 2 + 1 + PERSIST_BCOLS - 1) / PERSIST_BCOLS;
  const int grid = std::min(per * nsm, std::max(w.nparts * B, TB * B));
  // BSCT_PERSIST_SKIP (timing probes only: the result is wrong): bit 0/1/2 skips the pass A/B/C tiles
  const char *sk = getenv("BSCT_PERSIST_SKIP");
  int skip = sk ? atoi(sk) : 0;
  void *args[] = {&N, &B, &iters, &x, &r, &p, &T1, (void *)&S, (void *)&tw2, &w, &gparts, &skip};
  return cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(256), args, sm, s);
}

}  // namespace bsct
