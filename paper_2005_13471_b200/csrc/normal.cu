// normal.cu -- K2 filter spectrum and K5 three-pass FFT normal operator.
//
// y = G x with G Toeplitz-block-Toeplitz is the crop of an L x L circular
// convolution of pad(x) with the circulant embedding E of the taps (L >= 2N-1):
//   pass A  row DFTs of the N nonzero rows of pad(x); two real rows per complex FFT
//           (z = x_a + i x_b, then Hermitian split), output T1[q][row] for q <= L/2
//   pass B  per column q: length-L DFT of the N nonzero entries, times S[q][p]
//           (real: G is even, so its DFT is real), inverse DFT, keep rows < N
//   pass C  per row pair: inverse row DFT (Z = X_a + i X_b), keep columns < N
// The 1/L^2 normalisation is folded into S.  <x, Gx> = sum_q w_q sum_p S|P~|^2
// (Parseval; pad(x) is zero outside the crop) is reduced in pass B for the solvers.
#include "fft.cuh"
#include "fft32.cuh"
#include "pass_b2048.cuh"

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include "kernels.cuh"

namespace bsct {

// ---------------------------------------------------------------- pass A
template <typename T, int L>
__global__ void __launch_bounds__(FftLaunch<L>::THREADS) pass_a_kernel(int N, const T *__restrict__ x,
                                                                       cplx<T> *__restrict__ T1,
                                                                       const cplx<T> *__restrict__ tw) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunch<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * 2 * G;
  const int ra = row0 + 2 * g, rb = ra + 1;
  const T *xs = x + (size_t)b * N * N;
  V v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int j = t + r * P;
    T va = 0, vb = 0;
    if (j < N) {
      if (ra < N) va = xs[(size_t)ra * N + j];
      if (rb < N) vb = xs[(size_t)rb * N + j];
    }
    v[r] = V{va, vb};
  }
  V *sm = smem + g * Cf::SMEM;
  fft_group<T, L, false>(v, sm, tw, t);
  // Hermitian split X_a[q] = (Z[q] + conj Z[-q]) / 2, X_b[q] = -i (Z[q] - conj Z[-q]) / 2
  V *T1s = T1 + (size_t)b * Q * N;
  for (int idx = threadIdx.x; idx < Q * G; idx += blockDim.x) {
    const int q = idx / G, gg = idx % G;
    const int ra2 = row0 + 2 * gg;
    if (ra2 >= N) continue;
    const V *s2 = smem + gg * Cf::SMEM;
    const V z = s2[pidx(q)];
    const V zc = s2[pidx((L - q) & (L - 1))];
    const V xa = V{(T)0.5 * (z.x + zc.x), (T)0.5 * (z.y - zc.y)};
    const V xb = V{(T)0.5 * (z.y + zc.y), (T)0.5 * (zc.x - z.x)};
    T1s[(size_t)q * N + ra2] = xa;
    if (ra2 + 1 < N) T1s[(size_t)q * N + ra2 + 1] = xb;
  }
}

// ---------------------------------------------------------------- pass B
template <typename T, int L>
__global__ void __launch_bounds__(FftLaunchB<L>::THREADS) pass_b_kernel(int N, cplx<T> *__restrict__ T1,
                                                                       const T *__restrict__ S,
                                                                       const cplx<T> *__restrict__ tw,
                                                                       double *__restrict__ gpart) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunchB<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  __shared__ double red[32];
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int b = blockIdx.y;
  const int q = blockIdx.x * G + g;
  const bool qv = q < Q;
  V *col = T1 + ((size_t)b * Q + (qv ? q : 0)) * N;
  V v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int j = t + r * P;
    v[r] = (qv && j < N) ? col[j] : V{0, 0};
  }
  V *sm = smem + g * Cf::SMEM;
  fft_group<T, L, false>(v, sm, tw, t);
  double gam = 0.0;
  const T *Sq = S + (size_t)(qv ? q : 0) * L;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int p = t + r * P;
    const V y = sm[pidx(p)];
    const T sv = qv ? Sq[p] : (T)0;
    gam += (double)sv * ((double)y.x * y.x + (double)y.y * y.y);
    v[r] = V{y.x * sv, y.y * sv};
  }
  if (qv && q != 0 && q != L / 2) gam *= 2.0;  // the other half of the Hermitian spectrum
  __syncthreads();
  fft_group<T, L, true>(v, sm, tw, t);
  if (qv) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = t + r * P;
      if (i < N) col[i] = sm[pidx(i)];
    }
  }
  if (gpart) {  // deterministic CTA reduction
    for (int o = 16; o > 0; o >>= 1) gam += __shfl_xor_sync(0xffffffffu, gam, o);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[wid] = gam;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0;
      for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) s += red[i];
      gpart[(size_t)b * gridDim.x + blockIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------- pass B, L = 1024 (FP32)
// One warp per column q (fft32.cuh): rows >= N of the column are zero (N <= L/2), so the
// first DFT_32 sees 16 literal zeros, and only the N <= 512 kept rows of the inverse are
// formed.  No block-wide barrier; PB_WARPS columns per CTA share the W_1024 table.
constexpr int PB_WARPS = 4;
#ifndef BSCT_PB_CPW
#define BSCT_PB_CPW 2  // measured: pass B 145 -> 139 ms per config-5 step (4: same as 2)
#endif
constexpr int PB_CPW = BSCT_PB_CPW;  // columns per warp (the W_1024 table fill is per CTA)

// FULL: N == L / 2 (every load and store in range, no per-element guards; halves the code the
// compiler emits, which otherwise versions the FFT body on the guards)
template <bool FULL>
__global__ void __launch_bounds__(PB_WARPS * 32, 4) pass_b_1024_kernel(int N, float2 *__restrict__ T1,
                                                                  const float *__restrict__ S,
                                                                  const float2 *__restrict__ tw1024,
                                                                  double *__restrict__ gpart) {
  constexpr int L = 1024, Q = L / 2 + 1;
  __shared__ float2 twl[32 * 32];            // W_1024^{j t}, [j][t] (symmetric)
  __shared__ float2 trs[PB_WARPS][32 * 33];  // per-warp transpose buffers
  __shared__ double red[PB_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) twl[i] = tw1024[i];
  __syncthreads();
  const int b = blockIdx.y;
  // warps past the last column recompute column Q - 1 and store nothing: no branch around the
  // FFT (its __syncwarp transposes in possibly-divergent code made the compiler emit a second,
  // divergent-path copy of the whole body)
  double gam = 0.0;
#pragma unroll 1
  for (int cc = 0; cc < PB_CPW; ++cc) {
    const int q0 = (blockIdx.x * PB_CPW + cc) * PB_WARPS + warp;
    const bool live = q0 < Q;
    const int q = live ? q0 : Q - 1;
    float2 *col = T1 + ((size_t)b * Q + q) * N;
    float2 v[32];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int n = lane + 32 * r;
      v[r] = (FULL || n < N) ? col[n] : float2{0.f, 0.f};
    }
    dft32<false, true>(v);  // over r (v[16..31] = 0): v[j] = sum_r x[lane + 32 r] W_32^{r j}
#pragma unroll
    for (int j = 1; j < 32; ++j) v[j] = cmul(v[j], twl[j * 32 + lane]);
    float2 *tr = trs[warp];
    warp_transpose32(v, tr, lane);  // lane j: v[t]
    dft32<false>(v);                // v[k] = X[lane + 32 k]
    const float *Sq = S + (size_t)q * L + lane;
    // per-lane Parseval partials in FP32 (4 interleaved sums of 8 positive terms each:
    // relative error <= 8 eps), combined in FP64 across lanes and CTAs
    // (packed: g2[k & 1] += (s x, s y) * (x, y), then v = s v)
    float2 g2[2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float2 w = cscale(v[k], Sq[32 * k]);
      g2[k & 1] = cfma2(w, v[k], g2[k & 1]);
      v[k] = w;
    }
    double gc = (double)(g2[0].x + g2[1].x) + (double)(g2[0].y + g2[1].y);
    if (q != 0 && q != L / 2) gc *= 2.0;  // the other half of the Hermitian spectrum
    if (live) gam += gc;
    dft32<true>(v);  // over k: v[a] = U[lane][a]
#pragma unroll
    for (int a = 1; a < 32; ++a) v[a] = cmulc(v[a], twl[a * 32 + lane]);
    warp_transpose32(v, tr, lane);  // lane a: v[j] = U[j][a]
    dft32<true>(v);                 // v[m] = z[lane + 32 m]
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int n = lane + 32 * m;
      if (live && (FULL || n < N)) col[n] = v[m];
    }
  }
  if (gpart) {  // deterministic CTA reduction
    for (int o = 16; o > 0; o >>= 1) gam += __shfl_xor_sync(0xffffffffu, gam, o);
    if (lane == 0) red[warp] = gam;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int i = 0; i < PB_WARPS; ++i) t += red[i];
      gpart[(size_t)b * gridDim.x + blockIdx.x] = t;
    }
  }
}

// ---------------------------------------------------------------- pass B, L = 2048 (FP32)
// Two warps per column (pass_b2048.cuh), PB2_COLS columns per CTA.
constexpr int PB2_COLS = 2;  // columns per CTA (2 warps each)

template <bool FULL>
__global__ void __launch_bounds__(PB2_COLS * 64, 4) pass_b_2048_kernel(int N, float2 *__restrict__ T1,
                                                                     const float *__restrict__ S,
                                                                     const float2 *__restrict__ tw2,
                                                                     double *__restrict__ gpart) {
  extern __shared__ __align__(16) float2 pb2_smem[];
  pass_b_2048_tile<FULL, PB2_COLS>(blockIdx.x, blockIdx.y, gridDim.x, N, T1, S, tw2, gpart, pb2_smem);
}

// ---------------------------------------------------------------- pass B, L = 512 (FP32)
// Half-warp 16 x 32 four-step FFT per column (two columns per warp): lane t < 16 holds
// x[t + 16 r] (r < 32; rows >= N <= 256 are zero, so r < 16), DFT_32 over r in registers,
// twiddle W_512^{t j} (= W_1024^{2 t j}, the L = 1024 table), a padded 32 x 17 transpose so that
// lane t holds columns j = t and t + 16, two in-register DFT_16 over t: X[j + 32 k].  The inverse
// runs the steps backwards and forms only the first N <= 256 outputs.
#ifndef BSCT_PB5_WARPS
#define BSCT_PB5_WARPS 4
#endif
#ifndef BSCT_PB5_MINB
#define BSCT_PB5_MINB 4
#endif
constexpr int PB5_WARPS = BSCT_PB5_WARPS;
#ifndef BSCT_PB5_CPW
#define BSCT_PB5_CPW 2
#endif
constexpr int PB5_CPW = BSCT_PB5_CPW;

template <bool FULL>
__global__ void __launch_bounds__(PB5_WARPS * 32, BSCT_PB5_MINB) pass_b_512_kernel(int N, float2 *__restrict__ T1,
                                                                     const float *__restrict__ S,
                                                                     const float2 *__restrict__ tw1024,
                                                                     double *__restrict__ gpart) {
  constexpr int L = 512, Q = L / 2 + 1;
  __shared__ float2 twl[32 * 32];
  __shared__ float2 trs[PB5_WARPS][2][32 * 17];
  __shared__ double red[PB5_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, t = lane & 15;
  // twl holds W_1024^{r c} (symmetric in r, c) with each row's even columns first: entry (r, c)
  // at r * 32 + (c >> 1) + 16 * (c & 1), so that both W_512^{t j} = (j, 2t) over lanes t (forward)
  // and W_512^{j tt} = (2 tt, j) over lanes j = t or t + 16 (inverse) hit 16 distinct bank pairs
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
    const int r = i >> 5, c = i & 31;
    twl[r * 32 + (c >> 1) + 16 * (c & 1)] = tw1024[i];
  }
  __syncthreads();
  const int b = blockIdx.y;
  double gam = 0.0;
#pragma unroll 1
  for (int cc = 0; cc < PB5_CPW; ++cc) {  // columns per half-warp (the table fill is per CTA)
    const int q0 = ((blockIdx.x * PB5_CPW + cc) * PB5_WARPS + warp) * 2 + h;
    const bool live = q0 < Q;  // the last half-warps recompute column Q - 1 and store nothing
    const int q = live ? q0 : Q - 1;
    float2 *col = T1 + ((size_t)b * Q + q) * N;
    float2 *tr = trs[warp][h];
    float2 v[32];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int n = t + 16 * r;
      v[r] = (FULL || n < N) ? col[n] : float2{0.f, 0.f};
    }
    dft32<false, true>(v);  // v[j] = sum_r x[t + 16 r] W_32^{r j}
#pragma unroll
    for (int j = 1; j < 32; ++j) v[j] = cmul(v[j], twl[j * 32 + t]);  // W_512^{t j} = entry (j, 2t)
#pragma unroll
    for (int j = 0; j < 32; ++j) tr[j * 17 + t] = v[j];
    __syncwarp();
    float2 a0[16], a1[16];
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) {
      a0[tt] = tr[t * 17 + tt];
      a1[tt] = tr[(t + 16) * 17 + tt];
    }
    __syncwarp();
    dft_reg<16, false>(a0);  // a0[k] = X[t + 32 k]
    dft_reg<16, false>(a1);  // a1[k] = X[t + 16 + 32 k]
    const float *Sq = S + (size_t)q * L;
    float2 g2[2] = {{0.f, 0.f}, {0.f, 0.f}};  // packed Parseval partials, as in pass_b_1024_kernel
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float2 w0 = cscale(a0[k], Sq[t + 32 * k]), w1 = cscale(a1[k], Sq[t + 16 + 32 * k]);
      g2[0] = cfma2(w0, a0[k], g2[0]);
      g2[1] = cfma2(w1, a1[k], g2[1]);
      a0[k] = w0;
      a1[k] = w1;
    }
    double gc = (double)(g2[0].x + g2[1].x) + (double)(g2[0].y + g2[1].y);
    if (q != 0 && q != L / 2) gc *= 2.0;  // the other half of the Hermitian spectrum
    if (live) gam += gc;
    dft_reg<16, true>(a0);  // a0[tt] = U[j = t][tt]
    dft_reg<16, true>(a1);  // a1[tt] = U[j = t + 16][tt]
#pragma unroll
    for (int tt = 1; tt < 16; ++tt) {
      a0[tt] = cmulc(a0[tt], twl[tt * 64 + (t >> 1) + 16 * (t & 1)]);       // entry (2 tt, t)
      a1[tt] = cmulc(a1[tt], twl[tt * 64 + 8 + (t >> 1) + 16 * (t & 1)]);   // entry (2 tt, t + 16)
    }
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) {
      tr[t * 17 + tt] = a0[tt];
      tr[(t + 16) * 17 + tt] = a1[tt];
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = tr[j * 17 + t];  // lane t: U[j][t]
    __syncwarp();
    dft32<true>(v);  // v[r] = z[t + 16 r]
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int n = t + 16 * r;
      if (live && (FULL || n < N)) col[n] = v[r];
    }
  }
  if (gpart) {  // deterministic CTA reduction
    for (int o = 16; o > 0; o >>= 1) gam += __shfl_xor_sync(0xffffffffu, gam, o);
    if (lane == 0) red[warp] = gam;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0;
      for (int i = 0; i < PB5_WARPS; ++i) tot += red[i];
      gpart[(size_t)b * gridDim.x + blockIdx.x] = tot;
    }
  }
}

// ---------------------------------------------------------------- pass C
template <typename T, int L>
__global__ void __launch_bounds__(FftLaunch<L>::THREADS) pass_c_kernel(int N, const cplx<T> *__restrict__ T1,
                                                                       T *__restrict__ y,
                                                                       const cplx<T> *__restrict__ tw) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunch<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * 2 * G;
  const V *T1s = T1 + (size_t)b * Q * N;
  // Z[q] = X_a[q] + i X_b[q] (q <= L/2), Z[L-q] = conj X_a[q] + i conj X_b[q]
  for (int idx = threadIdx.x; idx < Q * G; idx += blockDim.x) {
    const int q = idx / G, gg = idx % G;
    const int ra2 = row0 + 2 * gg;
    V xa = V{0, 0}, xb = V{0, 0};
    if (ra2 < N) {
      xa = T1s[(size_t)q * N + ra2];
      if (ra2 + 1 < N) xb = T1s[(size_t)q * N + ra2 + 1];
    }
    if (q == 0 || q == L / 2) { xa.y = 0; xb.y = 0; }  // real rows: DC and Nyquist are real
    V *s2 = smem + gg * Cf::SMEM;
    s2[pidx(q)] = V{xa.x - xb.y, xa.y + xb.x};
    if (q != 0 && q != L / 2) s2[pidx(L - q)] = V{xa.x + xb.y, xb.x - xa.y};
  }
  __syncthreads();
  V *sm = smem + g * Cf::SMEM;
  V v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = sm[pidx(t + r * P)];
  __syncthreads();
  fft_group<T, L, true>(v, sm, tw, t);
  const int ra = row0 + 2 * g, rb = ra + 1;
  T *ys = y + (size_t)b * N * N;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int n = t + r * P;
    if (n < N) {
      const V z = sm[pidx(n)];
      if (ra < N) ys[(size_t)ra * N + n] = z.x;
      if (rb < N) ys[(size_t)rb * N + n] = z.y;
    }
  }
}

// ---------------------------------------------------------------- spectrum (K2)
// rows of the L x L embedding E[i][j] = taps[i'][j'] for |i'|,|j'| <= N-1 (i = i' mod L)
template <typename T, int L>
__global__ void __launch_bounds__(FftLaunch<L>::THREADS) spec_rows_kernel(int N, const T *__restrict__ taps,
                                                                          cplx<T> *__restrict__ W,
                                                                          const cplx<T> *__restrict__ tw) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunch<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int row0 = blockIdx.x * 2 * G;
  const int D = 2 * N - 1;
  auto tap_index = [&](int i) -> int {  // embedding row/col -> tap index, -1 if zero
    if (i >= L) return -1;
    if (i <= N - 1) return i + N - 1;
    if (i >= L - (N - 1)) return i - L + N - 1;
    return -1;
  };
  const int ia = tap_index(row0 + 2 * g), ib = tap_index(row0 + 2 * g + 1);
  V v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int jj = tap_index(t + r * P);
    T va = 0, vb = 0;
    if (jj >= 0) {
      if (ia >= 0) va = taps[(size_t)ia * D + jj];
      if (ib >= 0) vb = taps[(size_t)ib * D + jj];
    }
    v[r] = V{va, vb};
  }
  V *sm = smem + g * Cf::SMEM;
  fft_group<T, L, false>(v, sm, tw, t);
  for (int idx = threadIdx.x; idx < Q * G; idx += blockDim.x) {
    const int q = idx / G, gg = idx % G;
    const int ra2 = row0 + 2 * gg;
    if (ra2 >= L) continue;
    const V *s2 = smem + gg * Cf::SMEM;
    const V z = s2[pidx(q)];
    const V zc = s2[pidx((L - q) & (L - 1))];
    W[(size_t)q * L + ra2] = V{(T)0.5 * (z.x + zc.x), (T)0.5 * (z.y - zc.y)};
    W[(size_t)q * L + ra2 + 1] = V{(T)0.5 * (z.y + zc.y), (T)0.5 * (zc.x - z.x)};
  }
}

template <typename T, int L>
__global__ void __launch_bounds__(FftLaunch<L>::THREADS) spec_cols_kernel(const cplx<T> *__restrict__ W,
                                                                          T *__restrict__ S,
                                                                          const cplx<T> *__restrict__ tw) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  constexpr int G = FftLaunch<L>::G, P = Cf::P, E = Cf::E, Q = L / 2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *smem = reinterpret_cast<V *>(smem_raw);
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  const int q = blockIdx.x * G + g;
  const bool qv = q < Q;
  V v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = qv ? W[(size_t)q * L + t + r * P] : V{0, 0};
  V *sm = smem + g * Cf::SMEM;
  fft_group<T, L, false>(v, sm, tw, t);
  const T scale = (T)(1.0 / ((double)L * (double)L));
  if (qv) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int p = t + r * P;
      S[(size_t)q * L + p] = sm[pidx(p)].x * scale;
    }
  }
}

// ---------------------------------------------------------------- dispatch
template <int L>
constexpr size_t fft_smem_bytes(size_t elem) { return (size_t)FftLaunch<L>::G * FftCfg<L>::SMEM * elem; }

template <typename K>
static cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

#define BSCT_L_SWITCH(L, CALL)          \
  switch (L) {                          \
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

template <typename T, int L>
static cudaError_t pass_a_L(int N, int B, const T *x, cplx<T> *T1, const cplx<T> *tw, cudaStream_t s) {
  constexpr int G = FftLaunch<L>::G;
  const size_t sm = fft_smem_bytes<L>(sizeof(cplx<T>));
  cudaError_t e = set_smem(pass_a_kernel<T, L>, sm);
  if (e != cudaSuccess) return e;
  dim3 grid((N + 2 * G - 1) / (2 * G), B);
  pass_a_kernel<T, L><<<grid, FftLaunch<L>::THREADS, sm, s>>>(N, x, T1, tw);
  return cudaGetLastError();
}
// W_1024^{j t} for j, t < 32 ([32][32], FP32 rounded from long double), one copy per device,
// uploaded on first use (outside any stream capture: plan creation runs pass B once).
const float2 *tw1024_table() {
  static float2 *tab[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!tab[dev]) {
    float2 h[32 * 32];
    for (int j = 0; j < 32; ++j)
      for (int t = 0; t < 32; ++t) {
        const long double ang = 6.283185307179586476925286766559L * (long double)((j * t) % 1024) / 1024.0L;
        h[j * 32 + t] = float2{(float)cosl(ang), (float)-sinl(ang)};
      }
    float2 *d = nullptr;
    if (cudaMalloc((void **)&d, sizeof(h)) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    tab[dev] = d;
  }
  return tab[dev];
}

// [4][32][32]: [e][m][t] = W_2048^{(2m + e) t}, [2 + e][t][m] = the same for the inverse reads
const float2 *tw2048_table() {
  static float2 *tab[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!tab[dev]) {
    static float2 h[4 * 32 * 32];
    for (int e = 0; e < 2; ++e)
      for (int m = 0; m < 32; ++m)
        for (int t = 0; t < 32; ++t) {
          const long double ang = 6.283185307179586476925286766559L * (long double)(((2 * m + e) * t) % 2048) / 2048.0L;
          const float2 w{(float)cosl(ang), (float)-sinl(ang)};
          h[(e * 32 + m) * 32 + t] = w;
          h[((2 + e) * 32 + t) * 32 + m] = w;
        }
    float2 *d = nullptr;
    if (cudaMalloc((void **)&d, sizeof(h)) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    tab[dev] = d;
  }
  return tab[dev];
}

template <typename T, int L>
static cudaError_t pass_b_L(int N, int B, cplx<T> *T1, const T *S, const cplx<T> *tw, double *gpart, cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value && L == 1024) {
    const float2 *twl = tw1024_table();
    if (!twl) return cudaErrorMemoryAllocation;
    if (pass_b_warp_enabled()) {
      const dim3 grid((L / 2 + 1 + PB_WARPS * PB_CPW - 1) / (PB_WARPS * PB_CPW), B);
      if (N == L / 2)
        pass_b_1024_kernel<true><<<grid, PB_WARPS * 32, 0, s>>>(N, T1, S, twl, gpart);
      else
        pass_b_1024_kernel<false><<<grid, PB_WARPS * 32, 0, s>>>(N, T1, S, twl, gpart);
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value && L == 2048) {
    if (pass_b_warp_enabled()) {
      const float2 *tw2 = tw2048_table();
      if (!tw2) return cudaErrorMemoryAllocation;
      const dim3 grid((L / 2 + 1 + PB2_COLS - 1) / PB2_COLS, B);
      constexpr size_t sm = pass_b_2048_smem<PB2_COLS>();
      cudaError_t e = set_smem(pass_b_2048_kernel<true>, sm);
      if (e == cudaSuccess) e = set_smem(pass_b_2048_kernel<false>, sm);
      if (e != cudaSuccess) return e;
      if (N == L / 2)
        pass_b_2048_kernel<true><<<grid, PB2_COLS * 64, sm, s>>>(N, T1, S, tw2, gpart);
      else
        pass_b_2048_kernel<false><<<grid, PB2_COLS * 64, sm, s>>>(N, T1, S, tw2, gpart);
      return cudaGetLastError();
    }
  }
  if constexpr (std::is_same<T, float>::value && L == 512) {
    const float2 *twl = tw1024_table();
    if (!twl) return cudaErrorMemoryAllocation;
    if (pass_b_warp_enabled()) {
      const dim3 grid((L / 2 + 1 + 2 * PB5_WARPS * PB5_CPW - 1) / (2 * PB5_WARPS * PB5_CPW), B);
      if (N == L / 2)
        pass_b_512_kernel<true><<<grid, PB5_WARPS * 32, 0, s>>>(N, T1, S, twl, gpart);
      else
        pass_b_512_kernel<false><<<grid, PB5_WARPS * 32, 0, s>>>(N, T1, S, twl, gpart);
      return cudaGetLastError();
    }
  }
  constexpr int G = FftLaunchB<L>::G;
  const size_t sm = (size_t)G * FftCfg<L>::SMEM * sizeof(cplx<T>);
  cudaError_t e = set_smem(pass_b_kernel<T, L>, sm);
  if (e != cudaSuccess) return e;
  dim3 grid((L / 2 + 1 + G - 1) / G, B);
  pass_b_kernel<T, L><<<grid, FftLaunchB<L>::THREADS, sm, s>>>(N, T1, S, tw, gpart);
  return cudaGetLastError();
}
template <typename T, int L>
static cudaError_t pass_c_L(int N, int B, const cplx<T> *T1, T *y, const cplx<T> *tw, cudaStream_t s) {
  constexpr int G = FftLaunch<L>::G;
  const size_t sm = fft_smem_bytes<L>(sizeof(cplx<T>));
  cudaError_t e = set_smem(pass_c_kernel<T, L>, sm);
  if (e != cudaSuccess) return e;
  dim3 grid((N + 2 * G - 1) / (2 * G), B);
  pass_c_kernel<T, L><<<grid, FftLaunch<L>::THREADS, sm, s>>>(N, T1, y, tw);
  return cudaGetLastError();
}
template <typename T, int L>
static cudaError_t spectrum_L(int N, const T *taps, T *S, cplx<T> *work, const cplx<T> *tw, cudaStream_t s) {
  constexpr int G = FftLaunch<L>::G;
  const size_t sm = fft_smem_bytes<L>(sizeof(cplx<T>));
  cudaError_t e = set_smem(spec_rows_kernel<T, L>, sm);
  if (e != cudaSuccess) return e;
  e = set_smem(spec_cols_kernel<T, L>, sm);
  if (e != cudaSuccess) return e;
  spec_rows_kernel<T, L><<<(L + 2 * G - 1) / (2 * G), FftLaunch<L>::THREADS, sm, s>>>(N, taps, work, tw);
  spec_cols_kernel<T, L><<<(L / 2 + 1 + G - 1) / G, FftLaunch<L>::THREADS, sm, s>>>(work, S, tw);
  return cudaGetLastError();
}

bool pass_b_warp_enabled() {
  const char *e = getenv("BSCT_PASSB_V1");  // read per call: tests switch it within one process
  return !(e && e[0] == '1');
}

int pass_b_blocks(int L, bool fp32) {
  if (fp32 && L == 1024 && pass_b_warp_enabled()) return (1024 / 2 + 1 + PB_WARPS * PB_CPW - 1) / (PB_WARPS * PB_CPW);
  if (fp32 && L == 512 && pass_b_warp_enabled()) return (512 / 2 + 1 + 2 * PB5_WARPS * PB5_CPW - 1) / (2 * PB5_WARPS * PB5_CPW);
  if (fp32 && L == 2048 && pass_b_warp_enabled()) return (2048 / 2 + 1 + PB2_COLS - 1) / PB2_COLS;
  switch (L) {
    case 2: return (2 / 2 + 1 + FftLaunchB<2>::G - 1) / FftLaunchB<2>::G;
    case 4: return (4 / 2 + 1 + FftLaunchB<4>::G - 1) / FftLaunchB<4>::G;
    case 8: return (8 / 2 + 1 + FftLaunchB<8>::G - 1) / FftLaunchB<8>::G;
    case 16: return (16 / 2 + 1 + FftLaunchB<16>::G - 1) / FftLaunchB<16>::G;
    case 32: return (32 / 2 + 1 + FftLaunchB<32>::G - 1) / FftLaunchB<32>::G;
    case 64: return (64 / 2 + 1 + FftLaunchB<64>::G - 1) / FftLaunchB<64>::G;
    case 128: return (128 / 2 + 1 + FftLaunchB<128>::G - 1) / FftLaunchB<128>::G;
    case 256: return (256 / 2 + 1 + FftLaunchB<256>::G - 1) / FftLaunchB<256>::G;
    case 512: return (512 / 2 + 1 + FftLaunchB<512>::G - 1) / FftLaunchB<512>::G;
    case 1024: return (1024 / 2 + 1 + FftLaunchB<1024>::G - 1) / FftLaunchB<1024>::G;
    case 2048: return (2048 / 2 + 1 + FftLaunchB<2048>::G - 1) / FftLaunchB<2048>::G;
    case 4096: return (4096 / 2 + 1 + FftLaunchB<4096>::G - 1) / FftLaunchB<4096>::G;
  }
  return 0;
}

template <typename T>
cudaError_t pass_a(int N, int L, int B, const T *x, cplx<T> *T1, const cplx<T> *tw, cudaStream_t s) {
  BSCT_L_SWITCH(L, return (pass_a_L<T, LL>(N, B, x, T1, tw, s)));
}
template <typename T>
cudaError_t pass_b(int N, int L, int B, cplx<T> *T1, const T *S, const cplx<T> *tw, double *gpart, cudaStream_t s) {
  BSCT_L_SWITCH(L, return (pass_b_L<T, LL>(N, B, T1, S, tw, gpart, s)));
}
template <typename T>
cudaError_t pass_c(int N, int L, int B, const cplx<T> *T1, T *y, const cplx<T> *tw, cudaStream_t s) {
  BSCT_L_SWITCH(L, return (pass_c_L<T, LL>(N, B, T1, y, tw, s)));
}
template <typename T>
cudaError_t filter_spectrum(int N, int L, const T *taps, T *S, cplx<T> *work, const cplx<T> *tw, cudaStream_t s) {
  BSCT_L_SWITCH(L, return (spectrum_L<T, LL>(N, taps, S, work, tw, s)));
}

#define BSCT_INST(T)                                                                                         \
  template cudaError_t pass_a<T>(int, int, int, const T *, cplx<T> *, const cplx<T> *, cudaStream_t);        \
  template cudaError_t pass_b<T>(int, int, int, cplx<T> *, const T *, const cplx<T> *, double *,             \
                                 cudaStream_t);                                                              \
  template cudaError_t pass_c<T>(int, int, int, const cplx<T> *, T *, const cplx<T> *, cudaStream_t);        \
  template cudaError_t filter_spectrum<T>(int, int, const T *, T *, cplx<T> *, const cplx<T> *, cudaStream_t);
BSCT_INST(float)
BSCT_INST(double)

}  // namespace bsct
