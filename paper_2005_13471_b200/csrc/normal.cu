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
template <typename T, int L>
static cudaError_t pass_b_L(int N, int B, cplx<T> *T1, const T *S, const cplx<T> *tw, double *gpart, cudaStream_t s) {
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

int pass_b_blocks(int L) {
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
