// fft.cuh -- register-blocked Stockham FFT in shared memory, power-of-two L <= 4096.
//
// One FFT of length L is computed by a group of P = L/16 threads (P = 1 for L < 16),
// each holding E = 16 (or L) complex values in registers.  Stage s has radix
// R_s = 16 (last stage: 2, 4 or 8) and span Ns = 16^s; butterfly j reads
// X[j + r L/R], multiplies by w_{Ns R}^{r (j mod Ns)}, does an R-point DFT in registers
// and writes Y[(j - j mod Ns) R + j mod Ns + r Ns] (Stockham autosort: natural order
// in and out, no bit reversal).  Shared memory is padded one slot per 16 so that the
// strided stage-0 writes and the Ns-strided reads are bank-conflict free for 8-byte
// (float2) accesses in each half warp.
//
// The paper gives no FFT detail (P:131 only states that Gx is a filter); this is the
// B200 realisation of the zero-padded circulant product (kernel K5).
#pragma once

#include <cmath>

#include "common.cuh"

namespace bsct {

__host__ __device__ constexpr double cos16(int m) {
  m &= 15;
  return m == 0    ? 1.0
         : m == 1  ? 0.92387953251128675613
         : m == 2  ? 0.70710678118654752440
         : m == 3  ? 0.38268343236508977173
         : m == 4  ? 0.0
         : m == 5  ? -0.38268343236508977173
         : m == 6  ? -0.70710678118654752440
         : m == 7  ? -0.92387953251128675613
         : m == 8  ? -1.0
         : m == 9  ? -0.92387953251128675613
         : m == 10 ? -0.70710678118654752440
         : m == 11 ? -0.38268343236508977173
         : m == 12 ? 0.0
         : m == 13 ? 0.38268343236508977173
         : m == 14 ? 0.70710678118654752440
                   : 0.92387953251128675613;
}
__host__ __device__ constexpr double sin16(int m) { return cos16(m - 4); }

// v * exp(-+ 2 pi i m / 16) (forward: minus sign), m compile-time after unrolling.
template <bool INV, typename V>
__device__ __forceinline__ V twiddle16(V v, int m) {
  using S = decltype(v.x);
  if (m == 0) return v;
  if (m == 4) return INV ? V{-v.y, v.x} : V{v.y, -v.x};
  const S c = (S)cos16(m);
  const S s = INV ? (S)sin16(m) : -(S)sin16(m);
  if constexpr (sizeof(S) == 4) return crot(v, c, s);
  else return V{v.x * c - v.y * s, v.x * s + v.y * c};
}

__host__ __device__ constexpr int bitrev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

// In-register R-point DFT (R <= 16), natural order in and out: radix-2 decimation in
// frequency with constant twiddles, then a compile-time bit-reversal permutation.
template <int R, bool INV, typename V>
__device__ __forceinline__ void dft_reg(V *a) {
  if constexpr (R == 1) {
    return;
  } else {
#pragma unroll
    for (int len = R; len >= 2; len >>= 1) {
#pragma unroll
      for (int blk = 0; blk < R; blk += len) {
#pragma unroll
        for (int j = 0; j < len / 2; ++j) {
          V u = a[blk + j], w = a[blk + j + len / 2];
          a[blk + j] = cadd(u, w);
          a[blk + j + len / 2] = twiddle16<INV>(csub(u, w), j * (16 / len));
        }
      }
    }
    V o[R];
#pragma unroll
    for (int i = 0; i < R; ++i) o[bitrev(i, ilog2(R))] = a[i];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = o[i];
  }
}

template <int L>
struct FftCfg {
  static_assert(L >= 2 && L <= 4096 && (L & (L - 1)) == 0, "FFT size must be a power of two in [2, 4096]");
  static constexpr int LOG = ilog2(L);
  static constexpr int E = L < 16 ? L : 16;
  static constexpr int P = L / E;
  static constexpr int NS16 = L < 16 ? 0 : LOG / 4;
  static constexpr int RLAST = L < 16 ? L : (1 << (LOG % 4));
  static constexpr int NSTAGES = L < 16 ? 1 : NS16 + (RLAST > 1 ? 1 : 0);
  static constexpr int SMEM = L + L / 16 + 1;  // padded complex slots per FFT
  __host__ __device__ static constexpr int radix(int s) { return L < 16 ? L : (s < NS16 ? 16 : RLAST); }
  __host__ __device__ static constexpr int span(int s) { return s == 0 ? 1 : 16 * span(s - 1); }
  // offset of stage s's twiddle block tw[r * Ns + k] (stages >= 1)
  __host__ __device__ static constexpr int tw_off(int s) {
    return s <= 1 ? 0 : tw_off(s - 1) + radix(s - 1) * span(s - 1);
  }
  static constexpr int TW_SIZE = tw_off(NSTAGES);
};

__device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }

// Barrier between the stages of one group's FFT.  A group of P <= 32 threads lies inside one
// warp (32 % P == 0), so a warp barrier orders its shared-memory exchanges; larger groups need
// the CTA barrier.  The barrier after the last stage is always CTA-wide: callers read other
// groups' buffers (Hermitian splits).
template <int L>
__device__ __forceinline__ void fft_group_sync() {
  if constexpr (FftCfg<L>::P <= 32) {
    __syncwarp();
  } else {
    __syncthreads();
  }
}

template <typename T, int L, bool INV, int S>
__device__ __forceinline__ void fft_stage(cplx<T> *sm, const cplx<T> *__restrict__ tw, int t) {
  using Cf = FftCfg<L>;
  using V = cplx<T>;
  if constexpr (S < Cf::NSTAGES) {
    constexpr int R = Cf::radix(S);
    constexpr int Ns = Cf::span(S);
    constexpr int NB = Cf::E / R;
    constexpr int STRIDE = L / R;
    V a[Cf::E];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int j = t + u * Cf::P;
#pragma unroll
      for (int r = 0; r < R; ++r) a[u * R + r] = sm[pidx(j + r * STRIDE)];
    }
    fft_group_sync<L>();
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int j = t + u * Cf::P;
      const int k = j & (Ns - 1);
      const V *twb = tw + Cf::tw_off(S) + k;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        V w = twb[r * Ns];
        if (INV) w.y = -w.y;
        a[u * R + r] = cmul(a[u * R + r], w);
      }
      dft_reg<R, INV>(a + u * R);
      const int base = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) sm[pidx(base + r * Ns)] = a[u * R + r];
    }
    if constexpr (S + 1 < Cf::NSTAGES) fft_group_sync<L>();
    else __syncthreads();
    fft_stage<T, L, INV, S + 1>(sm, tw, t);
  }
}

// Group FFT.  On entry v[r] = X[t + r P] (t = thread index in the group, 0 <= t < P).
// On exit sm[pidx(i)] = sum_n X[n] exp(-+2 pi i n i / L) (unnormalised), natural
// order, and the CTA has passed __syncthreads().  Every thread of the CTA must call
// this the same number of times (groups of one CTA run in lockstep).
template <typename T, int L, bool INV>
__device__ __forceinline__ void fft_group(cplx<T> *v, cplx<T> *sm, const cplx<T> *__restrict__ tw, int t) {
  using Cf = FftCfg<L>;
  constexpr int R0 = Cf::radix(0);
  dft_reg<R0, INV>(v);
#pragma unroll
  for (int r = 0; r < R0; ++r) sm[pidx(t * R0 + r)] = v[r];
  if constexpr (1 < FftCfg<L>::NSTAGES) fft_group_sync<L>();
  else __syncthreads();
  fft_stage<T, L, INV, 1>(sm, tw, t);
}

// Host-side twiddle table for FftCfg<L>: tw[off(s) + r*Ns + k] = exp(-2 pi i r k / (Ns R)).
template <int L>
inline void fft_twiddles_host(double *re, double *im) {
  using Cf = FftCfg<L>;
  for (int s = 1; s < Cf::NSTAGES; ++s) {
    const int R = Cf::radix(s), Ns = Cf::span(s), n = Ns * R;
    for (int r = 0; r < R; ++r)
      for (int k = 0; k < Ns; ++k) {
        const long m = ((long)r * k) % n;
        // exact argument reduction: angle = 2 pi m / n
        const long double ang = 6.283185307179586476925286766559L * (long double)m / (long double)n;
        re[Cf::tw_off(s) + r * Ns + k] = (double)cosl(ang);
        im[Cf::tw_off(s) + r * Ns + k] = (double)-sinl(ang);
      }
  }
}

// Number of FFT groups (row pairs / columns) per CTA for size L.
template <int L>
struct FftLaunch {
  static constexpr int P = FftCfg<L>::P;
  static constexpr int G = L <= 256 ? 16 : (L == 512 ? 16 : (L == 1024 ? 8 : 4));
  static constexpr int THREADS = G * P;
};

// Pass B (two FFTs per column, the heaviest register user) uses fewer columns per CTA so
// that several CTAs share an SM and hide each other's barrier stalls.
template <int L>
struct FftLaunchB {
  static constexpr int P = FftCfg<L>::P;
  static constexpr int G = L >= 512 ? 2 : FftLaunch<L>::G;
  static constexpr int THREADS = G * P;
};

}  // namespace bsct
