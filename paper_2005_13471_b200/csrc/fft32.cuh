// fft32.cuh -- warp-level length-1024 FFT for the K5 normal operator, FP32.
//
// One warp computes one length-1024 DFT as a 32 x 32 four-step transform:
//   x[t + 32 r] (lane t, register r) --DFT_32 over r--> * W_1024^{t j} --smem transpose-->
//   (lane j, register t) --DFT_32 over t--> X[j + 32 k] (lane j, register k),
// i.e. natural order in and out in the same lane-strided layout, one shared-memory
// exchange per transform (row stride 33 slots: conflict-free 8-byte accesses per half
// warp) and no block-wide barrier.  The in-register DFT_32 is radix-2 decimation in
// frequency with compile-time twiddles followed by a compile-time bit reversal; inputs a
// caller sets to literal zeros are folded away by the compiler, and outputs it never
// reads are dead code (the zero-padded inputs and cropped outputs of the Toeplitz embedding).
#pragma once

#include <utility>

#include "common.cuh"

namespace bsct {

__host__ __device__ constexpr double cos32(int m) {
  m &= 31;
  if (m > 16) m = 32 - m;  // cos is even
  return m == 0    ? 1.0
         : m == 1  ? 0.98078528040323044913
         : m == 2  ? 0.92387953251128675613
         : m == 3  ? 0.83146961230254523708
         : m == 4  ? 0.70710678118654752440
         : m == 5  ? 0.55557023301960222474
         : m == 6  ? 0.38268343236508977173
         : m == 7  ? 0.19509032201612826785
         : m == 8  ? 0.0
         : m == 9  ? -0.19509032201612826785
         : m == 10 ? -0.38268343236508977173
         : m == 11 ? -0.55557023301960222474
         : m == 12 ? -0.70710678118654752440
         : m == 13 ? -0.83146961230254523708
         : m == 14 ? -0.92387953251128675613
         : m == 15 ? -0.98078528040323044913
                   : -1.0;
}
__host__ __device__ constexpr double sin32(int m) { return cos32(m - 8); }

// v * exp(-+ 2 pi i m / 32) (forward: minus sign); m is a compile-time constant after unrolling
template <bool INV>
__device__ __forceinline__ float2 twiddle32(float2 v, int m) {
  m &= 31;
  if (m == 0) return v;
  if (m == 16) return float2{-v.x, -v.y};
  if (m == 8) return INV ? float2{-v.y, v.x} : float2{v.y, -v.x};
  if (m == 24) return INV ? float2{v.y, -v.x} : float2{-v.y, v.x};
  const float c = (float)cos32(m);
  const float s = INV ? (float)sin32(m) : -(float)sin32(m);
  return crot(v, c, s);
}

__host__ __device__ constexpr int bitrev5(int x) {
  return ((x & 1) << 4) | ((x & 2) << 2) | (x & 4) | ((x & 8) >> 2) | ((x & 16) >> 4);
}

// In-register DFT_32, radix-2 decimation in frequency (the round-1 form, BSCT_DFT32_DIF=1):
// a[k] <- sum_n a[n] exp(-+2 pi i n k / 32), natural order in and out.
// HALF_IN: a[16..31] are zero on entry (the zero-padded half of the Toeplitz embedding);
// the first radix-2 stage then reduces to a twiddle (x + 0 cannot be folded by the
// compiler without fast-math, so the pruning is explicit).
template <bool INV, bool HALF_IN = false>
__device__ __forceinline__ void dft32_dif(float2 *a) {
  if constexpr (HALF_IN) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j + 16] = twiddle32<INV>(a[j], j);
  }
#pragma unroll
  for (int len = HALF_IN ? 16 : 32; len >= 2; len >>= 1) {
#pragma unroll
    for (int blk = 0; blk < 32; blk += len) {
#pragma unroll
      for (int j = 0; j < len / 2; ++j) {
        const float2 u = a[blk + j], w = a[blk + j + len / 2];
        a[blk + j] = cadd(u, w);
        a[blk + j + len / 2] = twiddle32<INV>(csub(u, w), j * (32 / len));
      }
    }
  }
  float2 o[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[bitrev5(i)] = a[i];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = o[i];
}

// Radix-2 butterfly (e + W o, e - W o), W = exp(-+2 pi i M / 32), with the twiddle folded into
// the butterfly (Linzer & Feig's FMA form): for W = c (1 + i t), |t| <= 1,
//   u = (1 + i t) o          one FFMA2 (swapped operand, constants (-t, t))
//   e +- W o = e +- c u      two FFMA2
// and for |s| > |c| the same with W = s i (1 - i t), t = c / s.  A twiddled butterfly is 3 FP32x2
// instructions instead of 4 (complex multiply 2 + add/sub 2); trivial twiddles (M = 0, 8) are 2.
template <bool INV, int M>
__device__ __forceinline__ void bfly32(float2 &e, float2 &o) {
  if constexpr (M == 0) {
    const float2 a = cadd(e, o), b = csub(e, o);
    e = a;
    o = b;
  } else if constexpr (M == 8) {  // W = -i (forward) / +i (inverse)
    const float2 wo = INV ? float2{-o.y, o.x} : float2{o.y, -o.x};
    const float2 a = cadd(e, wo), b = csub(e, wo);
    e = a;
    o = b;
  } else {
    constexpr double cd = cos32(M), sd = INV ? sin32(M) : -sin32(M);
    constexpr bool cmaj = (cd < 0 ? -cd : cd) >= (sd < 0 ? -sd : sd);
#ifdef BSCT_F32X2
    if constexpr (cmaj) {
      constexpr float t = (float)(sd / cd), c = (float)cd;
      const float2 u = x2fma(float2{o.y, o.x}, float2{-t, t}, o), e0 = e;
      e = x2fma(u, float2{c, c}, e0);
      o = x2fma(u, float2{-c, -c}, e0);
    } else {
      constexpr float t = (float)(cd / sd), sv = (float)sd;
      const float2 u = x2fma(float2{o.y, o.x}, float2{t, -t}, o), e0 = e;
      const float2 us{u.y, u.x};
      e = x2fma(us, float2{-sv, sv}, e0);
      o = x2fma(us, float2{sv, -sv}, e0);
    }
#else
    const float2 wo = crot(o, (float)cd, (float)sd);
    const float2 a = cadd(e, wo), b = csub(e, wo);
    e = a;
    o = b;
#endif
  }
}

// one radix-2 DIT stage of butterfly span LEN: butterfly F (0..15) of the stage pairs
// x[blk + j], x[blk + j + LEN / 2] with twiddle index j (32 / LEN)
template <bool INV, int LEN, int F>
__device__ __forceinline__ void dit_bfly(float2 *x) {
  constexpr int H = LEN / 2, blk = (F / H) * LEN, j = F % H;
  bfly32<INV, j * (32 / LEN)>(x[blk + j], x[blk + j + H]);
}
template <bool INV, int LEN, int... F>
__device__ __forceinline__ void dit_stage(float2 *x, std::integer_sequence<int, F...>) {
  (dit_bfly<INV, LEN, F>(x), ...);
}

// In-register DFT_32, radix-2 decimation in time with the twiddles folded into the butterflies
// (bfly32): a[k] <- sum_n a[n] exp(-+2 pi i n k / 32), natural order in and out (the bit reversal
// of the input is register renaming).  194 FP32x2 instructions instead of the DIF form's 228;
// HALF_IN (a[16..31] = 0 on entry): the first stage is a copy (162); outputs a caller never reads
// are dead code (the last stage's e - W o of the output-pruned inverse transforms).
template <bool INV, bool HALF_IN = false>
__device__ __forceinline__ void dft32_dit(float2 *a) {
  float2 x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = a[bitrev5(i)];
  using Seq = std::make_integer_sequence<int, 16>;
  if constexpr (HALF_IN) {  // x[2i + 1] = a[bitrev5(2i) + 16] = 0: the first stage copies
#pragma unroll
    for (int i = 0; i < 16; ++i) x[2 * i + 1] = x[2 * i];
  } else {
    dit_stage<INV, 2>(x, Seq{});
  }
  dit_stage<INV, 4>(x, Seq{});
  dit_stage<INV, 8>(x, Seq{});
  dit_stage<INV, 16>(x, Seq{});
  dit_stage<INV, 32>(x, Seq{});
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = x[i];
}

template <bool INV, bool HALF_IN = false>
__device__ __forceinline__ void dft32(float2 *a) {
#ifdef BSCT_DFT32_DIF
  dft32_dif<INV, HALF_IN>(a);
#else
  dft32_dit<INV, HALF_IN>(a);
#endif
}

// cos(2 pi m / 64), compile-time (the W_64 factors of the L = 2048 parity split)
__host__ __device__ constexpr double cos64(int m) {
  m &= 63;
  if (m > 32) m = 64 - m;  // even
  const bool neg = m > 16;
  if (neg) m = 32 - m;     // cos(pi - a) = -cos(a)
  const double c = m == 0    ? 1.0
         : m == 1  ? 0.99518472667219693
         : m == 2  ? 0.98078528040323043
         : m == 3  ? 0.95694033573220882
         : m == 4  ? 0.92387953251128674
         : m == 5  ? 0.88192126434835505
         : m == 6  ? 0.83146961230254524
         : m == 7  ? 0.77301045336273699
         : m == 8  ? 0.70710678118654757
         : m == 9  ? 0.63439328416364549
         : m == 10 ? 0.55557023301960229
         : m == 11 ? 0.47139673682599781
         : m == 12 ? 0.38268343236508984
         : m == 13 ? 0.29028467725446233
         : m == 14 ? 0.19509032201612833
         : m == 15 ? 0.09801714032956077
                   : 0.0;
  return neg ? -c : c;
}
__host__ __device__ constexpr double sin64(int m) { return cos64(m - 16); }

// v * exp(-+ 2 pi i m / 64), m a compile-time constant after unrolling
template <bool INV>
__device__ __forceinline__ float2 twiddle64(float2 v, int m) {
  m &= 63;
  if (m == 0) return v;
  const float c = (float)cos64(m);
  const float s = INV ? (float)sin64(m) : -(float)sin64(m);
  return crot(v, c, s);
}

// L = 2048 parity-split twiddles from tw2048_table() ([e][m][t] = W_2048^{(2m + e) t} and
// [2 + e][t][m] the same): 8 + 3 table reads per 32 factors instead of 32 --
// W^{(2m + e) t} = [e][4i][t] * W^{2 j t} for m = 4i + j (forward, lane t, register m) and
// W^{(2m + e) t} = [2 + e][4i][m] * W^{(2m + e) j} for t = 4i + j (inverse, lane m, register t).
__device__ __forceinline__ void twiddle2048_fwd(float2 *v, const float2 *__restrict__ tw2, int e, int lane) {
  const float2 r1 = __ldg(tw2 + 1 * 32 + lane), r2 = __ldg(tw2 + 2 * 32 + lane), r3 = __ldg(tw2 + 3 * 32 + lane);
  const float2 *T = tw2 + e * 1024;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 b = __ldg(T + (4 * i) * 32 + lane);
    if (e || i) v[4 * i] = cmul(v[4 * i], b);
    v[4 * i + 1] = cmul(cmul(v[4 * i + 1], b), r1);
    v[4 * i + 2] = cmul(cmul(v[4 * i + 2], b), r2);
    v[4 * i + 3] = cmul(cmul(v[4 * i + 3], b), r3);
  }
}
__device__ __forceinline__ void twiddle2048_inv(float2 *v, const float2 *__restrict__ tw2, int e, int lane) {
  const float2 *T = tw2 + (2 + e) * 1024;
  const float2 s1 = __ldg(T + 1 * 32 + lane), s2 = __ldg(T + 2 * 32 + lane), s3 = __ldg(T + 3 * 32 + lane);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 b = __ldg(T + (4 * i) * 32 + lane);
    if (e || i) v[4 * i] = cmulc(v[4 * i], b);
    v[4 * i + 1] = cmulc(cmulc(v[4 * i + 1], b), s1);
    v[4 * i + 2] = cmulc(cmulc(v[4 * i + 2], b), s2);
    v[4 * i + 3] = cmulc(cmulc(v[4 * i + 3], b), s3);
  }
}

// v[j] *= W_1024^{j t} (INV: conj) for lane t, j = 1..31, from the [32][32] table with 8 + 3
// reads instead of 31: W^{(4i + jj) t} = [4i][t] * [jj][t]
template <bool INV>
__device__ __forceinline__ void twiddle1024(float2 *v, const float2 *__restrict__ tw, int lane) {
  const float2 r1 = __ldg(tw + 1 * 32 + lane), r2 = __ldg(tw + 2 * 32 + lane), r3 = __ldg(tw + 3 * 32 + lane);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 b = __ldg(tw + (4 * i) * 32 + lane);
    if (INV) {
      if (i) v[4 * i] = cmulc(v[4 * i], b);
      v[4 * i + 1] = i ? cmulc(cmulc(v[4 * i + 1], b), r1) : cmulc(v[1], r1);
      v[4 * i + 2] = i ? cmulc(cmulc(v[4 * i + 2], b), r2) : cmulc(v[2], r2);
      v[4 * i + 3] = i ? cmulc(cmulc(v[4 * i + 3], b), r3) : cmulc(v[3], r3);
    } else {
      if (i) v[4 * i] = cmul(v[4 * i], b);
      v[4 * i + 1] = i ? cmul(cmul(v[4 * i + 1], b), r1) : cmul(v[1], r1);
      v[4 * i + 2] = i ? cmul(cmul(v[4 * i + 2], b), r2) : cmul(v[2], r2);
      v[4 * i + 3] = i ? cmul(cmul(v[4 * i + 3], b), r3) : cmul(v[3], r3);
    }
  }
}

// twiddle1024 reading the table through generic loads (e.g. a shared-memory copy)
template <bool INV>
__device__ __forceinline__ void twiddle1024_any(float2 *v, const float2 *tw, int lane) {
  const float2 r1 = tw[1 * 32 + lane], r2 = tw[2 * 32 + lane], r3 = tw[3 * 32 + lane];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 b = tw[(4 * i) * 32 + lane];
    if (INV) {
      if (i) v[4 * i] = cmulc(v[4 * i], b);
      v[4 * i + 1] = i ? cmulc(cmulc(v[4 * i + 1], b), r1) : cmulc(v[1], r1);
      v[4 * i + 2] = i ? cmulc(cmulc(v[4 * i + 2], b), r2) : cmulc(v[2], r2);
      v[4 * i + 3] = i ? cmulc(cmulc(v[4 * i + 3], b), r3) : cmulc(v[3], r3);
    } else {
      if (i) v[4 * i] = cmul(v[4 * i], b);
      v[4 * i + 1] = i ? cmul(cmul(v[4 * i + 1], b), r1) : cmul(v[1], r1);
      v[4 * i + 2] = i ? cmul(cmul(v[4 * i + 2], b), r2) : cmul(v[2], r2);
      v[4 * i + 3] = i ? cmul(cmul(v[4 * i + 3], b), r3) : cmul(v[3], r3);
    }
  }
}

// Warp transpose through shared memory: on entry lane l holds a[i] = M[l][i]; on exit lane l
// holds a[i] = M[i][l].  tr: this warp's [32][33] float2 buffer.
__device__ __forceinline__ void warp_transpose32(float2 *a, float2 *tr, int lane) {
#pragma unroll
  for (int i = 0; i < 32; ++i) tr[i * 33 + lane] = a[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = tr[lane * 33 + i];
  __syncwarp();
}

}  // namespace bsct
