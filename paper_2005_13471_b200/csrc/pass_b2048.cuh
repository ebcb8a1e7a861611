// pass_b2048.cuh -- the FP32 L = 2048 column pass (pass B of the normal apply) as a
// CTA-tile device function, shared by the per-pass kernel (normal.cu, pass_b_2048_kernel) and
// the persistent single-launch CG solver (cg.cu, cg_persist_2048_kernel).
//
// Two warps per column, 64 x 32 four-step FFT split by the parity e of the first-stage index:
// lane t holds x[t + 32 r] (r < 32: rows >= N <= 1024 are zero), and warp e = 0, 1 computes
//   v[m] = DFT_32 over r of x_r W_64^{r e}          (= Y[2m + e], the half-input DFT_64)
//   * W_2048^{t (2m + e)}, transpose, DFT_32 over t  -> X[2 lane + e + 64 k]
//   * S, Parseval, and the same steps backwards, ending in
//   z_e[t + 32 r] = W_64^{-r e} IDFT_32 over m of U[2m + e][t]
// so only 32 complex values per lane are live; warp 1 hands z_1 to warp 0 through shared
// memory, which stores z_0 + z_1.  Twiddles come from tw2048_table() through L1:
// [e][m][t] = W_2048^{(2m + e) t} (forward, coalesced over t) and [2 + e][t][m] (inverse,
// coalesced over m).
#pragma once
#include "fft32.cuh"

namespace bsct {

// dynamic shared memory of one COLS-column tile: [2 COLS][32 * 33] transposes, [COLS][32 * 32] z_1
template <int COLS>
constexpr size_t pass_b_2048_smem() { return sizeof(float2) * (2 * COLS * 32 * 33 + COLS * 32 * 32); }

// Tile bx of slice b: columns bx * COLS + c (c = warp / 2) of T1, in place; COLS * 64 threads
// (COLS even).  gpart[b * gx + g] (if non-null) receives the Parseval partial of <x, G x> of
// column pair g (gx = (L / 2 + 2) / 2 pairs per slice), summed in the same order for any COLS.
// The caller synchronises the CTA before reusing smem for another tile.
template <bool FULL, int COLS>
__device__ __forceinline__ void pass_b_2048_tile(int bx, int b, int gx, int N, float2 *__restrict__ T1,
                                                 const float *__restrict__ S, const float2 *__restrict__ tw2,
                                                 double *__restrict__ gpart, float2 *smem) {
  constexpr int L = 2048, Q = L / 2 + 1, NWP = 2 * COLS;
  static_assert(COLS % 2 == 0, "partials per column pair");
  __shared__ double red[NWP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = warp >> 1, e = warp & 1;
  const int q0 = bx * COLS + c;
  const bool live = q0 < Q;  // warps past the last column recompute column Q - 1, store nothing
  const int q = live ? q0 : Q - 1;
  float2 *col = T1 + ((size_t)b * Q + q) * N;
  float2 *tr = smem + warp * (32 * 33), *zx = smem + NWP * (32 * 33) + c * (32 * 32);
  const float *Sq = S + (size_t)q * L + 2 * lane + e;
  float2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const int n = lane + 32 * r;
    const float2 xv = (FULL || n < N) ? col[n] : float2{0.f, 0.f};
    v[r] = e ? twiddle64<false>(xv, r) : xv;  // x_r W_64^{r e}
  }
  dft32<false>(v);                   // v[m] = Y[2m + e]
  twiddle2048_fwd(v, tw2, e, lane);  // W_2048^{(2m + e) t}
  warp_transpose32(v, tr, lane);     // lane m: v[t]
  dft32<false>(v);                   // v[k] = X[2 lane + e + 64 k]
  float2 g2[2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float2 w = cscale(v[k], Sq[64 * k]);
    g2[k & 1] = cfma2(w, v[k], g2[k & 1]);
    v[k] = w;
  }
  dft32<true>(v);                    // over k: v[t] = U[2 lane + e][t]
  twiddle2048_inv(v, tw2, e, lane);  // conj W_2048^{(2 lane + e) t}
  warp_transpose32(v, tr, lane);     // lane t: v[m] = U[2m + e][t]
  dft32<true>(v);                    // v[r] = sum_m U[2m + e][t] W_32^{-r m}
  if (e) {
#pragma unroll
    for (int r = 0; r < 32; ++r) zx[r * 32 + lane] = twiddle64<true>(v[r], r);
  }
  __syncthreads();
  if (!e) {
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int n = lane + 32 * r;
      if (live && (FULL || n < N)) col[n] = cadd(v[r], zx[r * 32 + lane]);
    }
  }
  double gam = (double)(g2[0].x + g2[1].x) + (double)(g2[0].y + g2[1].y);
  if (q != 0 && q != L / 2) gam *= 2.0;  // the other half of the Hermitian spectrum
  if (!live) gam = 0.0;
  if (gpart) {  // deterministic reduction per column pair (the same partials for any COLS)
    for (int o = 16; o > 0; o >>= 1) gam += __shfl_xor_sync(0xffffffffu, gam, o);
    if (lane == 0) red[warp] = gam;
    __syncthreads();
    const int g = bx * (COLS / 2) + (warp >> 2);  // column pair of warps 4 (g) .. 4 (g) + 3
    if ((threadIdx.x & 127) == 0 && g < gx) {
      const int w0 = warp;
      gpart[(size_t)b * gx + g] = red[w0] + red[w0 + 1] + red[w0 + 2] + red[w0 + 3];
    }
  }
}

}  // namespace bsct
