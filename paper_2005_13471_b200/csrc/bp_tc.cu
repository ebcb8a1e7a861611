// bp_tc.cu -- K4 v4: the back projection b = H^T g^ on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, accumulator in TMEM, operands staged by TMA and by the CTA).
//
// Per angle t the back projection of a pixel is a short dot product with the corrected
// sinogram row (K4 v1-v3):
//     b_s[k] += sum_i g~_s[c_k + imin + i] Q_{p_k, i}(tau_k),   i = 0 .. S-1,
// where (c_k, p_k, tau_k) locate pixel k's detector coordinate u_k = <theta_perp, x_k>/lambda_y
// (cell, sub-interval, local coordinate) and Q_{p,i} are the degree-5 basis polynomials of the
// box spline C_t = M_[l|c|, l|s|, zeta] U [lambda_y]^(d+1) (bp_tables_kernel).  For a tile of
// 128 pixels (8 x 16) every pixel's samples lie in one window of K = 32 consecutive detector
// samples [m_lo, m_lo + 32), so for SB = 128 slices at once the angle's contribution is a
// dense product
//     D[pixel][slice] += W_t[pixel][j] G_t[j][slice],   W_t[k][j] = Q_{p_k, j + m_lo - c_k - imin}(tau_k)
// (zero outside the pixel's S samples), M = 128, N = 128, K = 32: four tcgen05.mma K-steps per
// angle.  FP32 accuracy from TF32 inputs by the 3xTF32 split: W = W_hi + W_lo and
// G = G_hi + G_lo with W_hi, G_hi rounded to TF32 (cvt.rna.tf32) and the lo parts exact FP32
// residuals; D += W_hi G_hi + W_hi G_lo + W_lo G_hi (the dropped W_lo G_lo is <= 2^-22 |W||G|).
// Accumulation in FP32 in TMEM over all angles, in angle order (fixed: deterministic).
//
// Roles (192 threads, one CTA per SM, NS-stage smem ring):
//   warps 0-3  one thread per pixel: locate, evaluate the S basis polynomials (Horner on the
//              angle's basis table), write the W_hi / W_lo rows in the canonical K-major
//              SWIZZLE_128B layout, fence.proxy.async, arrive on full_w[s]; epilogue:
//              tcgen05.ld of the pixel's TMEM lane (128 slice columns) -> b.
//   warp 4     TMA producer: G_hi / G_lo tiles [128 slices][32 samples] of the angle by
//              cp.async.bulk.tensor (3-D maps over g~_hi / g~_lo, SWIZZLE_128B, zero fill outside
//              the detector and the batch), completion counted on full_g[s].
//   warp 5     TMEM allocation; one elected thread issues the 12 MMAs per angle and
//              tcgen05.commit -> empty[s] (releases the stage) / done (after the last angle).
// Every mbarrier wait traps after ~2^26 polls instead of hanging.

#include <cuda.h>

#include <cstdio>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "tma.cuh"

namespace bsct {

namespace {

constexpr int TC_M = 128, TC_N = 128, TC_K = 32;  // pixels, slices, samples per angle
constexpr int TC_TR = 8, TC_TCOL = 16;             // pixel tile: 8 rows x 16 columns
constexpr int TC_THREADS = 352;  // 8 W-producer warps, G TMA warp, MMA warp, table warp
constexpr int TC_ROWB = 128;                        // bytes per operand row (32 x FP32)
constexpr int TC_OPB = TC_M * TC_ROWB;              // one operand tile: 16 KB
constexpr int HCv = 25;                             // correction filter half-width (R8)

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// canonical K-major SWIZZLE_128B operand: row r (0..127) of 128 bytes, 16-byte chunk q -> q ^ (r & 7)
__device__ __forceinline__ uint32_t sw128(int r, int k) {
  return (uint32_t)(r * TC_ROWB + ((((k >> 2) ^ (r & 7))) << 4) + ((k & 3) << 2));
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4, LBO = 1 (unused when swizzled),
// SBO = 1024 B (8 rows x 128 B) >> 4, version 1 (sm_100), layout type 2 (128B swizzle)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor kind::tf32: D F32 (bits 4-5 = 1), A, B TF32 (bits 7-9, 10-12 = 2),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

}  // namespace

// Shared memory: three rings, so that the G tiles' L2 latency overlaps the weight production:
//   tables  TC_NT slots: the angle's basis table (per-p rows padded to TC_PSTR bytes: lanes at the
//           same row i but different sub-intervals p land in different banks) + its BPAngle record,
//           bulk-copied; released by the producers (t_empty) once they have built W.
//   W       TC_NW slots of W_hi, W_lo (16 KB each); released by the MMAs (w_empty).
//   G       TC_NG slots of G_hi, G_lo (16 KB each), TMA; released by the MMAs (g_empty).
constexpr int TC_PSTR = BP_SMAX * 8 * 4 + 16;                 // bytes per sub-interval in smem
constexpr int TC_PMAXT = 10;                                   // sub-intervals per angle (host-checked)
constexpr int TC_TABB = TC_PMAXT * TC_PSTR;                    // basis table slot
constexpr int TC_ANGB = (int)((sizeof(BPAngle) + 8 + 15) & ~(size_t)15);  // BPAngle + up to 8 B misalignment
constexpr int TC_TSLOT = (TC_TABB + TC_ANGB + 127) & ~127;
constexpr int TC_NT = 5, TC_NW = 2, TC_NG = 4;  // W slot a % 2 = the producer group of angle a
constexpr int TC_WOFF = 0, TC_GOFF = TC_NW * 2 * TC_OPB, TC_TOFF = TC_GOFF + TC_NG * 2 * TC_OPB;
constexpr int TC_BOFF = (TC_TOFF + TC_NT * TC_TSLOT + 127) & ~127;  // barriers
constexpr int TC_PROD = 256;  // producer threads: pixel t & 127, row half t >> 7

__device__ __forceinline__ void st_shared_v4z(uint32_t a) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(a), "f"(0.f) : "memory");
}
__device__ __forceinline__ void st_shared_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float4 ld_shared_v4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// the tile's 32-sample window start m_lo for one angle: the lowest cell over the 8 x 16 tile minus
// one (rounding margin) plus imin, aligned down so that column m_lo + HC is a multiple of 4 floats
// (TMA box starts must be 16-byte aligned in the innermost dimension: an unaligned start raised an
// illegal-instruction fault on B200)
__device__ __forceinline__ int tc_window(double u0, double du1, double du2, int imin, int tk1, int tk2) {
  const double ut = fma(du1, (double)tk1, fma(du2, (double)tk2, u0));
  const double umin = ut + fmin(0.0, du1 * (TC_TR - 1)) + fmin(0.0, du2 * (TC_TCOL - 1));
  return ((((int)floor(umin)) - 1 + imin + HCv) & ~3) - HCv;
}

__device__ __forceinline__ void st_shared_v4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
// the tensor cores read TF32 operands by ignoring the low 13 mantissa bits (measured: with raw FP32
// operands and lo = x - trunc(x) the 3xTF32 product is as accurate as with pre-rounded hi parts), so
// hi = x as stored and lo = x - trunc_tf32(x) (exact in FP32)
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Accumulation: the tensor cores' FP32 accumulation over many MMAs drifts (measured 3e-5 relative
// after 360 angles x 12 MMAs against the CUDA-core K4 v3), so each block of TC_F angles is
// accumulated from zero in one of two TMEM buffers (ping-pong, 2 x 128 columns) and the producer
// threads add every finished block into FP32 registers (round to nearest), one block behind.
constexpr int TC_F = 8;
#ifdef BSCT_TC_TRACE
__device__ long long g_tc_trace[8][512];
#define TC_TR_MARK(slot, a) \
  if (blockIdx.x == 7 && blockIdx.y == 20 && blockIdx.z == 3 && (a) < 512) g_tc_trace[slot][a] = clock64();
#else
#define TC_TR_MARK(slot, a)
#endif

// grid (ceil(N/16), ceil(N/8), ceil(B/128)); 320 threads; dynamic smem = bp_tc_smem()
__global__ void __launch_bounds__(TC_THREADS, 1) bp_tc_kernel(int N, int n_angles, int B,
                                                              const BPAngle *__restrict__ ang,
                                                              const float *__restrict__ Btab,
                                                              const __grid_constant__ CUtensorMap map_g,
                                                              const __grid_constant__ CUtensorMap map_lo,
                                                              float *__restrict__ out, float scale, int maxP) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (raw & 1023u)) & 1023u;
  unsigned char *smg = smem_raw + pad;  // generic view (shared window) of the aligned base
  const uint32_t sm = raw + pad;        // 32-bit shared address of the aligned base
  const uint32_t barb = sm + TC_BOFF;
  // barriers: full_t/t_empty [NT], full_w/w_empty [NW], full_g/g_empty [NG], acc_full/acc_empty [2]
  const uint32_t full_t = barb, t_empty = full_t + 8 * TC_NT, full_w = t_empty + 8 * TC_NT, w_empty = full_w + 8 * TC_NW,
                 full_g = w_empty + 8 * TC_NW, g_empty = full_g + 8 * TC_NG, acc_full = g_empty + 8 * TC_NG,
                 acc_empty = acc_full + 16;
  uint32_t *tmem_sh = reinterpret_cast<uint32_t *>(smg + TC_BOFF + 8 * (2 * TC_NT + 2 * TC_NW + 2 * TC_NG + 4));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tk1 = blockIdx.y * TC_TR, tk2 = blockIdx.x * TC_TCOL;
  const int b0 = blockIdx.z * TC_N;
  const int nblk = (n_angles + TC_F - 1) / TC_F;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_NT; ++s) {
      mbar_init(full_t + 8 * s, 1);
      mbar_init(t_empty + 8 * s, TC_PROD / 2 + 1);  // the angle's producer group + the G warp
    }
    for (int s = 0; s < TC_NW; ++s) {
      mbar_init(full_w + 8 * s, TC_PROD / 2);
      mbar_init(w_empty + 8 * s, 1);
    }
    for (int s = 0; s < TC_NG; ++s) {
      mbar_init(full_g + 8 * s, 1);
      mbar_init(g_empty + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + 8 * b, 1);
      mbar_init(acc_empty + 8 * b, TC_PROD);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {  // TMEM: 2 x 128 columns (ping-pong FP32 accumulators, N = 128), owned by this warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_sh)),
                 "n"(2 * TC_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_sh;

  if (warp < 8) {
    // ---------------------------------------------------------------- W producers
    // two groups of 128 threads (warps 0-3, 4-7) take alternate angles, one thread per pixel row,
    // so that two angles' locate / basis-evaluation latency chains are in flight at once
    const int t = threadIdx.x, r = t & 127, grp = t >> 7;
    const int k1 = tk1 + r / TC_TCOL, k2 = tk2 + r % TC_TCOL;
    const bool inside = k1 < N && k2 < N;
    const float f1 = (float)(r / TC_TCOL), f2 = (float)(r % TC_TCOL);  // pixel offset in the tile
    float acc[64];  // this group's accumulator columns [64 grp, 64 grp + 64) of pixel r
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.f;
    const uint32_t tlane = (uint32_t)((warp & 3) * 32) << 16;
    auto flush = [&](int jf) {  // add TMEM block jf (columns [64 grp, 64 grp + 64) of lane r) into acc
      const int buf = jf & 1;
      mbar_wait(acc_full + 8 * buf, (uint32_t)((jf >> 1) & 1), 6, jf);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + tlane + (uint32_t)(buf * TC_N + 64 * grp + 32 * c), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[32 * c + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(acc_empty + 8 * buf);
    };
    int next_flush = 0;
    int pc = 0;  // first chunk of this thread's previous weights in its slot
    {            // the slot starts as zero rows (no MMA has read it yet)
      const uint32_t w0 = sm + TC_WOFF + grp * 2 * TC_OPB;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        st_shared_v4z(w0 + r * TC_ROWB + (q << 4));
        st_shared_v4z(w0 + TC_OPB + r * TC_ROWB + (q << 4));
      }
    }
    static_assert(TC_NW == 2, "the W slot of angle a must be owned by producer group a % 2");
    for (int a = grp; a < n_angles; a += 2) {
      const int ts = a % TC_NT, ws = a % TC_NW;
      const uint32_t tab = sm + TC_TOFF + ts * TC_TSLOT;
      const uint32_t whi = sm + TC_WOFF + ws * 2 * TC_OPB, wlo = whi + TC_OPB;
      mbar_wait(full_t + 8 * ts, (uint32_t)((a / TC_NT) & 1), 1, a);  // basis table and BPAngle of angle a
      const size_t aoff = (size_t)((uintptr_t)(ang + a) & 15);  // the staged copy starts 16-byte aligned
      const BPAngle &A = *reinterpret_cast<const BPAngle *>(smg + TC_TOFF + ts * TC_TSLOT + TC_TABB + aoff);
      // locate: the tile origin in FP64 (uniform), the pixel's offset (|.| < 24 cells) in FP32, as K4 v3
      const double ut = fma(A.du1, (double)tk1, fma(A.du2, (double)tk2, A.u0));
      const double umin = ut + fmin(0.0, A.du1 * (TC_TR - 1)) + fmin(0.0, A.du2 * (TC_TCOL - 1));
      const int m_lo = ((((int)floor(umin)) - 1 + A.imin + HCv) & ~3) - HCv;
      const double ct = floor(ut);
      const float w0 = (float)(ut - ct) + fmaf((float)A.du1, f1, (float)A.du2 * f2);
      const float cf = floorf(w0);
      const float ph = w0 - cf;
      const int P = A.P;
      int p = 0;
#pragma unroll
      for (int k = 1; k < BP_PMAX; ++k) p += (k < P && ph >= A.bpf[k]) ? 1 : 0;
      const float tau = ph - A.bpf[p];
      const int o = (int)ct + (int)cf + A.imin - m_lo;  // window position of sample i = 0
      const int ilo = A.ilo[p], ihi = min((int)A.ihi[p], A.S - 1);
      float wv[8];
      const uint32_t bp = tab + (uint32_t)(p * TC_PSTR);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = ilo + q;
        wv[q] = 0.f;
        if (i <= ihi) {
          const float4 c03 = ld_shared_v4(bp + i * 32), c47 = ld_shared_v4(bp + i * 32 + 16);
          float w = c47.y;
          w = fmaf(w, tau, c47.x);
          w = fmaf(w, tau, c03.w);
          w = fmaf(w, tau, c03.z);
          w = fmaf(w, tau, c03.y);
          w = fmaf(w, tau, c03.x);
          wv[q] = inside ? w : 0.f;
        }
      }
      mbar_arrive(t_empty + 8 * ts);  // done with the tables of this slot
      mbar_wait(w_empty + 8 * ws, (uint32_t)(((a / TC_NW) & 1) ^ 1), 8, a);  // the MMAs of angle a - NW are done
      // the pixel's W_hi / W_lo rows.  Slot ws = a % 2 = grp is only ever written by this thread
      // (for this pixel): it holds the weights of angle a - 2 in chunks [pc, pc + 3) and zeros
      // elsewhere, so clearing those three chunks restores a zero row; then the new weights at
      // window positions o + ilo + q (program order: zero first)
#pragma unroll
      for (int q = 0; q < 3; ++q) {  // chunk c ^ (r & 7): the 8 lanes of a quarter warp hit distinct banks
        const int c = min(pc + q, 7);
        st_shared_v4z(whi + r * TC_ROWB + ((c ^ (r & 7)) << 4));
        st_shared_v4z(wlo + r * TC_ROWB + ((c ^ (r & 7)) << 4));
      }
      pc = (o + ilo) >> 2;  // <= 8 positions from here: <= 3 chunks
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (ilo + q <= ihi) {
          const uint32_t off = sw128(r, o + ilo + q);
          st_shared_f32(whi + off, wv[q]);
          st_shared_f32(wlo + off, tf32_lo(wv[q]));
        }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy (MMA)
      mbar_arrive(full_w + 8 * ws);
      // block jf is flushed once this group has produced its angles of block jf + 1 (their MMAs wait
      // for W only a few angles behind, so block jf's MMAs are done)
      while (next_flush + 2 <= (a + 2) / TC_F) flush(next_flush++);
    }
    while (next_flush < nblk) flush(next_flush++);
    // ---------------------------------------------------------------- epilogue: acc -> b[:, k1, k2]
    if (inside) {
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int b = b0 + 64 * grp + j;
        if (b < B) out[((size_t)b * N + k1) * N + k2] = scale * acc[j];
      }
    }
  } else if (warp == 10) {
    // ---------------------------------------------------------------- table producer (bulk copies, NT - 1 ahead)
    if (lane == 0) {
      for (int a = 0; a < n_angles; ++a) {
        const int ts = a % TC_NT;
        mbar_wait(t_empty + 8 * ts, (uint32_t)(((a / TC_NT) & 1) ^ 1), 9, a);
        const uint32_t tab = sm + TC_TOFF + ts * TC_TSLOT;
        const char *asrc = reinterpret_cast<const char *>(ang + a);
        const char *aal = reinterpret_cast<const char *>((uintptr_t)asrc & ~(uintptr_t)15);
        mbar_expect_tx(full_t + 8 * ts, (uint32_t)(maxP * BP_SMAX * 32 + TC_ANGB));
        const float *src = Btab + (size_t)a * BP_PMAX * BP_SMAX * 8;
        for (int q = 0; q < maxP; ++q)  // per-sub-interval rows into padded slots
          bulk_g2s(tab + q * TC_PSTR, src + q * BP_SMAX * 8, BP_SMAX * 32, full_t + 8 * ts);
        bulk_g2s(tab + TC_TABB, aal, TC_ANGB, full_t + 8 * ts);
      }
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- G producer (TMA)
    if (lane == 0) {
      for (int a = 0; a < n_angles; ++a) {
        const int gs = a % TC_NG, ts = a % TC_NT;
        // the window from the staged BPAngle record (the table warp runs ahead): no global load here
        mbar_wait(full_t + 8 * ts, (uint32_t)((a / TC_NT) & 1), 10, a);
        const size_t aoff = (size_t)((uintptr_t)(ang + a) & 15);
        const BPAngle &A = *reinterpret_cast<const BPAngle *>(smg + TC_TOFF + ts * TC_TSLOT + TC_TABB + aoff);
        const int m_lo = tc_window(A.u0, A.du1, A.du2, A.imin, tk1, tk2);
        mbar_arrive(t_empty + 8 * ts);  // done with this table slot
        mbar_wait(g_empty + 8 * gs, (uint32_t)(((a / TC_NG) & 1) ^ 1), 2, a);
        const uint32_t g = sm + TC_GOFF + gs * 2 * TC_OPB;
        mbar_expect_tx(full_g + 8 * gs, 2 * TC_OPB);
        // sample m <-> column m + HC of the corrected rows; outside the rows / batch: zero fill
        tma_load_3d(g, &map_g, m_lo + HCv, a, b0, full_g + 8 * gs);
        tma_load_3d(g + TC_OPB, &map_lo, m_lo + HCv, a, b0, full_g + 8 * gs);
      }
    }
  } else {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0) {
      for (int a = 0; a < n_angles; ++a) {
        const int ws = a % TC_NW, gs = a % TC_NG;
        const int j = a / TC_F, buf = j & 1;
        const bool first = a % TC_F == 0, last = a % TC_F == TC_F - 1 || a == n_angles - 1;
        if (first && j >= 2) mbar_wait(acc_empty + 8 * buf, (uint32_t)(((j - 2) >> 1) & 1), 7, a);
        mbar_wait(full_g + 8 * gs, (uint32_t)((a / TC_NG) & 1), 4, a);
        TC_TR_MARK(5, a);
        mbar_wait(full_w + 8 * ws, (uint32_t)((a / TC_NW) & 1), 3, a);
        TC_TR_MARK(6, a);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t whi = sm + TC_WOFF + ws * 2 * TC_OPB, wlo = whi + TC_OPB;
        const uint32_t ghi = sm + TC_GOFF + gs * 2 * TC_OPB, glo = ghi + TC_OPB;
        const uint32_t As[3] = {whi, whi, wlo}, Bs[3] = {ghi, glo, ghi};
        const uint32_t d = tmem + (uint32_t)(buf * TC_N);
#pragma unroll
        for (int pr = 0; pr < 3; ++pr)
#pragma unroll
          for (int kk = 0; kk < TC_K / 8; ++kk)  // K = 8 TF32 (32 bytes) per instruction
            umma_tf32(d, umma_desc(As[pr] + 32 * kk), umma_desc(Bs[pr] + 32 * kk),
                      (!first || pr > 0 || kk > 0) ? 1u : 0u);
        umma_commit(w_empty + 8 * ws);  // the W and G slots are free once these MMAs have read them
        umma_commit(g_empty + 8 * gs);
        if (last) umma_commit(acc_full + 8 * buf);  // block j complete in TMEM buffer j & 1
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 9) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * TC_N));
  }
}

// ------------------------------------------------------------------------------------ host side
EncodeTiled tma_encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

namespace {

// 3-D map over rows [B][n_angles][ldt] FP32 (Mt valid columns): box {32, 1, 128}, SWIZZLE_128B
bool make_map(CUtensorMap *map, const float *base, int Mt, int ldt, int n_angles, int B) {
  EncodeTiled enc = tma_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)Mt, (cuuint64_t)n_angles, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)ldt * 4, (cuuint64_t)ldt * 4 * n_angles};
  const cuuint32_t box[3] = {(cuuint32_t)TC_K, 1, (cuuint32_t)TC_N};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Geometry check (host, per plan): every 8 x 16 tile's samples fit the K = 32 window at every
// angle: ceil(7 |du1| + 15 |du2|) + 1 (margin) + 1 (floor) + 3 (16-byte aligned start) + S <= 32,
// du = lambda_x / lambda_y (sin, cos).
bool bp_tc_supported(int n, const double *angles, double lx, double ly, double zeta) {
  if (getenv("BSCT_BP_V3") && getenv("BSCT_BP_V3")[0] == '1') return false;
  for (int i = 0; i < n; ++i) {
    const double c = std::fabs(std::cos(angles[i])), s = std::fabs(std::sin(angles[i]));
    const double span = (lx / ly) * ((TC_TR - 1) * s + (TC_TCOL - 1) * c);
    const double H = 0.5 * (lx * (c + s) + zeta + 3.0 * ly);  // >= the half support of C_t
    const int cw = (int)std::ceil(H / ly - 1e-12);
    if ((int)std::ceil(span) + 2 + 3 + (2 * cw + 1) > TC_K) return false;  // + 3: aligned window start
    if (2 * cw + 1 > 8) return false;  // a producer thread holds at most 8 weights of its pixel
  }
  if (bp_v2_max_p(n, angles, lx, ly, zeta) > TC_PMAXT) return false;  // table slots hold TC_PMAXT sub-intervals
  return true;
}

size_t bp_tc_smem() { return (size_t)TC_BOFF + 8 * (2 * TC_NT + 2 * TC_NW + 2 * TC_NG + 4) + 16 + 1024; }

cudaError_t backproject_tc(int N, int n_angles, int M, int B, const BPAngle *ang, const float *Btab, const float *gt,
                           const float *gt_lo, int ldt, float *out, double scale, int maxP, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  CUtensorMap mg, ml;
  const int Mt = M + 2 * HCv;
  if (!make_map(&mg, gt, Mt, ldt, n_angles, B) || !make_map(&ml, gt_lo, Mt, ldt, n_angles, B))
    return cudaErrorNotSupported;
  const size_t sm = bp_tc_smem();
  cudaError_t e = cudaFuncSetAttribute(bp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  dim3 grid((N + TC_TCOL - 1) / TC_TCOL, (N + TC_TR - 1) / TC_TR, (B + TC_N - 1) / TC_N);
  bp_tc_kernel<<<grid, TC_THREADS, sm, s>>>(N, n_angles, B, ang, Btab, mg, ml, out, (float)scale, maxP);
#ifdef BSCT_TC_TRACE
  if (grid.z > 3 && grid.y > 20) {
    static long long h[8][512];
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(h, g_tc_trace, sizeof(h));
    const char *nm[8] = {"p:t_wait0", "p:t_got", "p:w_wait0", "p:w_got", "p:arrived", "m:g_got", "m:w_got", "tma:g_empty"};
    for (int a = 100; a < 112; ++a) {
      fprintf(stderr, "a=%d", a);
      for (int k = 0; k < 8; ++k) fprintf(stderr, " %s=%lld", nm[k], h[k][a] - h[0][100]);
      fprintf(stderr, "\n");
    }
  }
#endif
  return cudaGetLastError();
}

}  // namespace bsct
