// gram.cu -- K1: exact Gram filter taps.
//
//   G[dk] = lambda_x^4 sum_t M_[l|c|, l|c|, l|s|, l|s|, zeta, zeta](lambda_x (-s dk1 + c dk2))
//
// Tiled gather (deterministic, no atomics; R20).  Per angle, K0 (tables.cu) writes a compact
// record (GramRec layout in kernels.cuh): the argument coefficients, the half support H, the
// <= 16 right-half knots and the degree-5 local Taylor coefficients of every piece.  Angles
// are sorted by t mod pi on the host, so that the angles that can reach a tap form one
// (wrapping) run of the sorted order: with dk = r (cos phi, sin phi) the argument is
// lambda_x r sin(phi - t), nonzero only for |sin(phi - t)| < H / (lambda_x r).
//
//  * outer CTAs: a 32 x 16 tile of taps, two taps (rows r, r + 16) per thread.  The CTA derives the window of
//    angles that can reach any of its taps from the tile's polar-angle span and distance
//    (a superset: the per-term support test is exact), looks the run up in a bucket table
//    (no search), stages the run's records in shared memory 32 at a time (record-major,
//    16-byte aligned records) and
//    sums them in sorted order.  Far from the origin a tile sees ~5-20 angles.
//  * central CTAs (launched first): near the origin every angle reaches every tap, so the
//    outer tiles there are split into 4 x 4 sub-tiles with 16 threads per tap; the 16
//    threads take every 16th angle of the run and a fixed xor-shuffle tree sums them.
//  * dense mode (bench --dense-angles): every (tap, angle) pair, branch-free
//    (the FP32-pipe measurement of north_star's "Gram build >= 50% of FP32 peak").
//  * G[k] = G[-k] (G = H^T H): only the taps up to the centre in row-major order are
//    evaluated (rows above the centre row, and the centre row up to the centre); each thread
//    writes its value to both k and -k, so the filter is symmetric bitwise and half the work
//    is done.  (M_W is even and -u is formed exactly as -(u), so both orders agree anyway.)
//
// Argument accuracy (SURVEY.md 7 "Gram argument"): in FP32 the argument is formed from a
// hi/lo split of lambda_x cos t and lambda_x sin t: the hi parts are multiples of
// q0 = 2^(ceil(log2 lambda_x) - 11) with |hi / q0| <= 2^11, so -S_hi dk1 + C_hi dk2 is an
// integer multiple of q0 below 2^24 q0 for |dk| < 2^12 (N <= 2048) and is formed EXACTLY by
// one FMUL + FFMA; the lo parts add ~1e-7 lambda_x absolute error.  FP64 tables use the
// plain FP64 product.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "pptable.cuh"

namespace bsct {

// shared-memory record stride: 16-byte aligned (vector loads of the header and coefficients);
// lanes reading 16 different records (level 2) see at most 2-way bank conflicts
template <typename T>
struct GramSm {
  static constexpr int RS = sizeof(T) == 4 ? GR_WORDS + 4 : GR_WORDS + 2;
};

template <typename T>
struct GramArg;
template <>
struct GramArg<float> {
  float4 cs;  // (C_hi, C_lo, S_hi, S_lo): one 16-byte shared load
  __device__ __forceinline__ void load(const float *rec) { cs = *reinterpret_cast<const float4 *>(rec); }
  __device__ __forceinline__ float abs_u(float a, float b) const {
    // (u_hi, u_lo) = (-S_hi a + C_hi b, -S_lo a + C_lo b) on the packed FP32x2 pipe, each lane
    // the same rounding as fmaf(-S, a, C * b); u_hi exact (see header)
#ifdef BSCT_F32X2
    const float2 u = x2fma(float2{-cs.z, -cs.w}, float2{a, a}, x2mul(float2{cs.x, cs.y}, float2{b, b}));
    return fabsf(u.x + u.y);
#else
    const float uh = fmaf(-cs.z, a, cs.x * b);
    const float ul = fmaf(-cs.w, a, cs.y * b);
    return fabsf(uh + ul);
#endif
  }
};
template <>
struct GramArg<double> {
  double c, s;
  __device__ __forceinline__ void load(const double *rec) { c = rec[0]; s = rec[2]; }
  __device__ __forceinline__ double abs_u(double a, double b) const { return fabs(fma(-s, a, c * b)); }
};

// M(u) on one staged record for u = |argument| < H (4-step branch-free piece search over
// the 16 knots, +inf padded; degree-5 Horner in the local coordinate)
template <typename T>
__device__ __forceinline__ T gram_piece(const T *rec, T u) {
  const T *kn = rec + GR_KN;
  int j = 0;
  j += (kn[j + 8] <= u) ? 8 : 0;
  j += (kn[j + 4] <= u) ? 4 : 0;
  j += (kn[j + 2] <= u) ? 2 : 0;
  j += (kn[j + 1] <= u) ? 1 : 0;
  const T t = u - kn[j];
  using V2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;  // 8/16-byte loads
  const V2 *c = reinterpret_cast<const V2 *>(rec + GR_CO + j * GR_NC);
  const V2 c01 = c[0], c23 = c[1], c45 = c[2];
  T v = c45.y;
  v = fma(v, t, c45.x);
  v = fma(v, t, c23.y);
  v = fma(v, t, c23.x);
  v = fma(v, t, c01.y);
  v = fma(v, t, c01.x);
  return v;
}

// Sorted-order run [i0, i0 + cnt) (mod n) of the angles that can reach taps with
// dk1 in [a0, a1], dk2 in [b0, b1]; all angles when the rectangle comes within hmax
// (H_max / lambda_x, in taps) of the origin.  FP32 geometry with a margin: a superset.
// Called by one full warp (lanes 0-3 take the corners' polar angles, lane 4 the centre's);
// the result is valid in lane 0.
__device__ __forceinline__ void gram_window_warp(float a0, float a1, float b0, float b1, float hmax, int n,
                                                 const int *__restrict__ bucket, int nb, int &i0, int &cnt) {
  const float pi = 3.14159265358979f;
  const int lane = threadIdx.x & 31;
  const float ca = fminf(fmaxf(0.f, a0), a1), cb = fminf(fmaxf(0.f, b0), b1);
  const float rmin = sqrtf(ca * ca + cb * cb);
  i0 = 0;
  cnt = n;
  if (rmin <= hmax * 1.0001f + 1e-4f) return;  // warp-uniform
  const float px = lane == 4 ? 0.5f * (a0 + a1) : ((lane & 1) ? a1 : a0);
  const float py = lane == 4 ? 0.5f * (b0 + b1) : ((lane & 2) ? b1 : b0);
  const float ph = atan2f(py, px);
  const float phc = __shfl_sync(0xffffffffu, ph, 4);
  float d = ph - phc;
  d -= 2.f * pi * rintf(d * (0.5f / pi));
  if (lane > 3) d = 0.f;
  float dmin = d, dmax = d;
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  dmin = fminf(dmin, 0.f);
  dmax = fmaxf(dmax, 0.f);
  if (lane != 0) return;
  const float om = asinf(fminf(1.f, hmax / rmin)) * 1.0001f + 2e-5f;  // FP32 atan2/asin: ~1e-6 rad
  const float span = dmax - dmin + 2.f * om;
  if (span >= pi * 0.999f) return;
  float lo = phc + dmin - om;
  lo -= pi * floorf(lo * (1.f / pi));
  lo = fminf(fmaxf(lo, 0.f), pi);
  const float sc = (float)nb / pi;
  const int k0 = min(nb, max(0, (int)floorf(lo * sc)));
  i0 = bucket[k0];
  const float e = lo + span;
  if (e < pi) {
    const int k1 = min(nb, (int)floorf(e * sc) + 1);
    cnt = bucket[k1] - i0;
  } else {
    const int k1 = min(nb, (int)floorf((e - pi) * sc) + 1);
    cnt = (n - i0) + bucket[k1];
    if (cnt > n) cnt = n;
  }
  if (i0 >= n) i0 -= n;
}

// Records of a run are staged in chunks of CH, double buffered: the float4 loads of chunk k+1
// are issued into registers before chunk k is evaluated, so the L2 latency of the staging
// overlaps the arithmetic (central CTAs walk every angle: one L2 round trip per chunk).
template <typename T>
struct GramStage {
  static constexpr int CH = sizeof(T) == 4 ? 32 : 16;               // records per chunk
  static constexpr int V4 = GR_WORDS * (int)sizeof(T) / 16;           // float4 per record
  static constexpr int PF = (CH * V4 + 255) / 256;                    // float4 per thread
  float4 r[PF];
  // float4 elements [0, mv) of the run starting at float4 g0 of the table (nv = n V4: wraps)
  __device__ __forceinline__ void load(const float4 *__restrict__ g, int nv, int g0, int mv) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int f = threadIdx.x + 256 * k;
      if (f < mv) {
        int gi = g0 + f;
        if (gi >= nv) gi -= nv;
        r[k] = __ldg(g + gi);
      }
    }
  }
  // element f of record c = f / V4 goes to sm[c RS + (f - c V4) 16 / sizeof(T)]: one 16-byte store
  __device__ __forceinline__ void store(T *sm, int mv) const {
    constexpr int RS = GramSm<T>::RS, E = 16 / (int)sizeof(T);
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int f = threadIdx.x + 256 * k;
      if (f < mv) {
        const int c = f / V4;
        *reinterpret_cast<float4 *>(sm + f * E + c * (RS - GR_WORDS)) = r[k];
      }
    }
  }
};

// Three tile levels, each a contiguous range of blockIdx (innermost first), so that no CTA
// walks a long angle run alone: a 16 x 16 tile at distance r sees ~(23 + 2 H_max) n / (pi r)
// angles.  Level 0: 16 x 16 taps, one thread per tap.  Level 1: 8 x 8 taps, 4 threads per tap.
// Level 2: 4 x 4 taps, 16 threads per tap.  Level l covers the 16-tiles of the square sq_l
// (in 16-tile units, rows up to the centre row) outside sq_{l+1}; CTAs of a tile inside the
// next square return at once.
struct GramLevels {
  int a1, b1, a2, b2;  // squares [a_l, b_l)^2 of 16-tiles of levels 1 and 2 (level 0: the whole grid)
  int st1, st2;        // first blockIdx of level 1 and of level 0 (level 2 starts at 0)
  int t16, r16;        // 16-tiles per side; tile rows up to the centre row
};

template <typename T, bool DENSE>
__global__ void __launch_bounds__(256) gram_tiles_kernel(int N, int n, const T *__restrict__ rec,
                                                          const int *__restrict__ bucket, int nb, float hmax,
                                                          GramLevels lv, T scale, T *__restrict__ taps) {
  using St = GramStage<T>;
  constexpr int CH = St::CH, V4 = St::V4;
  constexpr int GRS = GramSm<T>::RS;
  __shared__ __align__(16) T sm[2][CH * GRS];
  __shared__ int win[2];
  const int D = 2 * N - 1;
  const int bid = blockIdx.x;
  const int level = bid < lv.st1 ? 2 : (bid < lv.st2 ? 1 : 0);
  const int lg = 2 * level;              // log2 threads per tap (= log2 sub-tiles per 16-tile)
  const int tw = 16 >> level;            // tile edge
  const int idx = bid - (level == 2 ? 0 : (level == 1 ? lv.st1 : lv.st2));
  const int qa = level == 2 ? lv.a2 : (level == 1 ? lv.a1 : 0);
  const int qb = level == 2 ? lv.b2 : (level == 1 ? lv.b1 : lv.t16);
  const int sub = idx & ((1 << lg) - 1), tile = idx >> lg;
  const int side = qb - qa;
  const int trq = tile / side;
  const int tr16 = qa + trq, tc16 = qa + (tile - trq * side);
  if (tr16 >= min(qb, lv.r16)) return;  // below the centre row: mirrored from above
  const int na = level == 2 ? qb : (level == 1 ? lv.a2 : lv.a1), nbq = level == 2 ? qb : (level == 1 ? lv.b2 : lv.b1);
  if (level < 2 && tr16 >= na && tr16 < nbq && tc16 >= na && tc16 < nbq) return;  // next level's tile
  const int r0 = tr16 * 16 + (sub >> level) * tw, c0 = tc16 * 16 + (sub & ((1 << level) - 1)) * tw;
  if (r0 > N - 1 || c0 >= D) return;
  const int h = min(tw, D - r0), w = min(tw, D - c0);
  int i0 = 0, cnt = n;
  if (!DENSE) {
    if (threadIdx.x < 32) {
      gram_window_warp((float)(r0 - (N - 1)), (float)(r0 + h - 1 - (N - 1)), (float)(c0 - (N - 1)),
                       (float)(c0 + w - 1 - (N - 1)), hmax, n, bucket, nb, i0, cnt);
      if (threadIdx.x == 0) {
        win[0] = i0;
        win[1] = cnt;
      }
    }
    __syncthreads();
    i0 = win[0];
    cnt = win[1];
  }
  // this thread's tap and its share of the run (every P-th angle, P = 1 << lg).  Each warp covers
  // a compact (4 x 8, 2 x 4, 1 x 2 at levels 0, 1, 2) block of taps: a support strip crosses
  // fewer warp blocks than with row-shaped blocks, so fewer warps take the evaluation branch.
  const int wp = threadIdx.x >> 5, q = (threadIdx.x & 31) >> lg, lane0 = threadIdx.x & ((1 << lg) - 1);
  const int bh = 4 >> level, bw = 8 >> level;
  const int tr = (wp >> 1) * bh + (q >> (3 - level)), tcl = (wp & 1) * bw + (q & (bw - 1));
  const int ri = r0 + tr, ci = c0 + tcl;  // this thread's tap, and its mirror (D-1-ri, D-1-ci)
  const bool valid = tr < h && tcl < w && (ri < N - 1 || (ri == N - 1 && ci <= N - 1));
  const T a = (T)(ri - (N - 1));  // dk1
  const T b = (T)(ci - (N - 1));  // dk2
  T acc = (T)0;
  St st;
  // K1 is launched as a programmatic dependent of K0 (PDL): everything above (tile indices, the
  // window from the host-built bucket table) overlapped K0; the records are K0's output
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const float4 *g4 = reinterpret_cast<const float4 *>(rec);
  const int nv = n * V4;
  if (cnt > 0) st.load(g4, nv, i0 * V4, min(CH, cnt) * V4);
  for (int cb = 0, buf = 0; cb < cnt; cb += CH, buf ^= 1) {
    const int m = min(CH, cnt - cb);
    st.store(sm[buf], m * V4);
    __syncthreads();  // also orders the previous reads of sm[buf] (two chunks ago) before this store
    if (cb + CH < cnt) {
      int g0 = (i0 + cb + CH) * V4;
      if (g0 >= nv) g0 -= nv;
      st.load(g4, nv, g0, min(CH, cnt - cb - CH) * V4);
    }
    if (!valid) continue;
#pragma unroll 4
    for (int c = lane0; c < m; c += (1 << lg)) {
      const T *rc = sm[buf] + c * GRS;
      GramArg<T> g;
      g.load(rc);
      const T H = rc[GR_H];
      const T u = g.abs_u(a, b);
      if (DENSE) {  // branch-free: every pair evaluated, zero outside the support
        const T v = gram_piece<T>(rc, fmin(u, H));
        acc += (u < H) ? v : (T)0;
      } else if (u < H) {
        acc += gram_piece<T>(rc, u);
      }
    }
  }
  // fixed-order tree over the threads of each tap
  if (level >= 2) {
    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  }
  if (level >= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  }
  if (lane0 == 0 && valid) {
    const T v = scale * acc;
    taps[(size_t)ri * D + ci] = v;
    taps[(size_t)(D - 1 - ri) * D + (D - 1 - ci)] = v;
  }
}

template <typename T>
cudaError_t gram_build_tiles(int N, double lx, int n, double n_dens, const T *rec, const int *bucket, int nb,
                             double Hmax, bool dense, T *taps, cudaStream_t s) {
  const int D = 2 * N - 1;
  const int T16 = (D + 15) / 16, R16 = (N - 1) / 16 + 1;  // 16-tiles per side, tile rows up to the centre
  // level radii (taps): about <= 64 angles per thread at every level (K1).  n_dens: the
  // angles per pi where the set is densest (= n for angles spread over [0, pi); an angle shard of
  // config 4 packs its n angles into a wedge, whose taps see n_dens / n times more of them)
  const double hm = Hmax / lx;
  // BSCT_GRAM_R1 / BSCT_GRAM_R2: scale the level radii (experiments).  Level 1 reaches 1.5x further
  // than the 64-angles-per-thread rule: config 5 31.0 -> 28.9 us, config 4 unchanged
  // (profiles/r02/gram_r_sweep.txt)
  double f1 = 1.5, f2 = 1.0;
  if (const char *e = getenv("BSCT_GRAM_R1")) f1 = atof(e);
  if (const char *e = getenv("BSCT_GRAM_R2")) f2 = atof(e);
  const double R1 = dense ? 0.0 : f1 * (23.0 + 2.0 * hm) * n_dens / (3.14159265 * 64.0);
  const double R2 = dense ? 0.0 : f2 * (11.3 + 2.0 * hm) * n_dens / (3.14159265 * 4.0 * 64.0);
  auto square = [&](double R, int &a, int &b) {  // 16-tiles meeting |dk| <= R in both coordinates
    if (R <= 0) {
      a = b = 0;
      return;
    }
    a = (int)std::ceil(((N - 1) - R - 15) / 16.0);
    b = (int)std::floor(((N - 1) + R) / 16.0) + 1;
    a = a < 0 ? 0 : a;
    b = b > T16 ? T16 : b;
    if (b < a) b = a;
  };
  GramLevels lv;
  lv.t16 = T16;
  lv.r16 = R16;
  square(std::max(R1, R2), lv.a1, lv.b1);
  square(R2, lv.a2, lv.b2);
  auto count = [&](int a, int b, int l) {
    const int rows = std::max(0, std::min(b, R16) - a);
    return rows * (b - a) * (1 << (2 * l));
  };
  const int c2 = count(lv.a2, lv.b2, 2), c1 = count(lv.a1, lv.b1, 1), c0 = count(0, T16, 0);
  lv.st1 = c2;
  lv.st2 = c2 + c1;
  const int blocks = c2 + c1 + c0;
  const double l2 = lx * lx;
  if (blocks == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap K0's tail (PDL)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const float hmf = (float)hm;
  const T sc = (T)(l2 * l2);
  if (dense) return cudaLaunchKernelEx(&cfg, gram_tiles_kernel<T, true>, N, n, rec, bucket, nb, hmf, lv, sc, taps);
  return cudaLaunchKernelEx(&cfg, gram_tiles_kernel<T, false>, N, n, rec, bucket, nb, hmf, lv, sc, taps);
}

template cudaError_t gram_build_tiles<float>(int, double, int, double, const float *, const int *, int, double, bool,
                                             float *, cudaStream_t);
template cudaError_t gram_build_tiles<double>(int, double, int, double, const double *, const int *, int, double, bool,
                                              double *, cudaStream_t);

}  // namespace bsct
