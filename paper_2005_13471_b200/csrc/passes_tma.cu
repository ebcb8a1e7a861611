// passes_tma.cu -- pass C of the fused CG iteration at L = 1024 (FP32) as a persistent,
// TMA-pipelined kernel ("apply the filter"; the CG recurrences of cg.cu).
//
// Same contract as cg_pass_c_1024_kernel (cg.cu): for each tile = (slice b, 16 image rows from
// row0) the inverse row DFTs of T1[b][q][row0 .. row0 + 16), q <= L/2 (the Hermitian half
// spectra after pass B) give (G d) rows; r -= alpha G d (and x += alpha r for steepest descent /
// Landweber, MODE 1 / 2), partial <r, r> per tile; MODE 3 writes y = G x into r.
//
// The round-1 kernel stages a tile, waits for all of it, transforms it and only then stages the
// next one (one tile per CTA, two CTAs per SM): its load and compute phases overlap only across
// the two CTAs (pass C ran at 0.70 of HBM).  Here one CTA per SM loops over tiles with a 2-stage
// shared-memory ring filled by the copy engine:
//   warp 8 (one lane): cp.async.bulk.tensor of tile i + 2 as soon as the consumers have released
//                      stage i % 2 -- three 3-D boxes {32 floats, 171 q, 1 slice} (128-byte rows,
//                      SWIZZLE_128B, zero fill past the last image row), completion on full[s];
//   warps 0-7:         warp w owns the row pair (2w, 2w + 1) of every tile: prefetch its r rows
//                      into registers, wait full[s], read its 513 row-pair entries (conflict-free:
//                      the swizzle spreads 8 consecutive q over the 8 16-byte chunks), release the
//                      stage, then the inverse four-step FFT (fft32.cuh) and the r update while the
//                      copy engine already streams the next tile.
// Every tile's arithmetic is the one of cg_pass_c_1024_kernel except the per-slice scalar
// reductions, which each consumer warp forms itself (fixed order: deterministic, identical in all
// warps).
#include "fft32.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "tma.cuh"

namespace bsct {

namespace {

constexpr int PC_ROWS = 16;                    // image rows per tile (8 row pairs, one per consumer warp)
constexpr int PC_CONS = PC_ROWS / 2;           // consumer warps
constexpr int PC_THREADS = 32 * (PC_CONS + 1);  // + the TMA warp
constexpr int PC_BOXQ = 171;                   // q rows per TMA box: 3 x 171 = 513 = L / 2 + 1
constexpr int PC_BOXB = 22528;                 // bytes per box region: 176 rows of 128 B (1024-aligned)
constexpr int PC_STAGEB = 3 * PC_BOXB;         // one tile
constexpr int PC_TRB = 32 * 33 * 8;            // one warp's transpose buffer
constexpr int PC_SMEM = 2 * PC_STAGEB + PC_CONS * PC_TRB + 1024;  // + 1024: alignment of the ring

// byte offset of the 16-byte entry (q, row pair w) in a stage (SWIZZLE_128B: chunk w ^ (row & 7))
__device__ __forceinline__ uint32_t pc_entry(int q, int w) {
  const int kk = q / PC_BOXQ, rr = q - kk * PC_BOXQ;
  return (uint32_t)(kk * PC_BOXB + rr * 128 + ((w ^ (rr & 7)) << 4));
}

// sum of n doubles in a fixed order by one warp (lane-strided partial sums, xor tree): every warp
// that calls it with the same data gets the same value
__device__ __forceinline__ double warp_sum_parts(const double *__restrict__ parts, int n, int lane) {
  double v = 0.0;
  for (int i = lane; i < n; i += 32) v += parts[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(PC_THREADS, 1)
    cg_pass_c_1024_tma_kernel(const __grid_constant__ CUtensorMap tmap, int N, int k, int gparts,
                              float *__restrict__ x, float *__restrict__ r, const float2 *__restrict__ tw1024,
                              FusedWork w) {
  constexpr int L = 1024;
  extern __shared__ unsigned char pc_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(((uintptr_t)pc_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t ring = smem_u32(smem);
  float2 *trs = reinterpret_cast<float2 *>(smem + 2 * PC_STAGEB);
  __shared__ __align__(8) unsigned long long bars[4];  // full[2], empty[2]
  __shared__ double red[2][PC_CONS];
  __shared__ double sc_rho[PC_CONS], sc_alpha[PC_CONS];
  __shared__ float2 twl[32 * 32];  // W_1024^{j t}
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[2]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // each CTA takes a contiguous range of tiles: consecutive tiles mostly share the slice, whose
  // scalars are then formed once
  const int ntiles = w.nparts * w.B;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = min(ntiles, (int)blockIdx.x * per), t_end = min(ntiles, t_begin + per);
  if (threadIdx.x == 0) {
    mbar_init(full0, 1);
    mbar_init(full0 + 8, 1);
    mbar_init(empty0, PC_CONS);
    mbar_init(empty0 + 8, PC_CONS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == PC_CONS) {  // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int i = 0;
      for (int t = t_begin; t < t_end; ++t, ++i) {
        const int s = i & 1;
        if (i >= 2) mbar_wait(empty0 + 8 * s, (uint32_t)(((i >> 1) - 1) & 1), 1, i);
        const int b = t / w.nparts, row0 = (t - b * w.nparts) * PC_ROWS;
        mbar_expect_tx(full0 + 8 * s, (uint32_t)(3 * PC_BOXQ * 128));
#pragma unroll
        for (int kk = 0; kk < 3; ++kk)
          tma_load_3d(ring + s * PC_STAGEB + kk * PC_BOXB, &tmap, 2 * row0, kk * PC_BOXQ, b, full0 + 8 * s);
      }
    }
    return;
  }

  // ------------------------------------------------------------------------------ consumer warps
  // W_1024 table in shared memory (read once per CTA; the loop reads it 11 times per tile and warp)
  for (int j = threadIdx.x; j < 32 * 32; j += 32 * PC_CONS) twl[j] = tw1024[j];
  asm volatile("bar.sync 1, %0;" ::"n"(32 * PC_CONS) : "memory");
  int i = 0, win = -1;  // scalars of slices [win, win + PC_CONS) are in sc_*
#pragma unroll 1
  for (int t = t_begin; t < t_end; ++t, ++i) {
    const int s = i & 1;
    const int b = t / w.nparts, bx = t - b * w.nparts;
    const int row0 = bx * PC_ROWS;
    const int ra = row0 + 2 * warp;
    const bool ha = ra < N, hb = ra + 1 < N;
    float *r0 = r + ((size_t)b * N + ra) * N, *x0 = x + ((size_t)b * N + ra) * N;
    // this warp's r rows into registers first: their latency overlaps the wait and the FFT.  The
    // loads are unconditional (clamped to a valid row and column; unused values are never read) so
    // that no select on the loaded value forces an early wait.
    float rv[2][16];
    if (MODE != 3) {
      const float *ka = r + ((size_t)b * N + min(ra, N - 1)) * N, *kb = r + ((size_t)b * N + min(ra + 1, N - 1)) * N;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int n = min(lane + 32 * m, N - 1);
        rv[0][m] = ka[n];
        rv[1][m] = kb[n];
      }
    }
    // scalars of the slices (as cg_pass_c_1024_kernel, each slice's partials reduced by one warp in
    // a fixed order), formed for PC_CONS slices at a time when the tile's slice leaves the window
    if (MODE != 3 && (win < 0 || b >= win + PC_CONS)) {
      asm volatile("bar.sync 1, %0;" ::"n"(32 * PC_CONS) : "memory");  // the old window is read out
      win = b;
      const int bs = b + warp;
      if (bs < w.B) {
        double rho = 0.0, alpha = 0.0;
        if (MODE == 0) {
          rho = w.rho[(size_t)bs * w.rho_stride + k];
        } else {
          rho = warp_sum_parts(w.rpart + ((size_t)(k & 1) * w.B + bs) * w.nparts, w.nparts, lane);
        }
        if (MODE == 2) {
          alpha = *w.tau;
        } else {
          const double gam = warp_sum_parts(w.gpart + (size_t)bs * gparts, gparts, lane);
          const bool bad = rho > 0 && !(gam > 0);
          const bool frozen = bad || (w.flags && w.flags[bs]);
          alpha = (rho > 0 && !frozen) ? rho / gam : 0.0;
          if (bad && w.flags && lane == 0) w.flags[bs] = 1;  // idempotent: any CTA holding slice bs may set it
        }
        if (lane == 0) {
          sc_rho[warp] = rho;
          sc_alpha[warp] = alpha;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * PC_CONS) : "memory");
    }
    double alpha = 0.0;
    if (MODE != 3) alpha = sc_alpha[b - win];
    if (MODE != 3 && bx == 0 && warp == 0 && lane == 0) {
      w.alpha[b] = alpha;
      if (MODE != 0) {
        const double rho = sc_rho[b - win];
        w.rho[(size_t)b * w.rho_stride + k] = rho;
        if (k > 0 && w.resid) w.resid[(size_t)b * w.iters + k - 1] = sqrt(rho);
      }
    }
    const float al = (float)alpha;
    // row pair (2 warp, 2 warp + 1): Z[q] = X_a[q] + i X_b[q], Z[L - q] = conj X_a[q] + i conj X_b[q]
    mbar_wait(full0 + 8 * s, (uint32_t)((i >> 1) & 1), 2, i);
    const uint32_t st = ring + s * PC_STAGEB;
    float2 v[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const int q = lane + 32 * rr;
      float4 e;
      if (rr < 16 || (rr == 16 && lane == 0)) {  // q <= 512: direct
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(e.x), "=f"(e.y), "=f"(e.z), "=f"(e.w)
                     : "r"(st + pc_entry(q, warp)));
        if (q == 0 || q == L / 2) {  // DC / Nyquist of real rows
          e.y = 0.f;
          e.w = 0.f;
        }
        v[rr] = float2{e.x - e.w, e.y + e.z};
      } else {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(e.x), "=f"(e.y), "=f"(e.z), "=f"(e.w)
                     : "r"(st + pc_entry(L - q, warp)));
        v[rr] = float2{e.x + e.w, e.z - e.y};
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);  // this warp is done with the stage
    float2 *tr = trs + warp * (32 * 33);
    dft32<true>(v);                      // over rr: v[a] = U[lane][a]
    twiddle1024_any<true>(v, twl, lane);  // conj W_1024^{a t}
    warp_transpose32(v, tr, lane);       // lane a: v[j] = U[j][a]
    dft32<true>(v);                      // v[m] = z[lane + 32 m] = y_a + i y_b
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
          const float tt = fmaf(-al, v[m].x, rv[0][m]);
          r0[n] = tt;
          ac = fmaf(tt, tt, ac);
        }
        if (hb) {
          if (MODE != 0) x0[N + n] = fmaf(al, rv[1][m], x0[N + n]);
          const float tt = fmaf(-al, v[m].y, rv[1][m]);
          r0[N + n] = tt;
          ac = fmaf(tt, tt, ac);
        }
      }
    }
    if (MODE != 3) {  // partial <r_{k+1}, r_{k+1}> of the tile: warps in order, one named barrier
      double d = (double)ac;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0) red[s][warp] = d;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * PC_CONS) : "memory");
      if (warp == 0 && lane == 0) {
        double tot = 0.0;
#pragma unroll
        for (int j = 0; j < PC_CONS; ++j) tot += red[s][j];
        w.rpart[((size_t)((k + 1) & 1) * w.B + b) * w.nparts + bx] = tot;
      }
    }
  }
}

// 3-D map over T1 viewed as FP32 [B][Q][2N]: box {32 floats = 16 rows' complex entries, 171 q, 1}
bool make_t1_map(CUtensorMap *map, const float2 *T1, int N, int B) {
  EncodeTiled enc = tma_encoder();
  if (!enc) return false;
  constexpr int Q = 1024 / 2 + 1;
  const cuuint64_t dims[3] = {(cuuint64_t)2 * N, (cuuint64_t)Q, (cuuint64_t)B};
  const cuuint64_t strides[2] = {(cuuint64_t)N * 8, (cuuint64_t)N * 8 * Q};
  const cuuint32_t box[3] = {32, (cuuint32_t)PC_BOXQ, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2 *>(T1), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int n[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

template <int MODE>
cudaError_t launch_c(const CUtensorMap &map, int N, int k, int gparts, float *x, float *r, const float2 *twl,
                     const FusedWork &w, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(cg_pass_c_1024_tma_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PC_SMEM);
  if (e != cudaSuccess) return e;
  const int tiles = w.nparts * w.B;
  const int grid = std::min(tiles, num_sms());
  cg_pass_c_1024_tma_kernel<MODE><<<grid, PC_THREADS, PC_SMEM, s>>>(map, N, k, gparts, x, r, twl, w);
  return cudaGetLastError();
}

}  // namespace

// Opt-in (BSCT_PASSC_TMA=1): measured on B200 (config 5, 2048 slices) at 1.00 us per slice against
// 0.94 us for cg_pass_c_1024_kernel -- with one CTA (8 consumer warps) per SM the r-row loads and
// the slice scalars stall the lock-stepped warps (ncu: long_scoreboard 2.7 warps per issue, issue
// 32%) more than the TMA ring saves.  Needs N even (16-byte T1 row strides), N <= 512 and 16 rows
// per tile (w.nparts = ceil(N / 16)).
bool pass_c_tma_enabled(int N, int nparts) {
  const char *e = getenv("BSCT_PASSC_TMA");
  if (!(e && e[0] == '1')) return false;
  return (N % 2) == 0 && N <= 512 && nparts == (N + PC_ROWS - 1) / PC_ROWS && tma_encoder() != nullptr;
}

cudaError_t pass_c_1024_tma(int N, int k, int mode, int gparts, const float2 *T1, float *x, float *r,
                            const float2 *twl, const FusedWork &w, cudaStream_t s) {
  if (w.B <= 0) return cudaSuccess;
  CUtensorMap map;
  if (!make_t1_map(&map, T1, N, w.B)) return cudaErrorNotSupported;
  switch (mode) {
    case 0: return launch_c<0>(map, N, k, gparts, x, r, twl, w, s);
    case 1: return launch_c<1>(map, N, k, gparts, x, r, twl, w, s);
    case 2: return launch_c<2>(map, N, k, gparts, x, r, twl, w, s);
    case 3: return launch_c<3>(map, N, k, gparts, x, r, twl, w, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace bsct
