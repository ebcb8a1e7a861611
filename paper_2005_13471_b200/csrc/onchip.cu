// onchip.cu -- NEXT-2: cluster-resident solver loop for small N.
//
// One thread-block cluster of CS CTAs per slice runs all iterations of CG / steepest descent /
// Landweber (same recurrences as cg.cu) in one launch.  The row-FFT intermediate
// T1[q][row] (q <= L/2) never leaves the chip: it is split by column ranges over the CTAs'
// shared memory (CTA c owns q in [c QP, (c+1) QP)).  Per iteration, for the search direction d:
//   A  each CTA transforms its own rows of pad(d) (two real rows per complex FFT) and scatters
//      every column's two entries into the owner CTA's shared memory through DSMEM;
//   B  each CTA transforms its columns (FFT, * spectrum, inverse FFT, keep N rows) in place,
//      <d, G d> by Parseval;
//   C  each CTA gathers its rows' spectra from all owners through DSMEM, inverse transforms,
//      and updates r, x (and p for CG) for those rows; <r, r>.
// Cluster-wide scalars: each CTA's block partial goes to rank 0's shared memory; after the
// cluster barrier every CTA sums the CS partials in rank order (identical on all CTAs,
// deterministic).  x, r, p live in global memory (L2) by rows; a CTA only reads and writes
// its own rows of them.  The FFTs are the block-level Stockham groups of fft.cuh.
#include <cooperative_groups.h>

#include <cstdlib>

#include "fft.cuh"
#include "kernels.cuh"

namespace cgr = cooperative_groups;

namespace bsct {

constexpr int OC_THREADS = 256;

template <int L>
struct OcCfg {
  static constexpr int P = FftCfg<L>::P;   // threads per FFT group
  static constexpr int G = OC_THREADS / P;  // groups per CTA
  static constexpr int Q = L / 2 + 1;
};

// MODE 0 CG, 1 steepest descent, 2 Landweber
template <typename T, int L, int CS, int MODE>
__global__ void __launch_bounds__(OC_THREADS) onchip_kernel(int N, int iters, const T *__restrict__ b,
                                                            T *__restrict__ x, T *__restrict__ r, T *__restrict__ p,
                                                            const T *__restrict__ S, const cplx<T> *__restrict__ tw,
                                                            const double *__restrict__ tau, double *__restrict__ resid,
                                                            int *__restrict__ flags) {
  using V = cplx<T>;
  using Cf = FftCfg<L>;
  constexpr int P = OcCfg<L>::P, G = OcCfg<L>::G, Q = OcCfg<L>::Q, E = Cf::E;
  cgr::cluster_group cl = cgr::this_cluster();
  const int crank = (int)cl.block_rank();
  const int bs = blockIdx.y;  // slice
  const int QP = (Q + CS - 1) / CS;
  const int qlo = min(Q, crank * QP), qhi = min(Q, qlo + QP);
  const int RP = ((N + CS - 1) / CS + 1) & ~1;  // rows per CTA, even (row pairs)
  const int rlo = min(N, crank * RP), rhi = min(N, rlo + RP);
  const int npairs = (rhi - rlo + 1) / 2;
  // FP32 row pairs start at even rows (rlo is even): (ra, ra + 1) are 16-byte aligned in T1 rows
  // when N is even
  const bool pair16 = sizeof(T) == 4 && (N % 2) == 0;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  V *T1 = reinterpret_cast<V *>(smem_raw);  // [QP][N]: this CTA's columns
  V *gbuf = T1 + (size_t)QP * N;            // [G][SMEM]: FFT group buffers
  __shared__ double red[32];
  __shared__ double cpart[2][CS];  // cluster partials (rank 0's copy is the one read)
  const int g = threadIdx.x / P, t = threadIdx.x % P;
  V *sm = gbuf + g * Cf::SMEM;
  const size_t so = (size_t)bs * N * N;

  auto block_sum = [&](double v) -> double {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0;
    for (int i = 0; i < OC_THREADS / 32; ++i) s += red[i];
    return s;
  };
  // cluster sum in rank order; also a cluster-wide barrier (release / acquire of shared memory)
  auto cluster_sum = [&](double v, int slot) -> double {
    const double s = block_sum(v);
    if (threadIdx.x == 0) cl.map_shared_rank(&cpart[slot][0], 0)[crank] = s;
    cl.sync();
    const double *src = cl.map_shared_rank(&cpart[slot][0], 0);
    double tot = 0;
    for (int i = 0; i < CS; ++i) tot += src[i];
    return tot;
  };

  if (flags && crank == 0 && threadIdx.x == 0) flags[bs] = 0;
  // init: x = 0, r = b, p = b (own rows); rho_0 = <b, b>
  double acc = 0;
  for (int i = threadIdx.x; i < (rhi - rlo) * N; i += OC_THREADS) {
    const size_t e = so + (size_t)rlo * N + i;
    const T v = b[e];
    x[e] = 0;
    r[e] = v;
    if (MODE == 0) p[e] = v;
    acc += (double)v * v;
  }
  double rho = cluster_sum(acc, 0);
  bool frozen = false;
  const T *d = MODE == 0 ? p : r;
  for (int k = 0; k < iters; ++k) {
    // ---- A: row FFTs of pad(d), own rows; scatter the half spectra to the column owners
    for (int j0 = 0; j0 < npairs; j0 += G) {
      const int ra = rlo + 2 * (j0 + g);
      const bool valid = j0 + g < npairs;
      V v[E];
#pragma unroll
      for (int rr = 0; rr < E; ++rr) {
        const int c = t + rr * P;
        T va = 0, vb = 0;
        if (valid && c < N) {
          va = d[so + (size_t)ra * N + c];
          if (ra + 1 < rhi) vb = d[so + (size_t)(ra + 1) * N + c];
        }
        v[rr] = V{va, vb};
      }
      fft_group<T, L, false>(v, sm, tw, t);
      if (valid)
        for (int q = t; q < Q; q += P) {
          const V z = sm[pidx(q)];
          const V zc = sm[pidx((L - q) & (L - 1))];
          const int own = q / QP;
          V *dst = cl.map_shared_rank(T1, own) + (size_t)(q - own * QP) * N;
          const V va = V{(T)0.5 * (z.x + zc.x), (T)0.5 * (z.y - zc.y)};
          const V vb = V{(T)0.5 * (z.y + zc.y), (T)0.5 * (zc.x - z.x)};
          if (ra + 1 < rhi && pair16) {  // one 16-byte DSMEM store for the pair (FP32)
            *reinterpret_cast<float4 *>(dst + ra) = make_float4((float)va.x, (float)va.y, (float)vb.x, (float)vb.y);
          } else {
            dst[ra] = va;
            if (ra + 1 < rhi) dst[ra + 1] = vb;
          }
        }
      __syncthreads();  // sm is rewritten by the next round
    }
    cl.sync();  // all of T1 written
    // ---- B: own columns: FFT, * S, inverse FFT, keep rows < N; gamma = <d, G d> (Parseval)
    double gam = 0;
    for (int q0 = qlo; q0 < qhi; q0 += G) {
      const int q = q0 + g;
      const bool valid = q < qhi;
      V *col = T1 + (size_t)(valid ? q - qlo : 0) * N;
      V v[E];
#pragma unroll
      for (int rr = 0; rr < E; ++rr) {
        const int i = t + rr * P;
        v[rr] = (valid && i < N) ? col[i] : V{0, 0};
      }
      fft_group<T, L, false>(v, sm, tw, t);
      const T *Sq = S + (size_t)(valid ? q : 0) * L;
      double gq = 0;
#pragma unroll
      for (int rr = 0; rr < E; ++rr) {
        const int pp = t + rr * P;
        const V y = sm[pidx(pp)];
        const T sv = valid ? Sq[pp] : (T)0;
        gq += (double)sv * ((double)y.x * y.x + (double)y.y * y.y);
        v[rr] = V{y.x * sv, y.y * sv};
      }
      if (valid && q != 0 && q != L / 2) gq *= 2.0;
      gam += gq;
      __syncthreads();
      fft_group<T, L, true>(v, sm, tw, t);
      if (valid)
#pragma unroll
        for (int rr = 0; rr < E; ++rr) {
          const int i = t + rr * P;
          if (i < N) col[i] = sm[pidx(i)];
        }
      __syncthreads();
    }
    double alpha;
    if (MODE == 2) {
      cl.sync();  // columns done before C gathers them
      alpha = *tau;
    } else {
      const double gt = cluster_sum(gam, 1);  // also orders B's stores before C's gathers
      const bool bad = rho > 0 && !(gt > 0);
      if (bad) frozen = true;
      alpha = (rho > 0 && !frozen) ? rho / gt : 0.0;
      if (bad && crank == 0 && threadIdx.x == 0 && flags) flags[bs] = 1;
    }
    const T al = (T)alpha;
    // ---- C: gather own rows' spectra, inverse row FFTs, update r (x, p) for own rows
    double rr2 = 0;
    for (int j0 = 0; j0 < npairs; j0 += G) {
      const int ra = rlo + 2 * (j0 + g);
      const bool valid = j0 + g < npairs;
      for (int q = t; q < Q; q += P) {
        V xa = V{0, 0}, xb = V{0, 0};
        if (valid) {
          const int own = q / QP;
          const V *src = cl.map_shared_rank(T1, own) + (size_t)(q - own * QP) * N;
          if (ra + 1 < rhi && pair16) {  // one 16-byte DSMEM load for the pair (FP32)
            const float4 f = *reinterpret_cast<const float4 *>(src + ra);
            xa = V{(T)f.x, (T)f.y};
            xb = V{(T)f.z, (T)f.w};
          } else {
            xa = src[ra];
            if (ra + 1 < rhi) xb = src[ra + 1];
          }
        }
        if (q == 0 || q == L / 2) { xa.y = 0; xb.y = 0; }  // real rows: DC and Nyquist are real
        sm[pidx(q)] = V{xa.x - xb.y, xa.y + xb.x};
        if (q != 0 && q != L / 2) sm[pidx(L - q)] = V{xa.x + xb.y, xb.x - xa.y};
      }
      __syncthreads();
      V v[E];
#pragma unroll
      for (int rr = 0; rr < E; ++rr) v[rr] = sm[pidx(t + rr * P)];
      __syncthreads();
      fft_group<T, L, true>(v, sm, tw, t);
      if (valid)
#pragma unroll
        for (int rr = 0; rr < E; ++rr) {
          const int n = t + rr * P;
          if (n < N) {
            const V z = sm[pidx(n)];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (ra + h >= rhi) break;
              const size_t e = so + (size_t)(ra + h) * N + n;
              const T gd = h == 0 ? z.x : z.y;
              const T ro = r[e];
              if (MODE == 0) x[e] = fma(al, p[e], x[e]);
              else x[e] = fma(al, ro, x[e]);  // SD: x += alpha r; Landweber: x += tau r
              const T rn = fma(-al, gd, ro);
              r[e] = rn;
              rr2 += (double)rn * rn;
            }
          }
        }
      __syncthreads();
    }
    const double rho_n = cluster_sum(rr2, 0);  // also: every CTA is done gathering before A scatters
    if (resid && crank == 0 && threadIdx.x == 0) resid[(size_t)bs * iters + k] = sqrt(rho_n);
    if (MODE == 0) {  // p = r + beta p, own rows
      const T be = (T)(rho > 0 ? rho_n / rho : 0.0);
      for (int i = threadIdx.x; i < (rhi - rlo) * N; i += OC_THREADS) {
        const size_t e = so + (size_t)rlo * N + i;
        p[e] = fma(be, p[e], r[e]);
      }
      __syncthreads();
    }
    rho = rho_n;
  }
  cl.sync();  // no CTA exits while another may still read its shared memory (cpart, T1)
}

// Cluster size for (T, L): the smallest of 1, 2, 4, 8 whose per-CTA share of T1 plus the FFT
// group buffers fit in 200 KB of shared memory; 0 if none (or L > 512: use the fused passes).
template <typename T, int L>
static int onchip_cs(int N, size_t *smem) {
  if (L > 512) return 0;
  const size_t grp = (size_t)OcCfg<L>::G * FftCfg<L>::SMEM * sizeof(cplx<T>);
  for (int cs = 1; cs <= 8; cs *= 2) {
    const size_t qp = (OcCfg<L>::Q + cs - 1) / cs;
    const size_t b = qp * N * sizeof(cplx<T>) + grp;
    if (b <= 200 * 1024 && (cs == 1 || N >= 2 * cs)) {
      *smem = b;
      return cs;
    }
  }
  return 0;
}

template <typename T, int L, int CS, int MODE>
static cudaError_t onchip_launch(int N, int B, int iters, const T *b, T *x, T *r, T *p, const T *S,
                                 const cplx<T> *tw, const double *tau, double *resid, int *flags, size_t smem,
                                 cudaStream_t s) {
  auto kern = onchip_kernel<T, L, CS, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, B, 1);
  cfg.blockDim = dim3(OC_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, N, iters, b, x, r, p, S, tw, tau, resid, flags);
}

template <typename T, int L, int MODE>
static cudaError_t onchip_cs_switch(int cs, int N, int B, int iters, const T *b, T *x, T *r, T *p, const T *S,
                                    const cplx<T> *tw, const double *tau, double *resid, int *flags, size_t smem,
                                    cudaStream_t s) {
  switch (cs) {
    case 1: return onchip_launch<T, L, 1, MODE>(N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
    case 2: return onchip_launch<T, L, 2, MODE>(N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
    case 4: return onchip_launch<T, L, 4, MODE>(N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
    case 8: return onchip_launch<T, L, 8, MODE>(N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int L>
static cudaError_t onchip_L(int N, int B, int iters, int mode, const T *b, T *x, T *r, T *p, const T *S,
                            const cplx<T> *tw, const double *tau, double *resid, int *flags, cudaStream_t s) {
  size_t smem = 0;
  const int cs = onchip_cs<T, L>(N, &smem);
  if (!cs) return cudaErrorNotSupported;
  switch (mode) {
    case 0: return onchip_cs_switch<T, L, 0>(cs, N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
    case 1: return onchip_cs_switch<T, L, 1>(cs, N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
    default: return onchip_cs_switch<T, L, 2>(cs, N, B, iters, b, x, r, p, S, tw, tau, resid, flags, smem, s);
  }
}

// Opt-in (BSCT_ONCHIP=1): measured on B200 (tools/time_onchip.py) this version is slower than the
// fused 3-launch iteration -- config 2 (N = 256, 50 CG iterations): 4.4 ms vs 1.6 ms for 16 slices,
// 17.9 ms vs 11.0 ms for 128 slices (16-byte DSMEM row-pair accesses; 22 ms with 8-byte ones);
// config 1 (N = 64, FP64): 0.57 vs 0.36 ms.  The block-level FFT groups, the DSMEM scatter/gather
// and three cluster barriers per iteration cost more than the HBM traffic they save at these
// sizes.  Kept as the parity-tested cluster/DSMEM design (NEXT-2, first version).
bool onchip_enabled() {
  const char *e = getenv("BSCT_ONCHIP");
  return e && e[0] == '1';
}

int onchip_cluster_size(int N, int L, bool fp32) {
  size_t smem = 0;
  switch (L) {
    case 2: return fp32 ? onchip_cs<float, 2>(N, &smem) : onchip_cs<double, 2>(N, &smem);
    case 4: return fp32 ? onchip_cs<float, 4>(N, &smem) : onchip_cs<double, 4>(N, &smem);
    case 8: return fp32 ? onchip_cs<float, 8>(N, &smem) : onchip_cs<double, 8>(N, &smem);
    case 16: return fp32 ? onchip_cs<float, 16>(N, &smem) : onchip_cs<double, 16>(N, &smem);
    case 32: return fp32 ? onchip_cs<float, 32>(N, &smem) : onchip_cs<double, 32>(N, &smem);
    case 64: return fp32 ? onchip_cs<float, 64>(N, &smem) : onchip_cs<double, 64>(N, &smem);
    case 128: return fp32 ? onchip_cs<float, 128>(N, &smem) : onchip_cs<double, 128>(N, &smem);
    case 256: return fp32 ? onchip_cs<float, 256>(N, &smem) : onchip_cs<double, 256>(N, &smem);
    case 512: return fp32 ? onchip_cs<float, 512>(N, &smem) : onchip_cs<double, 512>(N, &smem);
  }
  return 0;
}

template <typename T>
cudaError_t onchip_solve(int N, int L, int B, int iters, int mode, const T *b, T *x, T *r, T *p, const T *S,
                         const cplx<T> *tw, const double *tau, double *resid, int *flags, cudaStream_t s) {
  switch (L) {
    case 2: return onchip_L<T, 2>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 4: return onchip_L<T, 4>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 8: return onchip_L<T, 8>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 16: return onchip_L<T, 16>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 32: return onchip_L<T, 32>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 64: return onchip_L<T, 64>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 128: return onchip_L<T, 128>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 256: return onchip_L<T, 256>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
    case 512: return onchip_L<T, 512>(N, B, iters, mode, b, x, r, p, S, tw, tau, resid, flags, s);
  }
  return cudaErrorNotSupported;
}

template cudaError_t onchip_solve<float>(int, int, int, int, int, const float *, float *, float *, float *,
                                         const float *, const cplx<float> *, const double *, double *, int *,
                                         cudaStream_t);
template cudaError_t onchip_solve<double>(int, int, int, int, int, const double *, double *, double *, double *,
                                          const double *, const cplx<double> *, const double *, double *, int *,
                                          cudaStream_t);

}  // namespace bsct
