// api.cu -- the C ABI of include/bsct.h: validation, plans, launch sequencing.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/bsct.h"
#include "fft.cuh"
#include "kernels.cuh"

using namespace bsct;

namespace {

thread_local std::string g_err;

// NVTX range around every C entry point (header-only NVTX3; visible in nsys / ncu timelines)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

bsct_status fail(bsct_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? BSCT_ENOMEM : BSCT_ECUDA, "%s: %s (%s:%d)", #expr, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                          \
  } while (0)

constexpr int HC = 25;

int fft_size(int N) {
  int L = 2;
  while (L < 2 * N - 1) L *= 2;
  return L;
}

bsct_status validate(const bsct_geometry *g, bsct_dtype dt) {
  if (!g) return fail(BSCT_EINVAL, "geometry is NULL");
  if (g->N < 1 || g->N > 2048) return fail(BSCT_EINVAL, "N = %d outside [1, 2048]", g->N);
  if (dt != BSCT_F32 && dt != BSCT_F64) return fail(BSCT_EINVAL, "unknown dtype %d", (int)dt);
  if (dt == BSCT_F64 && g->N > 1024) return fail(BSCT_EINVAL, "FP64 plans support N <= 1024 (got %d)", g->N);
  if (!(g->lambda_x > 0) || !std::isfinite(g->lambda_x)) return fail(BSCT_EINVAL, "lambda_x must be > 0");
  if (!(g->lambda_y > 0) || !std::isfinite(g->lambda_y)) return fail(BSCT_EINVAL, "lambda_y must be > 0");
  if (!(g->zeta_blur >= 0) || !std::isfinite(g->zeta_blur)) return fail(BSCT_EINVAL, "zeta_blur must be >= 0");
  if (g->n_angles < 1 || g->n_angles > 65535) return fail(BSCT_EINVAL, "n_angles = %d outside [1, 65535]", g->n_angles);
  if (g->n_det < 1 || g->n_det > (1 << 20)) return fail(BSCT_EINVAL, "n_det = %d outside [1, 2^20]", g->n_det);
  if (!g->angles) return fail(BSCT_EINVAL, "angles is NULL");
  for (int i = 0; i < g->n_angles; ++i)
    if (!std::isfinite(g->angles[i])) return fail(BSCT_EINVAL, "angle %d is not finite", i);
  return BSCT_OK;
}

template <typename T>
size_t tables_bytes(int n) { return PPTables<T>::bytes(n); }

}  // namespace

struct GraphEntry {  // a captured solve: argument key -> instantiated graph
  const void *key[8];
  cudaGraphExec_t exec;
  int64_t launches;
};

struct bsct_plan_s {
  int N = 0, L = 0, n_angles = 0, M = 0, max_batch = 0;
  double lx = 1, ly = 1, zeta = 0;
  bsct_dtype dt = BSCT_F32;
  double *angles = nullptr;
  void *bp_mem = nullptr, *fw_mem = nullptr;
  void *S = nullptr, *tw = nullptr, *spec_work = nullptr;
  BPAngle *bp_ang = nullptr;  // K4 v2 per-angle parameters
  void *bp_B = nullptr;       // K4 v2 basis table
  int bp_cells = 0;           // K4 v2 tile cell capacity (0: use K4 v1)
  int bp_maxp = 9;            // K4 v2 sub-intervals per detector cell (max over angles)
  bool solver_v1 = false;     // unfused 5-launch iteration (A/B testing only)
  bool bp_v3 = true;          // FP32: K4 v3 (slices per CTA); BSCT_BP_V2=1 selects v2 (A/B testing)
  bool bp_tc = false;         // FP32: K4 v4 on the tensor cores (bp_tc.cu) where the geometry fits
  int ldt = 0;                // row stride of g~ (K4 v4: a multiple of 4 floats for TMA)
  void *gt_lo = nullptr;      // K4 v4: FP32 residual of the TF32-rounded g~
  // plain adjoint H^T and SIRT (NEXT-1): K4 tables without the interpolation widths, weights
  BPAngle *adj_ang = nullptr;
  void *adj_B = nullptr;
  void *sirt_R = nullptr, *sirt_C = nullptr, *sino_tmp = nullptr;
  void *T1 = nullptr, *gt = nullptr, *r = nullptr, *p = nullptr, *q = nullptr;
  void *sino_dev = nullptr, *b_dev = nullptr, *x_dev = nullptr;  // reconstruct_host staging
  double *alpha = nullptr, *gpart = nullptr, *rpart = nullptr, *tau = nullptr;
  double *rho = nullptr;
  int rho_iters = -1;
  int *flags = nullptr;
  int64_t launches = 0;
  // reconstruct pipeline: aux streams (BP / H2D, D2H) and per-chunk events
  cudaStream_t aux = nullptr, aux2 = nullptr, hi = nullptr;  // hi: solves, highest priority
  cudaStream_t cap = nullptr;                                  // graph capture of small solves
  std::vector<GraphEntry> graphs;
  std::vector<cudaEvent_t> pipe_ev;
  std::vector<cudaStream_t> gstreams;  // streams of the chunked solver (BSCT_CHUNK_STREAMS)
  std::vector<cudaEvent_t> gevents;
  // kernel-class profiler: CUDA events bracket every launch on the caller's stream
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_pool;
  std::vector<std::pair<int, size_t>> prof_marks;  // (class, index of the start event)
  size_t prof_used = 0;
  double prof_ms[BSCT_K_COUNT] = {};
  int64_t prof_cnt[BSCT_K_COUNT] = {};
  size_t esize() const { return dt == BSCT_F64 ? 8 : 4; }
};

namespace {

template <typename T>
PPTables<T> tables_of(void *mem, int n) {
  PPTables<T> t;
  t.carve(mem, n);
  return t;
}

cudaError_t prof_begin(bsct_plan p, int cls, cudaStream_t s) {
  if (!p->prof_on) return cudaSuccess;
  while (p->prof_pool.size() < p->prof_used + 2) {
    cudaEvent_t e;
    cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) return err;
    p->prof_pool.push_back(e);
  }
  p->prof_marks.push_back({cls, p->prof_used});
  cudaError_t err = cudaEventRecord(p->prof_pool[p->prof_used], s);
  p->prof_used += 2;
  return err;
}

cudaError_t prof_end(bsct_plan p, cudaStream_t s) {
  if (!p->prof_on) return cudaSuccess;
  return cudaEventRecord(p->prof_pool[p->prof_marks.back().second + 1], s);
}

// one library launcher call (nk kernels) of kernel class `cls`, bracketed by profiler events
#define LAUNCH(p, cls, nk, expr)    \
  do {                              \
    CU(prof_begin((p), (cls), s));  \
    CU(expr);                       \
    CU(prof_end((p), s));           \
    (p)->launches += (nk);          \
  } while (0)

bsct_status check_plan(bsct_plan p, int B) {
  if (!p) return fail(BSCT_EINVAL, "plan is NULL");
  if (B < 0) return fail(BSCT_EINVAL, "batch %d < 0", B);
  if (B > p->max_batch) return fail(BSCT_ESHAPE, "batch %d exceeds the plan's max_batch %d", B, p->max_batch);
  return BSCT_OK;
}

template <int L>
void twiddles_L(std::vector<double> &re, std::vector<double> &im) {
  re.assign(FftCfg<L>::TW_SIZE + 1, 0.0);
  im.assign(FftCfg<L>::TW_SIZE + 1, 0.0);
  fft_twiddles_host<L>(re.data(), im.data());
}

void twiddles(int L, std::vector<double> &re, std::vector<double> &im) {
  switch (L) {
    case 2: twiddles_L<2>(re, im); break;
    case 4: twiddles_L<4>(re, im); break;
    case 8: twiddles_L<8>(re, im); break;
    case 16: twiddles_L<16>(re, im); break;
    case 32: twiddles_L<32>(re, im); break;
    case 64: twiddles_L<64>(re, im); break;
    case 128: twiddles_L<128>(re, im); break;
    case 256: twiddles_L<256>(re, im); break;
    case 512: twiddles_L<512>(re, im); break;
    case 1024: twiddles_L<1024>(re, im); break;
    case 2048: twiddles_L<2048>(re, im); break;
    case 4096: twiddles_L<4096>(re, im); break;
  }
}

// Library-owned stream-ordered memory pool of device `dev` (release threshold: keep everything),
// so that the scratch of gram_build never touches the default pool other code in the process uses.
cudaError_t lib_pool(int dev, cudaMemPool_t *out) {
  static std::mutex mu;
  static std::vector<std::pair<int, cudaMemPool_t>> pools;
  std::lock_guard<std::mutex> lock(mu);
  for (auto &e : pools)
    if (e.first == dev) {
      *out = e.second;
      return cudaSuccess;
    }
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  cudaError_t e = cudaMemPoolCreate(&pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t thr = UINT64_MAX;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  if (e != cudaSuccess) return e;
  pools.push_back({dev, pool});
  *out = pool;
  return cudaSuccess;
}

// Device copies of sorted angle sets (K1's input: angles sorted by t mod pi, then the bucket
// table of gram.cu), cached per device by content so that repeated builds of the same geometry
// enqueue no host->device copy and never wait on the stream.  Least recently used entries are
// evicted beyond 64 per process; cudaFree of an evicted buffer waits for the device, so no
// kernel still in flight can be reading it.
constexpr int GRAM_NB = 4096;  // buckets of [0, pi)

struct AngleSet {
  int dev;
  std::vector<double> key;
  double *dptr;
  uint64_t used;
};

cudaError_t gram_angles(int dev, const std::vector<double> &key, const std::vector<double> &sorted,
                        const std::vector<int> &bucket, double **out) {
  static std::mutex mu;
  static std::vector<AngleSet> cache;
  static uint64_t tick = 0;
  std::lock_guard<std::mutex> lock(mu);
  ++tick;
  for (auto &e : cache)
    if (e.dev == dev && e.key == key) {
      e.used = tick;
      *out = e.dptr;
      return cudaSuccess;
    }
  if (cache.size() >= 64) {
    auto lru = std::min_element(cache.begin(), cache.end(), [](auto &x, auto &y) { return x.used < y.used; });
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(lru->dev);
    cudaFree(lru->dptr);
    cudaSetDevice(cur);
    cache.erase(lru);
  }
  const size_t n = sorted.size();
  double *d = nullptr;
  cudaError_t e = cudaMalloc((void **)&d, sizeof(double) * n + sizeof(int) * bucket.size());
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(d, sorted.data(), sizeof(double) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, bucket.data(), sizeof(int) * bucket.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d);
    return e;
  }
  cache.push_back({dev, key, d, tick});
  *out = d;
  return cudaSuccess;
}

template <typename T>
bsct_status gram_build_t(const bsct_geometry *g, int a0, int a1, T *taps, cudaStream_t s) {
  const int n = a1 - a0;
  const int N = g->N;
  const size_t D2 = (size_t)(2 * N - 1) * (2 * N - 1);
  if (n == 0) {
    CU(cudaMemsetAsync(taps, 0, D2 * sizeof(T), s));
    return BSCT_OK;
  }
  int dev = 0;
  CU(cudaGetDevice(&dev));
  const char *dense_env = getenv("BSCT_GRAM_DENSE");
  const bool dense = dense_env && dense_env[0] == '1';
  // angles of the shard sorted by t mod pi (K1's windows are runs of this order); the key is
  // the shard's angles in the given order
  const double pi = 3.141592653589793238462643383279502884;
  std::vector<double> key(g->angles + a0, g->angles + a1);
  std::vector<std::pair<double, double>> srt(n);
  for (int i = 0; i < n; ++i) {
    const double t = key[i];
    double m = t - pi * std::floor(t / pi);
    srt[i] = {std::min(std::max(m, 0.0), std::nextafter(pi, 0.0)), t};
  }
  std::stable_sort(srt.begin(), srt.end(), [](auto &x, auto &y) { return x.first < y.first; });
  std::vector<double> sorted(n);
  std::vector<int> bucket(GRAM_NB + 1);
  for (int i = 0; i < n; ++i) sorted[i] = srt[i].second;
  for (int k = 0, i = 0; k <= GRAM_NB; ++k) {  // bucket[k] = #{sorted: (t mod pi) < k pi / NB}
    const double edge = k * (pi / GRAM_NB);
    while (i < n && (k == GRAM_NB || srt[i].first < edge)) ++i;
    bucket[k] = i;
  }
  // angular density for K1's tile levels: the fullest pi / 16 window (with wrap) x 16; a set spread
  // over [0, pi) keeps n, an angle shard (config 4: a wedge of the angle range) gets ~n pi / wedge
  double n_dens = n;
  {
    const int W = GRAM_NB / 16;
    int most = 0;
    for (int k = 0; k < GRAM_NB; ++k) {
      const int e = k + W;
      const int c = e <= GRAM_NB ? bucket[e] - bucket[k] : (n - bucket[k]) + bucket[e - GRAM_NB];
      most = std::max(most, c);
    }
    if (16.0 * most > 1.5 * n) n_dens = 16.0 * most;
  }
  double *ang = nullptr;
  CU(gram_angles(dev, key, sorted, bucket, &ang));
  const int *bk = (const int *)(ang + n);
  cudaMemPool_t pool;
  CU(lib_pool(dev, &pool));
  void *mem = nullptr;
  const size_t tb_bytes = (tables_bytes<T>(n) + 255) & ~(size_t)255;
  CU(cudaMallocFromPoolAsync(&mem, tb_bytes + sizeof(T) * (size_t)n * GR_WORDS, pool, s));
  PPTables<T> tb = tables_of<T>(mem, n);
  tb.grec = (T *)((char *)mem + tb_bytes);
  CU(build_pp_tables<T>(ang, n, PP_GRAM, g->lambda_x, g->lambda_y, g->zeta_blur, tb, s));
  const double Hmax = (g->lambda_x * 1.4142135623730951 + g->zeta_blur) * (1.0 + 1e-12);
  CU(gram_build_tiles<T>(N, g->lambda_x, n, n_dens, tb.grec, bk, GRAM_NB, Hmax, dense, taps, s));
  CU(cudaFreeAsync(mem, s));
  return BSCT_OK;
}

template <typename T>
bsct_status plan_filter_t(bsct_plan p, const void *taps, cudaStream_t s) {
  const int N = p->N, L = p->L, n = p->n_angles;
  PPTables<T> bp = tables_of<T>(p->bp_mem, n), fw = tables_of<T>(p->fw_mem, n);
  LAUNCH(p, BSCT_K_TABLES, 1, (build_pp_tables<T>(p->angles, n, PP_BP, p->lx, p->ly, p->zeta, bp, s)));
  LAUNCH(p, BSCT_K_TABLES, 1, (build_pp_tables<T>(p->angles, n, PP_FWD, p->lx, p->ly, p->zeta, fw, s)));
  if (p->bp_cells > 0)
    LAUNCH(p, BSCT_K_TABLES, 1,
           (build_bp_tables<T>(N, p->M, p->lx, p->ly, p->zeta, n, bp, p->bp_ang, (T *)p->bp_B, s, 1)));
  LAUNCH(p, BSCT_K_SPECTRUM, 2,
         (filter_spectrum<T>(N, L, (const T *)taps, (T *)p->S, (cplx<T> *)p->spec_work, (const cplx<T> *)p->tw, s)));
  LAUNCH(p, BSCT_K_SPECTRUM, 2, (spectrum_max<T>(L, (const T *)p->S, p->tau, s)));
  return BSCT_OK;
}

template <typename T>
bsct_status plan_init_t(bsct_plan p, const void *taps, cudaStream_t s) {
  const int N = p->N, L = p->L, n = p->n_angles, M = p->M, Bm = p->max_batch;
  const size_t Q = L / 2 + 1;
  CU(cudaMalloc(&p->bp_mem, tables_bytes<T>(n)));
  CU(cudaMalloc(&p->fw_mem, tables_bytes<T>(n)));
  // FFT twiddles
  std::vector<double> re, im;
  twiddles(L, re, im);
  std::vector<cplx<T>> twh(re.size());
  for (size_t i = 0; i < re.size(); ++i) twh[i] = cplx<T>{(T)re[i], (T)im[i]};
  CU(cudaMalloc(&p->tw, sizeof(cplx<T>) * twh.size()));
  CU(cudaMemcpyAsync(p->tw, twh.data(), sizeof(cplx<T>) * twh.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMalloc(&p->S, sizeof(T) * Q * L));
  CU(cudaMalloc(&p->spec_work, sizeof(cplx<T>) * Q * L));
  CU(cudaMalloc((void **)&p->tau, sizeof(double) * 256));  // [0] tau, [1..148] partial maxima
  const char *force_v1 = getenv("BSCT_BP_V1");
  p->bp_cells = (force_v1 && force_v1[0] == '1') ? 0 : bp_v2_max_cells(p->lx, p->ly, p->zeta);
  if (p->bp_cells > 0) {
    // K4 v2's double-buffered tables must fit in shared memory (fine detectors, lambda_y << lambda_x,
    // have many cells per tile); otherwise K4 v1 (direct per-sample evaluation)
    const size_t buf = (size_t)p->bp_cells * (p->bp_maxp * 8 + 4) + p->bp_maxp * BP_SMAX * 8 +
                       ((p->bp_cells + BP_SMAX + 7) & ~7);
    if (p->esize() * 2 * buf > 227 * 1024) p->bp_cells = 0;
  }
  const char *bp2 = getenv("BSCT_BP_V2");
  p->bp_v3 = !(bp2 && bp2[0] == '1');
  if (p->bp_cells > 0) {
    CU(cudaMalloc((void **)&p->bp_ang, sizeof(BPAngle) * n + 64));  // + 64: K4 v4 stages 16-byte aligned copies
    CU(cudaMalloc(&p->bp_B, sizeof(T) * bp_table_floats(n)));
  }
  bsct_status st = plan_filter_t<T>(p, taps, s);
  if (st != BSCT_OK) return st;
  // workspaces
  const size_t nn = (size_t)N * N;
  const size_t Bz = Bm > 0 ? Bm : 1;
  CU(cudaMalloc(&p->T1, sizeof(cplx<T>) * Q * N * Bz));
  p->ldt = p->bp_tc ? ((M + 2 * HC + 3) & ~3) : (M + 2 * HC);
  CU(cudaMalloc(&p->gt, sizeof(T) * (size_t)n * p->ldt * Bz));
  if (p->bp_tc) CU(cudaMalloc(&p->gt_lo, sizeof(T) * (size_t)n * p->ldt * Bz));
  CU(cudaMalloc(&p->r, sizeof(T) * nn * Bz));
  CU(cudaMalloc(&p->p, sizeof(T) * nn * Bz));
  CU(cudaMalloc(&p->q, sizeof(T) * nn * Bz));
  CU(cudaMalloc((void **)&p->alpha, sizeof(double) * Bz));
  // gamma partials: room for either pass-B layout (BSCT_PASSB_V1 is read per call)
  CU(cudaMalloc((void **)&p->gpart, sizeof(double) * Bz * std::max(pass_b_blocks(L, false), pass_b_blocks(L, true))));
  // <r,r> partials: room for either pass layout (the warp passes use more CTAs per slice)
  const size_t nrp = std::max((size_t)vec_blocks(N), (size_t)2 * (fused_parts(N, L, false) + fused_parts(N, L, true)));
  CU(cudaMalloc((void **)&p->rpart, sizeof(double) * Bz * nrp));
  const char *sv1 = getenv("BSCT_SOLVER_V1");
  p->solver_v1 = sv1 && sv1[0] == '1';
  CU(cudaMalloc((void **)&p->flags, sizeof(int) * Bz));
  CU(cudaStreamSynchronize(s));
  return BSCT_OK;
}

SolverWork solver_work(bsct_plan p, double *resid, int *flags) {
  SolverWork w;
  w.rho = p->rho;
  w.alpha = p->alpha;
  w.gpart = p->gpart;
  w.gstride = pass_b_blocks(p->L, p->dt == BSCT_F32);
  w.rpart = p->rpart;
  w.rstride = vec_blocks(p->N);
  w.flags = flags ? flags : p->flags;
  w.resid = resid;
  w.tau = p->tau;
  return w;
}

template <typename T>
bsct_status normal_apply_t(bsct_plan p, const T *x, T *y, int B, double *gpart, cudaStream_t s) {
  auto *T1 = (cplx<T> *)p->T1;
  auto *tw = (const cplx<T> *)p->tw;
  // warp-level passes A and C at L = 512 / 1024 / 2048 (pass B dispatches itself)
  const bool warp = std::is_same<T, float>::value && pass_c_warp_enabled() &&
                    (p->L == 1024 || p->L == 512 || p->L == 2048);
  const bool warpc = warp;
  if (warp)
    LAUNCH(p, BSCT_K_PASS_A, 1, (warp_apply_a(p->N, p->L, B, (const float *)x, (float2 *)T1, s)));
  else
    LAUNCH(p, BSCT_K_PASS_A, 1, (pass_a<T>(p->N, p->L, B, x, T1, tw, s)));
  LAUNCH(p, BSCT_K_PASS_B, 1, (pass_b<T>(p->N, p->L, B, T1, (const T *)p->S, tw, gpart, s)));
  if (warpc)
    LAUNCH(p, BSCT_K_PASS_C, 1, (warp_apply_c(p->N, p->L, B, (const float2 *)T1, (float *)y, s)));
  else
    LAUNCH(p, BSCT_K_PASS_C, 1, (pass_c<T>(p->N, p->L, B, T1, y, tw, s)));
  return BSCT_OK;
}

template <typename T>
bsct_status backproject_t(bsct_plan p, const T *sino, T *b, int B, cudaStream_t s) {
  PPTables<T> bp = tables_of<T>(p->bp_mem, p->n_angles);
  if (std::is_same<T, float>::value && p->bp_tc && p->bp_cells > 0) {
    // K4 v4: the TF32 split of g~ (hi into gt, residual into gt_lo, rows padded to ldt for TMA), then
    // the tensor-core product per angle (bp_tc.cu)
    LAUNCH(p, BSCT_K_CORRECTION, 1,
           (correction_filter<T>(p->n_angles, p->M, B, bp.degree, sino, (T *)p->gt, s, (T *)p->gt_lo, p->ldt)));
    LAUNCH(p, BSCT_K_BACKPROJECT, 1,
           (backproject_tc(p->N, p->n_angles, p->M, B, p->bp_ang, (const float *)p->bp_B, (const float *)p->gt,
                           (const float *)p->gt_lo, p->ldt, (float *)b, p->lx * p->lx * p->ly, p->bp_maxp, s)));
    return BSCT_OK;
  }
  LAUNCH(p, BSCT_K_CORRECTION, 1, (correction_filter<T>(p->n_angles, p->M, B, bp.degree, sino, (T *)p->gt, s)));
  const int sb = (p->bp_cells > 0 && p->bp_v3 && std::is_same<T, float>::value)
                     ? bp_v3_slices(B, p->bp_maxp, p->bp_cells) : 0;
  if (sb > 0) {
    LAUNCH(p, BSCT_K_BACKPROJECT, 1,
           (backproject_v3(p->N, p->n_angles, p->M, B, p->bp_ang, (const float *)p->bp_B, (const float *)p->gt,
                           (float *)b, p->bp_cells, p->bp_maxp, p->lx * p->lx * p->ly, sb, s)));
  } else if (p->bp_cells > 0)
    LAUNCH(p, BSCT_K_BACKPROJECT, 1,
           (backproject_v2<T>(p->N, p->n_angles, p->M, B, p->bp_ang, (const T *)p->bp_B, (const T *)p->gt, b,
                              p->bp_cells, p->bp_maxp, p->lx * p->lx * p->ly, s)));
  else
    LAUNCH(p, BSCT_K_BACKPROJECT, 1,
           (backproject<T>(p->N, p->lx, p->ly, p->n_angles, p->M, B, bp.cs, bp.view(), (const T *)p->gt, b, s)));
  return BSCT_OK;
}

// Slices per solver chunk.  Default for the FP32 L = 1024 warp passes (config 5): chunks of
// SOLVE_CHUNK slices solved on SOLVE_STREAMS streams at once (chunk k on stream k % streams, all
// its iterations back to back, the whole schedule captured into one CUDA graph): the 12 slices in
// flight keep their x, r, p and T1 (61 MB) resident in the 126 MB L2, and the concurrent chunks fill
// each other's kernel tails.  Measured on B200 (config 5, 2048 slices x 50 CG iterations, DIT
// FFTs): 372 -> 325 ms (chunks of 2-4 on 3-6 streams within 2%; 1 stream or chunks >= 8 slower,
// profiles/r02/chunks_v4.txt).  BSCT_CG_CHUNK forces a chunk size (0 = whole batch),
// BSCT_L2_BUDGET_MB sizes chunks to an L2 budget, BSCT_CHUNK_STREAMS sets the streams.  The
// kernel-class profiler (prof_on) always sees the plain whole-batch launches.
constexpr int SOLVE_CHUNK = 3, SOLVE_STREAMS = 4;

bool default_chunking(bsct_plan p, int B) {
  return p->dt == BSCT_F32 && p->L == 1024 && !p->prof_on && B >= 8 * SOLVE_CHUNK && pass_c_warp_enabled() &&
         pass_b_warp_enabled() && !p->solver_v1;
}

int solver_chunk(bsct_plan p, int B) {
  if (const char *e = getenv("BSCT_CG_CHUNK")) {
    const int c = atoi(e);
    return c <= 0 ? std::max(B, 1) : std::min(c, std::max(B, 1));
  }
  double budget = 0.0;
  if (const char *e = getenv("BSCT_L2_BUDGET_MB")) budget = atof(e);
  if (budget <= 0) return default_chunking(p, B) ? SOLVE_CHUNK : std::max(B, 1);
  const double per = (double)p->esize() * (3.0 * p->N * p->N + 2.0 * (p->L / 2 + 1) * p->N);
  const int c = (int)(budget * 1048576.0 / per);
  return std::max(1, std::min(c, std::max(B, 1)));
}

int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// Streams of the chunked solve (chunk size cb < B): chunk k runs on stream k % ns
int chunk_streams(bsct_plan p, int cb, int B) {
  if (cb >= B) return 1;
  return std::min(std::max(env_int("BSCT_CHUNK_STREAMS", default_chunking(p, B) ? SOLVE_STREAMS : 1), 1), 8);
}

template <typename T>
bsct_status solve_launch_t(bsct_plan p, const T *b, T *x, int B, int iters, int solver, double *resid, int *flags,
                           cudaStream_t s);

bsct_status clear_graphs(bsct_plan p) {
  for (auto &gk : p->graphs) cudaGraphExecDestroy(gk.exec);
  p->graphs.clear();
  return BSCT_OK;
}

// Small problems (B N^2 <= 2^22 values, profiler off) are launch bound: the whole solve (init,
// 3 launches per iteration, finish) is captured once per argument set into a CUDA graph on a
// plan-owned stream and replayed on the caller's stream (BSCT_GRAPH=0: plain launches).
template <typename T>
bsct_status solve_t(bsct_plan p, const T *b, T *x, int B, int iters, int solver, double *resid, int *flags,
                    cudaStream_t s) {
  if (p->rho_iters < iters) {
    if (p->rho) CU(cudaFree(p->rho));
    p->rho = nullptr;
    CU(cudaMalloc((void **)&p->rho, sizeof(double) * (size_t)(iters + 1) * (p->max_batch > 0 ? p->max_batch : 1)));
    p->rho_iters = iters;
    clear_graphs(p);  // captured graphs hold the old rho pointer
  }
  const char *ge = getenv("BSCT_GRAPH");
  // chunked solves on several streams (L2-resident chunks) launch thousands of small kernels:
  // captured as well, so that the host enqueue does not bound them
  const int cb = solver_chunk(p, B);
  const int ns = chunk_streams(p, cb, B);
  // the persistent solver is 3 launches per solve: nothing to capture
  const bool persist = !p->solver_v1 && persist_enabled(p->L, p->dt == BSCT_F32, B, solver == BSCT_CG);
  const bool graph = !(ge && ge[0] == '0') && !p->prof_on && !persist &&
                     ((size_t)B * p->N * p->N <= ((size_t)1 << 22) || ns > 1);
  if (!graph) return solve_launch_t<T>(p, b, x, B, iters, solver, resid, flags, s);
  // the key includes every switch that selects the launched code path
  const intptr_t path = (onchip_enabled() ? 1 : 0) | (pass_b_warp_enabled() ? 2 : 0) | (pass_c_warp_enabled() ? 4 : 0) |
                        (bulk_stage_enabled() ? 8 : 0) | (p->solver_v1 ? 16 : 0) |
                        ((intptr_t)cb << 8) | ((intptr_t)ns << 40);
  const void *key[8] = {b, x, (const void *)(intptr_t)B, (const void *)(intptr_t)iters,
                        (const void *)(intptr_t)solver, resid, flags, (const void *)path};
  for (auto &gk : p->graphs)
    if (std::equal(key, key + 8, gk.key)) {
      CU(cudaGraphLaunch(gk.exec, s));
      p->launches = gk.launches;
      return BSCT_OK;
    }
  if (!p->cap) CU(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
  (void)tw1024_table();  // any lazy device allocation happens before capture
  (void)tw2048_table();
  CU(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
  p->launches = 0;
  bsct_status st = solve_launch_t<T>(p, b, x, B, iters, solver, resid, flags, p->cap);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(p->cap, &g);
  if (st != BSCT_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  CU(e);
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  CU(e);
  if (p->graphs.size() >= 16) {
    cudaGraphExecDestroy(p->graphs.front().exec);
    p->graphs.erase(p->graphs.begin());
  }
  GraphEntry gk;
  std::copy(key, key + 8, gk.key);
  gk.exec = ex;
  gk.launches = p->launches;
  p->graphs.push_back(gk);
  CU(cudaGraphLaunch(ex, s));
  return BSCT_OK;
}

template <typename T>
bsct_status solve_launch_t(bsct_plan p, const T *b, T *x, int B, int iters, int solver, double *resid, int *flags,
                           cudaStream_t s) {
  T *r = (T *)p->r, *pp = (T *)p->p, *q = (T *)p->q;
  if (!p->solver_v1 && onchip_enabled() && onchip_cluster_size(p->N, p->L, p->dt == BSCT_F32) > 0) {
    // NEXT-2: small N -- one thread-block cluster per slice runs every iteration on chip
    LAUNCH(p, BSCT_K_FUSED_CG, 1,
           (onchip_solve<T>(p->N, p->L, B, iters, solver, b, x, r, pp, (const T *)p->S, (const cplx<T> *)p->tw,
                            p->tau, resid, flags ? flags : p->flags, s)));
    return BSCT_OK;
  }
  if (!p->solver_v1) {
    // fused iteration (cg.cu): 3 launches per iteration.  Slices are solved in chunks whose
    // per-iteration working set (x, r, p, T1) stays resident in L2, so that the FFT
    // intermediates and the CG vectors cycle through L2 instead of HBM.
    const int nparts = fused_parts(p->N, p->L, p->dt == BSCT_F32);
    const int cb = solver_chunk(p, B);
    auto *T1 = (cplx<T> *)p->T1;
    auto *tw = (const cplx<T> *)p->tw;
    const int gparts = pass_b_blocks(p->L, p->dt == BSCT_F32);
    const size_t nn = (size_t)p->N * p->N;
    const size_t t1s = (size_t)(p->L / 2 + 1) * p->N;  // T1 entries per slice
    // launch j (0: init, 1 + 3 it + {0, 1, 2}: passes A, B, C of iteration it, 3 iters + 1:
    // final) of the chunk of nb slices from slice c0, on stream s; ws: workspaces at the chunk's
    // own offsets (concurrent groups) or shared (sequential chunks)
    const int nlaunch = 3 * iters + 2;
    if constexpr (std::is_same<T, float>::value) {
      if (persist_enabled(p->L, true, B, solver == BSCT_CG)) {
        // small batches at L = 2048: init, every iteration in one cooperative launch, finish
        FusedWork fw;
        fw.rho = p->rho;
        fw.rho_stride = iters + 1;
        fw.alpha = p->alpha;
        fw.gpart = p->gpart;
        fw.rpart = p->rpart;
        fw.nparts = nparts;
        fw.B = B;
        fw.flags = flags ? flags : p->flags;
        fw.resid = resid;
        fw.iters = iters;
        fw.tau = p->tau;
        LAUNCH(p, BSCT_K_SOLVER_INIT, 1, (fused_init<T>(p->N, B, b, x, r, pp, fw, s)));
        LAUNCH(p, BSCT_K_FUSED_CG, 1,
               (persist_cg_2048(p->N, B, iters, x, r, pp, T1, (const float *)p->S, fw, gparts, s)));
        LAUNCH(p, BSCT_K_SOLVER_FINISH, 1, (fused_final<T>(p->N, B, iters, 1, x, pp, fw, s)));
        return BSCT_OK;
      }
    }
    auto launch = [&](int c0, int nb, bool ws, int j, cudaStream_t s) -> bsct_status {
      const T *bc = b + c0 * nn;
      T *xc = x + c0 * nn;
      T *rc = ws ? r + c0 * nn : r, *pc = ws ? pp + c0 * nn : pp;
      cplx<T> *T1c = ws ? T1 + c0 * t1s : T1;
      FusedWork fw;
      fw.rho = p->rho + (size_t)c0 * (iters + 1);
      fw.rho_stride = iters + 1;
      fw.alpha = p->alpha + c0;
      fw.gpart = ws ? p->gpart + (size_t)c0 * gparts : p->gpart;
      fw.rpart = ws ? p->rpart + (size_t)2 * c0 * nparts : p->rpart;
      fw.nparts = nparts;
      fw.B = nb;
      fw.flags = (flags ? flags : p->flags) + c0;
      fw.resid = resid ? resid + (size_t)c0 * iters : nullptr;
      fw.iters = iters;
      fw.tau = p->tau;
      if (j == 0) {
        LAUNCH(p, BSCT_K_SOLVER_INIT, 1,
               (fused_init<T>(p->N, nb, bc, xc, rc, solver == BSCT_CG ? pc : (T *)nullptr, fw, s)));
      } else if (j == nlaunch - 1) {
        LAUNCH(p, BSCT_K_SOLVER_FINISH, 1, (fused_final<T>(p->N, nb, iters, solver == BSCT_CG, xc, pc, fw, s)));
      } else {
        const int it = (j - 1) / 3, ph = (j - 1) % 3;
        if (ph == 0) {
          if (solver == BSCT_CG)
            LAUNCH(p, BSCT_K_PASS_A, 1, (fused_pass_a<T>(p->N, p->L, nb, it, xc, rc, pc, T1c, tw, fw, s)));
          else
            LAUNCH(p, BSCT_K_PASS_A, 1, (pass_a<T>(p->N, p->L, nb, rc, T1c, tw, s)));
        } else if (ph == 1) {
          LAUNCH(p, BSCT_K_PASS_B, 1,
                 (pass_b<T>(p->N, p->L, nb, T1c, (const T *)p->S, tw, solver == BSCT_LANDWEBER ? nullptr : fw.gpart, s)));
        } else {
          LAUNCH(p, BSCT_K_PASS_C, 1, (fused_pass_c<T>(p->N, p->L, nb, it, solver, gparts, T1c, xc, rc, tw, fw, s)));
        }
      }
      return BSCT_OK;
    };
    const int ns = chunk_streams(p, cb, B);
    if (ns > 1) {
      // L2-resident chunks on ns streams: chunk k runs all its iterations on stream k % ns, with
      // its own workspace slices, so that ns chunks are in flight and fill each other's tails
      while ((int)p->gstreams.size() < ns) {
        cudaStream_t gs = nullptr;
        CU(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
        p->gstreams.push_back(gs);
      }
      while ((int)p->gevents.size() < 1 + ns) {
        cudaEvent_t e = nullptr;
        CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p->gevents.push_back(e);
      }
      CU(cudaEventRecord(p->gevents[0], s));
      for (int i = 0; i < ns; ++i) CU(cudaStreamWaitEvent(p->gstreams[i], p->gevents[0], 0));
      const int nch = (B + cb - 1) / cb;
      for (int k0 = 0; k0 < nch; k0 += ns)
        for (int j = 0; j < nlaunch; ++j)
          for (int k = k0; k < std::min(nch, k0 + ns); ++k) {
            bsct_status st = launch(k * cb, std::min(cb, B - k * cb), true, j, p->gstreams[k % ns]);
            if (st != BSCT_OK) return st;
          }
      for (int i = 0; i < ns; ++i) {
        CU(cudaEventRecord(p->gevents[1 + i], p->gstreams[i]));
        CU(cudaStreamWaitEvent(s, p->gevents[1 + i], 0));
      }
      return BSCT_OK;
    }
    for (int c0 = 0; c0 < B; c0 += cb)
      for (int j = 0; j < nlaunch; ++j) {
        bsct_status st = launch(c0, std::min(cb, B - c0), false, j, s);
        if (st != BSCT_OK) return st;
      }
    return BSCT_OK;
  }
  SolverWork w = solver_work(p, resid, flags);
  // rho rows have stride (iters + 1): the kernels index rho[b * (iters+1) + k]
  LAUNCH(p, BSCT_K_SOLVER_INIT, 2, (solver_init<T>(p->N, B, b, x, r, solver == BSCT_CG ? pp : (T *)nullptr, w, iters, s)));
  for (int it = 0; it < iters; ++it) {
    const T *d = solver == BSCT_CG ? pp : r;
    bsct_status st = normal_apply_t<T>(p, d, q, B, solver == BSCT_LANDWEBER ? nullptr : p->gpart, s);
    if (st != BSCT_OK) return st;
    LAUNCH(p, BSCT_K_SOLVER_UPDATE, 1, (solver_update<T>(p->N, B, solver, it, iters, x, r, pp, q, w, s)));
    LAUNCH(p, BSCT_K_SOLVER_FINISH, 1, (solver_finish<T>(p->N, B, solver, it, iters, r, pp, w, s)));
  }
  return BSCT_OK;
}

// Resume a solve from a saved state (x_j, r_j, p_j) for `iters` more iterations on the fused
// passes (the same kernels as solve_launch_t), then export (r, p) of the final state in place.
template <typename T>
bsct_status resume_t(bsct_plan p, T *x, T *r_io, T *p_io, int B, int iters, int solver, double *alpha_out,
                     double *resid, int *flags, cudaStream_t s) {
  if (p->rho_iters < iters) {
    if (p->rho) CU(cudaFree(p->rho));
    p->rho = nullptr;
    CU(cudaMalloc((void **)&p->rho, sizeof(double) * (size_t)(iters + 1) * (p->max_batch > 0 ? p->max_batch : 1)));
    p->rho_iters = iters;
    clear_graphs(p);
  }
  const bool cg = solver == BSCT_CG;
  T *r = (T *)p->r, *pp = (T *)p->p, *q = (T *)p->q;
  auto *T1 = (cplx<T> *)p->T1;
  auto *tw = (const cplx<T> *)p->tw;
  FusedWork fw;
  fw.rho = p->rho;
  fw.rho_stride = iters + 1;
  fw.alpha = p->alpha;
  fw.gpart = p->gpart;
  fw.rpart = p->rpart;
  fw.nparts = fused_parts(p->N, p->L, p->dt == BSCT_F32);
  fw.B = B;
  fw.flags = flags ? flags : p->flags;
  fw.resid = resid;
  fw.iters = iters;
  fw.tau = p->tau;
  const int gparts = pass_b_blocks(p->L, p->dt == BSCT_F32);
  LAUNCH(p, BSCT_K_SOLVER_INIT, 1, (fused_resume<T>(p->N, B, r_io, cg ? p_io : (const T *)nullptr, r, cg ? pp : nullptr, q, fw, s)));
  CU(cudaMemsetAsync(p->alpha, 0, sizeof(double) * B, s));
  for (int it = 0; it < iters; ++it) {
    if (cg)  // first resumed iteration: beta = alpha_prev = 0 and the "r" operand q = p_j, so p = p_j
      LAUNCH(p, BSCT_K_PASS_A, 1, (fused_pass_a<T>(p->N, p->L, B, it, x, it == 0 ? q : r, pp, T1, tw, fw, s)));
    else
      LAUNCH(p, BSCT_K_PASS_A, 1, (pass_a<T>(p->N, p->L, B, r, T1, tw, s)));
    LAUNCH(p, BSCT_K_PASS_B, 1,
           (pass_b<T>(p->N, p->L, B, T1, (const T *)p->S, tw, solver == BSCT_LANDWEBER ? nullptr : p->gpart, s)));
    LAUNCH(p, BSCT_K_PASS_C, 1, (fused_pass_c<T>(p->N, p->L, B, it, solver, gparts, T1, x, r, tw, fw, s)));
  }
  LAUNCH(p, BSCT_K_SOLVER_FINISH, 1, (fused_final<T>(p->N, B, iters, cg, x, pp, fw, s)));
  LAUNCH(p, BSCT_K_SOLVER_FINISH, 1, (fused_export<T>(p->N, B, iters, r, pp, r_io, cg ? p_io : nullptr, fw, s)));
  if (alpha_out) CU(cudaMemcpyAsync(alpha_out, p->alpha, sizeof(double) * B, cudaMemcpyDeviceToDevice, s));
  return BSCT_OK;
}

template <typename T>
bsct_status forward_t(bsct_plan p, const T *c, T *sino, int B, cudaStream_t s) {
  PPTables<T> fw = tables_of<T>(p->fw_mem, p->n_angles);
  // the plan's q workspace holds the transposed image (it is free outside a solve; SIRT overwrites
  // it only after the forward projection)
  LAUNCH(p, BSCT_K_FORWARD, 2,
         (forward_project<T>(p->N, p->lx, p->ly, p->n_angles, p->M, B, fw.cs, fw.view(), c, sino, s, (T *)p->q)));
  return BSCT_OK;
}

// ---- NEXT-1: plain adjoint H^T (K4 machinery with the forward model's kernel) and SIRT
template <typename T>
bsct_status adjoint_core(bsct_plan p, const T *gt, T *out, int B, cudaStream_t s) {
  const double scale = p->lx * p->lx;  // H[(t,m), k] = lambda_x^2 M_[l|c|, l|s|, zeta](y_m - k_t)
  const int sb = (std::is_same<T, float>::value && p->bp_v3) ? bp_v3_slices(B, p->bp_maxp, p->bp_cells) : 0;
  if (sb > 0)
    LAUNCH(p, BSCT_K_BACKPROJECT, 1,
           (backproject_v3(p->N, p->n_angles, p->M, B, p->adj_ang, (const float *)p->adj_B, (const float *)gt,
                           (float *)out, p->bp_cells, p->bp_maxp, scale, sb, s, 3)));
  else
    LAUNCH(p, BSCT_K_BACKPROJECT, 1,
           (backproject_v2<T>(p->N, p->n_angles, p->M, B, p->adj_ang, (const T *)p->adj_B, gt, out, p->bp_cells,
                              p->bp_maxp, scale, s)));
  return BSCT_OK;
}

template <typename T>
bsct_status adjoint_tables(bsct_plan p, cudaStream_t s) {
  if (p->adj_ang) return BSCT_OK;
  if (p->bp_cells <= 0) return fail(BSCT_EINVAL, "adjoint/SIRT need a geometry supported by K4 v2/v3");
  CU(cudaMalloc((void **)&p->adj_ang, sizeof(BPAngle) * p->n_angles));
  CU(cudaMalloc(&p->adj_B, sizeof(T) * bp_table_floats(p->n_angles)));
  PPTables<T> bp = tables_of<T>(p->bp_mem, p->n_angles);
  LAUNCH(p, BSCT_K_TABLES, 1,
         (build_bp_tables<T>(p->N, p->M, p->lx, p->ly, p->zeta, p->n_angles, bp, p->adj_ang, (T *)p->adj_B, s, 0)));
  return BSCT_OK;
}

template <typename T>
bsct_status adjoint_t(bsct_plan p, const T *sino, T *out, int B, cudaStream_t s) {
  bsct_status st = adjoint_tables<T>(p, s);
  if (st != BSCT_OK) return st;
  LAUNCH(p, BSCT_K_CORRECTION, 1, (pad_rows<T>(p->n_angles, p->M, B, sino, nullptr, nullptr, (T *)p->gt, s)));
  return adjoint_core<T>(p, (const T *)p->gt, out, B, s);
}

template <typename T>
bsct_status sirt_weights(bsct_plan p, cudaStream_t s) {
  if (p->sirt_R) return BSCT_OK;
  const size_t ns = (size_t)p->n_angles * p->M, nn = (size_t)p->N * p->N;
  CU(cudaMalloc(&p->sirt_R, sizeof(T) * ns));
  CU(cudaMalloc(&p->sirt_C, sizeof(T) * nn));
  T *ones_img = nullptr, *ones_sino = nullptr;
  CU(cudaMallocAsync((void **)&ones_img, sizeof(T) * nn, s));
  CU(cudaMallocAsync((void **)&ones_sino, sizeof(T) * ns, s));
  std::vector<T> h1(std::max(ns, nn), (T)1);
  CU(cudaMemcpyAsync(ones_img, h1.data(), sizeof(T) * nn, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(ones_sino, h1.data(), sizeof(T) * ns, cudaMemcpyHostToDevice, s));
  bsct_status st = forward_t<T>(p, ones_img, (T *)p->sirt_R, 1, s);  // row sums H 1
  if (st == BSCT_OK) st = adjoint_t<T>(p, ones_sino, (T *)p->sirt_C, 1, s);  // column sums H^T 1
  if (st != BSCT_OK) return st;
  CU(safe_reciprocal<T>((long)ns, (T *)p->sirt_R, s));
  CU(safe_reciprocal<T>((long)nn, (T *)p->sirt_C, s));
  CU(cudaStreamSynchronize(s));  // h1 is a host temporary
  CU(cudaFreeAsync(ones_img, s));
  CU(cudaFreeAsync(ones_sino, s));
  return BSCT_OK;
}

// x_{k+1} = x_k + C H^T R (g - H x_k), x_0 = 0 (oracle/sirt.py)
template <typename T>
bsct_status sirt_t(bsct_plan p, const T *sino, T *x, int B, int iters, cudaStream_t s) {
  bsct_status st = adjoint_tables<T>(p, s);
  if (st == BSCT_OK) st = sirt_weights<T>(p, s);
  if (st != BSCT_OK) return st;
  const size_t ns = (size_t)p->n_angles * p->M, nn = (size_t)p->N * p->N;
  if (!p->sino_tmp) CU(cudaMalloc(&p->sino_tmp, sizeof(T) * ns * p->max_batch));
  CU(cudaMemsetAsync(x, 0, sizeof(T) * nn * B, s));
  for (int it = 0; it < iters; ++it) {
    if (it > 0) {
      st = forward_t<T>(p, x, (T *)p->sino_tmp, B, s);
      if (st != BSCT_OK) return st;
    }
    LAUNCH(p, BSCT_K_CORRECTION, 1,
           (pad_rows<T>(p->n_angles, p->M, B, sino, it > 0 ? (const T *)p->sino_tmp : nullptr,
                        (const T *)p->sirt_R, (T *)p->gt, s)));
    st = adjoint_core<T>(p, (const T *)p->gt, (T *)p->q, B, s);
    if (st != BSCT_OK) return st;
    LAUNCH(p, BSCT_K_SOLVER_UPDATE, 1, (sirt_update<T>((long)nn, B, (const T *)p->sirt_C, (const T *)p->q, x, s)));
  }
  return BSCT_OK;
}

// Chebyshev semi-iteration (oracle/solvers.py chebyshev): per iteration y = G d (the same three
// FFT passes as bsct_normal_apply) and one update kernel; coefficients from the host.
template <typename T>
bsct_status chebyshev_t(bsct_plan p, const T *b, T *x, int B, int iters, double lmin, double lmax, double *resid,
                        cudaStream_t s) {
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma = theta / delta;
  T *r = (T *)p->r, *d = (T *)p->p, *y = (T *)p->q;
  LAUNCH(p, BSCT_K_SOLVER_INIT, 1, (cheb_init<T>(p->N, B, b, x, r, d, 1.0 / theta, s)));
  double rho = 1.0 / sigma;
  for (int it = 0; it < iters; ++it) {
    bsct_status st = normal_apply_t<T>(p, d, y, B, nullptr, s);
    if (st != BSCT_OK) return st;
    const double rn = 1.0 / (2.0 * sigma - rho);
    LAUNCH(p, BSCT_K_SOLVER_UPDATE, resid ? 2 : 1,
           (cheb_update<T>(p->N, B, rn * rho, 2.0 * rn / delta, x, r, d, y, p->rpart, resid, iters, it, s)));
    rho = rn;
  }
  return BSCT_OK;
}

}  // namespace

extern "C" {

int32_t bsct_version(void) { return 100; }

bsct_status bsct_chebyshev_solve(bsct_plan p, const void *b, void *x, int32_t B, int32_t iters, double lambda_min,
                                 double lambda_max, double *resid_hist, bsct_stream stream) {
  NvtxRange nvtx_("bsct_chebyshev_solve");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (iters < 0) return fail(BSCT_EINVAL, "iters < 0");
  cudaStream_t s = (cudaStream_t)stream;
  if (!(lambda_max > 0)) {  // the plan's bound: max of the embedding spectrum >= lambda_max(G)
    double tau = 0;
    CU(cudaMemcpyAsync(&tau, p->tau, sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    lambda_max = 1.0 / tau;
  }
  if (!(lambda_min > 0) || !(lambda_min < lambda_max) || !std::isfinite(lambda_max))
    return fail(BSCT_EINVAL, "need 0 < lambda_min < lambda_max (got %g, %g)", lambda_min, lambda_max);
  if (B == 0) return BSCT_OK;
  if (!b || !x) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  return p->dt == BSCT_F64
             ? chebyshev_t<double>(p, (const double *)b, (double *)x, B, iters, lambda_min, lambda_max, resid_hist, s)
             : chebyshev_t<float>(p, (const float *)b, (float *)x, B, iters, lambda_min, lambda_max, resid_hist, s);
}

bsct_status bsct_adjoint_project(bsct_plan p, const void *sino, void *img, int32_t B, bsct_stream stream) {
  NvtxRange nvtx_("bsct_adjoint_project");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (B == 0) return BSCT_OK;
  if (!sino || !img) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? adjoint_t<double>(p, (const double *)sino, (double *)img, B, s)
                           : adjoint_t<float>(p, (const float *)sino, (float *)img, B, s);
}

bsct_status bsct_sirt_solve(bsct_plan p, const void *sino, void *x, int32_t B, int32_t iters, bsct_stream stream) {
  NvtxRange nvtx_("bsct_sirt_solve");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (iters < 0) return fail(BSCT_EINVAL, "iters < 0");
  if (B == 0) return BSCT_OK;
  if (!sino || !x) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? sirt_t<double>(p, (const double *)sino, (double *)x, B, iters, s)
                           : sirt_t<float>(p, (const float *)sino, (float *)x, B, iters, s);
}

const char *bsct_last_error(void) { return g_err.c_str(); }

int32_t bsct_fft_size(int32_t N) { return N < 1 ? 0 : fft_size(N); }

bsct_status bsct_gram_build(const bsct_geometry *g, bsct_dtype dt, int32_t angle_begin, int32_t angle_end, void *taps,
                            bsct_stream stream) {
  NvtxRange nvtx_("bsct_gram_build");
  bsct_status st = validate(g, dt);
  if (st != BSCT_OK) return st;
  if (angle_begin < 0 || angle_end < angle_begin || angle_end > g->n_angles)
    return fail(BSCT_EINVAL, "angle range [%d, %d) not within [0, %d)", angle_begin, angle_end, g->n_angles);
  if (!taps) return fail(BSCT_EINVAL, "taps is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  return dt == BSCT_F64 ? gram_build_t<double>(g, angle_begin, angle_end, (double *)taps, s)
                        : gram_build_t<float>(g, angle_begin, angle_end, (float *)taps, s);
}

bsct_status bsct_plan_create(const bsct_geometry *g, bsct_dtype dt, const void *taps, int32_t max_batch,
                             bsct_plan *out, bsct_stream stream) {
  NvtxRange nvtx_("bsct_plan_create");
  if (!out) return fail(BSCT_EINVAL, "out is NULL");
  *out = nullptr;
  bsct_status st = validate(g, dt);
  if (st != BSCT_OK) return st;
  if (!taps) return fail(BSCT_EINVAL, "taps is NULL");
  if (max_batch < 0) return fail(BSCT_EINVAL, "max_batch < 0");
  // slices index gridDim.y / gridDim.z of the batched kernels (<= 65535)
  if (max_batch > 65535) return fail(BSCT_EINVAL, "max_batch = %d exceeds 65535 (shard the stack)", max_batch);
  bsct_plan p = new bsct_plan_s();
  p->N = g->N;
  p->L = fft_size(g->N);
  p->n_angles = g->n_angles;
  p->M = g->n_det;
  p->lx = g->lambda_x;
  p->ly = g->lambda_y;
  p->zeta = g->zeta_blur;
  p->dt = dt;
  p->max_batch = max_batch;
  p->bp_maxp = bp_v2_max_p(g->n_angles, g->angles, g->lambda_x, g->lambda_y, g->zeta_blur);
  p->bp_tc = dt == BSCT_F32 && bp_tc_supported(g->n_angles, g->angles, g->lambda_x, g->lambda_y, g->zeta_blur);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMalloc((void **)&p->angles, sizeof(double) * g->n_angles);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->angles, g->angles, sizeof(double) * g->n_angles, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    bsct_plan_destroy(p);
    return fail(BSCT_ECUDA, "angle upload: %s", cudaGetErrorString(e));
  }
  st = dt == BSCT_F64 ? plan_init_t<double>(p, taps, s) : plan_init_t<float>(p, taps, s);
  if (st != BSCT_OK) {
    std::string msg = g_err;
    bsct_plan_destroy(p);
    g_err = msg;
    return st;
  }
  *out = p;
  return BSCT_OK;
}

bsct_status bsct_plan_destroy(bsct_plan p) {
  NvtxRange nvtx_("bsct_plan_destroy");
  if (!p) return BSCT_OK;
  void *bufs[] = {p->adj_ang, p->adj_B, p->sirt_R, p->sirt_C, p->sino_tmp,
                  p->angles, p->bp_mem, p->fw_mem, p->S, p->tw, p->T1, p->gt, p->gt_lo, p->r, p->p, p->q,
                  p->sino_dev, p->b_dev, p->x_dev, p->spec_work, p->bp_ang, p->bp_B, p->alpha, p->gpart, p->rpart, p->tau, p->rho, p->flags};
  for (void *b : bufs)
    if (b) cudaFree(b);
  for (cudaEvent_t e : p->prof_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : p->pipe_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : p->gevents) cudaEventDestroy(e);
  for (cudaStream_t g : p->gstreams) cudaStreamDestroy(g);
  if (p->aux) cudaStreamDestroy(p->aux);
  if (p->aux2) cudaStreamDestroy(p->aux2);
  if (p->hi) cudaStreamDestroy(p->hi);
  for (auto &gk : p->graphs) cudaGraphExecDestroy(gk.exec);
  if (p->cap) cudaStreamDestroy(p->cap);
  delete p;
  return BSCT_OK;
}

bsct_status bsct_plan_profile(bsct_plan p, int32_t enable) {
  bsct_status st = check_plan(p, 0);
  if (st != BSCT_OK) return st;
  p->prof_on = enable != 0;
  return BSCT_OK;
}

bsct_status bsct_plan_profile_read(bsct_plan p, double *ms, int64_t *count, int32_t n) {
  bsct_status st = check_plan(p, 0);
  if (st != BSCT_OK) return st;
  if (!p->prof_marks.empty()) {
    CU(cudaEventSynchronize(p->prof_pool[p->prof_marks.back().second + 1]));
    for (auto &m : p->prof_marks) {
      float t = 0;
      CU(cudaEventElapsedTime(&t, p->prof_pool[m.second], p->prof_pool[m.second + 1]));
      p->prof_ms[m.first] += t;
      p->prof_cnt[m.first] += 1;
    }
    p->prof_marks.clear();
    p->prof_used = 0;
  }
  for (int i = 0; i < n && i < BSCT_K_COUNT; ++i) {
    if (ms) ms[i] = p->prof_ms[i];
    if (count) count[i] = p->prof_cnt[i];
  }
  for (int i = 0; i < BSCT_K_COUNT; ++i) {
    p->prof_ms[i] = 0;
    p->prof_cnt[i] = 0;
  }
  return BSCT_OK;
}

bsct_status bsct_plan_set_filter(bsct_plan p, const void *taps, bsct_stream stream) {
  NvtxRange nvtx_("bsct_plan_set_filter");
  bsct_status st = check_plan(p, 0);
  if (st != BSCT_OK) return st;
  if (!taps) return fail(BSCT_EINVAL, "taps is NULL");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? plan_filter_t<double>(p, taps, s) : plan_filter_t<float>(p, taps, s);
}

bsct_status bsct_plan_spectrum(bsct_plan p, void *out, bsct_stream stream) {
  NvtxRange nvtx_("bsct_plan_spectrum");
  bsct_status st = check_plan(p, 0);
  if (st != BSCT_OK) return st;
  if (!out) return fail(BSCT_EINVAL, "out is NULL");
  CU(cudaMemcpyAsync(out, p->S, p->esize() * (size_t)(p->L / 2 + 1) * p->L, cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  return BSCT_OK;
}

bsct_status bsct_correction_filter(bsct_plan p, const void *sino, void *g_tilde, int32_t B, bsct_stream stream) {
  NvtxRange nvtx_("bsct_correction_filter");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (B == 0) return BSCT_OK;
  if (!sino || !g_tilde) return fail(BSCT_EINVAL, "NULL buffer");
  cudaStream_t s = (cudaStream_t)stream;
  p->launches = 0;
  if (p->dt == BSCT_F64) {
    PPTables<double> bp = tables_of<double>(p->bp_mem, p->n_angles);
    LAUNCH(p, BSCT_K_CORRECTION, 0,
           (correction_filter<double>(p->n_angles, p->M, B, bp.degree, (const double *)sino, (double *)g_tilde, s)));
  } else {
    PPTables<float> bp = tables_of<float>(p->bp_mem, p->n_angles);
    LAUNCH(p, BSCT_K_CORRECTION, 0,
           (correction_filter<float>(p->n_angles, p->M, B, bp.degree, (const float *)sino, (float *)g_tilde, s)));
  }
  p->launches = 1;
  return BSCT_OK;
}

bsct_status bsct_backproject(bsct_plan p, const void *sino, void *b, int32_t B, bsct_stream stream) {
  NvtxRange nvtx_("bsct_backproject");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (B == 0) return BSCT_OK;
  if (!sino || !b) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? backproject_t<double>(p, (const double *)sino, (double *)b, B, s)
                           : backproject_t<float>(p, (const float *)sino, (float *)b, B, s);
}

bsct_status bsct_normal_apply(bsct_plan p, const void *x, void *y, int32_t B, bsct_stream stream) {
  NvtxRange nvtx_("bsct_normal_apply");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (B == 0) return BSCT_OK;
  if (!x || !y) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? normal_apply_t<double>(p, (const double *)x, (double *)y, B, nullptr, s)
                           : normal_apply_t<float>(p, (const float *)x, (float *)y, B, nullptr, s);
}

bsct_status bsct_cg_solve(bsct_plan p, const void *b, void *x, int32_t B, int32_t iters, int32_t solver,
                          double *resid_hist, int32_t *flags, bsct_stream stream) {
  NvtxRange nvtx_("bsct_cg_solve");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (iters < 0) return fail(BSCT_EINVAL, "iters < 0");
  if (solver < BSCT_CG || solver > BSCT_LANDWEBER) return fail(BSCT_EINVAL, "unknown solver %d", solver);
  if (B == 0) return BSCT_OK;
  if (!b || !x) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64
             ? solve_t<double>(p, (const double *)b, (double *)x, B, iters, solver, resid_hist, flags, s)
             : solve_t<float>(p, (const float *)b, (float *)x, B, iters, solver, resid_hist, flags, s);
}

bsct_status bsct_cg_resume(bsct_plan p, void *x, void *r, void *pdir, int32_t B, int32_t iters, int32_t solver,
                           double *alpha_last, double *resid_hist, int32_t *flags, bsct_stream stream) {
  NvtxRange nvtx_("bsct_cg_resume");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (iters < 0) return fail(BSCT_EINVAL, "iters < 0");
  if (solver < BSCT_CG || solver > BSCT_LANDWEBER) return fail(BSCT_EINVAL, "unknown solver %d", solver);
  if (B == 0) return BSCT_OK;
  if (!x || !r || (solver == BSCT_CG && !pdir)) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? resume_t<double>(p, (double *)x, (double *)r, (double *)pdir, B, iters, solver,
                                              alpha_last, resid_hist, flags, s)
                           : resume_t<float>(p, (float *)x, (float *)r, (float *)pdir, B, iters, solver, alpha_last,
                                             resid_hist, flags, s);
}

bsct_status bsct_forward_project(bsct_plan p, const void *c, void *sino, int32_t B, bsct_stream stream) {
  NvtxRange nvtx_("bsct_forward_project");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (B == 0) return BSCT_OK;
  if (!c || !sino) return fail(BSCT_EINVAL, "NULL buffer");
  p->launches = 0;
  cudaStream_t s = (cudaStream_t)stream;
  return p->dt == BSCT_F64 ? forward_t<double>(p, (const double *)c, (double *)sino, B, s)
                           : forward_t<float>(p, (const float *)c, (float *)sino, B, s);
}

}  // extern "C"

namespace {

int pipe_chunk(int B, bool host) {
  // host path: chunks overlap the PCIe copies with compute (measured e2e 132K -> 142K
  // slice-iterations/s on config 5, round 1); device path: one chunk unless BSCT_PIPE_CHUNK is set.
  // 512: the quarter-chunk edges are then 128 slices = one full K4 v4 slice tile (round 2, config 5
  // e2e per step: 128: 471.6, 256: 394.3, 384: 390.2, 512: 389.3, 768: 394.3, 1024: 393.6 ms)
  int c = host ? 512 : 0;
  if (const char *e = getenv("BSCT_PIPE_CHUNK")) c = atoi(e);
  if (c <= 0 || c >= B) return B;  // one chunk: no pipelining
  return c;
}

bsct_status pipe_resources(bsct_plan p, int nchunks) {
  if (!p->aux) CU(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking));
  if (!p->aux2) CU(cudaStreamCreateWithFlags(&p->aux2, cudaStreamNonBlocking));
  if (!p->hi) {
    int lo = 0, hiP = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hiP));
    CU(cudaStreamCreateWithPriority(&p->hi, cudaStreamNonBlocking, hiP));
  }
  while ((int)p->pipe_ev.size() < 3 * nchunks + 3) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->pipe_ev.push_back(e);
  }
  if (!p->b_dev) CU(cudaMalloc(&p->b_dev, p->esize() * (size_t)p->N * p->N * p->max_batch));
  return BSCT_OK;
}

// Chunked back projection -> solve.  Host buffers (non-null): chunk c's H2D copy runs on
// aux ahead of its back projection and its D2H copy on aux2 after its solve, so the PCIe
// transfers overlap the kernels.  Kernels run in order on the caller's stream, unless
// BSCT_PIPE_OVERLAP=1: back projections on aux and solves on the plan's highest-priority
// stream (measured 1-3% slower on config 5: K4 and the FFT passes contend for the same SM
// resources, so overlapping them buys nothing; kept for experiments).
bsct_status reconstruct_pipe(bsct_plan p, const void *sino, void *x, int B, int iters, int solver, double *resid,
                             int32_t *flags, cudaStream_t s, const void *sino_host, void *x_host) {
  const size_t es = p->esize();
  const size_t sino_b = es * (size_t)p->n_angles * p->M, img_b = es * (size_t)p->N * p->N;
  const int cb = pipe_chunk(B, sino_host != nullptr);
  // chunk boundaries: with host buffers the first and last chunks are a quarter chunk, so that
  // the copy before the first kernel and after the last one (the unhidden part) are short
  std::vector<int> c0s;
  {
    const int edge = (sino_host && cb < B) ? std::max(1, cb / 4) : cb;
    int c0 = 0;
    while (c0 < B) {
      c0s.push_back(c0);
      const int left = B - c0;
      c0 += (c0 == 0) ? std::min(edge, left) : (left <= cb + edge ? (left > edge ? left - edge : left) : cb);
    }
    c0s.push_back(B);
  }
  const int nch = (int)c0s.size() - 1;
  bsct_status st = pipe_resources(p, nch);
  if (st != BSCT_OK) return st;
  const char *oe = getenv("BSCT_PIPE_OVERLAP");
  const bool overlap = nch > 1 && oe && oe[0] == '1';
  cudaStream_t sb = overlap ? p->aux : s, ss = overlap ? p->hi : s;
  char *bdev = (char *)p->b_dev;
  int64_t launches = 0;
  cudaEvent_t *evH = &p->pipe_ev[0], *evB = &p->pipe_ev[nch], *evS = &p->pipe_ev[2 * nch];
  cudaEvent_t start = p->pipe_ev[3 * nch], done = p->pipe_ev[3 * nch + 1], solved = p->pipe_ev[3 * nch + 2];
  CU(cudaEventRecord(start, s));
  for (cudaStream_t o : {p->aux, p->aux2, p->hi}) CU(cudaStreamWaitEvent(o, start, 0));
  if (sino_host)
    for (int c = 0; c < nch; ++c) {
      const int c0 = c0s[c], nb = c0s[c + 1] - c0;
      CU(cudaMemcpyAsync((char *)sino + c0 * sino_b, (const char *)sino_host + c0 * sino_b, nb * sino_b,
                         cudaMemcpyHostToDevice, p->aux));
      CU(cudaEventRecord(evH[c], p->aux));
    }
  for (int c = 0; c < nch; ++c) {
    const int c0 = c0s[c], nb = c0s[c + 1] - c0;
    const char *sc = (const char *)sino + c0 * sino_b;
    char *bc = bdev + c0 * img_b;
    if (sino_host) CU(cudaStreamWaitEvent(sb, evH[c], 0));
    p->launches = 0;
    st = p->dt == BSCT_F64 ? backproject_t<double>(p, (const double *)sc, (double *)bc, nb, sb)
                           : backproject_t<float>(p, (const float *)sc, (float *)bc, nb, sb);
    if (st != BSCT_OK) return st;
    launches += p->launches;
    if (overlap) {  // the solves wait per chunk; otherwise stream order suffices
      CU(cudaEventRecord(evB[c], sb));
    } else {
      p->launches = 0;
      st = p->dt == BSCT_F64
               ? solve_t<double>(p, (const double *)bc, (double *)((char *)x + c0 * img_b), nb, iters, solver,
                                 resid ? resid + (size_t)c0 * iters : nullptr, flags ? flags + c0 : nullptr, ss)
               : solve_t<float>(p, (const float *)bc, (float *)((char *)x + c0 * img_b), nb, iters, solver,
                                resid ? resid + (size_t)c0 * iters : nullptr, flags ? flags + c0 : nullptr, ss);
      if (st != BSCT_OK) return st;
      launches += p->launches;
      if (x_host) {
        CU(cudaEventRecord(evS[c], ss));
        CU(cudaStreamWaitEvent(p->aux2, evS[c], 0));
        CU(cudaMemcpyAsync((char *)x_host + c0 * img_b, (const char *)x + c0 * img_b, nb * img_b,
                           cudaMemcpyDeviceToHost, p->aux2));
      }
    }
  }
  if (overlap)
    for (int c = 0; c < nch; ++c) {
      const int c0 = c0s[c], nb = c0s[c + 1] - c0;
      const char *bc = bdev + c0 * img_b;
      CU(cudaStreamWaitEvent(ss, evB[c], 0));
      p->launches = 0;
      st = p->dt == BSCT_F64
               ? solve_t<double>(p, (const double *)bc, (double *)((char *)x + c0 * img_b), nb, iters, solver,
                                 resid ? resid + (size_t)c0 * iters : nullptr, flags ? flags + c0 : nullptr, ss)
               : solve_t<float>(p, (const float *)bc, (float *)((char *)x + c0 * img_b), nb, iters, solver,
                                resid ? resid + (size_t)c0 * iters : nullptr, flags ? flags + c0 : nullptr, ss);
      if (st != BSCT_OK) return st;
      launches += p->launches;
      if (x_host) {
        CU(cudaEventRecord(evS[c], ss));
        CU(cudaStreamWaitEvent(p->aux2, evS[c], 0));
        CU(cudaMemcpyAsync((char *)x_host + c0 * img_b, (const char *)x + c0 * img_b, nb * img_b,
                           cudaMemcpyDeviceToHost, p->aux2));
      }
    }
  // join every side stream back into the caller's stream
  CU(cudaEventRecord(done, p->aux2));
  CU(cudaStreamWaitEvent(s, done, 0));
  CU(cudaEventRecord(solved, p->hi));
  CU(cudaStreamWaitEvent(s, solved, 0));
  CU(cudaEventRecord(done, p->aux));
  CU(cudaStreamWaitEvent(s, done, 0));
  p->launches = launches;
  return BSCT_OK;
}

}  // namespace

extern "C" {

bsct_status bsct_reconstruct(bsct_plan p, const void *sino, void *x, int32_t B, int32_t iters, int32_t solver,
                             double *resid_hist, int32_t *flags, bsct_stream stream) {
  NvtxRange nvtx_("bsct_reconstruct");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (iters < 0) return fail(BSCT_EINVAL, "iters < 0");
  if (solver < BSCT_CG || solver > BSCT_LANDWEBER) return fail(BSCT_EINVAL, "unknown solver %d", solver);
  if (B == 0) return BSCT_OK;
  if (!sino || !x) return fail(BSCT_EINVAL, "NULL buffer");
  return reconstruct_pipe(p, sino, x, B, iters, solver, resid_hist, flags, (cudaStream_t)stream, nullptr, nullptr);
}

bsct_status bsct_reconstruct_host(bsct_plan p, const void *sino_host, void *x_host, int32_t B, int32_t iters,
                                  int32_t solver, bsct_stream stream) {
  NvtxRange nvtx_("bsct_reconstruct_host");
  bsct_status st = check_plan(p, B);
  if (st != BSCT_OK) return st;
  if (B == 0) return BSCT_OK;
  if (iters < 0) return fail(BSCT_EINVAL, "iters < 0");
  if (solver < BSCT_CG || solver > BSCT_LANDWEBER) return fail(BSCT_EINVAL, "unknown solver %d", solver);
  if (!sino_host || !x_host) return fail(BSCT_EINVAL, "NULL buffer");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t es = p->esize();
  const size_t sino_b = es * (size_t)p->n_angles * p->M, img_b = es * (size_t)p->N * p->N;
  if (!p->sino_dev) CU(cudaMalloc(&p->sino_dev, sino_b * p->max_batch));
  if (!p->x_dev) CU(cudaMalloc(&p->x_dev, img_b * p->max_batch));
  st = reconstruct_pipe(p, p->sino_dev, p->x_dev, B, iters, solver, nullptr, nullptr, s, sino_host, x_host);
  if (st != BSCT_OK) return st;
  CU(cudaStreamSynchronize(s));
  return BSCT_OK;
}

int64_t bsct_plan_launch_count(bsct_plan p) { return p ? p->launches : 0; }

}  // extern "C"
