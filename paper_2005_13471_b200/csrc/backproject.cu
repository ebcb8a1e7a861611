// backproject.cu -- K3 correction filter (Eq.(5)) and K4 back projection
// b = H^T g^_psi.
//
// K3: for angles whose interpolation degree is 2 (blur, non-axis angle) the
//     sinogram row is convolved with q[m] = sqrt(2)(2 sqrt(2) - 3)^|m|, |m| <= 25
//     (readings R7, R8: zero-extended full linear convolution, M + 50 outputs);
//     otherwise q = delta and the row is copied into the middle.
// K4: b[k] = lambda_x^2 lambda_y sum_t sum_m g~[t][m] C_t(y_m - k_t), C_t the box spline
//     with widths [l|c|, l|s|, zeta] U [lambda_y]^(d+1) (the pixel footprint convolved with
//     the degree-d B-spline interpolant, Eq.(1)); only the <= floor(W/lambda_y)+1 samples
//     inside C_t's support contribute.
#include "kernels.cuh"
#include "pptable.cuh"

namespace bsct {

constexpr int HC = 25;  // correction filter half-width ("truncated", R8)

__constant__ double c_q64[2 * HC + 1];
__constant__ float c_q32[2 * HC + 1];

template <typename T> __device__ __forceinline__ T qtap(int i);
template <> __device__ __forceinline__ float qtap<float>(int i) { return c_q32[i]; }
template <> __device__ __forceinline__ double qtap<double>(int i) { return c_q64[i]; }

static bool g_q_ready = false;

static cudaError_t upload_q() {
  if (g_q_ready) return cudaSuccess;
  double q[2 * HC + 1];
  float qf[2 * HC + 1];
  const long double z = 2.0L * sqrtl(2.0L) - 3.0L;
  for (int m = -HC; m <= HC; ++m) {
    long double v = sqrtl(2.0L);
    for (int k = 0; k < (m < 0 ? -m : m); ++k) v *= z;
    q[m + HC] = (double)v;
    qf[m + HC] = (float)v;
  }
  cudaError_t e = cudaMemcpyToSymbol(c_q64, q, sizeof(q));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_q32, qf, sizeof(qf));
  if (e == cudaSuccess) g_q_ready = true;
  return e;
}

template <typename T>
__global__ void __launch_bounds__(256) correction_kernel(int n_angles, int M, const int *__restrict__ degree,
                                                         const T *__restrict__ sino, T *__restrict__ gt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *row = reinterpret_cast<T *>(smem_raw);
  const int a = blockIdx.x, b = blockIdx.y;
  const T *src = sino + ((size_t)b * n_angles + a) * M;
  T *dst = gt + ((size_t)b * n_angles + a) * (M + 2 * HC);
  const int d = degree[a];
  for (int i = threadIdx.x; i < M; i += blockDim.x) row[i] = src[i];
  __syncthreads();
  for (int j = threadIdx.x; j < M + 2 * HC; j += blockDim.x) {
    const int m = j - HC;  // detector index of output sample j
    T v = 0;
    if (d == 2) {
      // g~[m] = sum_i q[i] g[m - i], zero outside [0, M)
      const int ilo = max(-HC, m - (M - 1)), ihi = min(HC, m);
      for (int i = ilo; i <= ihi; ++i) v = fma(qtap<T>(i + HC), row[m - i], v);
    } else if (m >= 0 && m < M) {
      v = row[m];
    }
    dst[j] = v;
  }
}

template <typename T>
cudaError_t correction_filter(int n_angles, int M, int B, const int *degree, const T *sino, T *gt, cudaStream_t s) {
  cudaError_t e = upload_q();
  if (e != cudaSuccess) return e;
  const size_t sm = sizeof(T) * (size_t)M;
  if (sm > 48 * 1024) {
    e = cudaFuncSetAttribute(correction_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  correction_kernel<T><<<dim3(n_angles, B), 256, sm, s>>>(n_angles, M, degree, sino, gt);
  return cudaGetLastError();
}

// K4 v1: one thread per pixel, 16 x 16 pixel tiles, all angles in order.
template <typename T>
__global__ void __launch_bounds__(256) backproject_kernel(int N, double lx, double ly, int n_angles, int M,
                                                          const double *__restrict__ cs, PPView<T> tb,
                                                          const T *__restrict__ gt, T *__restrict__ out) {
  const int k2 = blockIdx.x * 16 + threadIdx.x;
  const int k1 = blockIdx.y * 16 + threadIdx.y;
  const int b = blockIdx.z;
  const double x1 = lx * (double)(k1 - N / 2);
  const double x2 = lx * (double)(k2 - N / 2);
  const int Mt = M + 2 * HC;
  const T *g = gt + (size_t)b * n_angles * Mt;
  const double m_off = (double)(M / 2);
  T acc = 0;
  for (int a = 0; a < n_angles; ++a) {
    const double c = cs[2 * a], s = cs[2 * a + 1];
    const double kt = fma(-s, x1, c * x2);
    const double H = tb.half[a];
    // samples with |y_m - k_t| < H, y_m = ly (m - floor(M/2))
    int m = (int)floor((kt - H) / ly + m_off) + 1;
    const T *ga = g + (size_t)a * Mt + HC;
    for (;; ++m) {
      const double arg = ly * ((double)m - m_off) - kt;
      if (arg >= H) break;
      const int j = m + HC;
      if (j < 0 || j >= Mt) continue;
      acc = fma(ga[m], pp_eval<T>(tb, a, arg), acc);
    }
  }
  if (k1 < N && k2 < N) out[((size_t)b * N + k1) * N + k2] = (T)(lx * lx * ly) * acc;
}

template <typename T>
cudaError_t backproject(int N, double lx, double ly, int n_angles, int M, int B, const double *cs, PPView<T> tb,
                        const T *gt, T *b, cudaStream_t s) {
  dim3 grid((N + 15) / 16, (N + 15) / 16, B);
  backproject_kernel<T><<<grid, dim3(16, 16), 0, s>>>(N, lx, ly, n_angles, M, cs, tb, gt, b);
  return cudaGetLastError();
}

template cudaError_t correction_filter<float>(int, int, int, const int *, const float *, float *, cudaStream_t);
template cudaError_t correction_filter<double>(int, int, int, const int *, const double *, double *, cudaStream_t);
template cudaError_t backproject<float>(int, double, double, int, int, int, const double *, PPView<float>,
                                        const float *, float *, cudaStream_t);
template cudaError_t backproject<double>(int, double, double, int, int, int, const double *, PPView<double>,
                                         const double *, double *, cudaStream_t);

}  // namespace bsct
