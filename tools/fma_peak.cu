// FP32 / FP64 FMA throughput microbenchmark (roofline denominator for the ALU-bound kernels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak tools/fma_peak.cu && ./fma_peak
// Each thread runs 8 independent FMA chains (enough ILP to cover the FMA latency); grid =
// 148 SMs x 8 CTAs x 256 threads.  Prints one JSON line: TFLOP/s counted as 2 flops per FMA.
#include <cstdio>

#include <cuda_runtime.h>

template <typename T>
__global__ void __launch_bounds__(256) fma_kernel(T *out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (T)(threadIdx.x + i);
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == (T)12345.678) out[0] = s;  // keeps the chains live
}

// packed FP32x2 FMA (fma.rn.f32x2 -> FFMA2): two FP32 FMAs per lane per instruction
__global__ void __launch_bounds__(256) fma2_kernel(float *out, int iters, float a, float b) {
  unsigned long long x[8], av, bv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float v = (float)(threadIdx.x + i);
    asm("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(v));
  }
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(bv));
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
    s += lo + hi;
  }
  if (s == 12345.678f) out[0] = s;
}

static double run2(int sms) {
  float *out = nullptr;
  cudaMalloc(&out, sizeof(float));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  fma2_kernel<<<blocks, threads>>>(out, 64, 0.999999f, 1e-7f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma2_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(out);
  const double fmas = 2.0 * blocks * threads * iters * 16 * 8;
  return 2.0 * fmas / (best / 1e3) / 1e12;
}

template <typename T>
static double run(int sms) {
  T *out = nullptr;
  cudaMalloc(&out, sizeof(T));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  fma_kernel<T><<<blocks, threads>>>(out, 64, (T)0.999999, (T)1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_kernel<T><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(out);
  const double fmas = (double)blocks * threads * iters * 16 * 8;
  return 2.0 * fmas / (best / 1e3) / 1e12;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double f32 = run<float>(prop.multiProcessorCount);
  const double f64 = run<double>(prop.multiProcessorCount);
  const double f2 = run2(prop.multiProcessorCount);
  printf("{\"device\": \"%s\", \"sms\": %d, \"max_clock_mhz\": %.0f, \"fp32_fma_tflops\": %.2f, "
         "\"fp32x2_fma_tflops\": %.2f, \"fp64_fma_tflops\": %.2f, \"how\": \"tools/fma_peak.cu: 148 x 8 CTAs x 256 "
         "threads, 8 independent FMA chains per thread, best of 5, 2 flops per FMA (FFMA2: 4 per instruction)\"}\n",
         prop.name, prop.multiProcessorCount, clk / 1e3, f32, f2, f64);
  return 0;
}
