// 2-D TMA check with the driver API linked directly (-lcuda).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, float *out) {
  __shared__ __align__(1024) float sm[8 * 32];
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(1024) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(d), "l"(&map), "r"(0), "r"(0), "r"(b) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(b) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}

int main() {
  cuInit(0);
  std::vector<float> h(64 * 64);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *g, *o;
  cudaMalloc(&g, h.size() * 4);
  cudaMalloc(&o, 1024);
  cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  const cuuint64_t dims[2] = {64, 64};
  const cuuint64_t str[1] = {64 * 4};
  const cuuint32_t box[2] = {32, 8};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(map, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> ho(256);
  cudaMemcpy(ho.data(), o, 1024, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < 8; ++y)
    for (int x = 0; x < 32; ++x) bad += ho[y * 32 + x] != h[y * 64 + x];
  printf("mismatches %d\n", bad);
  return 0;
}
