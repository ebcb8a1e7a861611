// Minimal TMA (cp.async.bulk.tensor) check: one 3-D box {32, 1, 8} of an FP32 array, SWIZZLE_128B.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

using EncodeTiled = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap *gmap, const float *src, float *out, int x,
                  int y, int z, int variant) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = (unsigned char *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(variant == 2 ? 1024 : 32 * 8 * 4) : "memory");
    if (variant == 2) {  // plain bulk copy (no tensor map): 1 KB contiguous
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                   "l"(src), "r"(1024), "r"(b) : "memory");
    } else if (variant == 3) {  // tensor map in global memory
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(d), "l"(gmap), "r"(x), "r"(y), "r"(z), "r"(b) : "memory");
    } else if (variant == 0)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(d), "l"(&map), "r"(x), "r"(y), "r"(z), "r"(b) : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(d), "l"(&map), "r"(x), "r"(y), "r"(z), "r"(b) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(b) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = ((float *)sm)[i];
}

int main(int argc, char **argv) {
  const int X = 201, Y = 60, Z = 3, LD = 204;
  std::vector<float> h((size_t)Z * Y * LD);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *g, *o;
  cudaMalloc(&g, h.size() * 4);
  cudaMalloc(&o, 256 * 4);
  cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiled enc = (EncodeTiled)p;
  if (getenv("DIRECT")) { cuInit(0); enc = cuTensorMapEncodeTiled; printf("direct\n"); }
  printf("entry %p direct %p\n", p, (void *)cuTensorMapEncodeTiled);
  CUtensorMap map;
  const cuuint64_t dims[3] = {X, Y, Z};
  const cuuint64_t str[2] = {(cuuint64_t)LD * 4, (cuuint64_t)LD * 4 * Y};
  const cuuint32_t box[3] = {32, 1, 8};
  const cuuint32_t es[3] = {1, 1, 1};
  int sw = argc > 1 ? atoi(argv[1]) : 3;
  CUtensorMapSwizzle swz = sw == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (query %d) sizeof %zu\n", (int)r, (int)q, sizeof(CUtensorMap));
  CUtensorMap *gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  int variant = argc > 2 ? atoi(argv[2]) : 0;
  {
    k<<<1, 128, 4096 + 1024>>>(map, gm, g, o, 5, 2, 0, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    if (variant == 2) return 0;
    std::vector<float> ho(256);
    cudaMemcpy(ho.data(), o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int zz = 0; zz < 8; ++zz)
      for (int xx = 0; xx < 32; ++xx) {
        const int chunk = xx >> 2, sc = sw == 3 ? (chunk ^ (zz & 7)) : chunk;
        const float got = ho[zz * 32 + sc * 4 + (xx & 3)];
        const float want = zz < Z ? h[((size_t)zz * Y + 2) * LD + 5 + xx] : 0.f;
        bad += got != want;
      }
    printf("variant %d mismatches %d\n", variant, bad);
  }
  return 0;
}
