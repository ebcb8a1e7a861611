// TMA variant matrix: argv = rank tilekw l2promo oob swz
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

template <int RANK, int TILEKW>
__global__ void k(const __grid_constant__ CUtensorMap map, float *out, int z0, int bytes) {
  __shared__ __align__(1024) float sm[2048];
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    if (RANK == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(d), "l"(&map), "r"(z0 >> 8), "r"(z0 & 255), "r"(b) : "memory");
    else if (TILEKW)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(d), "l"(&map), "r"(5), "r"(2), "r"(z0), "r"(b) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(d), "l"(&map), "r"(5), "r"(2), "r"(z0), "r"(b) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(b) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char **argv) {
  const int rank = atoi(argv[1]), tilekw = atoi(argv[2]), l2 = atoi(argv[3]), oob = atoi(argv[4]), swz = atoi(argv[5]);
  cuInit(0);
  const int X = 201, Y = 60, Z = oob ? 3 : 16, LD = 204;
  std::vector<float> h((size_t)Z * Y * LD);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000);
  float *g, *o;
  cudaMalloc(&g, h.size() * 4);
  cudaMalloc(&o, 1024);
  cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  CUresult r;
  if (rank == 3) {
    const cuuint64_t dims[3] = {X, Y, (cuuint64_t)Z};
    const cuuint64_t str[2] = {(cuuint64_t)LD * 4, (cuuint64_t)LD * 4 * Y};
    const cuuint32_t box[3] = {32, 1, 8};
    const cuuint32_t es[3] = {1, 1, 1};
    r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                               l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[2] = {X, (cuuint64_t)Y * Z};
    const cuuint64_t str[1] = {(cuuint64_t)LD * 4};
    const cuuint32_t box[2] = {32, 8};
    const cuuint32_t es[2] = {1, 1};
    r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                               l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const int x0 = argc > 6 ? atoi(argv[6]) : 5;
  if (rank == 2) k<2, 0><<<1, 128>>>(map, o, x0 << 8, 1024);
  else if (tilekw) k<3, 1><<<1, 128>>>(map, o, 0, 1024);
  else k<3, 0><<<1, 128>>>(map, o, 0, 1024);
  cudaError_t e = cudaDeviceSynchronize();
  printf("rank %d tile %d l2 %d oob %d swz %d: encode %d kernel %s\n", rank, tilekw, l2, oob, swz, (int)r,
         cudaGetErrorString(e));
  return 0;
}
