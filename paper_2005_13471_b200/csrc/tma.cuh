// tma.cuh -- mbarrier and TMA (cp.async.bulk / cp.async.bulk.tensor) helpers shared by the kernels
// that stage operands with the sm_100 copy engine (K4 v4, bp_tc.cu).
#pragma once

#include <cuda.h>

#include <cstdint>
#include <cstdio>

namespace bsct {

#ifdef BSCT_TC_DEBUG
#define TMA_DBG(...) printf(__VA_ARGS__)
#else
#define TMA_DBG(...)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Every wait traps after ~2^26 polls instead of hanging the GPU on a lost arrival.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int who = 0, int a = 0) {
  uint32_t done = 0;
  long long it = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (++it > (1ll << 26)) {
      TMA_DBG("mbarrier timeout: block (%d,%d,%d) thread %d who %d item %d bar %u parity %u\n", blockIdx.x,
              blockIdx.y, blockIdx.z, threadIdx.x, who, a, bar, parity);
      __trap();
    }
  }
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int x, int y, int z, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link); null if absent
using EncodeTiled = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled tma_encoder();

}  // namespace bsct
