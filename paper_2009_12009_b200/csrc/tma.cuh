// TMA / mbarrier helpers and the tensor-map description of a FabArray's
// storage (shared by the streaming GSRB sweep and the coarse kernels).
#pragma once

#include <cuda.h>

#include <vector>

#include "stencil_common.cuh"

namespace amrb {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
// 4-D tile load (k, j, i, block) into shared memory, completion on bar
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// One FabArray's storage as a 4-D tensor (k, j, i, block): every resident box
// has the same grown shape and the blocks are equally spaced.
struct TmaDesc {
  bool ok = false;
  int64_t base = 0;  // element offset of tensor element (0, 0, 0, 0) (16-byte aligned)
  int64_t pitch = 0, rows = 0, planes = 0, stride = 0;
  int f = 0, g = 0;  // tensor column of the grown box's first cell = f; ghost width g
  std::vector<int> slot;  // per box
};

TmaDesc describe(const Level& lv, const Field& f);
// box = box_rows x box_cols elements of one plane of one block
bool make_map(CUtensorMap* map, const double* base, const TmaDesc& d, int nblocks, int box_rows, int box_cols);

}  // namespace amrb
