// tma.h -- Tensor Memory Accelerator descriptors for the natural capsule
// layout [B][H][W][CS][16] (bf16), used to stage source windows into shared
// memory with cp.async.bulk.tensor (no thread involvement, zero fill for
// out-of-bounds coordinates, optional traversal stride for phase planes).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace capsconv {

// Map over a bf16 tensor viewed as 4-D (innermost first):
//   d0 = CS*16 elements of one pixel, d1 = W, d2 = H, d3 = B.
// Box (innermost first): (cc*16, box_w * stride, box_h * stride, box_b) with
// element strides (1, stride, stride, 1): one copy lands box_b x box_h rows of
// box_w pixels (every stride-th pixel), each cc*16 elements, as
// [b][row][x][cc*16].  Out-of-bounds coordinates read as zero.
bool make_capsule_tmap(CUtensorMap *map, const void *base, int64_t B, int64_t H, int64_t W, int64_t CS, int cc,
                       int box_w, int box_h, int box_b, int stride);

}  // namespace capsconv

#ifdef __CUDACC__
namespace capsconv {
namespace tma {

__device__ __forceinline__ void prefetch_desc(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// 4-D tile load (coordinates innermost first), completion on an mbarrier.
__device__ __forceinline__ void load4d(uint32_t dst_smem, const CUtensorMap *m, int c0, int c1, int c2, int c3,
                                       uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];\n" ::"r"(dst_smem),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
        : "memory");
}

}  // namespace tma
}  // namespace capsconv
#endif
