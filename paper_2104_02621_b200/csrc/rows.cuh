// rows.cuh -- shared pieces of the D1-outer ("rows") layout kernels.
//
// Layout CAPSCONV_LAYOUT_ROWS stores a capsule tensor as
//     I[B][H][W][D1][C][D2]        (O[B][Ho][Wo][D1][Cout][D3])
// i.e. every pixel is D1 consecutive "capsule rows", each holding row d1 of
// all C capsules (C*D2 contiguous elements).  The contraction of the paper
// (Algorithm 2) then maps onto the tensor core with no
// data movement beyond TMA:
//   forward / dI : A rows (pixel, d1), K = (c, d2)  -> K-major, TMA writes it
//   dK           : A = I^T, M = (c, d2), K = (pixel, d1) -> MN-major, same bytes
//                  B = dO,  N = (c', d3), K = (pixel, d1) -> MN-major
// (SURVEY §7 H1(d) / NEXT-3(i)).  Tensors are staged with TMA in the 64-/128-
// byte swizzled layouts whose descriptors were verified bit-exactly on B200
// (tests/test_rows_probe_gpu.py): K-major operands may start at any whole
// row (the tap shift) and MN-major atoms may sit at any row stride (several
// taps read from one staged window).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#ifdef __CUDACC__
#include "umma.cuh"
#endif

namespace capsconv {
namespace rows {

// Swizzle width (bytes) for a chunk of `e` bf16 elements per row.
__host__ __device__ constexpr int swz_bytes(int e) { return e * 2; }
// UMMA descriptor layout code (bits 61-63) of a swizzle width.
__host__ __device__ constexpr uint64_t layout_code(int swz) {
    return swz == 128 ? 2ull : swz == 64 ? 4ull : swz == 32 ? 6ull : 0ull;
}

#ifdef __CUDACC__
// Shared-memory matrix descriptor of a swizzled operand.
//   K-major : rows of `swz` bytes; SBO = 8 rows; LBO unused.
//   MN-major: atoms of swz/2 elements; LBO = atom stride, SBO = 8 k-rows.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, int swz) {
    return umma::smem_desc(addr, lbo, sbo) | (layout_code(swz) << 61);
}

// 5-D tile load (coordinates innermost first), completion on an mbarrier.
__device__ __forceinline__ void tma_load5d(uint32_t dst, const CUtensorMap *m, int c0, int c1, int c2, int c3, int c4,
                                           uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(mbar)
        : "memory");
}
// 4-D tile load over a merged-row view (E, 4, Ws, B*Hs).
__device__ __forceinline__ void tma_load4d_rows(uint32_t dst, const CUtensorMap *m, int c0, int c1, int c2, int c3,
                                                uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void tma_load3d(uint32_t dst, const CUtensorMap *m, int c0, int c1, int c2,
                                           uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void tma_load2d(uint32_t dst, const CUtensorMap *m, int c0, int c1, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}

// 4-D tile store shared -> global (bulk async-group completion); the box is
// clipped at the tensor bounds.
__device__ __forceinline__ void tma_store4d(const CUtensorMap *m, uint32_t src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void tma_store5d(const CUtensorMap *m, uint32_t src, int c0, int c1, int c2, int c3,
                                            int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// wait until at most N committed store groups still READ shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
// wait until all committed store groups have completed (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// The same MMA issued by one elected lane of a converged warp: the whole
// warp runs the (uniform) issue loop, so descriptors stay in uniform
// registers and each MMA costs an elect + a predicated UTCHMMA.
__device__ __forceinline__ void mma_ss_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld16x(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// 16 columns of zeros into this warp's 32 TMEM lanes (one zero register, 16 operands)
__device__ __forceinline__ void tmem_st_zero16(uint32_t taddr) {
    const uint32_t z = 0u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n"
        ::"r"(taddr), "r"(z) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
#endif

// Host: tensor maps over a rows-layout bf16 tensor [B][Hs][Ws][4][E]
// (E = C*D2 elements per capsule row).
//   map5: dims (E, 4, Ws, Hs, B), box (ce, 4, bx, by, bb), element strides
//         (1, 1, es_x, es_y, 1) -- a box lands [by'][bx'][4][ce] with
//         bx' = bx / es_x pixels per row (every es_x-th pixel), zero filled
//         outside the tensor; swizzle = 2*ce bytes.
bool make_rows_map5(CUtensorMap *map, const void *base, int64_t B, int64_t Hs, int64_t Ws, int64_t E, int ce, int bx,
                    int by, int es_x, int es_y,
                    int bb = 1);
//   map2: a row-major [rows][E] bf16 matrix, box (ce, br), swizzle 2*ce bytes
//         (ce = 16/32/64), or no swizzle when swz == 0 (then ce*2 must be 16).
bool make_rows_map2(CUtensorMap *map, const void *base, int64_t rows, int64_t E, int ce, int br, int swz);
//   map4m: dims (E, 4, Ws, rows) -- a rows tensor with all B*Hs pixel rows
//          merged (dense: image stride = Hs row strides), box (ce, 4, bx, by),
//          element strides (1, 1, es, es)
bool make_rows_map4m(CUtensorMap *map, const void *base, int64_t rows, int64_t Ws, int64_t E, int ce, int bx, int by,
                     int es);
//   map4: dims (E, 4, P, B) -- a rows tensor viewed with all P = H*W pixels of
//         an image flattened -- box (ce, 4, 1, bb): one pixel position of bb
//         images (the fully-connected view, R18).
bool make_rows_map4(CUtensorMap *map, const void *base, int64_t B, int64_t P, int64_t E, int ce, int bp, int bb);

}  // namespace rows
}  // namespace capsconv
