// primary.cu -- the primary layer of the P-CapsNet training step (SURVEY
// §8(f) NEXT-4, reading R25): the capsule convolution with one
// input channel of 1x1 capsules (C = D1 = D2 = 1), stride 1, no padding, i.e.
// a plain convolution of a one-channel image to N = Cout * D3 channels:
//   O[b,x,y,n]  = sum_{p,q} img[b, x+p, y+q] * K[p, q, n]
//   dK[p,q,n]   = sum_{b,x,y} img[b, x+p, y+q] * dO[b, x, y, n]
// (the general kernels of simt.cu take it too, one output element per thread
// with two loads per multiply-add, ~100x slower).  Both passes are bounded by
// the N-channel map they write (fwd) or read (dK).  bf16 with N = 128 runs on
// tcgen05 (an im2col tile gathered by producer warps is one MMA operand:
// primary_tc_fwd_kernel, primary_tc_dk_kernel); fp32 and other widths run the
// CUDA-core kernels (primary_fwd_kernel, primary_dk_kernel).
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "rows.cuh"
#include "umma.cuh"

namespace capsconv {
namespace {

template <typename T> __device__ __forceinline__ float pr_ld(const T *p);
template <> __device__ __forceinline__ float pr_ld<float>(const float *p) { return __ldg(p); }
template <> __device__ __forceinline__ float pr_ld<__nv_bfloat16>(const __nv_bfloat16 *p) {
    return __bfloat162float(__ldg(p));
}

// Forward: a warp = 64 consecutive output pixels (two per lane, 32 apart:
// the image loads stay consecutive across the lanes and every weight read --
// a shared-memory broadcast -- feeds both) x one group of 32 channels; the
// block's 4 warps are channel groups (N >= 128) or pixel groups.  Weights
// K[t][n] (fp32) in shared memory.
template <typename T>
__device__ __forceinline__ void pr_store32(T *op, const float (&acc)[32]) {
    if constexpr (sizeof(T) == 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t w4[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                __nv_bfloat162 h = __floats2bfloat162_rn(acc[8 * j + 2 * c], acc[8 * j + 2 * c + 1]);
                w4[c] = *reinterpret_cast<uint32_t *>(&h);
            }
            reinterpret_cast<uint4 *>(op)[j] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            reinterpret_cast<float4 *>(op)[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
}

template <typename T>
__global__ void __launch_bounds__(128) primary_fwd_kernel(const T *__restrict__ img, const T *__restrict__ K,
                                                          T *__restrict__ O, int B, int H, int W, int KH, int KW,
                                                          int N) {
    extern __shared__ __align__(16) float Ks[];   // [KH*KW][N]
    const int ntap = KH * KW;
    for (int e = threadIdx.x; e < ntap * N; e += blockDim.x) Ks[e] = pr_ld<T>(K + e);
    __syncthreads();
    const int Ho = H - KH + 1, Wo = W - KW + 1, npix = B * Ho * Wo;
    const int ngrp = N / 32, wpb = ngrp < 4 ? ngrp : 4;              // warps sharing a pixel chunk
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wg = warp % wpb, wpix = warp / wpb;
    const int ppb = 64 * (4 / wpb);                                   // pixels per block
    const int pix0 = blockIdx.x * ppb + wpix * 64 + lane, pix1 = pix0 + 32;
    if (pix0 >= npix) return;
    const bool v1 = pix1 < npix;
    const int y0 = pix0 % Wo, x0 = (pix0 / Wo) % Ho, b0 = pix0 / (Wo * Ho);
    const int q1 = v1 ? pix1 : pix0;
    const int y1 = q1 % Wo, x1 = (q1 / Wo) % Ho, b1 = q1 / (Wo * Ho);
    const T *ip0 = img + ((size_t)b0 * H + x0) * W + y0;
    const T *ip1 = img + ((size_t)b1 * H + x1) * W + y1;
    for (int g = wg; g < ngrp; g += wpb) {
        float a0[32], a1[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a0[j] = a1[j] = 0.f;
        for (int p = 0; p < KH; ++p)
            for (int q = 0; q < KW; ++q) {
                const float u = pr_ld<T>(ip0 + (size_t)p * W + q), v = pr_ld<T>(ip1 + (size_t)p * W + q);
                const float4 *kr = reinterpret_cast<const float4 *>(Ks + (p * KW + q) * N + g * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 k = kr[j];
                    a0[4 * j] = fmaf(u, k.x, a0[4 * j]);
                    a0[4 * j + 1] = fmaf(u, k.y, a0[4 * j + 1]);
                    a0[4 * j + 2] = fmaf(u, k.z, a0[4 * j + 2]);
                    a0[4 * j + 3] = fmaf(u, k.w, a0[4 * j + 3]);
                    a1[4 * j] = fmaf(v, k.x, a1[4 * j]);
                    a1[4 * j + 1] = fmaf(v, k.y, a1[4 * j + 1]);
                    a1[4 * j + 2] = fmaf(v, k.z, a1[4 * j + 2]);
                    a1[4 * j + 3] = fmaf(v, k.w, a1[4 * j + 3]);
                }
            }
        pr_store32<T>(O + (size_t)pix0 * N + g * 32, a0);
        if (v1) pr_store32<T>(O + (size_t)pix1 * N + g * 32, a1);
    }
}

// Forward on the tensor cores (bf16, N = 128, KH*KW <= 32): a tile of 128
// output pixels is one MMA row block; its A operand (128 pixels x 32 taps,
// the 5x5 patch padded with zeros) is gathered by the four producer warps
// straight into the no-swizzle K-major core-matrix layout (element (m, k) at
// (k/8)*2048 + m*16 + (k%8)*2: each thread writes its own pixel's four
// 16-byte chunks, conflict-free), B = the 128 x 32 weight image staged once;
// two 128x128x16 MMAs per tile into one of two TMEM accumulators; the same
// warps drain the previous tile (each thread its pixel's 128 channels =
// 256 contiguous bytes).  Persistent: one CTA per SM walks tiles blockIdx.x,
// + gridDim.x, ...
constexpr int kPtN = 128, kPtK = 32;
constexpr uint32_t kPtStage = 128u * kPtK * 2u;   // 8 KB A stage
constexpr uint32_t kPtB = kPtN * kPtK * 2u;       // 8 KB weights
constexpr uint32_t kPtSmem = 2 * kPtStage + kPtB + 4 * 8192u;

template <int KH, int KW>
__global__ void __launch_bounds__(160, 1) primary_tc_fwd_kernel(const __nv_bfloat16 *__restrict__ img,
                                                                const __nv_bfloat16 *__restrict__ K,
                                                                __nv_bfloat16 *__restrict__ O, int B, int H, int W) {
    using namespace umma;
    // A stages | weights | per-warp output staging (32 pixels x 256 B, 16-byte chunks swizzled by row)
    extern __shared__ __align__(1024) uint8_t sm[];   // kPtSmem bytes
    __shared__ uint64_t afull[2], aempty[2], accf[2], acce[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const uint32_t a0 = smem_u32(sm), bs = a0 + 2 * kPtStage, ob = bs + kPtB + (uint32_t)(warp & 3) * 8192u;
    constexpr int ntap = KH * KW;
    const int Ho = H - KH + 1, Wo = W - KW + 1, npix = B * Ho * Wo;
    const int ntiles = (npix + 127) / 128;
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(afull + i, 128);
            mbar_init(aempty + i, 1);
            mbar_init(accf + i, 1);
            mbar_init(acce + i, 128);
        }
        mbar_fence_init();
    }
    if (warp == 4) tmem_alloc_dyn(&tslot, 256);
    pdl_wait();
    if (tid < 128) {   // weights: row n = tid, k = tap (zero past ntap)
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int k0 = 2 * j, k1 = 2 * j + 1;
            __nv_bfloat162 h;
            h.x = k0 < ntap ? K[(size_t)k0 * kPtN + tid] : __float2bfloat16_rn(0.f);
            h.y = k1 < ntap ? K[(size_t)k1 * kPtN + tid] : __float2bfloat16_rn(0.f);
            w[j] = *reinterpret_cast<uint32_t *>(&h);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(bs + (uint32_t)c * 2048u + (uint32_t)tid * 16u),
                         "r"(w[4 * c]), "r"(w[4 * c + 1]), "r"(w[4 * c + 2]), "r"(w[4 * c + 3])
                         : "memory");
        fence_proxy_async_smem();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = tslot;
    const int nk = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (warp == 4) {
        // ------------------------------------------------------------ MMA
        const uint32_t idesc = idesc_bf16(128, kPtN, 0, 0);
        for (int k = 0; k < nk; ++k) {
            const int s = k & 1;
            const uint32_t ph = (uint32_t)(k >> 1) & 1u;
            mbar_wait(afull + s, ph);
            mbar_wait(acce + s, ph ^ 1u);
            fence_after_sync();
            const uint32_t as = a0 + (uint32_t)s * kPtStage;
#pragma unroll
            for (int ks = 0; ks < kPtK / 16; ++ks) {
                const uint64_t ad = smem_desc(as + (uint32_t)ks * 4096u, 2048u, 128u);
                const uint64_t bd = smem_desc(bs + (uint32_t)ks * 4096u, 2048u, 128u);
                rows::mma_ss_elect(tmem + (uint32_t)s * kPtN, ad, bd, idesc, ks > 0 ? 1u : 0u);
            }
            if (elect_one()) {
                mma_commit(aempty + s);
                mma_commit(accf + s);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ im2col producer + epilogue
        for (int k = 0; k <= nk; ++k) {
            if (k < nk) {
                const int s = k & 1;
                mbar_wait(aempty + s, ((uint32_t)(k >> 1) & 1u) ^ 1u);
                const int pix = ((int)blockIdx.x + k * (int)gridDim.x) * 128 + tid;
                uint32_t w[16];
                if (pix < npix) {
                    const int y = pix % Wo, x = (pix / Wo) % Ho, b = pix / (Wo * Ho);
                    const __nv_bfloat16 *ip = img + ((size_t)b * H + x) * W + y;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int t0 = 2 * j, t1 = 2 * j + 1;
                        __nv_bfloat162 h;
                        h.x = t0 < ntap ? ip[(size_t)(t0 / KW) * W + t0 % KW] : __float2bfloat16_rn(0.f);
                        h.y = t1 < ntap ? ip[(size_t)(t1 / KW) * W + t1 % KW] : __float2bfloat16_rn(0.f);
                        w[j] = *reinterpret_cast<uint32_t *>(&h);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) w[j] = 0u;
                }
                const uint32_t as = a0 + (uint32_t)s * kPtStage + (uint32_t)tid * 16u;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(as + (uint32_t)c * 2048u),
                                 "r"(w[4 * c]), "r"(w[4 * c + 1]), "r"(w[4 * c + 2]), "r"(w[4 * c + 3])
                                 : "memory");
                fence_proxy_async_smem();
                mbar_arrive(afull + s);
            }
            if (k >= 1) {
                const int kk = k - 1, s = kk & 1;
                mbar_wait(accf + s, (uint32_t)(kk >> 1) & 1u);
                fence_after_sync();
                const uint32_t tb = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)s * kPtN;
                // row `lane` of the warp's staging: 16 chunks of 16 B, chunk j at (j ^ (lane & 15))
#pragma unroll
                for (int c = 0; c < kPtN / 32; ++c) {
                    float v[32];
                    rows::tmem_ld32(tb + (uint32_t)c * 32u, v);
                    tmem_wait_ld();
                    if (c == kPtN / 32 - 1) {   // accumulator drained: hand the slot back
                        fence_before_sync();
                        mbar_arrive(acce + s);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint32_t u[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
                            u[e] = *reinterpret_cast<uint32_t *>(&h);
                        }
                        const uint32_t ch = (uint32_t)((c * 4 + j) ^ (lane & 15));
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(ob + (uint32_t)lane * 256u + ch * 16u),
                                     "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3])
                                     : "memory");
                    }
                }
                __syncwarp();
                // the warp's 32 consecutive pixels are 8 KB contiguous in O: 512 B per store instruction
                const int wpix0 = ((int)blockIdx.x + kk * (int)gridDim.x) * 128 + warp * 32;
                uint4 *wo = reinterpret_cast<uint4 *>(O + (size_t)wpix0 * kPtN);
#pragma unroll 4
                for (int i = 0; i < 16; ++i) {
                    const int u = i * 32 + lane, r = u >> 4, j = u & 15;   // row r, chunk j of the warp's block
                    if (wpix0 + r < npix) wo[u] = ld_shared_v4(ob + (uint32_t)r * 256u + (uint32_t)((j ^ (r & 15)) * 16));
                }
                __syncwarp();
            }
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 4) tmem_dealloc_dyn(tmem, 256);
}

// Weight gradient on the tensor cores (bf16, N = 128, KH*KW <= 64): the
// transposed product dK^T[n][t] = sum_pix dO[pix][n] * A[pix][t] with the
// pixels as the reduction.  A = dO^T is MN-major straight from two TMA boxes
// (64 channels x 128 pixels, SWIZZLE_128B) per 128-pixel tile; B = the
// im2col tile (128 pixels x 64 taps, zero past KH*KW), MN-major in the same
// swizzled layout, gathered by four producer warps (row = pixel, 16-byte
// chunk c at c ^ (row & 7)); eight 128x64x16 MMAs per tile accumulate into
// one TMEM accumulator for the CTA's whole pixel range; the producers then
// write the CTA's partial (fixed-order sum in primary_dk_reduce).
constexpr int kPdStg = 3;
constexpr uint32_t kPdA = 2u * 16384u, kPdB = 16384u, kPdStage = kPdA + kPdB;
constexpr uint32_t kPdSmem = 1024u + kPdStg * kPdStage;

template <int KH, int KW>
__global__ void __launch_bounds__(192, 1) primary_tc_dk_kernel(const __grid_constant__ CUtensorMap tmD,
                                                               const __nv_bfloat16 *__restrict__ img,
                                                               float *__restrict__ part, int B, int H, int W) {
    using namespace umma;
    extern __shared__ __align__(1024) uint8_t smd[];
    __shared__ uint64_t full[kPdStg], empty[kPdStg], accf;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t s0 = (smem_u32(smd) + 1023u) & ~1023u;
    constexpr int ntap = KH * KW;
    const int Ho = H - KH + 1, Wo = W - KW + 1, npix = B * Ho * Wo;
    const int ntiles = (npix + 127) / 128;
    const int nk = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPdStg; ++i) {
            mbar_init(full + i, 1 + 128);
            mbar_init(empty + i, 1);
        }
        mbar_init(&accf, 1);
        mbar_fence_init();
    }
    if (warp == 5) tmem_alloc_dyn(&tslot, 64);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = tslot;
    pdl_wait();
    if (warp == 0) {
        // ------------------------------------------------------------ TMA: dO^T boxes
        if (lane == 0) {
            for (int k = 0; k < nk; ++k) {
                const int s = k % kPdStg;
                mbar_wait(empty + s, ((uint32_t)(k / kPdStg) & 1u) ^ 1u);
                const uint32_t stg = s0 + (uint32_t)s * kPdStage, mb = smem_u32(full + s);
                mbar_arrive_expect_tx(full + s, kPdA);
                const int r0 = ((int)blockIdx.x + k * (int)gridDim.x) * 128;
                rows::tma_load2d(stg, &tmD, 0, r0, mb);
                rows::tma_load2d(stg + 16384u, &tmD, 64, r0, mb);
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA
        const uint32_t idesc = idesc_bf16(128, 64, 1, 1);
        for (int k = 0; k < nk; ++k) {
            const int s = k % kPdStg;
            mbar_wait(full + s, (uint32_t)(k / kPdStg) & 1u);
            fence_after_sync();
            const uint32_t stg = s0 + (uint32_t)s * kPdStage;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t ad = rows::sdesc(stg + (uint32_t)kk * 2048u, 16384u, 1024u, 128);
                const uint64_t bd = rows::sdesc(stg + kPdA + (uint32_t)kk * 2048u, 16384u, 1024u, 128);
                rows::mma_ss_elect(tmem, ad, bd, idesc, (k > 0 || kk > 0) ? 1u : 0u);
            }
            if (elect_one()) mma_commit(empty + s);
            __syncwarp();
        }
        if (elect_one()) mma_commit(&accf);
        __syncwarp();
    } else {
        // ------------------------------------------------------------ im2col producers (warps 1-4), then the partial
        const int row = threadIdx.x - 32;   // pixel row of the tile
        for (int k = 0; k < nk; ++k) {
            const int s = k % kPdStg;
            mbar_wait(empty + s, ((uint32_t)(k / kPdStg) & 1u) ^ 1u);
            const int pix = ((int)blockIdx.x + k * (int)gridDim.x) * 128 + row;
            uint32_t w[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) w[j] = 0u;
            if (pix < npix) {
                const int y = pix % Wo, x = (pix / Wo) % Ho, b = pix / (Wo * Ho);
                const __nv_bfloat16 *ip = img + ((size_t)b * H + x) * W + y;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int t0 = 2 * j, t1 = 2 * j + 1;
                    if (t0 < ntap) {
                        __nv_bfloat162 h;
                        h.x = ip[(size_t)(t0 / KW) * W + t0 % KW];
                        h.y = t1 < ntap ? ip[(size_t)(t1 / KW) * W + t1 % KW] : __float2bfloat16_rn(0.f);
                        w[j] = *reinterpret_cast<uint32_t *>(&h);
                    }
                }
            }
            const uint32_t rb = s0 + (uint32_t)s * kPdStage + kPdA + (uint32_t)row * 128u;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(rb + (uint32_t)((c ^ (row & 7)) * 16)),
                             "r"(w[4 * c]), "r"(w[4 * c + 1]), "r"(w[4 * c + 2]), "r"(w[4 * c + 3])
                             : "memory");
            fence_proxy_async_smem();
            mbar_arrive(full + s);
        }
        if (nk > 0) {
            mbar_wait(&accf, 0u);
            fence_after_sync();
            const int q = warp & 3, n = q * 32 + lane;   // TMEM lane quarter of this warp = channels n
            float v[32];
            rows::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16), v);
            tmem_wait_ld();
            float *pp = part + (size_t)blockIdx.x * ntap * kPtN + n;
#pragma unroll
            for (int t = 0; t < 32; ++t)
                if (t < ntap) pp[(size_t)t * kPtN] = v[t];
            if (ntap > 32) {
                rows::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 32u, v);
                tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 32; ++t)
                    if (32 + t < ntap) pp[(size_t)(32 + t) * kPtN] = v[t];
            }
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 5) tmem_dealloc_dyn(tmem, 64);
}

// Weight gradient: thread = channel n (blockDim = N), block = a range of
// image rows (b, x); the KH x KW window of the image slides along y in
// registers (KH new values per output pixel, warp-wide broadcasts) and meets
// the pixel's dO[n] (one coalesced load per pixel and thread).  Partials
// part[block][t][n], summed in block order by primary_dk_reduce.
template <typename T, int KH, int KW>
__global__ void __launch_bounds__(256) primary_dk_kernel(const T *__restrict__ img, const T *__restrict__ dO,
                                                         float *__restrict__ part, int B, int H, int W, int N,
                                                         int rows_per_block) {
    const int n = threadIdx.x;
    const int Ho = H - KH + 1, Wo = W - KW + 1;
    float acc[KH][KW];
#pragma unroll
    for (int p = 0; p < KH; ++p)
#pragma unroll
        for (int q = 0; q < KW; ++q) acc[p][q] = 0.f;
    const int r0 = blockIdx.x * rows_per_block, r1 = min(B * Ho, r0 + rows_per_block);
    for (int r = r0; r < r1; ++r) {
        const int b = r / Ho, x = r - b * Ho;
        const T *ib = img + ((size_t)b * H + x) * W;
        const T *gb = dO + ((size_t)r * Wo) * N + n;
        float win[KH][KW];   // before pixel y: win[p][q] = img[x+p][y+q-1] for q >= 1
#pragma unroll
        for (int p = 0; p < KH; ++p) {
            win[p][0] = 0.f;
#pragma unroll
            for (int q = 1; q < KW; ++q) win[p][q] = pr_ld<T>(ib + (size_t)p * W + q - 1);
        }
        for (int y = 0; y < Wo; ++y) {
#pragma unroll
            for (int p = 0; p < KH; ++p) {   // shift left, load column y + KW - 1
#pragma unroll
                for (int q = 0; q + 1 < KW; ++q) win[p][q] = win[p][q + 1];
                win[p][KW - 1] = pr_ld<T>(ib + (size_t)p * W + y + KW - 1);
            }
            const float g = pr_ld<T>(gb + (size_t)y * N);
#pragma unroll
            for (int p = 0; p < KH; ++p)
#pragma unroll
                for (int q = 0; q < KW; ++q) acc[p][q] = fmaf(win[p][q], g, acc[p][q]);
        }
    }
    float *pp = part + (size_t)blockIdx.x * (KH * KW) * N + n;
#pragma unroll
    for (int p = 0; p < KH; ++p)
#pragma unroll
        for (int q = 0; q < KW; ++q) pp[(size_t)(p * KW + q) * N] = acc[p][q];
}

// One warp per output element: lane l adds partials l, l+32, ... in order,
// then a fixed butterfly over the lanes -- a fixed summation order for every
// element (deterministic), with nblk/32 loads per lane instead of nblk.
__global__ void __launch_bounds__(256) primary_dk_reduce(const float *__restrict__ part, float *__restrict__ dK,
                                                         int nblk, int n_out) {
    const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= n_out) return;
    float s = 0.f;
    for (int k = lane; k < nblk; k += 32) s += part[(size_t)k * n_out + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dK[i] = s;
}

int primary_dk_blocks(const Problem &p) {
    const int rows = (int)(p.B * p.Ho);
    const int want = 8 * device_info().num_sms;   // ~8 blocks of N threads per SM: latency hiding
    return rows < want ? rows : want;
}

}  // namespace

bool primary_supported(const Problem &p) {
    const int64_t N = p.Cout * p.D3;
    const bool k_ok = p.KH == p.KW && (p.KH == 3 || p.KH == 5 || p.KH == 7);   // instantiated windows
    return p.layout == CAPSCONV_LAYOUT_NATURAL && p.C == 1 && p.D1 == 1 && p.D2 == 1 && p.s == 1 && p.pad == 0 &&
           (N == 32 || N == 64 || N == 128 || N == 256) && k_ok && p.B * p.H * p.W < ((int64_t)1 << 30) &&
           p.B * p.Ho * p.Wo * N < ((int64_t)1 << 31);
}

bool primary_tc(capsconv_op_t op, const Problem &p) {
    if (!primary_supported(p) || p.dt != CAPSCONV_BF16 || p.Cout * p.D3 != kPtN) return false;
    if (op == CAPSCONV_OP_FWD) return p.KH == 3 || p.KH == 5;                 // <= 32 taps per im2col row
    if (op == CAPSCONV_OP_BWD_KERNEL) return p.KH == 3 || p.KH == 5 || p.KH == 7;   // <= 64 taps
    return false;
}

size_t primary_workspace_bytes(capsconv_op_t op, const Problem &p) {
    if (op != CAPSCONV_OP_BWD_KERNEL) return 0;
    return (size_t)primary_dk_blocks(p) * (size_t)(p.KH * p.KW) * (size_t)(p.Cout * p.D3) * sizeof(float);
}

cudaError_t primary_fwd(const Problem &p, const void *img, const void *K, void *O, cudaStream_t st) {
    const int N = (int)(p.Cout * p.D3), ngrp = N / 32, wpb = ngrp < 4 ? ngrp : 4;
    if (primary_tc(CAPSCONV_OP_FWD, p) && !(kProbes && probe_env("CAPSCONV_PRIMARY_SIMT"))) {
        const int64_t npix = p.B * p.Ho * p.Wo;
        const int grid = (int)std::min<int64_t>((npix + 127) / 128, device_info().num_sms);
        const auto *ip = static_cast<const __nv_bfloat16 *>(img);
        const auto *kp = static_cast<const __nv_bfloat16 *>(K);
        auto *op = static_cast<__nv_bfloat16 *>(O);
        auto kern = p.KH == 5 ? primary_tc_fwd_kernel<5, 5> : primary_tc_fwd_kernel<3, 3>;
        cudaError_t e = smem_optin(reinterpret_cast<const void *>(kern), (int)kPtSmem);
        if (e != cudaSuccess) return e;
        e = launch_k(kern, dim3(grid), dim3(160), kPtSmem, st, ip, kp, op, (int)p.B, (int)p.H, (int)p.W);
        note_launches(1);
        return e;
    }
    const int ppb = 64 * (4 / wpb);
    const int64_t npix = p.B * p.Ho * p.Wo;
    const size_t smem = (size_t)p.KH * p.KW * N * sizeof(float);
    const dim3 grid((unsigned)((npix + ppb - 1) / ppb));
    if (p.dt == CAPSCONV_BF16)
        primary_fwd_kernel<__nv_bfloat16><<<grid, 128, smem, st>>>(
            static_cast<const __nv_bfloat16 *>(img), static_cast<const __nv_bfloat16 *>(K),
            static_cast<__nv_bfloat16 *>(O), (int)p.B, (int)p.H, (int)p.W, (int)p.KH, (int)p.KW, N);
    else
        primary_fwd_kernel<float><<<grid, 128, smem, st>>>(static_cast<const float *>(img),
                                                            static_cast<const float *>(K), static_cast<float *>(O),
                                                            (int)p.B, (int)p.H, (int)p.W, (int)p.KH, (int)p.KW, N);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t primary_bwd_kernel(const Problem &p, const void *img, const void *dO, float *dK, void *ws, cudaStream_t st) {
    const int N = (int)(p.Cout * p.D3);
    if (primary_tc(CAPSCONV_OP_BWD_KERNEL, p) && !(kProbes && probe_env("CAPSCONV_PRIMARY_SIMT"))) {
        const int64_t npix = p.B * p.Ho * p.Wo;
        const int grid = (int)std::min<int64_t>((npix + 127) / 128, device_info().num_sms);
        CUtensorMap tm;
        if (!rows::make_rows_map2(&tm, dO, npix, kPtN, 64, 128, 128)) return cudaErrorInvalidValue;
        auto kern = p.KH == 5 ? primary_tc_dk_kernel<5, 5>
                    : p.KH == 3 ? primary_tc_dk_kernel<3, 3> : primary_tc_dk_kernel<7, 7>;
        cudaError_t e = smem_optin(reinterpret_cast<const void *>(kern), (int)kPdSmem);
        if (e != cudaSuccess) return e;
        e = launch_k(kern, dim3(grid), dim3(192), kPdSmem, st, tm, static_cast<const __nv_bfloat16 *>(img),
                     static_cast<float *>(ws), (int)p.B, (int)p.H, (int)p.W);
        if (e != cudaSuccess) return e;
        const int n_out = (int)(p.KH * p.KW) * N;
        primary_dk_reduce<<<(n_out + 7) / 8, 256, 0, st>>>(static_cast<const float *>(ws), dK, grid, n_out);
        note_launches(2);
        return cudaGetLastError();
    }
    const int nblk = primary_dk_blocks(p);
    const int rows = (int)(p.B * p.Ho), rpb = (rows + nblk - 1) / nblk;
    float *part = static_cast<float *>(ws);
    const int B = (int)p.B, H = (int)p.H, W = (int)p.W;
#define CAPSCONV_PRIMARY_DK(KK)                                                                                    \
    if (p.dt == CAPSCONV_BF16)                                                                                     \
        primary_dk_kernel<__nv_bfloat16, KK, KK><<<nblk, N, 0, st>>>(static_cast<const __nv_bfloat16 *>(img),      \
                                                                     static_cast<const __nv_bfloat16 *>(dO), part, \
                                                                     B, H, W, N, rpb);                             \
    else                                                                                                           \
        primary_dk_kernel<float, KK, KK><<<nblk, N, 0, st>>>(static_cast<const float *>(img),                      \
                                                             static_cast<const float *>(dO), part, B, H, W, N, rpb);
    if (p.KH == 3) { CAPSCONV_PRIMARY_DK(3) }
    else if (p.KH == 5) { CAPSCONV_PRIMARY_DK(5) }
    else { CAPSCONV_PRIMARY_DK(7) }
#undef CAPSCONV_PRIMARY_DK
    const int n_out = (int)(p.KH * p.KW) * N;
    primary_dk_reduce<<<(n_out + 7) / 8, 256, 0, st>>>(part, dK, nblk, n_out);
    note_launches(2);
    return cudaGetLastError();
}

}  // namespace capsconv
