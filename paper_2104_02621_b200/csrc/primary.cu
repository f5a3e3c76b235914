// primary.cu -- the primary layer of the P-CapsNet training step (SURVEY
// §8(f) NEXT-4, reading R25): the capsule convolution with one
// input channel of 1x1 capsules (C = D1 = D2 = 1), stride 1, no padding, i.e.
// a plain convolution of a one-channel image to N = Cout * D3 channels:
//   O[b,x,y,n]  = sum_{p,q} img[b, x+p, y+q] * K[p, q, n]
//   dK[p,q,n]   = sum_{b,x,y} img[b, x+p, y+q] * dO[b, x, y, n]
// (the general kernels of simt.cu take it too, one output element per thread
// with two loads per multiply-add, ~100x slower).  CUDA cores: K = KH*KW <= 32
// multiply-adds per output is far too short a reduction for the tensor cores'
// 16-deep k-steps to pay, and both passes are bounded by the N-channel map
// they write (fwd) or read (dK).
#include <cuda_bf16.h>

#include "internal.h"

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

__global__ void __launch_bounds__(256) primary_dk_reduce(const float *__restrict__ part, float *__restrict__ dK,
                                                         int nblk, int n_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_out) return;
    float s = 0.f;
    for (int k = 0; k < nblk; ++k) s += part[(size_t)k * n_out + i];   // fixed order: deterministic
    dK[i] = s;
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

size_t primary_workspace_bytes(capsconv_op_t op, const Problem &p) {
    if (op != CAPSCONV_OP_BWD_KERNEL) return 0;
    return (size_t)primary_dk_blocks(p) * (size_t)(p.KH * p.KW) * (size_t)(p.Cout * p.D3) * sizeof(float);
}

cudaError_t primary_fwd(const Problem &p, const void *img, const void *K, void *O, cudaStream_t st) {
    const int N = (int)(p.Cout * p.D3), ngrp = N / 32, wpb = ngrp < 4 ? ngrp : 4;
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
    primary_dk_reduce<<<(n_out + 255) / 256, 256, 0, st>>>(part, dK, nblk, n_out);
    note_launches(2);
    return cudaGetLastError();
}

}  // namespace capsconv
