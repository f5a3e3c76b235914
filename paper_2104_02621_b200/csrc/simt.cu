// simt.cu -- the SIMT ("custom APIs", Algorithm 5 lineage) path of libcapsconv.
//
// PAPER.md:210-229 (Algorithm 5) and :274-275: every small matrix product
// I_caps(D1xD2) * K_caps(D2xD3) is computed by CUDA cores and "accumulat[ed]
// ... at each output position".  Here each thread OWNS its outputs (gather
// form, no atomics) and keeps them in registers, so there is no index table
// and no replicated buffer.  This path is total: it takes every valid problem
// (any capsule size, stride, alignment) and is the exact-fp32 path.
//
// Two flavours per pass:
//   *_d4  : D1=D2=D3=4 capsules, 16-byte aligned pointers; register-blocked
//           (one thread per output capsule x CG output channels), vector loads.
//   *_gen : any extents; one thread per output element.
// dK is a reduction over (b, x', y', d1): split over the pixel range into a
// workspace of fp32 partials, then a fixed-order reduce (deterministic).
#include <cuda_bf16.h>

#include "internal.h"

namespace capsconv {
namespace {

template <typename T> __device__ __forceinline__ float ldf(const T *p);
template <> __device__ __forceinline__ float ldf<float>(const float *p) { return __ldg(p); }
template <> __device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16 *p) {
    return __bfloat162float(__ldg(p));
}
template <typename T> __device__ __forceinline__ T cvt(float v);
template <> __device__ __forceinline__ float cvt<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// 16 consecutive elements (one 4x4 capsule) -> fp32 registers.
template <typename T> __device__ __forceinline__ void load_caps16(const T *p, float (&v)[16]);
template <> __device__ __forceinline__ void load_caps16<float>(const float *p, float (&v)[16]) {
    const float4 *q = reinterpret_cast<const float4 *>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float4 t = __ldg(q + i);
        v[4 * i + 0] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
    }
}
template <> __device__ __forceinline__ void load_caps16<__nv_bfloat16>(const __nv_bfloat16 *p, float (&v)[16]) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        uint4 t = __ldg(q + i);
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162 *>(&w[j]);
            float2 f = __bfloat1622float2(h);
            v[8 * i + 2 * j] = f.x;
            v[8 * i + 2 * j + 1] = f.y;
        }
    }
}

template <typename T> __device__ __forceinline__ void store_caps16(T *p, const float (&v)[16]);
template <> __device__ __forceinline__ void store_caps16<float>(float *p, const float (&v)[16]) {
    float4 *q = reinterpret_cast<float4 *>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
template <> __device__ __forceinline__ void store_caps16<__nv_bfloat16>(__nv_bfloat16 *p, const float (&v)[16]) {
    uint4 *q = reinterpret_cast<uint4 *>(p);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
            w[j] = *reinterpret_cast<uint32_t *>(&h);
        }
        q[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <typename IX>
struct DimsT {
    IX B, H, W, C, Cout, KH, KW, D1, D2, D3, s, Ho, Wo;
    IX pad;   // symmetric zero padding: input pixel (x*s + p - pad, y*s + q - pad); outside = 0
};
using Dims = DimsT<int64_t>;
// The vectorised kernels index in 32 bits when every offset they form fits
// (one IMAD instead of a 64-bit multiply chain per address).
template <typename IX>
DimsT<IX> dims_as(const Dims &d) {
    return DimsT<IX>{(IX)d.B, (IX)d.H, (IX)d.W, (IX)d.C, (IX)d.Cout, (IX)d.KH, (IX)d.KW,
                     (IX)d.D1, (IX)d.D2, (IX)d.D3, (IX)d.s, (IX)d.Ho, (IX)d.Wo, (IX)d.pad};
}

// ============================================================ forward
// Thread = (b, x', y', group of CG output channels); acc[CG][d1][d3].
template <typename T, int CG, typename IX>
__global__ void __launch_bounds__(128) fwd_d4(DimsT<IX> d, const T *__restrict__ I, const T *__restrict__ K,
                                              T *__restrict__ O, float *__restrict__ part, int nsplit) {
    const IX ngroups = (d.Cout + CG - 1) / CG;
    const IX total = d.B * d.Ho * d.Wo * ngroups;
    const IX idx = (IX)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    IX r = idx;
    const IX y = r % d.Wo; r /= d.Wo;
    const IX x = r % d.Ho; r /= d.Ho;
    const IX b = r % d.B;
    const IX g = r / d.B;
    const IX co0 = g * CG;
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    // split blockIdx.y of nsplit takes the taps [t0, t1) (fixed ranges: the
    // partials are summed in split order, deterministic)
    const IX ntap = d.KH * d.KW, t0 = ntap * blockIdx.y / nsplit, t1 = ntap * (blockIdx.y + 1) / nsplit;
    for (IX t = t0; t < t1; ++t) {
        const IX p = t / d.KW, q = t - p * d.KW;
        const IX h = x * d.s + p - d.pad;
        if (h < 0 || h >= d.H) continue;
        {
            const IX w = y * d.s + q - d.pad;
            if (w < 0 || w >= d.W) continue;
            const T *ip = I + (((b * d.H + h) * d.W + w) * d.C) * 16;
            const T *kp = K + (((p * d.KW + q) * d.C) * d.Cout + co0) * 16;
            for (IX c = 0; c < d.C; ++c) {
                float a[16];
                load_caps16<T>(ip + c * 16, a);
#pragma unroll
                for (int j = 0; j < CG; ++j) {
                    if (co0 + j < d.Cout) {
                        float k[16];
                        load_caps16<T>(kp + (c * d.Cout + j) * 16, k);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int t = 0; t < 4; ++t)
#pragma unroll
                                for (int n = 0; n < 4; ++n)
                                    acc[j][i * 4 + n] = fmaf(a[i * 4 + t], k[t * 4 + n], acc[j][i * 4 + n]);
                    }
                }
            }
        }
    }
    const IX oo = (((b * d.Ho + x) * d.Wo + y) * d.Cout + co0) * 16;
    if (nsplit > 1) {
        float *pp = part + (IX)blockIdx.y * (d.B * d.Ho * d.Wo * d.Cout * 16) + oo;
#pragma unroll
        for (int j = 0; j < CG; ++j)
            if (co0 + j < d.Cout) store_caps16<float>(pp + j * 16, acc[j]);
        return;
    }
#pragma unroll
    for (int j = 0; j < CG; ++j)
        if (co0 + j < d.Cout) store_caps16<T>(O + oo + j * 16, acc[j]);
}

template <typename T>
__global__ void __launch_bounds__(256) fwd_gen(Dims d, const T *__restrict__ I, const T *__restrict__ K,
                                               T *__restrict__ O) {
    const int64_t total = d.B * d.Ho * d.Wo * d.Cout * d.D1 * d.D3;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int64_t r = idx;
    const int64_t d3 = r % d.D3; r /= d.D3;
    const int64_t d1 = r % d.D1; r /= d.D1;
    const int64_t co = r % d.Cout; r /= d.Cout;
    const int64_t y = r % d.Wo; r /= d.Wo;
    const int64_t x = r % d.Ho;
    const int64_t b = r / d.Ho;
    float acc = 0.f;
    for (int64_t p = 0; p < d.KH; ++p)
        for (int64_t q = 0; q < d.KW; ++q) {
            const int64_t h = x * d.s + p - d.pad, w = y * d.s + q - d.pad;
            if (h < 0 || h >= d.H || w < 0 || w >= d.W) continue;
            const T *ip = I + ((((b * d.H + h) * d.W + w) * d.C) * d.D1 + d1) * d.D2;
            const T *kp = K + ((((p * d.KW + q) * d.C) * d.Cout + co) * d.D2) * d.D3 + d3;
            for (int64_t c = 0; c < d.C; ++c)
                for (int64_t t = 0; t < d.D2; ++t)
                    acc = fmaf(ldf(ip + c * d.D1 * d.D2 + t), ldf(kp + (c * d.Cout * d.D2 + t) * d.D3), acc);
        }
    O[idx] = cvt<T>(acc);
}

// ============================================================ backward data
// Thread = (b, h, w, c) input capsule; acc[d1][d2] (gather form).
// Thread = (b, h, w, group of CG input channels); acc[CG][d1][d2]: each dO
// capsule is loaded once per (tap, c') and reused for the CG channels.
template <typename T, int CG, typename IX>
__global__ void __launch_bounds__(128) bwd_data_d4(DimsT<IX> d, const T *__restrict__ dO, const T *__restrict__ K,
                                                   T *__restrict__ dI) {
    const IX ngroups = (d.C + CG - 1) / CG;
    const IX total = d.B * d.H * d.W * ngroups;
    const IX idx = (IX)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    IX r = idx;
    const IX g = r % ngroups; r /= ngroups;
    const IX w = r % d.W; r /= d.W;
    const IX h = r % d.H;
    const IX b = r / d.H;
    const IX c0 = g * CG;
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    for (IX p = 0; p < d.KH; ++p) {
        const IX hx = h + d.pad - p;
        if (hx < 0 || hx % d.s) continue;
        const IX x = hx / d.s;
        if (x >= d.Ho) continue;
        for (IX q = 0; q < d.KW; ++q) {
            const IX wy = w + d.pad - q;
            if (wy < 0 || wy % d.s) continue;
            const IX y = wy / d.s;
            if (y >= d.Wo) continue;
            const T *gp = dO + ((b * d.Ho + x) * d.Wo + y) * d.Cout * 16;
            const T *kp = K + (((p * d.KW + q) * d.C + c0) * d.Cout) * 16;
            for (IX co = 0; co < d.Cout; ++co) {
                float gv[16];
                load_caps16<T>(gp + co * 16, gv);
#pragma unroll
                for (int j = 0; j < CG; ++j) {
                    if (c0 + j < d.C) {
                        float k[16];
                        load_caps16<T>(kp + ((IX)j * d.Cout + co) * 16, k);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int t = 0; t < 4; ++t)
#pragma unroll
                                for (int n = 0; n < 4; ++n)
                                    acc[j][i * 4 + t] = fmaf(gv[i * 4 + n], k[t * 4 + n], acc[j][i * 4 + t]);
                    }
                }
            }
        }
    }
    T *ip = dI + (((b * d.H + h) * d.W + w) * d.C + c0) * 16;
#pragma unroll
    for (int j = 0; j < CG; ++j)
        if (c0 + j < d.C) store_caps16<T>(ip + j * 16, acc[j]);
}

template <typename T>
__global__ void __launch_bounds__(256) bwd_data_gen(Dims d, const T *__restrict__ dO, const T *__restrict__ K,
                                                    T *__restrict__ dI) {
    const int64_t total = d.B * d.H * d.W * d.C * d.D1 * d.D2;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int64_t r = idx;
    const int64_t t = r % d.D2; r /= d.D2;
    const int64_t i = r % d.D1; r /= d.D1;
    const int64_t c = r % d.C; r /= d.C;
    const int64_t w = r % d.W; r /= d.W;
    const int64_t h = r % d.H;
    const int64_t b = r / d.H;
    float acc = 0.f;
    for (int64_t p = 0; p < d.KH; ++p) {
        const int64_t hx = h + d.pad - p;
        if (hx < 0 || hx % d.s) continue;
        const int64_t x = hx / d.s;
        if (x >= d.Ho) continue;
        for (int64_t q = 0; q < d.KW; ++q) {
            const int64_t wy = w + d.pad - q;
            if (wy < 0 || wy % d.s) continue;
            const int64_t y = wy / d.s;
            if (y >= d.Wo) continue;
            const T *gp = dO + (((b * d.Ho + x) * d.Wo + y) * d.Cout * d.D1 + i) * d.D3;
            const T *kp = K + (((p * d.KW + q) * d.C + c) * d.Cout * d.D2 + t) * d.D3;
            for (int64_t co = 0; co < d.Cout; ++co)
                for (int64_t n = 0; n < d.D3; ++n)
                    acc = fmaf(ldf(gp + co * d.D1 * d.D3 + n), ldf(kp + co * d.D2 * d.D3 + n), acc);
        }
    }
    dI[idx] = cvt<T>(acc);
}

// ============================================================ staged-weight variants
// The same gather loops with the block's weight slice in shared memory: a block
// is 128 pixels x ONE channel group (grid.x = group, fastest, so consecutive
// blocks share their pixels in L2), every thread of the block reads the same
// weight capsule at the same time (a shared-memory broadcast instead of an
// L1/L2 round trip per capsule), 32-bit indexing.  Used when the slice fits
// (kSimtSmemMax); the per-thread-load kernels above serve the rest.
constexpr int kSimtSmemMax = 100 * 1024;

__device__ __forceinline__ void lds_caps16(const float *p, float (&v)[16]) {
    const float4 *q = reinterpret_cast<const float4 *>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float4 t = q[i];
        v[4 * i + 0] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
    }
}

// Forward: Ks[t][c][j] = K[p][q][c][co0 + j] (zero past Cout); thread = one output pixel.
template <typename T>
__global__ void __launch_bounds__(128) fwd_d4s(DimsT<int> d, const T *__restrict__ I, const T *__restrict__ K,
                                               T *__restrict__ O) {
    extern __shared__ __align__(16) float Ks[];
    constexpr int CG = 4;
    const int g = blockIdx.x, co0 = g * CG;
    const int ntap = d.KH * d.KW;
    for (int e = threadIdx.x; e < ntap * d.C * CG * 16; e += blockDim.x) {
        const int k16 = e & 15, j = (e >> 4) % CG, tc = (e >> 4) / CG;   // tc = t * C + c
        Ks[e] = co0 + j < d.Cout ? ldf<T>(K + ((size_t)tc * d.Cout + co0 + j) * 16 + k16) : 0.f;
    }
    __syncthreads();
    const int n = blockIdx.y * blockDim.x + threadIdx.x;
    if (n >= d.B * d.Ho * d.Wo) return;
    const int y = n % d.Wo, x = (n / d.Wo) % d.Ho, b = n / (d.Wo * d.Ho);
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    for (int p = 0; p < d.KH; ++p) {
        const int h = x * d.s + p - d.pad;
        if (h < 0 || h >= d.H) continue;
        for (int q = 0; q < d.KW; ++q) {
            const int w = y * d.s + q - d.pad;
            if (w < 0 || w >= d.W) continue;
            const T *ip = I + (((size_t)(b * d.H + h) * d.W + w) * d.C) * 16;
            const float *kt = Ks + (size_t)(p * d.KW + q) * d.C * CG * 16;
            for (int c = 0; c < d.C; ++c) {
                float a[16];
                load_caps16<T>(ip + c * 16, a);
#pragma unroll
                for (int j = 0; j < CG; ++j) {
                    float k[16];
                    lds_caps16(kt + (c * CG + j) * 16, k);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int t = 0; t < 4; ++t)
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                acc[j][i * 4 + m] = fmaf(a[i * 4 + t], k[t * 4 + m], acc[j][i * 4 + m]);
                }
            }
        }
    }
    T *op = O + ((size_t)n * d.Cout + co0) * 16;
#pragma unroll
    for (int j = 0; j < CG; ++j)
        if (co0 + j < d.Cout) store_caps16<T>(op + j * 16, acc[j]);
}

// Data gradient: Ks[t][j][co] = K[p][q][c0 + j][co] (zero past C); thread = one input pixel.
template <typename T>
__global__ void __launch_bounds__(128) bwd_data_d4s(DimsT<int> d, const T *__restrict__ dO, const T *__restrict__ K,
                                                    T *__restrict__ dI) {
    extern __shared__ __align__(16) float Ks[];
    constexpr int CG = 4;
    const int g = blockIdx.x, c0 = g * CG;
    const int ntap = d.KH * d.KW;
    for (int e = threadIdx.x; e < ntap * CG * d.Cout * 16; e += blockDim.x) {
        const int k16 = e & 15, co = (e >> 4) % d.Cout, tj = (e >> 4) / d.Cout, j = tj % CG, t = tj / CG;
        Ks[e] = c0 + j < d.C ? ldf<T>(K + (((size_t)t * d.C + c0 + j) * d.Cout + co) * 16 + k16) : 0.f;
    }
    __syncthreads();
    // stride > 1: threads walk the input pixels phase by phase ((h mod s, w mod s)
    // outermost per image) so that a warp's lanes take the same taps
    const int Hq = (d.H + d.s - 1) / d.s, Wq = (d.W + d.s - 1) / d.s, s2 = d.s * d.s;
    const int v = blockIdx.y * blockDim.x + threadIdx.x;
    if (v >= d.B * s2 * Hq * Wq) return;
    const int ww = v % Wq, hh = (v / Wq) % Hq, ph = (v / (Wq * Hq)) % s2, b = v / (Wq * Hq * s2);
    const int h = hh * d.s + ph / d.s, w = ww * d.s + ph % d.s;
    if (h >= d.H || w >= d.W) return;
    const int n = (b * d.H + h) * d.W + w;
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    for (int p = 0; p < d.KH; ++p) {
        const int hx = h + d.pad - p;
        if (hx < 0 || hx % d.s) continue;
        const int x = hx / d.s;
        if (x >= d.Ho) continue;
        for (int q = 0; q < d.KW; ++q) {
            const int wy = w + d.pad - q;
            if (wy < 0 || wy % d.s) continue;
            const int y = wy / d.s;
            if (y >= d.Wo) continue;
            const T *gp = dO + ((size_t)(b * d.Ho + x) * d.Wo + y) * d.Cout * 16;
            const float *kt = Ks + (size_t)(p * d.KW + q) * CG * d.Cout * 16;
            for (int co = 0; co < d.Cout; ++co) {
                float gv[16];
                load_caps16<T>(gp + co * 16, gv);
#pragma unroll
                for (int j = 0; j < CG; ++j) {
                    float k[16];
                    lds_caps16(kt + (j * d.Cout + co) * 16, k);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int t = 0; t < 4; ++t)
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                acc[j][i * 4 + t] = fmaf(gv[i * 4 + m], k[t * 4 + m], acc[j][i * 4 + t]);
                }
            }
        }
    }
    T *ip = dI + ((size_t)n * d.C + c0) * 16;
#pragma unroll
    for (int j = 0; j < CG; ++j)
        if (c0 + j < d.C) store_caps16<T>(ip + j * 16, acc[j]);
}

// Weight gradient, four output channels per thread: thread = (tap, c, group of
// 4 c') x one split of the (b, x', y') range; each input capsule is loaded once
// per pixel for the four dO capsules (20 loads per 256 FMAs instead of 8 per 64).
template <typename T>
__global__ void __launch_bounds__(128) bwd_kernel_d4g(DimsT<int> d, const T *__restrict__ I, const T *__restrict__ dO,
                                                      float *__restrict__ part, int nsplit) {
    constexpr int CG = 4;
    const int ng = (d.Cout + CG - 1) / CG;
    const int nthr = d.KH * d.KW * d.C * ng;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nthr) return;
    const int split = blockIdx.y;
    const int gq = idx % ng, rest = idx / ng;
    const int c = rest % d.C, t = rest / d.C;
    const int q = t % d.KW, p = t / d.KW;
    const int co0 = gq * CG;
    const int npix = d.B * d.Ho * d.Wo;
    const int n0 = (int)((int64_t)npix * split / nsplit), n1 = (int)((int64_t)npix * (split + 1) / nsplit);
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    int y = n0 % d.Wo, x = (n0 / d.Wo) % d.Ho, b = n0 / (d.Wo * d.Ho);
    for (int n = n0; n < n1; ++n) {
        const int h = x * d.s + p - d.pad, w = y * d.s + q - d.pad;
        if (h >= 0 && h < d.H && w >= 0 && w < d.W) {
            float a[16];
            load_caps16<T>(I + (((size_t)(b * d.H + h) * d.W + w) * d.C + c) * 16, a);
            const T *gp = dO + ((size_t)n * d.Cout + co0) * 16;
#pragma unroll
            for (int j = 0; j < CG; ++j) {
                if (co0 + j < d.Cout) {
                    float g[16];
                    load_caps16<T>(gp + j * 16, g);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int tt = 0; tt < 4; ++tt)
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                acc[j][tt * 4 + m] = fmaf(a[i * 4 + tt], g[i * 4 + m], acc[j][tt * 4 + m]);
                }
            }
        }
        if (++y == d.Wo) { y = 0; if (++x == d.Ho) { x = 0; ++b; } }
    }
    const int ncaps = d.KH * d.KW * d.C * d.Cout;
#pragma unroll
    for (int j = 0; j < CG; ++j) {
        if (co0 + j >= d.Cout) continue;
        float *out = part + ((size_t)split * ncaps + ((size_t)t * d.C + c) * d.Cout + co0 + j) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            reinterpret_cast<float4 *>(out)[i] =
                make_float4(acc[j][4 * i], acc[j][4 * i + 1], acc[j][4 * i + 2], acc[j][4 * i + 3]);
    }
}

// Weight gradient, four input channels per thread: thread = (tap, group of 4 c,
// c') x one split; lanes run over c' so the four input capsules of a pixel are
// warp-wide broadcasts and the dO capsule loads are contiguous (20 loads per
// 256 FMAs; for many output channels, where bwd_kernel_d4g's wider threads lose).
template <typename T>
__global__ void __launch_bounds__(128) bwd_kernel_d4c(DimsT<int> d, const T *__restrict__ I, const T *__restrict__ dO,
                                                      float *__restrict__ part, int nsplit) {
    constexpr int CC = 4;
    const int ngc = d.C / CC;
    const int nthr = d.KH * d.KW * ngc * d.Cout;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nthr) return;
    const int split = blockIdx.y;
    const int co = idx % d.Cout, rest = idx / d.Cout;
    const int c0 = (rest % ngc) * CC, t = rest / ngc;
    const int q = t % d.KW, p = t / d.KW;
    const int npix = d.B * d.Ho * d.Wo;
    const int n0 = (int)((int64_t)npix * split / nsplit), n1 = (int)((int64_t)npix * (split + 1) / nsplit);
    float acc[CC][16];
#pragma unroll
    for (int j = 0; j < CC; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    int y = n0 % d.Wo, x = (n0 / d.Wo) % d.Ho, b = n0 / (d.Wo * d.Ho);
    for (int n = n0; n < n1; ++n) {
        const int h = x * d.s + p - d.pad, w = y * d.s + q - d.pad;
        if (h >= 0 && h < d.H && w >= 0 && w < d.W) {
            float g[16];
            load_caps16<T>(dO + ((size_t)n * d.Cout + co) * 16, g);
            const T *ip = I + (((size_t)(b * d.H + h) * d.W + w) * d.C + c0) * 16;
#pragma unroll
            for (int j = 0; j < CC; ++j) {
                float a[16];
                load_caps16<T>(ip + j * 16, a);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt)
#pragma unroll
                        for (int m = 0; m < 4; ++m)
                            acc[j][tt * 4 + m] = fmaf(a[i * 4 + tt], g[i * 4 + m], acc[j][tt * 4 + m]);
            }
        }
        if (++y == d.Wo) { y = 0; if (++x == d.Ho) { x = 0; ++b; } }
    }
    const int ncaps = d.KH * d.KW * d.C * d.Cout;
#pragma unroll
    for (int j = 0; j < CC; ++j) {
        float *out = part + ((size_t)split * ncaps + ((size_t)t * d.C + c0 + j) * d.Cout + co) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            reinterpret_cast<float4 *>(out)[i] =
                make_float4(acc[j][4 * i], acc[j][4 * i + 1], acc[j][4 * i + 2], acc[j][4 * i + 3]);
    }
}

// ============================================================ backward kernel
// Thread = (tap, c, c') kernel capsule x one split of the (b, x', y') range;
// acc[d2][d3] partial written to part[split][...].
template <typename T, typename IX>
__global__ void __launch_bounds__(128) bwd_kernel_d4(DimsT<IX> d, const T *__restrict__ I, const T *__restrict__ dO,
                                                     float *__restrict__ part, IX nsplit) {
    const IX ncaps = d.KH * d.KW * d.C * d.Cout;
    const IX idx = (IX)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncaps) return;
    const IX split = blockIdx.y;
    IX r = idx;
    const IX co = r % d.Cout; r /= d.Cout;
    const IX c = r % d.C; r /= d.C;
    const IX q = r % d.KW;
    const IX p = r / d.KW;
    const IX npix = d.B * d.Ho * d.Wo;
    const IX n0 = (IX)((int64_t)npix * split / nsplit), n1 = (IX)((int64_t)npix * (split + 1) / nsplit);
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
    for (IX n = n0; n < n1; ++n) {
        IX rr = n;
        const IX y = rr % d.Wo; rr /= d.Wo;
        const IX x = rr % d.Ho;
        const IX b = rr / d.Ho;
        const IX h = x * d.s + p - d.pad, w = y * d.s + q - d.pad;
        if (h < 0 || h >= d.H || w < 0 || w >= d.W) continue;
        float a[16], g[16];
        load_caps16<T>(I + (((b * d.H + h) * d.W + w) * d.C + c) * 16, a);
        load_caps16<T>(dO + (n * d.Cout + co) * 16, g);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    acc[t * 4 + m] = fmaf(a[i * 4 + t], g[i * 4 + m], acc[t * 4 + m]);
    }
    float *out = part + (split * ncaps + idx) * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        reinterpret_cast<float4 *>(out)[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
}

template <typename T>
__global__ void __launch_bounds__(256) bwd_kernel_gen(Dims d, const T *__restrict__ I, const T *__restrict__ dO,
                                                      float *__restrict__ part, int64_t nsplit) {
    const int64_t nk = d.KH * d.KW * d.C * d.Cout * d.D2 * d.D3;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nk) return;
    const int64_t split = blockIdx.y;
    int64_t r = idx;
    const int64_t n3 = r % d.D3; r /= d.D3;
    const int64_t t = r % d.D2; r /= d.D2;
    const int64_t co = r % d.Cout; r /= d.Cout;
    const int64_t c = r % d.C; r /= d.C;
    const int64_t q = r % d.KW;
    const int64_t p = r / d.KW;
    const int64_t npix = d.B * d.Ho * d.Wo;
    const int64_t n0 = npix * split / nsplit, n1 = npix * (split + 1) / nsplit;
    float acc = 0.f;
    for (int64_t n = n0; n < n1; ++n) {
        int64_t rr = n;
        const int64_t y = rr % d.Wo; rr /= d.Wo;
        const int64_t x = rr % d.Ho;
        const int64_t b = rr / d.Ho;
        const int64_t h = x * d.s + p - d.pad, w = y * d.s + q - d.pad;
        if (h < 0 || h >= d.H || w < 0 || w >= d.W) continue;
        const T *ip = I + ((((b * d.H + h) * d.W + w) * d.C + c) * d.D1) * d.D2 + t;
        const T *gp = dO + ((n * d.Cout + co) * d.D1) * d.D3 + n3;
        for (int64_t i = 0; i < d.D1; ++i) acc = fmaf(ldf(ip + i * d.D2), ldf(gp + i * d.D3), acc);
    }
    part[split * nk + idx] = acc;
}

// Fixed-order sum of the split partials (deterministic).
__global__ void __launch_bounds__(256) reduce_splits(const float *__restrict__ part, float *__restrict__ out,
                                                     int64_t n, int64_t nsplit) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    float acc = 0.f;
    for (int64_t s = 0; s < nsplit; ++s) acc += part[s * n + idx];
    out[idx] = acc;
}

// Fixed-order sum of forward tap-split partials into T outputs.
template <typename T>
__global__ void __launch_bounds__(256) reduce_splits_to(const float *__restrict__ part, T *__restrict__ out,
                                                        int64_t n, int64_t nsplit) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    float acc = 0.f;
    for (int64_t s = 0; s < nsplit; ++s) acc += part[s * n + idx];
    out[idx] = static_cast<T>(acc);
}

Dims dims_of(const Problem &p) {
    return Dims{p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW, p.D1, p.D2, p.D3, p.s, p.Ho, p.Wo, p.pad};
}

bool is_d4(const Problem &p) { return p.D1 == 4 && p.D2 == 4 && p.D3 == 4; }

inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// Every element offset the vectorised kernels form stays below n_in, n_out
// (x the forward tap splits) or n_k (x the dK splits): 32-bit indexing when
// those fit in an int.
bool fits32(const Problem &p, int64_t fwd_split, int64_t dk_split) {
    const int64_t lim = (int64_t)1 << 30;
    return p.n_in() < lim && p.n_out() * fwd_split < lim && p.n_k() * dk_split < lim;
}

// Number of splits of the (b, x', y') reduction for dK: enough threads to
// fill the machine a few times over, never more than the pixel count.
int64_t dk_splits(const Problem &p) {
    const int64_t units = !is_d4(p) ? p.n_k()
                          : p.C % 4 == 0 ? p.KH * p.KW * (p.C / 4) * p.Cout                       // bwd_kernel_d4c
                          : p.Cout >= 4 && p.Cout <= 8 ? p.KH * p.KW * p.C * ((p.Cout + 3) / 4)   // bwd_kernel_d4g
                                         : p.KH * p.KW * p.C * p.Cout;
    const int64_t target = (int64_t)device_info().num_sms * 2048;
    int64_t s = (target + units - 1) / units;
    const int64_t npix = p.n_pix_out();
    if (s > npix) s = npix;
    if (s > 1024) s = 1024;
    if (s < 1) s = 1;
    return s;
}

// Tap splits of the vectorised forward: when few output capsule groups exist
// (the FC layer: B*Cout/4 threads, each a 64-tap reduction) the taps are split
// over blockIdx.y into fp32 partials, summed in split order afterwards.
int64_t fwd_splits(const Problem &p) {
    if (!is_d4(p)) return 1;
    const int64_t units = p.B * p.Ho * p.Wo * (p.Cout >= 4 ? (p.Cout + 3) / 4 : p.Cout);
    const int64_t target = (int64_t)device_info().num_sms * 1024;
    int64_t s = units >= target ? 1 : (target + units - 1) / units;
    if (s > p.KH * p.KW) s = p.KH * p.KW;
    while (s > 1 && (size_t)s * (size_t)p.n_out() * 4 > ((size_t)64 << 20)) --s;
    return s < 1 ? 1 : s;
}

template <typename T>
cudaError_t fwd_impl(const Problem &p, const void *I, const void *K, void *O, void *ws, cudaStream_t st) {
    const Dims d = dims_of(p);
    const bool vec = is_d4(p) && ((uintptr_t)I % 16 == 0) && ((uintptr_t)K % 16 == 0) && ((uintptr_t)O % 16 == 0) &&
                     ((uintptr_t)ws % 16 == 0);
    if (vec) {
        const int64_t nsplit = ws ? fwd_splits(p) : 1;
        float *part = static_cast<float *>(ws);
        const bool i32 = fits32(p, nsplit, 1);
        const size_t ks_bytes = (size_t)p.KH * p.KW * p.C * 4 * 16 * sizeof(float);
        const int64_t npix = p.B * p.Ho * p.Wo;
        if (nsplit == 1 && i32 && p.Cout >= 4 && ks_bytes <= (size_t)kSimtSmemMax && (npix + 127) / 128 <= 65535) {
            cudaError_t e = smem_optin(reinterpret_cast<const void *>(fwd_d4s<T>), (int)ks_bytes);
            if (e != cudaSuccess) return e;
            fwd_d4s<T><<<dim3((unsigned)((p.Cout + 3) / 4), blocks_for(npix, 128)), 128, ks_bytes, st>>>(
                dims_as<int>(d), (const T *)I, (const T *)K, (T *)O);
            note_launches(1);
            return cudaGetLastError();
        }
        const int64_t n = p.B * p.Ho * p.Wo * (p.Cout >= 4 ? (p.Cout + 3) / 4 : p.Cout);
        const dim3 grid(blocks_for(n, 128), (unsigned)nsplit);
        if (p.Cout >= 4 && i32)
            fwd_d4<T, 4, int><<<grid, 128, 0, st>>>(dims_as<int>(d), (const T *)I, (const T *)K, (T *)O, part, (int)nsplit);
        else if (p.Cout >= 4)
            fwd_d4<T, 4, int64_t><<<grid, 128, 0, st>>>(d, (const T *)I, (const T *)K, (T *)O, part, (int)nsplit);
        else if (i32)
            fwd_d4<T, 1, int><<<grid, 128, 0, st>>>(dims_as<int>(d), (const T *)I, (const T *)K, (T *)O, part, (int)nsplit);
        else
            fwd_d4<T, 1, int64_t><<<grid, 128, 0, st>>>(d, (const T *)I, (const T *)K, (T *)O, part, (int)nsplit);
        if (nsplit > 1) {
            note_launches(1);
            reduce_splits_to<T><<<blocks_for(p.n_out(), 256), 256, 0, st>>>(part, (T *)O, p.n_out(), nsplit);
        }
    } else {
        fwd_gen<T><<<blocks_for(p.n_out(), 256), 256, 0, st>>>(d, (const T *)I, (const T *)K, (T *)O);
    }
    note_launches(1);
    return cudaGetLastError();
}

template <typename T>
cudaError_t bwd_data_impl(const Problem &p, const void *dO, const void *K, void *dI, cudaStream_t st) {
    const Dims d = dims_of(p);
    const bool vec = is_d4(p) && ((uintptr_t)dO % 16 == 0) && ((uintptr_t)K % 16 == 0) && ((uintptr_t)dI % 16 == 0);
    if (vec) {
        const bool i32 = fits32(p, 1, 1);
        const size_t ks_bytes = (size_t)p.KH * p.KW * 4 * p.Cout * 16 * sizeof(float);
        const int64_t npix = p.B * (p.s * p.s) * ((p.H + p.s - 1) / p.s) * ((p.W + p.s - 1) / p.s);   // phase grid
        if (i32 && p.C >= 4 && ks_bytes <= (size_t)kSimtSmemMax && (npix + 127) / 128 <= 65535 && npix < (1 << 30)) {
            cudaError_t e = smem_optin(reinterpret_cast<const void *>(bwd_data_d4s<T>), (int)ks_bytes);
            if (e != cudaSuccess) return e;
            bwd_data_d4s<T><<<dim3((unsigned)((p.C + 3) / 4), blocks_for(npix, 128)), 128, ks_bytes, st>>>(
                dims_as<int>(d), (const T *)dO, (const T *)K, (T *)dI);
            note_launches(1);
            return cudaGetLastError();
        }
        const int64_t n = p.B * p.H * p.W * (p.C >= 4 ? (p.C + 3) / 4 : p.C);
        const unsigned nb = blocks_for(n, 128);
        if (p.C >= 4 && i32)
            bwd_data_d4<T, 4, int><<<nb, 128, 0, st>>>(dims_as<int>(d), (const T *)dO, (const T *)K, (T *)dI);
        else if (p.C >= 4)
            bwd_data_d4<T, 4, int64_t><<<nb, 128, 0, st>>>(d, (const T *)dO, (const T *)K, (T *)dI);
        else if (i32)
            bwd_data_d4<T, 1, int><<<nb, 128, 0, st>>>(dims_as<int>(d), (const T *)dO, (const T *)K, (T *)dI);
        else
            bwd_data_d4<T, 1, int64_t><<<nb, 128, 0, st>>>(d, (const T *)dO, (const T *)K, (T *)dI);
    } else {
        bwd_data_gen<T><<<blocks_for(p.n_in(), 256), 256, 0, st>>>(d, (const T *)dO, (const T *)K, (T *)dI);
    }
    note_launches(1);
    return cudaGetLastError();
}

template <typename T>
cudaError_t bwd_kernel_impl(const Problem &p, const void *I, const void *dO, float *dK, void *ws,
                            cudaStream_t st) {
    const Dims d = dims_of(p);
    const int64_t nsplit = dk_splits(p);
    const bool vec = is_d4(p) && ((uintptr_t)I % 16 == 0) && ((uintptr_t)dO % 16 == 0) && ((uintptr_t)dK % 16 == 0) &&
                     ((uintptr_t)ws % 16 == 0);
    float *part = nsplit == 1 ? dK : (float *)ws;
    if (vec) {
        const int64_t ncaps = p.KH * p.KW * p.C * p.Cout;
        dim3 grid(blocks_for(ncaps, 128), (unsigned)nsplit);
        // four channels per thread pays for few output channels (stack L1, Cout = 8:
        // 2.71 -> 2.46 ms fp32); with many (L3, Cout = 32) the one-channel
        // threads' broadcast input loads and lower register count win (2.79 vs 4.88)
        if (fits32(p, 1, nsplit) && p.Cout >= 4 && p.Cout <= 8 && p.C % 4 != 0) {
            const int64_t nthr = p.KH * p.KW * p.C * ((p.Cout + 3) / 4);
            bwd_kernel_d4g<T><<<dim3(blocks_for(nthr, 128), (unsigned)nsplit), 128, 0, st>>>(
                dims_as<int>(d), (const T *)I, (const T *)dO, part, (int)nsplit);
        } else if (fits32(p, 1, nsplit) && p.C % 4 == 0) {
            const int64_t nthr = p.KH * p.KW * (p.C / 4) * p.Cout;
            bwd_kernel_d4c<T><<<dim3(blocks_for(nthr, 128), (unsigned)nsplit), 128, 0, st>>>(
                dims_as<int>(d), (const T *)I, (const T *)dO, part, (int)nsplit);
        } else if (fits32(p, 1, nsplit))
            bwd_kernel_d4<T, int><<<grid, 128, 0, st>>>(dims_as<int>(d), (const T *)I, (const T *)dO, part, (int)nsplit);
        else
            bwd_kernel_d4<T, int64_t><<<grid, 128, 0, st>>>(d, (const T *)I, (const T *)dO, part, nsplit);
    } else {
        dim3 grid(blocks_for(p.n_k(), 256), (unsigned)nsplit);
        bwd_kernel_gen<T><<<grid, 256, 0, st>>>(d, (const T *)I, (const T *)dO, part, nsplit);
    }
    note_launches(1);
    if (nsplit > 1) {
        reduce_splits<<<blocks_for(p.n_k(), 256), 256, 0, st>>>(part, dK, p.n_k(), nsplit);
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace

size_t simt_workspace_bytes(capsconv_op_t op, const Problem &p) {
    if (op == CAPSCONV_OP_FWD) {
        const int64_t s = fwd_splits(p);
        return s <= 1 ? 0 : (size_t)s * (size_t)p.n_out() * sizeof(float);
    }
    if (op != CAPSCONV_OP_BWD_KERNEL) return 0;
    const int64_t s = dk_splits(p);
    if (s <= 1) return 0;
    return (size_t)s * (size_t)p.n_k() * sizeof(float);
}

cudaError_t simt_fwd(const Problem &p, const void *I, const void *K, void *O, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
    if (ws_bytes < simt_workspace_bytes(CAPSCONV_OP_FWD, p)) ws = nullptr;   // no room: no tap split
    return p.dt == CAPSCONV_BF16 ? fwd_impl<__nv_bfloat16>(p, I, K, O, ws, st) : fwd_impl<float>(p, I, K, O, ws, st);
}

cudaError_t simt_bwd_data(const Problem &p, const void *dO, const void *K, void *dI, cudaStream_t st) {
    return p.dt == CAPSCONV_BF16 ? bwd_data_impl<__nv_bfloat16>(p, dO, K, dI, st)
                                 : bwd_data_impl<float>(p, dO, K, dI, st);
}

cudaError_t simt_bwd_kernel(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                            cudaStream_t st) {
    (void)ws_bytes;
    return p.dt == CAPSCONV_BF16 ? bwd_kernel_impl<__nv_bfloat16>(p, I, dO, dK, ws, st)
                                 : bwd_kernel_impl<float>(p, I, dO, dK, ws, st);
}

}  // namespace capsconv
