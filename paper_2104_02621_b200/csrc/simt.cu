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

struct Dims {
    int64_t B, H, W, C, Cout, KH, KW, D1, D2, D3, s, Ho, Wo;
    int64_t pad;   // symmetric zero padding: input pixel (x*s + p - pad, y*s + q - pad); outside = 0
};

// ============================================================ forward
// Thread = (b, x', y', group of CG output channels); acc[CG][d1][d3].
template <typename T, int CG>
__global__ void __launch_bounds__(128) fwd_d4(Dims d, const T *__restrict__ I, const T *__restrict__ K,
                                              T *__restrict__ O, float *__restrict__ part, int nsplit) {
    const int64_t ngroups = (d.Cout + CG - 1) / CG;
    const int64_t total = d.B * d.Ho * d.Wo * ngroups;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int64_t r = idx;
    const int64_t y = r % d.Wo; r /= d.Wo;
    const int64_t x = r % d.Ho; r /= d.Ho;
    const int64_t b = r % d.B;
    const int64_t g = r / d.B;
    const int64_t co0 = g * CG;
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
    // split blockIdx.y of nsplit takes the taps [t0, t1) (fixed ranges: the
    // partials are summed in split order, deterministic)
    const int64_t ntap = d.KH * d.KW, t0 = ntap * blockIdx.y / nsplit, t1 = ntap * (blockIdx.y + 1) / nsplit;
    for (int64_t t = t0; t < t1; ++t) {
        const int64_t p = t / d.KW, q = t - p * d.KW;
        const int64_t h = x * d.s + p - d.pad;
        if (h < 0 || h >= d.H) continue;
        {
            const int64_t w = y * d.s + q - d.pad;
            if (w < 0 || w >= d.W) continue;
            const T *ip = I + (((b * d.H + h) * d.W + w) * d.C) * 16;
            const T *kp = K + (((p * d.KW + q) * d.C) * d.Cout + co0) * 16;
            for (int64_t c = 0; c < d.C; ++c) {
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
    const int64_t oo = (((b * d.Ho + x) * d.Wo + y) * d.Cout + co0) * 16;
    if (nsplit > 1) {
        float *pp = part + (int64_t)blockIdx.y * (d.B * d.Ho * d.Wo * d.Cout * 16) + oo;
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
template <typename T, int CG>
__global__ void __launch_bounds__(128) bwd_data_d4(Dims d, const T *__restrict__ dO, const T *__restrict__ K,
                                                   T *__restrict__ dI) {
    const int64_t ngroups = (d.C + CG - 1) / CG;
    const int64_t total = d.B * d.H * d.W * ngroups;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int64_t r = idx;
    const int64_t g = r % ngroups; r /= ngroups;
    const int64_t w = r % d.W; r /= d.W;
    const int64_t h = r % d.H;
    const int64_t b = r / d.H;
    const int64_t c0 = g * CG;
    float acc[CG][16];
#pragma unroll
    for (int j = 0; j < CG; ++j)
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[j][e] = 0.f;
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
            const T *gp = dO + ((b * d.Ho + x) * d.Wo + y) * d.Cout * 16;
            const T *kp = K + (((p * d.KW + q) * d.C + c0) * d.Cout) * 16;
            for (int64_t co = 0; co < d.Cout; ++co) {
                float gv[16];
                load_caps16<T>(gp + co * 16, gv);
#pragma unroll
                for (int j = 0; j < CG; ++j) {
                    if (c0 + j < d.C) {
                        float k[16];
                        load_caps16<T>(kp + ((int64_t)j * d.Cout + co) * 16, k);
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

// ============================================================ backward kernel
// Thread = (tap, c, c') kernel capsule x one split of the (b, x', y') range;
// acc[d2][d3] partial written to part[split][...].
template <typename T>
__global__ void __launch_bounds__(128) bwd_kernel_d4(Dims d, const T *__restrict__ I, const T *__restrict__ dO,
                                                     float *__restrict__ part, int64_t nsplit) {
    const int64_t ncaps = d.KH * d.KW * d.C * d.Cout;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncaps) return;
    const int64_t split = blockIdx.y;
    int64_t r = idx;
    const int64_t co = r % d.Cout; r /= d.Cout;
    const int64_t c = r % d.C; r /= d.C;
    const int64_t q = r % d.KW;
    const int64_t p = r / d.KW;
    const int64_t npix = d.B * d.Ho * d.Wo;
    const int64_t n0 = npix * split / nsplit, n1 = npix * (split + 1) / nsplit;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
    for (int64_t n = n0; n < n1; ++n) {
        int64_t rr = n;
        const int64_t y = rr % d.Wo; rr /= d.Wo;
        const int64_t x = rr % d.Ho;
        const int64_t b = rr / d.Ho;
        const int64_t h = x * d.s + p - d.pad, w = y * d.s + q - d.pad;
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

// Number of splits of the (b, x', y') reduction for dK: enough threads to
// fill the machine a few times over, never more than the pixel count.
int64_t dk_splits(const Problem &p) {
    const int64_t units = is_d4(p) ? p.KH * p.KW * p.C * p.Cout : p.n_k();
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
        if (p.Cout >= 4) {
            const int64_t n = p.B * p.Ho * p.Wo * ((p.Cout + 3) / 4);
            fwd_d4<T, 4><<<dim3(blocks_for(n, 128), (unsigned)nsplit), 128, 0, st>>>(d, (const T *)I, (const T *)K,
                                                                                  (T *)O, part, (int)nsplit);
        } else {
            const int64_t n = p.B * p.Ho * p.Wo * p.Cout;
            fwd_d4<T, 1><<<dim3(blocks_for(n, 128), (unsigned)nsplit), 128, 0, st>>>(d, (const T *)I, (const T *)K,
                                                                                  (T *)O, part, (int)nsplit);
        }
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
        if (p.C >= 4) {
            const int64_t n = p.B * p.H * p.W * ((p.C + 3) / 4);
            bwd_data_d4<T, 4><<<blocks_for(n, 128), 128, 0, st>>>(d, (const T *)dO, (const T *)K, (T *)dI);
        } else {
            const int64_t n = p.B * p.H * p.W * p.C;
            bwd_data_d4<T, 1><<<blocks_for(n, 128), 128, 0, st>>>(d, (const T *)dO, (const T *)K, (T *)dI);
        }
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
        bwd_kernel_d4<T><<<grid, 128, 0, st>>>(d, (const T *)I, (const T *)dO, part, nsplit);
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
