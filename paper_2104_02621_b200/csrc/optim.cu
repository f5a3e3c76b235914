// optim.cu -- the optimizer step of the training step:
// plain SGD on an fp32 master copy of a weight tensor, with the working copy
// (bf16 or fp32, the dtype the convolution calls read) rewritten in the same
// pass.  Memory-bound elementwise work: 4 + 4 + 4 + |w_out| bytes per
// element, one 16-byte vector per thread and 4 elements per vector.
#include <cuda_bf16.h>

#include "internal.h"

namespace capsconv {
namespace {

template <typename T>
__device__ __forceinline__ void store4(T *p, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16 *p, float4 v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t *>(&a);
    u.y = *reinterpret_cast<uint32_t *>(&b);
    *reinterpret_cast<uint2 *>(p) = u;
}

template <typename T>
__global__ void __launch_bounds__(256) sgd_kernel(int64_t n, float lr, float *w, const float *__restrict__ g,
                                                  T *out) {   // out may be w (fp32): no __restrict__ on either
    const int64_t i4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i4 + 4 <= n) {
        float4 a = *reinterpret_cast<const float4 *>(w + i4);
        const float4 d = __ldg(reinterpret_cast<const float4 *>(g + i4));
        a.x = fmaf(-lr, d.x, a.x);
        a.y = fmaf(-lr, d.y, a.y);
        a.z = fmaf(-lr, d.z, a.z);
        a.w = fmaf(-lr, d.w, a.w);
        *reinterpret_cast<float4 *>(w + i4) = a;
        store4<T>(out + i4, a);
    } else {
        for (int64_t i = i4; i < n; ++i) {   // ragged tail
            const float a = fmaf(-lr, g[i], w[i]);
            w[i] = a;
            if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(a);
            else out[i] = a;
        }
    }
}

}  // namespace

cudaError_t sgd_update(capsconv_dtype_t wdt, int64_t n, float lr, float *w, const float *g, void *out,
                       cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int64_t nthr = (n + 3) / 4;
    const dim3 grid((unsigned)((nthr + 255) / 256));
    if (wdt == CAPSCONV_BF16)
        sgd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(n, lr, w, g, static_cast<__nv_bfloat16 *>(out));
    else
        sgd_kernel<float><<<grid, 256, 0, st>>>(n, lr, w, g, static_cast<float *>(out));
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace capsconv
