// slices.cu -- S-slice capsules (R22) as a
// channel-expanded capsule convolution.
//
// With I [..][C][S][D1][D2] and O [..][Cout][S][D1][D3], slice s of every
// capsule is its own matrix capsule: the slice-wise convolution is exactly the
// matrix-capsule convolution over C*S input and Cout*S output channels whose
// kernel is block-diagonal in the slice index,
//     K'[p][q][(c, s)][(c', s')][d2][d3] = (s == s') ? K[p][q][c][c'][s][d2][d3] : 0,
// and I, O are the same memory read as [..][C*S][D1][D2] / [..][Cout*S][D1][D3].
// dK is the diagonal of the expanded dK'.  Every stage runs on the library's
// tensor-core / SIMT kernels; the price is S x the useful flops (the zero
// blocks), stated in the bench line.
#include <cuda_bf16.h>

#include "internal.h"

namespace capsconv {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) expand_blockdiag(const T *__restrict__ K, T *__restrict__ Kx, int64_t taps,
                                                        int64_t C, int64_t Cout, int64_t S, int64_t D23) {
    const int64_t n = taps * C * S * Cout * S * D23;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    int64_t r = idx;
    const int64_t e = r % D23; r /= D23;
    const int64_t so = r % S; r /= S;
    const int64_t co = r % Cout; r /= Cout;
    const int64_t si = r % S; r /= S;
    const int64_t c = r % C;
    const int64_t tap = r / C;
    T v = (T)0.f;
    if (si == so) v = K[((((tap * C + c) * Cout + co) * S + si) * D23) + e];
    Kx[idx] = v;
}

__global__ void __launch_bounds__(256) extract_diag(const float *__restrict__ dKx, float *__restrict__ dK, int64_t taps,
                                                    int64_t C, int64_t Cout, int64_t S, int64_t D23) {
    const int64_t n = taps * C * Cout * S * D23;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    int64_t r = idx;
    const int64_t e = r % D23; r /= D23;
    const int64_t s = r % S; r /= S;
    const int64_t co = r % Cout; r /= Cout;
    const int64_t c = r % C;
    const int64_t tap = r / C;
    dK[idx] = dKx[((((tap * C + c) * S + s) * Cout + co) * S + s) * D23 + e];
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t slices_expand_kernel(capsconv_dtype_t dt, const void *K, void *Kx, int64_t taps, int64_t C, int64_t Cout,
                                 int64_t S, int64_t D23, cudaStream_t st) {
    const int64_t n = taps * C * S * Cout * S * D23;
    if (dt == CAPSCONV_BF16)
        expand_blockdiag<__nv_bfloat16><<<nblk(n), 256, 0, st>>>(static_cast<const __nv_bfloat16 *>(K),
                                                                 static_cast<__nv_bfloat16 *>(Kx), taps, C, Cout, S, D23);
    else
        expand_blockdiag<float><<<nblk(n), 256, 0, st>>>(static_cast<const float *>(K), static_cast<float *>(Kx), taps,
                                                         C, Cout, S, D23);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t slices_extract_dk(const float *dKx, float *dK, int64_t taps, int64_t C, int64_t Cout, int64_t S,
                              int64_t D23, cudaStream_t st) {
    const int64_t n = taps * C * Cout * S * D23;
    extract_diag<<<nblk(n), 256, 0, st>>>(dKx, dK, taps, C, Cout, S, D23);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace capsconv
