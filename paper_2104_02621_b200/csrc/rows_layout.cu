// rows_layout.cu -- capsule-row permutation between the natural layout
// [..pixel][C][D1][D2] and the D1-outer ("rows") layout [..pixel][D1][C][D2].
//
// The rows layout is an internal layout choice (reading R3: memory order is
// invisible to the mathematics; PAPER.md's Algorithm 2 itself is
// channel-major).  Problems the rows-layout tensor-core kernels do not take
// (fp32, capsules other than 4x4, padding, ...) run the natural-layout path
// between two of these permutations, so every valid rows-layout call has a
// path (the dispatch rule stays total).
#include <cuda_bf16.h>

#include "internal.h"

namespace capsconv {
namespace {

// One thread per (pixel, c, d1) capsule row of D2 elements.
template <typename T>
__global__ void permute_kernel(const T *__restrict__ src, T *__restrict__ dst, long long nrows, int C, int D1, int D2,
                               int to_rows) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const long long pix = r / ((long long)C * D1);
    const int rem = (int)(r - pix * C * D1);
    const int c = rem / D1, d1 = rem - c * D1;          // natural order of this capsule row
    const long long nat = (((pix * C + c) * D1) + d1) * D2;
    const long long row = (((pix * D1 + d1) * C) + c) * D2;
    const T *s = src + (to_rows ? nat : row);
    T *d = dst + (to_rows ? row : nat);
    for (int i = 0; i < D2; ++i) d[i] = s[i];
}

// Capsule rows of 4 bf16 (8 bytes) or 4 fp32 (16 bytes) moved whole: one
// thread per row, consecutive threads read consecutive rows of the source.
template <typename V>
__global__ void permute_rows_kernel(const V *__restrict__ src, V *__restrict__ dst, long long nrows, int C, int D1,
                                    int to_rows) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int per = C * D1;
    const long long pix = r / per;
    const int rem = (int)(r - pix * per);
    // the source is read in order: decompose r in the SOURCE layout
    int c, d1;
    if (to_rows) { c = rem / D1; d1 = rem - c * D1; }      // natural source: (c, d1)
    else { d1 = rem / C; c = rem - d1 * C; }                // rows source: (d1, c)
    const long long nat = pix * per + (long long)c * D1 + d1;
    const long long row = pix * per + (long long)d1 * C + c;
    dst[to_rows ? row : nat] = __ldg(src + (to_rows ? nat : row));
}

}  // namespace

cudaError_t permute_layout(capsconv_dtype_t dt, const void *src, void *dst, int64_t npix, int64_t C, int64_t D1,
                           int64_t D2, int to_rows, cudaStream_t st) {
    const long long nrows = (long long)npix * C * D1;
    if (nrows == 0) return cudaSuccess;
    const dim3 grid((unsigned)((nrows + 255) / 256));
    if (D2 == 4) {   // whole capsule rows: 8 bytes (bf16) / 16 bytes (fp32)
        if (dt == CAPSCONV_BF16)
            permute_rows_kernel<uint2><<<grid, 256, 0, st>>>(static_cast<const uint2 *>(src), static_cast<uint2 *>(dst),
                                                             nrows, (int)C, (int)D1, to_rows);
        else
            permute_rows_kernel<uint4><<<grid, 256, 0, st>>>(static_cast<const uint4 *>(src), static_cast<uint4 *>(dst),
                                                             nrows, (int)C, (int)D1, to_rows);
        note_launches(1);
        return cudaGetLastError();
    }
    if (dt == CAPSCONV_BF16)
        permute_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16 *>(src),
                                                            static_cast<__nv_bfloat16 *>(dst), nrows, (int)C, (int)D1,
                                                            (int)D2, to_rows);
    else
        permute_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float *>(src), static_cast<float *>(dst), nrows,
                                                    (int)C, (int)D1, (int)D2, to_rows);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace capsconv
