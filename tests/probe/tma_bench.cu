// TMA throughput microbenchmark: every CTA (one per SM) streams `iters` rounds
// of `nbox` copies into shared memory (mode 0: 4-D tensor boxes of the capsule
// map; mode 1: 1-D bulk copies of the same byte count), one mbarrier per round.
#include <cuda.h>
#include <cstdio>
#include "umma.cuh"
#include "tma.h"
using namespace capsconv;
using namespace capsconv::umma;

__global__ void tbench(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2, const uint8_t *src, int mode, int nbox, int iters,
                       int box_bytes, int W, int nrows_total, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, never;
    __shared__ volatile int done;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&never, 1); mbar_fence_init(); done = 0; }
    __syncthreads();
    if (threadIdx.x >= 32) {            // extra warps poll a barrier until the copier finishes
        while (!done) { mbar_try_wait(&never, 0); }
        return;
    }
    if (threadIdx.x != 0) return;
    const uint32_t dst = smem_u32(smem);
    unsigned long long t0 = clock64(), tissue = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned long long ta = clock64();
        mbar_arrive_expect_tx(&bar, (uint32_t)(nbox * box_bytes));
        for (int b = 0; b < nbox; ++b) {
            const int row = (blockIdx.x * 37 + it * nbox + b + blockIdx.x * iters * nbox) % nrows_total;
            if (mode == 0) tma::load4d(dst + b * box_bytes, &tm, 0, 0, row % 24, row / 24, smem_u32(&bar));
            else if (mode == 2) tma::load4d(dst + b * box_bytes, (b * 8 / nbox) < 5 ? &tm : &tm2, 0, 0, row % 24, row / 24, smem_u32(&bar));
            else if (mode == 1) bulk_g2s_u32(dst + b * box_bytes, src + (size_t)row * W * 256, box_bytes, &bar);
        }
        tissue += clock64() - ta;
        mbar_wait(&bar, it & 1);
    }
    unsigned long long t1 = clock64();
    done = 1;
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = tissue; }
}

extern "C" double tma_bench(int mode, int nbox, int iters, int W, int rows_per_box, int B, int boxw, int nthreads) {
    // tensor: B images of 24 x W pixels, 8 channels x 16 bf16 (256 B / pixel)
    const int64_t H = 24, CS = 8;
    uint8_t *src;
    cudaMalloc(&src, (size_t)B * H * W * 256);
    cudaMemset(src, 1, (size_t)B * H * W * 256);
    CUtensorMap tm, tm2;
    if (!make_capsule_tmap(&tm, src, B, H, W, CS, 8, boxw, rows_per_box, 1, 1)) return -2;
    uint8_t *src2;
    cudaMalloc(&src2, (size_t)B * H * W * 256);
    cudaMemset(src2, 1, (size_t)B * H * W * 256);
    if (!make_capsule_tmap(&tm2, src2, B, H, W, CS, 8, boxw, rows_per_box, 1, 1)) return -2;
    unsigned long long *d;
    cudaMalloc(&d, 16);
    const int box_bytes = boxw * 256 * rows_per_box;
    cudaFuncSetAttribute(tbench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    tbench<<<148, nthreads, 200 * 1024>>>(tm, tm2, src, mode, nbox, iters, box_bytes, W, (int)(B * H - 8), d);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tbench<<<148, nthreads, 200 * 1024>>>(tm, tm2, src, mode, nbox, iters, box_bytes, W, (int)(B * H - 8), d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("   [cta0: total %llu cyc, issue %llu cyc (%.0f%%), per round total %.0f issue %.0f]\n", h[0], h[1],
           100.0 * h[1] / h[0], (double)h[0] / iters, (double)h[1] / iters);
    cudaFree(src); cudaFree(src2); cudaFree(d);
    if (e != cudaSuccess) return -1;
    const double bytes = 148.0 * iters * nbox * box_bytes;
    return bytes / (ms * 1e-3) / 1e9;   // GB/s chip-wide
}
