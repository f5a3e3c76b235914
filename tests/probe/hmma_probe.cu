// Throughput of legacy warp-level mma.sync m16n8k16 bf16 (fp32 accumulate) on
// sm_100a: many warps, register operands, no memory traffic.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void hmma_loop(float *out, int iters) {
    unsigned a0 = threadIdx.x * 0x3c003c00u, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 4, b1 = a0 ^ 5;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 4096, blocks = 148 * 2;
        hmma_loop<<<blocks, warps * 32>>>(out, 16);
        cudaEventRecord(e0);
        hmma_loop<<<blocks, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * warps * blocks;
        printf("warps/CTA=%d: %.1f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
