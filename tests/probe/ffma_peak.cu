// ffma_peak.cu -- FP32 FFMA peak of this GPU: every thread runs
// 8 independent dependent-FMA chains; 148 x 8 CTAs of 256 threads; timed with
// CUDA events.  The roofline of the fp32 (SIMT) path in bench.py uses the
// derived figure SMs x 128 lanes x 2 flop x max SM clock; this measures it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_peak ffma_peak.cu && ./ffma_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float *out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[threadIdx.x] = s;   // keep the chains alive
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 1024 * sizeof(float));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    ffma_kernel<<<blocks, threads>>>(out, 16, 0.999f, 0.001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    printf("{\"ffma_tflops\": %.2f, \"sms\": %d}\n", best, sms);
    return 0;
}
