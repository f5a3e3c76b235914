// umma_probe.cu -- test-only probe of the tcgen05 descriptor conventions in
// csrc/umma.cuh: one CTA computes D = A(MxK) * B(NxK)^T with A and B staged in
// shared memory in the canonical no-swizzle K-major or MN-major layouts,
// including a start-address shift (the tap shift the capsule kernels use).
#include <cuda_bf16.h>
#include "umma.cuh"

using namespace capsconv::umma;

// A: global [RA][K] row-major (RA >= 128 + shift rows for K-major shifts,
//    or K + kshift columns for MN-major k-shifts), B: global [N][K].
// a_mn: 0 K-major, 1 MN-major.  Elements are 16-bit (bf16) or 32-bit (tf32).
template <typename T>
__global__ void probe_kernel(const T *A, const T *B, float *D, int RA, int KA, int N, int K, int a_mn, int b_mn,
                             int shift, int swz) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    constexpr int E = sizeof(T);          // bytes per element
    constexpr int PER16 = 16 / E;         // elements per 16-byte row
    const int tid = threadIdx.x;
    uint8_t *sA = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
    const int RApad = (RA + 7) / 8 * 8;
    const int KApad = (KA + 7) / 8 * 8;
    // A layout
    uint32_t a_lbo, a_sbo;
    if (swz) {    // SWIZZLE_128B K-major: 128-byte rows, chunk ^ (row % 8); K == 64
        a_lbo = 16; a_sbo = 1024;
        for (int i = tid; i < RA * KA; i += blockDim.x) {
            int r = i / KA, k = i % KA;
            *(T *)(sA + (r / 8) * 1024 + (r % 8) * 128 + (((k * E / 16) ^ (r % 8)) * 16) + (k * E % 16)) = A[i];
        }
    } else if (!a_mn) {  // K-major: rows at 16 B, row groups SBO=128, k-chunks LBO = RApad*16
        a_lbo = RApad * 16; a_sbo = 128;
        for (int i = tid; i < RA * KA; i += blockDim.x) {
            int r = i / KA, k = i % KA;
            *(T *)(sA + (k / PER16) * a_lbo + r * 16 + (k % PER16) * E) = A[i];
        }
    } else {      // MN-major: k rows at 16 B (k-groups LBO=128), m-groups at SBO = KApad*16
        a_lbo = 128; a_sbo = KApad * 16;
        for (int i = tid; i < RA * KA; i += blockDim.x) {
            int m = i / KA, k = i % KA;
            *(T *)(sA + (m / PER16) * a_sbo + (m % PER16) * E + k * 16) = A[i];
        }
    }
    uint8_t *sB = sA + 65536;
    uint32_t b_lbo, b_sbo;
    const int Npad = (N + 7) / 8 * 8;
    if (swz) {
        b_lbo = 16; b_sbo = 1024;
        for (int i = tid; i < N * K; i += blockDim.x) {
            int n = i / K, k = i % K;
            *(T *)(sB + (n / 8) * 1024 + (n % 8) * 128 + (((k * E / 16) ^ (n % 8)) * 16) + (k * E % 16)) = B[i];
        }
    } else if (!b_mn) {
        b_lbo = Npad * 16; b_sbo = 128;
        for (int i = tid; i < N * K; i += blockDim.x) {
            int n = i / K, k = i % K;
            *(T *)(sB + (k / PER16) * b_lbo + n * 16 + (k % PER16) * E) = B[i];
        }
    } else {
        b_lbo = 128; b_sbo = ((K + 7) / 8 * 8) * 16;
        for (int i = tid; i < N * K; i += blockDim.x) {
            int n = i / K, k = i % K;
            *(T *)(sB + (n / PER16) * b_sbo + (n % PER16) * E + k * 16) = B[i];
        }
    }
    if (tid < 32) tmem_alloc<256>(&tmem_base);
    if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = (E == 2) ? idesc_bf16(128, N, a_mn, b_mn) : idesc_tf32(128, N, a_mn, b_mn);
        const int ksteps = K / (32 / E);   // 16 bf16 or 8 tf32 per MMA = 2 chunks
        for (int ks = 0; ks < ksteps; ++ks) {
            uint32_t a_addr, b_addr;
            // K-major: a K-step is (32/E)/PER16 = 2 chunks of 16 B; MN-major: (32/E)/8 k-groups.
            const int a_adv = a_mn ? (32 / E) / 8 : 2, b_adv = b_mn ? (32 / E) / 8 : 2;
            a_addr = smem_u32(sA) + shift * 16 + ks * a_adv * a_lbo;   // shift: rows (K-major) / k-rows (MN)
            b_addr = smem_u32(sB) + ks * b_adv * b_lbo;
            uint64_t ad = smem_desc(a_addr, a_lbo, a_sbo);
            uint64_t bd = smem_desc(b_addr, b_lbo, b_sbo);
            if (swz) {
                a_addr = smem_u32(sA) + shift * 128 + ks * 32;
                b_addr = smem_u32(sB) + ks * 32;
                ad = smem_desc(a_addr, 16, 1024) | (2ull << 61);
                bd = smem_desc(b_addr, 16, 1024) | (2ull << 61);
                if (swz == 2) ad |= (uint64_t)((a_addr >> 7) & 7) << 49;   // base offset
            }
            if (E == 2) mma_bf16_ss(tm, ad, bd, idesc, ks > 0);
            else mma_tf32_ss(tm, ad, bd, idesc, ks > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after_sync();
    const int warp = tid / 32, lane = tid % 32;
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
        float v[8];
        tmem_ld8(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_wait_ld();
        for (int j = 0; j < 8 && c0 + j < N; ++j) D[row * N + c0 + j] = v[j];
    }
    fence_before_sync();
    __syncthreads();
    if (tid < 32) tmem_dealloc<256>(tm);
}

extern "C" int umma_probe(int tf32, const void *A, const void *B, float *D, int RA, int KA, int N, int K, int a_mn,
                          int b_mn, int shift, int swz) {
    const size_t smem = 65536 * 2 + 1024;
    if (tf32) {
        cudaFuncSetAttribute(probe_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        probe_kernel<float><<<1, 128, smem>>>((const float *)A, (const float *)B, D, RA, KA, N, K, a_mn, b_mn, shift, swz);
    } else {
        cudaFuncSetAttribute(probe_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        probe_kernel<__nv_bfloat16><<<1, 128, smem>>>((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)B, D, RA, KA,
                                                       N, K, a_mn, b_mn, shift, swz);
    }
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}

// ---------------------------------------------------------------------------
// Throughput microbenchmark: `iters` back-to-back 128xNx16 bf16 MMAs into one
// accumulator, operands from shared memory (SS) or A from TMEM (TS).  All
// CTAs run the same loop; returns cycles per MMA measured by CTA 0.
__global__ void bench_kernel(int N, int iters, int a_tmem, int nacc, int lay, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    for (int i = tid; i < 65536 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    if (tid < 32) tmem_alloc<512>(&tmem_base);
    if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    if (tid < 32) {
        const uint32_t idesc = idesc_bf16(128, N, 0, 0);
        const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
        uint64_t ad = smem_desc(sa, lay == 1 ? 128 * 16 + 64 : 128 * 16, 128);
        uint64_t bd = smem_desc(sb, lay == 1 ? 256 * 16 + 64 : 256 * 16, 128);
        if (lay == 2) {
            ad = smem_desc((sa + 1023) & ~1023u, 16, 1024) | (2ull << 61);
            bd = smem_desc((sb + 1023) & ~1023u, 16, 1024) | (2ull << 61);
        }
        const uint32_t step = nacc > 1 ? (uint32_t)N : 0u;
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; it += 8) {
            if (elect_one()) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t dcol = tm + (uint32_t)(u & 1) * step;
                    if (a_tmem) {
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dcol),
                            "r"(tm + 384), "l"(bd), "r"(idesc), "r"(1));
                    } else {
                        mma_bf16_ss(dcol, ad, bd, idesc, 1);
                    }
                }
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) *cycles = (t1 - t0);
    }
    fence_before_sync();
    __syncthreads();
    if (tid < 32) tmem_dealloc<512>(tm);
}

extern "C" double umma_bench(int N, int iters, int a_tmem, int nblocks, int nacc, int lay) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 32768);
    bench_kernel<<<nblocks, 128, 65536 + 32768>>>(N, iters, a_tmem, nacc, lay, d);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h / iters;
}

// ---------------------------------------------------------------------------
// TS probe: A (128 x K bf16) written into TMEM with tcgen05.st (lane = row,
// 32-bit column j = k pair (2j, 2j+1)), B (N x K) K-major in shared memory;
// D = A * B^T with kind::f16 A-from-TMEM.
__global__ void probe_ts(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D, int N, int K) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    uint8_t *sB = smem;
    const int Npad = (N + 7) / 8 * 8;
    const uint32_t b_lbo = Npad * 16, b_sbo = 128;
    for (int i = tid; i < N * K; i += blockDim.x) {
        int n = i / K, k = i % K;
        *(__nv_bfloat16 *)(sB + (k / 8) * b_lbo + n * 16 + (k % 8) * 2) = B[i];
    }
    if (warp == 0) tmem_alloc<512>(&tmem_base);
    if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    const uint32_t a_col = 256;   // A at columns [256, 256 + K/2)
    // each warp writes its lane quarter: row = warp*32 + lane, 8 columns at a time
    const int row = warp * 32 + lane;
    for (int j0 = 0; j0 < K / 2; j0 += 8) {
        uint32_t r[8];
        for (int j = 0; j < 8; ++j) {
            __nv_bfloat162 h;
            h.x = A[row * K + 2 * (j0 + j)];
            h.y = A[row * K + 2 * (j0 + j) + 1];
            r[j] = *reinterpret_cast<uint32_t *>(&h);
        }
        const uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16) + a_col + j0;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                     : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (warp == 0) {
        const uint32_t idesc = idesc_bf16(128, N, 0, 0);
        if (elect_one()) {
            for (int ks = 0; ks < K / 16; ++ks) {
                const uint64_t bd = smem_desc(smem_u32(sB) + ks * 2 * b_lbo, b_lbo, b_sbo);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm),
                    "r"(tm + a_col + ks * 8), "l"(bd), "r"(idesc), "r"(ks > 0 ? 1 : 0));
            }
            mma_commit(&bar);
        }
        __syncwarp();
    }
    mbar_wait(&bar, 0);
    fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 8) {
        float v[8];
        tmem_ld8(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_wait_ld();
        for (int j = 0; j < 8 && c0 + j < N; ++j) D[row * N + c0 + j] = v[j];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" int umma_probe_ts(const void *A, const void *B, float *D, int N, int K) {
    cudaFuncSetAttribute(probe_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    probe_ts<<<1, 128, 65536>>>((const __nv_bfloat16 *)A, (const __nv_bfloat16 *)B, D, N, K);
    return (int)cudaDeviceSynchronize();
}

// Variant of bench_kernel with wgrad's operand forms: B MN-major (LBO 128,
// SBO = 8 k-rows... see wgrad.cu) or K-major, A from TMEM walking `a_step`
// columns per MMA over 8 k-steps.  Returns cycles per MMA (CTA 0).
__global__ void bench2_kernel(int N, int iters, int b_mn, int a_step, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, done;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    for (int i = tid; i < 65536 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    if (tid < 32) tmem_alloc<512>(&tmem_base);
    if (tid == 0) { mbar_init(&bar, 1); mbar_init(&done, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    if (tid >= 32) {
        mbar_wait(&done, 0);   // spinning waiters (as the idle roles of a warp-specialised kernel)
    } else {
        const uint32_t idesc = idesc_bf16(128, N, 0, b_mn);
        const uint32_t sb = smem_u32(smem);
        // MN-major: n-groups of 8 at SBO = 128 * (k rows per stage = 128) ... use K=128 rows of 16 B per n-group
        const uint64_t bd = b_mn ? smem_desc(sb, 128, 128 * 16) : smem_desc(sb, 256 * 16, 128);
        unsigned long long t0 = clock64();
        // a_step: 0 -> one A block; 8 -> 8 blocks; -1 -> 24 blocks, 3 accumulators (wgrad);
        // -2 -> 24 blocks, one accumulator; -3 -> 8 blocks, 3 accumulators.  Constant offsets.
        for (int it = 0; it < iters; it += 24) {
            if (elect_one()) {
#pragma unroll
                for (int u = 0; u < 24; ++u) {
                    uint32_t acol, dcol;
                    if (a_step >= 0) { acol = 256 + (u % 8) * a_step; dcol = 0; }
                    else if (a_step == -1) { acol = 128 + u * 8; dcol = (u / 8) * N; }
                    else if (a_step == -2) { acol = 128 + u * 8; dcol = 0; }
                    else { acol = 256 + (u % 8) * 8; dcol = (u / 8) * N; }
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm + dcol),
                        "r"(tm + acol), "l"(bd + (uint64_t)(b_mn ? (u % 8) * 16 : (u % 8) * 2)), "r"(idesc), "r"(1));
                }
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) *cycles = (t1 - t0);
        if (tid == 0) mbar_arrive(&done);
    }
    fence_before_sync();
    __syncthreads();
    if (tid < 32) tmem_dealloc<512>(tm);
}

extern "C" double umma_bench2(int N, int iters, int b_mn, int a_step, int nblocks, int nthreads) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(bench2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 32768);
    bench2_kernel<<<nblocks, nthreads, 65536 + 32768>>>(N, iters, b_mn, a_step, d);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h / iters;
}
