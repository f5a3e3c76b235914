// rows_probe.cu -- test-only probe for the D1-outer ("rows") capsule layout.
//
// TMA stages row-major bf16 matrices (rows of E = 32 / 64 elements, 64 / 128
// bytes) into shared memory with SWIZZLE_64B / SWIZZLE_128B, and tcgen05.mma
// reads them in place, either
//   mode 0  K-major A and B; A starts `a_shift` rows into the staged buffer
//           (the forward / data-gradient tap shift: one pixel = D1 rows), or
//   mode 1  MN-major A and B; the MN atoms (E elements each) of A sit
//           `a_shift` rows apart and those of B `b_shift` rows apart, i.e.
//           every atom is the same staged buffer read at another k-row
//           offset (the kernel-gradient slot / column shifts).
// D (128 x N, fp32) is written to global memory for comparison with a
// float64 reference in tests/test_rows_probe_gpu.py.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>

#include "umma.cuh"

using namespace capsconv::umma;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool make_map(CUtensorMap *m, const void *g, int rows, int E, int swz) {
    cuuint64_t dims[2] = {(cuuint64_t)E, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)E * 2};
    cuuint32_t box[2] = {(cuuint32_t)E, 64u};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle sw = swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(g), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap *m, int c0, int c1, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}

__host__ __device__ constexpr uint64_t layout_code(int swz) {
    return swz == 128 ? 2ull : swz == 64 ? 4ull : swz == 32 ? 6ull : 0ull;
}

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int swz) {
    return smem_desc(addr, lbo, sbo) | (layout_code(swz) << 61);
}

struct Args {
    CUtensorMap tmA, tmB;
    int RA, RB, E, swz, mode, N, K, a_shift, b_shift, a_k0;
    float *D;
};

__global__ void __launch_bounds__(128, 1) rows_probe_kernel(const __grid_constant__ Args P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar_tma, bar_mma;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const uint32_t rowb = (uint32_t)P.E * 2;
    const uint32_t sA = (smem_u32(smem) + 1023u) & ~1023u;
    const uint32_t sB = sA + (((uint32_t)P.RA * rowb + 1023u) & ~1023u);
    if (warp == 0) tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        mbar_init(&bar_tma, 1);
        mbar_init(&bar_mma, 1);
        mbar_fence_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar_tma, (uint32_t)(P.RA + P.RB) * rowb);
        for (int r = 0; r < P.RA; r += 64) tma2d(sA + (uint32_t)r * rowb, &P.tmA, 0, r, smem_u32(&bar_tma));
        for (int r = 0; r < P.RB; r += 64) tma2d(sB + (uint32_t)r * rowb, &P.tmB, 0, r, smem_u32(&bar_tma));
    }
    mbar_wait(&bar_tma, 0);
    const uint32_t tm = tmem_base;
    if (warp == 0) {
        const int mn = P.mode == 1;
        const uint32_t idesc = idesc_bf16(128, P.N, mn, mn);
        if (elect_one()) {
            const int nk = mn ? P.K / 16 : P.E / 16;
            for (int ks = 0; ks < nk; ++ks) {
                uint64_t ad, bd;
                if (!mn) {
                    ad = desc(sA + (uint32_t)P.a_shift * rowb + ks * 32, 16, 8 * rowb, P.swz);
                    bd = desc(sB + ks * 32, 16, 8 * rowb, P.swz);
                } else {
                    ad = desc(sA + (uint32_t)(P.a_k0 + 16 * ks) * rowb, (uint32_t)P.a_shift * rowb, 8 * rowb, P.swz);
                    bd = desc(sB + (uint32_t)(16 * ks) * rowb, (uint32_t)P.b_shift * rowb, 8 * rowb, P.swz);
                }
                mma_bf16_ss(tm, ad, bd, idesc, ks > 0);
            }
            mma_commit(&bar_mma);
        }
        __syncwarp();
    }
    mbar_wait(&bar_mma, 0);
    fence_after_sync();
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < P.N; c0 += 8) {
        float v[8];
        tmem_ld8(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_wait_ld();
        for (int j = 0; j < 8 && c0 + j < P.N; ++j) P.D[row * P.N + c0 + j] = v[j];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tm);
}

// MMA-issue throughput with the rows-layout descriptors: `iters` SS MMAs of
// 128 x N x 16 (mode 0 K-major / mode 1 MN-major, swizzled), operands
// garbage; returns cycles per MMA measured by CTA 0.
__global__ void rows_bench_kernel(int mode, int swz, int N, int iters, int nacc, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    for (int i = tid; i < 98304 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    if (tid < 32) tmem_alloc<512>(&tmem_base);
    if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    if (tid < 32) {
        const uint32_t rowb = swz == 128 ? 128 : 64;
        const uint32_t sa = (smem_u32(smem) + 1023u) & ~1023u, sb = sa + 49152;
        const uint32_t idesc = idesc_bf16(128, N, mode, mode);
        uint64_t ad, bd;
        if (mode == 0) {
            ad = desc(sa, 16, 8 * rowb, swz);
            bd = desc(sb, 16, 8 * rowb, swz);
        } else {
            ad = desc(sa, 24 * 4 * rowb, 8 * rowb, swz);
            bd = desc(sb, 4 * rowb, 8 * rowb, swz);
        }
        const uint32_t kadv = mode == 0 ? 2u : (16u * rowb) >> 4;   // descriptor units (16 B)
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; it += 8) {
            if (elect_one()) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t dcol = tm + (uint32_t)((u % nacc) * N);
                    const uint64_t o = (uint64_t)((u & 1) * kadv);
                    mma_bf16_ss(dcol, ad + o, bd + o, idesc, 1);
                }
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) *cycles = t1 - t0;
    }
    fence_before_sync();
    __syncthreads();
    if (tid < 32) tmem_dealloc<512>(tm);
}

}  // namespace

extern "C" int rows_probe(const void *A, const void *B, float *D, int RA, int RB, int E, int swz, int mode, int N,
                          int K, int a_shift, int b_shift, int a_k0) {
    if (!encode_fn()) return -1;
    Args P;
    if (!make_map(&P.tmA, A, RA, E, swz) || !make_map(&P.tmB, B, RB, E, swz)) return -2;
    P.RA = RA; P.RB = RB; P.E = E; P.swz = swz; P.mode = mode; P.N = N; P.K = K;
    P.a_shift = a_shift; P.b_shift = b_shift; P.a_k0 = a_k0; P.D = D;
    const size_t smem = (size_t)((RA * E * 2 + 1023) / 1024 * 1024) + (size_t)RB * E * 2 + 2048;
    cudaFuncSetAttribute(rows_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rows_probe_kernel<<<1, 128, smem>>>(P);
    return (int)cudaDeviceSynchronize();
}

extern "C" double rows_bench(int mode, int swz, int N, int iters, int nacc, int nblocks) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int smem = 98304 + 1024;
    cudaFuncSetAttribute(rows_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rows_bench_kernel<<<nblocks, 128, smem>>>(mode, swz, N, iters, nacc, d);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h / iters;
}
