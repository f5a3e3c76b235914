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
__global__ void rows_bench_kernel(int mode, int swz, int N, int iters, int nacc, unsigned long long *cycles,
                                  int aoff, int walk) {
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
        const uint32_t idesc = idesc_bf16(128, N, mode == 1, mode == 1);
        uint64_t ad, bd;
        if (mode == 0) {
            ad = desc(sa + (uint32_t)aoff, 16, 8 * rowb, swz);
            bd = desc(sb, 16, 8 * rowb, swz);
        } else if (mode == 2) {   // B K-major without swizzle (the packed-weight image)
            ad = desc(sa + (uint32_t)aoff, 16, 8 * rowb, swz);
            bd = smem_desc(sb, (uint32_t)N * 16u, 128u);
        } else {
            ad = desc(sa + (uint32_t)aoff, 24 * 4 * rowb, 8 * rowb, swz);
            bd = desc(sb, 4 * rowb, 8 * rowb, swz);
        }
        const uint32_t kadv = mode != 1 ? 2u : (16u * rowb) >> 4;   // descriptor units (16 B)
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; it += 8) {
            if (elect_one()) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t dcol = tm + (uint32_t)((u % nacc) * N);
                    const uint64_t o = (uint64_t)((u & 1) * kadv);
                    // walk: every MMA starts `walk` bytes further (a moving tap window)
                    const uint64_t w = (uint64_t)(((u * walk) & 8191) >> 4);
                    const uint64_t ob = mode == 2 ? (uint64_t)((u & 1) * 2u * (uint32_t)N) : o;
                    mma_bf16_ss(dcol, ad + o + w, bd + ob, idesc, 1);
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

extern "C" double rows_bench(int mode, int swz, int N, int iters, int nacc, int nblocks, int aoff, int walk) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int smem = 98304 + 1024;
    cudaFuncSetAttribute(rows_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rows_bench_kernel<<<nblocks, 128, smem>>>(mode, swz, N, iters, nacc, d, aoff, walk);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h / iters;
}


namespace capsconv {
__device__ __forceinline__ void rows_probe_mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
}
// ---------------------------------------------------------------------------
// Synchronisation costs (one CTA per SM, globaltimer-free: clock64 of warp 0):
//  mode 0: `iters` tcgen05.commit -> mbarrier arrive, each waited by the same
//          warp (round trip commit -> phase flip -> try_wait returns)
//  mode 1: `iters` commits back to back (issue cost), then one wait
//  mode 2: producer/consumer ping-pong between warp 0 and warp 1 through two
//          mbarriers with plain arrives (round trip / 2 = one hand-off)
__global__ void sync_bench_kernel(int mode, int iters, unsigned long long *cycles) {
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32;
    if (warp == 0) tmem_alloc<32>(&tmem_base);
    if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_fence_init(); }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    unsigned long long t0 = clock64();
    if (mode == 0 && warp == 0) {
        for (int i = 0; i < iters; ++i) {
            if (elect_one()) mma_commit(&bar[0]);
            __syncwarp();
            mbar_wait(&bar[0], (uint32_t)(i & 1));
        }
    } else if (mode == 1 && warp == 0) {
        for (int i = 0; i < iters; ++i) {
            if (elect_one()) mma_commit(&bar[i & 1]);
            __syncwarp();
        }
        mbar_wait(&bar[(iters - 1) & 1], (uint32_t)(((iters - 1) >> 1) & 1));
    } else if (mode == 2) {
        if (warp == 0) {
            for (int i = 0; i < iters; ++i) {
                if (tid == 0) mbar_arrive(&bar[0]);
                mbar_wait(&bar[1], (uint32_t)(i & 1));
            }
        } else if (warp == 1) {
            for (int i = 0; i < iters; ++i) {
                mbar_wait(&bar[0], (uint32_t)(i & 1));
                if (tid == 32) mbar_arrive(&bar[1]);
            }
        }
    }
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) *cycles = t1 - t0;
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<32>(tmem_base);
}

extern "C" double sync_bench(int mode, int iters, int nblocks) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    sync_bench_kernel<<<nblocks, 64>>>(mode, iters, d);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h / iters;
}

__global__ void tile_bench_kernel(int N, int tiles, int per, int nslot, int ovw, int com, unsigned long long *cycles,
                                  int bmode) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[8];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    for (int i = tid; i < 98304 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    if (tid < 32) tmem_alloc<512>(&tmem_base);
    if (tid == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); mbar_fence_init(); }
    fence_proxy_async_smem();
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    if (tid < 32) {
        const uint32_t sa = (smem_u32(smem) + 1023u) & ~1023u, sb = sa + 49152;
        const uint32_t idesc = idesc_bf16(128, N, 0, 0);
        const uint64_t ad = desc(sa, 16, 512, 64);
        // bmode 0: one B (no swizzle); 1: three B slices in turn (no swizzle);
        // 2: one B (SW64 K-major); 3: three SW64 slices in turn
        const uint64_t bd = (bmode & 2) ? desc(sb, 16, 512, 64) : smem_desc(sb, (uint32_t)N * 16u, 128u);
        const uint32_t bslice = (bmode & 2) ? ((uint32_t)N * 64u) >> 4 : ((uint32_t)N * 64u) >> 4;
        unsigned long long t0 = clock64();
        const int pair = bmode >= 4;
        for (int t = 0; t < tiles; t += pair ? 2 : 1) {
            const uint32_t d = tm + (uint32_t)((t % nslot) * N);
            if (pair) {   // two independent accumulator chains interleaved
                const uint32_t d2 = tm + (uint32_t)(((t + 1) % nslot) * N);
                for (int u = 0; u < per; ++u) {
                    const uint64_t o = (uint64_t)((u & 1) * 2u);
                    capsconv::rows_probe_mma_elect(d, ad + o + (uint64_t)(u * 16), bd + (uint64_t)((u & 1) * 2u * N), idesc,
                                                   (ovw && u == 0) ? 0u : 1u);
                    capsconv::rows_probe_mma_elect(d2, ad + o + (uint64_t)(u * 16 + 32), bd + (uint64_t)((u & 1) * 2u * N),
                                                   idesc, (ovw && u == 0) ? 0u : 1u);
                }
                if (com) {
                    if (elect_one()) { mma_commit(&bar[t % 8]); mma_commit(&bar[(t + 1) % 8]); }
                    __syncwarp();
                }
                continue;
            }
            for (int u = 0; u < per; ++u) {
                const uint64_t o = (uint64_t)((u & 1) * 2u);
                const uint64_t bo = (bmode & 2) ? (uint64_t)((u & 1) * 2u) : (uint64_t)((u & 1) * 2u * N);
                const uint64_t bs = (bmode & 1) ? (uint64_t)((u % 3) * bslice) : 0ull;
                capsconv::rows_probe_mma_elect(d, ad + o + (uint64_t)(u * 16), bd + bo + bs, idesc,
                                               (ovw && u == 0) ? 0u : 1u);
            }
            if (com) { if (elect_one()) mma_commit(&bar[t % 8]); __syncwarp(); }
        }
        if (elect_one()) mma_commit(&bar[0]);
        __syncwarp();
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && tid == 0) *cycles = (t1 - t0);
    }
    fence_before_sync();
    __syncthreads();
    if (tid < 32) tmem_dealloc<512>(tm);
}

extern "C" double tile_bench(int N, int tiles, int per, int nslot, int ovw, int com, int bmode) {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    const int smem = 98304 + 1024;
    cudaFuncSetAttribute(tile_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_bench_kernel<<<148, 128, smem>>>(N, tiles, per, nslot, ovw, com, d, bmode);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h / ((double)tiles * per);
}

// TMEM read bandwidth: nwarps warps (warp w reads lane quarter w % 4), each
// `iters` times tcgen05.ld.32x32b.x32 (4 KB per warp) + wait::ld.
__global__ void tmem_bw_kernel(int iters, int ncol, unsigned long long *cycles, float *sink) {
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid / 32;
    if (warp == 0) tmem_alloc<512>(&tmem_base);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tm = tmem_base;
    float acc = 0.f;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r[32];
        const uint32_t a = tm + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((i * 32) % ncol);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
            "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
              "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(a));
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) *cycles = t1 - t0;
    if (acc == 12345.f) sink[tid] = acc;
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" double tmem_bw(int nwarps, int iters) {
    unsigned long long *d;
    float *sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 4096);
    tmem_bw_kernel<<<148, nwarps * 32>>>(iters, 512, d, sink);
    unsigned long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(sink);
    if (e != cudaSuccess) return -1.0;
    return (double)nwarps * iters * 4096.0 / (double)h;   // bytes per cycle per SM
}

// ---------------------------------------------------------------------------
// MMA queue depth: the issuing warp alternates K back-to-back 128xNx16 MMAs
// (uniform operands, one warp, elect per MMA) with `spin` dependent uniform
// integer steps of bookkeeping.  cycles/iteration ~ max(K*t_mma, spin + issue)
// if the tensor pipe queues the MMAs, ~ K*t_mma + spin if the issuing warp
// waits for them.
__global__ void queue_bench_kernel(int N, int K, int spin, int iters, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_base;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
    if (warp == 0) tmem_alloc<512>(&tmem_base);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (warp == 0) {
        const uint32_t sa = (smem_u32(smem) + 1023u) & ~1023u, sb = sa + 32768;
        const uint64_t ad = desc(sa, 16, 512, 64);
        const uint64_t bd = desc(sb, 16, 512, 64);
        const uint32_t idesc = idesc_bf16(128, N, 0, 0);
        uint32_t x = (uint32_t)clock();
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < K; ++k) {
                asm volatile(
                    "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(0u),
                    "l"(ad + (uint64_t)((k & 1) * 2)), "l"(bd), "r"(idesc), "r"(1u));
            }
            for (int j = 0; j < spin; ++j) x = x * 1664525u + 1013904223u;   // dependent bookkeeping
        }
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[0] = (t1 - t0) / (unsigned long long)iters, out[1] = x;
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem_base);
}

extern "C" double queue_bench(int N, int K, int spin, int iters) {
    unsigned long long *d;
    cudaMalloc(&d, 16);
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(queue_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    queue_bench_kernel<<<148, 64, smem>>>(N, K, spin, iters, d);
    unsigned long long h[2] = {0, 0};
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1.0;
    return (double)h[0];
}
