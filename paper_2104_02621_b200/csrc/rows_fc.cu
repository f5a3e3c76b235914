// rows_fc.cu -- the fully-connected capsule layer (the full-extent
// convolution KH = H, KW = W of reading R18) for the D1-outer
// ("rows") layout: three TMA-fed tcgen05 GEMMs.
//
// With I stored [B][P = H*W][D1][E = C*D2] (rows.cuh) the three passes are
// plain GEMMs whose operands TMA writes directly in the swizzled UMMA layouts:
//   fwd   O[(b,d1), (c',d3)]       = sum_{(p,c,d2)} I[b,p,d1,(c,d2)] K[p,c,c',d2,d3]
//         A = I rows (b, d1) K-major (one 128-byte chunk of (c,d2) per k-chunk),
//         B = K packed K-major; split-K, fp32 partials, fixed-order finalize.
//   dI    dI[(b,d1), (p,c,d2)]     = sum_{(c',d3)} dO[b,d1,(c',d3)] K[p,c,c',d2,d3]
//         A = dO rows K-major (K = Cout*D3, TMA zero fill to the k-step), B = K^T
//         packed; one k-block, N = 256 tiles, bf16 through swizzled staging + TMA stores.
//   dK    dK[(p,c,d2), (c',d3)]    = sum_{(b,d1)} I[b,p,d1,(c,d2)] dO[b,d1,(c',d3)]
//         A = I^T MN-major (two 64-element atoms per tile), B = dO MN-major;
//         split-K over images, fp32 partials, fixed-order finalize into dK.
// Roles (320 threads): warp 0 TMA, warp 1 MMA (TMEM owner), warps 2-9 epilogue (two per TMEM
// lane quarter, each taking half of the columns).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "internal.h"
#include "rows.cuh"
#include "umma.cuh"

namespace capsconv {
using namespace umma;

namespace {

constexpr int kFcEpw = 2;                      // epilogue warps per TMEM lane quarter
constexpr int kFcThreads = 64 + 128 * kFcEpw;  // warp 0 TMA, warp 1 MMA, then the epilogue warps
constexpr uint32_t kFcSmemLimit = 227 * 1024;

struct RowsFc {
    alignas(64) CUtensorMap tmA;   // fwd/dK: I as (E, 4, P, B); dI: dO as (EO, B*4)
    alignas(64) CUtensorMap tmB;   // dK: dO as (EO, B*4)
    alignas(64) CUtensorMap tmO;   // dI: dI as (E, 4, P, B), SWIZZLE_128B boxes (64, 4, 1, 8) for the stores
    int mode;                      // 0 fwd, 1 dI, 2 dK
    int B, P, E, EO, Cout, C;
    int N;                         // MMA N
    int nmt, nnt, ksplit, n_items;
    int kst;                       // K stages per M tile (whole K)
    int kps;                       // k-steps per stage
    int cps;                       // fwd: 64-element chunks per stage
    uint32_t a_bytes, b_bytes, stage_bytes;
    int nstg, nacc;
    const uint8_t *wpack;          // fwd: [chunk][N rows][128 B swizzled]; dI: [n][128 B swizzled]
    float *part;                   // fwd / dK: [ksplit][M][N] fp32 partials
    __nv_bfloat16 *out;            // dI output
    uint32_t epi_off;              // dI: per-warp store staging (2 x 4 KB per epilogue warp) from stg0
    int dst_direct;                // dI: 1 coalesced 16-byte stores from the staging, 0 TMA box stores
    uint32_t smem_bytes;
};

__device__ __forceinline__ void fc_decode(const RowsFc &P, int item, int &mt, int &nt, int &ks) {
    ks = item % P.ksplit;
    const int r = item / P.ksplit;
    nt = r % P.nnt;
    mt = r / P.nnt;
}

__global__ void __launch_bounds__(kFcThreads, 1) rows_fc_kernel(const __grid_constant__ RowsFc P) {
    // no early PDL trigger: the packed weights (and split partials) in the
    // workspace are read until the end
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *full = bars, *empty = bars + 8, *accf = bars + 16, *acce = bars + 18;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + 512);
    const uint32_t stg0 = (smem_u32(smem_raw) + 1024u + 1023u) & ~1023u;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P.nstg; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(accf + i, 1);
            mbar_init(acce + i, 4 * kFcEpw);
        }
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc_dyn(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (*tmem_slot != 0u) __trap();
    pdl_wait();
    const int nkb = P.kst / P.ksplit;   // stages per item

    if (warp == 0) {
        // ------------------------------------------------------------ TMA
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmB)) : "memory");
            int sb = 0;
            uint32_t ph = 0;
            for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
                int mt, nt, ks;
                fc_decode(P, item, mt, nt, ks);
                for (int s = ks * nkb; s < (ks + 1) * nkb; ++s) {
                    mbar_wait(empty + sb, ph ^ 1);
                    const uint32_t stg = stg0 + (uint32_t)sb * P.stage_bytes;
                    const uint32_t mb = smem_u32(full + sb);
                    mbar_arrive_expect_tx(full + sb, P.a_bytes + P.b_bytes);
                    if (P.mode == 0) {
                        // chunks c = s*cps .. : p = c / (E/64), element offset (c % (E/64)) * 64
                        const int cpp = P.E / 64;
                        for (int j = 0; j < P.cps; ++j) {
                            const int c = s * P.cps + j;
                            rows::tma_load4d_rows(stg + (uint32_t)j * 16384u, &P.tmA, (c % cpp) * 64, 0, c / cpp,
                                                  32 * mt, mb);
                        }
                        bulk_g2s_u32(stg + P.a_bytes, P.wpack + (size_t)s * P.b_bytes, P.b_bytes, full + sb);
                    } else if (P.mode == 1) {
                        // dO rows (b, d1): two 32-element boxes cover K (zero fill past EO)
                        rows::tma_load2d(stg, &P.tmA, 0, 128 * mt, mb);
                        rows::tma_load2d(stg + 8192u, &P.tmA, 32, 128 * mt, mb);
                        bulk_g2s_u32(stg + P.a_bytes, P.wpack + (size_t)nt * P.b_bytes, P.b_bytes, full + sb);
                    } else {
                        // I^T atoms (p = mt / (E/128), elements e0, e0 + 64) over 32 images; dO rows
                        const int tpp = P.E / 128;
                        const int p = mt / tpp, e0 = (mt % tpp) * 128;
                        rows::tma_load4d_rows(stg, &P.tmA, e0, 0, p, 32 * s, mb);
                        rows::tma_load4d_rows(stg + 16384u, &P.tmA, e0 + 64, 0, p, 32 * s, mb);
                        rows::tma_load2d(stg + P.a_bytes, &P.tmB, 0, 128 * s, mb);
                    }
                    if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA
        int sb = 0, slot = 0;
        uint32_t ph = 0, aph = 0;
        const uint32_t idesc = P.mode == 2 ? idesc_bf16(128, P.N, 1, 1) : idesc_bf16(128, P.N, 0, 0);
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            mbar_wait(acce + slot, aph ^ 1);
            fence_after_sync();
            const uint32_t d = (uint32_t)slot * 256u;
            for (int s = 0; s < nkb; ++s) {
                mbar_wait(full + sb, ph);
                fence_after_sync();
                const uint32_t stg = stg0 + (uint32_t)sb * P.stage_bytes;
                if (P.mode == 0) {
                    for (int j = 0; j < P.cps; ++j)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t ad = rows::sdesc(stg + (uint32_t)j * 16384u + kk * 32u, 16u, 1024u, 128);
                            const uint64_t bd = rows::sdesc(stg + P.a_bytes + (uint32_t)j * (uint32_t)P.N * 128u + kk * 32u,
                                                            16u, 1024u, 128);
                            rows::mma_ss_elect(d, ad, bd, idesc, (s > 0 || j > 0 || kk > 0) ? 1u : 0u);
                        }
                } else if (P.mode == 1) {
                    for (int kk = 0; kk < P.kps; ++kk) {
                        // A: 64-byte swizzled rows, k-steps 0,1 in box 0 and 2,3 in box 1
                        const uint64_t ad =
                            rows::sdesc(stg + (uint32_t)(kk >> 1) * 8192u + (uint32_t)(kk & 1) * 32u, 16u, 512u, 64);
                        const uint64_t bd = rows::sdesc(stg + P.a_bytes + (uint32_t)kk * 32u, 16u, 1024u, 128);
                        rows::mma_ss_elect(d, ad, bd, idesc, kk > 0 ? 1u : 0u);
                    }
                } else {
                    for (int kk = 0; kk < P.kps; ++kk) {
                        // MN-major: A atoms 16 KB apart, 16 k-rows (2 KB) per k-step
                        const uint64_t ad = rows::sdesc(stg + (uint32_t)kk * 2048u, 16384u, 1024u, 128);
                        const uint64_t bd = rows::sdesc(stg + P.a_bytes + (uint32_t)kk * 2048u, 16384u, 1024u, 128);
                        rows::mma_ss_elect(d, ad, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
                    }
                }
                if (elect_one()) mma_commit(empty + sb);
                __syncwarp();
                if (++sb == P.nstg) { sb = 0; ph ^= 1; }
            }
            if (elect_one()) mma_commit(accf + slot);
            __syncwarp();
            if (++slot == P.nacc) { slot = 0; aph ^= 1; }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3, half = (warp - 2) >> 2;   // lane quarter; column part (of kFcEpw)
        const int row = q * 32 + lane;
        int slot = 0, ebi = 0;
        uint32_t aph = 0;
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            int mt, nt, ks;
            fc_decode(P, item, mt, nt, ks);
            mbar_wait(accf + slot, aph);
            fence_after_sync();
            const uint32_t tb = ((uint32_t)(q * 32) << 16) + (uint32_t)slot * 256u;
            if (P.mode == 1) {
                // rows (b, d1) of dI, 8 images x 4 d1 per warp; columns (p, c, d2).  Each
                // 64-column chunk (one pixel p, 64 elements of E) is converted to bf16,
                // written to a per-warp SWIZZLE_128B staging box (row = lane, 16-byte
                // chunk j at j ^ (lane & 7): conflict-free) and stored by one TMA
                // (64, 4, 1, 8) box; two staging buffers alternate.
                const uint32_t ebuf = stg0 + P.epi_off + (uint32_t)(warp - 2) * 8192u;
                const int b0 = 32 * mt + 8 * q;
                for (int c0 = half * (P.N / kFcEpw); c0 < (half + 1) * (P.N / kFcEpw); c0 += 64) {
                    float v[64];
                    rows::tmem_ld32(tb + (uint32_t)c0, *reinterpret_cast<float(*)[32]>(v));
                    rows::tmem_ld32(tb + (uint32_t)c0 + 32u, *reinterpret_cast<float(*)[32]>(v + 32));
                    tmem_wait_ld();
                    const uint32_t buf = ebuf + (uint32_t)(ebi & 1) * 4096u;
                    if (lane == 0 && !P.dst_direct) rows::bulk_wait_read<1>();
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        uint32_t w[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * j + 2 * c], v[8 * j + 2 * c + 1]);
                            w[c] = *reinterpret_cast<uint32_t *>(&h);
                        }
                        const uint32_t a = buf + (uint32_t)lane * 128u + (uint32_t)((j ^ (lane & 7)) * 16);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(w[0]), "r"(w[1]),
                                     "r"(w[2]), "r"(w[3])
                                     : "memory");
                    }
                    const int n = nt * P.N + c0, p = n / P.E, e = n - p * P.E;
                    if (P.dst_direct) {
                        // coalesced 16-byte stores: 8 lanes write one 128-byte capsule-row piece
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int k = i * 32 + lane, r = k >> 3, j = k & 7;
                            const int b = b0 + (r >> 2);
                            if (b < P.B) {
                                const uint4 x = ld_shared_v4(buf + (uint32_t)r * 128u + (uint32_t)((j ^ (r & 7)) * 16));
                                *reinterpret_cast<uint4 *>(P.out + ((((size_t)b * P.P + p) * 4 + (r & 3)) * (size_t)P.E + e +
                                                                    (size_t)j * 8)) = x;
                            }
                        }
                        __syncwarp();
                    } else {
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0 && b0 < P.B) {
                            rows::tma_store4d(&P.tmO, buf, e, 0, p, b0);
                            rows::bulk_commit();
                        }
                    }
                    ++ebi;
                }
            } else {
                // fp32 partial rows [ks][M][N]
                float *dst = P.part + ((size_t)ks * P.nmt * 128 + (size_t)mt * 128 + row) * P.N;
                for (int c0 = 16 * half; c0 < P.N; c0 += 16 * kFcEpw) {
                    float v[16];
                    tmem_ld16(tb + (uint32_t)c0, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        reinterpret_cast<float4 *>(dst + c0)[g] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                }
            }
            fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(acce + slot);
            if (++slot == P.nacc) { slot = 0; aph ^= 1; }
        }
        if (P.mode == 1 && lane == 0 && !P.dst_direct) rows::bulk_wait_all();
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_dealloc_dyn(0u, 512);
}

// fwd: O[r][n] = bf16(sum_k part[k][r][n]), n < EO (rows r = (b, d1) < 4B)
__global__ void fc_fin_fwd(const float *__restrict__ part, __nv_bfloat16 *__restrict__ O, int rows, int N, int EO,
                           int ksplit, long long mstride) {
    pdl_wait();   // no early trigger: the partials in the workspace are read to the end
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)rows * EO) return;
    const int r = (int)(i / EO), n = (int)(i - (long long)r * EO);
    float acc = 0.f;
    for (int k = 0; k < ksplit; ++k) acc += part[(size_t)k * mstride + (size_t)r * N + n];
    O[i] = __float2bfloat16_rn(acc);
}

// dK: rows m = (p, c, d2) over E per pixel, columns n = (c', d3) < EO
__global__ void fc_fin_dk(const float *__restrict__ part, float *__restrict__ dK, int M, int N, int C, int Cout,
                          int ksplit, long long mstride) {
    pdl_wait();   // no early trigger: the partials in the workspace are read to the end
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int EO = 4 * Cout;
    if (i >= (long long)M * EO) return;
    const int m = (int)(i / EO), n = (int)(i - (long long)m * EO);
    float acc = 0.f;
    for (int k = 0; k < ksplit; ++k) acc += part[(size_t)k * mstride + (size_t)m * N + n];
    const int E = 4 * C;
    const int p = m / E, e = m - p * E, c = e >> 2, d2 = e & 3, co = n >> 2, d3 = n & 3;
    dK[((((size_t)p * C + c) * Cout + co) * 4 + d2) * 4 + d3] = acc;
}

// Packed weight images, SWIZZLE_128B K-major rows of 64 bf16 (128 B):
//   fwd: chunk c (p = c / (E/64), (c,d2) block (c % (E/64))*64), rows n < N = (c', d3)
//   dI : rows n = (p, c, d2) < P*E, k = (c', d3) < 64 (zero past EO)
__device__ __forceinline__ void fc_pack_unit(const __nv_bfloat16 *__restrict__ K, uint8_t *__restrict__ dst, int mode,
                                             int C, int Cout, int N, long long g) {
    const int E = 4 * C, EO = 4 * Cout;
    const long long rowi = g / 8;            // 8 sixteen-byte units per 128-byte row
    const int unit = (int)(g - rowi * 8);    // physical unit in the row
    int n, p, ebase;
    if (mode == 0) {
        const int cpp = E / 64;
        const long long c = rowi / N;
        n = (int)(rowi - c * N);
        p = (int)(c / cpp);
        ebase = (int)(c % cpp) * 64;
    } else {
        n = (int)rowi;
        p = 0;
        ebase = 0;
    }
    const int lunit = unit ^ (int)(rowi & 7);   // logical 16-byte chunk (Swizzle<3,4,3>)
    __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int k = lunit * 8 + e;
        float x = 0.f;
        if (mode == 0) {
            const int ee = ebase + k, c = ee >> 2, d2 = ee & 3, co = n >> 2, d3 = n & 3;
            if (n < EO) x = __bfloat162float(K[((((size_t)p * C + c) * Cout + co) * 4 + d2) * 4 + d3]);
        } else {
            const int pp = n / E, ee = n - pp * E, c = ee >> 2, d2 = ee & 3, co = k >> 2, d3 = k & 3;
            if (k < EO) x = __bfloat162float(K[((((size_t)pp * C + c) * Cout + co) * 4 + d2) * 4 + d3]);
        }
        v[e] = __float2bfloat16_rn(x);
    }
    uint4 w;
    memcpy(&w, v, 16);
    reinterpret_cast<uint4 *>(dst)[g] = w;
}

// Runs alongside the previous kernel's tail (see rc_pack_kernel): reads only K,
// writes only the workspace, and waits for the previous grid before it exits.
__global__ void __launch_bounds__(64) fc_pack(const __nv_bfloat16 *__restrict__ K, uint8_t *__restrict__ dst, int mode,
                                              int P, int C, int Cout, int N, long long total16) {
    (void)P;
    pdl_launch_dependents();
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < total16) fc_pack_unit(K, dst, mode, C, Cout, N, g);
    pdl_wait();
}

struct FcPlan {
    bool ok = false;
    RowsFc P;
    size_t wpack_bytes = 0, part_bytes = 0;
};

FcPlan make_fc_plan(const Problem &p, int mode) {
    FcPlan pl;
    RowsFc &P = pl.P;
    memset(&P, 0, sizeof(P));
    if (p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4 || p.pad != 0) return pl;
    if (p.KH != p.H || p.KW != p.W || p.s != 1) return pl;   // full extent: one output pixel
    const int E = 4 * (int)p.C, EO = 4 * (int)p.Cout;
    if (E % 128 != 0 || EO > 64 || (long long)p.B * 4 > (1 << 24) || p.H * p.W > 256) return pl;
    P.mode = mode;
    P.B = (int)p.B; P.P = (int)(p.H * p.W); P.E = E; P.EO = EO; P.C = (int)p.C; P.Cout = (int)p.Cout;
    P.nmt = (P.B + 31) / 32;
    const int nsm = device_info().num_sms;
    if (mode == 0) {
        P.N = (EO + 15) / 16 * 16;
        P.cps = 2;
        const int nchunks = P.P * E / 64;
        if (nchunks % P.cps) return pl;
        P.kst = nchunks / P.cps;
        P.kps = 4 * P.cps;
        P.a_bytes = (uint32_t)P.cps * 16384u;
        P.b_bytes = (uint32_t)P.cps * (uint32_t)P.N * 128u;
        P.nnt = 1;
        P.ksplit = 1;
        for (int k = 1; k <= P.kst; ++k)
            if (P.kst % k == 0 && P.nmt * k <= nsm) P.ksplit = k;
        pl.wpack_bytes = (size_t)nchunks * P.N * 128;
    } else if (mode == 1) {
        P.N = 256;
        if ((P.P * E) % 256) return pl;
        P.nnt = P.P * E / 256;
        P.kst = 1;
        P.kps = (EO + 15) / 16;
        P.a_bytes = 2u * 8192u;
        P.b_bytes = 256u * 128u;
        P.ksplit = 1;
        pl.wpack_bytes = (size_t)P.P * E * 128;
    } else {
        P.N = (EO + 15) / 16 * 16;
        P.nmt = P.P * E / 128;     // M tiles over (p, c, d2)
        P.nnt = 1;
        if (P.B % 32) return pl;
        P.kst = P.B / 32;           // stages of 32 images (128 k-rows)
        P.kps = 8;
        P.a_bytes = 2u * 16384u;
        P.b_bytes = 128u * 128u;
        P.ksplit = 1;
        for (int k = 1; k <= P.kst; ++k)
            if (P.kst % k == 0 && P.nmt * k <= 2 * nsm) P.ksplit = k;
    }
    P.stage_bytes = (P.a_bytes + P.b_bytes + 1023u) & ~1023u;
    const uint32_t epi = mode == 1 ? 4u * kFcEpw * 8192u : 0u;
    P.nstg = std::min(8, (int)((kFcSmemLimit - 2048u - epi) / P.stage_bytes));
    if (P.nstg < 2) return pl;
    P.nacc = 2;
    P.n_items = P.nmt * P.nnt * P.ksplit;
    P.epi_off = (uint32_t)P.nstg * P.stage_bytes;
    P.dst_direct = 1;
    if (kProbes && probe_env("CAPSCONV_FC_TMASTORE")) P.dst_direct = 0;
    P.smem_bytes = 2048u + P.epi_off + epi;
    if (mode != 1) pl.part_bytes = (size_t)P.ksplit * P.nmt * 128 * P.N * 4;
    pl.ok = true;
    return pl;
}

std::shared_ptr<const FcPlan> cached_fc_plan(const Problem &p, int mode) {
    static std::mutex mu;
    static std::vector<std::pair<std::vector<int64_t>, std::shared_ptr<const FcPlan>>> cache;
    const DeviceInfo &di = device_info();
    std::vector<int64_t> k = {mode, di.device, di.num_sms, p.dt, p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW,
                              p.D1, p.D2, p.D3, p.s, p.pad};
    std::lock_guard<std::mutex> lock(mu);
    for (auto &kv : cache)
        if (kv.first == k) return kv.second;
    if (cache.size() > 256) cache.clear();
    cache.emplace_back(k, std::make_shared<const FcPlan>(make_fc_plan(p, mode)));
    return cache.back().second;
}

int fc_mode(capsconv_op_t op) { return op == CAPSCONV_OP_FWD ? 0 : op == CAPSCONV_OP_BWD_DATA ? 1 : 2; }

}  // namespace

bool rows_fc_supported(capsconv_op_t op, const Problem &p) { return cached_fc_plan(p, fc_mode(op))->ok; }

size_t rows_fc_workspace_bytes(capsconv_op_t op, const Problem &p) {
    std::shared_ptr<const FcPlan> pl = cached_fc_plan(p, fc_mode(op));
    if (!pl->ok) return 0;
    return ((pl->wpack_bytes + 255) & ~(size_t)255) + ((pl->part_bytes + 255) & ~(size_t)255);
}

cudaError_t rows_fc_run(capsconv_op_t op, const Problem &p, const void *a, const void *b, void *out, void *ws,
                        size_t ws_bytes, cudaStream_t st) {
    const int mode = fc_mode(op);
    FcPlan pl = *cached_fc_plan(p, mode);
    if (!pl.ok || ws_bytes < rows_fc_workspace_bytes(op, p)) return cudaErrorNotSupported;
    RowsFc &P = pl.P;
    uint8_t *w8 = static_cast<uint8_t *>(ws);
    const size_t wb = (pl.wpack_bytes + 255) & ~(size_t)255;
    P.wpack = w8;
    P.part = reinterpret_cast<float *>(w8 + wb);
    cudaError_t e = cudaSuccess;
    if (mode == 0) {
        // a = I, b = K
        if (!rows::make_rows_map4(&P.tmA, a, P.B, P.P, P.E, 64, 1, 32)) return cudaErrorInvalidValue;
    } else if (mode == 1) {
        // a = dO, b = K
        if (!rows::make_rows_map2(&P.tmA, a, (int64_t)P.B * 4, P.EO, 32, 128, 64) ||
            !rows::make_rows_map4(&P.tmO, out, P.B, P.P, P.E, 64, 1, 8))
            return cudaErrorInvalidValue;
        P.out = static_cast<__nv_bfloat16 *>(out);
    } else {
        // a = I, b = dO
        if (!rows::make_rows_map4(&P.tmA, a, P.B, P.P, P.E, 64, 1, 32) ||
            !rows::make_rows_map2(&P.tmB, b, (int64_t)P.B * 4, P.EO, 64, 128, 128))
            return cudaErrorInvalidValue;
    }
    if (mode != 2 && !probe_skip_pack()) {
        const long long total16 = (long long)pl.wpack_bytes / 16;
        e = launch_pack(fc_pack, dim3((unsigned)((total16 + 63) / 64)), dim3(64), 0, st,
                     static_cast<const __nv_bfloat16 *>(b), w8, mode, P.P, P.C, P.Cout, P.N, total16);
        if (e != cudaSuccess) return e;
        note_launches(1);
    }
    e = smem_optin(reinterpret_cast<const void *>(rows_fc_kernel), (int)P.smem_bytes);
    if (e != cudaSuccess) return e;
    const int grid = std::min(P.n_items, device_info().num_sms);
    e = launch_k(rows_fc_kernel, dim3(grid), dim3(kFcThreads), P.smem_bytes, st, P);
    if (e != cudaSuccess) return e;
    note_launches(1);
    const long long mstride = (long long)P.nmt * 128 * P.N;
    if (probe_skip_fin()) {
    } else if (mode == 0) {
        const long long n = (long long)P.B * 4 * P.EO;
        e = launch_k(fc_fin_fwd, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, static_cast<const float *>(P.part),
                     static_cast<__nv_bfloat16 *>(out), P.B * 4, P.N, P.EO, P.ksplit, mstride);
        note_launches(1);
    } else if (mode == 2) {
        const long long n = (long long)P.P * P.E * P.EO;
        e = launch_k(fc_fin_dk, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, static_cast<const float *>(P.part),
                     static_cast<float *>(out), P.P * P.E, P.N, P.C, P.Cout, P.ksplit, mstride);
        note_launches(1);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace capsconv
