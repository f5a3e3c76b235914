// fc_hmma.cu -- the fully-connected capsule layer (R18: a full-extent
// capsule convolution viewed as 1x1 over C = KH*KW*Cin channels) on warp-level
// mma.sync tensor-core instructions: forward, dI and dK.
//
// Why not tcgen05 here: the FC passes are streaming GEMMs (forward: M = B*4,
// K = 4*C = 8192, N = 4*Cout = 40; 40 flop/byte, HBM-bound at ~260 TFLOP/s,
// well inside the ~550 TFLOP/s legacy HMMA sustains on B200, tests/probe/
// hmma_probe.cu).  With the k index inside each 16-step permuted, a thread's
// whole m16n8k16 A fragment is 16 contiguous bytes of the capsule layout, so
// the operand needs no D1 repack, which is what bounds the tcgen05 path on
// this layer (producer repack and split-K bookkeeping).
//
//   O[b, c', d1, d3]  = sum_{c, d2}   I[b, c, d1, d2] * K[c, c', d2, d3]     rows (b, d1),  k (c, d2)
//   dI[b, c, d1, d2]  = sum_{c', d3}  dO[b, c', d1, d3] * K[c, c', d2, d3]   rows (b, d1),  k (c', d3)
//   dK[c, c', d2, d3] = sum_{b, d1}   I[b, c, d1, d2] * dO[b, c', d1, d3]    rows (c, d2),  k (b, d1)
//                                                            (Alg. 4, R18)
//
// fwd: CTA = (K split, 64 images); the CTA's I rows stream through a 4-stage
// cp.async ring, the K slice of the weights (prepacked in fragment order)
// sits in shared memory.  dI: CTA = (column block, 64 images), dO fragments
// in registers, weights of the column block in shared memory.  dK: CTA =
// (image slice, 64 channels), I and dO rows of 8 images per stage by 1-D bulk
// copies on an mbarrier ring, capsule-column fragments built with PRMT.
// Split partials are summed in a fixed order by the finalize kernels
// (deterministic).  DESIGN.md 5.3c has the measurements.
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "umma.cuh"

namespace capsconv {
namespace {

constexpr int kFcWarps = 8;
constexpr int kFcMt = 2;          // m-tiles (16 rows) per warp
constexpr int kFcMaxNt = 8;       // n-tiles of 8 columns (N <= 64)

// I stream of the forward kernel: a ring of kFwdStages stages, each kFwdKs
// k-steps of the CTA's 64 images (image row = kFwdKs * 4 channels * 32 B,
// contiguous in I); a warp's fragment read (4 images x 128 B) is 4 wavefronts.
constexpr int kFwdStages = 4;
constexpr int kFwdKs = 2;
constexpr int kFwdRowBytes = kFwdKs * 128;
constexpr int kFwdStageBytes = 64 * kFwdRowBytes;
static_assert(kFcWarps * kFcMt * 4 == 64, "fc_fwd_kernel stages 64 images per CTA");

struct FcPlan {
    bool ok = false;
    int B, C, Cout, NT;           // NT = n-tiles of 8
    int ksteps;                   // K steps of 16 (4 channels)
    int ksplit, kslice;           // K splits, k-steps per split
    int mblocks;                  // M blocks of kFcWarps * kFcMt * 16 rows
    size_t wpack_bytes, part_bytes;
    uint32_t smem;
};

FcPlan fc_plan(const Problem &p) {
    FcPlan f;
    const bool full = p.KH == p.H && p.KW == p.W && p.pad == 0;
    if (!full || p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4) return f;
    f.B = (int)p.B;
    f.C = (int)(p.KH * p.KW * p.C);
    f.Cout = (int)p.Cout;
    f.NT = (int)((p.Cout * 4 + 7) / 8);
    if (f.NT > kFcMaxNt || f.C % 4 != 0 || p.B > (1 << 24)) return f;
    f.ksteps = f.C / 4;
    const int rows = f.B * 4;
    f.mblocks = (rows + kFcWarps * kFcMt * 16 - 1) / (kFcWarps * kFcMt * 16);
    // K splits: one wave of two CTAs per SM (a partial second wave doubles the
    // kernel time), weight slices of at most 48 KB (beside the 64 KB I ring)
    const int nsm = device_info().num_sms;
    int ks = std::max(1, (2 * nsm) / f.mblocks);
    const int kmax = (48 * 1024) / (f.NT * 256);   // weight slice <= 48 KB: two CTAs per SM with the I ring
    ks = std::max(ks, (f.ksteps + kmax - 1) / kmax);
    ks = std::min(ks, f.ksteps);
    f.kslice = (f.ksteps + ks - 1) / ks;
    f.ksplit = (f.ksteps + f.kslice - 1) / f.kslice;
    f.smem = kFwdStages * kFwdStageBytes + (uint32_t)f.kslice * f.NT * 256u;
    f.wpack_bytes = ((size_t)f.ksteps * f.NT * 256 + 255) & ~(size_t)255;
    f.part_bytes = ((size_t)f.ksplit * rows * f.NT * 8 * 4 + 255) & ~(size_t)255;
    f.ok = true;
    return f;
}

// Fragment k order.  The MMA's k index inside a 16-step may be any
// permutation shared by A and B; here fragment k-pair (2t, 2t+1) is
// (channel 4*kstep + t, d2 0..1) and (2t+8, 2t+9) is (same channel, d2 2..3),
// and fragment rows g, g+8 are capsule rows d1 = 2(g%2), 2(g%2)+1 of image g/2:
// a thread's whole A fragment is then the 16 contiguous bytes
// I[b][c][d1..d1+1][0..3] -- one vector load.
//
// Weights -> fragment order: wp[kstep][nt][lane] = {b0, b1} (two bf16x2),
// b0 = (c = 4*kstep + t, d2 = 0, 1; n = g), b1 = (same c, d2 = 2, 3; n = g), with
// g = lane/4, t = lane%4, n = (c' = (8nt+g)/4, d3 = (8nt+g)%4), value
// K[c][c'][d2][d3]; columns past 4*Cout are zero.
__global__ void __launch_bounds__(256) fc_pack(const __nv_bfloat16 *__restrict__ K, uint32_t *__restrict__ wp,
                                               int ksteps, int NT, int Cout) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)ksteps * NT * 32;
    if (idx >= total) return;
    const int lane = (int)(idx % 32);
    const int nt = (int)((idx / 32) % NT);
    const int kstep = (int)(idx / 32 / NT);
    const int g = lane >> 2, t = lane & 3;
    const int n = nt * 8 + g;
    uint32_t out[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        __nv_bfloat16 v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 4 * kstep + t, d2 = 2 * h + e;
            v[e] = __float2bfloat16_rn(0.f);
            if (n < 4 * Cout) v[e] = K[(((size_t)c * Cout + n / 4) * 4 + d2) * 4 + (n % 4)];
        }
        out[h] = (uint32_t)__bfloat16_as_ushort(v[0]) | ((uint32_t)__bfloat16_as_ushort(v[1]) << 16);
    }
    reinterpret_cast<uint2 *>(wp)[idx] = make_uint2(out[0], out[1]);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ void hmma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragment of m-tile (4 images from b0) at k-step kstep: lane (g, t) loads
// I[b0 + g/2][4*kstep + t][2(g%2) .. 2(g%2)+1][0..3] (16 bytes) = {a0, a2, a1, a3}.
__device__ __forceinline__ void load_a(const uint4 *__restrict__ I16, int C, int B, int b0, int kstep, int g, int t,
                                       uint32_t (&a)[4]) {
    const int b = b0 + (g >> 1);
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (b < B) v = __ldg(I16 + ((size_t)b * C + 4 * kstep + t) * 2 + (g & 1));
    a[0] = v.x;   // row g:     d2 0..1
    a[2] = v.y;   // row g:     d2 2..3
    a[1] = v.z;   // row g + 8: d2 0..1
    a[3] = v.w;   // row g + 8: d2 2..3
}

template <int NT>
__global__ void __launch_bounds__(kFcWarps * 32) fc_fwd_kernel(const __nv_bfloat16 *__restrict__ I,
                                                                const uint32_t *__restrict__ wp,
                                                                float *__restrict__ part, int B, int C, int kslice,
                                                                int ksteps) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    extern __shared__ __align__(128) uint8_t fw_smem[];
    uint8_t *ring = fw_smem;
    uint32_t *wsm = reinterpret_cast<uint32_t *>(fw_smem + kFwdStages * kFwdStageBytes);
    const int ks = blockIdx.x, mb = blockIdx.y;
    const int k0 = ks * kslice, k1 = min(ksteps, k0 + kslice);
    const int nk = k1 - k0;
    const int nst = (nk + kFwdKs - 1) / kFwdKs;
    const int b_lo = mb * 64;
    const uint4 *I16 = reinterpret_cast<const uint4 *>(I);
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    // per-thread copy slots: 64 images x kFwdKs*8 chunks of 16 B per stage
    constexpr int kChunks = 64 * kFwdKs * 8 / (kFcWarps * 32);
    auto issue = [&](int st) {
        if (st < nst) {
            const uint32_t dst0 = ring_s + (uint32_t)(st % kFwdStages) * kFwdStageBytes;
#pragma unroll
            for (int r = 0; r < kChunks; ++r) {
                const int e = threadIdx.x + r * kFcWarps * 32;
                const int img = e / (kFwdKs * 8), j = e % (kFwdKs * 8);
                const int b = b_lo + img, kstep = k0 + st * kFwdKs + j / 8;
                const bool ok = b < B && kstep < k1;
                const uint4 *src = ok ? I16 + (((size_t)b * C + 4 * kstep) * 2 + (j & 7)) : I16;
                cp_async16(dst0 + img * kFwdRowBytes + j * 16, src, ok);
            }
        }
        cp_async_commit();
    };
    // weight slice -> shared memory (fragment order, contiguous in global), committed
    // with I stage 0, so the first stage wait covers it
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(wp + (size_t)k0 * NT * 64);
        const uint32_t ws0 = (uint32_t)__cvta_generic_to_shared(wsm);
        for (int i = threadIdx.x; i < nk * NT * 16; i += blockDim.x) cp_async16(ws0 + i * 16, src + i, true);
    }
#pragma unroll
    for (int s0 = 0; s0 < kFwdStages - 1; ++s0) issue(s0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int rows = B * 4;
    const int r0 = (mb * kFcWarps + warp) * kFcMt * 16;   // first row (= 4 * first image) of the warp
    float acc[kFcMt][NT][4];
#pragma unroll
    for (int m = 0; m < kFcMt; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[m][n][e] = 0.f;
    // lane (g, t) of m-tile m: image 8*warp + 4m + g/2, channel 4*kstep + t, half g%2
    // = {a0, a2, a1, a3} (see load_a)
    const uint8_t *abase = ring + (8 * warp + (g >> 1)) * kFwdRowBytes + t * 32 + (g & 1) * 16;
    for (int st = 0; st < nst; ++st) {
        cp_async_wait<kFwdStages - 2>();
        __syncthreads();   // stage st landed for all threads (and, at st = 0, the weights); st-1 is free
        issue(st + kFwdStages - 1);
        const uint8_t *pa = abase + (st % kFwdStages) * kFwdStageBytes;
#pragma unroll
        for (int j = 0; j < kFwdKs; ++j) {
            const int kk = st * kFwdKs + j;
            if (kk < nk) {
                uint32_t a[kFcMt][4];
#pragma unroll
                for (int m = 0; m < kFcMt; ++m) {
                    const uint4 v = *reinterpret_cast<const uint4 *>(pa + 4 * m * kFwdRowBytes + j * 128);
                    a[m][0] = v.x; a[m][2] = v.y; a[m][1] = v.z; a[m][3] = v.w;
                }
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const uint2 bb = reinterpret_cast<const uint2 *>(wsm)[(kk * NT + n) * 32 + lane];
#pragma unroll
                    for (int m = 0; m < kFcMt; ++m) hmma16816(acc[m][n], a[m], bb.x, bb.y);
                }
            }
        }
    }
    cp_async_wait<0>();
    // partials part[ks][row = 4b + d1][NT*8]: c0,c1 -> fragment row g = (image g/2,
    // d1 = 2(g%2)), cols 2t, 2t+1; c2,c3 -> row g + 8 = (same image, d1 + 1)
    const int ncol = NT * 8;
    float *pk = part + (size_t)ks * rows * ncol;
#pragma unroll
    for (int m = 0; m < kFcMt; ++m) {
        const int b = (r0 >> 2) + 4 * m + (g >> 1);
        const int ra = 4 * b + 2 * (g & 1);
        if (b < B) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const int col = n * 8 + 2 * t;
                *reinterpret_cast<float2 *>(pk + (size_t)ra * ncol + col) = make_float2(acc[m][n][0], acc[m][n][1]);
                *reinterpret_cast<float2 *>(pk + (size_t)(ra + 1) * ncol + col) =
                    make_float2(acc[m][n][2], acc[m][n][3]);
            }
        }
    }
}

// O[b][c'][d1][d3] = sum over splits (fixed order) of part[ks][(b, d1)][(c', d3)], rounded to bf16
__global__ void __launch_bounds__(256) fc_finalize(const float *__restrict__ part, __nv_bfloat16 *__restrict__ O,
                                                   int B, int Cout, int ncol, int ksplit) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (row, c')
    const int64_t rows = (int64_t)B * 4;
    if (idx >= rows * Cout) return;
    const int co = (int)(idx % Cout);
    const int64_t r = idx / Cout;
    const int64_t b = r >> 2;
    const int d1 = (int)(r & 3);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int k = 0; k < ksplit; ++k) {
        const float4 v = *reinterpret_cast<const float4 *>(part + ((size_t)k * rows + r) * ncol + co * 4);
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(s.x, s.y), hi = __floats2bfloat162_rn(s.z, s.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t *>(&lo);
    w.y = *reinterpret_cast<uint32_t *>(&hi);
    *reinterpret_cast<uint2 *>(O + (((size_t)b * Cout + co) * 4 + d1) * 4) = w;
}

// ------------------------------------------------------------------ dI
// dI[b, c, d1, d2] = sum_{c', d3} dO[b, c', d1, d3] * K[c, c', d2, d3]
// rows m = (b, d1), k = (c', d3) (K = 4*Cout, zero-padded to 16-steps),
// columns n = (c, d2) (N = 4*C).  Same fragment permutation as the forward:
// k-pair (2t, 2t+1) = (c' = 4*kstep + t, d3 0..1), (2t+8, 2t+9) = (same c',
// d3 2..3); fragment rows g, g+8 = d1 = 2(g%2), 2(g%2)+1 of image g/2, so a
// thread's A fragment is the 16 bytes dO[b][c'][d1..d1+1][0..3].
//
// Weights -> wpd[kstep][nt][lane] = {b0, b1}: b0 = (c' = 4*kstep + t, d3 = 0, 1;
// n = 8nt + g), b1 = (same c', d3 = 2, 3), n = (c = n/4, d2 = n%4), value
// K[c][c'][d2][d3]; c' >= Cout is zero.
__global__ void __launch_bounds__(256) fc_pack_dgrad(const __nv_bfloat16 *__restrict__ K, uint32_t *__restrict__ wp,
                                                     int ksteps, int NT, int Cout) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)ksteps * NT * 32;
    if (idx >= total) return;
    const int lane = (int)(idx % 32);
    const int nt = (int)((idx / 32) % NT);
    const int kstep = (int)(idx / 32 / NT);
    const int g = lane >> 2, t = lane & 3;
    const int n = nt * 8 + g;
    const int co = 4 * kstep + t;
    uint32_t out[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        __nv_bfloat16 v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int d3 = 2 * h + e;
            v[e] = __float2bfloat16_rn(0.f);
            if (co < Cout) v[e] = K[(((size_t)(n / 4) * Cout + co) * 4 + (n % 4)) * 4 + d3];
        }
        out[h] = (uint32_t)__bfloat16_as_ushort(v[0]) | ((uint32_t)__bfloat16_as_ushort(v[1]) << 16);
    }
    reinterpret_cast<uint2 *>(wp)[idx] = make_uint2(out[0], out[1]);
}

constexpr int kFcDgKs = 4;     // max k-steps (4*Cout <= 64)
constexpr int kFcDgNt = 64;    // max n-tiles per CTA column block (512 columns)

// CTA = (column block of kFcDgNt n-tiles, 8 warps x 2 m-tiles of rows); each
// warp loads its dO fragments once and walks the column block.
__global__ void __launch_bounds__(kFcWarps * 32) fc_dgrad_kernel(const __nv_bfloat16 *__restrict__ dO,
                                                                  const uint32_t *__restrict__ wp,
                                                                  __nv_bfloat16 *__restrict__ dI, int B, int C,
                                                                  int Cout, int ksteps, int NTall, int ntper) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    extern __shared__ __align__(16) uint32_t wsm[];
    const int nb = blockIdx.x, mb = blockIdx.y;
    const int nt0 = nb * ntper, nt1 = min(NTall, nt0 + ntper);
    const int nnt = nt1 - nt0;
    // weights of this column block, all k-steps: wsm[kstep][ntl][lane] (async, overlaps the dO loads)
    {
        const uint32_t ws0 = (uint32_t)__cvta_generic_to_shared(wsm);
        for (int i = threadIdx.x; i < ksteps * nnt * 16; i += blockDim.x) {
            const int kstep = i / (nnt * 16), rem = i - kstep * nnt * 16;
            cp_async16(ws0 + i * 16, reinterpret_cast<const uint4 *>(wp) + ((size_t)kstep * NTall + nt0) * 16 + rem,
                       true);
        }
        cp_async_commit();
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int img0 = (mb * kFcWarps + warp) * kFcMt * 4;   // first image of the warp
    uint32_t a[kFcDgKs][kFcMt][4];
#pragma unroll
    for (int j = 0; j < kFcDgKs; ++j)
#pragma unroll
        for (int m = 0; m < kFcMt; ++m) {
            a[j][m][0] = a[j][m][1] = a[j][m][2] = a[j][m][3] = 0u;
            const int b = img0 + 4 * m + (g >> 1), co = 4 * j + t;
            if (j < ksteps && b < B && co < Cout) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(dO) + ((size_t)b * Cout + co) * 2 + (g & 1));
                a[j][m][0] = v.x; a[j][m][2] = v.y; a[j][m][1] = v.z; a[j][m][3] = v.w;
            }
        }
    cp_async_wait<0>();
    __syncthreads();
    for (int ntl = 0; ntl < nnt; ++ntl) {
        float acc[kFcMt][4];
#pragma unroll
        for (int m = 0; m < kFcMt; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
#pragma unroll
        for (int j = 0; j < kFcDgKs; ++j) {
            if (j < ksteps) {
                const uint2 bb = reinterpret_cast<const uint2 *>(wsm)[(j * nnt + ntl) * 32 + lane];
#pragma unroll
                for (int m = 0; m < kFcMt; ++m) hmma16816(acc[m], a[j][m], bb.x, bb.y);
            }
        }
        // c0,c1: row (image g/2, d1 = 2(g%2)), columns n = 8nt + 2t, +1 =
        // (c = n/4, d2 = 2(t%2) .. +1); c2,c3: row d1 + 1.  Lanes t and t^1 hold
        // the two d2 halves of the same capsule rows: one exchange gives the
        // even lane row d1 and the odd lane row d1 + 1 whole (8 bytes), so a warp
        // store writes full 64-byte capsule pairs.
        const int n = (nt0 + ntl) * 8 + 2 * t;
        const int c = n >> 2;
        const bool odd = t & 1;
#pragma unroll
        for (int m = 0; m < kFcMt; ++m) {
            const int b = img0 + 4 * m + (g >> 1);
            __nv_bfloat162 lo = __floats2bfloat162_rn(acc[m][0], acc[m][1]);
            __nv_bfloat162 hi = __floats2bfloat162_rn(acc[m][2], acc[m][3]);
            const uint32_t ulo = *reinterpret_cast<uint32_t *>(&lo), uhi = *reinterpret_cast<uint32_t *>(&hi);
            const uint32_t x = __shfl_xor_sync(0xffffffffu, odd ? ulo : uhi, 1);
            if (b < B && c < C) {
                const int row = 2 * (g & 1) + (odd ? 1 : 0);
                const uint2 w = odd ? make_uint2(x, uhi) : make_uint2(ulo, x);
                *reinterpret_cast<uint2 *>(dI + (((size_t)b * C + c) * 4 + row) * 4) = w;
            }
        }
    }
}

// ------------------------------------------------------------------ dK
// dK[c, c', d2, d3] = sum_{b, d1} I[b, c, d1, d2] * dO[b, c', d1, d3]
// rows m = (c, d2), columns n = (c', d3), k = (b, d1).  The contraction runs
// over d1, the row index of both capsules, so a fragment register needs two
// elements of one capsule *column*: fragment rows g, g+8 = (channel c0 + g/4,
// c0 + 2 + g/4; d2 = g%4), k-pair (2t, 2t+1) = (image b0 + t, d1 0..1), (2t+8,
// 2t+9) = (same image, d1 2..3).  A thread loads the whole 32-byte capsule
// (the four threads of a channel read the same address: an L1 broadcast) and
// extracts its column pair with one PRMT per register; B (dO) likewise with
// n = 8nt + g = (c' = 2nt + g/4, d3 = g%4).
__device__ __forceinline__ void caps_cols(const uint4 &lo, const uint4 &hi, int col, uint32_t &r01, uint32_t &r23) {
    // capsule words: row d1 = words 2*d1, 2*d1+1 (element d2 at word 2*d1 + d2/2, half d2%2)
    const uint32_t sel = (col & 1) ? 0x7632u : 0x5410u;
    const uint32_t w0 = (col & 2) ? lo.y : lo.x;   // row 0
    const uint32_t w1 = (col & 2) ? lo.w : lo.z;   // row 1
    const uint32_t w2 = (col & 2) ? hi.y : hi.x;   // row 2
    const uint32_t w3 = (col & 2) ? hi.w : hi.z;   // row 3
    r01 = __byte_perm(w0, w1, sel);
    r23 = __byte_perm(w2, w3, sel);
}

using namespace umma;   // mbarriers and 1-D bulk copies of the dK stream
constexpr int kFcDkNt = 8;     // n-tiles (4*Cout <= 64)

// I / dO stream of the dK kernel: a ring of kDkStages stages, each the 4
// images of one k-step: the CTA's 64 channels of I (one 1-D bulk copy per
// image, <= 2 KB) and the image's dO (<= 16 capsules), completion on one
// mbarrier per stage.  Image row t sits at t * row + {0, 16, 64, 80}[t] bytes:
// a warp's 32-bit fragment read touches, per image, the banks {0,1,8,9} + x
// (two channels 32 B apart, two column words), and the per-image offsets
// {0, 4, 16, 20} banks keep the four images disjoint -- one wavefront.
constexpr int kDkStages = 4;
constexpr int kDkKs = 2;            // k-steps (4 images each) per stage
constexpr int kDkImg = 4 * kDkKs;   // images per stage
static_assert(kFcWarps * kFcMt * 4 == 64, "fc_dk_kernel stages 64 channels per CTA");
constexpr int kDkIRow = 64 * 32 + 128;
constexpr int kDkORow = 16 * 32 + 128;
constexpr int kDkStageBytes = kDkImg * kDkIRow + kDkImg * kDkORow;
constexpr uint32_t kDkBfrBytes = 2 * kDkKs * kFcDkNt * 32 * 8;
__device__ __forceinline__ int dk_row_extra(int t) { return ((t & 1) ? 16 : 0) + ((t & 2) ? 64 : 0); }

template <int NT>
__global__ void __launch_bounds__(kFcWarps * 32) fc_dk_kernel(const __nv_bfloat16 *__restrict__ I,
                                                               const __nv_bfloat16 *__restrict__ dO,
                                                               float *__restrict__ part, int B, int C, int Cout,
                                                               int bslice, int dbg) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    extern __shared__ __align__(128) uint8_t dk_smem[];
    uint8_t *ring = dk_smem;   // kDkStages x (4 I rows, then 4 dO rows)
    uint2 *bfr = reinterpret_cast<uint2 *>(dk_smem + kDkStages * kDkStageBytes);   // [2][kDkKs][NT][32] B fragments
    uint64_t *full = reinterpret_cast<uint64_t *>(dk_smem + kDkStages * kDkStageBytes + kDkBfrBytes);
    const int ks = blockIdx.x, mb = blockIdx.y;
    const int b_lo = ks * bslice, b_hi = min(B, b_lo + bslice);
    const int nimg = b_hi - b_lo;
    const int nks = (nimg + 3) / 4;                 // k-steps
    const int nst = (nimg + kDkImg - 1) / kDkImg;   // stages
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int c0 = mb * 64, nc = min(64, C - c0);
    if (threadIdx.x == 0) {
        for (int s0 = 0; s0 < kDkStages; ++s0) mbar_init(&full[s0], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // thread 0: stage ss <- images b_lo + kDkImg*ss .. (valid ones only; the rest are masked in the fragments)
    auto issue = [&](int ss) {
        if (ss >= nst || (kProbes && (dbg & 1))) return;
        uint8_t *st = ring + (ss % kDkStages) * kDkStageBytes;
        const int ni = min(kDkImg, nimg - kDkImg * ss);
        mbar_arrive_expect_tx(&full[ss % kDkStages], (uint32_t)ni * (nc + Cout) * 32u);
        for (int tt = 0; tt < ni; ++tt) {
            const size_t b = (size_t)(b_lo + kDkImg * ss + tt);
            bulk_g2s(st + tt * kDkIRow + dk_row_extra(tt), I + (b * C + c0) * 16, (uint32_t)nc * 32u,
                     &full[ss % kDkStages]);
            bulk_g2s(st + kDkImg * kDkIRow + tt * kDkORow + dk_row_extra(tt), dO + b * Cout * 16,
                     (uint32_t)Cout * 32u, &full[ss % kDkStages]);
        }
    };
    auto wait_stage = [&](int ss) {
        if (ss < nst && !(kProbes && (dbg & 1))) mbar_wait(&full[ss % kDkStages], (uint32_t)(ss / kDkStages) & 1u);
    };
    if (threadIdx.x == 0)
        for (int s0 = 0; s0 < kDkStages - 1; ++s0) issue(s0);
    float acc[kFcMt][NT][4];
#pragma unroll
    for (int m = 0; m < kFcMt; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[m][n][e] = 0.f;
    // Fragment reads: lane (g, t) needs column d2 (A) / d3 (B) = g % 4 of capsules of image t;
    // column j sits in word j/2 of every capsule row (8 B), half j%2.
    const int cw = warp * kFcMt * 4;   // first channel of the warp within the CTA block
    const uint32_t sel = (g & 1) ? 0x7632u : 0x5410u;
    const int wofs = (g & 2) ? 4 : 0;
    const uint8_t *abase = ring + t * kDkIRow + dk_row_extra(t) + (cw + (g >> 2)) * 32 + wofs;
    auto w32 = [](const uint8_t *p) { return *reinterpret_cast<const uint32_t *>(p); };
    // B fragments are the same for every warp: the CTA extracts those of stage ss
    // into bfr[ss % 2] one iteration ahead (entry e = (j, n, lane), j the k-step in the stage)
    auto extract_b = [&](int ss) {
        if (ss >= nst) return;
        for (int e = threadIdx.x; e < kDkKs * NT * 32; e += kFcWarps * 32) {
            const int j = e / (NT * 32), n = (e >> 5) % NT, ln = e & 31, gg = ln >> 2, tt = ln & 3;
            const int im = 4 * j + tt;   // image within the stage
            uint2 v = make_uint2(0u, 0u);
            if (kDkImg * ss + im < nimg) {
                const uint32_t sl = (gg & 1) ? 0x7632u : 0x5410u;
                const uint8_t *q = ring + (ss % kDkStages) * kDkStageBytes + kDkImg * kDkIRow + im * kDkORow +
                                   dk_row_extra(tt) + (2 * n + (gg >> 2)) * 32 + ((gg & 2) ? 4 : 0);
                v = make_uint2(__byte_perm(w32(q), w32(q + 8), sl), __byte_perm(w32(q + 16), w32(q + 24), sl));
            }
            bfr[(ss & 1) * kDkKs * NT * 32 + e] = v;
        }
    };
    wait_stage(0);
    extract_b(0);
    for (int ss = 0; ss < nst; ++ss) {
        wait_stage(ss + 1);
        __syncthreads();   // B(ss) extracted; every thread is done with stage ss-1 (and waited for ss, ss+1)
        if (threadIdx.x == 0) issue(ss + kDkStages - 1);
        extract_b(ss + 1);
        if (kProbes && (dbg & 2)) continue;
#pragma unroll
        for (int j = 0; j < kDkKs; ++j) {
        const int k = ss * kDkKs + j;
        if (k >= nks) break;
        const uint8_t *pa = abase + (ss % kDkStages) * kDkStageBytes + 4 * j * kDkIRow;
        const bool tv = 4 * k + t < nimg;   // past the slice: zero A (smem holds stale data)
        uint32_t a[kFcMt][4];
#pragma unroll
        for (int m = 0; m < kFcMt; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint8_t *q = pa + (4 * m + 2 * h) * 32;   // a0/a1: d1 0..1, a2/a3: d1 2..3
                a[m][h] = tv ? __byte_perm(w32(q), w32(q + 8), sel) : 0u;
                a[m][h + 2] = tv ? __byte_perm(w32(q + 16), w32(q + 24), sel) : 0u;
            }
#pragma unroll
        for (int n = 0; n < NT; ++n) {   // c' = 2n + g/4; past Cout: garbage columns, never stored
            const uint2 bb = bfr[((ss & 1) * kDkKs + j) * NT * 32 + n * 32 + lane];
#pragma unroll
            for (int m = 0; m < kFcMt; ++m) hmma16816(acc[m][n], a[m], bb.x, bb.y);
        }
        }
    }
    // partials in dK layout: part[ks][c][c'][d2][d3]; c0,c1 -> row g (c, d2 = g%4),
    // cols n = 8nt + 2t, +1 = (c' = 2nt + t/2, d3 = 2(t%2), +1); c2,c3 -> channel c + 2
    float *pk = part + (size_t)ks * C * Cout * 16;
#pragma unroll
    for (int m = 0; m < kFcMt; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = c0 + cw + 4 * m + 2 * h + (g >> 2), d2 = g & 3;
            if (c >= C) continue;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                const int co = 2 * n + (t >> 1), d3 = 2 * (t & 1);
                if (co < Cout)
                    *reinterpret_cast<float2 *>(pk + (((size_t)c * Cout + co) * 4 + d2) * 4 + d3) =
                        make_float2(acc[m][n][2 * h], acc[m][n][2 * h + 1]);
            }
        }
}

__global__ void __launch_bounds__(256) fc_dk_finalize(const float *__restrict__ part, float *__restrict__ dK,
                                                      int64_t n, int ksplit) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // float4 index, n % 4 == 0
    if (i >= n / 4) return;
    const float4 *p4 = reinterpret_cast<const float4 *>(part);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int k = 0; k < ksplit; ++k) {
        const float4 v = p4[(size_t)k * (n / 4) + i];
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    reinterpret_cast<float4 *>(dK)[i] = s;
}

}  // namespace

bool fc_hmma_fwd_supported(const Problem &p) {
    static const bool off = probe_env("CAPSCONV_NO_FC_HMMA") != nullptr;
    return !off && fc_plan(p).ok;
}

size_t fc_hmma_fwd_workspace(const Problem &p) {
    const FcPlan f = fc_plan(p);
    return f.ok ? f.wpack_bytes + f.part_bytes : 0;
}

cudaError_t fc_hmma_fwd(const Problem &p, const void *I, const void *K, void *O, void *ws, size_t ws_bytes,
                        cudaStream_t st) {
    const FcPlan f = fc_plan(p);
    if (!f.ok || ws_bytes < f.wpack_bytes + f.part_bytes) return cudaErrorInvalidValue;
    uint32_t *wp = static_cast<uint32_t *>(ws);
    float *part = reinterpret_cast<float *>(static_cast<uint8_t *>(ws) + f.wpack_bytes);
    const int64_t npk = (int64_t)f.ksteps * f.NT * 32;
    launch_k(fc_pack, dim3((unsigned)((npk + 255) / 256)), dim3(256), 0, st, static_cast<const __nv_bfloat16 *>(K), wp, f.ksteps, f.NT,
                                                            f.Cout);
    note_launches(1);
    const dim3 grid((unsigned)f.ksplit, (unsigned)f.mblocks);
    const __nv_bfloat16 *Ib = static_cast<const __nv_bfloat16 *>(I);
    cudaError_t e = cudaSuccess;
    switch (f.NT) {
#define FC_CASE(nt)                                                                                               \
    case nt:                                                                                                      \
        e = smem_optin(reinterpret_cast<const void *>(fc_fwd_kernel<nt>), (int)f.smem);    \
        if (e != cudaSuccess) return e;                                                                           \
        launch_k(fc_fwd_kernel<nt>, dim3(grid), dim3(kFcWarps * 32), f.smem, st, Ib, wp, part, f.B, f.C, f.kslice, f.ksteps);        \
        break;
        FC_CASE(1) FC_CASE(2) FC_CASE(3) FC_CASE(4) FC_CASE(5) FC_CASE(6) FC_CASE(7) FC_CASE(8)
#undef FC_CASE
        default: return cudaErrorInvalidValue;
    }
    note_launches(1);
    const int64_t nfin = (int64_t)f.B * 4 * f.Cout;
    launch_k(fc_finalize, dim3((unsigned)((nfin + 255) / 256)), dim3(256), 0, st, part, static_cast<__nv_bfloat16 *>(O), f.B, f.Cout,
                                                                f.NT * 8, f.ksplit);
    note_launches(1);
    return cudaGetLastError();
}


namespace {
struct FcDgPlan {
    bool ok = false;
    int B, C, Cout, ksteps, NTall, ntper, nblocks, mblocks;
    size_t wpack_bytes;
    uint32_t smem;
};
FcDgPlan fc_dg_plan(const Problem &p) {
    FcDgPlan f;
    const bool full = p.KH == p.H && p.KW == p.W && p.pad == 0;
    if (!full || p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4) return f;
    f.B = (int)p.B;
    f.C = (int)(p.KH * p.KW * p.C);
    f.Cout = (int)p.Cout;
    f.ksteps = (f.Cout + 3) / 4;
    if (f.ksteps > kFcDgKs || p.B > (1 << 24)) return f;
    f.NTall = (f.C * 4 + 7) / 8;
    f.mblocks = (f.B + kFcWarps * kFcMt * 4 - 1) / (kFcWarps * kFcMt * 4);
    // column blocks: one wave of three CTAs per SM (72 registers x 256 threads)
    const int nsm = device_info().num_sms;
    const int nb = std::max(1, (3 * nsm) / f.mblocks);
    f.ntper = std::min(kFcDgNt, (f.NTall + nb - 1) / nb);
    f.nblocks = (f.NTall + f.ntper - 1) / f.ntper;
    f.smem = (uint32_t)f.ksteps * f.ntper * 256u;
    f.wpack_bytes = ((size_t)f.ksteps * f.NTall * 256 + 255) & ~(size_t)255;
    f.ok = true;
    return f;
}
}  // namespace

bool fc_hmma_dgrad_supported(const Problem &p) {
    static const bool off = probe_env("CAPSCONV_NO_FC_HMMA") != nullptr;
    return !off && fc_dg_plan(p).ok;
}

size_t fc_hmma_dgrad_workspace(const Problem &p) {
    const FcDgPlan f = fc_dg_plan(p);
    return f.ok ? f.wpack_bytes : 0;
}

cudaError_t fc_hmma_dgrad(const Problem &p, const void *dO, const void *K, void *dI, void *ws, size_t ws_bytes,
                          cudaStream_t st) {
    const FcDgPlan f = fc_dg_plan(p);
    if (!f.ok || ws_bytes < f.wpack_bytes) return cudaErrorInvalidValue;
    uint32_t *wp = static_cast<uint32_t *>(ws);
    const int64_t npk = (int64_t)f.ksteps * f.NTall * 32;
    launch_k(fc_pack_dgrad, dim3((unsigned)((npk + 255) / 256)), dim3(256), 0, st, static_cast<const __nv_bfloat16 *>(K), wp, f.ksteps,
                                                                  f.NTall, f.Cout);
    note_launches(1);
    cudaError_t e = smem_optin(reinterpret_cast<const void *>(fc_dgrad_kernel), (int)f.smem);
    if (e != cudaSuccess) return e;
    launch_k(fc_dgrad_kernel, dim3(dim3((unsigned)f.nblocks, (unsigned)f.mblocks)), dim3(kFcWarps * 32), f.smem, st, 
        static_cast<const __nv_bfloat16 *>(dO), wp, static_cast<__nv_bfloat16 *>(dI), f.B, f.C, f.Cout, f.ksteps,
        f.NTall, f.ntper);
    note_launches(1);
    return cudaGetLastError();
}


namespace {
struct FcDkPlan {
    bool ok = false;
    int B, C, Cout, NT, mblocks, ksplit, bslice;
    size_t part_bytes;
};
FcDkPlan fc_dk_plan(const Problem &p) {
    FcDkPlan f;
    const bool full = p.KH == p.H && p.KW == p.W && p.pad == 0;
    if (!full || p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4) return f;
    f.B = (int)p.B;
    f.C = (int)(p.KH * p.KW * p.C);
    f.Cout = (int)p.Cout;
    f.NT = (f.Cout * 4 + 7) / 8;
    if (f.NT > kFcDkNt || p.B > (1 << 24)) return f;
    f.mblocks = (f.C + kFcWarps * kFcMt * 4 - 1) / (kFcWarps * kFcMt * 4);
    // image splits: one wave of two CTAs per SM
    const int nsm = device_info().num_sms;
    int ks = std::max(1, (2 * nsm) / f.mblocks);
    ks = std::min(ks, (f.B + 3) / 4);
    f.bslice = ((f.B + ks - 1) / ks + 3) / 4 * 4;
    f.ksplit = (f.B + f.bslice - 1) / f.bslice;
    f.part_bytes = ((size_t)f.ksplit * f.C * f.Cout * 16 * 4 + 255) & ~(size_t)255;
    f.ok = true;
    return f;
}
}  // namespace

bool fc_hmma_dk_supported(const Problem &p) {
    static const bool off = probe_env("CAPSCONV_NO_FC_HMMA") != nullptr;
    return !off && fc_dk_plan(p).ok;
}

size_t fc_hmma_dk_workspace(const Problem &p) {
    const FcDkPlan f = fc_dk_plan(p);
    return f.ok ? f.part_bytes : 0;
}

cudaError_t fc_hmma_dk(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                       cudaStream_t st) {
    const FcDkPlan f = fc_dk_plan(p);
    if (!f.ok || ws_bytes < f.part_bytes) return cudaErrorInvalidValue;
    float *part = static_cast<float *>(ws);
    const dim3 grid((unsigned)f.ksplit, (unsigned)f.mblocks);
    const __nv_bfloat16 *Ib = static_cast<const __nv_bfloat16 *>(I), *Ob = static_cast<const __nv_bfloat16 *>(dO);
    const uint32_t smem = kDkStages * kDkStageBytes + kDkBfrBytes + kDkStages * 8;
    static const int dbg = probe_env("CAPSCONV_FC_DBG") ? atoi(probe_env("CAPSCONV_FC_DBG")) : 0;   // probe only
    cudaError_t e = cudaSuccess;
    switch (f.NT) {
#define DK_CASE(nt)                                                                                         \
    case nt:                                                                                                \
        e = smem_optin(reinterpret_cast<const void *>(fc_dk_kernel<nt>), (int)smem);     \
        if (e != cudaSuccess) return e;                                                                         \
        launch_k(fc_dk_kernel<nt>, dim3(grid), dim3(kFcWarps * 32), smem, st, Ib, Ob, part, f.B, f.C, f.Cout, f.bslice, dbg);       \
        break;
        DK_CASE(1) DK_CASE(2) DK_CASE(3) DK_CASE(4) DK_CASE(5) DK_CASE(6) DK_CASE(7) DK_CASE(8)
#undef DK_CASE
        default: return cudaErrorInvalidValue;
    }
    note_launches(1);
    const int64_t n = (int64_t)f.C * f.Cout * 16;
    launch_k(fc_dk_finalize, dim3((unsigned)((n / 4 + 255) / 256)), dim3(256), 0, st, part, dK, n, f.ksplit);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace capsconv
