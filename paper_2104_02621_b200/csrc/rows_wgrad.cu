// rows_wgrad.cu -- the kernel gradient dK for the D1-outer ("rows") layout on
// tcgen05, fed by TMA only (no loader warps, no shared-memory repack).
//
// Algorithm 4, read as the adjoint (R10/R11):
//     dK[p,q,c,c',d2,d3] = sum_{b,Y,X,d1} I[b, sY+p, sX+q, c, d1, d2] * dO[b, Y, X, c', d1, d3]
// With I stored [B][H][W][D1][C][D2] and dO [B][Ho][Wo][D1][Cout][D3], one
// staged capsule row (pixel, d1) holds all (c, d2) -- the M index of the GEMM
// -- contiguously, and the reduction index (pixel, d1) advances by whole rows:
// both operands are MN-major matrices exactly as TMA writes them.
//
// Row walk.  The reduction runs over output rows Y and, within a row, over
// k-steps of 4 pixels X0 = -bmax + 4*kx (16 capsule rows = one MMA K).  Column
// plane b holds input columns s*Xp + b (all input rows; element-strided TMA).
// One MMA covers a whole block of taps:
//   * M = 128 = up to 128/Ea "slots": slot j reads the plane at input row
//     s*Y + p0 + j -- the SAME staged buffer at a descriptor atom stride of
//     one plane row (Ea = elements of one staged I chunk);
//   * N = na*Eb "atoms": atom beta reads dO at column X + beta -- the same
//     staged dO buffer at an atom stride of one pixel.
// Slot j x atom beta accumulates  sum_X I[sY+p, s(X + qhi) + b] dO[Y, X + beta],
// i.e. tap (p0 + j, s*(qhi - beta) + b) once X + beta ranges over the dO row
// (columns outside [0, Wo) are TMA zero fill).  Slots past KH read whatever
// lies in shared memory; their D rows are never stored.
//
// Work items = (group set, split of the stage list); a CTA keeps its item's
// accumulators in TMEM over all its stages and writes fp32 partials, summed
// in a fixed order by rw_finalize (deterministic, no atomics).
// Roles (192 threads): warp 0 TMA, warp 1 MMA (TMEM owner), warps 2-5 epilogue.
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

constexpr int kRwMaxGroups = 8;    // MMA groups per set
constexpr int kRwMaxSets = 8;
constexpr int kRwMaxBufs = 8;      // staged buffers per stage
constexpr int kRwThreads = 192;
constexpr uint32_t kRwSmemLimit = 227 * 1024;

struct RwGroup {
    int ibuf, obuf;       // staged buffers (indices into the set's buffer list)
    int p0;               // tap row of slot 0
    int b, qhi, na;       // column plane, largest qq, atoms (qq = qhi - beta)
    int ci, co;           // I chunk, dO chunk
    int acol;             // plane column offset of this group inside its staged rows
    uint32_t dcol;        // TMEM column of the accumulator block
    uint32_t idesc;
};

struct RwBuf {
    int kind;             // 0: I plane chunk, 1: dO chunk
    int b, chunk;
    uint32_t off;         // byte offset inside a stage
};

struct RwSet {
    int ngroups, nbufs;
    RwGroup g[kRwMaxGroups];
    RwBuf buf[kRwMaxBufs];
    uint32_t stage_bytes;  // TMA bytes per stage
};

struct RowsWgrad {
    alignas(64) CUtensorMap tmI;   // I: box (Ea, 4, Wpb*s, rowsI, 1), element stride s on x
    alignas(64) CUtensorMap tmO;   // dO: box (Eb, 4, Wv, R, 1)
    float *part;                   // [ksplit][nK] partials, or dK itself (ksplit == 1)
    int s, KH, KW, C, Cout, B, H, W, Ho, Wo;
    int Ea, Eb;
    int R, nYst, nkx, bmax, Wpb, Wv, rowsI;
    int x0[4];                     // per plane: first staged plane column
    uint32_t pxA, pxO;             // bytes per staged pixel (4 capsule rows)
    uint32_t lboA, sboA, lboB, sboB;
    int nsets, ksplit, n_items, n_st;
    RwSet set[kRwMaxSets];
    uint32_t stage_stride;         // bytes between stage buffers (1024-aligned)
    int nstg;
    uint32_t smem_bytes;
    long long nK;
    int dbg;                       // probe builds only: 1 skip MMAs, 2 skip TMA loads, 4 skip the k-loop
};

// MMA issue of one work item: NG accumulator groups, descriptors built once
// per item and advanced by constant offsets (descriptor units of 16 bytes),
// so every operand lives in uniform registers; two k-steps per elected region.
template <int NG>
__device__ __forceinline__ void rw_mma_item(const RowsWgrad &P, const RwSet &S, uint32_t stg0, uint64_t *full,
                                            uint64_t *empty, int t0, int t1, int &sb, uint32_t &ph) {
    uint64_t ad[NG], bd[NG];
    uint32_t dc[NG], id[NG];
    const int ng = min(NG, S.ngroups);
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        const RwGroup &G = S.g[g < ng ? g : 0];
        ad[g] = rows::sdesc(stg0 + S.buf[G.ibuf].off + (uint32_t)(G.p0 * P.Wpb + G.acol) * P.pxA, P.lboA, P.sboA,
                            2 * P.Ea);
        bd[g] = rows::sdesc(stg0 + S.buf[G.obuf].off, P.lboB, P.sboB, 2 * P.Eb);
        dc[g] = G.dcol;
        id[g] = G.idesc;
    }
    const uint32_t rowa = ((uint32_t)(P.s * P.Wpb) * P.pxA) >> 4;   // one output row, A
    const uint32_t rowb = ((uint32_t)P.Wv * P.pxO) >> 4;
    const uint32_t ka = P.pxA >> 2, kb = P.pxO >> 2;                  // one k-step = 4 pixels
    const uint32_t sstr = P.stage_stride >> 4;
    const int nkx = P.nkx;
    uint32_t acc = 0;
    for (int t = t0; t < t1; ++t) {
        const int img = t / P.nYst, Y0 = (t - img * P.nYst) * P.R;
        const int Reff = min(P.R, P.Ho - Y0);
        mbar_wait(full + sb, ph);
        fence_after_sync();
        const uint32_t so = (uint32_t)sb * sstr;
        if (!(kProbes && (P.dbg & 4))) {
            for (int yl = 0; yl < Reff; ++yl) {
                const uint32_t oa0 = so + (uint32_t)yl * rowa, ob0 = so + (uint32_t)yl * rowb;
                for (int kx = 0; kx < nkx; ++kx) {
                    const uint32_t oa = oa0 + (uint32_t)kx * ka, ob = ob0 + (uint32_t)kx * kb;
                    if (!(kProbes && (P.dbg & 1))) {
#pragma unroll
                        for (int g = 0; g < NG; ++g)
                            if (g < ng) rows::mma_ss_elect(dc[g], ad[g] + oa, bd[g] + ob, id[g], acc);
                    }
                    acc = 1;
                }
            }
        }
        if (elect_one()) mma_commit(empty + sb);
        __syncwarp();
        if (++sb == P.nstg) { sb = 0; ph ^= 1; }
    }
}

__global__ void __launch_bounds__(kRwThreads, 1) rows_wgrad_kernel(const __grid_constant__ RowsWgrad P) {
    pdl_wait();   // no early PDL trigger: the split partials go to the workspace at the end
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *full = bars, *empty = bars + 8, *acc_full = bars + 16, *acc_empty = bars + 17;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + 512);
    const uint32_t stg0 = (smem_u32(smem_raw) + 1024u + 1023u) & ~1023u;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P.nstg; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 4);
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc_dyn(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (*tmem_slot != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmI)) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmO)) : "memory");
            int sb = 0;
            uint32_t ph = 0;
            for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
                const int gs = item / P.ksplit, ks = item - gs * P.ksplit;
                const RwSet &S = P.set[gs];
                const int t0 = (int)((long long)ks * P.n_st / P.ksplit);
                const int t1 = (int)((long long)(ks + 1) * P.n_st / P.ksplit);
                for (int t = t0; t < t1; ++t) {
                    const int img = t / P.nYst, Y0 = (t - img * P.nYst) * P.R;
                    mbar_wait(empty + sb, ph ^ 1);
                    const uint32_t stg = stg0 + (uint32_t)sb * P.stage_stride;
                    const uint32_t mb = smem_u32(full + sb);
                    if (kProbes && (P.dbg & 2)) {
                        mbar_arrive(full + sb);
                        if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                        continue;
                    }
                    mbar_arrive_expect_tx(full + sb, S.stage_bytes);
                    for (int i = 0; i < S.nbufs; ++i) {
                        const RwBuf &bf = S.buf[i];
                        if (bf.kind == 0)
                            rows::tma_load5d(stg + bf.off, &P.tmI, bf.chunk * P.Ea, 0, P.s * P.x0[bf.b] + bf.b,
                                             P.s * Y0, img, mb);
                        else
                            rows::tma_load5d(stg + bf.off, &P.tmO, bf.chunk * P.Eb, 0, -P.bmax, Y0, img, mb);
                    }
                    if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA
        int sb = 0;
        uint32_t ph = 0, aph = 0;
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            const int gs = item / P.ksplit, ks = item - gs * P.ksplit;
            const RwSet &S = P.set[gs];
            const int t0 = (int)((long long)ks * P.n_st / P.ksplit);
            const int t1 = (int)((long long)(ks + 1) * P.n_st / P.ksplit);
            mbar_wait(acc_empty, aph ^ 1);
            fence_after_sync();
            switch (S.ngroups) {
                case 1: rw_mma_item<1>(P, S, stg0, full, empty, t0, t1, sb, ph); break;
                case 2: rw_mma_item<2>(P, S, stg0, full, empty, t0, t1, sb, ph); break;
                case 3: rw_mma_item<3>(P, S, stg0, full, empty, t0, t1, sb, ph); break;
                case 4: rw_mma_item<4>(P, S, stg0, full, empty, t0, t1, sb, ph); break;
                default: rw_mma_item<8>(P, S, stg0, full, empty, t0, t1, sb, ph); break;
            }
            if (elect_one()) mma_commit(acc_full);
            __syncwarp();
            aph ^= 1;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;           // TMEM lane quarter of this warp
        const int m = q * 32 + lane;      // accumulator row
        uint32_t eph = 0;
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            const int gs = item / P.ksplit, ks = item - gs * P.ksplit;
            const RwSet &S = P.set[gs];
            mbar_wait(acc_full, eph);
            fence_after_sync();
            float *out = P.part + (size_t)ks * (size_t)P.nK;
            for (int g = 0; g < S.ngroups; ++g) {
                const RwGroup &G = S.g[g];
                const int j = m / P.Ea, r = m - j * P.Ea;
                const int p = G.p0 + j;
                const int c = G.ci * (P.Ea / 4) + (r >> 2), d2 = r & 3;
                const int N = G.na * P.Eb;
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + G.dcol;
                for (int n0 = 0; n0 < N; n0 += 16) {
                    float v[16];
                    tmem_ld16(taddr + (uint32_t)n0, v);
                    tmem_wait_ld();
                    if (p < P.KH) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int col = n0 + 4 * u;
                            const int beta = col / P.Eb, cl = (col - beta * P.Eb) >> 2;
                            const int qq = G.qhi - beta, qcol = P.s * qq + G.b;
                            const int co = G.co * (P.Eb / 4) + cl;
                            float *dst = out + ((((size_t)(p * P.KW + qcol) * P.C + c) * P.Cout + co) * 16 + d2 * 4);
                            *reinterpret_cast<float4 *>(dst) = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                        }
                    }
                }
            }
            fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
            eph ^= 1;
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_dealloc_dyn(0u, 512);
}

// dK[e] = sum_k part[k][e] in a fixed order: a block owns 32 float4 columns;
// warp w sums splits w, w + 16, w + 32, ... (independent loads in flight),
// then the 16 warp partials are added in warp order.  Deterministic.
constexpr int kFinWarps = 16;
__global__ void __launch_bounds__(kFinWarps * 32) rw_finalize(const float *__restrict__ part, float *__restrict__ dK,
                                                              long long n4, long long nK, int ksplit) {
    
    pdl_wait();
    __shared__ float4 red[kFinWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long i = (long long)blockIdx.x * 32 + lane;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n4) {
        const float4 *p = reinterpret_cast<const float4 *>(part) + i;
        const long long st4 = nK / 4;
        int k = w;
#pragma unroll 4
        for (; k < ksplit; k += kFinWarps) {
            const float4 v = __ldg(p + (size_t)k * (size_t)st4);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && i < n4) {
        float4 r = red[0][lane];
        for (int j = 1; j < kFinWarps; ++j) {
            const float4 v = red[j][lane];
            r.x += v.x; r.y += v.y; r.z += v.z; r.w += v.w;
        }
        reinterpret_cast<float4 *>(dK)[i] = r;
    }
}

struct RwPlan {
    bool ok = false;
    RowsWgrad P;
    size_t part_bytes = 0;
};

int chunk_width(int E) { return E % 64 == 0 ? 64 : E % 32 == 0 ? 32 : E % 16 == 0 ? 16 : 0; }

RwPlan make_rw_plan(const Problem &p) {
    RwPlan pl;
    RowsWgrad &P = pl.P;
    memset(&P, 0, sizeof(P));
    if (p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4 || p.pad != 0) return pl;
    if (p.s > 4 || p.B > (1 << 24)) return pl;
    const int s = (int)p.s, KH = (int)p.KH, KW = (int)p.KW;
    const int EI = 4 * (int)p.C, EO = 4 * (int)p.Cout;
    const int Ea = chunk_width(EI), Eb = chunk_width(EO);
    if (!Ea || !Eb) return pl;
    const int Sa = 128 / Ea;
    P.s = s; P.KH = KH; P.KW = KW; P.C = (int)p.C; P.Cout = (int)p.Cout; P.B = (int)p.B;
    P.H = (int)p.H; P.W = (int)p.W; P.Ho = (int)p.Ho; P.Wo = (int)p.Wo;
    P.Ea = Ea; P.Eb = Eb;
    P.pxA = 4u * Ea * 2u; P.pxO = 4u * Eb * 2u;
    // atoms per MMA: N = na * Eb <= 256
    const int na_max = std::max(1, 256 / Eb);
    // groups (before set packing)
    std::vector<RwGroup> gl;
    int bmax = 0;
    for (int b = 0; b < s && b < KW; ++b) {
        const int nqq = (KW - b + s - 1) / s;
        for (int qa = 0; qa < nqq; qa += na_max) {
            const int na = std::min(na_max, nqq - qa);
            bmax = std::max(bmax, na - 1);
            for (int p0 = 0; p0 < KH; p0 += Sa)
                for (int ci = 0; ci < EI / Ea; ++ci)
                    for (int co = 0; co < EO / Eb; ++co) {
                        RwGroup G{};
                        G.p0 = p0; G.b = b; G.qhi = qa + na - 1; G.na = na; G.ci = ci; G.co = co;
                        G.idesc = idesc_bf16(128, na * Eb, 1, 1);
                        gl.push_back(G);
                    }
        }
    }
    P.bmax = bmax;
    P.nkx = (P.Wo + bmax + 3) / 4;
    // staged plane columns per plane: [min qhi - bmax, 4 nkx + max qhi - bmax)
    int wpb = 0;
    for (int b = 0; b < s && b < KW; ++b) {
        int lo = 1 << 30, hi = -1;
        for (auto &G : gl)
            if (G.b == b) { lo = std::min(lo, G.qhi); hi = std::max(hi, G.qhi); }
        P.x0[b] = lo - bmax;
        for (auto &G : gl)
            if (G.b == b) G.acol = G.qhi - lo;
        wpb = std::max(wpb, 4 * P.nkx + hi - lo);
    }
    P.Wpb = wpb;
    P.Wv = 4 * P.nkx + bmax;
    if (P.Wpb * s > 256 || P.Wv > 256) return pl;
    P.lboA = (uint32_t)P.Wpb * P.pxA;   // slot stride: one plane row
    P.sboA = 8u * Ea * 2u;
    P.lboB = P.pxO;                     // atom stride: one pixel
    P.sboB = 8u * Eb * 2u;
    if ((P.lboA >> 4) >= (1u << 14)) return pl;
    // pack groups into sets of <= 512 TMEM columns, dO chunk outermost
    std::stable_sort(gl.begin(), gl.end(), [](const RwGroup &x, const RwGroup &y) { return x.co < y.co; });
    std::vector<std::vector<RwGroup>> sets;
    int cols = 0;
    for (auto &G : gl) {
        const int n = G.na * Eb;
        if (sets.empty() || cols + n > 512 || (int)sets.back().size() >= kRwMaxGroups) {
            sets.emplace_back();
            cols = 0;
        }
        G.dcol = (uint32_t)cols;
        cols += n;
        sets.back().push_back(G);
    }
    if ((int)sets.size() > kRwMaxSets) return pl;
    P.nsets = (int)sets.size();
    // rows per stage: the largest R that double-buffers in shared memory
    const uint32_t slack = (uint32_t)Sa * P.lboA + 4096u;   // garbage slots read past the last I buffer
    auto set_bytes = [&](const std::vector<RwGroup> &S, int R, RwSet *out) -> uint32_t {
        const int rowsI = s * (R - 1) + KH;
        std::vector<RwBuf> bufs;
        uint32_t off = 0;
        auto find = [&](int kind, int b, int ch) {
            for (size_t i = 0; i < bufs.size(); ++i)
                if (bufs[i].kind == kind && bufs[i].b == b && bufs[i].chunk == ch) return (int)i;
            RwBuf bf{kind, b, ch, off};
            off += kind == 0 ? (uint32_t)rowsI * P.Wpb * P.pxA : (uint32_t)R * P.Wv * P.pxO;
            off = (off + 1023u) & ~1023u;
            bufs.push_back(bf);
            return (int)bufs.size() - 1;
        };
        std::vector<RwGroup> G2 = S;
        for (auto &G : G2) G.ibuf = find(0, G.b, G.ci);
        for (auto &G : G2) G.obuf = find(1, 0, G.co);
        if (out) {
            if ((int)bufs.size() > kRwMaxBufs) return ~0u;
            out->ngroups = (int)G2.size();
            for (size_t i = 0; i < G2.size(); ++i) out->g[i] = G2[i];
            out->nbufs = (int)bufs.size();
            uint32_t tx = 0;
            for (size_t i = 0; i < bufs.size(); ++i) {
                out->buf[i] = bufs[i];
                tx += bufs[i].kind == 0 ? (uint32_t)rowsI * P.Wpb * P.pxA : (uint32_t)R * P.Wv * P.pxO;
            }
            out->stage_bytes = tx;
        }
        return (int)bufs.size() > kRwMaxBufs ? ~0u : off;
    };
    int best_R = 0, best_nstg = 0;
    uint32_t best_stride = 0;
    const int force_nstg = probe_env("CAPSCONV_RW_NSTG") ? atoi(probe_env("CAPSCONV_RW_NSTG")) : 0;
    for (int nstg = force_nstg ? force_nstg : 3; nstg >= 1 && !best_R; --nstg) {
        for (int R = std::min(P.Ho, 64); R >= 1; --R) {
            const int rowsI = s * (R - 1) + KH;
            if (rowsI > 256 || R > 256) continue;
            uint32_t stride = 0;
            for (auto &S : sets) stride = std::max(stride, set_bytes(S, R, nullptr));
            if (stride == ~0u) continue;
            const uint64_t need = 2048ull + (uint64_t)nstg * stride + slack;
            if (need <= kRwSmemLimit && (nstg < 3 || R >= std::min(P.Ho, 4))) {
                best_R = R; best_nstg = nstg; best_stride = stride;
                break;
            }
        }
    }
    if (!best_R) return pl;
    P.R = best_R;
    P.nstg = best_nstg;
    P.stage_stride = best_stride;
    P.rowsI = s * (P.R - 1) + KH;
    for (int i = 0; i < P.nsets; ++i)
        if (set_bytes(sets[i], P.R, &P.set[i]) == ~0u) return pl;
    P.smem_bytes = 2048u + (uint32_t)P.nstg * P.stage_stride + slack;
    P.nYst = (P.Ho + P.R - 1) / P.R;
    P.n_st = P.B * P.nYst;
    const int nsm = device_info().num_sms;
    P.ksplit = std::max(1, std::min(P.n_st, nsm / P.nsets));
    P.n_items = P.nsets * P.ksplit;
    P.nK = (long long)KH * KW * p.C * p.Cout * 16;
    pl.part_bytes = P.ksplit > 1 ? (((size_t)P.ksplit * (size_t)P.nK * 4 + 255) & ~(size_t)255) : 0;
    pl.ok = true;
    return pl;
}

struct RwKey {
    int dev, nsm;
    int64_t e[12];
    bool operator==(const RwKey &o) const {
        if (dev != o.dev || nsm != o.nsm) return false;
        for (int i = 0; i < 12; ++i)
            if (e[i] != o.e[i]) return false;
        return true;
    }
};

std::shared_ptr<const RwPlan> cached_rw_plan(const Problem &p) {
    static std::mutex mu;
    static std::vector<std::pair<RwKey, std::shared_ptr<const RwPlan>>> cache;
    const DeviceInfo &di = device_info();
    RwKey k{di.device, di.num_sms, {p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW, p.D1, p.D2, p.D3, p.s, p.pad}};
    if (p.dt != CAPSCONV_BF16) k.e[7] = -1;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &kv : cache)
        if (kv.first == k) return kv.second;
    if (cache.size() > 256) cache.clear();
    cache.emplace_back(k, std::make_shared<const RwPlan>(make_rw_plan(p)));
    std::shared_ptr<const RwPlan> sp = cache.back().second;
    if (probe_env("CAPSCONV_DEBUG") && sp->ok) {
        const RowsWgrad &P = sp->P;
        fprintf(stderr,
                "[capsconv] rows wgrad plan: s=%d Ea=%d Eb=%d R=%d nkx=%d bmax=%d Wpb=%d Wv=%d sets=%d groups0=%d "
                "ksplit=%d items=%d nstg=%d stage=%u smem=%u\n",
                P.s, P.Ea, P.Eb, P.R, P.nkx, P.bmax, P.Wpb, P.Wv, P.nsets, P.set[0].ngroups, P.ksplit, P.n_items,
                P.nstg, P.stage_stride, P.smem_bytes);
    }
    return sp;
}

}  // namespace

bool rows_wgrad_supported(const Problem &p) { return cached_rw_plan(p)->ok; }

size_t rows_wgrad_workspace_bytes(const Problem &p) {
    std::shared_ptr<const RwPlan> pl = cached_rw_plan(p);
    return pl->ok ? pl->part_bytes : 0;
}

cudaError_t rows_wgrad_run(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                           cudaStream_t st) {
    RwPlan pl = *cached_rw_plan(p);
    if (!pl.ok || ws_bytes < pl.part_bytes) return cudaErrorNotSupported;
    RowsWgrad &P = pl.P;
    if (!rows::make_rows_map5(&P.tmI, I, P.B, P.H, P.W, 4 * P.C, P.Ea, P.Wpb * P.s, P.rowsI, P.s, 1) ||
        !rows::make_rows_map5(&P.tmO, dO, P.B, P.Ho, P.Wo, 4 * P.Cout, P.Eb, P.Wv, P.R, 1, 1))
        return cudaErrorInvalidValue;
    P.part = P.ksplit > 1 ? static_cast<float *>(ws) : dK;
    P.dbg = probe_env("CAPSCONV_RW_DBG") ? atoi(probe_env("CAPSCONV_RW_DBG")) : 0;
    cudaError_t e = smem_optin(reinterpret_cast<const void *>(rows_wgrad_kernel), (int)P.smem_bytes);
    if (e != cudaSuccess) return e;
    const int grid = std::min(P.n_items, device_info().num_sms);
    e = launch_k(rows_wgrad_kernel, dim3(grid), dim3(kRwThreads), P.smem_bytes, st, P);
    if (e != cudaSuccess) return e;
    note_launches(1);
    if (P.ksplit > 1 && !probe_skip_fin()) {
        const long long n4 = P.nK / 4;
        e = launch_k(rw_finalize, dim3((unsigned)((n4 + 31) / 32)), dim3(kFinWarps * 32), 0, st,
                     static_cast<const float *>(P.part), dK, n4, P.nK, P.ksplit);
        if (e != cudaSuccess) return e;
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace capsconv
