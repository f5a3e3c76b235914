// rows_conv.cu -- forward O and data gradient dI for the D1-outer ("rows")
// layout on tcgen05, fed by TMA only (no producer / repack warps).
//
// The contraction (Algorithm 2; dI = the adjoint of
// Algorithm 4, reading R10/R11) is an implicit GEMM over a
// *virtual pixel grid*: rows M = (virtual pixel u, d1), reduction K = the
// source capsule row (c, d2) [fwd] or (c', d3) [dI], columns N = stacked
// output capsule rows.  With capsule rows stored contiguously ([..][D1][C][D2],
// rows.cuh) a staged window of source pixels IS the K-major A operand, and a
// kernel tap is the same window at another start row (one pixel = 4 rows):
//
//   fwd, stride s:  O[u]  = sum_{a,b,pp,qq} P_ab[u + pp*Wg + qq] . K[s pp + a, s qq + b]
//                   (P_ab = input phase plane (sY + a, sX + b); Wg = plane width)
//   dI,  stride s:  dI_ab[u] = sum_{pp,qq} dO[u - pp*Wg - qq] . K[s pp + a, s qq + b]^T
//                   (dI_ab = output phase (sY + a, sX + b); dO placed in the phase grid)
//
// Column-tap stacking.  The qq taps of one (plane, pp) share the A window up to
// a shift of qq pixels, so their weights are stacked side by side in N: one
// MMA of N = nq * E computes D_j[v] = sum A[v + sigma] W_j for every j, and the
// epilogue forms O[u] = sum_j D_j[u + j] (dI: D_j[u - j]) -- a shift of 4*j
// accumulator rows, i.e. lanes: warp shuffles inside a TMEM lane quarter and a
// small shared-memory hand-off across quarters.  N = 96..256 instead of 32..128
// per MMA (an SS MMA costs ~max(60 + N/8, N/2) cycles, tests/probe/rows_probe).
// Tiles of 32 virtual pixels overlap by the stacking span (T = 32 - span).
//
// Work item = G consecutive tiles sharing one staged window (whole virtual
// rows, one 5-D TMA box per row, element-strided for the stride-2 planes,
// zero filled outside the tensors).  Weights are prepacked once per call into
// the exact shared-memory image (K-major, no swizzle) and stay resident.
// Roles (448 threads): warps 0-11 three epilogue groups of four (one per TMEM
// lane quarter; each group owns a set of accumulator slots and drains their
// tiles in order), warp 12 MMA (TMEM owner), warp 13 TMA.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "conv_mma.cuh"
#include "internal.h"
#include "rows.cuh"
#include "umma.cuh"

namespace capsconv {
using namespace umma;

namespace {

constexpr int kRcMaxMma = 40;
constexpr int kRcMaxOut = 4;
constexpr int kRcMaxBlk = 4;
constexpr int kRcGroups = 3;                        // epilogue groups (4 warps each)
constexpr int kRcThreads = 64 + kRcGroups * 128;
constexpr uint32_t kRcSmemLimit = 227 * 1024;

struct RcMma {
    int pl;             // source plane
    int sig;            // A shift (virtual pixels) minus the smallest A shift
    uint32_t woff;      // byte offset of the packed B slice (all K) in the weight image
    int N;
    uint32_t dcol;      // accumulator column (inside a TMEM slot)
    uint32_t idesc;
    int zero;           // first writer of its D region: overwrite at the first k-step
    // packing: N = nblk * Eblk rows; row block i is tap (tp[i], tq[i]) (-1: zero)
    int nblk, tp[kRcMaxBlk], tq[kRcMaxBlk];
};

struct RcOut {
    int oy, ox, os;     // output pixel = (os*Y + oy, os*X + ox) of virtual (Y, X)
    int nblk;
    int dcol[kRcMaxBlk];
    int delta[kRcMaxBlk];   // lane offset 4*(sigma_j - sigma_min) >= 0
    int xo[kRcMaxBlk];      // first hand-off lane of block j (prefix sum of deltas)
    int kind;               // epilogue instantiation (block count and delta sequence)
};

struct RowsConv {
    alignas(64) CUtensorMap tmS;   // source, one virtual row: box (Ea, 4, Wg*es, 1, 1), element strides (1,1,es,1,1)
    alignas(64) CUtensorMap tmH;   // source, hb virtual rows: 5-D (per image) or, when merged, 4-D over B*Hs rows
    const uint8_t *wpack;          // packed weights (global)
    __nv_bfloat16 *out;
    int dgrad;
    int Bn, Hg, Wg, es;            // virtual grid per image; plane element stride
    int npl, pl_oy[4], pl_ox[4];   // plane p: source pixel (es*Y + oy, es*X + ox)
    int nch, Ea, kpc;              // source chunks, elements per chunk, k-steps per chunk
    uint32_t pxS;                  // staged bytes per pixel per chunk (4 rows of Ea bf16)
    int nmma;
    RcMma mma[kRcMaxMma];
    int nout;
    RcOut outp[kRcMaxOut];
    int T, smin;                   // output pixels per tile; smallest output shift
    int sAmin, sAspan;             // smallest A shift; span of A shifts
    int G, ntiles, n_items;
    int Hout, Wout, Eout;          // output tensor extents, elements per capsule row
    int ngrp;                      // epilogue groups in use (divides nacc: a slot always has one group)
    int pair;                      // MMA warp issues two tiles at a time (nacc == 4)
    int cstage;                    // one source chunk per pipeline stage (wide K, one tile per item)
    int prog;                      // compile-time MMA program (tap groups x k-steps), see the dispatch
    int dmax;                      // largest lane offset of any output
    int xl;                        // hand-off lanes per quarter (largest sum of an output's deltas)
    uint32_t wbytes;               // weight image bytes
    int rows_max;                  // staged virtual rows per plane per item (max, incl. box overshoot)
    int hb;                        // virtual rows per multi-row TMA box
    int merged;                    // virtual row R <-> source row es*R + oy over all images (4-D map)
    uint32_t plane_bytes;          // rows_max * Wg * pxS
    uint32_t chunk_bytes;          // npl * plane_bytes
    uint32_t stage_bytes;          // nch * chunk_bytes (1024 aligned)
    int nstg, nacc;
    uint32_t ND;                   // accumulator columns per tile
    uint32_t xoff, woff_s, stg_off;   // shared-memory offsets: hand-off buffer, weights, stages
    uint32_t soff;                    // per-warp store staging (2 KB per epilogue warp), 0 = none
    uint32_t smem_bytes;
    FastDiv fd_hw, fd_wg;          // virtual pixel -> (image, row, column)
    int dbg;                       // probe builds only: 1 skip MMAs, 2 skip TMA loads, 4 skip the epilogue body
    unsigned long long *prof;      // probe builds only: per-CTA cycle counters [cta][8]
};

// Window of item `it`: virtual rows [Ra, Ra + nrows) cover pixels
// [v0(first tile) + sAmin, v0(last tile) + 32 + sAmin + sAspan).
__device__ __forceinline__ void rc_window(const RowsConv &P, int it, int &t0, int &t1, int &Ra, int &nrows) {
    t0 = it * P.G;
    t1 = min(t0 + P.G, P.ntiles);
    const int w0 = t0 * P.T + P.smin + P.sAmin;
    const int w1 = (t1 - 1) * P.T + P.smin + 32 + P.sAmin + P.sAspan;
    Ra = w0 >= 0 ? w0 / P.Wg : -((-w0 + P.Wg - 1) / P.Wg);
    const int Rb = (w1 - 1) >= 0 ? (w1 - 1) / P.Wg : -((-(w1 - 1) + P.Wg - 1) / P.Wg);
    nrows = Rb - Ra + 1;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

struct RcOutS {   // shared-memory copy of RcOut
    int oy, ox, os, nblk, kind;
    int dcol[kRcMaxBlk], delta[kRcMaxBlk], xo[kRcMaxBlk];
};

// MMA issue.  The per-tile MMA program (NM tap groups x K k-steps) is the
// same for every tile except the A base and the accumulator slot, so it is
// unrolled at compile time: every MMA is two 32-bit adds on descriptor low
// words (start address field) and the UTCHMMA itself, all in uniform
// registers.  Descriptors: A = tile window + aoff[m] + 2*ks (32 bytes per
// k-step inside the swizzled row), B = packed slice + ks * 32 N bytes.
template <int NM, int KPC, int NCH>
__device__ __forceinline__ void rc_issue(uint32_t alo, uint32_t ahi, uint32_t dslot, const uint32_t (&aoff)[NM],
                                         const uint32_t (&blo)[NM], uint32_t bhi, const uint32_t (&bst)[NM],
                                         const uint32_t (&dcol)[NM], const uint32_t (&idesc)[NM], uint32_t zmask,
                                         uint32_t cstep) {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
#pragma unroll
        for (int ks = 0; ks < KPC * NCH; ++ks) {
            const uint64_t ad = ((uint64_t)ahi << 32) |
                                (uint64_t)(alo + aoff[m] + (uint32_t)(ks / KPC) * cstep + 2u * (uint32_t)(ks % KPC));
            const uint64_t bd = ((uint64_t)bhi << 32) | (uint64_t)(blo[m] + (uint32_t)ks * bst[m]);
            const uint32_t acc = (ks > 0 || !((zmask >> m) & 1u)) ? 1u : 0u;
            rows::mma_ss_elect(dslot + dcol[m], ad, bd, idesc[m], acc);
        }
    }
}

// Uniform program (every MMA has the same N, accumulator block and instruction
// descriptor; B slices laid out back to back): only the A offsets differ.
template <int NM, int KPC, int NCH>
__device__ __forceinline__ void rc_issue_u(uint32_t alo, uint32_t ahi, uint32_t dslot, const uint32_t (&aoff)[NM],
                                           uint32_t blo0, uint32_t bhi, uint32_t bst, uint32_t wst, uint32_t dcol,
                                           uint32_t idesc, uint32_t cstep) {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
#pragma unroll
        for (int ks = 0; ks < KPC * NCH; ++ks) {
            const uint64_t ad = ((uint64_t)ahi << 32) |
                                (uint64_t)(alo + aoff[m] + (uint32_t)(ks / KPC) * cstep + 2u * (uint32_t)(ks % KPC));
            const uint64_t bd = ((uint64_t)bhi << 32) | (uint64_t)(blo0 + (uint32_t)m * wst + (uint32_t)ks * bst);
            rows::mma_ss_elect(dslot + dcol, ad, bd, idesc, (m > 0 || ks > 0) ? 1u : 0u);
        }
    }
}

// Chunk-staged issue: the stage holds one source chunk (kpc k-steps) of the
// window; its B k-steps start at ks0; the very first MMA overwrites.
template <int NM, int KPC>
__device__ __forceinline__ void rc_issue_uc(uint32_t alo, uint32_t ahi, uint32_t dslot, const uint32_t (&aoff)[NM],
                                            uint32_t blo0, uint32_t bhi, uint32_t bst, uint32_t wst, uint32_t dcol,
                                            uint32_t idesc, uint32_t ks0, bool first) {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
#pragma unroll
        for (int kk = 0; kk < KPC; ++kk) {
            const uint64_t ad = ((uint64_t)ahi << 32) | (uint64_t)(alo + aoff[m] + 2u * (uint32_t)kk);
            const uint64_t bd = ((uint64_t)bhi << 32) | (uint64_t)(blo0 + (uint32_t)m * wst + (ks0 + (uint32_t)kk) * bst);
            rows::mma_ss_elect(dslot + dcol, ad, bd, idesc, (first && m == 0 && kk == 0) ? 0u : 1u);
        }
    }
}

template <int NM, int KPC, int NCH>
__device__ __forceinline__ void rc_mma_loop(const RowsConv &P, uint32_t stg0, uint32_t wsm, uint64_t *full,
                                            uint64_t *empty, uint64_t *accf, uint64_t *acce) {
    constexpr bool kU = NM == 9;       // uniform 3x3 program: compact state (see rc_issue_u)
    constexpr int NA = kU ? 1 : NM;
    uint32_t aoff[NM], blo[NA], bst[NA], dcol[NA], idesc[NA];
    uint32_t zmask = 0;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        const RcMma &M = P.mma[m];
        aoff[m] = ((uint32_t)M.pl * P.plane_bytes + (uint32_t)M.sig * P.pxS) >> 4;
        if (m < NA) {
            blo[m] = (uint32_t)smem_desc(wsm + M.woff, (uint32_t)M.N * 16u, 128u);
            bst[m] = (uint32_t)M.N * 2u;      // 32*N bytes per k-step, in 16-byte units
            dcol[m] = M.dcol;
            idesc[m] = M.idesc;
        }
        zmask |= (uint32_t)M.zero << m;
    }
    const uint32_t wst = (P.nmma > 1 ? (P.mma[1].woff - P.mma[0].woff) : 0u) >> 4;
    const uint32_t bhi = (uint32_t)(smem_desc(wsm, 16u, 128u) >> 32);
    const uint32_t sbo_a = 8u * (uint32_t)P.Ea * 2u;
    const int swz = 2 * P.Ea;
    const uint32_t tstep = ((uint32_t)P.T * P.pxS) >> 4;   // next tile of a pair: T pixels on
    const uint32_t cstep = P.chunk_bytes >> 4;               // next source chunk
    unsigned long long prof[4] = {0, 0, 0, 0};
    const unsigned long long cstart = kProbes ? clock64() : 0;
    int sb = 0, slot = 0;
    uint32_t ph = 0, aph = 0;
    if constexpr (kU && NCH > 1) {
        if (P.cstage) {
            // one chunk per stage, one tile per item: acquire the tile's slot,
            // then accumulate chunk by chunk as the stages arrive
            for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
                int t0, t1, Ra, nrows;
                rc_window(P, it, t0, t1, Ra, nrows);
                mbar_wait(acce + slot, aph ^ 1);
                fence_after_sync();
                const int v0 = t0 * P.T + P.smin;
                const uint32_t dslot = (uint32_t)slot * P.ND;
                for (int ci = 0; ci < NCH; ++ci) {
                    mbar_wait(full + sb, ph);
                    fence_after_sync();
                    const uint32_t stg = stg0 + (uint32_t)sb * P.stage_bytes;
                    const uint64_t at =
                        rows::sdesc(stg + (uint32_t)(v0 + P.sAmin - Ra * P.Wg) * P.pxS, 16u, sbo_a, swz);
                    rc_issue_uc<NM, KPC>((uint32_t)at, (uint32_t)(at >> 32), dslot, aoff, blo[0], bhi, bst[0], wst,
                                         dcol[0], idesc[0], (uint32_t)(ci * KPC), ci == 0);
                    if (elect_one()) mma_commit(empty + sb);
                    __syncwarp();
                    if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                }
                if (elect_one()) mma_commit(accf + slot);
                __syncwarp();
                if (++slot == P.nacc) { slot = 0; aph ^= 1; }
            }
            return;
        }
    }
    for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
        int t0, t1, Ra, nrows;
        rc_window(P, it, t0, t1, Ra, nrows);
        unsigned long long c0 = kProbes ? clock64() : 0;
        mbar_wait(full + sb, ph);
        fence_after_sync();
        if (kProbes && P.prof) { const unsigned long long c1 = clock64(); prof[0] += c1 - c0; c0 = c1; }
        const uint32_t stg = stg0 + (uint32_t)sb * P.stage_bytes;
        for (int t = t0; t < t1;) {
            // two tiles at a time when there are four accumulator slots: their
            // MMA chains interleave, hiding each chain's fill / drain latency
            const bool two = P.pair && t + 1 < t1;
            const int slot2 = slot + 1 == P.nacc ? 0 : slot + 1;
            const uint32_t aph2 = slot + 1 == P.nacc ? (aph ^ 1u) : aph;
            if (!(kProbes && (P.dbg & 16))) {
                mbar_wait(acce + slot, aph ^ 1);
                if (two) mbar_wait(acce + slot2, aph2 ^ 1);
            }
            fence_after_sync();
            if (kProbes && P.prof) { const unsigned long long c1 = clock64(); prof[1] += c1 - c0; c0 = c1; }
            const int v0 = t * P.T + P.smin;
            const uint64_t at = rows::sdesc(stg + (uint32_t)(v0 + P.sAmin - Ra * P.Wg) * P.pxS, 16u, sbo_a, swz);
            const uint32_t alo = (uint32_t)at, ahi = (uint32_t)(at >> 32);
            if (!(kProbes && (P.dbg & 1))) {
                if constexpr (kU) {
                    rc_issue_u<NM, KPC, NCH>(alo, ahi, (uint32_t)slot * P.ND, aoff, blo[0], bhi, bst[0], wst, dcol[0],
                                             idesc[0], cstep);
                    if (two)
                        rc_issue_u<NM, KPC, NCH>(alo + tstep, ahi, (uint32_t)slot2 * P.ND, aoff, blo[0], bhi, bst[0],
                                                 wst, dcol[0], idesc[0], cstep);
                } else {
                    rc_issue<NM, KPC, NCH>(alo, ahi, (uint32_t)slot * P.ND, aoff, blo, bhi, bst, dcol, idesc, zmask,
                                           cstep);
                    if (two)
                        rc_issue<NM, KPC, NCH>(alo + tstep, ahi, (uint32_t)slot2 * P.ND, aoff, blo, bhi, bst, dcol,
                                               idesc, zmask, cstep);
                }
            }
            if (kProbes && P.prof) { const unsigned long long c1 = clock64(); prof[2] += c1 - c0; c0 = c1; }
            if (elect_one()) {
                mma_commit(accf + slot);
                if (two) mma_commit(accf + slot2);
            }
            __syncwarp();
            if (kProbes && P.prof) { const unsigned long long c1 = clock64(); prof[3] += c1 - c0; c0 = c1; }
            if (two) {
                t += 2;
                slot = slot2 + 1 == P.nacc ? 0 : slot2 + 1;
                aph = slot2 + 1 == P.nacc ? (aph2 ^ 1u) : aph2;
            } else {
                t += 1;
                slot = slot2;
                aph = aph2;
            }
        }
        if (elect_one()) mma_commit(empty + sb);
        __syncwarp();
        if (++sb == P.nstg) { sb = 0; ph ^= 1; }
    }
    if (kProbes && P.prof && threadIdx.x % 32 == 0) {
        unsigned long long *o = P.prof + (size_t)blockIdx.x * 8;
        o[0] = prof[0]; o[1] = prof[1]; o[2] = prof[2]; o[3] = prof[3]; o[4] = clock64() - cstart;
    }
}

// Epilogue of one output (phase) of a tile: TMEM -> registers -> column-tap
// shift-sum -> bf16 capsule rows.  Block j of the output (NB blocks, lane
// offset DL_j = D0 + DS*j, compile-time) is added at row R + DL_j: a shuffle
// down inside the TMEM lane quarter; the top DL_j lanes take the first DL_j
// rows of the next quarter, which that quarter's warp leaves in the group's
// hand-off buffer (lanes [XO_j, XO_j + DL_j) of its quarter row).
template <int NB, int D0, int DS>
__device__ __forceinline__ void rc_epi_out(const RowsConv &P, const RcOutS &O, uint32_t tbase, bool ok,
                                           __nv_bfloat16 *dst, float *xb, int q, int lane, int grp, int c_lo,
                                           int c_hi, uint32_t &par) {
    constexpr bool kHand = (D0 > 0) || (DS > 0 && NB > 1) || (DS < 0 && D0 + DS * (NB - 1) > 0);
    const int xl = P.xl;
    (void)par;
    for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
        uint32_t v[NB][16];
#pragma unroll
        for (int j = 0; j < NB; ++j) rows::tmem_ld16x(tbase + (uint32_t)(O.dcol[j] + c0), v[j]);
        tmem_wait_ld();
        float acc[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = 0.f;
        int xo = 0;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int dl = D0 + DS * j;
            if (dl == 0) {
#pragma unroll
                for (int c = 0; c < 16; ++c) acc[c] += __uint_as_float(v[j][c]);
            } else {
                const float fm = lane + dl < 32 ? 1.f : 0.f;
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    acc[c] = fmaf(__uint_as_float(__shfl_down_sync(0xffffffffu, v[j][c], dl)), fm, acc[c]);
                if (q > 0 && lane < dl) {
                    uint4 *w = reinterpret_cast<uint4 *>(xb + ((size_t)q * xl + xo + lane) * 16);
#pragma unroll
                    for (int c = 0; c < 4; ++c) w[c] = make_uint4(v[j][4 * c], v[j][4 * c + 1], v[j][4 * c + 2], v[j][4 * c + 3]);
                }
                xo += dl;
            }
        }
        if (kHand && !(kProbes && (P.dbg & 32))) {
            named_bar(1 + grp, 128);
            if (q < 3) {
                int xo2 = 0;
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    const int dl = D0 + DS * j;
                    if (dl > 0) {
                        if (lane >= 32 - dl) {
                            const float4 *rd = reinterpret_cast<const float4 *>(
                                xb + ((size_t)(q + 1) * xl + xo2 + (lane - (32 - dl))) * 16);
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const float4 x4 = rd[c];
                                acc[4 * c] += x4.x; acc[4 * c + 1] += x4.y; acc[4 * c + 2] += x4.z; acc[4 * c + 3] += x4.w;
                            }
                        }
                        xo2 += dl;
                    }
                }
            }
            named_bar(1 + grp, 128);
        }
        if (ok) {
            uint32_t w[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * c], acc[2 * c + 1]);
                w[c] = *reinterpret_cast<uint32_t *>(&h);
            }
            uint4 *d4 = reinterpret_cast<uint4 *>(dst + c0);
            d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
            d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
    }
}

// Epilogue warps.  Group grp (four warps, one per TMEM lane quarter) owns
// accumulator slot grp % nacc and, when two groups share a slot, one half of
// its column passes.  A group walks only its own tiles: tile k of this CTA
// lands in slot k % nacc, so the group's tiles are k = slot, slot + nacc, ...
// (item i = k / G, tile i*gridDim.x*G + k % G), kept with counters.
// Single unshifted block (no column-tap stacking): 32 columns (one 64-byte
// piece of every capsule row) per pass, straight to bf16.  With a per-warp
// staging buffer the warp writes its 32 rows through shared memory so that
// every global store instruction covers 512 contiguous bytes (rows are
// consecutive capsule rows): lane l writes row 8i + l/4, piece l%4.  Without
// it each lane stores its own row (32 rows per instruction).
__device__ __forceinline__ void rc_epi_plain(const RcOutS &O, uint32_t tbase, bool ok, __nv_bfloat16 *dst, int c_lo,
                                             int c_hi, int dbg, uint32_t sbuf, int lane) {
    for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
        uint32_t v[32];
        rows::tmem_ld16x(tbase + (uint32_t)(O.dcol[0] + c0), *reinterpret_cast<uint32_t(*)[16]>(v));
        rows::tmem_ld16x(tbase + (uint32_t)(O.dcol[0] + c0 + 16), *reinterpret_cast<uint32_t(*)[16]>(v + 16));
        tmem_wait_ld();
        if (kProbes && (dbg & 128)) ok = ok && __uint_as_float(v[0]) == 1.2345f;   // probe: no stores
        uint32_t w[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1]));
            w[c] = *reinterpret_cast<uint32_t *>(&h);
        }
        if (sbuf) {
            // stage: row `lane` at lane*64, pieces rotated by lane/2 (conflict-free)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int c = (i + (lane >> 1)) & 3;
                const uint32_t a = sbuf + (uint32_t)lane * 64u + (uint32_t)c * 16u;
                uint32_t x0 = 0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc)
                    if (cc == c) { x0 = w[4 * cc]; x1 = w[4 * cc + 1]; x2 = w[4 * cc + 2]; x3 = w[4 * cc + 3]; }
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(x0), "r"(x1), "r"(x2), "r"(x3)
                             : "memory");
            }
            __syncwarp();
            const unsigned long long my = reinterpret_cast<unsigned long long>(dst + c0);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = 8 * i + (lane >> 2);
                const unsigned long long ra = __shfl_sync(0xffffffffu, my, r);
                const int rok = __shfl_sync(0xffffffffu, ok ? 1 : 0, r);
                const uint4 x = ld_shared_v4(sbuf + (uint32_t)i * 512u + (uint32_t)lane * 16u);
                if (rok) reinterpret_cast<uint4 *>(ra)[lane & 3] = x;
            }
            __syncwarp();
        } else if (ok) {
            uint4 *d4 = reinterpret_cast<uint4 *>(dst + c0);
#pragma unroll
            for (int g = 0; g < 4; ++g) d4[g] = make_uint4(w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
        }
    }
}

template <int NBX>
__device__ __forceinline__ void rc_epi_dispatch(const RowsConv &P, const RcOutS &O, uint32_t tbase, bool ok,
                                                __nv_bfloat16 *dst, float *xb, int q, int lane, int grp, int c_lo,
                                                int c_hi, uint32_t &par, uint32_t sbuf) {
    if (O.kind == 0 || !kProbes) {   // stacked epilogues exist in probe builds only (CAPSCONV_RC_GQ)
        rc_epi_plain(O, tbase, ok, dst, c_lo, c_hi, P.dbg, sbuf, lane);
        return;
    }
    if constexpr (kProbes) {
        switch (O.kind) {
            case 1: rc_epi_out<2, 0, 4>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
            case 2: rc_epi_out<3, 0, 4>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
            case 3: rc_epi_out<4, 0, 4>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
            case 4: rc_epi_out<2, 4, -4>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
            case 5: rc_epi_out<3, 8, -4>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
            case 6: rc_epi_out<1, 4, 0>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
            default: rc_epi_out<1, 8, 0>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par); break;
        }
    }
}

__device__ __forceinline__ void rc_epilogue(const RowsConv &P, float *xbuf, const RcOutS *ot, uint64_t *accf,
                                            uint64_t *acce, int warp, int lane) {
    const int grp = warp >> 2, q = warp & 3;
    const int nacc = P.nacc, G = P.G, ntiles = P.ntiles, n_items = P.n_items, T = P.T;
    // ngrp <= nacc: group g owns slots g, g + ngrp, ... and takes the tiles
    // k = g (mod ngrp); ngrp = 2*nacc: two groups share slot g % nacc and split
    // its columns, taking the tiles k = g (mod nacc)
    if (grp >= P.ngrp) return;
    const bool split = P.ngrp > nacc;
    const int kstep = split ? nacc : P.ngrp;
    const int part = split ? grp / nacc : 0;
    const int cspan = split ? P.Eout / 2 : P.Eout, c_lo = part * cspan, c_hi = c_lo + cspan;
    const int R = q * 32 + lane, px = R >> 2, d1 = R & 3;
    float *xb = xbuf + (size_t)grp * 4 * P.xl * 16;
    // per-warp 2 KB staging buffer for coalesced stores (0: store directly)
    const uint32_t sbuf = P.soff ? (((smem_u32(xbuf) - P.xoff) + P.soff) + (uint32_t)warp * 2048u) : 0u;
    uint32_t par = 0;                           // hand-off buffer parity (per group, across tiles)
    const uint32_t hw = (uint32_t)(P.Hg * P.Wg), Wg = (uint32_t)P.Wg;
    const int Bn = P.Bn, Hout = P.Hout, Wout = P.Wout, Eout = P.Eout, nout = P.nout;
    const uint32_t ND = P.ND;
    __nv_bfloat16 *const out = P.out;
    int slot = split ? grp % nacc : grp;        // tile k of this CTA lands in slot k % nacc
    int i = 0, r = slot;                        // k = i*G + r
    while (r >= G) { r -= G; ++i; }
    uint32_t aph = 0;
    for (;;) {
        const int it = blockIdx.x + i * (int)gridDim.x;
        if (it >= n_items) break;
        const int t = it * G + r;
        if (t >= ntiles) break;
        const unsigned long long e0 = kProbes ? clock64() : 0;
        mbar_wait(accf + slot, aph);
        const unsigned long long e1 = kProbes ? clock64() : 0;
        fence_after_sync();
        const uint32_t tbase = ((uint32_t)(q * 32) << 16) + (uint32_t)slot * ND;
        if (!(kProbes && (P.dbg & 4))) {
            const uint32_t u = (uint32_t)(t * T + px);
            const uint32_t img = P.fd_hw.div(u), rr = u - img * hw;
            const uint32_t Y = P.fd_wg.div(rr), X = rr - Y * Wg;
            const bool valid = px < T && (int)img < Bn;
            for (int o = 0; o < nout; ++o) {
                const RcOutS &O = ot[o];
                const int oy = O.os * (int)Y + O.oy, ox = O.os * (int)X + O.ox;
                const bool ok = valid && oy < Hout && ox < Wout;
                __nv_bfloat16 *dst = out + ((((size_t)img * Hout + oy) * Wout + ox) * 4 + d1) * (size_t)Eout;
                rc_epi_dispatch<0>(P, O, tbase, ok, dst, xb, q, lane, grp, c_lo, c_hi, par, sbuf);
            }
        }
        fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(acce + slot);
        if (kProbes && P.prof && warp == 0 && lane == 0) {
            unsigned long long *o = P.prof + (size_t)blockIdx.x * 8;
            o[5] += e1 - e0;
            o[6] += clock64() - e1;
            o[7] += 1;
        }
        slot += kstep;
        while (slot >= nacc) { slot -= nacc; aph ^= 1; }
        r += kstep;
        while (r >= G) { r -= G; ++i; }
    }
}

__global__ void __launch_bounds__(kRcThreads, 1) rows_conv_kernel(const __grid_constant__ RowsConv P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *full = bars, *empty = bars + 4, *accf = bars + 8, *acce = bars + 24, *wbar = bars + 40;   // up to 16 slots
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + 512);
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t wsm = base + P.woff_s, stg0 = base + P.stg_off;
    float *xbuf = reinterpret_cast<float *>(smem_raw + (base - smem_u32(smem_raw)) + P.xoff);
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P.nstg; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < P.nacc; ++i) {
            mbar_init(accf + i, 1);
            mbar_init(acce + i, P.ngrp > P.nacc ? 8 : 4);
        }
        mbar_init(wbar, 1);
        mbar_fence_init();
    }
    // warp roles: 0 .. 4*kRcGroups-1 epilogue, then MMA, then TMA -- the
    // scheduler favours higher warp ids, so the issue warps win every slot
    constexpr int kMmaWarp = 4 * kRcGroups, kTmaWarp = kMmaWarp + 1;
    if (warp == kMmaWarp) tmem_alloc_dyn(tmem_slot, 512);
    if (threadIdx.x < (unsigned)P.nout) {
        // the epilogue's output table, read from shared memory in the hot loop
        RcOutS *os = reinterpret_cast<RcOutS *>(smem_raw + 640) + threadIdx.x;
        const RcOut &O = P.outp[threadIdx.x];
        os->oy = O.oy; os->ox = O.ox; os->os = O.os; os->nblk = O.nblk; os->kind = O.kind;
        for (int j = 0; j < kRcMaxBlk; ++j) { os->dcol[j] = O.dcol[j]; os->delta[j] = O.delta[j]; os->xo[j] = O.xo[j]; }
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (*tmem_slot != 0u) __trap();
    pdl_wait();   // the previous grid's writes (source, weights) are visible from here on
    // The packed weights are the only workspace bytes this kernel reads: once
    // they are in shared memory the next kernel may launch (PDL) -- e.g. the
    // next call's weight pack, which rewrites the workspace.
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(wbar, P.wbytes);
        for (uint32_t o = 0; o < P.wbytes; o += 32768u) {
            const uint32_t n = min(32768u, P.wbytes - o);
            bulk_g2s_u32(wsm + o, P.wpack + o, n, wbar);
        }
    }
    mbar_wait(wbar, 0);
    pdl_launch_dependents();

    if (warp == kTmaWarp) {
        // ------------------------------------------------------------ TMA
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmS)) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmH)) : "memory");
            int sb = 0;
            uint32_t ph = 0;
            for (int it = blockIdx.x; it < P.n_items; it += gridDim.x) {
                int t0, t1, Ra, nrows;
                rc_window(P, it, t0, t1, Ra, nrows);
                if (P.cstage) {
                    // one stage per source chunk (rows of the window, this chunk's columns)
                    const uint32_t rowb = (uint32_t)P.Wg * P.pxS;
                    for (int ci = 0; ci < P.nch; ++ci) {
                        mbar_wait(empty + sb, ph ^ 1);
                        const uint32_t stg = stg0 + (uint32_t)sb * P.stage_bytes;
                        const uint32_t mb = smem_u32(full + sb);
                        mbar_arrive_expect_tx(full + sb, (uint32_t)(nrows * P.npl) * rowb);
                        int r = 0;
                        while (r < nrows) {
                            const int R = Ra + r;
                            const int img = R >= 0 ? R / P.Hg : -((-R + P.Hg - 1) / P.Hg);
                            const int Y = R - img * P.Hg;
                            const int len = min(P.Hg - Y, nrows - r);
                            int k = 0;
                            for (; k + P.hb <= len; k += P.hb)
                                for (int pl = 0; pl < P.npl; ++pl)
                                    rows::tma_load5d(stg + (uint32_t)pl * P.plane_bytes + (uint32_t)(r + k) * rowb,
                                                     &P.tmH, ci * P.Ea, 0, P.pl_ox[pl], P.es * (Y + k) + P.pl_oy[pl],
                                                     img, mb);
                            for (; k < len; ++k)
                                for (int pl = 0; pl < P.npl; ++pl)
                                    rows::tma_load5d(stg + (uint32_t)pl * P.plane_bytes + (uint32_t)(r + k) * rowb,
                                                     &P.tmS, ci * P.Ea, 0, P.pl_ox[pl], P.es * (Y + k) + P.pl_oy[pl],
                                                     img, mb);
                            r += len;
                        }
                        if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                    }
                    continue;
                }
                mbar_wait(empty + sb, ph ^ 1);
                if (kProbes && (P.dbg & 2)) {
                    mbar_arrive(full + sb);
                    if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                    continue;
                }
                const uint32_t stg = stg0 + (uint32_t)sb * P.stage_bytes;
                const uint32_t rowb = (uint32_t)P.Wg * P.pxS;
                const uint32_t mb = smem_u32(full + sb);
                auto dst = [&](int ci, int pl, int r) {
                    return stg + (uint32_t)ci * P.chunk_bytes + (uint32_t)pl * P.plane_bytes + (uint32_t)r * rowb;
                };
                if (P.merged) {
                    // one box per hb virtual rows (the last may overshoot into the stage's slack rows)
                    const int nbox = (nrows + P.hb - 1) / P.hb;
                    mbar_arrive_expect_tx(full + sb, (uint32_t)(nbox * P.hb * P.npl * P.nch) * rowb);
                    for (int r = 0; r < nrows; r += P.hb)
                        for (int ci = 0; ci < P.nch; ++ci)
                            for (int pl = 0; pl < P.npl; ++pl)
                                rows::tma_load4d_rows(dst(ci, pl, r), &P.tmH, ci * P.Ea, 0, P.pl_ox[pl],
                                                      P.es * (Ra + r) + P.pl_oy[pl], mb);
                } else {
                    // per image segment: hb-row boxes, then single rows (never past the image)
                    mbar_arrive_expect_tx(full + sb, (uint32_t)(nrows * P.npl * P.nch) * rowb);
                    int r = 0;
                    while (r < nrows) {
                        const int R = Ra + r;
                        const int img = R >= 0 ? R / P.Hg : -((-R + P.Hg - 1) / P.Hg);
                        const int Y = R - img * P.Hg;
                        const int len = min(P.Hg - Y, nrows - r);
                        int k = 0;
                        for (; k + P.hb <= len; k += P.hb)
                            for (int ci = 0; ci < P.nch; ++ci)
                                for (int pl = 0; pl < P.npl; ++pl)
                                    rows::tma_load5d(dst(ci, pl, r + k), &P.tmH, ci * P.Ea, 0, P.pl_ox[pl],
                                                     P.es * (Y + k) + P.pl_oy[pl], img, mb);
                        for (; k < len; ++k)
                            for (int ci = 0; ci < P.nch; ++ci)
                                for (int pl = 0; pl < P.npl; ++pl)
                                    rows::tma_load5d(dst(ci, pl, r + k), &P.tmS, ci * P.Ea, 0, P.pl_ox[pl],
                                                     P.es * (Y + k) + P.pl_oy[pl], img, mb);
                        r += len;
                    }
                }
                if (++sb == P.nstg) { sb = 0; ph ^= 1; }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA
        mbar_wait(wbar, 0);
        switch (P.prog) {
            case 0: rc_mma_loop<9, 2, 1>(P, stg0, wsm, full, empty, accf, acce); break;     // 3x3, C*D2 = 32
            case 1: rc_mma_loop<9, 4, 1>(P, stg0, wsm, full, empty, accf, acce); break;     // 3x3, 64
            case 2: rc_mma_loop<9, 4, 2>(P, stg0, wsm, full, empty, accf, acce); break;     // 3x3, 128
            case 3: rc_mma_loop<9, 2, 2>(P, stg0, wsm, full, empty, accf, acce); break;     // 3x3, 2 x 32
            case 4: rc_mma_loop<6, 4, 1>(P, stg0, wsm, full, empty, accf, acce); break;     // 3x3 s2 dI, 64
            case 5: rc_mma_loop<6, 2, 1>(P, stg0, wsm, full, empty, accf, acce); break;     // 3x3 s2 dI, 32
            default:
                if constexpr (kProbes) {   // stacked programs (probe builds, CAPSCONV_RC_GQ)
                    switch (P.prog) {
                        case 6: rc_mma_loop<3, 2, 1>(P, stg0, wsm, full, empty, accf, acce); break;
                        case 7: rc_mma_loop<3, 4, 1>(P, stg0, wsm, full, empty, accf, acce); break;
                        default: break;
                    }
                }
                break;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        rc_epilogue(P, xbuf, reinterpret_cast<const RcOutS *>(smem_raw + 640), accf, acce, warp, lane);
    }
    fence_before_sync();
    __syncthreads();
    if (warp == kMmaWarp) tmem_dealloc_dyn(0u, 512);
}

// ---------------------------------------------------------------- weight packing
struct RcPackMma {
    uint32_t woff;
    int N, nblk, tp[kRcMaxBlk], tq[kRcMaxBlk];
};
struct RcPackArgs {
    const __nv_bfloat16 *K;
    uint8_t *dst;
    int KW, C, Cout, ES, Eblk, dgrad, nmma;
    RcPackMma m[kRcMaxMma];
    uint32_t total16;   // 16-byte units
};

// One thread per 16-byte unit (8 consecutive k of one row n) of the K-major
// no-swizzle image: unit (k/8, n) of slice m at woff + (k/8)*N*16 + n*16.
__device__ __forceinline__ void rc_pack_unit(const RcPackArgs &A, uint32_t g) {
    int m = 0;
    while (m + 1 < A.nmma && A.m[m + 1].woff / 16 <= g) ++m;
    const RcPackMma &M = A.m[m];
    const uint32_t loc = g - M.woff / 16;
    const int kc = (int)(loc / (uint32_t)M.N), n = (int)(loc - (uint32_t)kc * M.N);
    const int blk = n / A.Eblk, r = n - blk * A.Eblk;
    const int p = blk < M.nblk ? M.tp[blk] : -1, qq = blk < M.nblk ? M.tq[blk] : -1;
    uint32_t w[4] = {0, 0, 0, 0};
    if (p >= 0) {
        __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = kc * 8 + e;
            int c, co, d2, d3;
            if (!A.dgrad) { c = k >> 2; d2 = k & 3; co = r >> 2; d3 = r & 3; }
            else { co = k >> 2; d3 = k & 3; c = r >> 2; d2 = r & 3; }
            v[e] = A.K[((((size_t)(p * A.KW + qq) * A.C + c) * A.Cout + co) * 4 + d2) * 4 + d3];
        }
        memcpy(w, v, 16);
    }
    reinterpret_cast<uint4 *>(A.dst)[g] = make_uint4(w[0], w[1], w[2], w[3]);
}

// The pack reads only K and writes only the workspace, which the previous
// libcapsconv kernel no longer reads once it has triggered its dependents
// (rows_walk / rows_conv: after their weights landed in shared memory; every
// other kernel: at completion): so it runs alongside that kernel's tail (64-
// thread blocks fit next to a resident conv CTA), and waits for the previous
// grid only before it exits, so that its own completion keeps stream order.
__global__ void __launch_bounds__(64) rc_pack_kernel(const __grid_constant__ RcPackArgs A) {
    pdl_launch_dependents();
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < A.total16) rc_pack_unit(A, g);
    pdl_wait();
}

struct RcPlan {
    bool ok = false;
    RowsConv P;
    RcPackArgs pack;
    size_t ws_bytes = 0;
};

int rc_chunk(int E) { return E % 64 == 0 ? 64 : E % 32 == 0 ? 32 : E % 16 == 0 ? 16 : 0; }

RcPlan make_rc_plan(const Problem &p, bool dgrad) {
    RcPlan pl;
    RowsConv &P = pl.P;
    memset(&P, 0, sizeof(P));
    memset(&pl.pack, 0, sizeof(pl.pack));
    if (p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4 || p.pad != 0) return pl;
    if (p.s > 2 || p.B > (1 << 20)) return pl;
    const int s = (int)p.s, KH = (int)p.KH, KW = (int)p.KW;
    if (KH * KW > 64) return pl;
    const int EI = 4 * (int)p.C, EO = 4 * (int)p.Cout;
    const int ES = dgrad ? EO : EI;      // source (K dimension) elements per capsule row
    const int EN = dgrad ? EI : EO;      // output elements per capsule row (one stacked block)
    const int Ea = rc_chunk(ES);
    if (!Ea || EN % 32 != 0 || EN > 256) return pl;
    if (dgrad && (KH < s || KW < s)) return pl;   // every output phase needs a tap
    P.dgrad = dgrad ? 1 : 0;
    P.Ea = Ea;
    P.nch = ES / Ea;
    P.kpc = Ea / 16;
    P.pxS = 4u * Ea * 2u;
    P.Bn = (int)p.B;
    P.es = s;
    P.Hg = (int)((p.H + s - 1) / s);
    P.Wg = (int)((p.W + s - 1) / s);
    if (P.Wg * s > 256) return pl;
    if ((long long)P.Bn * P.Hg * P.Wg > (1ll << 30)) return pl;
    P.Eout = EN;
    P.Hout = dgrad ? (int)p.H : (int)p.Ho;
    P.Wout = dgrad ? (int)p.W : (int)p.Wo;
    auto nqq = [&](int b) { return b < KW ? (KW - b + s - 1) / s : 0; };
    auto npp = [&](int a) { return a < KH ? (KH - a + s - 1) / s : 0; };
    // stacking depth: as many column taps per MMA as fit N <= 256
    // Column-tap stacking depth.  Stacking widens N (cheaper MMAs) but moves the
    // tap sum into the epilogue (shuffles + a cross-quarter hand-off); on the
    // config-5 layers the unstacked form measured faster end to end
    // (tests/probe/time_layers.py: L1 fwd 93 vs 116 us), so it is the default.
    int Gq_cap = 1;
    if (probe_env("CAPSCONV_RC_GQ")) Gq_cap = std::max(1, std::min(256 / EN, atoi(probe_env("CAPSCONV_RC_GQ"))));
    std::vector<RcMma> ml;
    std::vector<RcOut> ol;
    uint32_t woff = 0;
    auto add_mma = [&](int pln, int sig, int N, int dcol, int zero, int nblk, const int *tp, const int *tq) {
        RcMma M{};
        M.pl = pln; M.sig = sig; M.N = N; M.dcol = (uint32_t)dcol; M.zero = zero;
        M.idesc = idesc_bf16(128, N, 0, 0);
        M.woff = woff;
        woff += (uint32_t)N * (uint32_t)ES * 2u;
        M.nblk = nblk;
        for (int i = 0; i < nblk; ++i) { M.tp[i] = tp[i]; M.tq[i] = tq[i]; }
        ml.push_back(M);
    };
    int ND = 0;
    if (!dgrad) {
        // planes (a, b); D blocks j = stacked qq (shift +j)
        P.npl = 0;
        int plid[2][2];
        for (int a = 0; a < s && a < KH; ++a)
            for (int b = 0; b < s && b < KW; ++b) {
                plid[a][b] = P.npl;
                P.pl_oy[P.npl] = a;
                P.pl_ox[P.npl] = b;
                ++P.npl;
            }
        const int Gq = std::min(Gq_cap, nqq(0));
        ND = Gq * EN;
        bool first = true;
        for (int a = 0; a < s && a < KH; ++a)
            for (int b = 0; b < s && b < KW; ++b)
                for (int pp = 0; pp < npp(a); ++pp)
                    for (int q0 = 0; q0 < nqq(b); q0 += Gq) {
                        const int nj = std::min(Gq, nqq(b) - q0);
                        int tp[kRcMaxBlk], tq[kRcMaxBlk];
                        for (int j = 0; j < nj; ++j) { tp[j] = s * pp + a; tq[j] = s * (q0 + j) + b; }
                        add_mma(plid[a][b], pp * P.Wg + q0, nj * EN, 0, first && nj == Gq ? 1 : 0, nj, tp, tq);
                        first = first && !(nj == Gq);
                    }
        RcOut O{};
        O.oy = 0; O.ox = 0; O.os = 1; O.nblk = Gq;
        for (int j = 0; j < Gq; ++j) { O.dcol[j] = j * EN; O.delta[j] = 4 * j; }
        ol.push_back(O);
        P.smin = 0;
        P.T = 32 - (Gq - 1);
    } else {
        // one source plane (dO in the phase grid); output phases (a, b); per a one D
        // region holding the blocks (b, j) (shift -j), stacked in N when they fit
        P.npl = 1;
        P.pl_oy[0] = 0; P.pl_ox[0] = 0;
        P.es = 1;
        int Gq = std::min(Gq_cap, std::max(nqq(0), nqq(1 % s)));
        int span = 0;
        for (int b = 0; b < s; ++b) span += std::min(Gq, nqq(b));
        while (span * EN > 256 && Gq > 1) {
            --Gq;
            span = 0;
            for (int b = 0; b < s; ++b) span += std::min(Gq, nqq(b));
        }
        int region = 0;
        for (int a = 0; a < s && a < KH; ++a) {
            int boff[2] = {0, 0}, gqb[2] = {0, 0}, acc = 0;
            for (int b = 0; b < s; ++b) { gqb[b] = std::min(Gq, nqq(b)); boff[b] = acc; acc += gqb[b]; }
            const int rcols = acc * EN;
            for (int pp = 0; pp < npp(a); ++pp) {
                // chunk 0: every b stacked in one MMA over the whole region
                {
                    int tp[kRcMaxBlk], tq[kRcMaxBlk], nb = 0;
                    for (int b = 0; b < s; ++b)
                        for (int j = 0; j < gqb[b]; ++j) { tp[nb] = s * pp + a; tq[nb] = s * j + b; ++nb; }
                    if (nb > kRcMaxBlk) return pl;
                    add_mma(0, -(pp * P.Wg), nb * EN, region, pp == 0 ? 1 : 0, nb, tp, tq);
                }
                // later chunks (taps beyond the stacking depth): one MMA per b
                for (int b = 0; b < s; ++b)
                    for (int q0 = Gq; q0 < nqq(b); q0 += Gq) {
                        const int nj = std::min(Gq, nqq(b) - q0);
                        int tp[kRcMaxBlk], tq[kRcMaxBlk];
                        for (int j = 0; j < nj; ++j) { tp[j] = s * pp + a; tq[j] = s * (q0 + j) + b; }
                        add_mma(0, -(pp * P.Wg + q0), nj * EN, region + boff[b] * EN, 0, nj, tp, tq);
                    }
            }
            for (int b = 0; b < s && b < (int)p.W; ++b) {
                if (gqb[b] == 0) continue;
                RcOut O{};
                O.oy = a; O.ox = b; O.os = s; O.nblk = gqb[b];
                for (int j = 0; j < gqb[b]; ++j) { O.dcol[j] = region + (boff[b] + j) * EN; O.delta[j] = 4 * (Gq - 1 - j); }
                ol.push_back(O);
            }
            region += rcols;
        }
        ND = region;
        // shifts of block j are -j: sigma_min = -(Gq - 1); delta_j = 4*(sigma_j - sigma_min)
        P.smin = -(Gq - 1);
        P.T = 32 - (Gq - 1);
    }
    P.fd_hw.init((uint32_t)(P.Hg * P.Wg));
    P.fd_wg.init((uint32_t)P.Wg);
    if ((int)ml.size() > 9 || (int)ol.size() > kRcMaxOut || ND > 256 || ND % 16 != 0) return pl;
    // A shifts relative to the smallest
    int smn = 1 << 30, smx = -(1 << 30);
    for (auto &M : ml) { smn = std::min(smn, M.sig); smx = std::max(smx, M.sig); }
    for (auto &M : ml) M.sig -= smn;
    P.sAmin = smn;
    P.sAspan = smx - smn;
    P.nmma = (int)ml.size();
    for (int i = 0; i < P.nmma; ++i) P.mma[i] = ml[i];
    {
        // the issue loop is compiled per (tap groups, k-steps) with one source chunk
        static const int progs[][3] = {{9, 2, 1}, {9, 4, 1}, {9, 4, 2}, {9, 2, 2},
                                       {6, 4, 1}, {6, 2, 1}, {3, 2, 1}, {3, 4, 1}};
        P.prog = -1;
        for (int i = 0; i < (kProbes ? 8 : 6); ++i)
            if (progs[i][0] == P.nmma && progs[i][1] == P.kpc && progs[i][2] == P.nch) P.prog = i;
        if (P.prog < 0) return pl;
        if (P.nmma == 9) {   // the compact issue path needs a uniform program
            for (int i = 0; i < 9; ++i) {
                const RcMma &M = P.mma[i];
                if (M.N != P.mma[0].N || M.dcol != P.mma[0].dcol || M.idesc != P.mma[0].idesc ||
                    M.woff != P.mma[0].woff + (uint32_t)i * (P.mma[1].woff - P.mma[0].woff) || M.zero != (i == 0))
                    return pl;
            }
        }
    }
    P.nout = (int)ol.size();
    // epilogue instantiation per output: deltas 0,4,8,.. (fwd) / 4(n-1),..,4,0 (dI)
    for (auto &O : ol) {
        const int n = O.nblk;
        bool up = true, down = true;
        for (int j = 0; j < n; ++j) {
            up = up && O.delta[j] == 4 * j;
            down = down && O.delta[j] == 4 * (n - 1 - j);
        }
        if (up && n >= 1 && n <= 4) O.kind = n - 1;
        else if (down && n == 2) O.kind = 4;
        else if (down && n == 3) O.kind = 5;
        else if (n == 1 && O.delta[0] == 4) O.kind = 6;
        else if (n == 1 && O.delta[0] == 8) O.kind = 7;
        else return pl;
    }
    P.dmax = 0;
    P.xl = 0;
    for (int i = 0; i < P.nout; ++i) {
        int acc = 0;
        for (int j = 0; j < ol[i].nblk; ++j) {
            P.dmax = std::max(P.dmax, ol[i].delta[j]);
            ol[i].xo[j] = acc;
            acc += ol[i].delta[j];
        }
        P.xl = std::max(P.xl, acc);
        P.outp[i] = ol[i];
    }
    if (P.dmax > 12) return pl;
    P.ND = (uint32_t)ND;
    // accumulator slots; each slot belongs to one epilogue group (group = slot mod
    // ngrp), so a group never waits on a phase two ahead of its barrier
    // accumulator slots: as many as TMEM holds (up to 16), a multiple of the
    // epilogue groups when there are at least as many slots as groups
    P.nacc = std::min(16, 512 / ND);
    if (P.nacc < 2) return pl;
    if (P.nacc >= kRcGroups) P.nacc -= P.nacc % kRcGroups;
    // group g owns slot g % nacc; with two slots, two groups share each slot and
    // split its columns (when the columns split into 16-wide passes)
    P.ngrp = std::min(kRcGroups, P.nacc);
    if (P.nacc * 2 <= kRcGroups && (P.Eout / 2) % 32 == 0) P.ngrp = 2 * P.nacc;
    P.pair = P.nacc >= 4 ? 1 : 0;
    P.wbytes = woff;
    // shared memory: barriers 1 KB | hand-off (groups x 4 quarters x blocks x 12 lanes x 16 floats) | weights | stages
    // virtual rows map linearly onto source rows across images when the source
    // grid is the (phase of the) input itself: forward with H a multiple of s
    P.merged = (!dgrad && p.H % s == 0) ? 1 : 0;
    P.xoff = 1024;
    P.soff = (P.xoff + (uint32_t)kRcGroups * 4u * (uint32_t)P.xl * 16u * 4u + 1023u) & ~1023u;
    P.woff_s = P.soff + (uint32_t)kRcGroups * 4u * 2048u;
    P.stg_off = (P.woff_s + P.wbytes + 1023u) & ~1023u;
    const long long ntiles_ll = ((long long)P.Bn * P.Hg * P.Wg + P.T - 1) / P.T;
    P.ntiles = (int)ntiles_ll;
    const int nsm = device_info().num_sms;
    int bestG = 0, best_nstg = 0;
    uint32_t best_stage = 0;
    for (int nstg = 2; nstg >= 1 && !bestG; --nstg) {
        for (int G = 16; G >= 1; --G) {
            // at least ~2 items per SM when there are enough tiles
            if (G > 1 && (long long)P.ntiles < (long long)G * nsm * 2) continue;
            const int span_px = (G - 1) * P.T + 32 + P.sAspan;
            const int rows0 = span_px / P.Wg + 2;
            const int hb = std::max(1, std::min(rows0, std::min(16, 256 / P.es)));
            const int rows = P.merged ? (rows0 + hb - 1) / hb * hb : rows0;
            const uint32_t plane_b = (uint32_t)rows * P.Wg * P.pxS;
            const uint32_t chunk_b = plane_b * (uint32_t)P.npl;
            const uint32_t stage_b = ((chunk_b * (uint32_t)P.nch) + 1023u) & ~1023u;
            const uint64_t need = 1024ull + P.stg_off + (uint64_t)nstg * stage_b;
            if (need <= kRcSmemLimit && rows <= 256) {
                bestG = G; best_nstg = nstg; best_stage = stage_b;
                P.rows_max = rows;
                P.hb = hb;
                P.plane_bytes = plane_b;
                P.chunk_bytes = chunk_b;
                break;
            }
        }
    }
    if ((!bestG || best_nstg < 2) && P.soff) {
        // retry without the store staging buffers (double-buffered windows win)
        bestG = 0;
        P.woff_s = P.soff;
        P.soff = 0;
        P.stg_off = (P.woff_s + P.wbytes + 1023u) & ~1023u;
        for (int nstg = 2; nstg >= 1 && !bestG; --nstg) {
            for (int G = 16; G >= 1; --G) {
                if (G > 1 && (long long)P.ntiles < (long long)G * nsm * 2) continue;
                const int span_px = (G - 1) * P.T + 32 + P.sAspan;
                const int rows0 = span_px / P.Wg + 2;
                const int hb = std::max(1, std::min(rows0, std::min(16, 256 / P.es)));
                const int rows = P.merged ? (rows0 + hb - 1) / hb * hb : rows0;
                const uint32_t plane_b = (uint32_t)rows * P.Wg * P.pxS;
                const uint32_t chunk_b = plane_b * (uint32_t)P.npl;
                const uint32_t stage_b = ((chunk_b * (uint32_t)P.nch) + 1023u) & ~1023u;
                const uint64_t need = 1024ull + P.stg_off + (uint64_t)nstg * stage_b;
                if (need <= kRcSmemLimit && rows <= 256) {
                    bestG = G; best_nstg = nstg; best_stage = stage_b;
                    P.rows_max = rows;
                    P.hb = hb;
                    P.plane_bytes = plane_b;
                    P.chunk_bytes = chunk_b;
                    break;
                }
            }
        }
    }
    if ((!bestG || best_nstg < 2) && P.nch > 1 && !P.merged && P.nmma == 9) {
        // wide K (several source chunks): stage one chunk at a time, one tile per item
        const int span_px = 32 + P.sAspan;
        const int rows = span_px / P.Wg + 2;
        const uint32_t plane_b = (uint32_t)rows * P.Wg * P.pxS;
        const uint32_t stage_b = ((plane_b * (uint32_t)P.npl) + 1023u) & ~1023u;
        for (int nstg = 4; nstg >= 2; --nstg)
            if (1024ull + P.stg_off + (uint64_t)nstg * stage_b <= kRcSmemLimit) {
                bestG = 1; best_nstg = nstg; best_stage = stage_b;
                P.rows_max = rows;
                P.hb = std::max(1, std::min(rows, 16));
                P.plane_bytes = plane_b;
                P.chunk_bytes = (uint32_t)P.npl * plane_b;
                P.cstage = 1;
                P.pair = 0;
                break;
            }
    }
    if (!bestG) return pl;
    P.G = bestG;
    P.nstg = best_nstg;
    P.stage_bytes = best_stage;
    P.n_items = (P.ntiles + P.G - 1) / P.G;
    P.smem_bytes = 1024u + P.stg_off + (uint32_t)P.nstg * P.stage_bytes;
    // packing arguments
    RcPackArgs &A = pl.pack;
    A.KW = KW; A.C = (int)p.C; A.Cout = (int)p.Cout; A.ES = ES; A.Eblk = EN; A.dgrad = P.dgrad;
    A.nmma = P.nmma;
    for (int i = 0; i < P.nmma; ++i) {
        A.m[i].woff = ml[i].woff;
        A.m[i].N = ml[i].N;
        A.m[i].nblk = ml[i].nblk;
        for (int j = 0; j < ml[i].nblk; ++j) { A.m[i].tp[j] = ml[i].tp[j]; A.m[i].tq[j] = ml[i].tq[j]; }
    }
    A.total16 = P.wbytes / 16;
    pl.ws_bytes = ((size_t)P.wbytes + 255) & ~(size_t)255;
    pl.ok = true;
    return pl;
}

struct RcKey {
    int dg, dev, nsm;
    int64_t e[12];
    bool operator==(const RcKey &o) const {
        if (dg != o.dg || dev != o.dev || nsm != o.nsm) return false;
        for (int i = 0; i < 12; ++i)
            if (e[i] != o.e[i]) return false;
        return true;
    }
};

std::shared_ptr<const RcPlan> cached_rc_plan(const Problem &p, bool dgrad) {
    static std::mutex mu;
    static std::vector<std::pair<RcKey, std::shared_ptr<const RcPlan>>> cache;
    const DeviceInfo &di = device_info();
    RcKey k{dgrad ? 1 : 0, di.device, di.num_sms, {p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW, p.D1, p.D2, p.D3, p.s, p.pad}};
    if (p.dt != CAPSCONV_BF16) k.e[7] = -1;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &kv : cache)
        if (kv.first == k) return kv.second;
    if (cache.size() > 256) cache.clear();
    cache.emplace_back(k, std::make_shared<const RcPlan>(make_rc_plan(p, dgrad)));
    std::shared_ptr<const RcPlan> sp = cache.back().second;
    if (probe_env("CAPSCONV_DEBUG") && sp->ok) {
        const RowsConv &P = sp->P;
        fprintf(stderr,
                "[capsconv] rows conv plan: %s Ea=%d nch=%d Hg=%d Wg=%d npl=%d mma=%d out=%d ND=%u T=%d G=%d "
                "tiles=%d items=%d rows=%d stage=%u nstg=%d nacc=%d wbytes=%u smem=%u\n",
                dgrad ? "dI" : "fwd", P.Ea, P.nch, P.Hg, P.Wg, P.npl, P.nmma, P.nout, P.ND, P.T, P.G, P.ntiles,
                P.n_items, P.rows_max, P.stage_bytes, P.nstg, P.nacc, P.wbytes, P.smem_bytes);
    }
    return sp;
}

}  // namespace

bool rows_conv_supported(capsconv_op_t op, const Problem &p) {
    if (op == CAPSCONV_OP_BWD_KERNEL) return false;
    return cached_rc_plan(p, op == CAPSCONV_OP_BWD_DATA)->ok;
}

size_t rows_conv_workspace_bytes(capsconv_op_t op, const Problem &p) {
    std::shared_ptr<const RcPlan> pl = cached_rc_plan(p, op == CAPSCONV_OP_BWD_DATA);
    return pl->ok ? pl->ws_bytes : 0;
}

cudaError_t rows_conv_run(capsconv_op_t op, const Problem &p, const void *src, const void *K, void *out, void *ws,
                          size_t ws_bytes, cudaStream_t st) {
    const bool dgrad = op == CAPSCONV_OP_BWD_DATA;
    RcPlan pl = *cached_rc_plan(p, dgrad);
    if (!pl.ok || ws_bytes < pl.ws_bytes) return cudaErrorNotSupported;
    RowsConv &P = pl.P;
    // source map: fwd = I [B][H][W][4][EI] (planes, element stride s);
    //             dI  = dO [B][Ho][Wo][4][EO] in the phase grid (stride 1)
    const int64_t sH = dgrad ? p.Ho : p.H, sW = dgrad ? p.Wo : p.W;
    const int64_t ES = dgrad ? 4 * p.Cout : 4 * p.C;
    if (!rows::make_rows_map5(&P.tmS, src, p.B, sH, sW, ES, P.Ea, P.Wg * P.es, 1, P.es, 1))
        return cudaErrorInvalidValue;
    if (P.merged) {
        if (!rows::make_rows_map4m(&P.tmH, src, p.B * sH, sW, ES, P.Ea, P.Wg * P.es, P.hb * P.es, P.es))
            return cudaErrorInvalidValue;
    } else if (!rows::make_rows_map5(&P.tmH, src, p.B, sH, sW, ES, P.Ea, P.Wg * P.es, P.hb * P.es, P.es, P.es)) {
        return cudaErrorInvalidValue;
    }
    P.wpack = static_cast<const uint8_t *>(ws);
    P.out = static_cast<__nv_bfloat16 *>(out);
    P.dbg = probe_env("CAPSCONV_RC_DBG") ? atoi(probe_env("CAPSCONV_RC_DBG")) : 0;
    P.prof = nullptr;
    static unsigned long long *prof_buf = nullptr;
    if (kProbes && probe_env("CAPSCONV_RC_PROF")) {
        if (!prof_buf) cudaMalloc(&prof_buf, 148 * 8 * sizeof(unsigned long long));
        cudaMemsetAsync(prof_buf, 0, 148 * 8 * sizeof(unsigned long long), st);
        P.prof = prof_buf;
    }
    RcPackArgs &A = pl.pack;
    A.K = static_cast<const __nv_bfloat16 *>(K);
    A.dst = static_cast<uint8_t *>(ws);
    cudaError_t e = probe_skip_pack() ? cudaSuccess
                                       : launch_pack(rc_pack_kernel, dim3((A.total16 + 63) / 64), dim3(64), 0, st, A);
    if (e != cudaSuccess) return e;
    note_launches(1);
    e = smem_optin(reinterpret_cast<const void *>(rows_conv_kernel), (int)P.smem_bytes);
    if (e != cudaSuccess) return e;
    const int grid = std::min(P.n_items, device_info().num_sms);
    e = launch_k(rows_conv_kernel, dim3(grid), dim3(kRcThreads), P.smem_bytes, st, P);
    if (e != cudaSuccess) return e;
    note_launches(1);
    if (kProbes && P.prof) {
        unsigned long long h[148 * 8];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, P.prof, sizeof(h), cudaMemcpyDeviceToHost);
        double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int b = 0; b < grid; ++b)
            for (int i = 0; i < 8; ++i) a[i] += (double)h[b * 8 + i] / grid;
        fprintf(stderr,
                "[rc prof] %s cycles/CTA: wait_full %.0f wait_acce %.0f issue %.0f commit %.0f total %.0f | epi warp0: "
                "tiles %.1f wait %.0f/tile work %.0f/tile\n",
                dgrad ? "dI" : "fwd", a[0], a[1], a[2], a[3], a[4], a[7], a[5] / a[7], a[6] / a[7]);
    }
    return cudaGetLastError();
}

}  // namespace capsconv
