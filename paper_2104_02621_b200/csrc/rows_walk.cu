// rows_walk.cu -- row-walk forward O (stride 1, 2) and data gradient dI
// (stride 1) for the D1-outer ("rows") layout on tcgen05.
//
// Same contraction as rows_conv.cu (Algorithm 2; dI =
// the adjoint of Algorithm 4, readings R10/R11), organised around
// the SOURCE row instead of the output tile:
//
//   fwd:  O[y]  += I[Ys]  . K[p]      for every tap row p with Ys = s*y + p
//   dI:   dI[y] += dO[Ys] . K[p]^T    for every tap row p with y  = Ys + p
//
// One staged source row (a TMA box of 32 virtual pixels x 4 d1 rows = the
// M = 128 A operand, shifted by whole pixels for the column taps q) feeds all
// output rows it touches at once: the row taps are stacked in N, B = [W_p]
// ordered by ascending output row, and the accumulators of consecutive output
// rows sit side by side in TMEM (a ring of R slots of NB columns), so one MMA of
// N = (taps) * NB adds into all of them -- no epilogue shifts.  An SS MMA costs
// ~max(60 + N/8, N/2) cycles (tests/probe/rows_probe), so N = 96..192 instead
// of 32..64 per MMA cuts the issue cost of the thin layers 2-3x.
//
// Tiles: M = 32 virtual pixels = G images x Xs pixels (Xs a power of two >= the
// source row width incl. the halo, so G images share one MMA), or 32-pixel
// x-tiles of one image for wide rows.  The first MMA that touches an output
// row overwrites it (the first tap-group MMA of a source row is split at that
// boundary), an output row is committed to the epilogue after the last source
// row that touches it, and an MMA is split where its rows wrap around the ring.
//
// Epilogue: TMEM -> bf16 -> per-warp swizzled staging -> TMA box store (clipped
// at the tensor bounds, so the virtual pixels past the row end are dropped).
// Roles: warp 0 TMA, warp 1 MMA (TMEM owner), warps 2.. epilogue groups of four.
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

constexpr int kWkMaxR = 16;        // accumulator slots
constexpr int kWkMaxStg = 12;   // stages over all streams
constexpr int kWkMaxQ = 4;         // column taps (KW)
constexpr int kWkMaxRows = 64;     // walked source rows (the schedule lives in the kernel parameters)
constexpr uint32_t kWkSmemLimit = 227 * 1024;

struct RowsWalk {
    alignas(64) CUtensorMap tmS;   // source (Es, 4, Ws, Hs, B): box (Ea, 4, bx*s, 1, G), element strides (1,1,s,1,1)
    alignas(64) CUtensorMap tmO;   // output (Eo, 4, Wo, Ho, B): box (cw, 4, 8, ey, 1), swizzle 2*cw bytes
    const uint8_t *wpack;          // packed weight image (global), copied to shared memory once
    int dgrad, s, KW;
    int B, Hs, Ho, Wo;
    int G, Xs, nxt, ngi, n_items;  // images per tile, pixel slot per image, x tiles, image groups, items
    int x0mul, x0off;              // source pixel of plane 0, x tile xt: x0mul*xt + x0off
    int box_px;                    // pixels per plane of one source-row box (per image)
    int npl, nch, Ea;              // planes (= s), source chunks per row, elements per chunk
    int ncls, ncl[2], pm[2];       // row classes (Ys mod s); taps per class; y0 = (Ys - pm)/s
    int NB, R;                     // accumulator columns per output row; ring slots
    int nmw, Rw;                   // MMA streams (TMA + MMA warp pairs, alternate strips); slots per stream
    int nepi, nbuf, cw;            // epilogue groups of 4 warps; staging buffers per warp; store box columns
    int ys_lo, ys_hi;              // walked source rows
    uint32_t plane_bytes, stage_bytes, stage_tx;
    int nstg;
    uint32_t woff_s, wbytes, soff, sbytes;   // shared offsets (from the 1024-aligned base): weights, staging
    uint32_t roff;                 // shared offset of the per-source-row schedule (32 B per row)
    int ey;                        // output rows per epilogue store box
    int dyn;                       // streams take strips from a CTA-shared counter (see wk_take)
    uint32_t foff;                 // shared offset (from the 1024-aligned base) of the strip lists
    int espin;                     // epilogue waits: 1 poll (try_wait loop), 0 suspend with a time hint
    int est;                       // epilogue stores: 0 one TMA box per group, 2 per-warp coalesced 16-byte stores
    int rps;                       // source rows per pipeline step (1 or 2): stage = rps rows x planes of one chunk
    __nv_bfloat16 *out;
    uint32_t smem_bytes;
    uint32_t wof[2][kWkMaxQ];      // weight block (class, q) byte offsets in the image
    uint32_t aoff[kWkMaxQ];        // A offset of column tap q: plane * plane_bytes + shift * 4 rows
    uint32_t sched[kWkMaxRows][8]; // per-source-row MMA schedule (wk_make_rec), built on the host
    unsigned long long *prof;      // probe builds only: per-CTA cycle counters [cta][8]
    int zfill;                     // drained slots are zeroed by the epilogue: every MMA accumulates
    int dbg;                       // probe builds only: 1 skip epilogue stores, 2 skip source loads, 4 skip MMAs
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

#ifdef CAPSCONV_NOCLK   // probe builds without the cycle counters (product-like timing with the dbg knobs)
__device__ __forceinline__ unsigned long long wk_clk() { return 0ull; }
#else
__device__ __forceinline__ unsigned long long wk_clk() { return kProbes ? clock64() : 0ull; }
#endif

__host__ __device__ __forceinline__ int wk_min(int a, int b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int wk_max(int a, int b) { return a > b ? a : b; }

__host__ __device__ __forceinline__ int wk_y0(const RowsWalk &P, int Ys, int &cl) {
    cl = P.s == 2 ? (Ys & 1) : 0;
    return P.s == 2 ? (Ys - P.pm[cl]) >> 1 : Ys - P.pm[0];   // exact: Ys - pm[cl] is a multiple of s
}

// valid output rows [ya, yb] of source row Ys (empty if ya > yb)
__host__ __device__ __forceinline__ void wk_rows(const RowsWalk &P, int Ys, int &cl, int &y0, int &ya, int &yb) {
    y0 = wk_y0(P, Ys, cl);
    ya = wk_max(y0, 0);
    yb = wk_min(y0 + P.ncl[cl] - 1, P.Ho - 1);
}

// Per-source-row MMA schedule, identical for every strip (the accumulator of
// output row y lives in slot y mod R; slot phases are tracked per slot), built
// once per CTA in shared memory.  Record of 8 words:
//   w0: slots to wait free (rows touched first here) | slots to commit << 16
//   w1: bit 0 valid, bit 1 row class
//   w2..w5: segments of the first MMA (split where the fresh rows start; with
//           zfill the fresh slots already hold zeros and w2..w3 = w6..w7)
//   w6..w7: segments of the other MMAs (split only where the rows wrap the ring)
// segment word: dcol (10 bits) | B row offset in 16-byte units (10) << 10 |
//               accumulate << 20 | N/8 << 21 (0: no segment)
constexpr uint32_t kWkRecBytes = 32;

__host__ __device__ __forceinline__ void wk_seg(const RowsWalk &P, int y0, int u, int v, uint32_t acc, uint32_t &a,
                                                uint32_t &b) {
    a = 0u;
    b = 0u;
    if (u > v) return;
    const int slot = u % P.Rw;
    const int w = wk_min(v, u + (P.Rw - slot) - 1);
    a = (uint32_t)(slot * P.NB) | ((uint32_t)((u - y0) * P.NB) << 10) | (acc << 20) |
        ((uint32_t)((w - u + 1) * P.NB / 8) << 21);
    if (w < v)
        b = ((uint32_t)((w + 1 - y0) * P.NB) << 10) | (acc << 20) | ((uint32_t)((v - w) * P.NB / 8) << 21);
}

__host__ __device__ void wk_make_rec(const RowsWalk &P, int Ys, uint32_t (&w)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = 0u;
    int cl, y0, ya, yb;
    wk_rows(P, Ys, cl, y0, ya, yb);
    if (ya > yb) return;
    int yfresh = 0, ynext = P.Ho;
    for (int Yp = Ys - 1; Yp >= P.ys_lo; --Yp) {
        int c2, y02, ya2, yb2;
        wk_rows(P, Yp, c2, y02, ya2, yb2);
        if (ya2 <= yb2) { yfresh = yb2 + 1; break; }
    }
    for (int Yn = Ys + 1; Yn <= P.ys_hi; ++Yn) {
        int c2, y02, ya2, yb2;
        wk_rows(P, Yn, c2, y02, ya2, yb2);
        if (ya2 <= yb2) { ynext = ya2; break; }
    }
    const int yf = wk_max(ya, yfresh);
    uint32_t wm = 0u, cm = 0u;
    for (int y = yf; y <= yb; ++y) wm |= 1u << (y % P.Rw);
    for (int y = ya; y < ynext; ++y) cm |= 1u << (y % P.Rw);
    w[0] = wm | (cm << 16);
    w[1] = 1u | ((uint32_t)cl << 1);
    wk_seg(P, y0, ya, yb, 1u, w[6], w[7]);
    if (P.zfill) {
        w[2] = w[6];
        w[3] = w[7];
    } else {
        wk_seg(P, y0, ya, yf - 1, 1u, w[2], w[3]);
        wk_seg(P, y0, yf, yb, 0u, w[4], w[5]);
    }
}

__device__ __forceinline__ void wk_mma_seg(uint32_t sg, uint32_t dbase, uint64_t ad, uint32_t bhi, uint32_t bk,
                                           uint32_t ibase, uint32_t acc) {
    rows::mma_ss_elect(dbase + (sg & 1023u), ad, ((uint64_t)bhi << 32) | (uint64_t)(bk + ((sg >> 10) & 1023u)),
                       ibase | ((sg >> 21) << 17), acc);
}

// Strip assignment.  Static: stream w of a CTA takes the CTA's strips
// w, w + nmw, ...; dynamic (P.dyn): the streams' TMA warps take the CTA's
// strips from a shared counter in the order they finish (the CTA's 6-7 strips
// split 3/2/2 over three streams statically), and publish each taken strip --
// or -1 at the end -- in a per-stream list of single-use mbarrier slots that
// the stream's MMA warp and epilogue groups read in the same order.
constexpr int kWkFifo = 16;
struct WkFifo {
    uint64_t *bar;   // [3][kWkFifo]
    int *id;         // [3][kWkFifo]
    int *ctr;
};
__device__ __forceinline__ int wk_take(const RowsWalk &P, const WkFifo &F, int w, int e) {   // TMA warp lane 0
    int it;
    if (P.dyn) {
        const int k = atomicAdd(F.ctr, 1);
        it = blockIdx.x + k * (int)gridDim.x;
        if (it >= P.n_items) it = -1;
        F.id[w * kWkFifo + e] = it;
        mbar_arrive(F.bar + w * kWkFifo + e);   // release: the id is visible to the waiters
    } else {
        it = blockIdx.x + (w + P.nmw * e) * (int)gridDim.x;
        if (it >= P.n_items) it = -1;
    }
    return it;
}
__device__ __forceinline__ int wk_read(const RowsWalk &P, const WkFifo &F, int w, int e) {   // MMA / epilogue warps
    if (!P.dyn) {
        const int it = blockIdx.x + (w + P.nmw * e) * (int)gridDim.x;
        return it < P.n_items ? it : -1;
    }
    mbar_wait(F.bar + w * kWkFifo + e, 0u);
    return *(volatile int *)(F.id + w * kWkFifo + e);
}

template <int KWT, int KPC>
__device__ __forceinline__ void wk_mma(const RowsWalk &P, int w, uint32_t stg0, uint32_t wsm, uint32_t sched,
                                       uint64_t *full, uint64_t *empty, uint64_t *accf, uint64_t *acce,
                                       const WkFifo &F) {
    const int swz = 2 * P.Ea;
    const uint32_t sbo_a = 16u * (uint32_t)P.Ea;              // 8 rows of 2*Ea bytes
    const uint64_t a0 = rows::sdesc(stg0, 16u, sbo_a, swz);
    const uint32_t ahi = (uint32_t)(a0 >> 32);
    const uint32_t bhi = (uint32_t)(smem_desc(wsm, 16u, 128u) >> 32);
    const uint32_t ibase = idesc_bf16(128, 16, 0, 0) & ~(63u << 17);   // N field filled per segment
    uint32_t bl[2], bst[2], aoff[KWT], wq[2][KWT];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const uint32_t Ncl = (uint32_t)(P.ncl[c] * P.NB);
        bl[c] = (uint32_t)smem_desc(wsm, Ncl * 16u, 128u);
        bst[c] = Ncl * 2u;                                    // 32*N bytes per k-step, 16-byte units
#pragma unroll
        for (int q = 0; q < KWT; ++q) wq[c][q] = bl[c] + (P.wof[c][q] >> 4);
    }
#pragma unroll
    for (int q = 0; q < KWT; ++q) aoff[q] = P.aoff[q] >> 4;
    const int nrow = P.ys_hi - P.ys_lo + 1, nch = P.nch, nstg = P.nstg;
    const uint32_t sbytes16 = P.stage_bytes >> 4;
    // stream w: its own stages, barriers and accumulator slots [w*Rw, (w+1)*Rw)
    full += w * nstg;
    empty += w * nstg;
    accf += w * P.Rw;
    acce += w * P.Rw;
    const uint32_t dbase = (uint32_t)(w * P.Rw * P.NB);
    const uint32_t a0lo = (uint32_t)a0 + (((uint32_t)(w * nstg) * P.stage_bytes) >> 4);
    int sb = 0;
    uint32_t ph = 0, mph = 0;   // stage phase; per-slot acce phases
    unsigned long long pw_full = 0, pw_acce = 0;
    const unsigned long long pstart = wk_clk();
    const int rps = P.rps;                                       // source rows per pipeline step
    const uint32_t rowb16 = (uint32_t)P.npl * (P.plane_bytes >> 4);  // next row of a step
    for (int e = 0;; ++e) {
        if (wk_read(P, F, w, e) < 0) break;
        for (int r0 = 0; r0 < nrow; r0 += rps) {
            // the step's rows: records, then the slots their first touches need
            uint4 h0[2], h1[2];
            bool v[2];
            uint32_t wm = 0u, cm = 0u;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                v[j] = false;
                h0[j] = make_uint4(0u, 0u, 0u, 0u);
                h1[j] = h0[j];
                if (j < rps && r0 + j < nrow) {
                    const uint32_t *rec = P.sched[r0 + j];
                    h0[j] = make_uint4(rec[0], rec[1], rec[2], rec[3]);
                    v[j] = (h0[j].y & 1u) != 0u;
                    if (v[j]) {
                        h1[j] = make_uint4(rec[4], rec[5], rec[6], rec[7]);
                        wm |= h0[j].x & 0xffffu;
                        cm |= h0[j].x >> 16;
                    }
                }
            }
            if (!v[0] && !v[1]) continue;
            unsigned long long t0 = wk_clk();
            for (uint32_t m = wm; m; m &= m - 1u) {   // slots first touched in this step
                const int j = __ffs(m) - 1;
                mbar_wait(acce + j, ((mph >> j) & 1u) ^ 1u);
                mph ^= 1u << j;
            }
            if (kProbes) pw_acce += wk_clk() - t0;
            fence_after_sync();
            for (int c = 0; c < nch; ++c) {
                t0 = wk_clk();
                mbar_wait(full + sb, ph);
                if (kProbes) pw_full += wk_clk() - t0;
                fence_after_sync();
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (!v[j]) continue;
                    const uint32_t alo = a0lo + (uint32_t)sb * sbytes16 + (uint32_t)j * rowb16;
                    const int cl = (h0[j].y >> 1) & 1u;
                    const uint32_t bstc = cl ? bst[1] : bst[0];
#pragma unroll
                    for (int q = 0; q < (kProbes && (P.dbg & 4) ? 0 : KWT); ++q) {
                        const uint32_t wqc = cl ? wq[1][q] : wq[0][q];
#pragma unroll
                        for (int kk = 0; kk < KPC; ++kk) {
                            const uint64_t ad = ((uint64_t)ahi << 32) | (uint64_t)(alo + aoff[q] + 2u * (uint32_t)kk);
                            const uint32_t bk = wqc + (uint32_t)(c * KPC + kk) * bstc;
                            if (q == 0 && kk == 0 && c == 0) {
                                const uint4 a = h0[j], b = h1[j];
                                if (a.z >> 21) wk_mma_seg(a.z, dbase, ad, bhi, bk, ibase, (a.z >> 20) & 1u);
                                if (a.w >> 21) wk_mma_seg(a.w, dbase, ad, bhi, bk, ibase, (a.w >> 20) & 1u);
                                if (b.x >> 21) wk_mma_seg(b.x, dbase, ad, bhi, bk, ibase, (b.x >> 20) & 1u);
                                if (b.y >> 21) wk_mma_seg(b.y, dbase, ad, bhi, bk, ibase, (b.y >> 20) & 1u);
                            } else {
                                wk_mma_seg(h1[j].z, dbase, ad, bhi, bk, ibase, 1u);
                                if (h1[j].w >> 21) wk_mma_seg(h1[j].w, dbase, ad, bhi, bk, ibase, 1u);
                            }
                        }
                    }
                }
                if (elect_one()) mma_commit(empty + sb);
                __syncwarp();
                if (++sb == nstg) { sb = 0; ph ^= 1; }
            }
            if (elect_one())   // rows no later source row touches
                for (uint32_t m = cm; m; m &= m - 1u) mma_commit(accf + (__ffs(m) - 1));
            __syncwarp();
        }
    }
    if (kProbes && P.prof && w == 0 && (threadIdx.x & 31) == 0) {
        unsigned long long *o = P.prof + (size_t)blockIdx.x * 8;
        o[0] = pw_full;
        o[1] = pw_acce;
        o[2] = wk_clk() - pstart;
    }
}

// Epilogue: one accumulator row chunk of this warp (32 lanes = 8 pixels x 4
// d1) converted to bf16 and staged as rows yy*32 + lane of a SWIZZLE_(2*CW)
// box image (16-byte chunk j of row r at j ^ (r * 2CW / 128 mod 2CW/16):
// conflict-free); the box is stored by one TMA per EY output rows.
template <int CW>
__device__ __forceinline__ void wk_stage(const float *v, uint32_t buf, int r) {
    constexpr uint32_t rowb = (uint32_t)CW * 2u;
    constexpr uint32_t zsh = rowb == 128u ? 0u : rowb == 64u ? 1u : 2u;
    const uint32_t rsw = ((uint32_t)r >> zsh) & (rowb / 16u - 1u);
#pragma unroll
    for (int j = 0; j < CW / 8; ++j) {
        uint32_t w[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * j + 2 * c], v[8 * j + 2 * c + 1]);
            w[c] = *reinterpret_cast<uint32_t *>(&h);
        }
        const uint32_t a = buf + (uint32_t)r * rowb + ((((uint32_t)j) ^ rsw) * 16u);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                     : "memory");
    }
}

// Epilogue warps.  Group g serves stream w = g / gps and its row blocks
// y0 = EY*gl (mod EY*gps).  Each warp owns TMEM lane quarter qq = 32 rows of
// the accumulator (8 pixels x 4 d1).  EST 2: per-warp swizzled staging, then
// coalesced 16-byte stores (the SM's TMA unit serves only the source loads);
// EST 0: the group's four warps stage one box (cw, 4, Xs, ey, G) and its first
// warp issues one TMA store.
template <int CW, int EST>
__device__ __forceinline__ void wk_epilogue(const RowsWalk &P, int warp, int lane, uint32_t base, uint64_t *accf,
                                            uint64_t *acce, const WkFifo &F) {
    const int nmw = P.nmw;
    const int e = warp - 2 * nmw, grp = e >> 2, qq = warp & 3;
    const int gps = P.nepi / nmw, w = grp / gps, gl = grp - w * gps;
    constexpr uint32_t rowb = (uint32_t)CW * 2u;             // staged row bytes (= swizzle span)
    constexpr int cpr = CW / 8;                               // 16-byte chunks per staged row
    constexpr uint32_t zsh = rowb == 128u ? 0u : rowb == 64u ? 1u : 2u;
    const int EY = P.ey, nbuf = P.nbuf;
    const uint32_t bufb = (uint32_t)EY * 128u * rowb;         // one group staging box
    const uint32_t sbuf0 = base + P.soff + (uint32_t)(grp * nbuf) * bufb;
    const uint32_t wbuf = sbuf0 + (uint32_t)(e & 3) * (uint32_t)EY * 32u * rowb;   // EST 2: this warp's rows
    const bool leader = (e & 3) == 0 && lane == 0;
    const int bar_id = 1 + grp;
    const int pxl = 8 * qq + (lane >> 2), d1 = lane & 3;      // this lane's tile pixel and d1 row
    const int Rw = P.Rw, NB = P.NB;
    const int lb = P.G > 1 ? pxl / P.Xs : 0, lx = P.G > 1 ? pxl - lb * P.Xs : pxl;
    const int sxs = P.G > 1 ? P.Xs : 32;
    const int wimg_off = P.G > 1 ? (8 * qq) / P.Xs : 0, wx_off = P.G > 1 ? (8 * qq) % P.Xs : 8 * qq;
    accf += w * Rw;
    acce += w * Rw;
    const uint32_t tl = ((uint32_t)(qq * 32) << 16) + (uint32_t)(w * Rw * NB);
    uint32_t eph = 0;                                         // per-slot accf phases
    int bi = 0;
    unsigned long long pe_wait = 0, pe_rows = 0;
    const unsigned long long pe_start = wk_clk();
    for (int fe = 0;; ++fe) {
        const int it = wk_read(P, F, w, fe);
        if (it < 0) break;
        const int gi = it / P.nxt, xt = it - gi * P.nxt;
        const int img0 = gi * P.G, xg0 = P.G > 1 ? 0 : 32 * xt;
        const int wimg = img0 + wimg_off, wx0 = xg0 + wx_off;
        int slot = EY * gl;
        for (int y0 = EY * gl; y0 < P.Ho; y0 += EY * gps) {
            const int ny = min(EY, P.Ho - y0);
            const unsigned long long e0 = wk_clk();
            for (int yy = 0; yy < ny; ++yy) {
                if (P.espin) mbar_wait(accf + slot + yy, (eph >> (slot + yy)) & 1u);
                else mbar_wait_sleep(accf + slot + yy, (eph >> (slot + yy)) & 1u);
                eph ^= 1u << (slot + yy);
            }
            if (kProbes) { pe_wait += wk_clk() - e0; pe_rows += ny; }
            fence_after_sync();
            for (int c0 = 0; c0 < NB; c0 += CW) {
                const uint32_t buf = sbuf0 + (uint32_t)(nbuf > 1 ? (bi & 1) : 0) * bufb;
                if (EST == 0) {
                    if (leader) {   // this buffer's previous store has read it
                        if (nbuf > 1) rows::bulk_wait_read<1>();
                        else rows::bulk_wait_read<0>();
                    }
                    named_bar_sync(bar_id, 128);
                }
                for (int yy = 0; yy < ny; ++yy) {
                    const uint32_t tb = tl + (uint32_t)((slot + yy) * NB + c0);
                    float v[CW];
                    if (CW == 16) {
                        tmem_ld16(tb, *reinterpret_cast<float(*)[16]>(v));
                    } else {
                        rows::tmem_ld32(tb, *reinterpret_cast<float(*)[32]>(v));
                        if (CW == 64) rows::tmem_ld32(tb + 32u, *reinterpret_cast<float(*)[32]>(v + 32 % CW));
                    }
                    tmem_wait_ld();
                    if (P.zfill) {   // leave zeros behind: the slot's next row starts by accumulating
#pragma unroll
                        for (int z = 0; z < CW; z += 16) rows::tmem_st_zero16(tb + (uint32_t)z);
                    }
                    if (c0 + CW >= NB) {   // slot drained: hand it back to the MMA warp
                        if (P.zfill) rows::tmem_wait_st();
                        fence_before_sync();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(acce + slot + yy);
                    }
                    if (kProbes && (P.dbg & 1)) continue;
                    if (EST == 0) {
                        wk_stage<CW>(v, buf, ((lb * EY + yy) * sxs + lx) * 4 + d1);
                    } else {
                        const uint32_t ybuf = wbuf + (uint32_t)yy * 32u * rowb;
                        wk_stage<CW>(v, ybuf, lane);
                        __syncwarp();
                        if (wimg < P.B) {
                            uint8_t *gb = reinterpret_cast<uint8_t *>(P.out) +
                                          ((((size_t)wimg * P.Ho + (y0 + yy)) * P.Wo + wx0) * 4 * (size_t)NB + c0) * 2;
#pragma unroll
                            for (int i = 0; i < cpr; ++i) {
                                const int k = i * 32 + lane, r = k / cpr, j = k % cpr;
                                if (wx0 + (r >> 2) < P.Wo) {
                                    const uint32_t rsw = ((uint32_t)r >> zsh) & (uint32_t)(cpr - 1);
                                    const uint4 x = ld_shared_v4(ybuf + (uint32_t)r * rowb + ((uint32_t)j ^ rsw) * 16u);
                                    *reinterpret_cast<uint4 *>(gb + (size_t)r * NB * 2 + (size_t)j * 16) = x;
                                }
                            }
                        }
                        __syncwarp();
                    }
                }
                if (EST == 0) {
                    fence_proxy_async_smem();
                    named_bar_sync(bar_id, 128);
                    if (leader && img0 < P.B && !(kProbes && (P.dbg & 1))) {
                        rows::tma_store5d(&P.tmO, buf, c0, 0, xg0, y0, img0);
                        rows::bulk_commit();
                    }
                }
                ++bi;
            }
            slot += EY * gps;
            if (slot >= Rw) slot -= Rw;
        }
    }
    if (EST == 0 && leader) rows::bulk_wait_all();
    if (kProbes && P.prof && e == 0 && lane == 0) {
        unsigned long long *o = P.prof + (size_t)blockIdx.x * 8;
        o[3] = pe_wait;
        o[4] = pe_rows;
        o[5] = wk_clk() - pe_start;
    }
}

__global__ void __launch_bounds__(640, 1) rows_walk_kernel(const __grid_constant__ RowsWalk P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *full = bars, *empty = bars + kWkMaxStg, *accf = bars + 2 * kWkMaxStg,
             *acce = bars + 2 * kWkMaxStg + kWkMaxR, *wbar = bars + 2 * kWkMaxStg + 2 * kWkMaxR;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + 768);
    const uint32_t base = (smem_u32(smem_raw) + 1024u + 1023u) & ~1023u;
    const uint32_t stg0 = base, wsm = base + P.woff_s, sched = base + P.roff;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
    WkFifo F;
    F.bar = reinterpret_cast<uint64_t *>(smem_raw + (base - smem_u32(smem_raw)) + P.foff);
    F.id = reinterpret_cast<int *>(F.bar + 3 * kWkFifo);
    F.ctr = F.id + 3 * kWkFifo;
    if (threadIdx.x == 0) {
        for (int i = 0; i < P.nstg * P.nmw; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        if (P.dyn) {
            for (int i = 0; i < 3 * kWkFifo; ++i) mbar_init(F.bar + i, 1);
            *F.ctr = 0;
        }
        for (int i = 0; i < P.R; ++i) {
            mbar_init(accf + i, 1);
            mbar_init(acce + i, 4);
        }
        mbar_init(wbar, 1);
        mbar_fence_init();
    }
    if (warp == 1) tmem_alloc_dyn(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (*tmem_slot != 0u) __trap();
    if (P.zfill) {   // every accumulator column starts at zero (epilogue warps, own lane quarter)
        const int e = warp - 2 * P.nmw;
        if (e >= 0) {
            const uint32_t tl = (uint32_t)((warp & 3) * 32) << 16;
            for (int c = (e >> 2) * 16; c < 512; c += 16 * P.nepi) rows::tmem_st_zero16(tl + (uint32_t)c);
            rows::tmem_wait_st();
        }
        fence_before_sync();
        __syncthreads();
        fence_after_sync();
    }
    pdl_wait();
    // The packed weights are the only workspace bytes this kernel reads: once
    // they are in shared memory the next kernel may launch (PDL) -- e.g. the
    // next call's weight pack, which rewrites the workspace.
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(wbar, P.wbytes);
        for (uint32_t o = 0; o < P.wbytes; o += 32768u)
            bulk_g2s_u32(wsm + o, P.wpack + o, min(32768u, P.wbytes - o), wbar);
    }
    mbar_wait(wbar, 0);
    pdl_launch_dependents();

    const int nmw = P.nmw;
    if (warp < 2 * nmw && !(warp & 1)) {
        // ------------------------------------------------------------ TMA (stream w)
        const int w = warp >> 1;
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&P.tmS)) : "memory");
            uint64_t *fullw = full + w * P.nstg, *emptyw = empty + w * P.nstg;
            const uint32_t stgw = stg0 + (uint32_t)(w * P.nstg) * P.stage_bytes;
            int sb = 0;
            uint32_t ph = 0;
            unsigned long long pt_wait = 0;
            const int nrow = P.ys_hi - P.ys_lo + 1;
            for (int e = 0;; ++e) {
                const int it = wk_take(P, F, w, e);
                if (it < 0) break;
                const int gi = it / P.nxt, xt = it - gi * P.nxt;
                const int X0 = P.x0mul * xt + P.x0off;
                for (int r0 = 0; r0 < nrow; r0 += P.rps) {
                    bool v[2];
                    int nv = 0;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        v[j] = j < P.rps && r0 + j < nrow && (P.sched[r0 + j][1] & 1u);
                        nv += v[j] ? 1 : 0;
                    }
                    if (!nv) continue;
                    for (int c = 0; c < P.nch; ++c) {
                        const unsigned long long t0 = wk_clk();
                        mbar_wait(emptyw + sb, ph ^ 1);
                        if (kProbes) pt_wait += wk_clk() - t0;
                        const uint32_t stg = stgw + (uint32_t)sb * P.stage_bytes;
                        const uint32_t mb = smem_u32(fullw + sb);
                        if (kProbes && (P.dbg & 2)) {
                            mbar_arrive(fullw + sb);
                            if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                            continue;
                        }
                        mbar_arrive_expect_tx(fullw + sb, P.stage_tx * (uint32_t)nv);
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            if (v[j])
                                for (int pl = 0; pl < P.npl; ++pl)
                                    rows::tma_load5d(stg + (uint32_t)(j * P.npl + pl) * P.plane_bytes, &P.tmS, c * P.Ea,
                                                     0, X0 + pl, P.ys_lo + r0 + j, gi * P.G, mb);
                        if (++sb == P.nstg) { sb = 0; ph ^= 1; }
                    }
                }
            }
            if (kProbes && P.prof && w == 0) P.prof[(size_t)blockIdx.x * 8 + 6] = pt_wait;
        }
    } else if (warp < 2 * nmw) {
        // ------------------------------------------------------------ MMA (stream w)
        const int w = warp >> 1;
        mbar_wait(wbar, 0);
        const int KPC = P.Ea / 16;
        if (P.KW == 3 && KPC == 2) wk_mma<3, 2>(P, w, stg0, wsm, sched, full, empty, accf, acce, F);
        else if (P.KW == 3 && KPC == 4) wk_mma<3, 4>(P, w, stg0, wsm, sched, full, empty, accf, acce, F);
        else if (P.KW == 2 && KPC == 2) wk_mma<2, 2>(P, w, stg0, wsm, sched, full, empty, accf, acce, F);
        else if (P.KW == 2 && KPC == 4) wk_mma<2, 4>(P, w, stg0, wsm, sched, full, empty, accf, acce, F);
        else if (P.KW == 4 && KPC == 2) wk_mma<4, 2>(P, w, stg0, wsm, sched, full, empty, accf, acce, F);
        else if (P.KW == 4 && KPC == 4) wk_mma<4, 4>(P, w, stg0, wsm, sched, full, empty, accf, acce, F);
        else __trap();
    } else {
        // ------------------------------------------------------------ epilogue
        if (P.est == 2) {
            if (P.cw == 16) wk_epilogue<16, 2>(P, warp, lane, base, accf, acce, F);
            else if (P.cw == 32) wk_epilogue<32, 2>(P, warp, lane, base, accf, acce, F);
            else wk_epilogue<64, 2>(P, warp, lane, base, accf, acce, F);
        } else {
            if (P.cw == 16) wk_epilogue<16, 0>(P, warp, lane, base, accf, acce, F);
            else if (P.cw == 32) wk_epilogue<32, 0>(P, warp, lane, base, accf, acce, F);
            else wk_epilogue<64, 0>(P, warp, lane, base, accf, acce, F);
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_dealloc_dyn(0u, 512);
}

struct WkPackArgs {
    const __nv_bfloat16 *K;
    uint8_t *dst;
    int dgrad, KW, C, Cout, NB, Es;
    int nblk;                   // (class, q) blocks
    uint32_t bo[8];             // block start, 16-byte units
    int bcl[8], bq[8], bN[8];   // class, column tap, rows of the block
    int tp[2][8];               // class taps in B row order
    uint32_t total16;
};

// One thread per 16-byte unit (8 consecutive k of one row n) of the K-major
// no-swizzle image: unit (k/8, n) of block (cl, q) at bo + (k/8)*Ncl + n.
__device__ __forceinline__ void wk_pack_unit(const WkPackArgs &A, uint32_t g) {
    int b = 0;
    while (b + 1 < A.nblk && A.bo[b + 1] <= g) ++b;
    const uint32_t loc = g - A.bo[b];
    const int N = A.bN[b];
    const int kc = (int)(loc / (uint32_t)N), n = (int)(loc - (uint32_t)kc * N);
    const int j = n / A.NB, r = n - j * A.NB;
    const int p = A.tp[A.bcl[b]][j], q = A.bq[b];
    __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int k = kc * 8 + e;
        int c, co, d2, d3;
        if (!A.dgrad) { c = k >> 2; d2 = k & 3; co = r >> 2; d3 = r & 3; }
        else { co = k >> 2; d3 = k & 3; c = r >> 2; d2 = r & 3; }
        v[e] = A.K[((((size_t)(p * A.KW + q) * A.C + c) * A.Cout + co) * 4 + d2) * 4 + d3];
    }
    uint4 w;
    memcpy(&w, v, 16);
    reinterpret_cast<uint4 *>(A.dst)[g] = w;
}

// Runs alongside the previous kernel's tail (see rc_pack_kernel): it reads only
// K and writes only the workspace, and waits for the previous grid before it
// exits so that its completion keeps stream order.
__global__ void __launch_bounds__(64) wk_pack_kernel(const __grid_constant__ WkPackArgs A) {
    pdl_launch_dependents();
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < A.total16) wk_pack_unit(A, g);
    pdl_wait();
}

struct WkPlan {
    bool ok = false;
    RowsWalk P;
    WkPackArgs pack;
    size_t ws_bytes = 0;
};

WkPlan make_wk_plan(const Problem &p, bool dgrad) {
    WkPlan pl;
    RowsWalk &P = pl.P;
    memset(&P, 0, sizeof(P));
    memset(&pl.pack, 0, sizeof(pl.pack));
    if (p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4 || p.pad != 0) return pl;
    const int s = (int)p.s, KH = (int)p.KH, KW = (int)p.KW;
    if (dgrad ? s != 1 : (s < 1 || s > 2)) return pl;
    if (KW < 2 || KW > kWkMaxQ || KH < 2 || KH > 8) return pl;
    if (p.B > (1 << 20) || p.H > 4096 || p.W > 4096) return pl;
    P.dgrad = dgrad ? 1 : 0;
    P.s = s;
    P.KW = KW;
    P.B = (int)p.B;
    const int Es = (int)(dgrad ? 4 * p.Cout : 4 * p.C), Eo = (int)(dgrad ? 4 * p.C : 4 * p.Cout);
    P.Hs = (int)(dgrad ? p.Ho : p.H);
    const int Ws = (int)(dgrad ? p.Wo : p.W);
    P.Ho = (int)(dgrad ? p.H : p.Ho);
    P.Wo = (int)(dgrad ? p.W : p.Wo);
    if (P.Ho < 1 || P.Wo < 1 || P.Hs < 1 || Ws < 1) return pl;
    if (Es % 32 || Eo % 16 || Eo > 256) return pl;
    P.Ea = Es % 64 == 0 ? 64 : 32;
    P.nch = Es / P.Ea;
    P.NB = Eo;
    // row classes: taps p of class cl (Ys = s*y + p, p = cl mod s), ordered by ascending y
    P.ncls = s;
    int tp[2][8];
    for (int cl = 0; cl < s; ++cl) {
        P.ncl[cl] = 0;
        if (!dgrad) {
            for (int pp = KH - 1; pp >= 0; --pp)
                if (pp % s == cl) tp[cl][P.ncl[cl]++] = pp;
            P.pm[cl] = tp[cl][0];
        } else {
            for (int pp = 0; pp < KH; ++pp) tp[cl][P.ncl[cl]++] = pp;
            P.pm[cl] = 0;
        }
    }
    if (s == 1) P.ncl[1] = P.ncl[0], P.pm[1] = P.pm[0];
    const int nmax = std::max(P.ncl[0], P.ncl[1]);
    if (nmax * P.NB > 256 || nmax < 2) return pl;   // nothing to stack: rows_conv serves it
    P.R = std::min(kWkMaxR, 512 / P.NB);
    if (P.R < nmax + 2) return pl;
    // two TMA + MMA warp pairs (alternate strips, half the slots each) when the
    // halves still hold a window plus slack: one warp's issue rate is the limit
    // for thin rows
    P.nmw = P.R / 3 >= nmax + 2 ? 3 : P.R / 2 >= nmax + 2 ? 2 : 1;
    if (kProbes && probe_env("CAPSCONV_WK_NMW")) P.nmw = std::max(1, std::min(3, atoi(probe_env("CAPSCONV_WK_NMW"))));
    const int slack = kProbes && probe_env("CAPSCONV_WK_SLACK") ? atoi(probe_env("CAPSCONV_WK_SLACK")) : 2;
    if (P.R / P.nmw < nmax + slack) P.nmw = 1;
    P.Rw = P.R / P.nmw;
    // columns: plane q mod s, shift q / s (fwd); one plane, shift KW-1-q (dI)
    P.npl = dgrad ? 1 : s;
    const int kwp = dgrad ? KW : (KW + s - 1) / s;   // shifts per plane
    const int win = P.Wo + kwp - 1;                  // source pixels per plane an output row reads
    int box_px;
    if (win <= 32) {
        P.Xs = 8;
        while (P.Xs < win) P.Xs *= 2;
        P.G = 32 / P.Xs;
        P.nxt = 1;
        box_px = P.Xs;
    } else {
        P.Xs = 32;
        P.G = 1;
        P.nxt = (P.Wo + 31) / 32;
        box_px = 32 + kwp - 1;
    }
    if (box_px * s > 256) return pl;
    P.box_px = box_px;
    P.x0mul = dgrad ? 32 : 32 * s;
    P.x0off = dgrad ? -(KW - 1) : 0;
    P.ngi = (P.B + P.G - 1) / P.G;
    P.n_items = P.ngi * P.nxt;
    P.ys_lo = 0;
    P.ys_hi = dgrad ? P.Hs - 1 : std::min(P.Hs - 1, s * (P.Ho - 1) + KH - 1);
    const uint32_t pxb = 4u * 2u * (uint32_t)P.Ea;    // bytes per staged pixel (4 rows)
    const int plane_px = P.G * P.Xs + kwp - 1;
    P.plane_bytes = ((uint32_t)plane_px * pxb + 1023u) & ~1023u;
    P.stage_bytes = P.plane_bytes * (uint32_t)P.npl;
    P.stage_tx = (uint32_t)(P.npl * P.G * box_px) * pxb;
    for (int q = 0; q < KW; ++q) {
        const int pl_ = dgrad ? 0 : q % s, sh = dgrad ? KW - 1 - q : q / s;
        P.aoff[q] = (uint32_t)pl_ * P.plane_bytes + (uint32_t)sh * pxb;
    }
    // weight image: blocks (class, q), K-major no swizzle, Ncl = ncl * NB rows
    uint32_t off = 0;
    WkPackArgs &A = pl.pack;
    A.nblk = 0;
    for (int cl = 0; cl < s; ++cl)
        for (int q = 0; q < KW; ++q) {
            P.wof[cl][q] = off;
            A.bo[A.nblk] = off / 16;
            A.bcl[A.nblk] = cl;
            A.bq[A.nblk] = q;
            A.bN[A.nblk] = P.ncl[cl] * P.NB;
            ++A.nblk;
            off += (uint32_t)(Es * P.ncl[cl] * P.NB * 2);
        }
    if (s == 1)
        for (int q = 0; q < KW; ++q) P.wof[1][q] = P.wof[0][q];
    P.wbytes = off;
    for (int cl = 0; cl < 2; ++cl)
        for (int j = 0; j < 8; ++j) A.tp[cl][j] = (cl < s && j < P.ncl[cl]) ? tp[cl][j] : 0;
    A.dgrad = P.dgrad;
    A.KW = KW;
    A.C = (int)p.C;
    A.Cout = (int)p.Cout;
    A.NB = P.NB;
    A.Es = Es;
    A.total16 = off / 16;
    // store boxes of cw columns (swizzle span 2*cw bytes)
    P.cw = P.NB % 64 == 0 ? 64 : P.NB % 32 == 0 ? 32 : 16;
    // shared memory: [1024 barriers][stages][weights][row schedule][staging];
    // prefer >= 4 stages, then more epilogue groups, then double-buffered stores
    if (kProbes && probe_env("CAPSCONV_WK_DBG")) P.dbg = atoi(probe_env("CAPSCONV_WK_DBG"));
    P.zfill = 1;
    if (kProbes && probe_env("CAPSCONV_WK_ZFILL")) P.zfill = atoi(probe_env("CAPSCONV_WK_ZFILL"));
    P.espin = 0;
    if (kProbes && probe_env("CAPSCONV_WK_ESPIN")) P.espin = atoi(probe_env("CAPSCONV_WK_ESPIN"));
    P.est = 0;
    if (kProbes && probe_env("CAPSCONV_WK_EST")) P.est = atoi(probe_env("CAPSCONV_WK_EST"));
    const size_t limit = std::min<size_t>(kWkSmemLimit, device_info().smem_optin ? device_info().smem_optin : kWkSmemLimit);
    const uint32_t rbytes = 0u;   // the schedule lives in the kernel parameters
    int max_epi = 4, max_ey = 2;
    if (kProbes && probe_env("CAPSCONV_WK_NEPI")) max_epi = atoi(probe_env("CAPSCONV_WK_NEPI"));
    if (kProbes && probe_env("CAPSCONV_WK_EY")) max_ey = atoi(probe_env("CAPSCONV_WK_EY"));
    bool found = false;
    // candidates (epilogue groups, rows per store box, staging buffers)
    const int cand[12][3] = {{4, 2, 2}, {4, 2, 1}, {4, 1, 2}, {2, 2, 2}, {4, 1, 1}, {3, 1, 2},
                             {2, 2, 1}, {2, 1, 2}, {3, 1, 1}, {2, 1, 1}, {1, 1, 2}, {1, 1, 1}};
    // two source rows per pipeline step when >= 3 such stages fit (halves the
    // per-row waits and releases of the MMA and TMA warps), else one
    int rps_max = 2;
    if (kProbes && probe_env("CAPSCONV_WK_RPS")) rps_max = std::max(1, std::min(2, atoi(probe_env("CAPSCONV_WK_RPS"))));
    const uint32_t row_bytes = P.plane_bytes * (uint32_t)P.npl;
    for (int rps = rps_max; rps >= 1 && !found; --rps)
        for (int want = rps == 2 ? 4 : 4; want >= (rps == 2 ? 3 : 2) && !found; --want)
            for (int ci = 0; ci < 12 && !found; ++ci) {
                const int nepi = cand[ci][0], ey = cand[ci][1], nbuf = cand[ci][2];
                if (nepi > max_epi || ey > max_ey || nepi % P.nmw || P.Rw % (ey * (nepi / P.nmw)) ||
                    64 * P.nmw + 128 * nepi > 640)
                    continue;
                const uint32_t sb = (uint32_t)(nepi * nbuf * ey) * 128u * (uint32_t)P.cw * 2u;
                const uint32_t stage = row_bytes * (uint32_t)rps;
                for (int nstg = kWkMaxStg / P.nmw; nstg >= want; --nstg) {
                    const uint32_t wo = (uint32_t)(nstg * P.nmw) * stage;
                    const uint32_t ro = (wo + P.wbytes + 127u) & ~127u;
                    const uint32_t so = (ro + rbytes + 1023u) & ~1023u;
                    const size_t tot = 2048u + (size_t)so + sb + 1024u;   // + the strip lists
                    if (tot <= limit) {
                        P.rps = rps;
                        P.stage_bytes = stage;
                        P.nstg = nstg;
                        P.nepi = nepi;
                        P.ey = ey;
                        P.nbuf = nbuf;
                        P.woff_s = wo;
                        P.roff = ro;
                        P.soff = so;
                        P.sbytes = sb;
                        P.smem_bytes = (uint32_t)tot;
                        P.foff = so + sb;
                        found = true;
                        break;
                    }
                }
            }
    if (!found) return pl;
    // dynamic strip assignment when several streams share a CTA (each stream's
    // list holds the strips it takes plus the end marker)
    {
        const int grid = std::min(P.n_items, device_info().num_sms);
        P.dyn = P.nmw > 1 && (P.n_items + grid - 1) / grid + 1 <= kWkFifo;
        if (kProbes && probe_env("CAPSCONV_WK_DYN")) P.dyn = P.dyn && atoi(probe_env("CAPSCONV_WK_DYN"));
    }
    // the per-source-row schedule (identical for every strip)
    if (P.ys_hi - P.ys_lo + 1 > kWkMaxRows) return pl;
    for (int r = 0; r <= P.ys_hi - P.ys_lo; ++r) wk_make_rec(P, P.ys_lo + r, P.sched[r]);
    // the walk must touch every output row, with windows moving forward
    {
        int yfresh = 0, last_ya = 0;
        for (int Ys = P.ys_lo; Ys <= P.ys_hi; ++Ys) {
            const int cl = s == 2 ? (Ys & 1) : 0;
            const int y0 = s == 2 ? (Ys - P.pm[cl]) / 2 : Ys - P.pm[0];
            const int ya = std::max(y0, 0), yb = std::min(y0 + P.ncl[cl] - 1, P.Ho - 1);
            if (ya > yb) continue;
            if (ya < last_ya || ya > yfresh) return pl;
            last_ya = ya;
            yfresh = std::max(yfresh, yb + 1);
        }
        if (yfresh != P.Ho) return pl;
    }
    pl.ws_bytes = ((size_t)P.wbytes + 255) & ~(size_t)255;
    if (kProbes && probe_env("CAPSCONV_WK_DEBUG"))
        fprintf(stderr,
                "[wk plan] %s s=%d G=%d Xs=%d nxt=%d items=%d Ea=%d nch=%d NB=%d R=%d nmw=%d ncl=%d/%d stage=%u nstg=%d "
                "nepi=%d nbuf=%d cw=%d ey=%d rps=%d wbytes=%u smem=%u ys=[%d,%d]\n",
                dgrad ? "dI" : "fwd", s, P.G, P.Xs, P.nxt, P.n_items, P.Ea, P.nch, P.NB, P.R, P.nmw, P.ncl[0], P.ncl[1],
                P.stage_bytes, P.nstg, P.nepi, P.nbuf, P.cw, P.ey, P.rps, P.wbytes, P.smem_bytes, P.ys_lo, P.ys_hi);
    pl.ok = true;
    return pl;
}

std::shared_ptr<const WkPlan> cached_wk_plan(const Problem &p, bool dgrad) {
    static std::mutex mu;
    static std::vector<std::pair<std::vector<int64_t>, std::shared_ptr<const WkPlan>>> cache;
    const DeviceInfo &di = device_info();
    std::vector<int64_t> k = {dgrad ? 1 : 0, di.device, di.num_sms, p.dt, p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW,
                              p.D1, p.D2, p.D3, p.s, p.pad};
    std::lock_guard<std::mutex> lock(mu);
    for (auto &kv : cache)
        if (kv.first == k) return kv.second;
    if (cache.size() > 256) cache.clear();
    cache.emplace_back(k, std::make_shared<const WkPlan>(make_wk_plan(p, dgrad)));
    return cache.back().second;
}

}  // namespace

bool rows_walk_supported(capsconv_op_t op, const Problem &p) {
    if (op == CAPSCONV_OP_BWD_KERNEL) return false;
    if (kProbes && probe_env("CAPSCONV_NO_WALK")) return false;
    return cached_wk_plan(p, op == CAPSCONV_OP_BWD_DATA)->ok;
}

size_t rows_walk_workspace_bytes(capsconv_op_t op, const Problem &p) {
    std::shared_ptr<const WkPlan> pl = cached_wk_plan(p, op == CAPSCONV_OP_BWD_DATA);
    return pl->ok ? pl->ws_bytes : 0;
}

cudaError_t rows_walk_run(capsconv_op_t op, const Problem &p, const void *src, const void *K, void *out, void *ws,
                          size_t ws_bytes, cudaStream_t st) {
    const bool dgrad = op == CAPSCONV_OP_BWD_DATA;
    WkPlan pl = *cached_wk_plan(p, dgrad);
    if (!pl.ok || ws_bytes < pl.ws_bytes || ws == nullptr) return cudaErrorNotSupported;
    RowsWalk &P = pl.P;
    const int64_t Es = dgrad ? 4 * p.Cout : 4 * p.C, Eo = dgrad ? 4 * p.C : 4 * p.Cout;
    const int64_t Ws = dgrad ? p.Wo : p.W;
    if (!rows::make_rows_map5(&P.tmS, src, p.B, P.Hs, Ws, Es, P.Ea, P.box_px * P.s, 1, P.s, 1, P.G) ||
        !rows::make_rows_map5(&P.tmO, out, p.B, P.Ho, P.Wo, Eo, P.cw, P.G > 1 ? P.Xs : 32, P.ey, 1, 1, P.G))
        return cudaErrorInvalidValue;
    P.wpack = static_cast<const uint8_t *>(ws);
    P.out = static_cast<__nv_bfloat16 *>(out);
    WkPackArgs &A = pl.pack;
    A.K = static_cast<const __nv_bfloat16 *>(K);
    A.dst = static_cast<uint8_t *>(ws);
    cudaError_t e = probe_skip_pack() ? cudaSuccess
                                       : launch_pack(wk_pack_kernel, dim3((A.total16 + 63) / 64), dim3(64), 0, st, A);
    if (e != cudaSuccess) return e;
    note_launches(1);
    static unsigned long long *prof_buf = nullptr;
    if (kProbes && probe_env("CAPSCONV_WK_PROF")) {
        if (!prof_buf) cudaMalloc(&prof_buf, 148 * 8 * sizeof(unsigned long long));
        cudaMemsetAsync(prof_buf, 0, 148 * 8 * sizeof(unsigned long long), st);
        P.prof = prof_buf;
    }
    e = smem_optin(reinterpret_cast<const void *>(rows_walk_kernel), (int)P.smem_bytes);
    if (e != cudaSuccess) return e;
    const int grid = std::min(P.n_items, device_info().num_sms);
    e = launch_k(rows_walk_kernel, dim3(grid), dim3(64 * P.nmw + 128 * P.nepi), P.smem_bytes, st, P);
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
                "[wk prof] %s cycles/CTA: mma wait_full %.0f wait_acce %.0f total %.0f | epi warp2 wait %.0f rows %.0f "
                "total %.0f | tma wait_empty %.0f\n",
                dgrad ? "dI" : "fwd", a[0], a[1], a[2], a[3], a[4], a[5], a[6]);
    }
    return cudaGetLastError();
}

}  // namespace capsconv
