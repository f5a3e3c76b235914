// mma.cu -- tcgen05 / TMEM path of libcapsconv: forward and data gradient as
// one shifted-window implicit GEMM (conv_mma.cuh), plus host planning.
//
// Roles in a CTA (288 threads, persistent over work items):
//   warps 0-7  producers: stage the source window of the current channel chunk
//              into shared memory (16-byte coalesced loads; each 16 B holds
//              two D1 rows of one capsule, stored as two 8-byte pieces into the
//              K-major rows (pixel, d1) -- the D1 repack of SURVEY H1); one
//              thread also streams the prepacked weights with bulk copies.
//   warps 8-15 epilogue (two per TMEM lane quarter, alternating tiles): TMEM -> registers -> bf16 -> capsule layout in HBM.
//   warp 16    MMA issuer: for every tap, the same window at a different row
//              offset; accumulators stay in TMEM across taps and chunks
//              (the paper's output_reduce, becomes free).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <vector>

#include "conv_mma.cuh"
#include "internal.h"
#include "tma.h"
#include "umma.cuh"

namespace capsconv {
using namespace umma;

namespace {

constexpr int kMaxStages = 8;
constexpr int kMaxStg = 4;     // staging buffers


struct Item {
    int g, ig, nt, ks;
    int tile0, ntl;      // first M tile, tiles in this item
    int c_begin, c_end;  // channel chunks
};

__device__ __forceinline__ Item decode_item(const ConvMma &P, int item) {
    // every role decodes every item: host-computed reciprocals, no runtime division
    Item it;
    uint32_t r = (uint32_t)item, q;
    q = P.fd_ksplit.div(r); it.ks = (int)(r - q * (uint32_t)P.ksplit); r = q;
    q = P.fd_nnt.div(r);    it.nt = (int)(r - q * (uint32_t)P.n_ntiles); r = q;
    q = P.fd_nig.div(r);    it.ig = (int)(r - q * (uint32_t)P.n_igroups);
    it.g = (int)q * P.gpi;   // first output group of the item
    it.tile0 = it.ig * P.G;
    it.ntl = min(P.G, P.n_mtiles - it.tile0);
    it.c_begin = (int)P.fd_ksplit.div((uint32_t)(it.ks * P.nchunks));
    it.c_end = (int)P.fd_ksplit.div((uint32_t)((it.ks + 1) * P.nchunks));
    return it;
}

// floor(a / d) for any sign of a, with a host-computed reciprocal of d
__device__ __forceinline__ int fd_floor(const FastDiv &fd, int a) {
    return a >= 0 ? (int)fd.div((uint32_t)a) : -(int)fd.div((uint32_t)(-a) + fd.d - 1u);
}

#define TRACE(role, idx, ev)                                                                      \
    do {                                                                                          \
        if (kProbes && P.trace && blockIdx.x == 0 && (idx) < 64)                                             \
            P.trace[((role) * 64 + (idx)) * 4 + (ev)] = gtime();                                  \
    } while (0)


// ------------------------------------------------------------------ producers

// Window of virtual pixels [v0, v0 + len) of the current item; with the
// staging layout of whole virtual rows the window starts `off` pixels in.
__device__ __forceinline__ int window_v0(const ConvMma &P, const Item &it) {
    return it.tile0 * kTilePix + P.ib_offmin[it.g];
}
__device__ __forceinline__ int staging_off(const ConvMma &P, int v0) {
    return P.stg_batch_mode ? 0 : v0 - fd_floor(P.fd_Wg, v0) * P.Wg;
}

// rows mode: global input rows [rA, rB] covering the window [v0, v0 + win_px)
// of every plane (virtual row R = b*Hg + Y -> input rows b*H + 2Y + a)
__device__ __forceinline__ void conv_in_rows(const ConvMma &P, int v0, int &rA, int &rB) {
    const int wlo = max(v0, 0), whi = min(v0 + P.win_px, P.Bn * P.Hg * P.Wg) - 1;
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const uint32_t bA = P.fd_HgWg.div((uint32_t)wlo), bB = P.fd_HgWg.div((uint32_t)max(whi, 0));
    const int YA = (int)P.fd_Wg.div((uint32_t)wlo - bA * HgWg), YB = (int)P.fd_Wg.div((uint32_t)max(whi, 0) - bB * HgWg);
    // input rows 2Y + a - pad of both parities; rows inside the padding are not
    // staged (a window starting in the bottom padding of image bA starts at
    // row 0 of bA + 1, one ending in the top padding of bB ends in bB - 1)
    const int ylo = 2 * YA - P.src_pad, yhi = 2 * YB + 1 - P.src_pad;
    rA = ylo >= P.Hin ? ((int)bA + 1) * P.Hin : (int)bA * P.Hin + max(0, ylo);
    rB = yhi < 0 ? (int)bB * P.Hin - 1 : (int)bB * P.Hin + min(P.Hin - 1, yhi);
    rB = min(rB, P.Bin * P.Hin - 1);
    if (whi < wlo || rB < rA) rB = rA - 1;
}

// Tall-box staging: the window's source rows, image by image.  Segment of
// image b = rows [yfirst, yhi] (yfirst pulled up so the last box never runs
// past yhi; a segment occupies max(rows, h_box) staged rows), staged at row
// offset rowbase.  Slot i is image ba + i (the planner bounds the window to
// <= 4 images); slots are statically indexed so the segments stay in registers.
struct TallSegs {
    bool ok[4];
    int b[4], yfirst[4], yhi[4], rowbase[4];
};
__device__ __forceinline__ void tall_segments(const ConvMma &P, int v0, TallSegs &S) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { S.ok[i] = false; S.b[i] = S.yfirst[i] = S.yhi[i] = S.rowbase[i] = 0; }
    const int vtot = P.Bn * P.Hg * P.Wg;
    const int vlo = max(v0, 0), vhi = min(v0 + P.win_px, vtot) - 1;
    if (vhi < vlo) return;
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const int ba = (int)P.fd_HgWg.div((uint32_t)vlo), bb = (int)P.fd_HgWg.div((uint32_t)vhi);
    const int ya = (int)P.fd_Wg.div((uint32_t)vlo - (uint32_t)ba * HgWg);
    const int yb = (int)P.fd_Wg.div((uint32_t)vhi - (uint32_t)bb * HgWg);
    int rowbase = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int b = ba + i;
        const int ylo = b == ba ? ya : 0;
        const int yhi = min(b == bb ? yb : P.Hg - 1, P.src_H - 1);
        if (b > bb || yhi < ylo) continue;   // past the window, or only zero-padding rows of this image
        const int yfirst = max(0, min(ylo, yhi - P.h_box + 1));
        S.ok[i] = true; S.b[i] = b; S.yfirst[i] = yfirst; S.yhi[i] = yhi; S.rowbase[i] = rowbase;
        rowbase += max(yhi - yfirst + 1, P.h_box);
    }
}
__device__ __forceinline__ int tall_nbox(const ConvMma &P, const TallSegs &S, int k) {
    return max(1, (int)P.fd_hbox.div((uint32_t)(S.yhi[k] - S.yfirst[k] + P.h_box)));
}
__device__ __forceinline__ uint32_t tall_issue(const ConvMma &P, int v0, int ch, uint32_t stg, uint32_t mbar, bool issue) {
    TallSegs S;
    tall_segments(P, v0, S);
    const uint32_t px_bytes = (uint32_t)P.CC * 32u;
    const uint32_t box_bytes = (uint32_t)P.h_box * P.src_W * px_bytes;
    const int c0 = ch * P.CC * 16;
    uint32_t bytes = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!S.ok[k]) continue;
        const int nb = tall_nbox(P, S, k);
        for (int j = 0; j < nb; ++j) {
            const int ys = j == nb - 1 ? max(S.yfirst[k], S.yhi[k] - P.h_box + 1) : S.yfirst[k] + j * P.h_box;
            if (issue)
                tma::load4d(stg + (uint32_t)((S.rowbase[k] + ys - S.yfirst[k]) * P.src_W) * px_bytes, &P.tmap, c0, 0,
                            ys, S.b[k], mbar);
            bytes += box_bytes;
        }
    }
    return bytes;
}
// table of the window: tab[vl] = staged pixel of window pixel vl, -1 = zero
__device__ __forceinline__ void build_table_tall(const ConvMma &P, const Item &it, uint32_t tab, int tid) {
    const int v0 = window_v0(P, it);
    TallSegs S;
    tall_segments(P, v0, S);
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const int vtotal = P.Bn * P.Hg * P.Wg;
    for (int e = tid; e < P.win_px; e += kProducerThreads) {
        const int v = v0 + e;
        int idx = -1;
        if (v >= 0 && v < vtotal) {
            const uint32_t b = P.fd_HgWg.div((uint32_t)v);
            const uint32_t rr = (uint32_t)v - b * HgWg;
            const int Y = (int)P.fd_Wg.div(rr);
            const int X = (int)rr - Y * P.Wg;
            if (Y < P.src_H && X < P.src_W) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (S.ok[k] && S.b[k] == (int)b) idx = (S.rowbase[k] + Y - S.yfirst[k]) * P.src_W + X;
            }
        }
        asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(tab + (uint32_t)e * 4u), "r"(idx) : "memory");
    }
}

// TMA thread: stage the natural-layout source pixels covering the window of
// channel chunk `ch` for every plane.  Rows mode: one box per virtual row
// (Wg pixels, every pl_s-th source pixel, rows/batches outside the tensor
// read as zero).  Batch mode (Hg*Wg == 1): boxes of BB images.
__device__ __forceinline__ uint32_t issue_staging(const ConvMma &P, const Item &it, int ch, uint32_t stg,
                                                  uint32_t mbar) {
    if (P.stg_tall) return tall_issue(P, window_v0(P, it), ch, stg, mbar, true);
    if (P.I_rows) {
        int rA, rB;
        conv_in_rows(P, window_v0(P, it), rA, rB);
        if (rB < rA) return 0;
        const uint32_t nb = (uint32_t)(rB - rA + 1) * P.Win * P.CS * 32u;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         stg),
                     "l"(reinterpret_cast<const uint8_t *>(P.src) + (size_t)rA * P.Win * P.CS * 32), "r"(nb), "r"(mbar)
                     : "memory");
        return nb;
    }
    const int v0 = window_v0(P, it);
    const int len = P.win_px;
    const int c0 = ch * P.CC * 16;
    const uint32_t px_bytes = (uint32_t)P.CC * 32u;
    uint32_t bytes = 0;
    for (int k = 0; k < P.npl; ++k) {
        const uint32_t base = stg + k * P.stg_plane_bytes;
        if (P.stg_batch_mode) {
            for (int b0 = v0; b0 < v0 + len; b0 += P.BB) {
                tma::load4d(base + (uint32_t)(b0 - v0) * px_bytes, &P.tmap, c0, 0, 0, b0, mbar);
                bytes += (uint32_t)P.BB * px_bytes;
            }
        } else {
            const int Ra = fd_floor(P.fd_Wg, v0), Rb = fd_floor(P.fd_Wg, v0 + len - 1);
            for (int R = Ra; R <= Rb; ++R) {
                const int b = fd_floor(P.fd_Hg, R);
                const int Y = R - b * P.Hg;
                tma::load4d(base + (uint32_t)((R - Ra) * P.Wg) * px_bytes, &P.tmap, c0, P.pl_ox[k] - P.src_pad,
                            P.pl_s * Y + P.pl_oy[k] - P.src_pad, b, mbar);
                bytes += (uint32_t)P.Wg * px_bytes;
            }
        }
    }
    return bytes;
}



// Producers: repack the staged natural layout [pixel][c][d1][d2] into the
// K-major window rows (pixel, d1) x k-chunks (c pair, d2): each 16-byte unit
// (c, rows 2i, 2i+1) becomes two 8-byte pieces (the D1 repack of SURVEY H1).
// rows mode: tab[k*win_px + vl] = staged pixel of plane k, window pixel vl (-1: outside)
__device__ __forceinline__ void build_table(const ConvMma &P, const Item &it, uint32_t tab, int tid) {
    const int v0 = window_v0(P, it);
    int rA, rB;
    conv_in_rows(P, v0, rA, rB);
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const int vtotal = P.Bn * P.Hg * P.Wg;
    for (int e = tid; e < P.npl * P.win_px; e += kProducerThreads) {
        int k = 0, vl = e;
        while (vl >= P.win_px) { vl -= P.win_px; ++k; }
        const int v = v0 + vl;
        int idx = -1;
        if (v >= 0 && v < vtotal) {
            const uint32_t b = P.fd_HgWg.div((uint32_t)v);
            const uint32_t rr = (uint32_t)v - b * HgWg;
            const uint32_t Y = P.fd_Wg.div(rr);
            const uint32_t X = rr - Y * (uint32_t)P.Wg;
            const int y = 2 * (int)Y + P.pl_oy[k] - P.src_pad, x = 2 * (int)X + P.pl_ox[k] - P.src_pad;
            if (y >= 0 && x >= 0 && y < P.Hin && x < P.Win) idx = ((int)b * P.Hin + y - rA) * P.Win + x;
        }
        asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(tab + (uint32_t)e * 4u), "r"(idx) : "memory");
    }
}

__device__ __forceinline__ void repack_rows(const ConvMma &P, uint32_t stg, uint32_t tab, uint32_t a_stage, int tid) {
    // thread -> fixed unit (c, i); pixels advance by pstep = threads / units.
    // Plane-outer loop and batches of 4 pixels: the table loads, then the
    // staged-unit loads, then the stores, so each thread has 4 smem round
    // trips in flight instead of one dependent chain per pixel.
    const int upp = 2 * P.CC;
    const int pstep = kProducerThreads / upp;
    const int p0 = tid / upp, u2 = tid - p0 * upp;
    if (p0 >= pstep) return;
    const int c = u2 >> 1, i = u2 & 1;
    const uint32_t px_bytes = (uint32_t)P.CC * 32u;
    const uint32_t soff = (uint32_t)u2 * 16u;
    const uint32_t dcol = a_stage + (c >> 1) * P.a_lbo + (uint32_t)(2 * i) * 16u + (c & 1) * 8u;
    for (int k = 0; k < P.npl; ++k) {
        const uint32_t tabk = tab + (uint32_t)(k * P.win_px) * 4u;
        const uint32_t dstk = dcol + k * P.plane_bytes;
        for (int vl = p0; vl < P.win_px; vl += 4 * pstep) {
            int idx[4];
            uint4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                idx[j] = -1;
                if (vl + j * pstep < P.win_px)
                    asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(idx[j]) : "r"(tabk + (uint32_t)(vl + j * pstep) * 4u));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[j] = make_uint4(0, 0, 0, 0);
                if (idx[j] >= 0) v[j] = ld_shared_v4(stg + (uint32_t)idx[j] * px_bytes + soff);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (vl + j * pstep < P.win_px) {
                    const uint32_t dst = dstk + (uint32_t)(vl + j * pstep) * 64u;
                    st_shared_v2(dst, v[j].x, v[j].y);
                    st_shared_v2(dst + 16u, v[j].z, v[j].w);
                }
            }
        }
    }
}

__device__ __forceinline__ void repack_window(const ConvMma &P, const Item &it, uint32_t stg, uint32_t a_stage,
                                              int tid) {
    const int off = staging_off(P, window_v0(P, it));
    if (!P.stg_batch_mode) {
        // thread -> fixed unit (c, i), incremental (plane, pixel) counters
        // (measured: 2% faster for row staging, 8% slower for FC batch boxes)
        const int upp = 2 * P.CC;
        const int pstep = kProducerThreads / upp;
        const int p0 = tid / upp, u2 = tid - p0 * upp;
        if (p0 >= pstep) return;
        const int c = u2 >> 1, i = u2 & 1;
        const uint32_t px_bytes = (uint32_t)P.CC * 32u;
        const uint32_t src0 = stg + (uint32_t)off * px_bytes + (uint32_t)u2 * 16u;
        const uint32_t dcol = a_stage + (c >> 1) * P.a_lbo + (uint32_t)(2 * i) * 16u + (c & 1) * 8u;
        int k = 0, vl = p0;
        while (vl >= P.win_px) { vl -= P.win_px; ++k; }
#pragma unroll 2
        for (; k < P.npl;) {
            const uint4 v = ld_shared_v4(src0 + k * P.stg_plane_bytes + (uint32_t)vl * px_bytes);
            const uint32_t dst = dcol + k * P.plane_bytes + (uint32_t)vl * 64u;
            st_shared_v2(dst, v.x, v.y);
            st_shared_v2(dst + 16u, v.z, v.w);
            vl += pstep;
            while (vl >= P.win_px) { vl -= P.win_px; ++k; }
        }
        return;
    }
    const int upp = 2 * P.CC;
    const int total = P.npl * P.win_px * upp;
    const uint32_t px_bytes = (uint32_t)P.CC * 32u;
#pragma unroll 4
    for (int L = tid; L < total; L += kProducerThreads) {
        const int pix = (int)P.fd_units.div((uint32_t)L);
        const int u2 = L - pix * upp;
        const int c = u2 >> 1, i = u2 & 1;
        int k = 0, vl = pix;
        while (vl >= P.win_px) { vl -= P.win_px; ++k; }
        const uint4 v = ld_shared_v4(stg + k * P.stg_plane_bytes + (uint32_t)(vl + off) * px_bytes + (uint32_t)u2 * 16u);
        const uint32_t dst = a_stage + k * P.plane_bytes + (c >> 1) * P.a_lbo + (uint32_t)(vl * 4 + 2 * i) * 16u +
                             (c & 1) * 8u;
        st_shared_v2(dst, v.x, v.y);
        st_shared_v2(dst + 16u, v.z, v.w);
    }
}

// Epilogue store of 16 accumulator columns (4 output channels x 4) of one row
// (virtual pixel u, capsule row d1): bf16 into the capsule layout, or fp32
// split-K partials.
__device__ __forceinline__ void epi_store16(const ConvMma &P, const Item &it, const float (&v)[16], int n0, int u,
                                            int d1, bool valid, size_t opix) {
    if (P.ksplit == 1) {
        if (!valid) return;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int ch = it.nt * (P.N_tile / 4) + n0 / 4 + j;
            if (ch < P.NCH) {
                __nv_bfloat162 lo = __floats2bfloat162_rn(v[4 * j], v[4 * j + 1]);
                __nv_bfloat162 hi = __floats2bfloat162_rn(v[4 * j + 2], v[4 * j + 3]);
                uint2 w;
                w.x = *reinterpret_cast<uint32_t *>(&lo);
                w.y = *reinterpret_cast<uint32_t *>(&hi);
                *reinterpret_cast<uint2 *>(P.out + (opix * P.NCH + ch) * 16 + d1 * 4) = w;
            }
        }
    } else if (u < P.Bn * P.Hg * P.Wg) {
        const size_t rows_total = (size_t)P.n_mtiles * 128;
        const size_t ntot = (size_t)P.n_ntiles * P.N_tile;
        float *dst = P.part + ((size_t)it.ks * rows_total + (size_t)u * 4 + d1) * ntot + (size_t)it.nt * P.N_tile + n0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            reinterpret_cast<float4 *>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
}

// MMA warp: the taps of one staged chunk.  Descriptors of a tap are computed
// by the whole (converged) warp; one elected lane then issues the tap's
// KS k-steps x NTL tiles.  KS = NTL = 0: runtime counts (ks, ntl).
struct TapIssue {
    uint64_t a_desc0, b_desc0;
    uint32_t a_lbo16, b_lbo16, n_tile, idesc, d_base;
    int offmin, T0;
    bool first_chunk;
};
template <int KS, int NTL>
__device__ __forceinline__ void mma_taps(const ConvMma &P, const Item &it, const TapIssue &ti, int ks = KS,
                                         int ntl = NTL) {
    for (int gg = 0; gg < P.gpi; ++gg) {
        const int g = it.g + gg;
        const uint32_t d0 = ti.d_base + (uint32_t)(gg * P.G * P.N_tile);
        for (int t = P.og_t0[g]; t < P.og_t1[g]; ++t) {
            const uint64_t a_tap = ti.a_desc0 + ((P.tap_plane[t] * P.plane_bytes +
                                                  (uint32_t)(P.tap_shift[t] - ti.offmin) * 64u) >> 4);
            const uint64_t b_tap = ti.b_desc0 + (uint64_t)((t - ti.T0) * (P.CC / 2)) * ti.b_lbo16;
            const bool first_tap = (ti.first_chunk && t == P.og_t0[g]);
            if (elect_one()) {
                if constexpr (KS > 0) {
#pragma unroll
                    for (int j = 0; j < KS; ++j)
#pragma unroll
                        for (int gi = 0; gi < NTL; ++gi)
                            mma_bf16_ss(d0 + (uint32_t)gi * ti.n_tile,
                                        a_tap + 2u * j * ti.a_lbo16 + (uint32_t)gi * ((kTilePix * 64) >> 4),
                                        b_tap + 2u * j * ti.b_lbo16, ti.idesc, (first_tap && j == 0) ? 0u : 1u);
                } else {
                    for (int j = 0; j < ks; ++j) {
                        const uint64_t bd = b_tap + 2u * j * ti.b_lbo16;
                        const uint64_t aj = a_tap + 2u * j * ti.a_lbo16;
                        const uint32_t acc = (first_tap && j == 0) ? 0u : 1u;
                        uint32_t d = d0;
                        uint64_t ad = aj;
                        for (int gi = 0; gi < ntl; ++gi) {
                            mma_bf16_ss(d, ad, bd, ti.idesc, acc);
                            d += ti.n_tile;
                            ad += (kTilePix * 64) >> 4;
                        }
                    }
                }
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(kConvThreads, 1) conv_mma_kernel(const __grid_constant__ ConvMma P) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *a_full = bars;
    uint64_t *a_empty = bars + kMaxStages;
    uint64_t *b_full = bars + 2 * kMaxStages;
    uint64_t *acc_full = bars + 3 * kMaxStages;
    uint64_t *acc_empty = acc_full + 2;
    uint64_t *b_res = acc_empty + 2;
    uint64_t *stg_full = b_res + 1;
    uint64_t *stg_empty = stg_full + kMaxStg;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + 512);
    const uint32_t stg0 = smem_u32(smem_raw) + 1024;
    const uint32_t stage0 = stg0 + P.nstg * P.stg_bytes;
    const uint32_t stage_stride = P.a_stage_bytes + (P.b_resident ? 0u : P.b_stage_bytes);
    const uint32_t bres_addr = stage0 + P.nstages * stage_stride;

    // warp index broadcast from lane 0: role branches are then known to be
    // warp-uniform and the MMA operands stay in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
    const int lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        for (int s = 0; s < P.nstages; ++s) {
            mbar_init(a_full + s, kProducerThreads);
            mbar_init(a_empty + s, 1);
            mbar_init(b_full + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(acc_full + i, 1);
            mbar_init(acc_empty + i, kEpilogueThreads / 32);
        }
        mbar_init(b_res, 1);
        for (int i = 0; i < kMaxStg; ++i) {
            mbar_init(stg_full + i, 1);
            mbar_init(stg_empty + i, kProducerThreads);
        }
        mbar_fence_init();
    }
    constexpr int kEpiWarp0 = kProducerThreads / 32;
    constexpr int kMmaWarp = kEpiWarp0 + kEpilogueThreads / 32;
    constexpr int kTmaWarp = kMmaWarp + 1;
    // all 512 columns (one CTA per SM): the allocation then starts at column 0
    if (warp == kMmaWarp) tmem_alloc_dyn(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    if (*tmem_slot != 0u) __trap();
    constexpr uint32_t tmem = 0u;   // constant base: no R2UR per MMA

    if (warp < kEpiWarp0) {
        // ================================================= producers
        const int tid = threadIdx.x;
        if (P.b_resident && tid == 0) {
            const uint32_t bytes = (uint32_t)(P.og_t1[P.gpi - 1] - P.og_t0[0]) * (P.CC / 2) * P.N_tile * 16;
            mbar_arrive_expect_tx(b_res, bytes);
            bulk_g2s_u32(bres_addr, P.wpack, bytes, b_res);
        }
        int stage = 0, sb = 0;
        uint32_t phase = 0, sphase = 0;
        for (int item = blockIdx.x, ii = 0; item < P.n_items; item += gridDim.x, ++ii) {
            const Item it = decode_item(P, item);
            for (int ch = it.c_begin; ch < it.c_end; ++ch) {
                if (tid == 0) TRACE(0, ii, 0);
                mbar_wait(a_empty + stage, phase ^ 1);
                const uint32_t a_stage = stage0 + stage * stage_stride;
                if (!P.b_resident && tid == 0) {
                    const int t0 = P.og_t0[it.g], t1 = P.og_t1[it.g + P.gpi - 1];
                    const size_t blk = (size_t)(P.CC / 2) * P.N_tile * 16;
                    const size_t off = (((size_t)it.nt * P.nchunks + ch) * P.ntaps + t0) * blk;
                    const uint32_t bytes = (uint32_t)((t1 - t0) * blk);
                    mbar_arrive_expect_tx(b_full + stage, bytes);
                    bulk_g2s_u32(a_stage + P.a_stage_bytes, P.wpack + off, bytes, b_full + stage);
                }
                mbar_wait(stg_full + sb, sphase);
                if (tid == 0) TRACE(0, ii, 1);
                if (kProbes && (P.dbg & 64)) {
                } else if (P.I_rows || P.stg_tall) {
                    const uint32_t tab = smem_u32(smem_raw) + P.tab_off;
                    if (P.stg_tall) build_table_tall(P, it, tab, tid);
                    else build_table(P, it, tab, tid);
                    asm volatile("bar.sync 1, %0;\n" ::"r"(kProducerThreads) : "memory");
                    repack_rows(P, stg0 + sb * P.stg_bytes, tab, a_stage, tid);
                    asm volatile("bar.sync 1, %0;\n" ::"r"(kProducerThreads) : "memory");   // table reuse
                } else if (!(kProbes && (P.dbg & 1))) {
                    repack_window(P, it, stg0 + sb * P.stg_bytes, a_stage, tid);
                }
                fence_proxy_async_smem();
                mbar_arrive(a_full + stage);
                mbar_arrive(stg_empty + sb);
                if (tid == 0) TRACE(0, ii, 2);
                if (++stage == P.nstages) { stage = 0; phase ^= 1; }
                if (++sb == P.nstg) { sb = 0; sphase ^= 1; }
            }
        }
    } else if (warp < kMmaWarp) {
        // ================================================= epilogue
        const int wq = warp & 3;   // TMEM lane quarter this warp may access
        const int ehalf = (warp - kEpiWarp0) >> 2;   // which of the two warps of this quarter
        const int row = wq * 32 + lane;
        const int vtotal = P.Bn * P.Hg * P.Wg;
        const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
        int abuf = 0;
        uint32_t aphase = 0;
        for (int item = blockIdx.x, ii = 0; item < P.n_items; item += gridDim.x, ++ii) {
            const Item it = decode_item(P, item);
            if (row == 0) TRACE(2, ii, 0);
            mbar_wait(acc_full + abuf, aphase);
            if (row == 0) TRACE(2, ii, 1);
            fence_after_sync();
            // work units (output group, tile, 32-column chunk) alternate between
            // the two warps of this lane quarter -- both stay busy even for
            // one tile per item (G = 1)
            const int nch = (P.N_tile + 31) / 32;
            const int nunits = (kProbes && (P.dbg & 32)) ? 0 : P.gpi * it.ntl * nch;
            int cur_t = -1;
            int u = 0, d1 = row & 3;
            bool valid = false;
            size_t opix = 0;
            for (int w = ehalf; w < nunits; w += 2) {
                const int t = w / nch, n0 = (w - t * nch) * 32;
                const int gg = t / it.ntl, gi = t - gg * it.ntl;   // output group, tile
                if (t != cur_t) {
                    cur_t = t;
                    const int g = it.g + gg;
                    u = (it.tile0 + gi) * kTilePix + (row >> 2);
                    valid = u < vtotal;
                    opix = 0;
                    if (valid) {
                        const uint32_t b = P.fd_HgWg.div((uint32_t)u);
                        const uint32_t rr = (uint32_t)u - b * HgWg;
                        const uint32_t Y = P.fd_Wg.div(rr);
                        const uint32_t X = rr - Y * (uint32_t)P.Wg;
                        const int oy = P.og_s * (int)Y + P.og_oy[g] - P.out_pad;
                        const int ox = P.og_s * (int)X + P.og_ox[g] - P.out_pad;
                        valid = oy >= 0 && ox >= 0 && oy < P.out_H && ox < P.out_W;
                        opix = valid ? ((size_t)b * P.out_H + oy) * P.out_W + ox : 0;
                    }
                }
                const uint32_t tcol = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(((abuf * P.gpi + gg) * P.G + gi) * P.N_tile);
                {
                    float va[16], vb[16];
                    const bool two = n0 + 16 < P.N_tile;
                    if (!(kProbes && (P.dbg & 16))) {
                        tmem_ld16(tcol + n0, va);
                        if (two) tmem_ld16(tcol + n0 + 16, vb);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) va[e] = vb[e] = (float)e;
                    }
                    if (!(kProbes && (P.dbg & 4))) {
                        epi_store16(P, it, va, n0, u, d1, valid, opix);
                        if (two) epi_store16(P, it, vb, n0 + 16, u, d1, valid, opix);
                    }
                }
            }
            if (row == 0) TRACE(2, ii, 2);
            fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + abuf);
            if (row == 0) TRACE(2, ii, 3);
            if (++abuf == 2) { abuf = 0; aphase ^= 1; }
        }
    } else if (warp == kTmaWarp) {
        // ================================================= TMA staging
        if (lane == 0) {
            tma::prefetch_desc(&P.tmap);
            int sb = 0;
            uint32_t sphase = 0;
            for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
                const Item it = decode_item(P, item);
                for (int ch = it.c_begin; ch < it.c_end; ++ch) {
                    mbar_wait(stg_empty + sb, sphase ^ 1);
                    const uint32_t stg = stg0 + sb * P.stg_bytes;
                    const uint32_t mb = smem_u32(stg_full + sb);
                    if (!(kProbes && (P.dbg & 1))) {
                        // issue the copies, then arm with their byte count (the transaction
                        // count may go transiently negative; the phase cannot complete
                        // before this arrival) -- one walk over the staging plan
                        const uint32_t bytes = issue_staging(P, it, ch, stg, mb);
                        mbar_arrive_expect_tx(stg_full + sb, bytes);
                    } else {
                        mbar_arrive(stg_full + sb);
                    }
                    if (++sb == P.nstg) { sb = 0; sphase ^= 1; }
                }
            }
        }
    } else {
        // ================================================= MMA issuer
        const uint32_t idesc = idesc_bf16(128, P.N_tile, 0, 0);
        const uint32_t b_lbo = (uint32_t)P.N_tile * 16;
        int stage = 0;
        uint32_t phase = 0;
        int abuf = 0;
        uint32_t aphase = 0;
        if (P.b_resident) mbar_wait(b_res, 0);
        for (int item = blockIdx.x, ii = 0; item < P.n_items; item += gridDim.x, ++ii) {
            const Item it = decode_item(P, item);
            if (lane == 0) TRACE(1, ii, 0);
            mbar_wait(acc_empty + abuf, aphase ^ 1);
            if (lane == 0) TRACE(1, ii, 1);
            fence_after_sync();
            const int T0 = P.og_t0[it.g];
            const int offmin = P.ib_offmin[it.g];
            for (int ch = it.c_begin; ch < it.c_end; ++ch) {
                mbar_wait(a_full + stage, phase);
                if (!P.b_resident) mbar_wait(b_full + stage, phase);
                if (lane == 0) TRACE(1, ii, 2);
                fence_proxy_async_smem();   // cp.async (generic proxy) data -> tensor core (async proxy)
                fence_after_sync();
                const uint32_t a_stage = stage0 + stage * stage_stride;
                const uint32_t b_base = P.b_resident ? bres_addr : a_stage + P.a_stage_bytes;
                // descriptors: the 14-bit start-address field (16-byte units) is the low
                // bits, so a byte offset is added as (offset >> 4).
                const uint64_t a_desc0 = smem_desc(a_stage, P.a_lbo, 128);
                const uint64_t b_desc0 = smem_desc(b_base, b_lbo, 128);
                const int ksteps = P.CC / 4;
                // warp-converged tap loop; one elected lane issues the tap's
                // (k-step x tile) MMAs, fully unrolled for the common shapes
                if (!(kProbes && (P.dbg & 2))) {
                    const TapIssue ti{a_desc0, b_desc0, P.a_lbo >> 4, b_lbo >> 4, (uint32_t)P.N_tile, idesc,
                                      tmem + (uint32_t)(abuf * P.gpi * P.G * P.N_tile), offmin, T0,
                                      ch == it.c_begin};
                    const int ntl = it.ntl;
                    if (ksteps == 1 && ntl == 8) mma_taps<1, 8>(P, it, ti);
                    else if (ksteps == 1 && ntl == 2) mma_taps<1, 2>(P, it, ti);
                    else if (ksteps == 2 && ntl == 1) mma_taps<2, 1>(P, it, ti);
                    else if (ksteps == 2 && ntl == 2) mma_taps<2, 2>(P, it, ti);
                    else if (ksteps == 2 && ntl == 4) mma_taps<2, 4>(P, it, ti);
                    else if (ksteps == 2 && ntl == 8) mma_taps<2, 8>(P, it, ti);
                    else if (ksteps == 4 && ntl == 2) mma_taps<4, 2>(P, it, ti);
                    else mma_taps<0, 0>(P, it, ti, ksteps, ntl);
                }
                if (elect_one()) mma_commit(a_empty + stage);

                __syncwarp();
                if (++stage == P.nstages) { stage = 0; phase ^= 1; }
            }
            if (elect_one()) mma_commit(acc_full + abuf);
            __syncwarp();
            if (lane == 0) TRACE(1, ii, 3);
            if (++abuf == 2) { abuf = 0; aphase ^= 1; }
        }
    }

    fence_before_sync();
    __syncthreads();
    if (warp == kMmaWarp) {
        fence_after_sync();
        tmem_dealloc_dyn(tmem, 512);
    }
}

// ------------------------------------------------------------------ weight repack
// B for tap t, chunk ch, N tile nt: [kc][n][8 elements], element (k = kc*8+e, n):
//   forward : B[n=(c',d3)][k=(c,d2)]  = K[p][q][c][c'][d2][d3]
//   dgrad   : B[n=(c,d2)][k=(c',d3)]  = K[p][q][c][c'][d2][d3]
// K is viewed as [KHv][KWv][Cv][Coutv][4][4] (a full-extent layer is viewed as
// 1x1 over Cv = KH*KW*C channels, the same memory).
struct PackArgs {
    const __nv_bfloat16 *K;
    uint8_t *dst;
    int KWv, Cv, Coutv;
    int dgrad;
    int CS, NCH, CC, nchunks, ntaps, N_tile, n_ntiles;
    int tap_p[kMaxTaps], tap_q[kMaxTaps];
};

__global__ void __launch_bounds__(256) pack_weights_kernel(const __grid_constant__ PackArgs A) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    const int kcpc = A.CC / 2;
    const long long total = (long long)A.n_ntiles * A.nchunks * A.ntaps * kcpc * A.N_tile;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    long long r = idx;
    const int n = (int)(r % A.N_tile); r /= A.N_tile;
    const int kc = (int)(r % kcpc); r /= kcpc;
    const int t = (int)(r % A.ntaps); r /= A.ntaps;
    const int ch = (int)(r % A.nchunks);
    const int nt = (int)(r / A.nchunks);
    const int ng = nt * A.N_tile + n;
    const int oc = ng >> 2, dn = ng & 3;
    const int p = A.tap_p[t], q = A.tap_q[t];
    __align__(16) __nv_bfloat16 vals[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int kl = kc * 8 + e;
        const int cs = ch * A.CC + (kl >> 2);
        const int dk = kl & 3;
        __nv_bfloat16 w = __float2bfloat16_rn(0.f);
        if (cs < A.CS && oc < A.NCH) {
            size_t off;
            if (!A.dgrad)  // K[p][q][c=cs][c'=oc][d2=dk][d3=dn]
                off = ((((size_t)p * A.KWv + q) * A.Cv + cs) * A.Coutv + oc) * 16 + dk * 4 + dn;
            else           // K[p][q][c=oc][c'=cs][d2=dn][d3=dk]
                off = ((((size_t)p * A.KWv + q) * A.Cv + oc) * A.Coutv + cs) * 16 + dn * 4 + dk;
            w = A.K[off];
        }
        vals[e] = w;
    }
    *reinterpret_cast<uint4 *>(A.dst + idx * 16) = *reinterpret_cast<const uint4 *>(vals);
}

// ------------------------------------------------------------------ split-K finalize
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ ConvMma P) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    // one thread per (virtual row R = u*4 + d1, output channel)
    const long long rows = (long long)P.Bn * P.Hg * P.Wg * 4;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * P.NCH) return;
    const int ch = (int)(idx % P.NCH);
    const long long R = idx / P.NCH;
    const int u = (int)(R >> 2), d1 = (int)(R & 3);
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const uint32_t b = P.fd_HgWg.div((uint32_t)u);
    const uint32_t rr = (uint32_t)u - b * HgWg;
    const uint32_t Y = P.fd_Wg.div(rr);
    const uint32_t X = rr - Y * (uint32_t)P.Wg;
    const int g = 0;  // split-K is planned only for single-group problems
    const int oy = P.og_s * (int)Y + P.og_oy[g] - P.out_pad;
    const int ox = P.og_s * (int)X + P.og_ox[g] - P.out_pad;
    if (oy < 0 || ox < 0 || oy >= P.out_H || ox >= P.out_W) return;
    const size_t rows_total = (size_t)P.n_mtiles * 128;
    const size_t ntot = (size_t)P.n_ntiles * P.N_tile;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int ks = 0; ks < P.ksplit; ++ks) {
        const float4 v = *reinterpret_cast<const float4 *>(P.part + ((size_t)ks * rows_total + R) * ntot + ch * 4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const size_t opix = ((size_t)b * P.out_H + oy) * P.out_W + ox;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t *>(&lo);
    w.y = *reinterpret_cast<uint32_t *>(&hi);
    *reinterpret_cast<uint2 *>(P.out + (opix * P.NCH + ch) * 16 + d1 * 4) = w;
}

// ------------------------------------------------------------------ planning
struct Plan {
    bool ok = false;
    ConvMma P{};
    PackArgs pack{};
    size_t wpack_bytes = 0, part_bytes = 0;
};

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr uint32_t kSmemLimit = 227 * 1024;

Plan make_plan(const Problem &p, bool dgrad) {
    Plan pl;
    ConvMma &P = pl.P;
    if (p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4) return pl;
    const bool full_extent = (p.KH == p.H && p.KW == p.W && p.pad == 0);
    P.src_pad = dgrad ? 0 : (int)p.pad;
    P.out_pad = dgrad ? (int)p.pad : 0;
    const int s = (int)p.s;
    P.Bn = (int)p.B;
    int KWv, Cv, Coutv;
    std::vector<int> tp, tq, tplane, tshift, tgroup;
    if (full_extent) {
        // fully-connected capsule layer viewed as a 1x1 convolution over
        // KH*KW*C channels (reading R18)
        const int Ceff = (int)(p.KH * p.KW * p.C);
        KWv = 1; Cv = Ceff; Coutv = (int)p.Cout;
        P.src_H = P.src_W = 1;
        P.src_vH = P.src_vW = 1;
        P.Hg = P.Wg = 1;
        P.npl = 1; P.pl_s = 1; P.pl_oy[0] = P.pl_ox[0] = 0;
        P.CS = dgrad ? (int)p.Cout : Ceff;
        P.NCH = dgrad ? Ceff : (int)p.Cout;
        P.nog = 1; P.og_s = 1; P.og_oy[0] = P.og_ox[0] = 0;
        P.out_H = P.out_W = 1;
        tp.push_back(0); tq.push_back(0); tplane.push_back(0); tshift.push_back(0); tgroup.push_back(0);
    } else {
        if (s > 2 || p.KH * p.KW > kMaxTaps) return pl;
        if (dgrad && (p.KH < s || p.KW < s)) return pl;   // a dI phase with no taps
        KWv = (int)p.KW; Cv = (int)p.C; Coutv = (int)p.Cout;
        // the virtual grid covers the zero-padded input (pad = 0: the input)
        P.Hg = ceil_div(p.H + 2 * p.pad, s);
        P.Wg = ceil_div(p.W + 2 * p.pad, s);
        if (!dgrad) {
            P.CS = (int)p.C; P.NCH = (int)p.Cout;
            P.src_H = (int)p.H; P.src_W = (int)p.W;
            P.src_vH = (int)p.H; P.src_vW = (int)p.W;
            P.pl_s = s;
            int plane_of[2][2] = {{-1, -1}, {-1, -1}};
            P.npl = 0;
            for (int pp = 0; pp < p.KH; ++pp)
                for (int qq = 0; qq < p.KW; ++qq) {
                    const int a = pp % s, b = qq % s;
                    if (plane_of[a][b] < 0) {
                        plane_of[a][b] = P.npl;
                        P.pl_oy[P.npl] = a; P.pl_ox[P.npl] = b;
                        ++P.npl;
                    }
                    tp.push_back(pp); tq.push_back(qq);
                    tplane.push_back(plane_of[a][b]);
                    tshift.push_back((pp / s) * P.Wg + qq / s);
                    tgroup.push_back(0);
                }
            P.nog = 1; P.og_s = 1; P.og_oy[0] = P.og_ox[0] = 0;
            P.out_H = (int)p.Ho; P.out_W = (int)p.Wo;
        } else {
            P.CS = (int)p.Cout; P.NCH = (int)p.C;
            P.src_H = (int)p.Ho; P.src_W = (int)p.Wo;
            P.src_vH = (int)p.Ho; P.src_vW = (int)p.Wo;
            P.npl = 1; P.pl_s = 1; P.pl_oy[0] = P.pl_ox[0] = 0;
            P.nog = s * s; P.og_s = s;
            P.out_H = (int)p.H; P.out_W = (int)p.W;
            for (int a = 0; a < s; ++a)
                for (int b = 0; b < s; ++b) {
                    const int g = a * s + b;
                    P.og_oy[g] = a; P.og_ox[g] = b;
                    for (int pp = a; pp < p.KH; pp += s)
                        for (int qq = b; qq < p.KW; qq += s) {
                            tp.push_back(pp); tq.push_back(qq); tplane.push_back(0);
                            tshift.push_back(-((pp / s) * P.Wg + qq / s));
                            tgroup.push_back(g);
                        }
                }
        }
    }
    P.ntaps = (int)tp.size();
    for (int t = 0; t < P.ntaps; ++t) {
        P.tap_p[t] = tp[t]; P.tap_q[t] = tq[t]; P.tap_plane[t] = tplane[t]; P.tap_shift[t] = tshift[t];
    }
    int max_taps_g = 0, max_span = 0;
    for (int g = 0; g < P.nog; ++g) {
        int t0 = P.ntaps, t1 = 0, mn = 1 << 30, mx = -(1 << 30);
        for (int t = 0; t < P.ntaps; ++t)
            if (tgroup[t] == g) { t0 = std::min(t0, t); t1 = std::max(t1, t + 1); mn = std::min(mn, tshift[t]); mx = std::max(mx, tshift[t]); }
        if (t1 <= t0) return pl;
        P.og_t0[g] = t0; P.og_t1[g] = t1; P.og_offmin[g] = mn;
        max_taps_g = std::max(max_taps_g, t1 - t0);
        max_span = std::max(max_span, mx - mn);
    }
    // all output groups in one item (stride-2 dI): one staged window covering
    // every group's taps, nog accumulator sets
    int span_all = 0, offmin_all = 1 << 30;
    {
        int mx = -(1 << 30);
        for (int t = 0; t < P.ntaps; ++t) { offmin_all = std::min(offmin_all, tshift[t]); mx = std::max(mx, tshift[t]); }
        span_all = mx - offmin_all;
    }
    static const int no_merge = probe_env("CAPSCONV_NO_MERGE") ? 1 : 0;
    const long long vtotal = (long long)P.Bn * P.Hg * P.Wg;
    if (vtotal * 4 >= (1ll << 31) || (long long)P.src_H * P.src_W * P.Bn >= (1ll << 31)) return pl;

    // ---- N tiling
    const int N = P.NCH * 4;
    P.n_ntiles = ceil_div(N, 256);
    P.N_tile = ceil_div(ceil_div(N, P.n_ntiles), 16) * 16;
    // ---- channel chunks, split-K, tiles per item, stages
    P.CSpad = ceil_div(P.CS, 4) * 4;
    P.n_mtiles = ceil_div(vtotal, kTilePix);
    const int nsm = device_info().num_sms;
    const long long base_items = (long long)P.nog * P.n_ntiles * P.n_mtiles;
    std::vector<int> ccs;
    for (int cc = std::min(P.CSpad, 16); cc >= 4; cc -= 4)   // TMA box: cc*16 <= 256 elements
        if (P.CSpad % cc == 0) ccs.push_back(cc);
    bool found = false;
    ConvMma best;
    long long best_score = -1;
    static const int force_g = probe_env("CAPSCONV_FORCE_G") ? atoi(probe_env("CAPSCONV_FORCE_G")) : 0;
    const int gpis[2] = {P.nog, 1};
    for (int gq = (P.nog > 1 && !no_merge) ? 0 : 1; gq < 2; ++gq) {
    const int gpi = gpis[gq];
    if (gq == 1 && found) break;   // merged plan found: keep it
    for (int G : {8, 4, 2, 1}) {
        if (force_g && G != force_g) continue;
        for (int cc : ccs) {
            static const int force_cc = probe_env("CAPSCONV_FORCE_CC") ? atoi(probe_env("CAPSCONV_FORCE_CC")) : 0;
            if (force_cc && cc != force_cc) continue;
            const int nchunks = P.CSpad / cc;
            int ksplit = 1;
            if (base_items < nsm && P.nog == 1) {
                // split-K: at least ~2 items per SM, then the factor (up to 2x
                // that) whose items fill the last wave best; ties -> fewer partials
                const int ks0 = std::min(nchunks, ceil_div(2 * nsm, base_items));
                double best_eff = -1.0;
                for (int k = ks0; k <= std::min(nchunks, 2 * ks0); ++k) {
                    const long long it = base_items * k;
                    const double eff = (double)it / (double)(ceil_div(it, nsm) * nsm);
                    if (eff > best_eff + 1e-9) { best_eff = eff; ksplit = k; }
                }
            }
            if (2 * gpi * G * P.N_tile > 512) continue;
            const long long items = (long long)(P.nog / gpi) * P.n_ntiles * ceil_div(P.n_mtiles, G) * ksplit;
            if (G > 1 && items < 2 * nsm && !force_g) continue;
            const int span = gpi > 1 ? span_all : max_span;
            const int win_px = ((G * kTilePix + span) + 1) & ~1;
            // k-chunk planes staggered by 16 bytes mod 128: the repack's 8-byte
            // stores of a warp (lanes = (pixel, c, i) units) then hit every
            // bank exactly twice -- two wavefronts, the minimum for 256 bytes
            const uint32_t a_lbo = (uint32_t)win_px * 64 + 16;
            const uint32_t plane = (uint32_t)(cc / 2) * a_lbo;
            const uint32_t a_stage = (uint32_t)P.npl * plane;
            const uint32_t b_stage = (uint32_t)(gpi > 1 ? P.ntaps : max_taps_g) * (cc / 2) * P.N_tile * 16;
            const bool bres = (gpi == P.nog && nchunks == 1 && P.n_ntiles == 1);
            // staging of the natural layout (whole virtual rows, or BB-image boxes)
            const bool batch_mode = (P.Hg * P.Wg == 1);
            // (whole rows are staged in the natural layout: the pixel stride is
            // CS*32 bytes, so the channel count must equal the padded chunk)
            const bool rows_mode = !dgrad && !full_extent && s == 2 && nchunks == 1 && P.CS == P.CSpad;
            if (!batch_mode && !rows_mode && P.Wg * s > 256) continue;
            const int BB = std::min(win_px, 256);
            // tall boxes: unit-stride source planes outside batch/rows mode
            static const int no_tall = probe_env("CAPSCONV_NO_TALL") ? 1 : 0;
            // (only when a virtual-row box is small: <= 2.5 KB per TMA op is
            // op-rate bound, measured: L3 dI 146 -> 99 us; 3 KB rows are not)
            const bool tall_ok = !batch_mode && !rows_mode && P.pl_s == 1 && !no_tall && P.src_W <= 256 &&
                                 p.pad == 0 &&
                                 P.Wg * cc * 32 <= 2560;
            const int nrows = (win_px - 1) / P.Wg + 2;
            const int nseg = (nrows - 1) / P.Hg + 2;
            int best_st = 0, best_nstg = 0, cap = 0, hbox = 0;
            uint32_t stg_plane = 0, stg = 0, tab_bytes = 0;
            // batch mode (fully-connected view) is a streaming GEMM: deeper
            // staging keeps more HBM bytes in flight per SM
            const int max_nstg = batch_mode ? kMaxStg : 2;
            static const int force_h = probe_env("CAPSCONV_TALL_H") ? atoi(probe_env("CAPSCONV_TALL_H")) : -1;
            for (int h : {8, 4, 2, 1, 0}) {            // h = 0: one virtual row per box
                if (force_h >= 0 && h > 0 && h != force_h) continue;   // (row boxes stay the fallback)
                if (h > 0 && (!tall_ok || h > P.src_H || nseg > 4)) continue;
                if (h == 0 && tall_ok && best_st) break;
                cap = batch_mode ? ceil_div(win_px, BB) * BB
                      : rows_mode ? 2 * ((win_px - 1) / P.Wg + 2) * (int)p.W
                      : h > 0 ? (nrows + nseg * h) * P.src_W
                              : ((win_px - 1) / P.Wg + 2) * P.Wg;
                stg_plane = (uint32_t)cap * cc * 32;
                stg = rows_mode ? stg_plane : (uint32_t)P.npl * stg_plane;
                tab_bytes = (rows_mode || h > 0) ? (uint32_t)(P.npl * win_px * 4 + 15) & ~15u : 0u;
                best_st = 0; best_nstg = 0;
                for (int nstg = max_nstg; nstg >= (h > 0 ? 2 : 1) && !best_st; --nstg)
                    for (int st = std::min(kMaxStages, 4); st >= (nstg >= 2 ? 2 : 3); --st) {
                        const uint64_t bytes = 1024 + (uint64_t)nstg * stg +
                                               (uint64_t)st * (a_stage + (bres ? 0 : b_stage)) + (bres ? b_stage : 0) +
                                               tab_bytes;
                        if (bytes <= kSmemLimit) { best_st = st; best_nstg = nstg; break; }
                    }
                if (best_st) { hbox = h; break; }
            }
            if (!best_st) continue;
            P.stg_tall = hbox > 0 ? 1 : 0; P.h_box = hbox;
            P.stg_batch_mode = batch_mode ? 1 : 0; P.BB = BB; P.stg_cap_px = cap;
            P.stg_plane_bytes = stg_plane; P.stg_bytes = stg; P.nstg = best_nstg;
            P.I_rows = rows_mode ? 1 : 0;
            P.Hin = (int)p.H; P.Win = (int)p.W; P.Bin = (int)p.B;
            if (a_lbo >= (1u << 18) || b_stage >= (1u << 20)) continue;
            P.CC = cc; P.nchunks = nchunks; P.ksplit = ksplit; P.G = G; P.gpi = gpi;
            P.win_px = win_px; P.a_lbo = a_lbo; P.plane_bytes = plane;
            P.a_stage_bytes = a_stage; P.b_stage_bytes = b_stage;
            P.b_resident = bres ? 1 : 0; P.nstages = best_st;
            P.smem_bytes = 1024 + best_nstg * stg + best_st * (a_stage + (bres ? 0 : b_stage)) + (bres ? b_stage : 0) +
                           tab_bytes;
            P.tab_off = 1024 + best_nstg * stg + best_st * (a_stage + (bres ? 0 : b_stage)) + (bres ? b_stage : 0);
            // measured on the stack layers (tests/probe/gcc_sweep.sh): time
            // falls with G*CC (MMAs per staged window); at equal G*CC the
            // larger G wins (fewer items), except for stride 2, where the
            // wider chunk wins (fwd: whole-row staging needs one chunk;
            // dI: s*s phase groups each restage the window per chunk)
            const bool prefer_cc = s == 2 && !full_extent;
            const long long score = (long long)G * cc * 64 + (prefer_cc ? cc : G);
            if (!found || score > best_score) { best = P; best_score = score; }
            found = true;
        }
    }
    }
    if (!found) return pl;
    P = best;
    for (int g = 0; g < P.nog; ++g) P.ib_offmin[g] = P.gpi > 1 ? offmin_all : P.og_offmin[g];
    P.n_igroups = ceil_div(P.n_mtiles, P.G);
    P.n_items = (P.nog / P.gpi) * P.n_igroups * P.n_ntiles * P.ksplit;
    uint32_t cols = 32;
    while (cols < (uint32_t)(2 * P.gpi * P.G * P.N_tile)) cols <<= 1;
    P.tmem_cols = cols;
    P.fd_Wg.init((uint32_t)P.Wg);
    P.fd_Hg.init((uint32_t)P.Hg);
    P.fd_hbox.init((uint32_t)std::max(1, P.h_box));
    P.fd_HgWg.init((uint32_t)(P.Hg * P.Wg));
    P.fd_units.init((uint32_t)(2 * P.CC));
    P.fd_ksplit.init((uint32_t)P.ksplit);
    P.fd_nnt.init((uint32_t)P.n_ntiles);
    P.fd_nig.init((uint32_t)P.n_igroups);

    pl.wpack_bytes = align256((size_t)P.n_ntiles * P.nchunks * P.ntaps * (P.CC / 2) * P.N_tile * 16);
    pl.part_bytes = P.ksplit > 1 ? align256((size_t)P.ksplit * P.n_mtiles * 128 * P.n_ntiles * P.N_tile * 4) : 0;

    PackArgs &A = pl.pack;
    A.KWv = KWv; A.Cv = Cv; A.Coutv = Coutv; A.dgrad = dgrad ? 1 : 0;
    A.CS = P.CS; A.NCH = P.NCH; A.CC = P.CC; A.nchunks = P.nchunks; A.ntaps = P.ntaps;
    A.N_tile = P.N_tile; A.n_ntiles = P.n_ntiles;
    for (int t = 0; t < P.ntaps; ++t) { A.tap_p[t] = P.tap_p[t]; A.tap_q[t] = P.tap_q[t]; }
    pl.ok = true;
    return pl;
}

cudaError_t run_plan(Plan &pl, const void *src, const void *K, void *out, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
    ConvMma &P = pl.P;
    if (ws_bytes < pl.wpack_bytes + pl.part_bytes) return cudaErrorInvalidValue;
    static const int dbg_bits = probe_env("CAPSCONV_MMA_DBG") ? atoi(probe_env("CAPSCONV_MMA_DBG")) : 0;
    P.dbg = dbg_bits;
    uint8_t *w = static_cast<uint8_t *>(ws);
    P.src = static_cast<const __nv_bfloat16 *>(src);
    if (!make_capsule_tmap(&P.tmap, src, P.Bn, P.src_H, P.src_W, P.CS, P.CC,
                           P.stg_batch_mode ? 1 : P.stg_tall ? P.src_W : P.Wg, P.stg_tall ? P.h_box : 1,
                           P.stg_batch_mode ? P.BB : 1, P.stg_batch_mode ? 1 : P.pl_s))
        return cudaErrorInvalidValue;
    P.wpack = w;
    P.out = static_cast<__nv_bfloat16 *>(out);
    P.part = pl.part_bytes ? reinterpret_cast<float *>(w + pl.wpack_bytes) : nullptr;
    pl.pack.K = static_cast<const __nv_bfloat16 *>(K);
    pl.pack.dst = w;
    const long long npack = (long long)pl.wpack_bytes / 16;
    launch_k(pack_weights_kernel, dim3((unsigned)((npack + 255) / 256)), dim3(256), 0, st, pl.pack);
    note_launches(1);
    cudaError_t ea = smem_optin(reinterpret_cast<const void *>(conv_mma_kernel), (int)kSmemLimit);
    if (ea != cudaSuccess) return ea;
    const int grid = std::min(P.n_items, device_info().num_sms);
    static const bool tracing = probe_env("CAPSCONV_TRACE") != nullptr;
    P.trace = nullptr;
    if (tracing) {
        cudaMalloc(&P.trace, 3 * 64 * 4 * sizeof(unsigned long long));
        cudaMemset(P.trace, 0, 3 * 64 * 4 * sizeof(unsigned long long));
    }
    launch_k(conv_mma_kernel, dim3(grid), dim3(kConvThreads), P.smem_bytes, st, P);
    note_launches(1);
    if (tracing) {
        std::vector<unsigned long long> h(3 * 64 * 4);
        cudaStreamSynchronize(st);
        cudaMemcpy(h.data(), P.trace, h.size() * 8, cudaMemcpyDeviceToHost);
        cudaFree(P.trace);
        unsigned long long t0 = ~0ull;
        for (auto v : h) if (v && v < t0) t0 = v;
        const char *names[3] = {"prod", "mma ", "epi "};
        for (int i = 0; i < 20; ++i)
            for (int r = 0; r < 3; ++r) {
                fprintf(stderr, "[trace] item %2d %s", i, names[r]);
                for (int e = 0; e < 4; ++e) {
                    unsigned long long v = h[(r * 64 + i) * 4 + e];
                    fprintf(stderr, " %8lld", v ? (long long)(v - t0) : -1ll);
                }
                fprintf(stderr, "\n");
            }
    }
    if (P.ksplit > 1) {
        const long long n = (long long)P.Bn * P.Hg * P.Wg * 4 * P.NCH;
        launch_k(finalize_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, P);
        note_launches(1);
    }
    return cudaGetLastError();
}

// Plans depend only on (op, extents, device): cache them (host planning costs
// microseconds; a training step calls the same shapes every iteration).
struct PlanKey {
    int op, dt, dev, nsm;
    int64_t e[12];
    bool operator==(const PlanKey &o) const {
        if (op != o.op || dt != o.dt || dev != o.dev || nsm != o.nsm) return false;
        for (int i = 0; i < 12; ++i)
            if (e[i] != o.e[i]) return false;
        return true;
    }
};

// Entries are immutable and shared: a caller keeps its plan alive while another
// thread evicts or inserts (the returned pointer never dangles).
std::shared_ptr<const Plan> cached_plan(const Problem &p, bool dgrad) {
    static std::mutex mu;
    static std::vector<std::pair<PlanKey, std::shared_ptr<const Plan>>> cache;
    const DeviceInfo &di = device_info();
    PlanKey k{dgrad ? 1 : 0, (int)p.dt, di.device, di.num_sms, {p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW, p.D1, p.D2, p.D3, p.s, p.pad}};
    std::lock_guard<std::mutex> lock(mu);
    for (auto &kv : cache)
        if (kv.first == k) return kv.second;
    if (cache.size() > 256) cache.clear();
    cache.emplace_back(k, std::make_shared<const Plan>(make_plan(p, dgrad)));
    std::shared_ptr<const Plan> sp = cache.back().second;
    const Plan &pl = *sp;
    if (probe_env("CAPSCONV_DEBUG") && pl.ok) {
        const ConvMma &P = pl.P;
        fprintf(stderr,
                "[capsconv] mma plan: %s CS=%d NCH=%d Hg=%d Wg=%d npl=%d nog=%d taps=%d N_tile=%d n_ntiles=%d CC=%d "
                "nchunks=%d ksplit=%d G=%d mtiles=%d items=%d win_px=%d stages=%d bres=%d smem=%u tmem=%u nstg=%d "
                "stg_cap=%d batch=%d gpi=%d h_box=%d\n",
                dgrad ? "dgrad" : "fwd", P.CS, P.NCH, P.Hg, P.Wg, P.npl, P.nog, P.ntaps, P.N_tile, P.n_ntiles, P.CC,
                P.nchunks, P.ksplit, P.G, P.n_mtiles, P.n_items, P.win_px, P.nstages, P.b_resident, P.smem_bytes,
                P.tmem_cols, P.nstg, P.stg_cap_px, P.stg_batch_mode, P.gpi, P.stg_tall ? P.h_box : 0);
    }
    return sp;
}

}  // namespace

bool mma_supported(capsconv_op_t op, const Problem &p) {
    if (op == CAPSCONV_OP_BWD_KERNEL) return fc_hmma_dk_supported(p) || wgrad_supported(p);
    if (op == CAPSCONV_OP_FWD && fc_hmma_fwd_supported(p)) return true;
    if (op == CAPSCONV_OP_BWD_DATA && fc_hmma_dgrad_supported(p)) return true;
    return cached_plan(p, op == CAPSCONV_OP_BWD_DATA)->ok;
}

size_t mma_workspace_bytes(capsconv_op_t op, const Problem &p) {
    if (op == CAPSCONV_OP_BWD_KERNEL) return fc_hmma_dk_supported(p) ? fc_hmma_dk_workspace(p) : wgrad_workspace_bytes(p);
    if (op == CAPSCONV_OP_FWD && fc_hmma_fwd_supported(p)) return fc_hmma_fwd_workspace(p);
    if (op == CAPSCONV_OP_BWD_DATA && fc_hmma_dgrad_supported(p)) return fc_hmma_dgrad_workspace(p);
    std::shared_ptr<const Plan> pl = cached_plan(p, op == CAPSCONV_OP_BWD_DATA);
    return pl->ok ? pl->wpack_bytes + pl->part_bytes : 0;
}

cudaError_t mma_fwd(const Problem &p, const void *I, const void *K, void *O, void *ws, size_t ws_bytes,
                    cudaStream_t st) {
    if (fc_hmma_fwd_supported(p)) return fc_hmma_fwd(p, I, K, O, ws, ws_bytes, st);
    Plan pl = *cached_plan(p, false);
    if (!pl.ok) return cudaErrorNotSupported;
    return run_plan(pl, I, K, O, ws, ws_bytes, st);
}

cudaError_t mma_bwd_data(const Problem &p, const void *dO, const void *K, void *dI, void *ws, size_t ws_bytes,
                         cudaStream_t st) {
    if (fc_hmma_dgrad_supported(p)) return fc_hmma_dgrad(p, dO, K, dI, ws, ws_bytes, st);
    Plan pl = *cached_plan(p, true);
    if (!pl.ok) return cudaErrorNotSupported;
    return run_plan(pl, dO, K, dI, ws, ws_bytes, st);
}

cudaError_t mma_bwd_kernel(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                           cudaStream_t st) {
    if (fc_hmma_dk_supported(p)) return fc_hmma_dk(p, I, dO, dK, ws, ws_bytes, st);
    return wgrad_run(p, I, dO, dK, ws, ws_bytes, st);
}

}  // namespace capsconv
