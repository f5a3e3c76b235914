// wgrad.cu -- the kernel gradient dK on tcgen05 / TMEM.
//
// Algorithm 4 (output_extend -> strided_batched_matrix_
// multiply(O'_d, I') -> reduce to K_diff), read as the adjoint (DESIGN.md
// R10/R11):
//     dK[p,q,c,c',d2,d3] = sum_{b,x',y',d1} I[b, x's+p, y's+q, c, d1, d2] * dO[b,x',y',c',d1,d3]
// is one long-K GEMM per tap with M = (c, d2), N = (c', d3) and the reduction
// K = (virtual pixel v, d1).  The paper's replicated I'/O'_d buffers and its
// separate reduction pass become: a TMA-staged window of I and dO per stage,
// repacked in shared memory into MN-major operands (the D1 row transpose of a
// capsule is an 8-byte shuffle no TMA layout can express), and fp32
// accumulation in TMEM across the whole pixel range of a work item.
//
// M packing: one 128-row M tile holds several *slots* (tap, channel range);
// each slot is the staged input window read at that tap's shift, so small
// C (4*C < 128) still fills the tensor core.  Work items = (M tile, split of
// the pixel range); split partials are summed in a fixed order by a
// finalize kernel (deterministic, no atomics).
//
// Operands: A (rows m = slot (c, d2), K = (v, d1)) lives in TENSOR MEMORY:
// loader warps read each capsule row from the staged window (one 8-byte load
// per lane), transpose the 4x4 capsule in registers (d1 <-> d2, two shuffle
// rounds) and write the slot's shifted copy with tcgen05.st straight into the
// lane quarter it owns -- no shared-memory round trip for the replicated
// operand, and the TS-form MMA avoids re-reading A from shared memory
// (measured ~2x cheaper than SS at N = 32).  B (dO, columns (c', d3)) is one
// MN-major shared-memory operand.  A CTA accumulates a group of M tiles over
// a pixel range, so the staged window is shared by all the taps it holds.
//
// Roles (576 threads): warps 0-11 loaders (three per TMEM lane quarter),
// warps 12-15 epilogue, warp 16 MMA, warp 17 TMA.
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

// 16 loader warps (four per TMEM lane quarter); they also run the epilogue
// at the end of each work item (a CTA holds ~one item, so dedicated epilogue
// warps would idle through the whole main loop)
constexpr int kWLoad = 512, kWEpi = 0;
constexpr int kWThreads = kWLoad + kWEpi + 64;
constexpr int kWMaxTiles = 96;
constexpr int kWMaxSlots = 4;
constexpr int kWMaxStages = 4;

struct WSlot {
    int tap, plane, shift, c0, cn, row0;   // rows [row0, row0 + 4*cn) of the tile
    FastDiv fd_upp;                        // 2*cn units per pixel
};

struct WTile {
    int nslots;
    WSlot slot[kWMaxSlots];
    int np;                                // distinct input planes staged for this tile
    int plane[kWMaxSlots];
    int minsh[kWMaxSlots], span[kWMaxSlots];
    int c_lo, c_hi;                        // staged channel range
};

struct WgradMma {
    alignas(64) CUtensorMap tm_I;
    alignas(64) CUtensorMap tm_O;
    float *part;                           // [ksplit][KH*KW*C*Cout*16] (ksplit > 1) or dK itself
    int Bn, Hg, Wg, vtotal;
    FastDiv fd_Wg, fd_HgWg;
    int batch_mode;                        // Hg*Wg == 1 (fully-connected view)
    int C, Cout, ntaps, s;
    int pl_oy[4], pl_ox[4];
    int n_mtiles;
    WTile tile[kWMaxTiles];
    int TG, n_groups;                      // M tiles per CTA group, groups
    int g_np[kWMaxTiles];                  // per group: staged I planes (union over its tiles)
    int g_plane[kWMaxTiles][4], g_minsh[kWMaxTiles][4], g_span[kWMaxTiles][4];
    int g_clo[kWMaxTiles], g_chi[kWMaxTiles];
    uint32_t acc_cols, abuf_cols;          // TMEM: accumulators, then A buffers
    int N_tile;
    int KP;                                // virtual pixels per stage (multiple of 4)
    int ksplit, kpix;                      // pixels per split (multiple of KP)
    int n_items;
    int CBI, CBO;                          // channels per TMA box (I, dO)
    FastDiv fd_uppO;                       // 2*Cout units per pixel
    int capI, capO;                        // staging capacity (pixels) per I plane / for dO
    uint32_t stgI_plane, stgI_bytes, stgO_bytes, stg_bytes;
    uint32_t b_sbo, b_bytes;
    int nstg, nstages;
    uint32_t smem_bytes, tmem_cols;
    unsigned long long *trace;             // debug: globaltimer stamps of CTA 0 [role][stage][4]
    int dbg;                               // bench-only (wrong results): 1 skip transpose, 2 skip MMAs, 4 skip B, 16 skip A
    // contiguous staging (1-D bulk copies): dO always; I when stride 1 (not FC)
    const uint8_t *I_ptr, *O_ptr;
    int I_contig;
    // stride-2 input planes: whole contiguous input rows (both parities) are
    // staged with one bulk copy; a per-stage table maps plane pixels to them
    int I_rows;
    int Hin, Win, Bin;
    int TABW;                              // table entries per plane
    uint32_t tab_off;                      // tables (per staging buffer) offset from the dynamic smem base
    uint32_t tab_stride;                   // bytes of tables per staging buffer
    uint32_t btab_off;                     // B source table offset inside a buffer's tables
    // column shifts: B holds nq copies of the dO window,
    // copy j read at virtual pixel u - j, side by side in N; D column block j
    // of a slot for tap (p, q) is the gradient of tap (p, q + s*j)
    int nq, KWv;
    int tiles_uniform;   // FC view with more tiles than the table holds: tile mt = tile[0] shifted by 32*mt channels
    int pad;       // zero padding: input coordinates are virtual - pad (tensor-map boxes zero-fill outside)
    int b_pstep;                           // staged dO pixels per B-loader iteration (loader threads / (2*Cout))
    // bdesc: B holds ONE dO copy over KP + nq - 1 pixels; copy j is the same
    // buffer at descriptor offset (nq-1-j) pixels (64 B), one N = 4*Cout MMA per copy
    int bdesc;
    int bmat;      // bdesc: materialised copies F_a[e] = F_0[e + a], a < bmat, side by side in N;
                   // accumulator block bi (columns bi*4*Cout) is shift j = nq-1-bi
    // loader groups: stage s is built by group s % lgroups (lgroups divides nstg
    // and nstages, so every buffer always belongs to one group); the groups
    // work on different stages concurrently
    int lgroups;   // stage s is built by group s % lgroups
    int Ho, Wo;                            // dO extents (rows per image, pixels per row)
};
#define WTRACE(role, idx, ev)                                                              \
    do {                                                                                   \
        if (kProbes && P.trace && blockIdx.x == 0 && (idx) < 64) P.trace[((role) * 64 + (idx)) * 4 + (ev)] = gtime(); \
    } while (0)

__device__ __forceinline__ void wdecode(const WgradMma &P, int item, int &mt, int &ks, int &p0, int &p1) {
    ks = item % P.ksplit;
    mt = item / P.ksplit;                  // group index
    // balanced split of the nst = ceil(vtotal / KP) stages: split ks owns
    // stages [ks*nst/ksplit, (ks+1)*nst/ksplit)
    const int nst = (P.vtotal + P.KP - 1) / P.KP;
    p0 = (int)((long long)ks * nst / P.ksplit) * P.KP;
    p1 = min(P.vtotal, (int)((long long)(ks + 1) * nst / P.ksplit) * P.KP);
}

// Rows mode: the window [v0, v0 + len) as whole virtual rows; returns the
// staging pixel offset of v0.  Batch mode: boxes of KP images at v0.
__device__ __forceinline__ uint32_t w_stage_window(const WgradMma &P, const CUtensorMap *tm, int v0, int len,
                                                   int cb, int nbox, int c_first, int ox, int oy, int cs, int cap,
                                                   uint32_t dst, uint32_t mbar, bool issue, int &box_id, int lane) {
    // issue: every box gets an index; lane `lane` issues the boxes with index % 32 == lane
    const uint32_t px = (uint32_t)cb * 32u;
    uint32_t bytes = 0;
    for (int bx = 0; bx < nbox; ++bx) {
        const uint32_t base = dst + (uint32_t)bx * cap * px;
        const int c0 = (c_first + bx * cb) * 16;
        if (P.batch_mode) {
            if (issue && (box_id & 31) == lane) tma::load4d(base, tm, c0, 0, 0, v0, mbar);
            ++box_id;
            bytes += (uint32_t)P.KP * px;
        } else {
            const int Ra = floor_div(v0, P.Wg), Rb = floor_div(v0 + len - 1, P.Wg);
            for (int R = Ra; R <= Rb; ++R) {
                if (issue && (box_id & 31) == lane) {
                    const int b = floor_div(R, P.Hg);
                    const int Y = R - b * P.Hg;
                    tma::load4d(base + (uint32_t)((R - Ra) * P.Wg) * px, tm, c0, ox - P.pad, cs * Y + oy - P.pad, b,
                                mbar);
                }
                ++box_id;
                bytes += (uint32_t)P.Wg * px;
            }
        }
    }
    return bytes;
}

__device__ __forceinline__ int w_off(const WgradMma &P, int v0) {
    return P.batch_mode ? 0 : v0 - floor_div(v0, P.Wg) * P.Wg;
}

// dO rows [ra, rb) (global row index b*Ho + Y) covering virtual pixels [v0, v0 + KP)
// (v0 >= 0 on the forward grid; FastDiv: no runtime integer division)
__device__ __forceinline__ void w_dO_rows(const WgradMma &P, int v0, int &ra, int &rb) {
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const uint32_t va = (uint32_t)max(v0 - (P.nq - 1), 0), vb = (uint32_t)(min(v0 + P.KP, P.vtotal) - 1);
    const uint32_t ba = P.fd_HgWg.div(va), bb = P.fd_HgWg.div(vb);
    const int ya = (int)P.fd_Wg.div(va - ba * HgWg), yb = (int)P.fd_Wg.div(vb - bb * HgWg);
    ra = ya < P.Ho ? (int)ba * P.Ho + ya : ((int)ba + 1) * P.Ho;
    rb = yb < P.Ho ? (int)bb * P.Ho + yb + 1 : ((int)bb + 1) * P.Ho;
}

__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void *src, uint32_t bytes, uint64_t *, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

// stride-2 rows mode: global input rows [rA, rB] covering every plane window
// of the stage (virtual rows R = b*Hg + Y map to input rows b*H + 2Y + a)
// rows mode: global input rows [rA, rB] covering every plane window of the
// stage (virtual row Y of image b is input row s*Y + oy - pad of plane oy;
// rows outside the image are padding and are not staged)
__device__ __forceinline__ void w_in_rows(const WgradMma &P, int wlo, int whi, int &rA, int &rB) {
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const uint32_t bA = P.fd_HgWg.div((uint32_t)wlo), bB = P.fd_HgWg.div((uint32_t)whi);
    const int YA = (int)P.fd_Wg.div((uint32_t)wlo - bA * HgWg), YB = (int)P.fd_Wg.div((uint32_t)whi - bB * HgWg);
    // a window starting in the bottom padding of image bA starts at row 0 of
    // bA + 1; one ending in the top padding of bB ends at the last row of bB - 1
    const int ylo = P.s * YA - P.pad, yhi = P.s * YB + P.s - 1 - P.pad;
    rA = ylo >= P.Hin ? ((int)bA + 1) * P.Hin : (int)bA * P.Hin + max(0, ylo);
    rB = yhi < 0 ? (int)bB * P.Hin - 1 : (int)bB * P.Hin + min(P.Hin - 1, yhi);
    rB = min(rB, P.Bin * P.Hin - 1);
    if (rB < rA) rB = rA - 1;
}

struct WGroup {
    int np, nbI, clo;
    int minsh[4], span[4], ox[4], oy[4];
};

__device__ __forceinline__ void w_group_setup(const WgradMma &P, int g, WGroup &G) {
    G.np = P.g_np[g];
    G.clo = P.g_clo[g];
    G.nbI = (P.g_chi[g] - G.clo + P.CBI - 1) / P.CBI;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int pl = k < G.np ? P.g_plane[g][k] : 0;
        G.minsh[k] = k < G.np ? P.g_minsh[g][k] : 0;
        G.span[k] = k < G.np ? P.g_span[g][k] : 0;
        G.ox[k] = P.pl_ox[pl];
        G.oy[k] = P.pl_oy[pl];
    }
}

__device__ __forceinline__ uint32_t w_issue(const WgradMma &P, const WGroup &G, int v0, uint32_t stg, uint32_t mbar,
                                            bool issue, int lane) {
    uint32_t bytes = 0;
    int box_id = 0;
    if (P.I_rows) {
        int wlo = 1 << 30, whi = -1;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < G.np) { wlo = min(wlo, v0 + G.minsh[k]); whi = max(whi, v0 + G.minsh[k] + P.KP + G.span[k] - 1); }
        int rA, rB;
        w_in_rows(P, wlo, min(whi, P.vtotal - 1), rA, rB);
        if (rB >= rA) {
            const uint32_t nb = (uint32_t)(rB - rA + 1) * P.Win * P.C * 32u;
            if (issue && lane == 0) bulk_g2s_u32(stg, P.I_ptr + (size_t)rA * P.Win * P.C * 32, nb, (uint64_t *)0, mbar);
            bytes += nb;
        }
        ++box_id;
    } else if (P.I_contig) {
        // stride 1: the window of input pixels is contiguous in memory (one plane, all channels)
        const int lo = v0 + G.minsh[0];
        const int hi = min(v0 + P.KP + G.span[0] + G.minsh[0], P.vtotal);
        if (hi > lo) {
            const uint32_t nb = (uint32_t)(hi - lo) * P.C * 32u;
            if (issue && lane == 0) bulk_g2s_u32(stg, P.I_ptr + (size_t)lo * P.C * 32, nb, (uint64_t *)0, mbar);
            bytes += nb;
        }
        ++box_id;
    } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k >= G.np) break;
        bytes += w_stage_window(P, &P.tm_I, v0 + G.minsh[k], P.KP + G.span[k], P.CBI, G.nbI, G.clo, G.ox[k],
                                G.oy[k], P.s, P.capI, stg + k * P.stgI_plane, mbar, issue, box_id, lane);
    }
    }
    // dO: the valid rows of the window are consecutive rows of the dO tensor
    int ra, rb;
    w_dO_rows(P, v0, ra, rb);
    if (rb > ra) {
        const uint32_t nb = (uint32_t)(rb - ra) * P.Wo * P.Cout * 32u;
        if (issue && lane == (box_id & 31))
            bulk_g2s_u32(stg + P.stgI_bytes, P.O_ptr + (size_t)ra * P.Wo * P.Cout * 32, nb, (uint64_t *)0 + 0, mbar);
        bytes += nb;
    }
    ++box_id;
    return bytes;
}

// B source table: entry e (0 <= e < KP + nq - 1) = staged dO pixel of
// virtual pixel v0 - (nq - 1) + e, or -1 (outside dO: a zero row of B)
__device__ __forceinline__ void w_build_btab(const WgradMma &P, int v0, uint32_t btab, int tid, int nthr) {
    int ra, rb;
    w_dO_rows(P, v0, ra, rb);
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    const int n = P.KP + P.nq - 1;
    for (int e = tid; e < n; e += nthr) {
        const int vv = v0 - (P.nq - 1) + e;
        int idx = -1;
        if (vv >= 0 && vv < P.vtotal) {
            const uint32_t bq = P.fd_HgWg.div((uint32_t)vv);
            const uint32_t rr = (uint32_t)vv - bq * HgWg;
            const uint32_t Y = P.fd_Wg.div(rr);
            const uint32_t X = rr - Y * (uint32_t)P.Wg;
            if ((int)Y < P.Ho && (int)X < P.Wo) idx = ((int)bq * P.Ho + (int)Y - ra) * P.Wo + (int)X;
        }
        asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(btab + (uint32_t)e * 4u), "r"(idx) : "memory");
    }
}

// dO -> B: MN-major shared-memory operand, columns n = (j, c', d3) in groups
// of 8 (c' pair), k-rows (v, d1) at 16 bytes; a capsule unit (c', d1 rows
// 2i, 2i+1) becomes two 8-byte pieces (the D1 transpose).  Copy j holds
// dO[v - j]: each staged unit is loaded once and stored into every copy
// whose local row falls inside the stage.
constexpr int kWMaxNq = 4;
// loader group lg of NG: warps [lg*16/NG, (lg+1)*16/NG) (sizes differ by at most one warp)
__host__ __device__ __forceinline__ int w_group_w0(int lg, int ng) { return lg * (kWLoad / 32) / ng; }

__device__ __forceinline__ void w_load_B(const WgradMma &P, uint32_t stg, uint32_t btab, uint32_t b, int tid,
                                         int pstep) {
    // thread -> fixed unit (c', i) of a staged pixel; pixels advance by
    // P.b_pstep per iteration (b_pstep * upp <= loader threads): no division
    const uint32_t base = stg + P.stgI_bytes;
    const int upp = 2 * P.Cout;
    const int pix0 = tid / upp;                 // once per stage
    const int u = tid - pix0 * upp;
    if (pix0 >= pstep) return;
    const int c = u >> 1, i = u & 1;
    const uint32_t pxb = (uint32_t)P.Cout * 32u;
    const uint32_t src_off = (uint32_t)(c * 32 + i * 16);
    const int npx = P.KP + P.nq - 1;
    uint32_t dcol[kWMaxNq];                     // per copy: column-group offset of this unit
#pragma unroll
    for (int j = 0; j < kWMaxNq; ++j) {
        const int col = j * P.Cout + c;
        dcol[j] = b + (uint32_t)(col >> 1) * P.b_sbo + (uint32_t)(2 * i) * 16u + (col & 1) * 8u;
    }
    if (P.bdesc) {
#pragma unroll 4
        for (int e = pix0; e < npx; e += pstep) {
            int idx;
            asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(idx) : "r"(btab + (uint32_t)e * 4u));
            uint4 v = make_uint4(0, 0, 0, 0);
            if (idx >= 0) v = ld_shared_v4(base + (uint32_t)idx * pxb + src_off);
            const uint32_t dst = dcol[0] + (uint32_t)e * 64u;
            st_shared_v2(dst, v.x, v.y);
            st_shared_v2(dst + 16u, v.z, v.w);
            if (P.bmat > 1 && e >= 1) {          // F_1[e - 1] = F_0[e]
                const uint32_t d1 = dcol[1] + (uint32_t)(e - 1) * 64u;
                st_shared_v2(d1, v.x, v.y);
                st_shared_v2(d1 + 16u, v.z, v.w);
            }
        }
        return;
    }
#pragma unroll 4
    for (int e = pix0; e < npx; e += pstep) {
        int idx;
        asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(idx) : "r"(btab + (uint32_t)e * 4u));
        uint4 v = make_uint4(0, 0, 0, 0);
        if (idx >= 0) v = ld_shared_v4(base + (uint32_t)idx * pxb + src_off);
#pragma unroll
        for (int j = 0; j < kWMaxNq; ++j) {
            const int l = e - (P.nq - 1) + j;     // local row of copy j
            if (j < P.nq && l >= 0 && l < P.KP) {
                const uint32_t dst = dcol[j] + (uint32_t)l * 64u;
                st_shared_v2(dst, v.x, v.y);
                st_shared_v2(dst + 16u, v.z, v.w);
            }
        }
    }
}

// 4x4 transpose of bf16 capsule rows across the 4 lanes of a group:
// lane d1 holds row d1 (lo = d2 0..1, hi = d2 2..3); afterwards lane d2 holds
// column d2 (lo = d1 0..1, hi = d1 2..3).
__device__ __forceinline__ void transpose4x4(uint32_t &lo, uint32_t &hi, int r) {
    const uint32_t t = (r & 2) ? lo : hi;
    const uint32_t x = __shfl_xor_sync(0xffffffffu, t, 2);
    if (r & 2) lo = x; else hi = x;
    const uint32_t plo = __shfl_xor_sync(0xffffffffu, lo, 1);
    const uint32_t phi = __shfl_xor_sync(0xffffffffu, hi, 1);
    if (r & 1) {
        lo = __byte_perm(lo, plo, 0x3276);
        hi = __byte_perm(hi, phi, 0x3276);
    } else {
        lo = __byte_perm(lo, plo, 0x5410);
        hi = __byte_perm(hi, phi, 0x5410);
    }
}

// Transpose every staged input capsule in place (rows d1 -> columns d2), once
// per stage, so the per-slot loads below are plain 8-byte reads of a column.
// Lane groups of 4 own one 32-byte capsule.
__device__ __forceinline__ void w_transpose_stage(uint32_t base, uint32_t bytes, int tid, int nthr) {
    const int lane = tid & 31;
    const uint32_t n8 = bytes / 8;                      // 8-byte rows
    const uint32_t kStep = (uint32_t)nthr;
    constexpr int kU = 4;                               // independent rows in flight per lane
    // all lanes of a warp iterate together (shuffles need the full warp)
    for (uint32_t r0 = (uint32_t)(tid - lane); r0 < n8; r0 += kU * kStep) {
        uint32_t lo[kU], hi[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t r = r0 + u * kStep + (uint32_t)lane;
            lo[u] = 0; hi[u] = 0;
            if (r < n8) asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];\n" : "=r"(lo[u]), "=r"(hi[u]) : "r"(base + r * 8u));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) transpose4x4(lo[u], hi[u], lane & 3);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t r = r0 + u * kStep + (uint32_t)lane;
            if (r < n8) st_shared_v2(base + r * 8u, lo[u], hi[u]);
        }
    }
}

__device__ __forceinline__ void st_shared_v4z(uint32_t addr) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};\n" ::"r"(addr), "r"(0) : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// I -> A in TMEM for every tile of the group: this warp owns lane quarter q
// (rows q*32 .. q*32+31 of each tile) and k-steps kk = part (mod kParts).
// Lane group lane/4 is one (slot, channel), lane & 3 the capsule column d2:
// the staged capsules were transposed in place, so the 8 bytes at offset
// d2*8 are (d1 = 0..3) of column d2 -- two TMEM columns of the A operand.  The per-tile
// addressing is computed once per work item (WLane) -- the tile tables are
// large kernel parameters and must not be re-read per stage.
constexpr int kWMaxTG = 8;
struct WLane {
    uint32_t loff[kWMaxTG];   // lane offset inside a staged pixel: channel box + capsule column
    uint32_t base[kWMaxTG];   // staging byte offset of this lane's capsule row at window pixel 0 (minus plane start)
    int kpl[kWMaxTG];         // staged plane index (-1: padding row)
    int sp0[kWMaxTG];         // staged pixel (within its plane window) read for stage pixel 0
    int ntl, np;
    uint32_t live;            // bit tt: some lane of this warp holds a real row of tile tt
    int minsh[4];
};

__device__ __forceinline__ void w_lane_setup(const WgradMma &P, int g, int q, int lane, WLane &L) {
    const uint32_t pxb = (uint32_t)P.CBI * 32u;
    const int row = q * 32 + lane;
    const int d1 = lane & 3;
    L.ntl = min(P.TG, P.n_mtiles - g * P.TG);
    L.np = P.g_np[g];
#pragma unroll
    for (int k = 0; k < 4; ++k) L.minsh[k] = k < L.np ? P.g_minsh[g][k] : 0;
#pragma unroll
    for (int tt = 0; tt < kWMaxTG; ++tt) {
        L.kpl[tt] = -1;
        L.base[tt] = 0;
        L.loff[tt] = 0;
        L.sp0[tt] = 0;
        if (tt >= L.ntl) continue;
        const WTile &T = P.tile[P.tiles_uniform ? 0 : g * P.TG + tt];
        const int cshift = P.tiles_uniform ? (g * P.TG + tt) * 32 : 0;
        for (int j = 0; j < T.nslots; ++j) {
            const WSlot &S = T.slot[j];
            if (row >= S.row0 && row < S.row0 + 4 * S.cn) {
                const int c = S.c0 + cshift + ((row - S.row0) >> 2);
                if (c >= P.C) break;
                int k = 0;
                while (P.g_plane[g][k] != S.plane) ++k;
                const int cl = c - P.g_clo[g];
                const int bx = cl / P.CBI, cc = cl - bx * P.CBI;
                L.kpl[tt] = k;
                L.sp0[tt] = S.shift - P.g_minsh[g][k];
                L.loff[tt] = (uint32_t)bx * P.capI * pxb + (uint32_t)(cc * 32 + d1 * 8);
                L.base[tt] = k * P.stgI_plane + (uint32_t)bx * P.capI * pxb +
                             (uint32_t)(S.shift - P.g_minsh[g][k]) * pxb + (uint32_t)(cc * 32 + d1 * 8);
            }
        }
    }
    L.live = 0;
#pragma unroll
    for (int tt = 0; tt < kWMaxTG; ++tt)
        if (__any_sync(0xffffffffu, L.kpl[tt] >= 0)) L.live |= 1u << tt;
}

// Rows mode: table[k][w] = staged pixel of plane k's window position w
// (window of plane k starts at v0 + minsh_k), -1 outside the input.
__device__ __forceinline__ void w_build_table(const WgradMma &P, const WGroup &G, int v0, uint32_t tab, int tid,
                                              int nthr) {
    int wlo = 1 << 30, whi = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (k < G.np) { wlo = min(wlo, v0 + G.minsh[k]); whi = max(whi, v0 + G.minsh[k] + P.KP + G.span[k] - 1); }
    int rA, rB;
    w_in_rows(P, wlo, min(whi, P.vtotal - 1), rA, rB);
    const uint32_t HgWg = (uint32_t)(P.Hg * P.Wg);
    for (int e = tid; e < 4 * P.TABW; e += nthr) {
        const int k = e / P.TABW, w = e - k * P.TABW;
        int idx = -1;
        if (k < G.np && w < P.KP + G.span[k]) {
            const int v = v0 + G.minsh[k] + w;
            if (v < P.vtotal) {
                const uint32_t b = P.fd_HgWg.div((uint32_t)v);
                const uint32_t rr = (uint32_t)v - b * HgWg;
                const uint32_t Y = P.fd_Wg.div(rr);
                const uint32_t X = rr - Y * (uint32_t)P.Wg;
                const int y = P.s * (int)Y + G.oy[k] - P.pad, x = P.s * (int)X + G.ox[k] - P.pad;
                if (y >= 0 && x >= 0 && y < P.Hin && x < P.Win) idx = ((int)b * P.Hin + y - rA) * P.Win + x;
            }
        }
        asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(tab + (uint32_t)e * 4u), "r"(idx) : "memory");
    }
}

__device__ __forceinline__ void w_load_A_rows(const WgradMma &P, const WLane &L, uint32_t stg, uint32_t tab,
                                              uint32_t zero8, uint32_t tm_a, int q, int part, int kParts) {
    const uint32_t pxb = (uint32_t)P.CBI * 32u;
    const int nk = P.KP / 4;
    const uint32_t lane_q = (uint32_t)(q * 32) << 16;
#pragma unroll
    for (int tt = 0; tt < kWMaxTG; ++tt) {
        if (tt >= L.ntl) break;
        if (!((L.live >> tt) & 1u)) continue;   // rows of this lane quarter are all padding: never stored
        const int k = L.kpl[tt] < 0 ? 0 : L.kpl[tt];
        const uint32_t trow = tab + (uint32_t)(k * P.TABW + L.sp0[tt]) * 4u;
        const uint32_t dcol = tm_a + lane_q + (uint32_t)(tt * nk * 8);
        // two k-steps per batch (independent table and data loads in flight)
        for (int kk = part; kk < nk; kk += 2 * kParts) {
            const bool two = kk + kParts < nk;
            const int kk2 = two ? kk + kParts : kk;
            int idx[8];
#pragma unroll
            for (int px = 0; px < 4; ++px)
                asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(idx[px]) : "r"(trow + (uint32_t)(kk * 4 + px) * 4u));
#pragma unroll
            for (int px = 0; px < 4; ++px)
                asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(idx[4 + px]) : "r"(trow + (uint32_t)(kk2 * 4 + px) * 4u));
            uint32_t r[16];
#pragma unroll
            for (int px = 0; px < 8; ++px) {
                const uint32_t a = idx[px] >= 0 ? stg + (uint32_t)idx[px] * pxb + L.loff[tt] : zero8;
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];\n" : "=r"(r[2 * px]), "=r"(r[2 * px + 1]) : "r"(a));
            }
            tmem_st8(dcol + (uint32_t)(kk * 8), *reinterpret_cast<const uint32_t(*)[8]>(r));
            if (two) tmem_st8(dcol + (uint32_t)(kk2 * 8), *reinterpret_cast<const uint32_t(*)[8]>(r + 8));
        }
    }
}

__device__ __forceinline__ void w_load_A(const WgradMma &P, const WLane &L, int v0, uint32_t stg, uint32_t tm_a,
                                         int q, int part, int kParts) {
    // Unconditional loads: padding rows read harmless staged data (their D
    // rows are never stored) and the staging tail past the tensor end is zero.
    const uint32_t pxb = (uint32_t)P.CBI * 32u;
    const int nk = P.KP / 4;
    int wo[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int w0 = v0 + L.minsh[k];
        wo[k] = (P.batch_mode || P.I_contig) ? 0 : w0 - floor_div(w0, P.Wg) * P.Wg;
    }
    const uint32_t lane_q = (uint32_t)(q * 32) << 16;
#pragma unroll
    for (int tt = 0; tt < kWMaxTG; ++tt) {
        if (tt >= L.ntl) break;
        if (!((L.live >> tt) & 1u)) continue;   // rows of this lane quarter are all padding: never stored
        const int k = L.kpl[tt] < 0 ? 0 : L.kpl[tt];
        int wok = wo[0];
#pragma unroll
        for (int kx = 1; kx < 4; ++kx)
            if (k == kx) wok = wo[kx];
        const uint32_t src = stg + L.base[tt] + (uint32_t)wok * pxb;
        const uint32_t dcol = tm_a + lane_q + (uint32_t)(tt * nk * 8);
        // two k-steps per batch: 8 independent loads in flight before the TMEM stores
        for (int kk = part; kk < nk; kk += 2 * kParts) {
            const bool two = kk + kParts < nk;
            uint32_t r[8], r2[8];
            const uint32_t a = src + (uint32_t)(kk * 4) * pxb;
            const uint32_t a2 = two ? a + (uint32_t)(kParts * 4) * pxb : a;
#pragma unroll
            for (int px = 0; px < 4; ++px)
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];\n"
                             : "=r"(r[2 * px]), "=r"(r[2 * px + 1])
                             : "r"(a + (uint32_t)px * pxb));
#pragma unroll
            for (int px = 0; px < 4; ++px)
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];\n"
                             : "=r"(r2[2 * px]), "=r"(r2[2 * px + 1])
                             : "r"(a2 + (uint32_t)px * pxb));
            tmem_st8(dcol + (uint32_t)(kk * 8), r);
            if (two) tmem_st8(dcol + (uint32_t)((kk + kParts) * 8), r2);
        }
    }
}

__global__ void __launch_bounds__(kWThreads, 1) wgrad_kernel(const __grid_constant__ WgradMma P) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *stg_full = bars, *stg_empty = bars + 4;
    uint64_t *op_full = bars + 8, *op_empty = op_full + kWMaxStages;
    uint64_t *acc_full = op_empty + kWMaxStages, *acc_empty = acc_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem_raw + 512);
    const uint32_t stg0 = smem_u32(smem_raw) + 1024;
    const uint32_t op0 = stg0 + P.nstg * P.stg_bytes;
    // warp index broadcast from lane 0: the compiler then knows the role
    // branches are warp-uniform and keeps the MMA operands in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
    constexpr int kEpi0 = kWLoad / 32, kMma = kEpi0 + kWEpi / 32, kTma = kMma + 1;

    const uint32_t zero8 = smem_u32(smem_raw) + 768;   // 16 zero bytes (padding pixels)
    if (threadIdx.x < 4) reinterpret_cast<uint32_t *>(smem_raw + 768)[threadIdx.x] = 0u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(stg_full + i, 1);
            mbar_init(stg_empty + i, 32 * (w_group_w0(i % P.lgroups + 1, P.lgroups) - w_group_w0(i % P.lgroups, P.lgroups)));
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(acc_full + i, 1);
            mbar_init(acc_empty + i, kWLoad / 32);
        }
        for (int s = 0; s < P.nstages; ++s) {
            mbar_init(op_full + s, 32 * (w_group_w0(s % P.lgroups + 1, P.lgroups) - w_group_w0(s % P.lgroups, P.lgroups)));
            mbar_init(op_empty + s, 1);
        }
        mbar_fence_init();
    }
    if (warp == kMma) tmem_alloc_dyn(tmem_slot, 512);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    // all 512 columns belong to this CTA, so the allocation starts at lane 0,
    // column 0.  Using the constant (not the value read back from shared
    // memory) keeps every MMA operand in uniform registers -- no R2UR per MMA.
    if (*tmem_slot != 0u) __trap();
    constexpr uint32_t tmem = 0u;
    const int nk = P.KP / 4;

    if (warp == kTma) {
        if (lane == 0) {
            tma::prefetch_desc(&P.tm_I);
            tma::prefetch_desc(&P.tm_O);
        }
        int sb = 0;
        uint32_t sph = 0;
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            int g, ks, p0, p1;
            wdecode(P, item, g, ks, p0, p1);
            WGroup G;
            w_group_setup(P, g, G);
            for (int v0 = p0; v0 < p1; v0 += P.KP) {
                const int si = (v0 - p0) / P.KP;
                if (lane == 0) WTRACE(0, si, 0);
                mbar_wait(stg_empty + sb, sph ^ 1);
                if (lane == 0) WTRACE(0, si, 1);
                const uint32_t stg = stg0 + sb * P.stg_bytes;
                if (P.I_contig) {
                    const int lo = v0 + G.minsh[0];
                    const int valid = max(0, min(P.vtotal, lo + P.KP + G.span[0]) - lo);
                    const uint32_t zb = (uint32_t)valid * P.C * 32u, ze = (uint32_t)P.capI * P.C * 32u;
                    for (uint32_t z = zb + (uint32_t)lane * 16u; z < ze; z += 512u) st_shared_v4z(stg + z);
                    __syncwarp();
                }
                if (P.I_contig || P.I_rows) {
                    // at most two bulk copies: computed once, issued by lane 0
                    if (lane == 0) {
                        const uint32_t mb = smem_u32(stg_full + sb);
                        const uint8_t *srcI = nullptr;
                        uint32_t nbI = 0;
                        if (P.I_rows) {
                            int wlo = 1 << 30, whi = -1;
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                if (k < G.np) {
                                    wlo = min(wlo, v0 + G.minsh[k]);
                                    whi = max(whi, v0 + G.minsh[k] + P.KP + G.span[k] - 1);
                                }
                            int rA, rB;
                            w_in_rows(P, wlo, min(whi, P.vtotal - 1), rA, rB);
                            if (rB >= rA) {
                                nbI = (uint32_t)(rB - rA + 1) * P.Win * P.C * 32u;
                                srcI = P.I_ptr + (size_t)rA * P.Win * P.C * 32;
                            }
                        } else {
                            const int lo = v0 + G.minsh[0];
                            const int hi = min(v0 + P.KP + G.span[0] + G.minsh[0], P.vtotal);
                            if (hi > lo) {
                                nbI = (uint32_t)(hi - lo) * P.C * 32u;
                                srcI = P.I_ptr + (size_t)lo * P.C * 32;
                            }
                        }
                        int ra, rb;
                        w_dO_rows(P, v0, ra, rb);
                        const uint32_t nbO = rb > ra ? (uint32_t)(rb - ra) * P.Wo * P.Cout * 32u : 0u;
                        mbar_arrive_expect_tx(stg_full + sb, nbI + nbO);
                        if (nbI) bulk_g2s_u32(stg, srcI, nbI, nullptr, mb);
                        if (nbO)
                            bulk_g2s_u32(stg + P.stgI_bytes, P.O_ptr + (size_t)ra * P.Wo * P.Cout * 32, nbO, nullptr, mb);
                    }
                    __syncwarp();
                } else {
                    if (lane == 0) mbar_arrive_expect_tx(stg_full + sb, w_issue(P, G, v0, stg, 0, false, 0));
                    __syncwarp();
                    w_issue(P, G, v0, stg, smem_u32(stg_full + sb), true, lane);
                }
                if (lane == 0) WTRACE(0, si, 2);
                if (++sb == P.nstg) { sb = 0; sph ^= 1; }
            }
        }
    } else if (warp < kEpi0) {
        // ---------------------------------------------------------- loaders
        const int tid = threadIdx.x;
        // group lg = tid / gsize owns the stages s with s % lgroups == lg; the
        // warps of a group cover all four TMEM lane quarters (quarter = warp % 4)
        const int NG = P.lgroups;
        int lg = 0;
        while (lg + 1 < NG && warp >= w_group_w0(lg + 1, NG)) ++lg;
        const int gw0 = w_group_w0(lg, NG), gw1 = w_group_w0(lg + 1, NG);
        const int gsize = 32 * (gw1 - gw0), gtid = tid - 32 * gw0;
        const int bpstep = gsize / (2 * P.Cout);
        const int q = warp & 3;
        int part = 0, nparts = 0;
        for (int w = gw0; w < gw1; ++w)
            if ((w & 3) == q) { if (w < warp) ++part; ++nparts; }
        int s_glob = 0;
        uint32_t e_aph = 0;   // accumulator phase (one accumulator set)
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            int g, ks, p0, p1;
            wdecode(P, item, g, ks, p0, p1);
            WLane L;
            w_lane_setup(P, g, q, lane, L);
            WGroup G;
            w_group_setup(P, g, G);
            for (int v0 = p0; v0 < p1; v0 += P.KP, ++s_glob) {
                if (s_glob % NG != lg) continue;
                const int sb = s_glob % P.nstg, st = s_glob % P.nstages;
                const uint32_t sph = (uint32_t)(s_glob / P.nstg) & 1u, ph = (uint32_t)(s_glob / P.nstages) & 1u;
                // tables per staging buffer: a buffer is refilled (and its
                // tables rewritten) only after every loader thread released it
                const uint32_t tab = smem_u32(smem_raw) + P.tab_off + (uint32_t)sb * P.tab_stride;
                const uint32_t btab = tab + P.btab_off;
                const int si = (v0 - p0) / P.KP;
                if (tid == 0) WTRACE(1, si, 0);
                mbar_wait(stg_full + sb, sph);
                if (tid == 0) WTRACE(1, si, 1);
                if (P.I_rows) w_build_table(P, G, v0, tab, gtid, gsize);
                w_build_btab(P, v0, btab, gtid, gsize);
                if (!(kProbes && (P.dbg & 1))) w_transpose_stage(stg0 + sb * P.stg_bytes, P.stgI_bytes, gtid, gsize);
                named_bar_sync(1 + lg, gsize);
                mbar_wait(op_empty + st, ph ^ 1);
                fence_after_sync();
                if (tid == 0) WTRACE(1, si, 2);
                const uint32_t stg = stg0 + sb * P.stg_bytes;
                if (!(kProbes && (P.dbg & 4))) w_load_B(P, stg, btab, op0 + st * P.b_bytes, gtid, bpstep);
                if (kProbes && (P.dbg & 16)) {
                } else if (P.I_rows)
                    w_load_A_rows(P, L, stg, tab, zero8, tmem + P.acc_cols + (uint32_t)st * P.abuf_cols, q, part,
                                  nparts);
                else
                    w_load_A(P, L, v0, stg, tmem + P.acc_cols + (uint32_t)st * P.abuf_cols, q, part, nparts);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                fence_proxy_async_smem();
                fence_before_sync();
                if (tid == 0) WTRACE(1, si, 3);
                mbar_arrive(op_full + st);
                mbar_arrive(stg_empty + sb);
            }
            // ------------------------------------------------ epilogue of the item
            // units (tile, 16 columns) are spread over the four warps of this
            // warp's lane quarter
            {
                const int wq = q, wi = warp >> 2;
                const int row = wq * 32 + lane;
                const size_t nkel = (size_t)P.ntaps * P.C * P.Cout * 16;
                const int ntl = min(P.TG, P.n_mtiles - g * P.TG);
                const int nch = P.N_tile / 16;
                mbar_wait(acc_full + 0, e_aph);
                fence_after_sync();
                int cur_tt = -1, tap = -1, c = 0, q0 = 0;
                float *dst = nullptr;
                const int d2 = row & 3;
                for (int unit = wi; unit < ntl * nch; unit += 4) {
                    const int tt = unit / nch, n0 = (unit - tt * nch) * 16;
                    if (tt != cur_tt) {
                        cur_tt = tt;
                        const WTile &T = P.tile[P.tiles_uniform ? 0 : g * P.TG + tt];
                        const int cshift = P.tiles_uniform ? (g * P.TG + tt) * 32 : 0;
                        tap = -1; c = 0;
                        for (int j = 0; j < T.nslots; ++j) {
                            const WSlot &S = T.slot[j];
                            if (row >= S.row0 && row < S.row0 + 4 * S.cn) {
                                tap = S.tap;
                                c = S.c0 + cshift + ((row - S.row0) >> 2);
                            }
                        }
                        // column n = (block, c', d3); block bi is shift j of the slot's tap (p, q)
                        q0 = tap < 0 ? 0 : tap % P.KWv;
                        dst = P.part + (size_t)ks * nkel + (((size_t)(tap < 0 ? 0 : tap) * P.C + c) * P.Cout) * 16 + d2 * 4;
                    }
                    const uint32_t tcol = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(tt * P.N_tile);
                    float v[16];
                    tmem_ld16(tcol + n0, v);
                    tmem_wait_ld();
                    if (tap >= 0 && c < P.C) {
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int cn = n0 / 4 + jj;           // capsule column bi*Cout + c'
                            const int bi = cn / P.Cout, co = cn - bi * P.Cout;
                            const int j = P.bdesc ? P.nq - 1 - bi : bi;   // shift of this block
                            if (bi < P.nq && q0 + P.s * j < P.KWv)
                                *reinterpret_cast<float4 *>(dst + ((size_t)P.s * j * P.C * P.Cout + co) * 16) =
                                    make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
                        }
                    }
                }
                fence_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive(acc_empty + 0);
                e_aph ^= 1;
            }
        }
    } else if (warp == kMma) {
        const uint32_t idesc = idesc_bf16(128, P.N_tile, 0, 1);
        const uint32_t idesc_sub = idesc_bf16(128, P.Cout * 4, 0, 1);
        // 8 k-steps per elected region when possible (measured: L1 dK 130 -> 126 us)
        const bool unr8 = true;
        const uint32_t idesc_sub2 = idesc_bf16(128, (P.bmat > 1 ? 2 : 1) * P.Cout * 4, 0, 1);
        int st = 0, abuf = 0;
        uint32_t ph = 0, aph = 0;
        for (int item = blockIdx.x; item < P.n_items; item += gridDim.x) {
            int g, ks, p0, p1;
            wdecode(P, item, g, ks, p0, p1);
            const int ntl = min(P.TG, P.n_mtiles - g * P.TG);
            mbar_wait(acc_empty + abuf, aph ^ 1);
            fence_after_sync();
            bool first = true;
            for (int v0 = p0; v0 < p1; v0 += P.KP) {
                const int si = (v0 - p0) / P.KP;
                if (lane == 0) WTRACE(2, si, 0);
                mbar_wait(op_full + st, ph);
                if (lane == 0) WTRACE(2, si, 1);
                fence_after_sync();
                const uint64_t bd0 = smem_desc(op0 + st * P.b_bytes, 128, P.b_sbo);
                const uint32_t a0 = tmem + P.acc_cols + (uint32_t)st * P.abuf_cols;
                // the warp stays converged; one elected lane issues 4 k-steps at
                // a time (a long divergent single-lane loop issues far slower)
                if (kProbes && (P.dbg & 2)) {
                } else if (P.bdesc) {
                    // accumulator block bi = shift j = nq-1-bi reads F_0 from
                    // pixel bi (descriptor offset); one MMA covers bmat adjacent
                    // blocks through the materialised copies.  Block-major order:
                    // each accumulator takes its k-steps back to back.
                    const int nsub = P.Cout * 4;
                    for (int tt = 0; tt < ntl; ++tt) {
                        for (int b0 = 0; b0 < P.nq; b0 += P.bmat) {
                            const bool two = P.bmat > 1 && b0 + 1 < P.nq;
                            const uint32_t d = tmem + (uint32_t)(tt * P.N_tile + b0 * nsub);
                            const uint64_t bj = bd0 + (uint64_t)(b0 * 4);
                            const uint32_t idx = two ? idesc_sub2 : idesc_sub;
                            if (unr8 && (nk & 7) == 0) {
                                for (int k8 = 0; k8 < nk; k8 += 8) {
                                    if (elect_one()) {
#pragma unroll
                                        for (int u = 0; u < 8; ++u) {
                                            const int kk = k8 + u;
                                            asm volatile(
                                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                                                "r"(a0 + (uint32_t)((tt * nk + kk) * 8)), "l"(bj + (uint64_t)(kk * 16)),
                                                "r"(idx), "r"((first && kk == 0) ? 0u : 1u));
                                        }
                                    }
                                    __syncwarp();
                                }
                            } else
                            for (int k4 = 0; k4 < nk; k4 += 4) {
                                if (elect_one()) {
#pragma unroll
                                    for (int u = 0; u < 4; ++u) {
                                        const int kk = k4 + u;
                                        asm volatile(
                                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                                            "r"(a0 + (uint32_t)((tt * nk + kk) * 8)), "l"(bj + (uint64_t)(kk * 16)),
                                            "r"(idx), "r"((first && kk == 0) ? 0u : 1u));
                                    }
                                }
                                __syncwarp();
                            }
                        }
                    }
                } else
                for (int tt = 0; tt < ntl; ++tt) {
                    const uint32_t d = tmem + (uint32_t)(tt * P.N_tile);
                    for (int k4 = 0; k4 < nk; k4 += 4) {
                        if (elect_one()) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int kk = k4 + u;
                                asm volatile(
                                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                    "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                                    "r"(a0 + (uint32_t)((tt * nk + kk) * 8)), "l"(bd0 + (uint64_t)(kk * 16)),
                                    "r"(idesc), "r"((first && kk == 0) ? 0u : 1u));
                            }
                        }
                        __syncwarp();
                    }
                }
                if (elect_one()) mma_commit(op_empty + st);
                __syncwarp();
                first = false;
                if (++st == P.nstages) { st = 0; ph ^= 1; }
            }
            if (elect_one()) mma_commit(acc_full + abuf);
            __syncwarp();
            aph ^= 1;   // one accumulator set (abuf stays 0)
        }
    }

    fence_before_sync();
    __syncthreads();
    if (warp == kMma) {
        fence_after_sync();
        tmem_dealloc_dyn(tmem, 512);
    }
}

// Split-K partials -> dK, deterministic: a block of 256 threads is E = 256/nsl
// elements x nsl slices of the split range (nsl in {1, 2, 4, 8}, more slices
// for longer splits); each thread sums its slice in order, the slice sums are
// then added in slice order (a fixed summation tree for every launch).
__global__ void __launch_bounds__(256) w_finalize(const float *__restrict__ part, float *__restrict__ dK, int64_t n,
                                                  int ksplit, int nsl) {
    // (no early PDL trigger: the workspace may be read until the end, and the
    // rows-layout weight packs that may follow do not wait before writing it)
    pdl_wait();                // the previous grid has completed and its writes are visible
    __shared__ float red[256];
    const int E = 256 / nsl;
    const int el = threadIdx.x % E, sl = threadIdx.x / E;
    const int64_t i = (int64_t)blockIdx.x * E + el;
    const int k0 = sl * ksplit / nsl, k1 = (sl + 1) * ksplit / nsl;
    float acc = 0.f;
    if (i < n)
        for (int k = k0; k < k1; ++k) acc += part[(int64_t)k * n + i];
    red[threadIdx.x] = acc;
    __syncthreads();
    if (sl == 0 && i < n) {
        float t = red[el];
        for (int j = 1; j < nsl; ++j) t += red[j * E + el];
        dK[i] = t;
    }
}

// ------------------------------------------------------------------ planning
struct WPlan {
    bool ok = false;
    WgradMma P{};
    size_t part_bytes = 0;
    // tensor-map geometry
    int64_t I_B, I_H, I_W, I_C, O_B, O_H, O_W, O_C;
};

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
constexpr uint32_t kWSmemLimit = 227 * 1024;

WPlan make_wplan(const Problem &p, bool allow_nq) {
    WPlan pl;
    WgradMma &P = pl.P;
    if (p.dt != CAPSCONV_BF16 || p.D1 != 4 || p.D2 != 4 || p.D3 != 4) return pl;
    const bool fc = (p.KH == p.H && p.KW == p.W && p.pad == 0);
    P.pad = (int)p.pad;
    const int s = fc ? 1 : (int)p.s;
    if (s > 2) return pl;
    P.s = s;
    std::vector<int> tplane, tshift;
    if (fc) {
        // fully-connected view: one pixel per image, C_eff = KH*KW*C channels, one tap
        P.C = (int)(p.KH * p.KW * p.C);
        P.Cout = (int)p.Cout;
        P.Bn = (int)p.B; P.Hg = 1; P.Wg = 1; P.batch_mode = 1;
        P.ntaps = 1;
        P.pl_oy[0] = P.pl_ox[0] = 0;
        tplane.push_back(0); tshift.push_back(0);
        pl.I_B = p.B; pl.I_H = 1; pl.I_W = 1; pl.I_C = P.C;
        pl.O_B = p.B; pl.O_H = 1; pl.O_W = 1; pl.O_C = p.Cout;
    } else {
        if (p.KH * p.KW > kMaxTaps) return pl;
        P.C = (int)p.C; P.Cout = (int)p.Cout;
        P.Bn = (int)p.B;
        // the virtual grid covers the zero-padded input (pad = 0: the input)
        P.Hg = cdiv(p.H + 2 * p.pad, s); P.Wg = cdiv(p.W + 2 * p.pad, s); P.batch_mode = 0;
        if (P.Wg * s > 256) return pl;
        P.ntaps = (int)(p.KH * p.KW);
        int plane_of[2][2] = {{-1, -1}, {-1, -1}}, npl = 0;
        for (int pp = 0; pp < p.KH; ++pp)
            for (int qq = 0; qq < p.KW; ++qq) {
                const int a = pp % s, b = qq % s;
                if (plane_of[a][b] < 0) { plane_of[a][b] = npl; P.pl_oy[npl] = a; P.pl_ox[npl] = b; ++npl; }
                tplane.push_back(plane_of[a][b]);
                tshift.push_back((pp / s) * P.Wg + qq / s);
            }
        pl.I_B = p.B; pl.I_H = p.H; pl.I_W = p.W; pl.I_C = p.C;
        pl.O_B = p.B; pl.O_H = p.Ho; pl.O_W = p.Wo; pl.O_C = p.Cout;
    }
    // contiguous input staging needs the virtual grid to be the input itself
    P.I_contig = (!fc && s == 1 && P.C <= 16 && p.pad == 0) ? 1 : 0;
    // whole input rows + a plane table: stride 2, or any padded layer
    P.I_rows = (!fc && (s == 2 || p.pad > 0) && P.C <= 16) ? 1 : 0;
    P.Hin = (int)p.H; P.Win = (int)p.W; P.Bin = (int)p.B;
    P.Ho = (int)pl.O_H; P.Wo = (int)pl.O_W;
    const long long vt = (long long)P.Bn * P.Hg * P.Wg;
    if (vt * 4 >= (1ll << 31)) return pl;
    P.vtotal = (int)vt;
    // ---- column shifts: taps (p, q) with q >= s are served by B copy j = q / s
    // of the slot for tap (p, q mod s) -- fewer, wider MMAs and 1/nq of the A
    // operand to build.  bdesc: one B copy, the shifts are
    // descriptor offsets and each copy is its own N = 4*Cout MMA (the
    // accumulators, nq*4*Cout columns per tile, only have to fit TMEM);
    // otherwise the copies are materialised side by side in one N <= 256 MMA.
    static const int force_nq1 = probe_env("CAPSCONV_WG_NQ1") ? 1 : 0;
    static const int bdesc_env = probe_env("CAPSCONV_WG_BDESC") ? atoi(probe_env("CAPSCONV_WG_BDESC")) : -1;
    P.KWv = fc ? 1 : (int)p.KW;
    P.nq = 1;
    P.bdesc = 0;
    if (!fc && !force_nq1 && allow_nq) {
        const int nq = cdiv(p.KW, s);
        const bool bd = (P.Cout * 4) % 16 == 0 && P.Cout * 4 <= 256 && bdesc_env != 0;
        if (nq > 1 && nq <= kWMaxNq && (bd ? nq * P.Cout * 4 <= 384 : cdiv(nq * P.Cout * 4, 16) * 16 <= 256)) {
            P.nq = nq;
            P.bdesc = bd ? 1 : 0;
        }
    }
    {
        static const int bmat_env = probe_env("CAPSCONV_WG_BMAT") ? atoi(probe_env("CAPSCONV_WG_BMAT")) : 0;
        P.bmat = 1;
        // measured (tests/probe/ab.sh CAPSCONV_WG_BMAT 2 1): two copies are
        // slower on every stack layer (the bigger B costs pipeline depth), so
        // one copy is the default; 2 stays selectable
        if (P.bdesc && 2 * P.Cout * 4 <= 256 && bmat_env == 2) P.bmat = 2;
    }
    std::vector<int> stap;   // taps that own A slots
    for (int t = 0; t < P.ntaps; ++t)
        if (P.nq == 1 || t % P.KWv < s) stap.push_back(t);
    const int nst = (int)stap.size();
    P.N_tile = cdiv(P.nq * P.Cout * 4, 16) * 16;
    if (P.N_tile > (P.bdesc ? 384 : 256)) return pl;
    // ---- M tiles: slots (tap, channel range); channels in pairs (C odd -> padded slot rows)
    const int cpad = (P.C + 1) & ~1;
    std::vector<WTile> tiles;
    if (4 * cpad <= 128) {
        const int per = 128 / (4 * cpad);
        for (int t0 = 0; t0 < nst; t0 += per) {
            WTile T{};
            T.nslots = std::min(per, nst - t0);
            if (T.nslots > kWMaxSlots) return pl;
            T.c_lo = 0; T.c_hi = P.C;
            for (int j = 0; j < T.nslots; ++j) {
                const int t = stap[t0 + j];
                T.slot[j] = WSlot{t, tplane[t], tshift[t], 0, cpad, j * 4 * cpad, {}};
                T.slot[j].fd_upp.init((uint32_t)(2 * cpad));
            }
            tiles.push_back(T);
        }
    } else {
        for (int t : stap)
            for (int c0 = 0; c0 < P.C; c0 += 32) {
                WTile T{};
                T.nslots = 1;
                const int cn = std::min(32, P.C - c0);
                T.slot[0] = WSlot{t, tplane[t], tshift[t], c0, (cn + 1) & ~1, 0, {}};
                T.slot[0].fd_upp.init((uint32_t)(2 * ((cn + 1) & ~1)));
                T.c_lo = c0; T.c_hi = std::min(P.C, c0 + ((cn + 1) & ~1));
                tiles.push_back(T);
            }
    }
    // FC view (one tap, 32-channel tiles): beyond the table's capacity the
    // tiles are uniform and computed from tile 0 in the kernel
    P.tiles_uniform = 0;
    if ((int)tiles.size() > kWMaxTiles) {
        if (!fc || tiles[0].nslots != 1 || tiles[0].slot[0].cn != 32) return pl;
        P.tiles_uniform = 1;
    }
    P.n_mtiles = (int)tiles.size();
    for (int i = 0; i < P.n_mtiles; ++i) {
        WTile &T = tiles[i];
        T.np = 0;
        for (int j = 0; j < T.nslots; ++j) {
            int k = 0;
            while (k < T.np && T.plane[k] != T.slot[j].plane) ++k;
            if (k == T.np) { T.plane[k] = T.slot[j].plane; T.minsh[k] = 1 << 30; T.span[k] = -(1 << 30); ++T.np; }
            T.minsh[k] = std::min(T.minsh[k], T.slot[j].shift);
            T.span[k] = std::max(T.span[k], T.slot[j].shift);
        }
        for (int k = 0; k < T.np; ++k) T.span[k] -= T.minsh[k];
        if (i < kWMaxTiles) P.tile[i] = T;
    }
    const int nsm = device_info().num_sms;
    P.CBO = std::min(16, P.Cout);
    const int nbO = cdiv(P.Cout, P.CBO);
    static const int force_tg = probe_env("CAPSCONV_WG_TG") ? atoi(probe_env("CAPSCONV_WG_TG")) : 0;
    bool found = false;
    // tiles per CTA group: as many as TMEM holds (shared staged window), then
    // pixels per stage and pipeline depths that fit shared memory
    for (int TG = std::min(P.n_mtiles, kWMaxTG); TG >= 1 && !found; --TG) {
        if (force_tg && TG != force_tg) continue;
        const int ngroups = cdiv(P.n_mtiles, TG);
        if (ngroups > kWMaxTiles) continue;   // per-group tables hold kWMaxTiles entries
        // group unions
        int gmax_np = 1, gmax_span = 0, gmax_ci = 0, gmax_msh = 0;
        for (int g = 0; g < ngroups; ++g) {
            int np = 0, plane[4], mn[4], mx[4], clo = 1 << 30, chi = 0;
            for (int mt = g * TG; mt < std::min(P.n_mtiles, (g + 1) * TG); ++mt) {
                const WTile &T = tiles[mt];
                clo = std::min(clo, T.c_lo); chi = std::max(chi, T.c_hi);
                for (int j = 0; j < T.nslots; ++j) {
                    int k = 0;
                    while (k < np && plane[k] != T.slot[j].plane) ++k;
                    if (k == np) { if (np == 4) return pl; plane[k] = T.slot[j].plane; mn[k] = 1 << 30; mx[k] = -(1 << 30); ++np; }
                    mn[k] = std::min(mn[k], T.slot[j].shift);
                    mx[k] = std::max(mx[k], T.slot[j].shift);
                }
            }
            P.g_np[g] = np;
            for (int k = 0; k < np; ++k) {
                P.g_plane[g][k] = plane[k]; P.g_minsh[g][k] = mn[k]; P.g_span[g][k] = mx[k] - mn[k];
                gmax_span = std::max(gmax_span, mx[k] - mn[k]);
            }
            P.g_clo[g] = clo; P.g_chi[g] = chi;
            {
                int lo = 1 << 30, hi = -(1 << 30);
                for (int k = 0; k < np; ++k) { lo = std::min(lo, mn[k]); hi = std::max(hi, mx[k]); }
                gmax_msh = std::max(gmax_msh, hi - lo - 0);
            }
            gmax_np = std::max(gmax_np, np);
            gmax_ci = std::max(gmax_ci, chi - clo);
        }
        P.CBI = std::min(16, gmax_ci);
        const int nbI = cdiv(gmax_ci, P.CBI);
        static const int force_kp = probe_env("CAPSCONV_WG_KP") ? atoi(probe_env("CAPSCONV_WG_KP")) : 0;
        for (int KP : {128, 96, 64, 32, 16}) {
            if (force_kp ? KP != force_kp : KP > 64) continue;
            const uint32_t acc = (uint32_t)(TG * P.N_tile);
            const uint32_t abuf = (uint32_t)(2 * TG * KP);      // TG tiles x KP/4 k-steps x 8 columns
            // rows mode: both parities of every virtual row the union window touches
            const int rows_mode_cap = s * ((KP + gmax_span + gmax_msh - 1) / P.Wg + 2) * P.Win;
            const int capI = P.batch_mode ? KP
                             : P.I_contig ? KP + gmax_span
                             : P.I_rows   ? rows_mode_cap
                                          : ((KP + gmax_span - 1) / P.Wg + 2) * P.Wg;
            // dO: whole dO rows touched by the window
            const int capO = P.batch_mode ? KP : ((KP + P.nq - 2) / P.Wg + 2) * P.Wo;
            const uint32_t stgI_plane = (uint32_t)nbI * capI * P.CBI * 32;
            const uint32_t stgI = P.I_rows ? stgI_plane : (uint32_t)gmax_np * stgI_plane;
            const int TABW = KP + gmax_span;
            const uint32_t stgO = (uint32_t)capO * P.Cout * 32;
            const uint32_t stg = stgI + stgO;
            const uint32_t sbo = (uint32_t)(P.bdesc ? KP + P.nq - 1 : KP) * 64 + 16;
            const uint32_t bbytes = (uint32_t)((P.bdesc ? P.bmat * P.Cout * 4 : P.N_tile) / 8) * sbo;
            const uint32_t btab_off = P.I_rows ? 16u * TABW : 0u;
            const uint32_t tab_stride = btab_off + (((uint32_t)(KP + P.nq) * 4u + 15u) & ~15u);
            // (A buffers, staging buffers): equal counts first, so that the
            // loader can run that many stage groups concurrently
            static const int cmode = probe_env("CAPSCONV_WG_CMODE") ? atoi(probe_env("CAPSCONV_WG_CMODE")) : 0;
            // (A buffers, staging buffers): equal counts first, so that the
            // loader runs that many stage groups concurrently; 3/3 (three
            // groups of 5-6 warps) measured best where it fits (L1 dK 152 ->
            // 130 us vs 2/2)
            static const int combos_t[3][5][2] = {{{3, 3}, {2, 2}, {2, 3}, {3, 2}, {0, 0}},
                                                  {{2, 2}, {3, 3}, {2, 3}, {3, 2}, {0, 0}},
                                                  {{4, 4}, {2, 2}, {3, 3}, {2, 3}, {3, 2}}};
            const int (*combos)[2] = combos_t[cmode];
            for (int ci = 0; ci < 5 && combos[ci][0] && !found; ++ci) {
                const int ns = combos[ci][0], nstg = combos[ci][1];
                if (acc + ns * abuf > 512) continue;   // TMEM: accumulators + ns A buffers
                const uint64_t tot = 1024 + (uint64_t)nstg * stg + (uint64_t)ns * bbytes + (uint64_t)nstg * tab_stride;
                if (tot > kWSmemLimit) continue;
                P.TG = TG; P.n_groups = ngroups;
                P.KP = KP; P.capI = capI; P.capO = capO; P.stgI_plane = stgI_plane; P.stgI_bytes = stgI;
                P.stgO_bytes = stgO; P.stg_bytes = stg; P.b_sbo = sbo; P.b_bytes = bbytes;
                P.nstg = nstg; P.nstages = ns; P.smem_bytes = (uint32_t)tot;
                P.acc_cols = acc; P.abuf_cols = abuf;
                P.TABW = TABW;
                P.tab_off = 1024 + nstg * stg + ns * bbytes;
                P.tab_stride = tab_stride; P.btab_off = btab_off;
                if (P.I_rows) P.stgI_plane = 0;   // one staged region shared by all planes
                found = true;
            }
            if (found) break;
        }
    }
    if (!found) return pl;
    // ---- split of the pixel range so that items fill the machine
    const int nstage_total = cdiv(P.vtotal, P.KP);
    // one item per CTA: fewer fp32 partials for the finalize pass to read
    int ks = std::max(1, std::min(nstage_total, nsm / std::max(1, P.n_groups)));
    P.kpix = cdiv(nstage_total, ks) * P.KP;   // longest split (informational)
    P.ksplit = ks;
    P.n_items = P.n_groups * P.ksplit;
    P.tmem_cols = 512;
    P.fd_Wg.init((uint32_t)P.Wg);
    P.fd_HgWg.init((uint32_t)(P.Hg * P.Wg));
    P.fd_uppO.init((uint32_t)(2 * P.Cout));
    static const int lg_env = probe_env("CAPSCONV_WG_LG") ? atoi(probe_env("CAPSCONV_WG_LG")) : 0;
    P.lgroups = 1;
    // groups of 4 or 8 warps (every group covers the four lane quarters).
    // NG must divide both buffer counts: then a buffer is always used by the
    // same group, whose previous wait on it was the phase just before --
    // otherwise a group running ahead could wait two phases ahead and the
    // mbarrier parity test would pass falsely (observed: a hang).
    for (int ng : {4, 3, 2}) {
        if (lg_env && ng != lg_env) continue;
        const int min_threads = 32 * w_group_w0(1, ng);   // the smallest group is the first
        if (P.nstg % ng == 0 && P.nstages % ng == 0 && min_threads / (2 * P.Cout) >= 1) { P.lgroups = ng; break; }
    }
    P.b_pstep = 32 * w_group_w0(1, P.lgroups) / (2 * P.Cout);   // smallest group's (informational)
    if (P.b_pstep < 1) return WPlan{};
    const size_t nk = (size_t)P.ntaps * P.C * P.Cout * 16;
    pl.part_bytes = P.ksplit > 1 ? ((size_t)P.ksplit * nk * 4 + 255) & ~(size_t)255 : 0;
    pl.ok = true;
    return pl;
}

struct WKey {
    int dev, nsm;
    int64_t e[12];
    bool operator==(const WKey &o) const {
        if (dev != o.dev || nsm != o.nsm) return false;
        for (int i = 0; i < 12; ++i)
            if (e[i] != o.e[i]) return false;
        return true;
    }
};

// Entries are immutable and shared (see cached_plan in mma.cu).
std::shared_ptr<const WPlan> cached_wplan(const Problem &p) {
    static std::mutex mu;
    static std::vector<std::pair<WKey, std::shared_ptr<const WPlan>>> cache;
    const DeviceInfo &di = device_info();
    WKey k{di.device, di.num_sms, {p.B, p.H, p.W, p.C, p.Cout, p.KH, p.KW, p.D1, p.D2, p.D3, p.s, p.pad}};
    if (p.dt != CAPSCONV_BF16) k.e[7] = -1;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &kv : cache)
        if (kv.first == k) return kv.second;
    if (cache.size() > 256) cache.clear();
    WPlan w = make_wplan(p, true);
    if (!w.ok) w = make_wplan(p, false);   // column shifts do not fit TMEM/smem: one tap per slot
    cache.emplace_back(k, std::make_shared<const WPlan>(w));
    std::shared_ptr<const WPlan> sp = cache.back().second;
    const WPlan &pl = *sp;
    if (probe_env("CAPSCONV_DEBUG") && pl.ok) {
        const WgradMma &P = pl.P;
        fprintf(stderr,
                "[capsconv] wgrad plan: C=%d Cout=%d Hg=%d Wg=%d taps=%d mtiles=%d TG=%d groups=%d N_tile=%d KP=%d "
                "ksplit=%d items=%d capI=%d capO=%d nstg=%d stages=%d smem=%u acc=%u abuf=%u nq=%d bdesc=%d\n",
                P.C, P.Cout, P.Hg, P.Wg, P.ntaps, P.n_mtiles, P.TG, P.n_groups, P.N_tile, P.KP, P.ksplit, P.n_items,
                P.capI, P.capO, P.nstg, P.nstages, P.smem_bytes, P.acc_cols, P.abuf_cols, P.nq, P.bdesc);
    }
    return sp;
}

}  // namespace

bool wgrad_supported(const Problem &p) { return cached_wplan(p)->ok; }

size_t wgrad_workspace_bytes(const Problem &p) {
    std::shared_ptr<const WPlan> pl = cached_wplan(p);
    return pl->ok ? pl->part_bytes : 0;
}

cudaError_t wgrad_run(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                      cudaStream_t st) {
    WPlan pl = *cached_wplan(p);
    if (!pl.ok || ws_bytes < pl.part_bytes) return cudaErrorNotSupported;
    WgradMma &P = pl.P;
    const int boxw = P.batch_mode ? 1 : P.Wg;
    const int boxb = P.batch_mode ? P.KP : 1;
    if (!make_capsule_tmap(&P.tm_I, I, pl.I_B, pl.I_H, pl.I_W, pl.I_C, P.CBI, boxw, 1, boxb, P.batch_mode ? 1 : P.s))
        return cudaErrorInvalidValue;
    if (!make_capsule_tmap(&P.tm_O, dO, pl.O_B, pl.O_H, pl.O_W, pl.O_C, P.CBO, boxw, 1, boxb, 1))
        return cudaErrorInvalidValue;
    P.part = P.ksplit > 1 ? static_cast<float *>(ws) : dK;
    P.I_ptr = static_cast<const uint8_t *>(I);
    P.O_ptr = static_cast<const uint8_t *>(dO);
    P.dbg = probe_env("CAPSCONV_WG_DBG") ? atoi(probe_env("CAPSCONV_WG_DBG")) : 0;
    cudaError_t ea = smem_optin(reinterpret_cast<const void *>(wgrad_kernel), (int)kWSmemLimit);
    if (ea != cudaSuccess) return ea;
    const int grid = std::min(P.n_items, device_info().num_sms);
    static const bool tracing = probe_env("CAPSCONV_TRACE") != nullptr;
    P.trace = nullptr;
    if (tracing) {
        cudaMalloc(&P.trace, 3 * 64 * 4 * 8);
        cudaMemset(P.trace, 0, 3 * 64 * 4 * 8);
    }
    launch_k(wgrad_kernel, dim3(grid), dim3(kWThreads), P.smem_bytes, st, P);
    note_launches(1);
    if (tracing) {
        std::vector<unsigned long long> h(3 * 64 * 4);
        cudaStreamSynchronize(st);
        cudaMemcpy(h.data(), P.trace, h.size() * 8, cudaMemcpyDeviceToHost);
        cudaFree(P.trace);
        unsigned long long t0 = ~0ull;
        for (auto v : h) if (v && v < t0) t0 = v;
        const char *names[3] = {"tma ", "rpk ", "mma "};
        for (int i = 0; i < 12; ++i)
            for (int r = 0; r < 3; ++r) {
                fprintf(stderr, "[wtrace] stage %2d %s", i, names[r]);
                for (int e = 0; e < 4; ++e) {
                    unsigned long long v = h[(r * 64 + i) * 4 + e];
                    fprintf(stderr, " %8lld", v ? (long long)(v - t0) : -1ll);
                }
                fprintf(stderr, "\n");
            }
    }
    if (P.ksplit > 1) {
        const int64_t n = (int64_t)P.ntaps * P.C * P.Cout * 16;
        const int nsl = P.ksplit >= 64 ? 8 : P.ksplit >= 32 ? 4 : P.ksplit >= 16 ? 2 : 1;
        const int64_t E = 256 / nsl;
        launch_k(w_finalize, dim3((unsigned)((n + E - 1) / E)), dim3(256), 0, st, P.part, dK, n, P.ksplit, nsl);
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace capsconv
