// conv_mma.cuh -- host/device description of one "shifted-window" implicit GEMM
// on tcgen05, shared by the forward pass and the data-gradient pass.
//
// The capsule convolution (Algorithm 2) is one dense
// contraction: rows M = (pixel, d1), columns N = (out channel, d),
// reduction K = (tap, source channel, d).  Instead of materialising the
// paper's capsule_im2col / input_extend / kernel_extend buffers (PAPER.md:
// 125-131), a CTA stages a *window* of source pixels once in shared memory in
// the UMMA K-major layout, and every kernel tap becomes the same window read
// at a different row offset (one descriptor start address per tap):
//
//   O[u] = sum_taps  A_plane(t)[u + shift(t)] . B_t           (rows u = virtual pixels)
//
// Virtual pixel grids: every source plane and every output group is an
// Hg x Wg grid per image; a virtual pixel (b, Y, X) maps to a source pixel
// (b, s*Y + oy, s*X + ox) or to an output pixel likewise, valid only inside
// the real tensor.  Forward with stride s uses s*s source planes (phase
// decomposition of the input) and one output group; the data gradient uses
// one source plane (dO placed in a zero-padded Hg x Wg grid) and s*s output
// groups (the phases of dI), each with its own taps.  Invalid source pixels
// are zero in shared memory; invalid output rows are computed and dropped.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace capsconv {

constexpr int kTilePix = 32;     // M = 128 rows = 32 pixels x D1 (=4)
constexpr int kMaxTaps = 64;
constexpr int kProducerThreads = 256;
constexpr int kEpilogueThreads = 256;   // two warps per TMEM lane quarter
constexpr int kConvThreads = kProducerThreads + kEpilogueThreads + 64;  // + MMA warp + TMA warp

// n / d for n < 2^31 by multiply-high (host-computed magic).
struct FastDiv {
    uint32_t d, mul, shr;
    void init(uint32_t dd) {
        d = dd;
        shr = 0;
        while ((1ull << shr) < dd) ++shr;
        mul = (uint32_t)((((1ull << 32) * ((1ull << shr) - dd)) / dd) + 1);
        if (dd == 1) mul = 0;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return (uint32_t)(((uint64_t)__umulhi(n, mul) + n) >> shr);
    }
};

struct ConvMma {
    // ---- TMA descriptor of the source (natural layout), see tma.h
    alignas(64) CUtensorMap tmap;
    int stg_batch_mode;        // 0: one copy per virtual row (box Wg px); 1: Hg*Wg == 1, box of BB images
    int BB;
    int stg_cap_px;            // staging capacity per plane, pixels
    uint32_t stg_plane_bytes;  // stg_cap_px * CC * 32
    uint32_t stg_bytes;        // npl * stg_plane_bytes
    int nstg;                  // staging buffers (1 or 2)
    // stride-2 forward: whole input rows (both parities) staged with one bulk
    // copy; a per-stage table maps each plane pixel of the window to them
    int I_rows, Hin, Win, Bin;
    // tall-box staging (unit-stride source planes, not batch mode): per image
    // segment of the window, boxes of h_box source rows x src_W pixels; a
    // per-item table maps window pixels to staged pixels (-1: zero)
    int stg_tall, h_box;
    // zero padding: source (staging) coordinates are virtual - src_pad, output
    // pixels are virtual - out_pad (fwd: src_pad = pad; dI: out_pad = pad)
    int src_pad, out_pad;
    uint32_t tab_off;          // table offset from the dynamic smem base (npl * win_px int32)
    // ---- tensors
    const __nv_bfloat16 *src;  // A source, natural capsule layout, pixel = CS*16 elements
    const uint8_t *wpack;      // prepacked B: [ntile][chunk][tap][kc][N_tile][16 B]
    __nv_bfloat16 *out;        // output, pixel = NCH*16 elements (used when ksplit == 1)
    float *part;               // fp32 partials [ksplit][Bn*Hg*Wg*4][N_total] (ksplit > 1)
    // ---- source
    int Bn, CS, CSpad;
    int src_H, src_W;          // source tensor spatial extents (pitch)
    int src_vH, src_vW;        // valid source region (mapped coordinates)
    int Hg, Wg;                // virtual grid per image
    FastDiv fd_Wg, fd_HgWg, fd_Hg, fd_hbox;
    int npl, pl_s;             // source planes and their stride
    int pl_oy[4], pl_ox[4];
    // ---- taps (sorted by output group)
    int ntaps;
    int tap_plane[kMaxTaps];
    int tap_shift[kMaxTaps];   // in virtual pixels (signed)
    int tap_p[kMaxTaps], tap_q[kMaxTaps];
    // ---- output groups
    int nog, og_s;
    int og_t0[4], og_t1[4];
    int og_oy[4], og_ox[4];
    int og_offmin[4];          // min tap shift of the group
    int gpi;                   // output groups per work item (1, or nog: one staged window for all phases)
    int ib_offmin[4];          // window offset of the item block starting at group g (min shift over its groups)
    int out_H, out_W, NCH;
    // ---- tiling
    int N_tile, n_ntiles;
    int CC, nchunks, ksplit;
    int G;                     // M tiles per work item
    int n_mtiles;              // ceil(Bn*Hg*Wg / kTilePix)
    int n_igroups;             // ceil(n_mtiles / G)
    int n_items;
    FastDiv fd_units;          // 8-byte pieces per pixel in a chunk = 4*CC
    FastDiv fd_ksplit, fd_nnt, fd_nig;   // item decode: ksplit, n_ntiles, n_igroups
    // ---- shared memory plan
    int win_px;                // window pixels (max over groups, even)
    uint32_t a_lbo;            // win_px*4*16 + 16 (bank stagger)
    uint32_t plane_bytes;      // (CC/2) * a_lbo
    uint32_t a_stage_bytes;    // npl * plane_bytes
    uint32_t b_stage_bytes;    // max taps-per-group * (CC/2) * N_tile * 16
    int nstages;
    int b_resident;            // one B stage for the whole kernel
    uint32_t smem_bytes;
    uint32_t tmem_cols;
    int dbg;                   // bench-only bits: 1 skip loads, 2 skip MMAs, 4 skip stores, 64 skip repack
    unsigned long long *trace; // debug: globaltimer stamps of CTA 0 [role][item][4]
};

}  // namespace capsconv
