// internal.h -- shared declarations of libcapsconv's CUDA path (product code;
// nothing here is shared with oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>

#include "capsconv.h"

namespace capsconv {

// One validated problem: the extents of capsconv.h plus the derived output size.
struct Problem {
    capsconv_dtype_t dt;
    int64_t B, H, W, C, Cout, KH, KW, D1, D2, D3, s;
    int64_t pad;   // symmetric zero padding of H and W (0: the paper's valid convolution)
    int64_t Ho, Wo;
    int layout = CAPSCONV_LAYOUT_NATURAL;   // capsconv_layout_t of I, dI, O, dO

    size_t elem() const { return dt == CAPSCONV_BF16 ? 2 : 4; }
    int64_t n_in() const { return B * H * W * C * D1 * D2; }
    int64_t n_out() const { return B * Ho * Wo * Cout * D1 * D3; }
    int64_t n_k() const { return KH * KW * C * Cout * D2 * D3; }
    int64_t n_pix_out() const { return B * Ho * Wo; }
    size_t kernel_bytes() const { return (size_t)n_k() * elem(); }
    // bytes a call writes: O (fwd), dI (bwd_data), fp32 dK (bwd_kernel)
    size_t out_bytes(capsconv_op_t op) const {
        return op == CAPSCONV_OP_FWD ? (size_t)n_out() * elem()
               : op == CAPSCONV_OP_BWD_DATA ? (size_t)n_in() * elem() : (size_t)n_k() * 4;
    }
};

// Device facts, cached once per device.
struct DeviceInfo {
    int device = -1;
    int num_sms = 148;
    int cc_major = 0, cc_minor = 0;
    size_t smem_optin = 0;
};
const DeviceInfo &device_info();

// Counts kernels enqueued by the library (capsconv_launch_count()).
void note_launches(int n);

// Diagnostic knobs (planner overrides, switches that skip loads / MMAs /
// stores, timing traces, the PDL A/B switch) exist only in probe builds
// (-DCAPSCONV_PROBES, tests/probe/); the product library never reads the
// environment, so no variable can change its results or make a call
// synchronise.
#ifdef CAPSCONV_PROBES
constexpr bool kProbes = true;
inline const char *probe_env(const char *name) { return getenv(name); }
#else
constexpr bool kProbes = false;
inline const char *probe_env(const char *) { return nullptr; }
#endif

// Opt `func` in to `bytes` of dynamic shared memory on the CURRENT device
// (the attribute is per function and per device).  Thread-safe; the driver
// call is made once per (function, device, larger size).
cudaError_t smem_optin(const void *func, int bytes);
// probe builds only: skip the weight-pack and split-K finalize launches (timing
// experiments; results are then wrong)
inline bool probe_skip_small() { return kProbes && probe_env("CAPSCONV_SKIP_SMALL") != nullptr; }
inline bool probe_skip_pack() { return probe_skip_small() || (kProbes && probe_env("CAPSCONV_SKIP_PACK") != nullptr); }
inline bool probe_skip_fin() { return probe_skip_small() || (kProbes && probe_env("CAPSCONV_SKIP_FIN") != nullptr); }

// Programmatic dependent launch (PDL) for the kernels of the hot path: the
// launch may begin while the previous kernel in the stream is still running;
// every kernel launched this way calls pdl_launch_dependents() on entry and
// pdl_wait() before its first global-memory access, which blocks until the
// previous grid has completed and its writes are visible -- stream order is
// unchanged, only launch latency and CTA placement overlap the predecessor's
// tail.  Disabled with CAPSCONV_NO_PDL (A/B measurements).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
// Weight packs (K -> workspace) read K while the previous kernel on the stream
// may still run (they trigger their dependents on entry and wait for the
// previous grid only before exiting).  The API entry clears this per call
// when K overlaps the output of the previous libcapsconv call on the same
// stream; the pack then launches fully ordered (see capsconv.h, "Streams").
bool pack_may_overlap();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pack(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() && pack_may_overlap() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
#endif

// ---------------------------------------------------------------- primary layer (primary.cu)
// The one-channel plain convolution of the training step's primary layer
// (C = D1 = D2 = 1, stride 1, no padding, N = Cout*D3 in {32, 64, 128, 256},
// 3x3 / 5x5 / 7x7): fwd and dK (dI has no consumer; the general path takes it).
bool primary_supported(const Problem &p);
bool primary_tc(capsconv_op_t op, const Problem &p);   // ... and runs on tcgen05 (bf16, 128 channels)
size_t primary_workspace_bytes(capsconv_op_t op, const Problem &p);
cudaError_t primary_fwd(const Problem &p, const void *img, const void *K, void *O, cudaStream_t st);
cudaError_t primary_bwd_kernel(const Problem &p, const void *img, const void *dO, float *dK, void *ws, cudaStream_t st);

// ---------------------------------------------------------------- optimizer step (optim.cu)
cudaError_t sgd_update(capsconv_dtype_t wdt, int64_t n, float lr, float *w, const float *g, void *out,
                       cudaStream_t st);

// ---------------------------------------------------------------- SIMT path
size_t simt_workspace_bytes(capsconv_op_t op, const Problem &p);
cudaError_t simt_fwd(const Problem &p, const void *I, const void *K, void *O, void *ws, size_t ws_bytes,
                     cudaStream_t st);
cudaError_t simt_bwd_data(const Problem &p, const void *dO, const void *K, void *dI, cudaStream_t st);
cudaError_t simt_bwd_kernel(const Problem &p, const void *I, const void *dO, float *dK,
                            void *ws, size_t ws_bytes, cudaStream_t st);

// ---------------------------------------------------------------- tcgen05 (MMA) path
// Returns true when the MMA path can take the problem (alignment excluded).
bool mma_supported(capsconv_op_t op, const Problem &p);
// fully-connected view (R18) forward on warp-level mma.sync (csrc/fc_hmma.cu)
bool fc_hmma_fwd_supported(const Problem &p);
size_t fc_hmma_fwd_workspace(const Problem &p);
cudaError_t fc_hmma_fwd(const Problem &p, const void *I, const void *K, void *O, void *ws, size_t ws_bytes,
                        cudaStream_t st);
// S-slice capsules as a channel-expanded convolution (csrc/slices.cu)
cudaError_t slices_expand_kernel(capsconv_dtype_t dt, const void *K, void *Kx, int64_t taps, int64_t C, int64_t Cout,
                                 int64_t S, int64_t D23, cudaStream_t st);
cudaError_t slices_extract_dk(const float *dKx, float *dK, int64_t taps, int64_t C, int64_t Cout, int64_t S,
                              int64_t D23, cudaStream_t st);
bool fc_hmma_dk_supported(const Problem &p);
size_t fc_hmma_dk_workspace(const Problem &p);
cudaError_t fc_hmma_dk(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                       cudaStream_t st);
bool fc_hmma_dgrad_supported(const Problem &p);
size_t fc_hmma_dgrad_workspace(const Problem &p);
cudaError_t fc_hmma_dgrad(const Problem &p, const void *dO, const void *K, void *dI, void *ws, size_t ws_bytes,
                          cudaStream_t st);
size_t mma_workspace_bytes(capsconv_op_t op, const Problem &p);
cudaError_t mma_fwd(const Problem &p, const void *I, const void *K, void *O,
                    void *ws, size_t ws_bytes, cudaStream_t st);
cudaError_t mma_bwd_data(const Problem &p, const void *dO, const void *K, void *dI,
                         void *ws, size_t ws_bytes, cudaStream_t st);
cudaError_t mma_bwd_kernel(const Problem &p, const void *I, const void *dO, float *dK,
                           void *ws, size_t ws_bytes, cudaStream_t st);

// D1-outer ("rows") layout: tcgen05 kernels fed by TMA only (rows_*.cu)
bool rows_wgrad_supported(const Problem &p);
size_t rows_wgrad_workspace_bytes(const Problem &p);
cudaError_t rows_wgrad_run(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                           cudaStream_t st);
bool rows_conv_supported(capsconv_op_t op, const Problem &p);
size_t rows_conv_workspace_bytes(capsconv_op_t op, const Problem &p);
cudaError_t rows_conv_run(capsconv_op_t op, const Problem &p, const void *src, const void *K, void *out, void *ws,
                          size_t ws_bytes, cudaStream_t st);
bool rows_walk_supported(capsconv_op_t op, const Problem &p);
size_t rows_walk_workspace_bytes(capsconv_op_t op, const Problem &p);
cudaError_t rows_walk_run(capsconv_op_t op, const Problem &p, const void *src, const void *K, void *out, void *ws,
                          size_t ws_bytes, cudaStream_t st);
bool rows_fc_supported(capsconv_op_t op, const Problem &p);
size_t rows_fc_workspace_bytes(capsconv_op_t op, const Problem &p);
cudaError_t rows_fc_run(capsconv_op_t op, const Problem &p, const void *a, const void *b, void *out, void *ws,
                        size_t ws_bytes, cudaStream_t st);
// capsule-row permutation between the layouts: [npix][C][D1][D2] <-> [npix][D1][C][D2]
// (to_rows = 1: natural -> rows).  Used by the rows-layout fallback path.
cudaError_t permute_layout(capsconv_dtype_t dt, const void *src, void *dst, int64_t npix, int64_t C, int64_t D1,
                           int64_t D2, int to_rows, cudaStream_t st);

// tcgen05 kernel gradient (wgrad.cu)
bool wgrad_supported(const Problem &p);
size_t wgrad_workspace_bytes(const Problem &p);
cudaError_t wgrad_run(const Problem &p, const void *I, const void *dO, float *dK, void *ws, size_t ws_bytes,
                      cudaStream_t st);

}  // namespace capsconv
