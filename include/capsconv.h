/*
 * capsconv.h -- C ABI of libcapsconv, a B200 (sm_100a) implementation of the
 * capsule convolution of arXiv 2104.02621, "How to Accelerate Capsule
 * Convolutions in Capsule Networks", and of its two backward passes.
 *
 * The operation (§1.2; Algorithm 2):
 *   input  I(W, H, C, T1(D1, D2)), kernel K(w, h, c, T2(D2, D3)),
 *   output O(W', H', C', T3(D1, D3)); every output capsule is the sum over
 *   kernel taps and input channels of matrix_multiply(I_caps, K_caps), with
 *   row_offset = i*stride, col_offset = j*stride and no padding.
 *
 *   O[b,x',y',c',d1,d3] = sum_{p<KH, q<KW, c<C, d2<D2}
 *                           I[b, x'*s+p, y'*s+q, c, d1, d2] * K[p, q, c, c', d2, d3]
 *
 *   Ho = (H - KH) / s + 1, Wo = (W - KW) / s + 1   (integer division;
 *   PAPER.md:98-99 and the worked example PAPER.md:43-54, 5x5 * 4x4 -> 2x2).
 *
 * Backward (Algorithm 4, read as the analytic adjoints --
 * DESIGN.md readings R10/R11):
 *   dI[b,h,w,c,d1,d2] = sum_{p,q,c',d3 : h = x'*s+p, w = y'*s+q, x'<Ho, y'<Wo}
 *                          dO[b,x',y',c',d1,d3] * K[p,q,c,c',d2,d3]
 *   dK[p,q,c,c',d2,d3] = sum_{b,x',y',d1} I[b,x'*s+p,y'*s+q,c,d1,d2] * dO[b,x',y',c',d1,d3]
 *
 * ------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ------------------------------------------------------------------------
 * Extents      int64_t, all >= 1; KH <= H, KW <= W; stride >= 1.
 * Layouts      dense, row-major, element units, capsules contiguous:
 *                I, dI : [B][H][W][C][D1][D2]
 *                K     : [KH][KW][C][Cout][D2][D3]     dK: same, always fp32
 *                O, dO : [B][Ho][Wo][Cout][D1][D3]
 *              x' indexes H (rows, tap p over KH); y' indexes W (tap q over KW).
 * Dtypes       I, K, O, dO, dI share `dt` (fp32 or bf16).  Products are
 *              accumulated in fp32; bf16 results are rounded once (RNE) at the
 *              store.  dK is always fp32 (a long reduction that feeds an fp32
 *              all-reduce across GPUs).
 * Semantics    every call OVERWRITES its output (beta = 0).  Input positions
 *              covered by no window receive dI = 0.
 * Pointers     DEVICE pointers, caller-owned.  The library never allocates,
 *              frees or retains caller memory.  Input and output buffers must
 *              not alias (undefined behaviour).  The workspace is caller
 *              allocated device memory of at least capsconv_workspace_bytes();
 *              it may be NULL when that size is 0.  Its contents on entry are
 *              ignored and on return are unspecified.
 * Streams      calls enqueue on `stream` (NULL = legacy default stream) and
 *              return without synchronising.  Concurrent calls on different
 *              streams (with disjoint workspaces) are safe.  Calls on one
 *              stream run in order.  A call's weight packing (K into the
 *              workspace) may overlap the end of the previous libcapsconv
 *              call on that stream (programmatic dependent launch); the
 *              library remembers each stream's last output range and packs
 *              fully ordered when K overlaps it, so K may be any buffer,
 *              including the previous call's output.  Kernels of other
 *              libraries or of the caller are fully ordered as usual.
 * Errors       every call returns a status.  All validation happens before
 *              any launch, so a non-OK status other than CAPSCONV_ERR_CUDA
 *              guarantees nothing was written.  Asynchronous device faults
 *              surface at the caller's next synchronisation.  NaN/Inf inputs
 *              propagate per IEEE (no check).  capsconv_last_error() returns a
 *              thread-local detail string for the last failing call.
 * Dispatch     the library picks a kernel path per call (capsconv_select_path);
 *              every valid problem has a path (the SIMT path is total), so
 *              misalignment or unusual capsule sizes are never errors.
 */
#ifndef CAPSCONV_H_
#define CAPSCONV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CAPSCONV_API __attribute__((visibility("default")))
#else
#define CAPSCONV_API
#endif

/* ABI compatible with cudaStream_t / CUstream. */
typedef struct CUstream_st *capsconv_stream_t;

typedef enum {
    CAPSCONV_F32 = 0,
    CAPSCONV_BF16 = 1
} capsconv_dtype_t;

typedef enum {
    CAPSCONV_OK = 0,
    CAPSCONV_ERR_NULL = 1,       /* a required pointer is NULL */
    CAPSCONV_ERR_SHAPE = 2,      /* extent < 1, KH > H or KW > W */
    CAPSCONV_ERR_STRIDE = 3,     /* stride < 1 */
    CAPSCONV_ERR_DTYPE = 4,      /* unknown dtype / op / path */
    CAPSCONV_ERR_WORKSPACE = 5,  /* workspace smaller than capsconv_workspace_bytes() */
    CAPSCONV_ERR_OVERFLOW = 6,   /* an element count or index exceeds int64 / kernel limits */
    CAPSCONV_ERR_DEVICE = 7,     /* no CUDA device, or the current device is not sm_100 */
    CAPSCONV_ERR_CUDA = 8        /* a CUDA launch / runtime error; see capsconv_last_error() */
} capsconv_status_t;

typedef enum {
    CAPSCONV_OP_FWD = 0,
    CAPSCONV_OP_BWD_DATA = 1,
    CAPSCONV_OP_BWD_KERNEL = 2
} capsconv_op_t;

/* Memory layout of the capsule tensors I, dI, O, dO (K and dK always use
 * [KH][KW][C][Cout][D2][D3]).
 *   NATURAL  I [B][H][W][C][D1][D2],  O [B][Ho][Wo][Cout][D1][D3]  (the order
 *            of BASELINE.json's formula; every call without a layout argument)
 *   ROWS     I [B][H][W][D1][C][D2],  O [B][Ho][Wo][D1][Cout][D3]  ("D1-outer":
 *            row d1 of all C capsules of a pixel is contiguous).  Memory order
 *            is invisible to the mathematics (reading R3; the
 *            paper's Algorithm 2 is itself channel-major);
 *            this one lets TMA stage tensor-core operands with no repack
 *            (DESIGN.md §5.5), so chained layers should keep it. */
typedef enum {
    CAPSCONV_LAYOUT_NATURAL = 0,
    CAPSCONV_LAYOUT_ROWS = 1
} capsconv_layout_t;

typedef enum {
    CAPSCONV_PATH_AUTO = 0,   /* library's choice (only valid as an override) */
    CAPSCONV_PATH_SIMT = 1,   /* register-blocked small-matmul kernels (FFMA, fp32 accumulate) */
    CAPSCONV_PATH_MMA = 2     /* tcgen05 / TMEM implicit GEMM */
} capsconv_path_t;

/* Shape law.  Writes Ho, Wo.  Pure host function. */
CAPSCONV_API capsconv_status_t capsconv_output_dims(int64_t H, int64_t W, int64_t KH, int64_t KW,
                                       int64_t stride, int64_t *Ho, int64_t *Wo);

/* Bytes of device workspace the call `op` needs for these extents (0 if none).
 * Host only; no CUDA call except a one-time cached device-property query. */
CAPSCONV_API capsconv_status_t capsconv_workspace_bytes(capsconv_op_t op, capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        size_t *bytes);

/* The kernel path `op` would take for these extents (writes *path).  Pointer
 * alignment is not known here; a call whose pointers are not 16-byte aligned
 * takes the SIMT path even when this reports MMA. */
CAPSCONV_API capsconv_status_t capsconv_select_path(capsconv_op_t op, capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        capsconv_path_t *path);

/* Force a path for subsequent calls in this process (CAPSCONV_PATH_AUTO
 * restores the default).  Forcing MMA on a problem the MMA path cannot take
 * makes those calls fall back to SIMT. */
CAPSCONV_API capsconv_status_t capsconv_set_path_override(capsconv_path_t path);

/* Forward: O = I (*) K.  I [B][H][W][C][D1][D2], K [KH][KW][C][Cout][D2][D3]
 * (both dtype dt) -> O [B][Ho][Wo][Cout][D1][D3] (dtype dt). */
CAPSCONV_API capsconv_status_t capsconv_fwd(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        const void *I, const void *K, void *O,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

/* Backward data: dI = dO (*)^T K.  dO [B][Ho][Wo][Cout][D1][D3], K as above
 * (dtype dt) -> dI [B][H][W][C][D1][D2] (dtype dt). */
CAPSCONV_API capsconv_status_t capsconv_bwd_data(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        const void *dO, const void *K, void *dI,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

/* Backward kernel: dK = sum over (b, x', y', d1) of I^T dO.  I and dO of dtype
 * dt -> dK [KH][KW][C][Cout][D2][D3] in fp32.  The reduction is deterministic
 * (fixed order, no floating-point atomics). */
CAPSCONV_API capsconv_status_t capsconv_bwd_kernel(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        const void *I, const void *dO, float *dK,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

/* ---- Zero padding (SPEC.md:48-53 symmetric zero padding --
 * the paper's own convolution has none).  Each call below is
 * its unpadded namesake with one more extent, `pad` >= 0 (at most 2^20): the
 * input is read through a view padded with `pad` zero pixels on every side of
 * H and W, so Ho = (H + 2 pad - KH)/stride + 1, Wo likewise (KH <= H + 2 pad).
 * Layouts, ownership, stream semantics and error behaviour are those of the
 * unpadded calls; pad = 0 is exactly the unpadded call.  bwd_data returns dI
 * for the real H x W pixels only (the padding has no gradient). */
CAPSCONV_API capsconv_status_t capsconv_output_dims_pad(int64_t H, int64_t W, int64_t KH, int64_t KW,
                                       int64_t stride, int64_t pad, int64_t *Ho, int64_t *Wo);

CAPSCONV_API capsconv_status_t capsconv_workspace_bytes_pad(capsconv_op_t op, capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        size_t *bytes);

CAPSCONV_API capsconv_status_t capsconv_select_path_pad(capsconv_op_t op, capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        capsconv_path_t *path);

CAPSCONV_API capsconv_status_t capsconv_fwd_pad(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        const void *I, const void *K, void *O,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

CAPSCONV_API capsconv_status_t capsconv_bwd_data_pad(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        const void *dO, const void *K, void *dI,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

CAPSCONV_API capsconv_status_t capsconv_bwd_kernel_pad(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        const void *I, const void *dO, float *dK,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

/* ---- S-slice capsules (reading R22): a
 * capsule is S matrices multiplied slice-wise (PAPER.md:44-53's 3x3x3
 * capsules are S = 3 slices of 3x3).  Layouts, row-major, no padding:
 *   I, dI [B][H][W][C][S][D1][D2]; K [KH][KW][C][Cout][S][D2][D3];
 *   O, dO [B][Ho][Wo][Cout][S][D1][D3]; dK [KH][KW][C][Cout][S][D2][D3] (fp32)
 *   O[b,x',y',c',s,d1,d3] = sum_{p,q,c,d2} I[b,x's+p,y's+q,c,s,d1,d2] K[p,q,c,c',s,d2,d3].
 * Computed as the matrix-capsule convolution over C*S / Cout*S channels with a
 * block-diagonal kernel built in the workspace (S x the useful flops); the
 * workspace (query with capsconv_workspace_bytes_slices) is required, 1 <= S <= 64.
 * Errors, ownership and stream semantics are those of the matrix calls. */
CAPSCONV_API capsconv_status_t capsconv_workspace_bytes_slices(capsconv_op_t op, capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        size_t *bytes);

CAPSCONV_API capsconv_status_t capsconv_fwd_slices(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        const void *I, const void *K, void *O,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

CAPSCONV_API capsconv_status_t capsconv_bwd_data_slices(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        const void *dO, const void *K, void *dI,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

CAPSCONV_API capsconv_status_t capsconv_bwd_kernel_slices(capsconv_dtype_t dt,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
        const void *I, const void *dO, float *dK,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

/* ---- Layout-generic forms.  Each call below is its `_pad` namesake with a
 * capsconv_layout_t argument for I, dI, O and dO (see above); everything
 * else -- extents, padding, dtypes, ownership, stream semantics, errors --
 * is unchanged, and CAPSCONV_LAYOUT_NATURAL is exactly the `_pad` call.
 * An unknown layout value is CAPSCONV_ERR_DTYPE.  In the ROWS layout the
 * library runs its TMA-fed tensor-core kernels when they take the problem
 * (bf16, 4x4 capsules, C and Cout multiples of 4, pad 0, 16-byte aligned
 * pointers); any other valid problem runs the natural-layout path between
 * two on-device permutations held in the workspace (query the size with
 * capsconv_workspace_bytes_ex), so every valid call has a path. */
CAPSCONV_API capsconv_status_t capsconv_workspace_bytes_ex(capsconv_op_t op, capsconv_dtype_t dt,
        capsconv_layout_t layout, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        size_t *bytes);

CAPSCONV_API capsconv_status_t capsconv_select_path_ex(capsconv_op_t op, capsconv_dtype_t dt,
        capsconv_layout_t layout, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        capsconv_path_t *path);

CAPSCONV_API capsconv_status_t capsconv_fwd_ex(capsconv_dtype_t dt, capsconv_layout_t layout,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        const void *I, const void *K, void *O,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

CAPSCONV_API capsconv_status_t capsconv_bwd_data_ex(capsconv_dtype_t dt, capsconv_layout_t layout,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        const void *dO, const void *K, void *dI,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

CAPSCONV_API capsconv_status_t capsconv_bwd_kernel_ex(capsconv_dtype_t dt, capsconv_layout_t layout,
        int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
        const void *I, const void *dO, float *dK,
        void *workspace, size_t workspace_bytes, capsconv_stream_t stream);

/* ---- Training-step helper (the routing-free P-CapsNet
 * training step of PAPER.md:278 / Fig 7): one plain SGD step on a weight
 * tensor kept in fp32 ("master" copy), with its working copy re-rounded:
 *   w_master[i] -= lr * grad[i];   w_out[i] = round_wdt(w_master[i])
 * for i < n, elementwise, in fp32 (RNE to bf16 when wdt = CAPSCONV_BF16;
 * w_out may be w_master itself when wdt = CAPSCONV_F32).  grad is a dK of
 * this library (fp32, the layout of K).  w_master and grad are device fp32
 * arrays of n elements, w_out a device array of n `wdt` elements; caller-
 * owned, 16-byte aligned; w_out must not overlap grad.  n = 0 is a no-op.
 * Asynchronous on `stream` like every call; errors as above (NULL pointer
 * with n > 0 -> CAPSCONV_ERR_NULL, n < 0 or a non-finite lr ->
 * CAPSCONV_ERR_SHAPE, unknown wdt -> CAPSCONV_ERR_DTYPE). */
CAPSCONV_API capsconv_status_t capsconv_sgd_update(capsconv_dtype_t wdt, int64_t n, float lr, float *w_master,
        const float *grad, void *w_out, capsconv_stream_t stream);

/* Static description of a status code. */
CAPSCONV_API const char *capsconv_status_string(capsconv_status_t status);

/* Thread-local detail message of the last failing call on this thread ("" if none). */
CAPSCONV_API const char *capsconv_last_error(void);

/* Number of CUDA kernels this process has enqueued through libcapsconv so far
 * (monotonic, all threads).  Lets a caller count its device launches. */
CAPSCONV_API uint64_t capsconv_launch_count(void);

/* Library version, "MAJOR.MINOR.PATCH". */
CAPSCONV_API const char *capsconv_version(void);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* CAPSCONV_H_ */
