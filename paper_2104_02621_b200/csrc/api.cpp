// api.cpp -- the C ABI of libcapsconv (include/capsconv.h): validation,
// shape law, workspace query, path dispatch, error mapping.
//
// Every argument is validated before anything is enqueued, so a non-OK
// status other than CAPSCONV_ERR_CUDA leaves all buffers untouched.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>

#include <cuda_runtime.h>

#include "internal.h"

namespace capsconv {

static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_path_override{CAPSCONV_PATH_AUTO};
static thread_local std::string t_last_error;

void note_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

cudaError_t smem_optin(const void *func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> done;   // (function, device) -> bytes opted in
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    int &have = done[std::make_pair(func, dev)];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

// Per stream, the byte range of the last libcapsconv call's output: a call
// whose K overlaps it packs K fully ordered (no programmatic overlap).
static thread_local bool t_pack_overlap = true;
bool pack_may_overlap() { return t_pack_overlap; }

namespace {
struct OutRange {
    uintptr_t lo = 0, hi = 0;
};
std::mutex g_out_mu;
std::unordered_map<cudaStream_t, OutRange> g_last_out;

// Before a call: may its weight pack overlap the previous call on `cs`?
void pack_guard_begin(cudaStream_t cs, const void *K, size_t k_bytes) {
    bool ok = true;
    if (K) {
        const uintptr_t lo = reinterpret_cast<uintptr_t>(K), hi = lo + k_bytes;
        std::lock_guard<std::mutex> lock(g_out_mu);
        auto it = g_last_out.find(cs);
        if (it != g_last_out.end() && lo < it->second.hi && it->second.lo < hi) ok = false;
    }
    t_pack_overlap = ok;
}
// After a call: remember its output range on `cs`.
void pack_guard_end(cudaStream_t cs, const void *out, size_t out_bytes) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(out);
    std::lock_guard<std::mutex> lock(g_out_mu);
    if (g_last_out.size() > 4096) g_last_out.clear();   // bound the table (streams come and go)
    g_last_out[cs] = OutRange{lo, lo + out_bytes};
    t_pack_overlap = true;
}
}  // namespace

bool pdl_enabled() {
    static const bool on = probe_env("CAPSCONV_NO_PDL") == nullptr;
    return on;
}

static capsconv_status_t fail(capsconv_status_t st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static capsconv_status_t fail(capsconv_status_t st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_last_error = buf;
    return st;
}

const DeviceInfo &device_info() {
    // Cached per current device (the common case is one device per process).
    static thread_local DeviceInfo info;
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        info = DeviceInfo{};
        return info;
    }
    if (info.device != dev) {
        DeviceInfo d;
        d.device = dev;
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) d.num_sms = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess) d.cc_major = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess) d.cc_minor = v;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess)
            d.smem_optin = (size_t)v;
        cudaGetLastError();
        info = d;
    }
    return info;
}

// Product of extents with overflow detection.
static bool mul_ok(int64_t a, int64_t b, int64_t *out) {
    if (a > 0 && b > std::numeric_limits<int64_t>::max() / a) return false;
    *out = a * b;
    return true;
}

static capsconv_status_t make_problem(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C,
                                      int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                                      int64_t s, int64_t pad, Problem *p, int layout = CAPSCONV_LAYOUT_NATURAL) {
    if (dt != CAPSCONV_F32 && dt != CAPSCONV_BF16) return fail(CAPSCONV_ERR_DTYPE, "unknown dtype %d", (int)dt);
    if (layout != CAPSCONV_LAYOUT_NATURAL && layout != CAPSCONV_LAYOUT_ROWS)
        return fail(CAPSCONV_ERR_DTYPE, "unknown layout %d", layout);
    if (s < 1) return fail(CAPSCONV_ERR_STRIDE, "stride %lld < 1", (long long)s);
    if (pad < 0 || pad > (1 << 20)) return fail(CAPSCONV_ERR_SHAPE, "padding %lld out of [0, 2^20]", (long long)pad);
    const int64_t ext[] = {B, H, W, C, Cout, KH, KW, D1, D2, D3};
    const char *names[] = {"B", "H", "W", "C", "Cout", "KH", "KW", "D1", "D2", "D3"};
    for (int i = 0; i < 10; ++i)
        if (ext[i] < 1) return fail(CAPSCONV_ERR_SHAPE, "extent %s = %lld < 1", names[i], (long long)ext[i]);
    if (KH > H + 2 * pad || KW > W + 2 * pad)
        return fail(CAPSCONV_ERR_SHAPE, "kernel %lldx%lld larger than padded input %lldx%lld", (long long)KH,
                    (long long)KW, (long long)(H + 2 * pad), (long long)(W + 2 * pad));
    p->dt = dt;
    p->B = B; p->H = H; p->W = W; p->C = C; p->Cout = Cout;
    p->KH = KH; p->KW = KW; p->D1 = D1; p->D2 = D2; p->D3 = D3; p->s = s; p->pad = pad;
    p->Ho = (H + 2 * pad - KH) / s + 1;
    p->Wo = (W + 2 * pad - KW) / s + 1;
    p->layout = layout;
    // Element counts (and their byte sizes) must fit comfortably in int64.
    int64_t n = 1;
    const int64_t in_f[] = {B, H, W, C, D1, D2, 8};
    for (int64_t f : in_f)
        if (!mul_ok(n, f, &n)) return fail(CAPSCONV_ERR_OVERFLOW, "input element count overflows int64");
    n = 1;
    const int64_t out_f[] = {B, p->Ho, p->Wo, Cout, D1, D3, 8};
    for (int64_t f : out_f)
        if (!mul_ok(n, f, &n)) return fail(CAPSCONV_ERR_OVERFLOW, "output element count overflows int64");
    n = 1;
    const int64_t k_f[] = {KH, KW, C, Cout, D2, D3, 8};
    for (int64_t f : k_f)
        if (!mul_ok(n, f, &n)) return fail(CAPSCONV_ERR_OVERFLOW, "kernel element count overflows int64");
    // Grid limits of the SIMT path: one thread per output element at most.
    if (p->n_in() > (int64_t)1 << 40 || p->n_out() > (int64_t)1 << 40)
        return fail(CAPSCONV_ERR_OVERFLOW, "problem exceeds 2^40 elements per tensor");
    return CAPSCONV_OK;
}

// ---- rows layout (D1-outer): the TMA-fed tensor-core kernels when they take
// the problem, else the natural-layout path between two permutations.
static bool rows_mma(capsconv_op_t op, const Problem &p) {
    if (p.layout != CAPSCONV_LAYOUT_ROWS || g_path_override.load() == CAPSCONV_PATH_SIMT) return false;
    if (rows_fc_supported(op, p) || rows_walk_supported(op, p)) return true;
    return op == CAPSCONV_OP_BWD_KERNEL ? rows_wgrad_supported(p) : rows_conv_supported(op, p);
}
static size_t rows_mma_ws(capsconv_op_t op, const Problem &p) {
    if (rows_fc_supported(op, p)) return rows_fc_workspace_bytes(op, p);
    if (rows_walk_supported(op, p)) return rows_walk_workspace_bytes(op, p);
    return op == CAPSCONV_OP_BWD_KERNEL ? rows_wgrad_workspace_bytes(p) : rows_conv_workspace_bytes(op, p);
}
static Problem natural_of(const Problem &p) {
    Problem q = p;
    q.layout = CAPSCONV_LAYOUT_NATURAL;
    return q;
}
static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
// fallback workspace: [natural copy of the first operand][natural copy of the
// second operand or of the output][the natural path's own workspace]
static size_t rows_fb_a(capsconv_op_t op, const Problem &p) {
    return align256((size_t)(op == CAPSCONV_OP_BWD_DATA ? p.n_out() : p.n_in()) * p.elem());
}
static size_t rows_fb_b(capsconv_op_t op, const Problem &p) {
    return align256((size_t)(op == CAPSCONV_OP_BWD_DATA ? p.n_in() : p.n_out()) * p.elem());
}

static capsconv_path_t choose_path(capsconv_op_t op, const Problem &p) {
    const int ov = g_path_override.load();
    if (ov == CAPSCONV_PATH_SIMT) return CAPSCONV_PATH_SIMT;
    if (p.layout == CAPSCONV_LAYOUT_ROWS) {
        if (rows_mma(op, p)) return CAPSCONV_PATH_MMA;
        return choose_path(op, natural_of(p));
    }
    if (mma_supported(op, p) || primary_tc(op, p)) return CAPSCONV_PATH_MMA;
    return CAPSCONV_PATH_SIMT;
}

static size_t workspace_for(capsconv_op_t op, const Problem &p) {
    if (p.layout == CAPSCONV_LAYOUT_ROWS) {
        const size_t fb = rows_fb_a(op, p) + rows_fb_b(op, p) + workspace_for(op, natural_of(p));
        if (!rows_mma(op, p)) return fb;
        // misaligned pointers take the fallback: cover both
        return std::max(rows_mma_ws(op, p), fb);
    }
    // every kernel family that may take the call (misaligned pointers fall back
    // to the SIMT kernels), so the workspace covers all of them
    size_t need = simt_workspace_bytes(op, p);
    if (mma_supported(op, p)) need = std::max(need, mma_workspace_bytes(op, p));
    if (primary_supported(p)) need = std::max(need, primary_workspace_bytes(op, p));
    return need;
}

static capsconv_status_t check_device() {
    const DeviceInfo &d = device_info();
    if (d.device < 0) return fail(CAPSCONV_ERR_DEVICE, "no CUDA device available");
    if (d.cc_major != 10 || d.cc_minor != 0)
        return fail(CAPSCONV_ERR_DEVICE, "device %d is sm_%d%d; libcapsconv is built for sm_100a only", d.device,
                    d.cc_major, d.cc_minor);
    return CAPSCONV_OK;
}

static bool aligned16(const void *a) { return ((uintptr_t)a & 15u) == 0; }

static capsconv_status_t finish(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return fail(CAPSCONV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    t_last_error.clear();
    return CAPSCONV_OK;
}

// Path choice + launch for a validated problem (the body shared by the
// plain, padded and S-slice entry points).
static cudaError_t dispatch(capsconv_op_t op, const Problem &p, const void *a, const void *b, void *out, void *ws,
                            size_t ws_bytes, cudaStream_t cs);

// Rows-layout call: a = I (fwd, dK) or dO (dI); b = K (fwd, dI) or dO (dK).
static cudaError_t dispatch_rows(capsconv_op_t op, const Problem &p, const void *a, const void *b, void *out,
                                 void *ws, size_t ws_bytes, cudaStream_t cs) {
    const size_t need = rows_mma(op, p) ? rows_mma_ws(op, p) : 0;
    if (rows_mma(op, p) && aligned16(a) && aligned16(b) && aligned16(out) && (need == 0 || aligned16(ws))) {
        if (rows_fc_supported(op, p)) return rows_fc_run(op, p, a, b, out, ws, ws_bytes, cs);
        if (rows_walk_supported(op, p)) return rows_walk_run(op, p, a, b, out, ws, ws_bytes, cs);
        if (op == CAPSCONV_OP_BWD_KERNEL)
            return rows_wgrad_run(p, a, b, static_cast<float *>(out), ws, ws_bytes, cs);
        return rows_conv_run(op, p, a, b, out, ws, ws_bytes, cs);
    }
    const Problem q = natural_of(p);
    uint8_t *w8 = static_cast<uint8_t *>(ws);
    const size_t na = rows_fb_a(op, p), nb = rows_fb_b(op, p);
    if (ws_bytes < na + nb) return cudaErrorInvalidValue;
    void *wa = w8, *wb = w8 + na, *wr = w8 + na + nb;
    const size_t rest = ws_bytes - na - nb;
    const int64_t pin = p.B * p.H * p.W, pout = p.B * p.Ho * p.Wo;
    cudaError_t e;
    switch (op) {
        case CAPSCONV_OP_FWD:
            e = permute_layout(p.dt, a, wa, pin, p.C, p.D1, p.D2, 0, cs);
            if (e == cudaSuccess) e = dispatch(op, q, wa, b, wb, wr, rest, cs);
            if (e == cudaSuccess) e = permute_layout(p.dt, wb, out, pout, p.Cout, p.D1, p.D3, 1, cs);
            return e;
        case CAPSCONV_OP_BWD_DATA:
            e = permute_layout(p.dt, a, wa, pout, p.Cout, p.D1, p.D3, 0, cs);
            if (e == cudaSuccess) e = dispatch(op, q, wa, b, wb, wr, rest, cs);
            if (e == cudaSuccess) e = permute_layout(p.dt, wb, out, pin, p.C, p.D1, p.D2, 1, cs);
            return e;
        default:
            e = permute_layout(p.dt, a, wa, pin, p.C, p.D1, p.D2, 0, cs);
            if (e == cudaSuccess) e = permute_layout(p.dt, b, wb, pout, p.Cout, p.D1, p.D3, 0, cs);
            if (e == cudaSuccess) e = dispatch(op, q, wa, wb, out, wr, rest, cs);
            return e;
    }
}

static cudaError_t dispatch(capsconv_op_t op, const Problem &p, const void *a, const void *b, void *out, void *ws,
                            size_t ws_bytes, cudaStream_t cs) {
    if (p.layout == CAPSCONV_LAYOUT_ROWS) return dispatch_rows(op, p, a, b, out, ws, ws_bytes, cs);
    const size_t need = workspace_for(op, p);
    if (op != CAPSCONV_OP_BWD_DATA && primary_supported(p) && g_path_override.load() != CAPSCONV_PATH_SIMT &&
        aligned16(a) && aligned16(b) && aligned16(out) && aligned16(ws) &&
        ws_bytes >= primary_workspace_bytes(op, p))   // one-channel plain convolution (primary.cu)
        return op == CAPSCONV_OP_FWD ? primary_fwd(p, a, b, out, cs)
                                     : primary_bwd_kernel(p, a, b, static_cast<float *>(out), ws, cs);
    const bool mma = choose_path(op, p) == CAPSCONV_PATH_MMA && aligned16(a) && aligned16(b) && aligned16(out) &&
                     (need == 0 || aligned16(ws));
    switch (op) {
        case CAPSCONV_OP_FWD: return mma ? mma_fwd(p, a, b, out, ws, ws_bytes, cs) : simt_fwd(p, a, b, out, ws, ws_bytes, cs);
        case CAPSCONV_OP_BWD_DATA:
            return mma ? mma_bwd_data(p, a, b, out, ws, ws_bytes, cs) : simt_bwd_data(p, a, b, out, cs);
        default:
            return mma ? mma_bwd_kernel(p, a, b, static_cast<float *>(out), ws, ws_bytes, cs)
                       : simt_bwd_kernel(p, a, b, static_cast<float *>(out), ws, ws_bytes, cs);
    }
}

// S-slice capsules (R22): the expanded problem (C*S, Cout*S channels) and
// the workspace = [expanded kernel K' (fwd, dI) or expanded dK' (fp32, dK)] +
// the expanded problem's own workspace.
static capsconv_status_t make_slices(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                                     int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3,
                                     int64_t s, Problem *pe) {
    if (S < 1 || S > 64) return fail(CAPSCONV_ERR_SHAPE, "slice count S = %lld out of [1, 64]", (long long)S);
    int64_t cs = 0, cos = 0;
    if (!mul_ok(C, S, &cs) || !mul_ok(Cout, S, &cos)) return fail(CAPSCONV_ERR_OVERFLOW, "C*S or Cout*S overflows");
    return make_problem(dt, B, H, W, cs, cos, KH, KW, D1, D2, D3, s, 0, pe);
}

static size_t slices_aux_bytes(capsconv_op_t op, const Problem &pe) {
    const size_t n = (size_t)pe.KH * pe.KW * pe.C * pe.Cout * pe.D2 * pe.D3;   // expanded kernel elements
    const size_t b = op == CAPSCONV_OP_BWD_KERNEL ? 4 * n : pe.elem() * n;
    return (b + 255) & ~(size_t)255;
}

}  // namespace capsconv

using namespace capsconv;

extern "C" {

capsconv_status_t capsconv_output_dims_pad(int64_t H, int64_t W, int64_t KH, int64_t KW, int64_t stride,
                                           int64_t pad, int64_t *Ho, int64_t *Wo) {
    if (!Ho || !Wo) return fail(CAPSCONV_ERR_NULL, "Ho/Wo output pointer is NULL");
    if (stride < 1) return fail(CAPSCONV_ERR_STRIDE, "stride %lld < 1", (long long)stride);
    if (pad < 0 || pad > (1 << 20)) return fail(CAPSCONV_ERR_SHAPE, "padding %lld out of [0, 2^20]", (long long)pad);
    if (H < 1 || W < 1 || KH < 1 || KW < 1 || KH > H + 2 * pad || KW > W + 2 * pad)
        return fail(CAPSCONV_ERR_SHAPE, "invalid spatial extents H=%lld W=%lld KH=%lld KW=%lld pad=%lld",
                    (long long)H, (long long)W, (long long)KH, (long long)KW, (long long)pad);
    *Ho = (H + 2 * pad - KH) / stride + 1;
    *Wo = (W + 2 * pad - KW) / stride + 1;
    return CAPSCONV_OK;
}

capsconv_status_t capsconv_output_dims(int64_t H, int64_t W, int64_t KH, int64_t KW, int64_t stride, int64_t *Ho,
                                       int64_t *Wo) {
    return capsconv_output_dims_pad(H, W, KH, KW, stride, 0, Ho, Wo);
}

capsconv_status_t capsconv_workspace_bytes_pad(capsconv_op_t op, capsconv_dtype_t dt, int64_t B, int64_t H,
                                               int64_t W, int64_t C, int64_t Cout, int64_t KH, int64_t KW,
                                               int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
                                               size_t *bytes) {
    if (!bytes) return fail(CAPSCONV_ERR_NULL, "bytes pointer is NULL");
    if (op < CAPSCONV_OP_FWD || op > CAPSCONV_OP_BWD_KERNEL) return fail(CAPSCONV_ERR_DTYPE, "unknown op %d", (int)op);
    Problem p;
    capsconv_status_t st = make_problem(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, &p);
    if (st) return st;
    *bytes = workspace_for(op, p);
    return CAPSCONV_OK;
}

capsconv_status_t capsconv_workspace_bytes(capsconv_op_t op, capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W,
                                           int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2,
                                           int64_t D3, int64_t stride, size_t *bytes) {
    return capsconv_workspace_bytes_pad(op, dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, 0, bytes);
}

capsconv_status_t capsconv_select_path_pad(capsconv_op_t op, capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W,
                                           int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2,
                                           int64_t D3, int64_t stride, int64_t pad, capsconv_path_t *path) {
    if (!path) return fail(CAPSCONV_ERR_NULL, "path pointer is NULL");
    if (op < CAPSCONV_OP_FWD || op > CAPSCONV_OP_BWD_KERNEL) return fail(CAPSCONV_ERR_DTYPE, "unknown op %d", (int)op);
    Problem p;
    capsconv_status_t st = make_problem(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, &p);
    if (st) return st;
    *path = choose_path(op, p);
    return CAPSCONV_OK;
}

capsconv_status_t capsconv_select_path(capsconv_op_t op, capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W,
                                       int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2,
                                       int64_t D3, int64_t stride, capsconv_path_t *path) {
    return capsconv_select_path_pad(op, dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, 0, path);
}

capsconv_status_t capsconv_set_path_override(capsconv_path_t path) {
    if (path != CAPSCONV_PATH_AUTO && path != CAPSCONV_PATH_SIMT && path != CAPSCONV_PATH_MMA)
        return fail(CAPSCONV_ERR_DTYPE, "unknown path %d", (int)path);
    g_path_override.store((int)path);
    return CAPSCONV_OK;
}

capsconv_status_t capsconv_workspace_bytes_ex(capsconv_op_t op, capsconv_dtype_t dt, capsconv_layout_t layout,
                                              int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t KH,
                                              int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
                                              int64_t pad, size_t *bytes) {
    if (!bytes) return fail(CAPSCONV_ERR_NULL, "bytes pointer is NULL");
    if (op < CAPSCONV_OP_FWD || op > CAPSCONV_OP_BWD_KERNEL) return fail(CAPSCONV_ERR_DTYPE, "unknown op %d", (int)op);
    Problem p;
    capsconv_status_t st = make_problem(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, &p, (int)layout);
    if (st) return st;
    *bytes = workspace_for(op, p);
    return CAPSCONV_OK;
}

capsconv_status_t capsconv_select_path_ex(capsconv_op_t op, capsconv_dtype_t dt, capsconv_layout_t layout, int64_t B,
                                          int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t KH, int64_t KW,
                                          int64_t D1, int64_t D2, int64_t D3, int64_t stride, int64_t pad,
                                          capsconv_path_t *path) {
    if (!path) return fail(CAPSCONV_ERR_NULL, "path pointer is NULL");
    if (op < CAPSCONV_OP_FWD || op > CAPSCONV_OP_BWD_KERNEL) return fail(CAPSCONV_ERR_DTYPE, "unknown op %d", (int)op);
    Problem p;
    capsconv_status_t st = make_problem(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, &p, (int)layout);
    if (st) return st;
    *path = choose_path(op, p);
    return CAPSCONV_OK;
}

// Validation (all of it before any launch), then the path dispatch.
static capsconv_status_t run_op(capsconv_op_t op, capsconv_dtype_t dt, capsconv_layout_t layout, int64_t B,
                                int64_t H, int64_t W, int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1,
                                int64_t D2, int64_t D3, int64_t stride, int64_t pad, const void *a, const void *b,
                                void *out, void *workspace, size_t workspace_bytes, capsconv_stream_t stream,
                                const char *what) {
    Problem p;
    capsconv_status_t st = make_problem(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, &p, (int)layout);
    if (st) return st;
    if (!a || !b || !out) return fail(CAPSCONV_ERR_NULL, "a tensor pointer is NULL");
    const size_t need = workspace_for(op, p);
    if (workspace_bytes < need)
        return fail(CAPSCONV_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);
    if (need && !workspace) return fail(CAPSCONV_ERR_NULL, "workspace is NULL but %zu bytes are required", need);
    st = check_device();
    if (st) return st;
    const cudaStream_t cs = (cudaStream_t)stream;
    pack_guard_begin(cs, op == CAPSCONV_OP_BWD_KERNEL ? nullptr : b, p.kernel_bytes());
    const cudaError_t e = dispatch(op, p, a, b, out, workspace, workspace_bytes, cs);
    pack_guard_end(cs, out, p.out_bytes(op));
    return finish(e, what);
}

capsconv_status_t capsconv_fwd_ex(capsconv_dtype_t dt, capsconv_layout_t layout, int64_t B, int64_t H, int64_t W,
                                  int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                                  int64_t stride, int64_t pad, const void *I, const void *K, void *O, void *workspace,
                                  size_t workspace_bytes, capsconv_stream_t stream) {
    return run_op(CAPSCONV_OP_FWD, dt, layout, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, I, K, O, workspace,
                  workspace_bytes, stream, "capsconv_fwd");
}

capsconv_status_t capsconv_bwd_data_ex(capsconv_dtype_t dt, capsconv_layout_t layout, int64_t B, int64_t H,
                                       int64_t W, int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1,
                                       int64_t D2, int64_t D3, int64_t stride, int64_t pad, const void *dO,
                                       const void *K, void *dI, void *workspace, size_t workspace_bytes,
                                       capsconv_stream_t stream) {
    return run_op(CAPSCONV_OP_BWD_DATA, dt, layout, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, dO, K, dI,
                  workspace, workspace_bytes, stream, "capsconv_bwd_data");
}

capsconv_status_t capsconv_bwd_kernel_ex(capsconv_dtype_t dt, capsconv_layout_t layout, int64_t B, int64_t H,
                                         int64_t W, int64_t C, int64_t Cout, int64_t KH, int64_t KW, int64_t D1,
                                         int64_t D2, int64_t D3, int64_t stride, int64_t pad, const void *I,
                                         const void *dO, float *dK, void *workspace, size_t workspace_bytes,
                                         capsconv_stream_t stream) {
    return run_op(CAPSCONV_OP_BWD_KERNEL, dt, layout, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, I, dO, dK,
                  workspace, workspace_bytes, stream, "capsconv_bwd_kernel");
}

capsconv_status_t capsconv_fwd_pad(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                                   int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
                                   int64_t pad, const void *I, const void *K, void *O, void *workspace,
                                   size_t workspace_bytes, capsconv_stream_t stream) {
    return capsconv_fwd_ex(dt, CAPSCONV_LAYOUT_NATURAL, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, I, K, O,
                           workspace, workspace_bytes, stream);
}

capsconv_status_t capsconv_fwd(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                               int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
                               const void *I, const void *K, void *O, void *workspace, size_t workspace_bytes,
                               capsconv_stream_t stream) {
    return capsconv_fwd_pad(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, 0, I, K, O, workspace, workspace_bytes,
                            stream);
}

capsconv_status_t capsconv_bwd_data_pad(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C,
                                        int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                                        int64_t stride, int64_t pad, const void *dO, const void *K, void *dI,
                                        void *workspace, size_t workspace_bytes, capsconv_stream_t stream) {
    return capsconv_bwd_data_ex(dt, CAPSCONV_LAYOUT_NATURAL, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, dO, K,
                                dI, workspace, workspace_bytes, stream);
}

capsconv_status_t capsconv_bwd_data(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                                    int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
                                    const void *dO, const void *K, void *dI, void *workspace,
                                    size_t workspace_bytes, capsconv_stream_t stream) {
    return capsconv_bwd_data_pad(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, 0, dO, K, dI, workspace,
                                 workspace_bytes, stream);
}

capsconv_status_t capsconv_bwd_kernel_pad(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C,
                                          int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                                          int64_t stride, int64_t pad, const void *I, const void *dO, float *dK,
                                          void *workspace, size_t workspace_bytes, capsconv_stream_t stream) {
    return capsconv_bwd_kernel_ex(dt, CAPSCONV_LAYOUT_NATURAL, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, pad, I,
                                  dO, dK, workspace, workspace_bytes, stream);
}

capsconv_status_t capsconv_bwd_kernel(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C,
                                      int64_t Cout, int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                                      int64_t stride, const void *I, const void *dO, float *dK, void *workspace,
                                      size_t workspace_bytes, capsconv_stream_t stream) {
    return capsconv_bwd_kernel_pad(dt, B, H, W, C, Cout, KH, KW, D1, D2, D3, stride, 0, I, dO, dK, workspace,
                                   workspace_bytes, stream);
}

capsconv_status_t capsconv_workspace_bytes_slices(capsconv_op_t op, capsconv_dtype_t dt, int64_t B, int64_t H,
                                                  int64_t W, int64_t C, int64_t Cout, int64_t KH, int64_t KW,
                                                  int64_t S, int64_t D1, int64_t D2, int64_t D3, int64_t stride,
                                                  size_t *bytes) {
    if (!bytes) return fail(CAPSCONV_ERR_NULL, "bytes pointer is NULL");
    if (op < CAPSCONV_OP_FWD || op > CAPSCONV_OP_BWD_KERNEL) return fail(CAPSCONV_ERR_DTYPE, "unknown op %d", (int)op);
    Problem pe;
    capsconv_status_t st = make_slices(dt, B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride, &pe);
    if (st) return st;
    *bytes = slices_aux_bytes(op, pe) + workspace_for(op, pe);
    return CAPSCONV_OK;
}

#define CAPSCONV_SLICES_PROLOGUE(OP, A, B_, OUT)                                                              \
    Problem pe;                                                                                               \
    capsconv_status_t st = make_slices(dt, B, H, W, C, Cout, KH, KW, S, D1, D2, D3, stride, &pe);             \
    if (st) return st;                                                                                        \
    if (!(A) || !(B_) || !(OUT)) return fail(CAPSCONV_ERR_NULL, "a tensor pointer is NULL");                  \
    const size_t aux = slices_aux_bytes(OP, pe), need = aux + workspace_for(OP, pe);                          \
    if (workspace_bytes < need)                                                                               \
        return fail(CAPSCONV_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);     \
    if (!workspace) return fail(CAPSCONV_ERR_NULL, "workspace is NULL but %zu bytes are required", need);     \
    st = check_device();                                                                                      \
    if (st) return st;                                                                                        \
    cudaStream_t cs = (cudaStream_t)stream;                                                                   \
    uint8_t *ws8 = static_cast<uint8_t *>(workspace);                                                         \
    void *inner_ws = aux < workspace_bytes ? ws8 + aux : nullptr;                                             \
    const size_t inner_bytes = workspace_bytes - aux;

capsconv_status_t capsconv_fwd_slices(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                                      int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3,
                                      int64_t stride, const void *I, const void *K, void *O, void *workspace,
                                      size_t workspace_bytes, capsconv_stream_t stream) {
    CAPSCONV_SLICES_PROLOGUE(CAPSCONV_OP_FWD, I, K, O)
    cudaError_t e = slices_expand_kernel(dt, K, ws8, KH * KW, C, Cout, S, D2 * D3, cs);
    if (e == cudaSuccess) e = dispatch(CAPSCONV_OP_FWD, pe, I, ws8, O, inner_ws, inner_bytes, cs);
    pack_guard_end(cs, O, (size_t)pe.n_out() * pe.elem());
    return finish(e, "capsconv_fwd_slices");
}

capsconv_status_t capsconv_bwd_data_slices(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C,
                                           int64_t Cout, int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2,
                                           int64_t D3, int64_t stride, const void *dO, const void *K, void *dI,
                                           void *workspace, size_t workspace_bytes, capsconv_stream_t stream) {
    CAPSCONV_SLICES_PROLOGUE(CAPSCONV_OP_BWD_DATA, dO, K, dI)
    cudaError_t e = slices_expand_kernel(dt, K, ws8, KH * KW, C, Cout, S, D2 * D3, cs);
    if (e == cudaSuccess) e = dispatch(CAPSCONV_OP_BWD_DATA, pe, dO, ws8, dI, inner_ws, inner_bytes, cs);
    pack_guard_end(cs, dI, (size_t)pe.n_in() * pe.elem());
    return finish(e, "capsconv_bwd_data_slices");
}

capsconv_status_t capsconv_bwd_kernel_slices(capsconv_dtype_t dt, int64_t B, int64_t H, int64_t W, int64_t C,
                                             int64_t Cout, int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2,
                                             int64_t D3, int64_t stride, const void *I, const void *dO, float *dK,
                                             void *workspace, size_t workspace_bytes, capsconv_stream_t stream) {
    CAPSCONV_SLICES_PROLOGUE(CAPSCONV_OP_BWD_KERNEL, I, dO, dK)
    float *dKx = reinterpret_cast<float *>(ws8);
    cudaError_t e = dispatch(CAPSCONV_OP_BWD_KERNEL, pe, I, dO, dKx, inner_ws, inner_bytes, cs);
    if (e == cudaSuccess) e = slices_extract_dk(dKx, dK, KH * KW, C, Cout, S, D2 * D3, cs);
    pack_guard_end(cs, dK, (size_t)pe.n_k() * 4);   // bound: the expanded dK
    return finish(e, "capsconv_bwd_kernel_slices");
}

capsconv_status_t capsconv_sgd_update(capsconv_dtype_t wdt, int64_t n, float lr, float *w_master,
                                      const float *grad, void *w_out, capsconv_stream_t stream) {
    if (wdt != CAPSCONV_BF16 && wdt != CAPSCONV_F32) return fail(CAPSCONV_ERR_DTYPE, "unknown weight dtype %d", (int)wdt);
    if (n < 0) return fail(CAPSCONV_ERR_SHAPE, "n = %lld < 0", (long long)n);
    if (!std::isfinite(lr)) return fail(CAPSCONV_ERR_SHAPE, "learning rate is not finite");
    if (n == 0) return CAPSCONV_OK;
    if (!w_master || !grad || !w_out) return fail(CAPSCONV_ERR_NULL, "a tensor pointer is NULL");
    if (!aligned16(w_master) || !aligned16(grad) || !aligned16(w_out))
        return fail(CAPSCONV_ERR_SHAPE, "sgd_update pointers must be 16-byte aligned");
    const capsconv_status_t st = check_device();
    if (st) return st;
    const cudaStream_t cs = (cudaStream_t)stream;
    const cudaError_t e = sgd_update(wdt, n, lr, w_master, grad, w_out, cs);
    pack_guard_end(cs, w_out, (size_t)n * (wdt == CAPSCONV_BF16 ? 2 : 4));   // w_out is the next call's K
    return finish(e, "capsconv_sgd_update");
}

const char *capsconv_status_string(capsconv_status_t s) {
    switch (s) {
        case CAPSCONV_OK: return "CAPSCONV_OK";
        case CAPSCONV_ERR_NULL: return "CAPSCONV_ERR_NULL: a required pointer is NULL";
        case CAPSCONV_ERR_SHAPE: return "CAPSCONV_ERR_SHAPE: extent < 1 or kernel larger than input";
        case CAPSCONV_ERR_STRIDE: return "CAPSCONV_ERR_STRIDE: stride < 1";
        case CAPSCONV_ERR_DTYPE: return "CAPSCONV_ERR_DTYPE: unknown dtype, op or path";
        case CAPSCONV_ERR_WORKSPACE: return "CAPSCONV_ERR_WORKSPACE: workspace too small";
        case CAPSCONV_ERR_OVERFLOW: return "CAPSCONV_ERR_OVERFLOW: element count or index range too large";
        case CAPSCONV_ERR_DEVICE: return "CAPSCONV_ERR_DEVICE: no sm_100 CUDA device";
        case CAPSCONV_ERR_CUDA: return "CAPSCONV_ERR_CUDA: CUDA launch/runtime error";
    }
    return "CAPSCONV_ERR_UNKNOWN";
}

const char *capsconv_last_error(void) { return t_last_error.c_str(); }

uint64_t capsconv_launch_count(void) { return g_launches.load(); }

const char *capsconv_version(void) { return "0.1.0"; }

}  // extern "C"
