/*
 * capsconv_oracle.c -- CPU oracle for the capsule convolution of
 * arXiv 2104.02621 ("How to Accelerate Capsule Convolutions in Capsule
 * Networks").  TEST INFRASTRUCTURE ONLY: this file may be built and called
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg.  The product path (paper_2104_02621_b200/) never
 * links, imports or executes it, and it shares no code, header or table
 * with the CUDA path.
 *
 * What it computes (the plain definition, written out):
 *
 *   Paper PAPER.md:84  (§1.2): input I(W,H,C,T1(D1,D2)), kernel
 *   K(w,h,c,T2(D2,D3)), output O(W',H',C',T3(D1,D3)).
 *   Paper PAPER.md:92-108 (Algorithm 2 "General capsule convolution"):
 *   for every output channel, output position and input channel / kernel
 *   tap, O_caps += matrix_multiply(I_caps, K_caps) with
 *   row_offset = i*stride, col_offset = j*stride (no padding term).
 *   matrix_multiply of a (D1 x D2) capsule by a (D2 x D3) capsule is the
 *   ordinary matrix product ("we assume both T1 and T2 are
 *   matrices").
 *
 *   O[b,x',y',c',d1,d3] = sum_{p,q,c,d2} I[b, x'*s+p, y'*s+q, c, d1, d2]
 *                                      * K[p, q, c, c', d2, d3]
 *
 *   Layouts (readings R3/R4): dense row-major
 *     I, dI : [B][H][W][C][D1][D2]
 *     K, dK : [KH][KW][C][Cout][D2][D3]
 *     O, dO : [B][Ho][Wo][Cout][D1][D3]
 *   x indexes H (rows) with tap p over KH; y indexes W with tap q over KW.
 *
 *   Backward (Algorithm 4; its typos are resolved by the
 *   analytic adjoint of the linear map above, reading R10/R11):
 *     dI[b,h,w,c,d1,d2] = sum over (p,q,c',d3) with h = x'*s+p, w = y'*s+q,
 *                         0<=x'<Ho, 0<=y'<Wo of dO[b,x',y',c',d1,d3]*K[p,q,c,c',d2,d3]
 *     dK[p,q,c,c',d2,d3] = sum_{b,x',y',d1} I[b,x'*s+p,y'*s+q,c,d1,d2]*dO[b,x',y',c',d1,d3]
 *
 * Every accumulation is done in double precision on inputs that are exact
 * in double (fp32 and bf16 values upcast exactly).  Alongside each result
 * the oracle returns sum |term| over the same terms: the denominator of the
 * error metric (reading R19).  Parallelism: one owner per output element
 * (OpenMP over the outermost output index), so results are deterministic.
 */
#include <stdint.h>
#include <math.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_SHAPE 2
#define OR_ERR_STRIDE 3

/* Shape law, PAPER.md:98-99 (row_offset = i*stride, no padding) and the
 * worked example PAPER.md:43-54 (5x5 input, 4x4 kernel -> 2x2 output). */
int oracle_output_dims(int64_t H, int64_t W, int64_t KH, int64_t KW,
                       int64_t stride, int64_t *Ho, int64_t *Wo)
{
    if (stride < 1) return OR_ERR_STRIDE;
    if (H < 1 || W < 1 || KH < 1 || KW < 1 || KH > H || KW > W) return OR_ERR_SHAPE;
    *Ho = (H - KH) / stride + 1;
    *Wo = (W - KW) / stride + 1;
    return OR_OK;
}

/* Row-major offsets of the three layouts, written out once here. */
#define IDX_I(b, h, w, c, d1, d2) \
    ((((((int64_t)(b) * H + (h)) * W + (w)) * C + (c)) * D1 + (d1)) * D2 + (d2))
#define IDX_K(p, q, c, co, d2, d3) \
    ((((((int64_t)(p) * KW + (q)) * C + (c)) * Cout + (co)) * D2 + (d2)) * D3 + (d3))
#define IDX_O(b, x, y, co, d1, d3) \
    ((((((int64_t)(b) * Ho + (x)) * Wo + (y)) * Cout + (co)) * D1 + (d1)) * D3 + (d3))

/* Forward: Algorithm 2 with matrix_multiply written out as
 * sum_{d2} I[d1,d2] * K[d2,d3]. */
int oracle_fwd(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
               int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
               int64_t stride, const double *I, const double *K,
               double *O, double *Oabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims(H, W, KH, KW, stride, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_out = B * Ho * Wo * Cout * D1 * D3;
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < n_out; ++o) {
        int64_t r = o;
        const int64_t d3 = r % D3; r /= D3;
        const int64_t d1 = r % D1; r /= D1;
        const int64_t co = r % Cout; r /= Cout;
        const int64_t y = r % Wo; r /= Wo;
        const int64_t x = r % Ho; r /= Ho;
        const int64_t b = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t p = 0; p < KH; ++p)
            for (int64_t q = 0; q < KW; ++q)
                for (int64_t c = 0; c < C; ++c)
                    for (int64_t d2 = 0; d2 < D2; ++d2) {
                        const double t = I[IDX_I(b, x * stride + p, y * stride + q, c, d1, d2)]
                                       * K[IDX_K(p, q, c, co, d2, d3)];
                        acc += t;
                        aabs += fabs(t);
                    }
        O[o] = acc;
        if (Oabs) Oabs[o] = aabs;
    }
    return OR_OK;
}

/* dI by the adjoint (gather / owner-computes form): every (p,q) whose window
 * covers (h,w) at an integral output position contributes. */
int oracle_bwd_data(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                    int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                    int64_t stride, const double *dO, const double *K,
                    double *dI, double *dIabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims(H, W, KH, KW, stride, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_in = B * H * W * C * D1 * D2;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_in; ++e) {
        int64_t r = e;
        const int64_t d2 = r % D2; r /= D2;
        const int64_t d1 = r % D1; r /= D1;
        const int64_t c = r % C; r /= C;
        const int64_t w = r % W; r /= W;
        const int64_t h = r % H; r /= H;
        const int64_t b = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t p = 0; p < KH; ++p) {
            const int64_t hx = h - p;
            if (hx < 0 || hx % stride != 0) continue;
            const int64_t x = hx / stride;
            if (x >= Ho) continue;
            for (int64_t q = 0; q < KW; ++q) {
                const int64_t wy = w - q;
                if (wy < 0 || wy % stride != 0) continue;
                const int64_t y = wy / stride;
                if (y >= Wo) continue;
                for (int64_t co = 0; co < Cout; ++co)
                    for (int64_t d3 = 0; d3 < D3; ++d3) {
                        const double t = dO[IDX_O(b, x, y, co, d1, d3)]
                                       * K[IDX_K(p, q, c, co, d2, d3)];
                        acc += t;
                        aabs += fabs(t);
                    }
            }
        }
        dI[e] = acc;
        if (dIabs) dIabs[e] = aabs;
    }
    return OR_OK;
}

/* dK: sum over batch, output positions and the D1 row index. */
int oracle_bwd_kernel(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                      int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                      int64_t stride, const double *I, const double *dO,
                      double *dK, double *dKabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims(H, W, KH, KW, stride, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_k = KH * KW * C * Cout * D2 * D3;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_k; ++e) {
        int64_t r = e;
        const int64_t d3 = r % D3; r /= D3;
        const int64_t d2 = r % D2; r /= D2;
        const int64_t co = r % Cout; r /= Cout;
        const int64_t c = r % C; r /= C;
        const int64_t q = r % KW; r /= KW;
        const int64_t p = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t b = 0; b < B; ++b)
            for (int64_t x = 0; x < Ho; ++x)
                for (int64_t y = 0; y < Wo; ++y)
                    for (int64_t d1 = 0; d1 < D1; ++d1) {
                        const double t = I[IDX_I(b, x * stride + p, y * stride + q, c, d1, d2)]
                                       * dO[IDX_O(b, x, y, co, d1, d3)];
                        acc += t;
                        aabs += fabs(t);
                    }
        dK[e] = acc;
        if (dKabs) dKabs[e] = aabs;
    }
    return OR_OK;
}

/* Round a double to the nearest bfloat16 value (round-to-nearest-even on
 * the 8-bit significand), returned as a double.  Used only by the stack
 * oracle to round activations at layer boundaries exactly where the GPU
 * path stores bf16 (reading R13).  Non-finite values pass through. */
double oracle_round_bf16(double v)
{
    if (!isfinite(v) || v == 0.0) return v;
    int e;
    const double m = frexp(v, &e);          /* v = m * 2^e, 0.5 <= |m| < 1 */
    /* bf16 keeps 8 significant bits: quantum 2^(e-8) for normal numbers.
     * Subnormal bf16 (e <= -126) keeps a fixed quantum 2^-133. */
    int qexp = e - 8;
    if (qexp < -133) qexp = -133;
    const double scaled = ldexp(v, -qexp);  /* exact: power-of-two scaling */
    const double rounded = nearbyint(scaled); /* default FE_TONEAREST = ties-to-even */
    (void)m;
    return ldexp(rounded, qexp);
}

void oracle_round_bf16_array(double *x, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) x[i] = oracle_round_bf16(x[i]);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops (timing only: bench.py's single-thread and
   all-core baselines); the arithmetic and its order per output are unchanged. */
void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------------
 * Zero padding (SPEC.md:48-53 symmetric zero padding -- the
 * paper itself has no padding term).  The definition with
 * the input read through a zero-padded view: I_pad(h, w) = I(h - pad, w - pad)
 * inside the input, 0 outside.  Shape law H' = floor((H + 2 pad - KH)/s) + 1.
 * Written out separately so the unpadded functions above (and their pins)
 * are untouched.
 * ------------------------------------------------------------------------ */
int oracle_output_dims_pad(int64_t H, int64_t W, int64_t KH, int64_t KW,
                           int64_t stride, int64_t pad, int64_t *Ho, int64_t *Wo)
{
    if (pad < 0) return OR_ERR_SHAPE;
    return oracle_output_dims(H + 2 * pad, W + 2 * pad, KH, KW, stride, Ho, Wo);
}

int oracle_fwd_pad(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                   int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                   int64_t stride, int64_t pad, const double *I, const double *K,
                   double *O, double *Oabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims_pad(H, W, KH, KW, stride, pad, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_out = B * Ho * Wo * Cout * D1 * D3;
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < n_out; ++o) {
        int64_t r = o;
        const int64_t d3 = r % D3; r /= D3;
        const int64_t d1 = r % D1; r /= D1;
        const int64_t co = r % Cout; r /= Cout;
        const int64_t y = r % Wo; r /= Wo;
        const int64_t x = r % Ho; r /= Ho;
        const int64_t b = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t p = 0; p < KH; ++p)
            for (int64_t q = 0; q < KW; ++q) {
                const int64_t h = x * stride + p - pad, w = y * stride + q - pad;
                if (h < 0 || h >= H || w < 0 || w >= W) continue;   /* a zero of the padding */
                for (int64_t c = 0; c < C; ++c)
                    for (int64_t d2 = 0; d2 < D2; ++d2) {
                        const double t = I[IDX_I(b, h, w, c, d1, d2)] * K[IDX_K(p, q, c, co, d2, d3)];
                        acc += t;
                        aabs += fabs(t);
                    }
            }
        O[o] = acc;
        if (Oabs) Oabs[o] = aabs;
    }
    return OR_OK;
}

/* dI of the padded convolution: the adjoint restricted to real input pixels
 * (h + pad = x*s + p). */
int oracle_bwd_data_pad(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                        int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                        int64_t stride, int64_t pad, const double *dO, const double *K,
                        double *dI, double *dIabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims_pad(H, W, KH, KW, stride, pad, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_in = B * H * W * C * D1 * D2;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_in; ++e) {
        int64_t r = e;
        const int64_t d2 = r % D2; r /= D2;
        const int64_t d1 = r % D1; r /= D1;
        const int64_t c = r % C; r /= C;
        const int64_t w = r % W; r /= W;
        const int64_t h = r % H; r /= H;
        const int64_t b = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t p = 0; p < KH; ++p) {
            const int64_t hx = h + pad - p;
            if (hx < 0 || hx % stride != 0) continue;
            const int64_t x = hx / stride;
            if (x >= Ho) continue;
            for (int64_t q = 0; q < KW; ++q) {
                const int64_t wy = w + pad - q;
                if (wy < 0 || wy % stride != 0) continue;
                const int64_t y = wy / stride;
                if (y >= Wo) continue;
                for (int64_t co = 0; co < Cout; ++co)
                    for (int64_t d3 = 0; d3 < D3; ++d3) {
                        const double t = dO[IDX_O(b, x, y, co, d1, d3)] * K[IDX_K(p, q, c, co, d2, d3)];
                        acc += t;
                        aabs += fabs(t);
                    }
            }
        }
        dI[e] = acc;
        if (dIabs) dIabs[e] = aabs;
    }
    return OR_OK;
}

int oracle_bwd_kernel_pad(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                          int64_t KH, int64_t KW, int64_t D1, int64_t D2, int64_t D3,
                          int64_t stride, int64_t pad, const double *I, const double *dO,
                          double *dK, double *dKabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims_pad(H, W, KH, KW, stride, pad, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_k = KH * KW * C * Cout * D2 * D3;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_k; ++e) {
        int64_t r = e;
        const int64_t d3 = r % D3; r /= D3;
        const int64_t d2 = r % D2; r /= D2;
        const int64_t co = r % Cout; r /= Cout;
        const int64_t c = r % C; r /= C;
        const int64_t q = r % KW; r /= KW;
        const int64_t p = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t b = 0; b < B; ++b)
            for (int64_t x = 0; x < Ho; ++x)
                for (int64_t y = 0; y < Wo; ++y) {
                    const int64_t h = x * stride + p - pad, w = y * stride + q - pad;
                    if (h < 0 || h >= H || w < 0 || w >= W) continue;
                    for (int64_t d1 = 0; d1 < D1; ++d1) {
                        const double t = I[IDX_I(b, h, w, c, d1, d2)] * dO[IDX_O(b, x, y, co, d1, d3)];
                        acc += t;
                        aabs += fabs(t);
                    }
                }
        dK[e] = acc;
        if (dKabs) dKabs[e] = aabs;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * S-slice capsules (SPEC.md:30-35, 90 -- PoseDims (S, M, K):
 * a rank-3 capsule is S matrices, multiplied slice-wise, which is how
 * PAPER.md:44-53's 3x3x3 capsules are read).  Layouts (reading R22):
 *   I [B][H][W][C][S][D1][D2], K [KH][KW][C][Cout][S][D2][D3],
 *   O [B][Ho][Wo][Cout][S][D1][D3]
 *   O[b,x',y',c',s,d1,d3] = sum_{p,q,c,d2} I[b,x's+p,y's+q,c,s,d1,d2] K[p,q,c,c',s,d2,d3]
 * (no padding; S = 1 is the matrix-capsule convolution above).
 * ------------------------------------------------------------------------ */
int oracle_fwd_slices(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                      int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3,
                      int64_t stride, const double *I, const double *K, double *O, double *Oabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims(H, W, KH, KW, stride, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || S < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_out = B * Ho * Wo * Cout * S * D1 * D3;
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < n_out; ++o) {
        int64_t r = o;
        const int64_t d3 = r % D3; r /= D3;
        const int64_t d1 = r % D1; r /= D1;
        const int64_t sl = r % S; r /= S;
        const int64_t co = r % Cout; r /= Cout;
        const int64_t y = r % Wo; r /= Wo;
        const int64_t x = r % Ho; r /= Ho;
        const int64_t b = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t p = 0; p < KH; ++p)
            for (int64_t q = 0; q < KW; ++q)
                for (int64_t c = 0; c < C; ++c)
                    for (int64_t d2 = 0; d2 < D2; ++d2) {
                        const int64_t ii = ((((((b * H + x * stride + p) * W + y * stride + q) * C + c) * S + sl)
                                             * D1 + d1) * D2 + d2);
                        const int64_t kk = ((((((p * KW + q) * C + c) * Cout + co) * S + sl) * D2 + d2) * D3 + d3);
                        const double t = I[ii] * K[kk];
                        acc += t;
                        aabs += fabs(t);
                    }
        O[o] = acc;
        if (Oabs) Oabs[o] = aabs;
    }
    return OR_OK;
}

/* dI and dK of the slice-wise map, as adjoints (R10/R11 per slice). */
int oracle_bwd_data_slices(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                           int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3,
                           int64_t stride, const double *dO, const double *K, double *dI, double *dIabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims(H, W, KH, KW, stride, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || S < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_in = B * H * W * C * S * D1 * D2;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_in; ++e) {
        int64_t r = e;
        const int64_t d2 = r % D2; r /= D2;
        const int64_t d1 = r % D1; r /= D1;
        const int64_t sl = r % S; r /= S;
        const int64_t c = r % C; r /= C;
        const int64_t w = r % W; r /= W;
        const int64_t h = r % H; r /= H;
        const int64_t b = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t p = 0; p < KH; ++p) {
            const int64_t hx = h - p;
            if (hx < 0 || hx % stride != 0) continue;
            const int64_t x = hx / stride;
            if (x >= Ho) continue;
            for (int64_t q = 0; q < KW; ++q) {
                const int64_t wy = w - q;
                if (wy < 0 || wy % stride != 0) continue;
                const int64_t y = wy / stride;
                if (y >= Wo) continue;
                for (int64_t co = 0; co < Cout; ++co)
                    for (int64_t d3 = 0; d3 < D3; ++d3) {
                        const int64_t oo = ((((((b * Ho + x) * Wo + y) * Cout + co) * S + sl) * D1 + d1) * D3 + d3);
                        const int64_t kk = ((((((p * KW + q) * C + c) * Cout + co) * S + sl) * D2 + d2) * D3 + d3);
                        const double t = dO[oo] * K[kk];
                        acc += t;
                        aabs += fabs(t);
                    }
            }
        }
        dI[e] = acc;
        if (dIabs) dIabs[e] = aabs;
    }
    return OR_OK;
}

int oracle_bwd_kernel_slices(int64_t B, int64_t H, int64_t W, int64_t C, int64_t Cout,
                             int64_t KH, int64_t KW, int64_t S, int64_t D1, int64_t D2, int64_t D3,
                             int64_t stride, const double *I, const double *dO, double *dK, double *dKabs)
{
    int64_t Ho, Wo;
    int rc = oracle_output_dims(H, W, KH, KW, stride, &Ho, &Wo);
    if (rc) return rc;
    if (B < 1 || C < 1 || Cout < 1 || S < 1 || D1 < 1 || D2 < 1 || D3 < 1) return OR_ERR_SHAPE;
    const int64_t n_k = KH * KW * C * Cout * S * D2 * D3;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n_k; ++e) {
        int64_t r = e;
        const int64_t d3 = r % D3; r /= D3;
        const int64_t d2 = r % D2; r /= D2;
        const int64_t sl = r % S; r /= S;
        const int64_t co = r % Cout; r /= Cout;
        const int64_t c = r % C; r /= C;
        const int64_t q = r % KW; r /= KW;
        const int64_t p = r;
        double acc = 0.0, aabs = 0.0;
        for (int64_t b = 0; b < B; ++b)
            for (int64_t x = 0; x < Ho; ++x)
                for (int64_t y = 0; y < Wo; ++y)
                    for (int64_t d1 = 0; d1 < D1; ++d1) {
                        const int64_t ii = ((((((b * H + x * stride + p) * W + y * stride + q) * C + c) * S + sl)
                                             * D1 + d1) * D2 + d2);
                        const int64_t oo = ((((((b * Ho + x) * Wo + y) * Cout + co) * S + sl) * D1 + d1) * D3 + d3);
                        const double t = I[ii] * dO[oo];
                        acc += t;
                        aabs += fabs(t);
                    }
        dK[e] = acc;
        if (dKabs) dKabs[e] = aabs;
    }
    return OR_OK;
}
