/*
 * oracle_mlp.c — plain, slow, obviously-correct CPU oracle for the fully
 * integer Swin MLP sub-layer of arXiv 2402.01169 ("GELU-less quantized SWIN").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2402_01169_b200/csrc); it includes nothing but libc/libm.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (done by oracle/build.py, called from __graft_entry__.build()).
 * -ffp-contract=off forbids the compiler from fusing a*b+c into an FMA, so
 * every fp32 operation below rounds exactly once, where it is written, and
 * the only fused multiply-add is the explicit fmaf() of step O2/O4.
 * On x86-64 (SSE, FLT_EVAL_METHOD == 0) float arithmetic is done in float.
 *
 * The method (Fig. 1, lines 72-86; Sec. "GELU-less SWIN", lines
 * 244-247 and 326-328):
 *   FC1 GEMM (int8 x int8 -> int32)
 *   Fused op #5: dQ -> FC1 bias -> act -> Q
 *        act = ReLU ("replace GELU with ReLU") or GELU (control)
 *   FC2 GEMM (int8 x int8 -> int32)
 *   Fused op #6: dQ -> FC2 bias -> Add & LN
 *        plus a trailing Q (reading R4).
 * Step names O0..O6 follow SURVEY.md §8(c); every reading of the paper taken
 * here (rounding, zero points, residual, eps, ...) is listed in DESIGN.md §3.
 *
 * Notation: fl(.) = round to nearest-even fp32; rne(.) = round half to even
 * to an integer.  T tokens (rows), C channels, H hidden (= 4C for Swin).
 * Row-major everywhere; weights in nn.Linear layout [out][in].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EOVERFLOW 1

/* ------------------------------------------------------------------ */
/* Q / dQ primitives ("Q and dQ denote the quantization and
 * de-quantization operations").                          */
/* ------------------------------------------------------------------ */

/* rne(v): round half to even, in double (exact for any float v).        */
static double rne_double(double v) { return nearbyint(v); } /* FE_TONEAREST */

/* Q(v) on an already-scaled fp32 value v = x * (1/s):
 *   q = clamp(rne(v) + z, -128, 127), zero point added after rounding
 *   (reading R5: folding z into the float first is not exact).          */
static int8_t quant_from_scaled(float v, int32_t zp) {
    double r = rne_double((double)v);           /* exact: |v| < 2^128 */
    if (r > 1024.0) r = 1024.0;                 /* keep int conversion safe */
    if (r < -1024.0) r = -1024.0;
    int32_t q = (int32_t)r + zp;
    if (q < -128) q = -128;
    if (q > 127) q = 127;
    return (int8_t)q;
}

/* Exported Q and dQ on arrays, for the oracle's own pin tests (tests/).
 *   Q : q = clamp(rne(fl(x * inv_s)) + z, -128, 127)   (reading R11: multiply
 *       by the folded reciprocal fl(1/s), not divide)
 *   dQ: x = fl(fl(q - z) * s)                                              */
void oracle_q(const float* x, int64_t n, float inv_s, int32_t z, int8_t* q) {
    for (int64_t i = 0; i < n; ++i) q[i] = quant_from_scaled(x[i] * inv_s, z);
}
void oracle_dq(const int8_t* q, int64_t n, float s, int32_t z, float* x) {
    for (int64_t i = 0; i < n; ++i) x[i] = (float)((int32_t)q[i] - z) * s;
}

/* ------------------------------------------------------------------ */
/* O0: constant folding.  fp32 ops, one rounding each. */
/* ------------------------------------------------------------------ */
void oracle_fold_constants(int32_t C, int32_t H, float s_x, const float* s_w1,
                           float s_h, const float* s_w2, float s_y,
                           float* m1 /*[H]*/, float* inv_h /*[1]*/,
                           float* m2 /*[C]*/, float* inv_y /*[1]*/) {
    for (int32_t n = 0; n < H; ++n) m1[n] = s_x * s_w1[n];
    for (int32_t c = 0; c < C; ++c) m2[c] = s_h * s_w2[c];
    *inv_h = 1.0f / s_h;
    *inv_y = 1.0f / s_y;
}

/* ------------------------------------------------------------------ */
/* O1 / O3: integer GEMM with zero-point, int64 accumulation, checked to
 * fit int32 ("8-bit integer for the weights and input
 * activations of the linear layers ... integer tensor cores").
 *   A[t][n] = sum_k (X[t][k] - z) * W[n][k]
 * Rows are independent: rows[] selects which of the T rows to compute
 * (rows == NULL means all rows, out row i = row i).                      */
/* ------------------------------------------------------------------ */
int32_t oracle_gemm_i8(const int8_t* X, int64_t ldx, const int64_t* rows, int64_t nrows,
                       int32_t K, const int8_t* W /*[N][K]*/, int32_t N, int32_t zp,
                       int32_t* A /*[nrows][N]*/, int32_t nthreads) {
    int32_t status = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static) reduction(| : status)
#endif
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t t = rows ? rows[i] : i;
        const int8_t* x = X + t * ldx;
        for (int32_t n = 0; n < N; ++n) {
            const int8_t* w = W + (int64_t)n * K;
            int64_t acc = 0;
            for (int32_t k = 0; k < K; ++k)
                acc += (int64_t)((int32_t)x[k] - zp) * (int64_t)w[k];
            if (acc > INT32_MAX || acc < INT32_MIN) status |= ORACLE_EOVERFLOW;
            A[i * N + n] = (int32_t)acc;
        }
    }
    return status;
}

/* ------------------------------------------------------------------ */
/* O2 / O2': fused op #5 with ReLU in place of GELU
 * (PAPER.md:245, 327-328), or the GELU control.
 *   a = fl(A1)                      int32 -> fp32, RNE (reading R13)
 *   y = fmaf(a, m1[n], b1[n] or 0)  dQ + FC1 bias, one rounding (R12)
 *   ReLU: v = fl(max(y, 0) * inv_h)
 *   GELU: g = fl(0.5*y*(1+erf(y/sqrt(2)))) in double (R8), v = fl(g*inv_h)
 *   Hq = clamp(rne(v) + z_h, -128, 127)                                   */
/* ------------------------------------------------------------------ */
#define ORACLE_ACT_RELU 0
#define ORACLE_ACT_GELU 1

static float gelu_erf_double(float y) {
    double yd = (double)y;
    double g = 0.5 * yd * (1.0 + erf(yd / sqrt(2.0)));
    return (float)g;
}

void oracle_ep5(const int32_t* A1, int64_t nrows, int32_t H, const float* m1,
                const float* b1 /*[H] or NULL*/, float inv_h, int32_t z_h, int32_t act,
                int8_t* Hq /*[nrows][H]*/, float* pre /*[nrows][H] or NULL: y*/) {
    for (int64_t i = 0; i < nrows; ++i) {
        for (int32_t n = 0; n < H; ++n) {
            float a = (float)A1[i * H + n];
            float y = fmaf(a, m1[n], b1 ? b1[n] : 0.0f);
            if (pre) pre[i * H + n] = y;
            float f;
            if (act == ORACLE_ACT_RELU)
                f = y > 0.0f ? y : 0.0f;
            else
                f = gelu_erf_double(y);
            float v = f * inv_h;
            Hq[i * H + n] = quant_from_scaled(v, z_h);
        }
    }
}

/* ------------------------------------------------------------------ */
/* O2'': the I-ViT shift-GELU control of SURVEY.md §8(f) NEXT-4 (the integer GELU the paper
 * contrasts ReLU with: "needs to compute the maximum value of the input tensor",
 * PAPER.md:182-186, 246).  The paper gives no formula; this follows I-ViT's ShiftGELU as read
 * in DESIGN.md reading R28, every step integer except the two quantizer products:
 *   y  = fmaf(fl(A1), m1[n], b1[n] or 0)                     dQ + bias, as op #5
 *   I  = clamp(rne(fl(y * inv_g)), -32767, 32767)            the 16-bit GELU input grid s_g
 *   Im = max_n I[t][n]                                        per token row (the tensor max)
 *   e_x = ShiftExp(I - Im),  e_m = ShiftExp(min(-Im, 0))      2^(1.702 x s_g log2 e), integer
 *   sig = floor(e_x * floor((2^31-1) / min(e_x + e_m, 2^31-1)) / 2^24)   in [0, 128]
 *   G  = I * sig                                              GELU on the grid s_g * 2^-7
 *   Hq = clamp(rne(fl(fl(G) * k_g)) + z_h, -128, 127),  k_g = fl(fl(s_g * inv_h) * 2^-7)
 * ShiftExp(x <= 0), with S = fl(1.702 * s_g), x0 = floor(-1 / S) (double), n = 15:
 *   p = x + floor(x / 2) - floor(x / 16)            (x log2 e, by shifts)
 *   p = max(p, n * x0);  q = floor(p / x0);  r = p - q * x0        (r in (x0, 0])
 *   e = max(floor((r - 2 x0) * 2^(n - q - 1)), 0)                   (2^(r/x0) ~ 1 + r/(2|x0|))  */
/* ------------------------------------------------------------------ */
#define ORACLE_ACT_SHIFT_GELU 2
#define SHIFT_N 15

static int64_t floor_div(int64_t a, int64_t b) {   /* floor(a / b), b != 0 */
    int64_t q = a / b, r = a % b;
    if (r != 0 && ((r < 0) != (b < 0))) --q;
    return q;
}

static int64_t shift_exp(int64_t x, int64_t x0) {
    int64_t p = x + floor_div(x, 2) - floor_div(x, 16);
    if (p < SHIFT_N * x0) p = SHIFT_N * x0;
    const int64_t q = floor_div(p, x0);
    const int64_t r = p - q * x0;
    const int64_t m = r - 2 * x0;                       /* > 0 */
    int64_t e = SHIFT_N - q - 1 >= 0 ? m << (SHIFT_N - q - 1) : floor_div(m, 2);
    return e > 0 ? e : 0;
}

void oracle_ep5_shiftgelu(const int32_t* A1, int64_t nrows, int32_t H, const float* m1,
                          const float* b1 /*[H] or NULL*/, float s_g, float inv_h, int32_t z_h,
                          int8_t* Hq /*[nrows][H]*/, int32_t* I_out /*[nrows][H] or NULL*/) {
    const float inv_g = 1.0f / s_g;
    const float S = 1.702f * s_g;
    const int64_t x0 = (int64_t)floor(-1.0 / (double)S);
    const float k_g = (s_g * inv_h) * 0.0078125f;
    int32_t* I = (int32_t*)malloc(sizeof(int32_t) * (size_t)H);
    for (int64_t i = 0; i < nrows; ++i) {
        int32_t Im = -32768;
        for (int32_t n = 0; n < H; ++n) {
            const float y = fmaf((float)A1[i * H + n], m1[n], b1 ? b1[n] : 0.0f);
            double r = nearbyint((double)(y * inv_g));
            if (r > 32767.0) r = 32767.0;
            if (r < -32767.0) r = -32767.0;
            I[n] = (int32_t)r;
            if (I[n] > Im) Im = I[n];
            if (I_out) I_out[i * H + n] = I[n];
        }
        const int64_t e_m = shift_exp(-Im < 0 ? -(int64_t)Im : 0, x0);
        for (int32_t n = 0; n < H; ++n) {
            const int64_t e_x = shift_exp((int64_t)I[n] - Im, x0);
            int64_t sum = e_x + e_m;
            if (sum > 2147483647LL) sum = 2147483647LL;
            const int64_t factor = sum > 0 ? 2147483647LL / sum : 0;
            const int64_t sig = (e_x * factor) >> 24;
            const int64_t G = (int64_t)I[n] * sig;
            const float v = (float)G * k_g;
            Hq[i * H + n] = quant_from_scaled(v, z_h);
        }
    }
    free(I);
}

/* ------------------------------------------------------------------ */
/* O4-O6: fused op #6: dQ -> FC2 bias -> Add & LayerNorm,
 * then Q (reading R4).
 *   d = fmaf(fl(A2), m2[c], b2[c] or 0)
 *   z = fl(d + R[t][c])                          with an fp32 residual, else
 *   r = fl(fl(X[t][c] - z_x) * s_x)              dQ(X) (the dQ node), then
 *   z = fl(d + r)                                the Add node (Fig. 1, PAPER.md:82-86:
 *                                                dQ -> FC2 Bias -> Add, each its own step;
 *                                                reading R3)
 *   mu  = (sum_c z) / C          double, ascending c
 *   var = (sum_c (z-mu)^2) / C   double, ascending c, biased (R9)
 *   rstd = 1 / sqrt(var + eps)   double
 *   yhat = fl(((z - mu) * rstd) * gamma[c] + beta[c])   double ops, L to R
 *   Y = clamp(rne(fl(yhat * inv_y)) + z_y, -128, 127)                     */
/* ------------------------------------------------------------------ */
void oracle_ep6(const int32_t* A2, int64_t nrows, int32_t C, const float* m2,
                const float* b2 /*[C] or NULL*/,
                const float* R /*[nrows][C] or NULL*/,
                const int8_t* X /*[nrows][C], used when R == NULL*/, float s_x, int32_t z_x,
                const float* gamma, const float* beta, float eps,
                float inv_y, int32_t z_y,
                float* z_out /*[nrows][C] or NULL*/, float* yhat_out /*[nrows][C] or NULL*/,
                int8_t* Y /*[nrows][C]*/) {
    float* z = (float*)malloc(sizeof(float) * (size_t)C);
    for (int64_t i = 0; i < nrows; ++i) {
        for (int32_t c = 0; c < C; ++c) {
            float d = fmaf((float)A2[i * C + c], m2[c], b2 ? b2[c] : 0.0f);
            if (R)
                z[c] = d + R[i * C + c];
            else {
                float r = (float)((int32_t)X[i * C + c] - z_x) * s_x;   /* dQ(X) */
                z[c] = d + r;                                              /* Add  */
            }
            if (z_out) z_out[i * C + c] = z[c];
        }
        double sum = 0.0;
        for (int32_t c = 0; c < C; ++c) sum += (double)z[c];
        double mu = sum / (double)C;
        double ss = 0.0;
        for (int32_t c = 0; c < C; ++c) {
            double dz = (double)z[c] - mu;
            ss += dz * dz;
        }
        double var = ss / (double)C;
        double rstd = 1.0 / sqrt(var + (double)eps);
        for (int32_t c = 0; c < C; ++c) {
            double xh = ((double)z[c] - mu) * rstd;
            double yh = xh * (double)gamma[c] + (double)beta[c];
            float yhat = (float)yh;
            if (yhat_out) yhat_out[i * C + c] = yhat;
            float v = yhat * inv_y;
            Y[i * C + c] = quant_from_scaled(v, z_y);
        }
    }
    free(z);
}

/* ------------------------------------------------------------------ */
/* O7: whole layer = O0 -> O1 -> O2 -> O3 -> O4..O6 on a subset of rows
 * (rows are independent: the MLP is applied token-wise, Fig. 1).
 * Optional taps receive the intermediate tensors of the selected rows.   */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t C, H, act;
    float s_x; int32_t z_x;
    const int8_t* w1; const float* s_w1; const float* b1;
    float s_h; int32_t z_h;
    const int8_t* w2; const float* s_w2; const float* b2;
    const float* gamma; const float* beta; float eps;
    float s_y; int32_t z_y;
    float s_g;   /* shift-GELU input grid (act == 2 only) */
} oracle_layer_t;

int32_t oracle_mlp(const oracle_layer_t* L, const int8_t* X /*[T][C]*/,
                   const float* R /*[T][C] or NULL*/,
                   const int64_t* rows, int64_t nrows, int32_t nthreads,
                   int8_t* Y /*[nrows][C]*/,
                   int32_t* acc1 /*[nrows][H] or NULL*/, int8_t* hidden /*[nrows][H] or NULL*/,
                   int32_t* acc2 /*[nrows][C] or NULL*/, float* yhat /*[nrows][C] or NULL*/,
                   float* z_out /*[nrows][C] or NULL*/) {
    const int32_t C = L->C, H = L->H;
    float* m1 = (float*)malloc(sizeof(float) * (size_t)H);
    float* m2 = (float*)malloc(sizeof(float) * (size_t)C);
    float inv_h, inv_y;
    oracle_fold_constants(C, H, L->s_x, L->s_w1, L->s_h, L->s_w2, L->s_y, m1, &inv_h, m2, &inv_y);
    int32_t status = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : status)
#endif
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t t = rows ? rows[i] : i;
        int32_t* a1 = (int32_t*)malloc(sizeof(int32_t) * (size_t)H);
        int8_t* h = (int8_t*)malloc((size_t)H);
        int32_t* a2 = (int32_t*)malloc(sizeof(int32_t) * (size_t)C);
        status |= oracle_gemm_i8(X + t * C, C, NULL, 1, C, L->w1, H, L->z_x, a1, -1);
        if (L->act == ORACLE_ACT_SHIFT_GELU)
            oracle_ep5_shiftgelu(a1, 1, H, m1, L->b1, L->s_g, inv_h, L->z_h, h, NULL);
        else
            oracle_ep5(a1, 1, H, m1, L->b1, inv_h, L->z_h, L->act, h, NULL);
        status |= oracle_gemm_i8(h, H, NULL, 1, H, L->w2, C, L->z_h, a2, -1);
        oracle_ep6(a2, 1, C, m2, L->b2, R ? R + t * C : NULL, X + t * C, L->s_x, L->z_x,
                   L->gamma, L->beta, L->eps, inv_y, L->z_y,
                   z_out ? z_out + i * C : NULL, yhat ? yhat + i * C : NULL, Y + i * C);
        if (acc1) memcpy(acc1 + i * H, a1, sizeof(int32_t) * (size_t)H);
        if (hidden) memcpy(hidden + i * H, h, (size_t)H);
        if (acc2) memcpy(acc2 + i * C, a2, sizeof(int32_t) * (size_t)C);
        free(a1); free(h); free(a2);
    }
    free(m1); free(m2);
    return status;
}

int32_t oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
