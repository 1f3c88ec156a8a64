/*
 * oracle_attn.c — plain, slow, obviously-correct CPU oracle for the attention half of the
 * quantized Swin block of arXiv 2402.01169 (Fig. 1, lines 39-70):
 *
 *   Fused op #1  Layer-norm -> Window Shifting -> Q          PAPER.md:39-43 (nodes a1-a3)
 *   QKV GEMM (int8 x int8 -> int32)                          PAPER.md:45      (node b)
 *   Fused op #2  dQ -> QKV Bias -> Q                         PAPER.md:47-51   (nodes c1-c3)
 *   Q.K GEMM (per window and head)                           PAPER.md:53      (node d1)
 *   Fused op #3  dQ -> Softmax & Pos. Bias -> Q              PAPER.md:55-58   (nodes d2-d4)
 *   V.att GEMM, int8 output (the Proj GEMM consumes it)      PAPER.md:60, 62  (d5 -> e1)
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_2402_01169_b200/csrc); it includes nothing but libc/libm.
 * Built like oracle_mlp.c: gcc -O2 -ffp-contract=off -fno-fast-math (every fp32 op rounds where
 * it is written; the only fused multiply-add is the explicit fmaf of op #2, reading R12).
 *
 * The paper draws these nodes but does not spell out the window geometry, the shift, the
 * relative position bias, the shifted-window mask or the attention scale; it defers to the Swin
 * paper ("We avoid changing the Softmax fused operation as it also contains the relative
 * position bias").  The readings taken (R21-R27):
 *   - windows of M x M tokens, raster window order, raster token order inside a window;
 *   - Window Shifting = cyclic shift by -s along both image axes (s = 0 or M/2): output pixel
 *     (i, j) of the shifted map is input pixel ((i + s) mod Hs, (j + s) mod Ws);
 *   - LayerNorm statistics in double (as oracle O5), biased variance, eps;
 *   - op #2 quantizes q, k, v with their own scales (s_q, s_k, s_v), zero point 0;
 *   - the attention scale d^-1/2 (d = 32) is folded into op #3's dequant multiplier;
 *   - relative position bias B[h][i][j] = table[idx(i, j)][h], idx from the relative
 *     (row, col) displacement (2M-1)^2 entries; shifted blocks add -100 across regions;
 *   - softmax in double, the quantized probability Pq = Q(p, s_p = 1/127) in [0, 127];
 *   - the V.att GEMM writes int8 (requantized with fl(fl(s_p s_v) / s_a)); its rows go back to
 *     image (raster) order -- window reverse and the inverse shift -- so the Proj GEMM and its
 *     residual add (op #4) see tokens in the residual stream's order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Q on an already-scaled fp32 value: clamp(rne(v) + z, -128, 127) (readings R2, R5). */
static int8_t q_scaled(float v, int32_t zp) {
    double r = nearbyint((double)v);
    if (r > 1024.0) r = 1024.0;
    if (r < -1024.0) r = -1024.0;
    int32_t q = (int32_t)r + zp;
    if (q < -128) q = -128;
    if (q > 127) q = 127;
    return (int8_t)q;
}

/* ------------------------------------------------------------------ */
/* Window geometry (readings R21, R22).                                */
/* Row r of the window-ordered tensor [B * nW * M * M][C]:             */
/*   b = r / (nW M^2), w = (r / M^2) % nW, p = r % M^2,                */
/*   wy = w / (Ws/M), wx = w % (Ws/M), iy = p / M, ix = p % M,         */
/*   source pixel = ((wy M + iy + s) mod Hs, (wx M + ix + s) mod Ws).  */
/* Returns the raster row b * Hs * Ws + y * Ws + x of that pixel.       */
/* ------------------------------------------------------------------ */
int64_t oracle_window_src_row(int64_t r, int32_t Hs, int32_t Ws, int32_t M, int32_t s) {
    const int64_t N = (int64_t)M * M, nWx = Ws / M, nW = (int64_t)(Hs / M) * nWx;
    const int64_t b = r / (nW * N), w = (r / N) % nW, p = r % N;
    const int64_t wy = w / nWx, wx = w % nWx, iy = p / M, ix = p % M;
    const int64_t y = (wy * M + iy + s) % Hs, x = (wx * M + ix + s) % Ws;
    return b * (int64_t)Hs * Ws + y * Ws + x;
}

/* ------------------------------------------------------------------ */
/* Fused op #1: Layer-norm -> Window Shifting -> Q.    */
/* x: fp32 [B][Hs][Ws][C] (the block input, residual stream).            */
/* out row r (window order) = Q(LN(x[src(r)])):                          */
/*   mu = sum_c x / C, var = sum_c (x - mu)^2 / C (double, ascending c)  */
/*   yhat = fl(((x - mu) * rstd) * gamma + beta)  (double ops, L to R)   */
/*   out = clamp(rne(fl(yhat * inv_s)) + z, -128, 127)                   */
/* ------------------------------------------------------------------ */
void oracle_op1(const float* x, int32_t B, int32_t Hs, int32_t Ws, int32_t C, int32_t M, int32_t s,
                const float* gamma, const float* beta, float eps, float inv_s, int32_t z,
                const int64_t* rows, int64_t nrows, int8_t* out /*[nrows][C]*/, float* yhat_out /*or NULL*/) {
    (void)B;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t r = rows ? rows[i] : i;
        const float* xr = x + oracle_window_src_row(r, Hs, Ws, M, s) * C;
        double sum = 0.0;
        for (int32_t c = 0; c < C; ++c) sum += (double)xr[c];
        const double mu = sum / (double)C;
        double ss = 0.0;
        for (int32_t c = 0; c < C; ++c) {
            const double d = (double)xr[c] - mu;
            ss += d * d;
        }
        const double rstd = 1.0 / sqrt(ss / (double)C + (double)eps);
        for (int32_t c = 0; c < C; ++c) {
            const float yh = (float)((((double)xr[c] - mu) * rstd) * (double)gamma[c] + (double)beta[c]);
            if (yhat_out) yhat_out[i * C + c] = yh;
            out[i * C + c] = q_scaled(yh * inv_s, z);
        }
    }
}

/* ------------------------------------------------------------------ */
/* QKV GEMM + fused op #2: dQ -> QKV Bias -> Q.        */
/*   A[t][n] = sum_k (X[t][k] - z_x) W[n][k]        (int64, exact)      */
/*   y = fmaf(fl(A), m[n], b[n]),  m[n] = fl(s_x * s_w[n])  (R12)       */
/*   out = clamp(rne(fl(y * inv[n])), -128, 127), inv[n] = fl(1/s_q),   */
/*   fl(1/s_k) or fl(1/s_v) for n in the q, k, v thirds (zero point 0). */
/* ------------------------------------------------------------------ */
void oracle_qkv(const int8_t* X, int64_t T, int32_t C, int32_t z_x, const int8_t* W /*[3C][C]*/,
                const float* s_w /*[3C]*/, const float* b /*[3C] or NULL*/, float s_x, float s_q, float s_k,
                float s_v, int32_t* acc_out /*[T][3C] or NULL*/, int8_t* out /*[T][3C]*/) {
    const int32_t N = 3 * C;
    const float inv3[3] = {1.0f / s_q, 1.0f / s_k, 1.0f / s_v};
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t t = 0; t < T; ++t) {
        for (int32_t n = 0; n < N; ++n) {
            int64_t a = 0;
            for (int32_t k = 0; k < C; ++k) a += (int64_t)((int32_t)X[t * C + k] - z_x) * (int64_t)W[(int64_t)n * C + k];
            if (acc_out) acc_out[t * N + n] = (int32_t)a;
            const float m = s_x * s_w[n];
            const float y = fmaf((float)a, m, b ? b[n] : 0.0f);
            out[t * N + n] = q_scaled(y * inv3[n / C], 0);
        }
    }
}

/* ------------------------------------------------------------------ */
/* Relative position bias (reading R24): B[h][i][j] = table[idx][h],    */
/* i = (yi, xi), j = (yj, xj) inside an M x M window,                   */
/* idx = (yi - yj + M - 1) * (2M - 1) + (xi - xj + M - 1).              */
/* ------------------------------------------------------------------ */
void oracle_rel_bias(const float* table /*[(2M-1)^2][heads]*/, int32_t M, int32_t heads, float* out /*[heads][N][N]*/) {
    const int32_t N = M * M;
    for (int32_t h = 0; h < heads; ++h)
        for (int32_t i = 0; i < N; ++i)
            for (int32_t j = 0; j < N; ++j) {
                const int32_t dy = i / M - j / M + M - 1, dx = i % M - j % M + M - 1;
                out[((int64_t)h * N + i) * N + j] = table[(dy * (2 * M - 1) + dx) * heads + h];
            }
}

/* Shifted-window mask (reading R25): 0 when both tokens come from the same region of the
 * shifted image, -100 otherwise; regions split each axis at Hs - M and Hs - s.  s = 0: none. */
void oracle_shift_mask(int32_t Hs, int32_t Ws, int32_t M, int32_t s, float* out /*[nW][N][N]*/) {
    const int32_t N = M * M, nWx = Ws / M, nW = (Hs / M) * nWx;
    for (int32_t w = 0; w < nW; ++w) {
        int32_t reg[1024];
        for (int32_t p = 0; p < N; ++p) {
            const int32_t y = (w / nWx) * M + p / M, x = (w % nWx) * M + p % M;
            const int32_t ry = s == 0 ? 0 : (y < Hs - M ? 0 : y < Hs - s ? 1 : 2);
            const int32_t rx = s == 0 ? 0 : (x < Ws - M ? 0 : x < Ws - s ? 1 : 2);
            reg[p] = ry * 3 + rx;
        }
        for (int32_t i = 0; i < N; ++i)
            for (int32_t j = 0; j < N; ++j) out[((int64_t)w * N + i) * N + j] = reg[i] == reg[j] ? 0.0f : -100.0f;
    }
}

/* Folded constants of op #3 and the V.att requant (fp32, one rounding each, R23/R27):
 *   m3 = fl(fl(s_q * s_k) * fl(1 / sqrt(D))),  inv_p = fl(1 / s_p) with s_p = fl(1 / 127),
 *   m_o = fl(fl(s_p * s_v) * fl(1 / s_a)).                                                  */
void oracle_attn_fold(float s_q, float s_k, float s_v, float s_a, int32_t D, float* m3, float* inv_p, float* m_o) {
    const float rs = (float)(1.0 / sqrt((double)D));
    const float sqk = s_q * s_k;
    *m3 = sqk * rs;
    const float s_p = 1.0f / 127.0f;
    *inv_p = 1.0f / s_p;
    const float spv = s_p * s_v;
    const float inv_a = 1.0f / s_a;
    *m_o = spv * inv_a;
}

/* ------------------------------------------------------------------ */
/* Q.K GEMM + fused op #3 + V.att GEMM, one window w and head h:         */
/*   S[i][j] = sum_d q[i][d] k[j][d]                     int64, exact    */
/*   l = fl(fl(fl(S) * m3) + bias[h][i][j])  (+ mask, another rounding)  */
/*       m3 = fl(fl(s_q * s_k) * d^-1/2)     (attention scale, R23)      */
/*   p = exp(l - max_j l) / sum_j exp(l - max_j l)    double, ascending j */
/*   Pq = clamp(rne(fl(fl(p) * inv_p)), -128, 127),  inv_p = 127 (R26)   */
/*   O[i][n] = sum_j Pq[i][j] v[j][n]                 int64, exact        */
/*   out = clamp(rne(fl(fl(O) * m_o)) + z_a, -128, 127),                 */
/*       m_o = fl(fl(s_p * s_v) * fl(1/s_a)), s_p = 1/127          (R27) */
/* qkv: [T][3C] window order (q, k, v thirds; head h at columns h*32..); */
/* out: [T][C] in raster order (row src(r)); p_tap [nWin][heads][N][N].  */
/* ------------------------------------------------------------------ */
void oracle_attn(const int8_t* qkv, int64_t n_win, int32_t C, int32_t heads, int32_t M, int32_t Hs, int32_t Ws,
                 int32_t s, float m3, const float* bias /*[heads][N][N]*/, const float* mask /*[nW][N][N] or NULL*/,
                 float inv_p, float m_o, int32_t z_a, const int64_t* wins, int64_t nwins,
                 int8_t* out /*[n_win*N][C] raster*/, int8_t* p_tap /*[nwins][heads][N][N] or NULL*/) {
    (void)n_win;
    const int32_t N = M * M, D = C / heads, nW = (Hs / M) * (Ws / M);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t wi = 0; wi < nwins; ++wi) {
        const int64_t win = wins ? wins[wi] : wi;
        const int8_t* base = qkv + win * N * (int64_t)(3 * C);
        double* e = (double*)malloc(sizeof(double) * (size_t)N);
        float* l = (float*)malloc(sizeof(float) * (size_t)N);
        int8_t* P = (int8_t*)malloc((size_t)N * N);
        for (int32_t h = 0; h < heads; ++h) {
            for (int32_t i = 0; i < N; ++i) {
                for (int32_t j = 0; j < N; ++j) {
                    int64_t S = 0;
                    for (int32_t d = 0; d < D; ++d)
                        S += (int64_t)base[(int64_t)i * 3 * C + h * D + d] * (int64_t)base[(int64_t)j * 3 * C + C + h * D + d];
                    float v = (float)S * m3;
                    v = v + bias[((int64_t)h * N + i) * N + j];
                    if (mask) v = v + mask[((int64_t)(win % nW) * N + i) * N + j];
                    l[j] = v;
                }
                double mx = (double)l[0];
                for (int32_t j = 1; j < N; ++j) if ((double)l[j] > mx) mx = (double)l[j];
                double sum = 0.0;
                for (int32_t j = 0; j < N; ++j) { e[j] = exp((double)l[j] - mx); sum += e[j]; }
                for (int32_t j = 0; j < N; ++j) {
                    const float p = (float)(e[j] / sum);
                    P[(int64_t)i * N + j] = q_scaled(p * inv_p, 0);
                }
            }
            if (p_tap) memcpy(p_tap + (wi * heads + h) * (int64_t)N * N, P, (size_t)N * N);
            for (int32_t i = 0; i < N; ++i) {
                const int64_t orow = oracle_window_src_row(win * N + i, Hs, Ws, M, s);
                for (int32_t n = 0; n < D; ++n) {
                    int64_t O = 0;
                    for (int32_t j = 0; j < N; ++j)
                        O += (int64_t)P[(int64_t)i * N + j] * (int64_t)base[(int64_t)j * 3 * C + 2 * C + h * D + n];
                    out[orow * C + h * D + n] = q_scaled((float)O * m_o, z_a);
                }
            }
        }
        free(e); free(l); free(P);
    }
}
