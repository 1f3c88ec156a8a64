/*
 * swin_attn_int8.h — C ABI of the attention half of the quantized Swin block (arXiv 2402.01169,
 * PAPER.md Fig. 1 lines 39-62), B200 (sm_100a).  Same shared
 * library, status codes and error convention as swin_mlp_int8.h (validation before any launch;
 * on error nothing is launched and swin_mlp_int8_last_error() describes the failure).
 *
 *   op #1 (NEXT-4)  Y = Q_x(LayerNorm(x)) in shifted-window order
 *   QKV GEMM        A[t][n] = sum_k (Y[t][k] - z_x) * Wqkv[n][k]
 *   op #2           qkv[t][n] = Q_{q|k|v}(dQ(A) + b_qkv[n])
 *   Q.K GEMM        S = q_h k_h^T per window and head (d = 32)
 *   op #3           Pq = Q_p(softmax(dQ(S) / sqrt(d) + B_h [+ mask]))
 *   V.att GEMM      a[raster(t)][h*32 + n] = Q_a(sum_j Pq[i][j] v_h[j][n])
 *
 * Exact arithmetic (fl = fp32 round-to-nearest-even, rne = round half to even; the readings
 * are DESIGN.md R21-R27):
 *   geometry   windows of M x M tokens in raster order, tokens raster inside a window; the
 *              window-ordered row r reads image pixel ((wy M + iy + s) mod Hs, (wx M + ix + s)
 *              mod Ws) (cyclic shift by -s, s = shift); the attention output goes back to that
 *              pixel's raster row (window reverse + inverse shift)
 *   op #1      mu, var (biased) in fp32 over the row (two passes), rstd = fl(1/fl(sqrt(var+eps)));
 *              yhat = fmaf(fl(fl(x - mu) * rstd), gamma, beta); Y = clamp(rne(fl(yhat * fl(1/s_x))) + z_x)
 *              (the oracle's statistics are in double: Y within 1 LSB on <= 0.01 %)
 *   op #2      y = fmaf(fl(A), fl(s_x * s_w[n]), b[n] or 0); qkv = clamp(rne(fl(y * fl(1/s))), -128, 127),
 *              s = q_scale / k_scale / v_scale for the three C-column thirds (zero point 0)
 *   op #3      l = S * m3 + B[h][i][j] (+ mask), m3 = fl(fl(q_scale * k_scale) * fl(1/sqrt(32)));
 *              B from the (2M-1)^2 x heads table by the relative (row, col) displacement; mask
 *              0 / -100 across the shifted regions (shift > 0 only); p = softmax_j(l);
 *              Pq = clamp(rne(p * 127), 0, 127)   (s_p = 1/127).  The oracle rounds each step in
 *              fp32 and takes the softmax in double; the GPU uses one fma for l, ex2 of the
 *              max-shifted logits and one product e * fl(127 / sum): Pq within 1 LSB on <= 0.01 %
 *   V.att      a = clamp(rne(fl(fl(O) * m_o)) + z_a, -128, 127), O = sum_j Pq v (int32 exact),
 *              m_o = fl(fl(fl(1/127) * v_scale) * fl(1/a_scale))
 * Layout: x fp32 [B][Hs][Ws][C]; window-ordered and raster tensors [B*Hs*Ws][C] (int8);
 * qkv [T][3C] = q | k | v, head h at columns h*32 .. h*32+31 of each third; Wqkv [3C][C].
 */
#ifndef SWIN_ATTN_INT8_H_
#define SWIN_ATTN_INT8_H_

#include <stddef.h>
#include <stdint.h>

#include "swin_mlp_int8.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- fused op #1: LayerNorm -> window shift -> Q ---------------- */
typedef struct swin_op1_int8_s* swin_op1_int8_t;

typedef struct {
    int32_t C;                 /* channels, multiple of 4, 4 <= C <= 1536                       */
    int32_t M;                 /* window side (7, or 12 for Swin at 384), 1 <= M <= 16          */
    int32_t shift;             /* cyclic shift s, 0 <= s < M (Swin: 0 or M/2)                   */
    int32_t Hs, Ws;            /* feature map, multiples of M                                   */
    const float* ln_gamma;     /* [C], host or device, copied                                   */
    const float* ln_beta;      /* [C]                                                           */
    float ln_eps;              /* > 0                                                           */
    float y_scale;             /* output quantizer (the QKV GEMM input), finite normal > 0      */
    int32_t y_zero_point;      /* [-128, 127]                                                   */
    int32_t device;
} swin_op1_int8_desc_t;

swin_mlp_status_t swin_op1_int8_create(const swin_op1_int8_desc_t* desc, swin_op1_int8_t* out);
/*   x  [B][Hs][Ws][C] fp32, device, 16-byte aligned (the block input / residual stream)
 *   y  [B*Hs*Ws][C] int8, device, 4-byte aligned (window order)
 * B >= 0 (0: no launch).  One launch, stream-ordered, asynchronous. */
swin_mlp_status_t swin_op1_int8_run(swin_op1_int8_t h, const float* x, int64_t B, int8_t* y, void* stream);
swin_mlp_status_t swin_op1_int8_destroy(swin_op1_int8_t h);

/* ---- QKV GEMM + op #2 -> Q.K + op #3 -> V.att --------------------- */
typedef struct swin_attn_int8_s* swin_attn_int8_t;

typedef struct {
    int32_t C;                 /* channels, heads * 32, 64 <= C <= 1536 (3C a multiple of 32)   */
    int32_t heads;             /* C / 32 (Swin head dim 32)                                     */
    int32_t M, shift, Hs, Ws;  /* window geometry as op #1 (M = 7 or 12)                        */
    float x_scale;             /* QKV GEMM input quantizer (op #1's output)                     */
    int32_t x_zero_point;
    const int8_t* w_qkv;       /* [3C][C], symmetric (-128 not allowed), host or device, copied */
    const float* w_qkv_scale;  /* [3C] per output channel                                       */
    const float* b_qkv;        /* [3C] or NULL                                                  */
    float q_scale, k_scale, v_scale;  /* op #2 output quantizers (zero point 0)                 */
    const float* rel_bias_table;      /* [(2M-1)^2][heads] fp32                                 */
    float a_scale;             /* V.att output quantizer (the Proj GEMM input)                  */
    int32_t a_zero_point;
    int32_t device;
} swin_attn_int8_desc_t;

swin_mlp_status_t swin_attn_int8_create(const swin_attn_int8_desc_t* desc, swin_attn_int8_t* out);
/* Device workspace bytes for a run of B images: qkv [B*Hs*Ws][3C] int8 (128-byte aligned). */
size_t swin_attn_int8_workspace_bytes(swin_attn_int8_t h, int64_t B);
/*   xw  [B*Hs*Ws][C] int8, device, 16-byte aligned, window order (op #1's output)
 *   a   [B*Hs*Ws][C] int8, device, 16-byte aligned, RASTER order (the Proj GEMM input)
 * Two launches (QKV GEMM + op #2, then the attention core), PDL-chained, asynchronous. */
swin_mlp_status_t swin_attn_int8_run(swin_attn_int8_t h, const int8_t* xw, int64_t B, int8_t* a, void* workspace,
                                     size_t workspace_bytes, void* stream);
/* run + debug taps (device, any may be NULL): qkv [T][3C] int8 (op #2 output), acc [T][3C]
 * int32 (the QKV GEMM accumulators), p [B*nW][heads][N][N] int8 (Pq, N = M*M). */
swin_mlp_status_t swin_attn_int8_run_debug(swin_attn_int8_t h, const int8_t* xw, int64_t B, int8_t* a,
                                           void* workspace, size_t workspace_bytes, void* stream, int8_t* qkv,
                                           int32_t* acc, int8_t* p);
/* Folded constants (host): {m3, inv_p, m_o} and the expanded bias [heads][N][N] (may be NULL). */
swin_mlp_status_t swin_attn_int8_get_constants(swin_attn_int8_t h, float* m3_invp_mo, float* bias);
/* Native per-kernel timing (bench / tools): CUDA events around the QKV GEMM and the attention
 * core of the next max_runs runs on their launching stream; _end synchronizes on the events and
 * returns the summed milliseconds of each kernel.  Host-only; EINVAL on a NULL handle. */
swin_mlp_status_t swin_attn_int8_profile_begin(swin_attn_int8_t h, int32_t max_runs);
swin_mlp_status_t swin_attn_int8_profile_end(swin_attn_int8_t h, float* qkv_ms, float* core_ms, int32_t* runs);
swin_mlp_status_t swin_attn_int8_destroy(swin_attn_int8_t h);

#ifdef __cplusplus
}
#endif
#endif /* SWIN_ATTN_INT8_H_ */
