/*
 * swin_mlp_int8.h — C ABI of the B200-native (sm_100a) fully-integer Swin
 * MLP sub-layer of arXiv 2402.01169, "GELU-less quantized SWIN".
 *
 * The layer (Fig. 1, lines 72-86; "GELU-less SWIN", lines 244-247,
 * 326-328), for T tokens of C channels, hidden width H (= 4C in Swin):
 *
 *   FC1 GEMM   A1[t][n] = sum_k (X[t][k] - z_x) * W1[n][k]        int32
 *   op #5      Hq[t][n] = Q_h(act(dQ(A1) + b1[n]))                 int8
 *              act = ReLU (the paper's replacement, fused
 *              into the GEMM epilogue) or GELU (control)
 *   FC2 GEMM   A2[t][c] = sum_j (Hq[t][j] - z_h) * W2[c][j]        int32
 *   op #6      z = dQ(A2) + b2[c] + residual;  Y = Q_y(LayerNorm(z))
 *
 * Exact arithmetic (what "bit-exact" in the tests means) — fl() = fp32
 * round-to-nearest-even, rne() = round half to even:
 *   a  = fl(A1);  y = fmaf(a, m1[n], b1[n] or 0),  m1[n] = fl(x_scale*w1_scale[n])
 *   ReLU: v = fl(max(y,0) * inv_h)         GELU: v = fl(gelu_erf(y) * inv_h)
 *   Hq = clamp(rne(v) + h_zero_point, -128, 127),  inv_h = fl(1/h_scale)
 *   d  = fmaf(fl(A2), m2[c], b2[c] or 0),  m2[c] = fl(h_scale*w2_scale[c])
 *   z  = fl(d + residual[t][c])  or, when residual == NULL, the residual dQ(X) then the
 *        Add, each its own rounding (Fig. 1 node order, reading R3):
 *        r = fl(fl(X[t][c] - z_x) * x_scale),  z = fl(d + r);
 *   mu, var (biased), rstd = 1/sqrt(var+eps) in double;
 *   yhat = fl(((z-mu)*rstd)*gamma[c] + beta[c])  (double ops; desc.ln_fp64 = 1 —
 *   with ln_fp64 = 0 the same formula is evaluated in fp32 with one fmaf);
 *   Y  = clamp(rne(fl(yhat * inv_y)) + y_zero_point, -128, 127),  inv_y = fl(1/y_scale)
 * The readings behind these choices (rounding, zero points, residual
 * operand, trailing Q, eps) are listed in DESIGN.md §3.
 *
 * Layout: row-major.  X, Y: [T][C] int8.  W1: [H][C] int8, W2: [C][H] int8
 * (nn.Linear [out][in], i.e. both GEMMs are K-major "TN").  Weights are
 * symmetric (zero point 0), per-output-channel scales.
 *
 * Errors: every entry point returns a swin_mlp_status_t; no exception or
 * abort crosses the ABI.  Validation happens synchronously before any
 * launch; on error nothing is launched, outputs are untouched and
 * swin_mlp_int8_last_error() (thread-local) describes the failure.
 */
#ifndef SWIN_MLP_INT8_H_
#define SWIN_MLP_INT8_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct swin_mlp_int8_s* swin_mlp_int8_t;

typedef enum {
    SWIN_MLP_OK = 0,
    SWIN_MLP_EINVAL = 1,        /* bad argument (message in last_error)                 */
    SWIN_MLP_EUNSUPPORTED = 2,  /* valid but not supported by this build (e.g. C > 1536)   */
    SWIN_MLP_ENOMEM = 3,        /* device allocation failed                                */
    SWIN_MLP_ECUDA = 4          /* a CUDA runtime/driver call failed (message has the code) */
} swin_mlp_status_t;

typedef enum {
    SWIN_MLP_ACT_RELU = 0,      /* the paper's GELU-less block             */
    SWIN_MLP_ACT_GELU_ERF = 1,  /* control: exact erf GELU, 0.5*y*(1+erf(y/sqrt 2))       */
    SWIN_MLP_ACT_SHIFT_GELU = 2 /* control: I-ViT's integer shift-GELU (R28), which needs
                                 * the max of each token's FC1 row before any output: always
                                 * the unfused plan (FC1 -> A1 -> row-max op #5 kernel -> FC2) */
} swin_mlp_act_t;

/* Layer description passed to swin_mlp_int8_create.  All pointers may be
 * host or device memory (detected); they are read during create only —
 * the handle keeps its own device copies. */
typedef struct {
    int32_t C;                  /* channels; C % 32 == 0, 32 <= C <= 1536                  */
    int32_t H;                  /* hidden width; H % 32 == 0, C <= H <= 6144 (Swin: 4*C)   */
    swin_mlp_act_t act;
    float   x_scale;            /* input activation scale s_x > 0 (finite, normal)         */
    int32_t x_zero_point;       /* z_x in [-128, 127]                                      */
    const int8_t* w1;           /* [H][C]                                                  */
    const float*  w1_scale;     /* [H], > 0                                                */
    const float*  b1;           /* [H] or NULL (NULL = the paper's bias-free FC1) */
    float   h_scale;            /* hidden (post-activation) scale s_h > 0                  */
    int32_t h_zero_point;       /* z_h in [-128, 127]                                      */
    const int8_t* w2;           /* [C][H]                                                  */
    const float*  w2_scale;     /* [C], > 0                                                */
    const float*  b2;           /* [C] or NULL                                             */
    const float*  ln_gamma;     /* [C]                                                     */
    const float*  ln_beta;      /* [C]                                                     */
    float   ln_eps;             /* > 0 (1e-5)                                              */
    float   y_scale;            /* output scale s_y > 0                                    */
    int32_t y_zero_point;       /* z_y in [-128, 127]                                      */
    int32_t device;             /* CUDA device ordinal the handle lives on                 */
    int32_t ln_fp64;            /* LayerNorm statistics/normalisation precision:
                                 *   1: fp64 in the oracle's operation order (Y, yhat bit-exact
                                 *      up to the order of the row sums)
                                 *   0: fp32 (faster; Y within 1 LSB on <= 0.01 % of elements) */
    int32_t op5_unfused;        /* 0: op #5 fused into FC1's TMEM drain (this design).
                                 * 1: the paper's FasterTransformer baseline layout (SURVEY.md
                                 *    §8(f) NEXT-1): FC1 writes the int32
                                 *    accumulators A1 [T][H] to global memory, a separate
                                 *    elementwise kernel runs op #5 (dQ -> b1 -> act -> Q) into Hq,
                                 *    then FC2 + op #6.  Same arithmetic, same results; it exists
                                 *    to measure on B200 what fusing / deleting op #5 saves.  Uses
                                 *    the three-kernel plan for every C (the workspace grows by
                                 *    4*T*H bytes for A1). */
    float gelu_in_scale;        /* act == SWIN_MLP_ACT_SHIFT_GELU only: s_g, the 16-bit integer grid
                                 * of the shift-GELU input (I = clamp(rne(fl(y * fl(1/s_g))),
                                 * +-32767)); finite, normal, > 0.  Ignored otherwise.  The
                                 * control's arithmetic (reading R28):
                                 *   Im = max_n I[t][n];  e = ShiftExp(I - Im), e_m = ShiftExp(min(-Im, 0))
                                 *   sig = floor(e * floor((2^31-1) / min(e + e_m, 2^31-1)) / 2^24)
                                 *   Hq = clamp(rne(fl(fl(I * sig) * fl(fl(s_g * inv_h) * 2^-7))) + z_h)
                                 * ShiftExp(x <= 0): S = fl(1.702 s_g), x0 = floor(-1/S) (double),
                                 *   p = max(x + floor(x/2) - floor(x/16), 15 x0), q = floor(p / x0),
                                 *   e = max(floor((p - q x0 - 2 x0) * 2^(14 - q)), 0)
                                 * (integer throughout: Hq bit-exact with the oracle). */
} swin_mlp_int8_desc_t;

/* Create a layer handle: validates the description, folds the fp32
 * constants m1, inv_h, m2, inv_y, computes the int32 zero-point
 * corrections sum_k W1[n][k] and sum_j W2[c][j], uploads everything to
 * handle-owned device memory and encodes the weight TMA descriptors.
 * No device compute beyond copies.  *out is set only on SWIN_MLP_OK. */
swin_mlp_status_t swin_mlp_int8_create(const swin_mlp_int8_desc_t* desc, swin_mlp_int8_t* out);

/* Bytes of caller-provided device workspace `run` needs for T tokens
 * (the int8 hidden tensor Hq, [T][H], 128-byte aligned; with desc.op5_unfused
 * also the int32 A1 [T][H] behind it).  Returns 0 for a NULL handle, T <= 0, or
 * a layer on the one-kernel plan (C <= 256: the hidden tile stays in shared
 * memory; `run` then accepts workspace == NULL). */
size_t swin_mlp_int8_workspace_bytes(swin_mlp_int8_t h, int64_t T);

/* The hot path: Y = layer(X) for T tokens, stream-ordered, asynchronous.
 *   x            [T][C] int8, device, 16-byte aligned
 *   residual     [T][C] fp32, device, 16-byte aligned, or NULL (NULL: r = dQ(X), reading R3)
 *   y            [T][C] int8, device, 16-byte aligned (may not alias x)
 *   residual_out [T][C] fp32, device, or NULL: receives z (pre-LN sum) for pre-norm chaining
 *   T >= 0 (T == 0: no launch, SWIN_MLP_OK)
 *   workspace    >= swin_mlp_int8_workspace_bytes(h, T) bytes, device, 128-byte aligned
 *   stream       cudaStream_t (NULL = legacy default stream)
 * Ownership: all buffers are the caller's; nothing is retained after return.
 * Concurrency: for T <= 64 (the one-launch plan; clusters of up to 8 CTAs) the
 * kernel reduces FC2 into a handle-owned int32 scratch [64][C] and counter, which it leaves
 * zeroed on exit; two runs of ONE handle must therefore be ordered (same stream, or an event
 * between streams).  Distinct handles never share scratch, and runs with T > 64 use only the
 * caller's workspace. */
swin_mlp_status_t swin_mlp_int8_run(swin_mlp_int8_t h, const int8_t* x, const float* residual,
                                    int8_t* y, float* residual_out, int64_t T,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* Same as run, plus debug taps (any may be NULL), all device memory:
 *   acc1 [T][H] int32 (FC1 accumulators incl. zero-point term), hidden [T][H] int8 (Hq),
 *   acc2 [T][C] int32, ln_out [T][C] fp32 (yhat, the pre-quant LayerNorm output).
 * Runs the same kernels as `run` with their tap-writing variants. */
swin_mlp_status_t swin_mlp_int8_run_debug(swin_mlp_int8_t h, const int8_t* x, const float* residual,
                                          int8_t* y, float* residual_out, int64_t T,
                                          void* workspace, size_t workspace_bytes, void* stream,
                                          int32_t* acc1, int8_t* hidden, int32_t* acc2, float* ln_out);

/* End-to-end convenience: x, residual (or NULL) and y are HOST buffers
 * (pinned for full bandwidth); device staging is taken from `workspace`,
 * which must hold swin_mlp_int8_host_workspace_bytes(h, T, residual != NULL).
 * Pipelined over up to 8 token chunks: the copy-in of a chunk and the copy-out
 * of the previous one (on two handle-owned streams) overlap the kernels of the
 * current one (on `stream`).  Ordered after earlier work on `stream`; returns
 * after enqueueing, and `stream` completes only when y_host is written
 * (synchronize it before reading y).  Not re-entrant per handle: one run_host
 * at a time for a given handle. */
size_t swin_mlp_int8_host_workspace_bytes(swin_mlp_int8_t h, int64_t T, int32_t with_residual);
swin_mlp_status_t swin_mlp_int8_run_host(swin_mlp_int8_t h, const int8_t* x_host, const float* residual_host,
                                         int8_t* y_host, int64_t T, void* workspace, size_t workspace_bytes,
                                         void* stream);

/* End-to-end batch over several independent layers (e.g. the four stage MLPs of a
 * network step, or several batches through one layer): host inputs x_hosts[l]
 * ([Ts[l]][C_l] int8, pinned) -> host outputs y_hosts[l]; residual = dQ(x) (NULL
 * residual) for every layer.  One copy-in / kernels / copy-out pipeline over the
 * token chunks of all layers, so the transfers of one layer overlap the kernels and
 * transfers of its neighbours.  All handles must live on one device; their copy
 * streams and events are taken from hs[0] (one batch at a time per hs[0]).
 * `workspace` (device) must hold swin_mlp_int8_host_batch_workspace_bytes(n, hs, Ts).
 * Ordered after earlier work on `stream`; `stream` completes when every y_hosts[l]
 * is written. */
size_t swin_mlp_int8_host_batch_workspace_bytes(int32_t n, const swin_mlp_int8_t* hs, const int64_t* Ts);
swin_mlp_status_t swin_mlp_int8_run_host_batch(int32_t n, const swin_mlp_int8_t* hs, const int8_t* const* x_hosts,
                                               int8_t* const* y_hosts, const int64_t* Ts, void* workspace,
                                               size_t workspace_bytes, void* stream);

/* Debug getter: the folded fp32 constants exactly as the kernels use them
 * (host arrays m1[H], m2[C]; scalars inv_h, inv_y), and the int32
 * zero-point corrections wsum1[H], wsum2[C].  Any pointer may be NULL. */
swin_mlp_status_t swin_mlp_int8_get_constants(swin_mlp_int8_t h, float* m1, float* inv_h, float* m2,
                                              float* inv_y, int32_t* wsum1, int32_t* wsum2);

/* Number of kernel launches one `run` enqueues (for the bench's launch count). */
int32_t swin_mlp_int8_launches_per_run(swin_mlp_int8_t h);

/* Native per-kernel timing for the bench's roofline: after profile_begin,
 * every run/run_debug records CUDA events before FC1, between FC1 and FC2
 * and after FC2 on its stream (at most max_runs runs are recorded; later
 * runs are not).  profile_end synchronizes those events, returns the summed
 * FC1+ep5 and FC2+ep6 kernel durations in ms and the number of recorded runs,
 * and stops recording (desc.op5_unfused: the first interval holds FC1 and the
 * separate op #5 kernel).  Any output pointer may be NULL. */
swin_mlp_status_t swin_mlp_int8_profile_begin(swin_mlp_int8_t h, int32_t max_runs);
swin_mlp_status_t swin_mlp_int8_profile_end(swin_mlp_int8_t h, float* fc1_ms, float* fc2_ms, int32_t* runs);

/* Pipeline tracing (debug): while set, every run makes CTA `cta` of each
 * kernel record %globaltimer stamps (ns) into the device buffer `trace`
 * (8192 uint64: FC1 at [0, 4096), FC2 at [4096, 8192); within a kernel
 * trace[role*1024 + 2*i + {0,1}] for its i-th tile, roles 0 TMA producer
 * (first stage acquired, last k-block issued), 1 MMA (accumulator acquired,
 * tile committed), 2 epilogue (accumulator ready, tile stored), 3 constant
 * loader (buffer acquired, constants published)).  The trace buffer must then hold 9216
 * uint64: every CTA also stamps its entry / exit at [8192 + 2*cta + {0,1}] (FC1 or
 * the one-kernel plan) and [8704 + 2*cta + {0,1}] (FC2).  trace = NULL disables. */
swin_mlp_status_t swin_mlp_int8_set_trace(swin_mlp_int8_t h, void* trace, int32_t cta);

/* Introspection: the launch plan of this layer, out10[20] = {FC1 BN, FC1 cluster size,
 * FC1 stages, FC1 max co-resident clusters, FC2 BN, FC2 cluster size, FC2 stages,
 * FC2 max clusters, FC1 epilogue groups, FC2 epilogue groups, FC1 resident weights (1: all,
 * 2: each cluster's own column slice),
 * FC2 resident weights, one-kernel plan used (C <= 256, H % 128 == 0; 1/0), its weight
 * ring depth (0 = weights resident in smem), its hidden-tile buffers, its FC1 TMEM
 * buffers, FC1 CTA pair (cta_group::2 MMA, M = 256; 1/0), 0, 0, 0}.  Entries 0-11 and 16
 * describe the two-kernel plan, which runs when entry 12 is 0.
 * Returns 0, or -1 on a NULL argument. */
int32_t swin_mlp_int8_plan(swin_mlp_int8_t h, int32_t* out10);

/* Introspection: the plans a run of T tokens actually launches (the two-kernel path
 * chooses per run: the few-tile plans for one or two m-tiles, the CTA-pair op #6 for at
 * most one wave of pairs, else the defaults).  Same 20-entry layout as
 * swin_mlp_int8_plan with entries 0-11 and 16 describing the chosen plans, and entry 19 =
 * op5_unfused | (choice << 1), choice 0 = default, 1 = CTA-pair op #6, 2 = few-tile,
 * 3 = one launch for T <= 64 (entries 0 = CTAs, 4 = FC2 columns per CTA, 5 = cluster size), and
 * entry 13 = the op #6 split-K factor S of this run (1 = none; S > 1 splits FC2's K = H
 * over S clusters per m-tile when the unsplit grid would fill at most half the SMs).
 * The plan hint (swin_mlp_int8_set_plan_hint), when set, replaces T.  For a one-kernel
 * handle (entry 12 = 1) the result equals swin_mlp_int8_plan: one launch serves every T.
 * Host-only, no launch.  Returns 0, or -1 on a NULL argument or T < 0. */
int32_t swin_mlp_int8_plan_for(swin_mlp_int8_t h, int64_t T, int32_t* out20);

/* Plan hint (batch invariance, reading R20).  The two-kernel path chooses its
 * launch plans per run from T (few-tile plans for one or two m-tiles, the CTA-pair op #6
 * for one wave of pairs, else the defaults), and with fp32 LayerNorm statistics
 * (ln_fp64 = 0) Y can differ by 1 LSB between plans because the row statistics are summed
 * in a different order (within the R15 tier).  With T_hint > 0 every later run/run_debug
 * on this handle chooses its plans as a run of T_hint tokens would, so the shards of a
 * batch of T_hint tokens (multi-GPU token sharding, chunked serving) reproduce the
 * unsharded run bit for bit.  T_hint = 0 restores the per-run choice.  run_host and
 * run_host_batch always plan every chunk for the whole call's T (or the hint when set).
 * Host-only.  Returns OK, or EINVAL on a NULL handle or T_hint < 0. */
swin_mlp_status_t swin_mlp_int8_set_plan_hint(swin_mlp_int8_t h, int64_t T_hint);

/* Release the handle's device memory.  No run may be in flight. NULL is OK. */
swin_mlp_status_t swin_mlp_int8_destroy(swin_mlp_int8_t h);

/* ------------------------------------------------------------------------------------
 * the attention projection GEMM + fused op #4 (Fig. 1,
 * lines 63-70: Proj GEMM -> dQ -> Proj Bias -> Add (Residual) -> Q), the step that
 * produces the MLP sub-layer's input.  For T tokens of C channels:
 *
 *   Proj GEMM  A[t][c] = sum_k (Xa[t][k] - z_a) * W[c][k]          int32 (exact)
 *   op #4      d = fmaf(fl(A), m[c], b[c] or 0),  m[c] = fl(a_scale * w_scale[c])
 *              z = fl(d + residual[t][c])             (residual: the block's fp32 shortcut)
 *              yhat = LayerNorm2(z) (as op #6: fp64 or fp32 statistics, biased variance)
 *              Y = clamp(rne(fl(yhat * inv_y)) + y_zero_point, -128, 127)
 *
 * Reading (R18): Fig. 1 draws op #4 as dQ/bias/add/Q with no LayerNorm, but the
 * Swin block is pre-norm: FC1 consumes LN2(x + proj), so LN2 is fused into op #4's
 * epilogue here -- Y is the int8 MLP input, residual_out = z is the fp32 residual stream the
 * MLP sub-layer adds back (its `residual` argument).  The arithmetic is op #6's with K = C.
 *
 * Errors, ownership, layout and alignment follow swin_mlp_int8_* (Xa, Y [T][C] int8 row-major;
 * W [C][C] int8 nn.Linear [out][in], symmetric, per-output-channel scales).  `residual` is
 * required (op #4 always adds the shortcut).  No workspace. */
typedef struct swin_proj_int8_s* swin_proj_int8_t;

typedef struct {
    int32_t C;                  /* channels; C % 32 == 0, 32 <= C <= 1536                  */
    float   a_scale;            /* attention-output (Proj GEMM input) scale > 0           */
    int32_t a_zero_point;       /* in [-128, 127]                                          */
    const int8_t* w;            /* [C][C] proj weights                                     */
    const float*  w_scale;      /* [C], > 0                                                */
    const float*  b;            /* [C] proj bias or NULL                                   */
    const float*  ln_gamma;     /* [C] LN2                                                 */
    const float*  ln_beta;      /* [C]                                                     */
    float   ln_eps;             /* > 0                                                     */
    float   y_scale;            /* output (MLP input) scale > 0                            */
    int32_t y_zero_point;       /* in [-128, 127]                                          */
    int32_t device;
    int32_t ln_fp64;            /* as swin_mlp_int8_desc_t.ln_fp64                         */
} swin_proj_int8_desc_t;

swin_mlp_status_t swin_proj_int8_create(const swin_proj_int8_desc_t* desc, swin_proj_int8_t* out);
/*   a            [T][C] int8, device, 16-byte aligned (the V*att output, quantized)
 *   residual     [T][C] fp32, device, 16-byte aligned, required
 *   y            [T][C] int8, device, 16-byte aligned
 *   residual_out [T][C] fp32, device, or NULL: receives z
 * T >= 0 (0: no launch).  One kernel launch, stream-ordered, asynchronous. */
swin_mlp_status_t swin_proj_int8_run(swin_proj_int8_t h, const int8_t* a, const float* residual, int8_t* y,
                                     float* residual_out, int64_t T, void* stream);
/* run + debug taps (device, any may be NULL): acc [T][C] int32 (A), ln_out [T][C] fp32 (yhat). */
swin_mlp_status_t swin_proj_int8_run_debug(swin_proj_int8_t h, const int8_t* a, const float* residual, int8_t* y,
                                           float* residual_out, int64_t T, void* stream, int32_t* acc,
                                           float* ln_out);
/* Launch plan: out4 = {BN, cluster size, ring stages, CTA pair}.  Returns 0, or -1 on NULL. */
int32_t swin_proj_int8_plan(swin_proj_int8_t h, int32_t* out4);
swin_mlp_status_t swin_proj_int8_destroy(swin_proj_int8_t h);

/* Thread-local description of the last error on this thread ("" if none). */
const char* swin_mlp_int8_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SWIN_MLP_INT8_H_ */
