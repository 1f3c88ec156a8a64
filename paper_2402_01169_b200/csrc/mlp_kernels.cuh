// mlp_kernels.cuh — the sm_100a kernels of the INT8 Swin MLP sub-layer.
//
// One warp-specialised, persistent tcgen05 GEMM skeleton serves both GEMMs of
// the layer; the epilogue (the paper's fused ops, run inside the TMEM->register
// drain) is the template parameter:
//
//   EP5_RELU  FC1 + fused op #5 with ReLU (PAPER.md:74-78 with GELU replaced by
//             ReLU; "fused, as an integer operation, to the previous
//             GEMM")
//   EP5_GELU  FC1 + fused op #5 with exact-erf GELU (the control the paper removes)
//   EP6_LN    FC2 + fused op #6: dQ, FC2 bias, residual add, LayerNorm, Q
//             (trailing Q per DESIGN.md reading R4)
//   EP2_QKV   QKV GEMM + fused op #2: dQ, QKV bias, Q with a per-column output scale (the q, k and
//             v thirds each on their own quantizer)
//   EP_ACC    FC1 alone, the int32 accumulators A1 (zero-point term included) written
//             to global memory: the FasterTransformer layout the paper starts from,
//             where op #5 is a separate kernel (SURVEY.md
//             §8(f) NEXT-1).  Used only by the desc.op5_unfused comparison plan.
//
// CTA = 640 threads, 1 per SM, persistent over 128-row tiles (a tile = 128 token
// rows x BN columns of one GEMM):
//   warp 0      TMA producer: A (activations) and B (weights) K-blocks of 128 B
//               into a `stages`-deep smem ring (128-B swizzle); A is multicast
//               across the CS CTAs of a cluster, which share one m-tile.
//   warp 1      MMA issuer: tcgen05.mma.kind::i8 (M=128, N=BN, K=32), int32
//               accumulators in TMEM, G accumulator buffers (tile it -> it % G).
//   warp 2      TMEM allocator, then the output store warp: writes each staged
//               int8 tile with TMA tensor stores ([128 rows][W bytes] boxes).
//   warp 3      loader: per tile, the per-column constants (dequant multiplier,
//               bias, zero-point correction, LN gamma/beta) into smem and, for
//               op #6, the residual x tile (TMA).
//   warps 4-19  epilogue, G ping-pong groups of 16/G warps; group g takes the
//               tiles with it % G == g.  Inside a group, warp w drains TMEM lane
//               quadrant (w % 4) (thread = token row) over one of P = 4/G column
//               parts.  16 columns per tcgen05.ld.  Output chunks go to a
//               per-group smem staging tile (16-B granules, swizzled like the
//               TMA box) that warp 2 stores.
//
// Op #6 row statistics: partial row sums of the P column parts combine through
// smem (named barrier of the group), the CS CTAs of a cluster (which split the C
// columns of the same rows) exchange partial sums through DSMEM with st.async +
// mbarrier complete_tx, always summed in the same (part, rank) order so every CTA
// derives identical mean and rstd.  z is parked in TMEM between the three passes
// (sum, centred sum of squares, normalise).
//
// Template flags F (so the hot loop carries no predicated-off work):
//   kHasB   bias present          kHasZc  A-operand zero point != 0 (int32 correction)
//   kZqNz   output zero point != 0 kS64   LayerNorm statistics/normalisation in fp64
//   kSmallK |acc| < 2^22 guaranteed (host-checked: (128+|z_A|)*127*K < 2^22): int32 ->
//           fp32 by the exact magic-number add instead of the half-rate I2FP.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <type_traits>

#include "sm100_ptx.cuh"

namespace swinmlp {

enum Epi : int { EP5_RELU = 0, EP5_GELU = 1, EP6_LN = 2, EP_ACC = 3, EP2_QKV = 4 };

constexpr int kBM = 128;             // rows per tile (UMMA M, TMEM lanes)
constexpr int kBK = 128;             // K bytes per pipeline stage (one 128-B swizzle row)
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
constexpr int kChunk = 16;           // columns per tcgen05.ld (32x32b.x16)
constexpr int kGMax = 4;             // max ping-pong groups / accumulator buffers
constexpr int kNConst = 5;           // m, b, zc, gamma, beta
constexpr int kHasB = 1, kHasZc = 2, kZqNz = 4, kS64 = 8, kSmallK = 16, kPair = 32;

__host__ __device__ constexpr int kernel_threads(int) { return kThreads; }

struct GemmArgs {
    int64_t M;             // token rows
    int32_t K;             // reduction length (bytes of int8)
    int32_t BN;            // columns per CTA tile (UMMA N)
    int32_t CS;            // CTAs per cluster (share one m-tile, A multicast)
    int32_t stages;        // smem ring depth
    int32_t G;             // ping-pong groups = accumulator buffers = staging tiles (2 or 4)
    int32_t xstage;        // op #6: residual x tile buffers in smem, loaded by TMA (G: one per
                           // group, 1: one shared by the groups, 0: pass 1 reads x from global)
    int32_t resb;          // B (weights) resident in smem for the whole kernel (requires mt_major)
    int32_t mt_major;      // tile order: the cluster's m-tiles with the n-groups innermost
    int32_t out_w;         // output TMA box width in bytes (128/64/32/16; swizzle of the same width)
    int32_t n_groups;      // column groups of CS*BN columns
    int64_t num_units;     // m_tiles * n_groups
    int32_t ldo;           // columns of the output (= N total)
    const float* m;        // [N] per-column dequant multiplier (m1 or m2)
    const float* b;        // [N] bias or nullptr
    const int32_t* zc;     // [N] zero-point correction z*sum_k W[n][k], or nullptr
    float inv_q;           // 1/s of the output quantizer (inv_h or inv_y)
    int32_t zq;            // output zero point (z_h or z_y)
    // EP6 only
    const int8_t* x;       // [M][ldo] layer input (op #6 residual when xstage == 0)
    float s_x;
    int32_t z_x;
    const float* resid;    // [M][ldo] fp32 residual or nullptr (nullptr: r = dQ(x), x via tmX)
    float* resid_out;      // [M][ldo] fp32 z or nullptr
    const float* gamma;    // EP6: LN gamma; EP2_QKV: [N] per-column output quantizer reciprocal
    const float* beta;
    float eps;
    float one;             // 1.0f (host-set): z = fma(dQ(x), one, d) keeps ptxas from fusing the
                           // dQ product into the Add (it contracts mul.rn.f32x2 + add.rn.f32x2)
    // debug taps
    int32_t* acc_tap;      // [M][ldo] int32 accumulators (incl. zero-point term)
    float* ln_tap;         // [M][ldo] fp32 yhat (EP6)
    // pipeline trace (debug): when non-null, CTA `trace_cta` records %globaltimer
    // stamps (see swin_mlp_int8_set_trace in the header for the layout)
    unsigned long long* trace;
    int32_t trace_cta;
    unsigned long long* cta_stamps;   // debug: per CTA %globaltimer at entry / exit ([2 * blockIdx.x + {0,1}])
    int32_t eg;                       // op #5 epilogue groups (1: all 16 warps drain every tile; or G)
    int32_t* acc_out;                 // EP_ACC: [M][ldo] int32 A1 (the unfused plan's GEMM output)
    int32_t yin;                      // op #6 with xstage == G: Y staged over its own x tile (no
                                      // separate output staging; the x buffer is released to the
                                      // loader by the store warp once the stores have read Y)
    int32_t dst;                      // op #5: Hq stored straight from registers to `out` (16-B
                                      // st.global per chunk; no staging tiles, no store warp work)
    int8_t* out;                      // [M][ldo] int8 output for dst
    int32_t wsl;                      // weight-stationary slice (op #5): each cluster owns ONE
                                      // column group, keeps that B slice resident in smem (its half
                                      // for a pair) and streams only A tiles through the ring
    // op #6 split-K (runs of few m-tiles): the units are (m-tile, split) pairs, one per cluster;
    // split s accumulates k-blocks [s kb_per, (s+1) kb_per).  Splits 1..S-1 add their int32
    // partial tiles into kacc with bulk reduce-add and count in; split 0 (the reducer) waits for
    // the S-1 arrivals, adds kacc to its own accumulator and runs op #6.  Integer sums are exact
    // in any order, so A2 -- and Y -- are bit-identical to the unsplit plan.
    int32_t ksplit;                   // S (<= 1: no split)
    int32_t kb_per;                   // k-blocks per split
    int32_t* kacc;                    // [M][ldo] int32 (zeroed by the preceding FC1 launch)
    int32_t* kcnt;                    // [m_tiles][CS] arrival counters (zeroed with kacc)
    // FC1: words of `zero_ptr` to clear (after griddepcontrol.wait) for the next launch's split-K
    int32_t* zero_ptr;
    int64_t zero_words;               // multiple of 4, zero_ptr 16-byte aligned
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct SmemLayout {
    uint32_t a, b, bres, out, xres, consts, bars, tmem_slot, red, xbuf, total;
};
__host__ __device__ constexpr uint32_t kNumBars(int stages) { return 2u * stages + 7u * kGMax + 2u * kGMax + 1u + kGMax + 1u; }
// split-K: row stride (bytes) of an int32 partial tile staged in the operand ring (16 B of padding
// per row: consecutive rows start in different 16-B bank groups)
__host__ __device__ constexpr uint32_t ksplit_row_bytes(int BN) { return (uint32_t)BN * 4u + 16u; }

// ebytes: size of one exchanged row statistic (4: fp32 LN, 8: fp64 LN);
// xstage: op #6 stages the residual x tiles in smem (else pass 1 reads x from global)
// resb_bytes: resident-B region (0 when B streams through the ring with A)
// bn_b: B rows per ring stage (BN; BN / 2 for a CTA pair, each CTA holds half of B)
// eg: epilogue groups (G ping-pong groups, or 1: all 16 warps per tile), 4/eg column parts
__host__ __device__ inline SmemLayout smem_layout(int epi, int BN, int CS, int stages, int G, int ebytes = 4,
                                                  int xstage = 1, uint32_t resb_bytes = 0, int bn_b = 0,
                                                  int eg = 0, int yin = 0, int csh = 0, int dst = 0) {
    SmemLayout L;
    const uint32_t tile = (uint32_t)BN * kBM;
    L.a = 0;
    L.b = L.a + (uint32_t)stages * kBM * kBK;
    L.bres = L.b + (resb_bytes ? 0u : (uint32_t)stages * (uint32_t)(bn_b ? bn_b : BN) * kBK);
    L.out = L.bres + resb_bytes;                                   // [G] output staging tiles
    L.xres = L.out + (epi == EP_ACC || yin || dst ? 0u : (uint32_t)G * tile);   // yin: out aliases xres   // (EP_ACC stores from registers)                           // op #6: [G] residual x tiles
    L.consts = L.xres + (epi == EP6_LN ? (uint32_t)xstage * tile : 0u);       // [G][kNConst][BN] fp32
    // csh: every tile of the CTA has the same columns (op #6, one column group) -> one
    // constant buffer shared by the accumulator buffers
    L.bars = L.consts + (csh ? 1u : (uint32_t)G) * kNConst * (uint32_t)BN * 4u;
    L.tmem_slot = L.bars + 8u * kNumBars(stages);
    const uint32_t eb = (uint32_t)ebytes;
    const uint32_t parts = 4u / (uint32_t)(eg ? eg : G);
    const uint32_t npass = eb == 8u ? 2u : 1u;  // fp64 statistics: two exchange passes; fp32: one
    L.red = (L.tmem_slot + 8 + 15) & ~15u;      // op #6: [G][pass][part][val][row] (parts > 1 only)
    L.xbuf = L.red + (epi == EP6_LN && parts > 1 ? (uint32_t)G * npass * parts * 2u * kBM * eb : 0u);
    L.total = L.xbuf + (epi == EP6_LN && CS > 1 ? (uint32_t)G * npass * (uint32_t)CS * 2u * kBM * eb : 0u);
    return L;
}

__host__ __device__ inline uint32_t tmem_cols_for(int BN, int G) {
    uint32_t need = (uint32_t)G * (uint32_t)BN, c = 32;
    while (c < need) c <<= 1;
    return c;
}

// Exact-erf GELU in fp32 (the control's activation; reading R8).
__device__ __forceinline__ float gelu_erf_f32(float y) {
    const float t = erff(__fmul_rn(y, 0.70710678118654752440f));
    return __fmul_rn(__fmul_rn(0.5f, y), __fadd_rn(1.0f, t));
}

// Q of 16 scaled values v (already multiplied by 1/s): clamp(rne(v) + zq, -128, 127),
// packed little-endian into 4 words.  zq == 0: F2IP (rne + saturate + pack 2 per
// instruction; with RELU the max(.,0) folds in as well).  zq != 0: rne saturated to
// int16, + zq, saturating pack (the zero point is added after rounding, reading R5).
template <bool RELU, bool ZQNZ>
__device__ __forceinline__ void quant_pack16(const float (&v)[16], int32_t zq, uint32_t (&w)[4]) {
    using namespace sm100;
    if constexpr (!ZQNZ) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int32_t q[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) q[j] = __float2int_rn(RELU ? fmaxf(v[4 * k + j], 0.0f) : v[4 * k + j]);
            w[k] = pack_sat_s8(q[1], q[0], pack_sat_s8(q[3], q[2], 0u));
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int32_t q[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                q[j] = f2i_rn_sat16(v[4 * k + j]) + zq;
                if (RELU) q[j] = max(q[j], zq);
            }
            w[k] = pack_sat_s8(q[1], q[0], pack_sat_s8(q[3], q[2], 0u));
        }
    }
}

// fl(int) of two accumulators.  SMALLK: |a| < 2^22, so the bits 0x4B400000 + a
// are the float 1.5*2^23 + a and subtracting 1.5*2^23 is exact (an FMA-pipe op
// instead of the half-rate I2FP conversion).
template <bool SMALLK>
__device__ __forceinline__ float2 i2f_pair(uint32_t a, uint32_t b) {
    using namespace sm100;
    if constexpr (SMALLK) {
        const float2 t = make_float2(__uint_as_float(a + 0x4B400000u), __uint_as_float(b + 0x4B400000u));
        return f2_sub(t, make_float2(12582912.0f, 12582912.0f));
    } else {
        return make_float2(__int2float_rn((int32_t)a), __int2float_rn((int32_t)b));
    }
}

template <int EPI, int F>
__global__ void __launch_bounds__(kThreads, 1)
mlp_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ GemmArgs p) {
    using namespace sm100;
    constexpr bool HAS_B = (F & kHasB) != 0, HAS_ZC = (F & kHasZc) != 0, ZQNZ = (F & kZqNz) != 0;
    constexpr bool STATS64 = (F & kS64) != 0, SMALLK = (F & kSmallK) != 0;
    constexpr bool IS_LN = (EPI == EP6_LN);
#ifndef SWIN_LN_PREFETCH
#define SWIN_LN_PREFETCH 0
#endif
    constexpr bool LN_PREFETCH = SWIN_LN_PREFETCH != 0;   // op #6 chunk loop keeps the next tcgen05.ld in flight
    // CTA pair (cta_group::2, M = 256 per MMA): the two CTAs of a cluster take m-tiles
    // 2u and 2u+1 of the same n-group; each loads its A rows and half of the B rows,
    // the leader issues the MMAs (op #5 only: no cross-CTA row statistics)
    constexpr bool PAIR = (F & kPair) != 0;
    // (op #6 in a pair: CS == 1, the whole row in each CTA's TMEM -- BN = C <= 512 as two
    // N = BN/2 MMAs when BN > 256 -- so the LayerNorm statistics never leave the CTA)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    if (p.cta_stamps && threadIdx.x == 0) p.cta_stamps[2 * blockIdx.x] = gtimer();

    const int BN = p.BN;
    const uint32_t CS = (uint32_t)p.CS;
    const int stages = p.stages;
    const uint32_t G = (uint32_t)p.G;
    const uint32_t lgG = G == 4 ? 2u : G == 2 ? 1u : 0u;   // (G = 1: the pair op #6 plan)
    // epilogue groups: op #6 G ping-pong groups (one per accumulator buffer); op #5 may
    // use one group of all 16 warps per tile (shorter per-tile drain, so the MMA of tile
    // t + G waits less for the drain of tile t)
    const uint32_t EG = (uint32_t)p.eg;
    const uint32_t lgEG = EG == 4u ? 2u : EG == 2u ? 1u : 0u;
    const uint32_t tile_warps = kEpiWarps / EG;
    using acc_t = typename std::conditional<STATS64, double, float>::type;   // LN statistics type
    const int bn_b = PAIR ? BN / 2 : BN;                 // B rows per ring stage in this CTA
    const bool wsl = !IS_LN && p.wsl != 0;               // weight-stationary slice (see GemmArgs)
    const uint32_t resb_bytes = p.resb ? (uint32_t)p.n_groups * (uint32_t)((p.K + kBK - 1) / kBK) * (uint32_t)BN * kBK
                              : wsl ? (uint32_t)((p.K + kBK - 1) / kBK) * (uint32_t)bn_b * kBK : 0u;
    // pair with BN > 256: two MMAs of N = BN/2 per K step; each CTA holds, per MMA half h,
    // B rows [h BN/2 + rank BN/4, + BN/4) as [h][BN/4 rows][128 B]
    const uint32_t nh2 = (PAIR && BN > 256) ? 2u : 1u;
    const uint32_t nmma = (uint32_t)BN / nh2;            // UMMA N
    const uint32_t hrows = PAIR ? nmma / 2u : nmma;      // B rows per MMA half in this CTA
    const bool csh = IS_LN && p.n_groups == 1;           // one shared constant buffer (see smem_layout)
    constexpr uint32_t NPASS = STATS64 ? 2u : 1u;         // row-statistics exchange passes
    const SmemLayout L = smem_layout(EPI, BN, p.CS, stages, p.G, (int)sizeof(acc_t), p.xstage, resb_bytes, bn_b, p.eg,
                                     IS_LN ? p.yin : 0, csh ? 1 : 0, p.dst);
    const bool dst = !IS_LN && EPI != EP_ACC && p.dst != 0;   // op #5 direct global stores
    const bool yin = IS_LN && p.yin != 0;                 // Y staged over its x tile (xstage == G)
    const uint32_t tile_bytes = (uint32_t)BN * kBM;
    const uint32_t sA = base + L.a, sB = base + L.b;
    const uint32_t bar_full = base + L.bars;              // [stages] operands landed (count 1 + tx)
    const uint32_t bar_empty = bar_full + 8u * stages;    // [stages] operands consumed (count CS)
    const uint32_t bar_tfull = bar_empty + 8u * stages;   // [G] accumulator ready (count 1)
    const uint32_t bar_tempty = bar_tfull + 8u * kGMax;   // [G] accumulator drained (tile warps)
    const uint32_t bar_cfull = bar_tempty + 8u * kGMax;   // [G] constants published (count 32)
    const uint32_t bar_sfull = bar_cfull + 8u * kGMax;    // [G] output tile staged (tile warps)
    const uint32_t bar_sfree = bar_sfull + 8u * kGMax;    // [G] staging tile reusable (count 1)
    const uint32_t bar_xfull = bar_sfree + 8u * kGMax;    // [G] op #6 x tile landed (count 1 + tx)
    const uint32_t bar_xfree = bar_xfull + 8u * kGMax;    // [G] op #6 x tile consumed (tile warps)
    const uint32_t bar_xst = bar_xfree + 8u * kGMax;      // [G][pass] op #6 DSMEM row stats (1 + tx)
    const uint32_t bar_bfull = bar_xst + 16u * kGMax;     // resident B landed (count 1 + tx)
    const uint32_t bar_ptempty = bar_bfull + 8u;          // [G] pair: accumulator drained in both CTAs
    const uint32_t bar_kfull = bar_ptempty + 8u * kGMax;  // split-K reducer: partial sums staged (1 + tx)
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gbase + L.tmem_slot);
    float* consts = reinterpret_cast<float*>(gbase + L.consts);
    acc_t* red = reinterpret_cast<acc_t*>(gbase + L.red);
    acc_t* xbuf = reinterpret_cast<acc_t*>(gbase + L.xbuf);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    unsigned long long* trc = (p.trace && (int)blockIdx.x == p.trace_cta) ? p.trace : nullptr;
    const uint32_t tmem_cols = tmem_cols_for(BN, p.G);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmO);
        if (IS_LN) tma_prefetch_desc(&tmX);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(bar_full + 8u * s, 1);
            mbar_init(bar_empty + 8u * s, CS);   // one tcgen05.commit from every CTA of the cluster
        }
        for (uint32_t i = 0; i < (uint32_t)kGMax; ++i) {
            mbar_init(bar_tfull + 8u * i, 1);
            mbar_init(bar_tempty + 8u * i, tile_warps);
            mbar_init(bar_cfull + 8u * i, 32);
            mbar_init(bar_sfull + 8u * i, tile_warps);
            mbar_init(bar_sfree + 8u * i, 1);
            mbar_init(bar_xfull + 8u * i, 1);
            mbar_init(bar_xfree + 8u * i, yin ? 1u : tile_warps);   // yin: the store warp frees it
            mbar_init(bar_xst + 16u * i, 1);
            mbar_init(bar_xst + 16u * i + 8u, 1);
        }
        mbar_init(bar_bfull, 1);
        for (uint32_t i = 0; i < (uint32_t)kGMax; ++i) mbar_init(bar_ptempty + 8u * i, 2u * tile_warps);
        mbar_init(bar_kfull, 1);
        fence_mbar_init();
    }
    if (warp == 2) {
        if constexpr (PAIR) tmem_alloc_pair(smem_u32(const_cast<uint32_t*>(tmem_slot)), tmem_cols);
        else tmem_alloc(smem_u32(const_cast<uint32_t*>(tmem_slot)), tmem_cols);
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the next kernel may start its prologue as soon as SMs free up; every access
    // to activation memory (written / read by the neighbouring kernels) waits below
    pdl_launch_dependents();

    const uint32_t CL = PAIR ? 2u : CS;                   // CTAs per cluster
    const uint32_t cid = blockIdx.x / CL, nclus = gridDim.x / CL;
    const uint32_t num_units = (uint32_t)p.num_units, n_groups = (uint32_t)p.n_groups;
    const uint32_t KS = (IS_LN && p.ksplit > 1) ? (uint32_t)p.ksplit : 1u;   // split-K (op #6 only)
    const uint32_t m_tiles = num_units / n_groups;
    const int num_kb = (p.K + kBK - 1) / kBK;
    const uint32_t a_bytes = kBM * kBK, b_bytes = (uint32_t)bn_b * kBK;
    const uint16_t cmask = (uint16_t)((1u << CS) - 1u);
    const uint32_t W = (uint32_t)p.out_w;
    const uint32_t lgW = 31u - (uint32_t)__clz((int)W);   // W is a power of two
    const bool resb = p.resb != 0;
    // This CTA's tile sequence (identical in every role).  m-major: the cluster
    // owns m-tiles cid, cid+nclus, ... and walks its n-groups innermost (the A tile
    // is reused across them; required by resident B).  Otherwise the (m, n) units
    // are dealt round-robin (more parallelism when there are few m-tiles).
    const uint32_t my_m = cid < m_tiles ? (m_tiles - cid + nclus - 1) / nclus : 0u;
    // weight-stationary slice: cluster cid owns column group g = cid % n_groups and the m units
    // li, li + cnt, ... of it (cnt clusters share the group)
    const uint32_t wg = cid % n_groups, wli = cid / n_groups;
    const uint32_t wcnt = (nclus - wg + n_groups - 1) / n_groups;
    const uint32_t my_tiles = wsl ? (wli < m_tiles ? (m_tiles - wli + wcnt - 1) / wcnt : 0u)
                            : p.mt_major ? my_m * n_groups
                                         : (cid < num_units ? (num_units - cid + nclus - 1) / nclus : 0u);
    auto tile_at = [&](uint32_t it, uint32_t& m_tile, uint32_t& ng) {
        if (wsl) {
            const uint32_t u = wli + it * wcnt;
            m_tile = PAIR ? 2u * u + rank : u;
            ng = wg;
        } else if (p.mt_major) {
            m_tile = cid + (it / n_groups) * nclus;
            ng = it % n_groups;
        } else {
            const uint32_t u = KS > 1u ? (cid + it * nclus) / KS : cid + it * nclus;
            m_tile = PAIR ? 2u * (u / n_groups) + rank : u / n_groups;   // pair: units are m-tile pairs
            ng = u % n_groups;
        }
    };
    // split-K: this unit's split and k-block range (split 0 reduces)
    auto split_of = [&](uint32_t it) -> uint32_t { return KS > 1u ? (cid + it * nclus) % KS : 0u; };
    auto kb_range = [&](uint32_t it, int& kb0, int& kb1) {
        kb0 = KS > 1u ? (int)split_of(it) * p.kb_per : 0;
        kb1 = KS > 1u ? min(num_kb, kb0 + p.kb_per) : num_kb;
    };
    auto n0_of = [&](uint32_t ng) -> int { return (int)((PAIR ? ng : ng * CS + rank) * (uint32_t)BN); };
    // op #6 x tile buffer of tile `it` and its phase (xstage buffers: 1 or G, powers of two)
    const uint32_t xsb = p.xstage > 0 ? (uint32_t)p.xstage : 1u;
    const uint32_t lgX = xsb == 4u ? 2u : xsb == 2u ? 1u : 0u;
    auto xbuf_of = [&](uint32_t it) -> uint32_t { return it & (xsb - 1u); };
    auto xph_of = [&](uint32_t it) -> uint32_t { return (it >> lgX) & 1u; };

    // Producer, MMA and store roles run on the whole warp with warp-uniform control
    // flow (addresses and descriptors stay in uniform registers); one elected lane
    // issues the TMA / tcgen05 instructions.
    if (warp == 0) {
        // ============================ TMA producer ============================
        int s = 0;
        uint32_t ph = 0;
        const int a_rows = kBM / (int)CS;
        auto load_a = [&](int kb, int row0) {
            if (CS == 1)
                tma_load_2d(&tmA, sA + (uint32_t)s * a_bytes, bar_full + 8u * s, kb * kBK, row0);
            else
                tma_load_2d_mc(&tmA, sA + (uint32_t)s * a_bytes + rank * (uint32_t)a_rows * kBK,
                               bar_full + 8u * s, kb * kBK, row0 + (int)rank * a_rows, cmask);
        };
        if (resb) {
            // resident B: every (n-group, k-block) weight tile of this CTA, loaded once
            if (elect_one()) {
                mbar_arrive_expect_tx(bar_bfull, n_groups * (uint32_t)num_kb * b_bytes);
                for (uint32_t ng = 0; ng < n_groups; ++ng)
                    for (int kb = 0; kb < num_kb; ++kb)
                        tma_load_2d(&tmB, base + L.bres + (ng * (uint32_t)num_kb + (uint32_t)kb) * b_bytes, bar_bfull,
                                    kb * kBK, n0_of(ng));
            }
            __syncwarp();
            pdl_wait();   // activations: produced by the previous kernel
            // the ring streams A only: one load per (m-tile, k-block)
            for (uint32_t j = 0; j < my_m; ++j) {
                const int row0 = (int)((cid + j * nclus) * kBM);
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(bar_empty + 8u * s, ph ^ 1u);
                    if (elect_one()) {
                        if (trc && kb == 0 && j < 512) trc[2 * j] = gtimer();
                        mbar_arrive_expect_tx(bar_full + 8u * s, a_bytes);
                        load_a(kb, row0);
                    }
                    __syncwarp();
                    if (++s == stages) { s = 0; ph ^= 1u; }
                }
            }
        } else if (wsl) {
            // this cluster's B slice (this CTA's half rows for a pair), loaded once; the bytes
            // of both CTAs of a pair complete on the leader's barrier
            if (elect_one()) {
                const uint32_t bb = PAIR ? mapa(bar_bfull, 0) : bar_bfull;
                if (!PAIR || rank == 0) mbar_arrive_expect_tx(bar_bfull, (PAIR ? 2u : 1u) * (uint32_t)num_kb * b_bytes);
                const int n0 = n0_of(wg) + (PAIR ? (int)(rank * hrows) : 0);
                for (int kb = 0; kb < num_kb; ++kb) {
                    if constexpr (PAIR) tma_load_2d_pair(&tmB, base + L.bres + (uint32_t)kb * b_bytes, bb, kb * kBK, n0);
                    else tma_load_2d(&tmB, base + L.bres + (uint32_t)kb * b_bytes, bb, kb * kBK, n0);
                }
            }
            __syncwarp();
            pdl_wait();   // activations: produced by the previous kernel
            for (uint32_t it = 0; it < my_tiles; ++it) {
                uint32_t m_tile, ng;
                tile_at(it, m_tile, ng);
                const int row0 = (int)(m_tile * kBM);
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(bar_empty + 8u * s, ph ^ 1u);
                    if (elect_one()) {
                        if (trc && kb == 0 && it < 512) trc[2 * it] = gtimer();
                        if constexpr (PAIR) {
                            if (rank == 0) mbar_arrive_expect_tx(bar_full + 8u * s, 2u * a_bytes);
                            tma_load_2d_pair(&tmA, sA + (uint32_t)s * a_bytes, mapa(bar_full + 8u * s, 0), kb * kBK, row0);
                        } else {
                            mbar_arrive_expect_tx(bar_full + 8u * s, a_bytes);
                            tma_load_2d(&tmA, sA + (uint32_t)s * a_bytes, bar_full + 8u * s, kb * kBK, row0);
                        }
                    }
                    __syncwarp();
                    if (++s == stages) { s = 0; ph ^= 1u; }
                }
            }
        } else {
            pdl_wait();   // activations: produced by the previous kernel
            for (uint32_t it = 0; it < my_tiles; ++it) {
                uint32_t m_tile, ng;
                tile_at(it, m_tile, ng);
                const int n0 = n0_of(ng), row0 = (int)(m_tile * kBM);
                int kbA, kbB;
                kb_range(it, kbA, kbB);
                for (int kb = kbA; kb < kbB; ++kb) {
                    mbar_wait(bar_empty + 8u * s, ph ^ 1u);
                    if constexpr (PAIR) {
                        // both CTAs load their halves; the bytes complete on the leader's barrier
                        if (elect_one()) {
                            if (trc && kb == 0 && it < 512) trc[2 * it] = gtimer();
                            if (rank == 0) mbar_arrive_expect_tx(bar_full + 8u * s, 2u * (a_bytes + b_bytes));
                            const uint32_t fb = mapa(bar_full + 8u * s, 0);
                            for (uint32_t h = 0; h < nh2; ++h)
                                tma_load_2d_pair(&tmB, sB + (uint32_t)s * b_bytes + h * hrows * kBK, fb, kb * kBK,
                                                 n0 + (int)(h * nmma + rank * hrows));
                            tma_load_2d_pair(&tmA, sA + (uint32_t)s * a_bytes, fb, kb * kBK, row0);
                        }
                        __syncwarp();
                        if (++s == stages) { s = 0; ph ^= 1u; }
                        continue;
                    }
                    if (elect_one()) {
                        if (trc && kb == 0 && it < 512) trc[2 * it] = gtimer();
                        if (trc && it < 4 && kb < 16) trc[2048 + 16 * (40 + it) + kb] = gtimer();
                        mbar_arrive_expect_tx(bar_full + 8u * s, a_bytes + b_bytes);
                        tma_load_2d(&tmB, sB + (uint32_t)s * b_bytes, bar_full + 8u * s, kb * kBK, n0);
                        load_a(kb, row0);
                    }
                    __syncwarp();
                    if (++s == stages) { s = 0; ph ^= 1u; }
                }
            }
        }
        // Drain: every stage's last fill released by all consumers of the cluster,
        // so no multicast commit can still target this CTA after it exits.
        for (int i = 0; i < stages; ++i) {
            mbar_wait(bar_empty + 8u * s, ph ^ 1u);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ==============================
        const uint32_t idesc = idesc_i8(PAIR ? 2u * kBM : kBM, nmma);
        const uint32_t hoff16 = (hrows * kBK) >> 4;      // descriptor step to MMA half 1's B rows
        int s = 0;
        uint32_t ph = 0;
        if (resb || (wsl && (!PAIR || rank == 0))) mbar_wait(bar_bfull, 0);
        // one tile: MMAs over its k-blocks starting at ring slot (s0, ph0); with resident B
        // the n-groups of an m-tile share the A slots (waited by the first, released by the last)
        auto mma_tile = [&](uint32_t it, uint32_t ng, bool first, bool last, int& ss, uint32_t& pp) {
            const uint32_t buf = it & (G - 1u), aph = (it >> lgG) & 1u;
            mbar_wait((PAIR ? bar_ptempty : bar_tempty) + 8u * buf, aph ^ 1u);
            tc_fence_after();
            if (trc && lane == 0 && it < 256) trc[1024 + 4 * it] = gtimer();
            const uint32_t d = tmem_base + buf * (uint32_t)BN;
            int kbA, kbB;
            kb_range(it, kbA, kbB);
            for (int kb = kbA; kb < kbB; ++kb) {
                if (first) mbar_wait(bar_full + 8u * ss, pp);
                tc_fence_after();
                if (trc && lane == 0 && it < 4 && kb < 16) trc[2048 + 16 * (44 + it) + kb] = gtimer();
                if (trc && lane == 0 && it < 256 && kb == 0) trc[1024 + 4 * it + 1] = gtimer();
                const uint64_t ad = umma_desc_k128(sA + (uint32_t)ss * a_bytes);
                const uint64_t bd = umma_desc_k128(resb ? base + L.bres + (ng * (uint32_t)num_kb + (uint32_t)kb) * b_bytes
                                                   : wsl ? base + L.bres + (uint32_t)kb * b_bytes
                                                        : sB + (uint32_t)ss * b_bytes);
                const int rem = p.K - kb * kBK;
                const int nk = rem >= kBK ? 4 : rem / 32;
                if (elect_one()) {
                    if constexpr (PAIR) {
                        for (uint32_t h = 0; h < nh2; ++h)
                            for (int k = 0; k < nk; ++k)
                                mma_i8_pair(d + h * nmma, ad + 2u * k, bd + h * hoff16 + 2u * k, idesc, (kb != kbA) | (k != 0));
                        mma_commit_pair_mc(bar_empty + 8u * ss, 3);   // both CTAs' slots free
                    } else {
                        for (int k = 0; k < nk; ++k)
                            mma_i8(d, ad + 2u * k, bd + 2u * k, idesc, (kb != kbA) | (k != 0));
                        if (last) {
                            if (CS == 1) mma_commit(bar_empty + 8u * ss);
                            else mma_commit_mc(bar_empty + 8u * ss, cmask);
                        }
                    }
                    if (trc && it < 256 && kb == 0) trc[1024 + 4 * it + 2] = gtimer();
                }
                __syncwarp();
                if (++ss == stages) { ss = 0; pp ^= 1u; }
            }
            if (elect_one()) {
                if constexpr (PAIR) mma_commit_pair_mc(bar_tfull + 8u * buf, 3);   // both CTAs' accumulators
                else mma_commit(bar_tfull + 8u * buf);
            }
            __syncwarp();
            if (trc && lane == 0 && it < 256) trc[1024 + 4 * it + 3] = gtimer();
        };
        if (resb) {
            uint32_t it = 0;
            for (uint32_t j = 0; j < my_m; ++j) {
                int ss = s;
                uint32_t pp = ph;
                for (uint32_t ng = 0; ng < n_groups; ++ng, ++it) {
                    ss = s;
                    pp = ph;
                    mma_tile(it, ng, ng == 0, ng + 1 == n_groups, ss, pp);
                }
                s = ss;
                ph = pp;
            }
        } else if (!PAIR || rank == 0) {   // pair: the leader issues for both CTAs
            for (uint32_t it = 0; it < my_tiles; ++it) {
                uint32_t m_tile, ng;
                tile_at(it, m_tile, ng);
                mma_tile(it, ng, true, true, s, ph);
            }
        }
    } else if (warp == 2) {
        // ============================ output store warp =========================
        pdl_wait();   // outputs may overwrite what the previous kernel still reads
        for (uint32_t it = 0; it < (dst ? 0u : my_tiles); ++it) {
            if (split_of(it) != 0u) continue;   // split-K partial: nothing to store
            const uint32_t sb = it & (G - 1u), sph = (it >> lgG) & 1u;
            mbar_wait(bar_sfull + 8u * sb, sph);
            if (trc && lane == 0 && it < 64) trc[2048 + 16 * it + 8] = gtimer();
            if (lane == 0) {
                uint32_t m_tile, ng;
                tile_at(it, m_tile, ng);
                const int n0 = n0_of(ng);
                const int32_t row0 = (int32_t)(m_tile * kBM);
                const uint32_t src = base + L.out + sb * tile_bytes;
                if (EPI != EP_ACC)
                for (uint32_t sub = 0; sub < ((uint32_t)BN >> lgW); ++sub)
                    tma_store_2d(&tmO, src + (sub << (lgW + 7u)), n0 + (int)(sub << lgW), row0);
                bulk_commit();
                bulk_wait_read<0>();              // the stores have read the staging tile
                if (trc && it < 64) trc[2048 + 16 * it + 9] = gtimer();
                mbar_arrive(bar_sfree + 8u * sb);
                if (yin && p.resid == nullptr) mbar_arrive(bar_xfree + 8u * sb);   // (x tile == staging tile)
            }
            __syncwarp();
        }
        if (lane == 0) bulk_wait_all();           // output writes complete before the CTA retires
        if (trc && lane == 0) trc[2048 + 16 * 63 + 10] = gtimer();
        __syncwarp();
    } else if (warp == 3) {
        // ============================ loader ====================================
        // Per tile: (op #6) TMA the residual x[rows][cols] tile into xres[buf] as soon
        // as the previous user of that buffer finished pass 1 (xfree), then copy the
        // per-column constants once the buffer's previous tile is fully drained (tempty).
        if (p.zero_ptr) {
            // clear the next launch's split-K partial sums and counters (after the previous
            // grid -- whose op #6 may still read them -- has completed)
            pdl_wait();
            int4* zp = reinterpret_cast<int4*>(p.zero_ptr);
            const int64_t n4 = p.zero_words >> 2;
            for (int64_t i = (int64_t)blockIdx.x * 32 + lane; i < n4; i += (int64_t)gridDim.x * 32)
                zp[i] = make_int4(0, 0, 0, 0);
        }
        const bool load_x = IS_LN && (p.resid == nullptr) && p.xstage;
        if (load_x) pdl_wait();
        for (uint32_t it = 0; it < my_tiles; ++it) {
            if (split_of(it) != 0u) continue;   // split-K partial: no constants / residual needed
            uint32_t m_tile, ng;
            tile_at(it, m_tile, ng);
            const int n0 = n0_of(ng);
            const uint32_t buf = it & (G - 1u), aph = (it >> lgG) & 1u;
            if (load_x) {
                const uint32_t xb = xbuf_of(it), xph = xph_of(it);
                mbar_wait(bar_xfree + 8u * xb, xph ^ 1u);
                if (lane == 0) {
                    const uint32_t dst = base + L.xres + xb * tile_bytes;
                    mbar_arrive_expect_tx(bar_xfull + 8u * xb, tile_bytes);
                    for (uint32_t sub = 0; sub < ((uint32_t)BN >> lgW); ++sub)
                        tma_load_2d(&tmX, dst + (sub << (lgW + 7u)), bar_xfull + 8u * xb, n0 + (int)(sub << lgW),
                                    (int32_t)(m_tile * kBM));
                }
                __syncwarp();
            }
            if (IS_LN && p.resid != nullptr) {
                // fp32 residual rows of this tile -> L2 ahead of pass 1 (its per-chunk loads are
                // otherwise HBM-latency bound: one dependent load round trip per 16 columns)
                if (it == 0) pdl_wait();
                for (uint32_t r = lane; r < (uint32_t)kBM; r += 32u) {
                    const int64_t row = (int64_t)m_tile * kBM + r;
                    if (row < p.M) bulk_prefetch_l2(p.resid + row * (int64_t)p.ldo + n0, (uint32_t)BN * 4u);
                }
            }
            mbar_wait(bar_tempty + 8u * buf, aph ^ 1u);
            if (trc && lane == 0 && it < 512) trc[3072 + 2 * it] = gtimer();
            float* cb = consts + (size_t)(csh ? 0u : buf) * kNConst * BN;
            if (!csh || it == 0)
            for (int c = (int)lane; c < BN; c += 32) {
                const int n = n0 + c;
                cb[0 * BN + c] = __ldg(p.m + n);
                cb[1 * BN + c] = HAS_B ? __ldg(p.b + n) : 0.0f;
                cb[2 * BN + c] = HAS_ZC ? __int_as_float(__ldg(p.zc + n)) : 0.0f;
                if (IS_LN) {
                    cb[3 * BN + c] = __ldg(p.gamma + n);
                    cb[4 * BN + c] = __ldg(p.beta + n);
                }
                if (EPI == EP2_QKV) cb[3 * BN + c] = __ldg(p.gamma + n);   // 1/s of this column's quantizer
            }
            if (trc && lane == 0 && it < 512) trc[3072 + 2 * it + 1] = gtimer();
            mbar_arrive(bar_cfull + 8u * buf);
            if (IS_LN && KS > 1u) {
                // split-K reducer: once the S-1 partners have counted in and this CTA's own MMAs
                // have completed (the operand ring is free: one unit per cluster), bulk-copy the
                // summed partial rows kacc[rows][n0, n0 + BN) into the ring, one row per copy
                const int32_t* cnt = p.kcnt + m_tile * CS + rank;
                if (lane == 0)
                    while (ld_acquire_gpu(cnt) < (int32_t)KS - 1) __nanosleep(32);
                __syncwarp();
                (void)ld_acquire_gpu(cnt);
                fence_proxy_async_global();   // (the copies below read through the async proxy)
                mbar_wait(bar_tfull + 8u * buf, aph);
                const int64_t r0 = (int64_t)m_tile * kBM;
                const uint32_t nrows = (uint32_t)min((int64_t)kBM, p.M - r0);
                if (lane == 0) mbar_arrive_expect_tx(bar_kfull, nrows * (uint32_t)BN * 4u);
                __syncwarp();
                for (uint32_t r = lane; r < nrows; r += 32u)
                    bulk_load_g2s(base + L.a + r * ksplit_row_bytes(BN), p.kacc + (r0 + r) * (int64_t)p.ldo + n0,
                                  (uint32_t)BN * 4u, bar_kfull);
            }
        }
    } else {
        // ============================ epilogue ================================
        const uint32_t ew = warp - kEpiWarp0;
        const uint32_t quad = warp & 3u;            // TMEM lane quadrant this warp may access
        const uint32_t grp = ew >> (4u - lgEG);     // ping-pong group: 16/EG warps each
        const uint32_t P = 4u >> lgEG;              // column parts per group (4/EG)
        const uint32_t part = (ew >> 2) & (P - 1u);
        const uint32_t rit = quad * 32u + lane;     // row in tile
        const int nch = BN / kChunk;
        const int per = (nch + (int)P - 1) / (int)P;
        const int ch_lo = min((int)part * per, nch), ch_hi = min(ch_lo + per, nch);
        // staging layout: [BN/W sub-boxes][128 rows][W bytes]; 16-B granule g of a row
        // XOR-swizzled like TMA SWIZZLE_{W}B (conflict-free 16-B writes per warp)
        const uint32_t swz_shift = W == 128 ? 0u : W == 64 ? 1u : 2u;
        const uint32_t swz_mask = W == 128 ? 7u : W == 64 ? 3u : W == 32 ? 1u : 0u;
        const uint32_t row_swz = (rit >> swz_shift) & swz_mask;
        const uint32_t lg = lgW - 4u, gm = (W >> 4) - 1u;
        const uint32_t gran_off_row = rit << lgW;
        auto gran = [&](int ch) -> uint32_t {        // offset of this row's granule of chunk ch
            const uint32_t c = (uint32_t)ch;
            return ((c >> lg) << (lgW + 7u)) + gran_off_row + (((c & gm) ^ row_swz) << 4);
        };
        const bool elected = (ew == 0 && lane == 0);
        const bool grp_leader = ((ew & (tile_warps - 1u)) == 0 && lane == 0);
        const float2 inv2 = make_float2(p.inv_q, p.inv_q);
        pdl_wait();   // (global residual / taps)

        for (uint32_t it = grp; it < my_tiles; it += EG) {
            uint32_t m_tile, ng;
            tile_at(it, m_tile, ng);
            const int n0 = n0_of(ng);
            const uint32_t buf = it & (G - 1u), aph = (it >> lgG) & 1u;
            if (IS_LN && KS > 1u && split_of(it) != 0u) {
                // ---- split-K partial: TMEM -> smem (row-major int32, in the operand ring,
                // free once every MMA of this cluster's only unit has completed) -> bulk
                // reduce-add into kacc; then count in for the reducer
                mbar_wait(bar_tfull + 8u * buf, aph);
                tc_fence_after();
                const int64_t prow = (int64_t)m_tile * kBM + rit;
                const uint32_t tbp = tmem_base + ((quad * 32u) << 16) + buf * (uint32_t)BN;
                const uint32_t stg = base + L.a + rit * ksplit_row_bytes(BN);
                for (int ch = ch_lo; ch < ch_hi; ++ch) {
                    uint32_t r[16];
                    tmem_ld16(tbp + (uint32_t)(ch * kChunk), r);
                    tmem_wait_ld_dep(r);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        st_shared_v4(stg + (uint32_t)ch * 64u + 16u * q, r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                }
                fence_proxy_async_smem();
                if (prow < p.M && ch_hi > ch_lo) {
                    bulk_reduce_add_s32(p.kacc + prow * (int64_t)p.ldo + n0 + ch_lo * kChunk,
                                        stg + (uint32_t)ch_lo * 64u, (uint32_t)(ch_hi - ch_lo) * 64u);
                    bulk_commit();
                    bulk_wait_all();
                    fence_proxy_async_global();
                }
                __threadfence();
                tc_fence_before();
                named_bar_sync(1u + buf, 32u * tile_warps);
                if (grp_leader) red_release_gpu_add(p.kcnt + m_tile * CS + rank, 1);
                continue;
            }
            const uint32_t sbuf = base + L.out + buf * tile_bytes;
            if (!dst) mbar_wait(bar_sfree + 8u * buf, aph ^ 1u);   // staging tile read by its last stores
            mbar_wait(bar_cfull + 8u * buf, aph);
            mbar_wait(bar_tfull + 8u * buf, aph);
            tc_fence_after();
            if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 2] = gtimer();
            const int64_t row = (int64_t)m_tile * kBM + rit;
            const bool valid = row < p.M;
            const uint32_t tb = tmem_base + ((quad * 32u) << 16) + buf * (uint32_t)BN;
            const float* cm = consts + (size_t)(csh ? 0u : buf) * kNConst * BN;

            // dQ (+bias) of one 16-column chunk, two columns per f32x2 op:
            // y = fl(fmaf(fl(acc - zc), m, b))  (bit-identical to the scalar form)
            auto dequant16 = [&](uint32_t (&r)[16], int cl, float2 (&y)[8]) {
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) {
                    const float4 mv = *reinterpret_cast<const float4*>(cm + cl + 4 * j4);
                    if constexpr (HAS_ZC) {
                        const int4 zv = *reinterpret_cast<const int4*>(cm + 2 * BN + cl + 4 * j4);
                        r[4 * j4 + 0] -= (uint32_t)zv.x; r[4 * j4 + 1] -= (uint32_t)zv.y;
                        r[4 * j4 + 2] -= (uint32_t)zv.z; r[4 * j4 + 3] -= (uint32_t)zv.w;
                    }
                    const float2 a0 = i2f_pair<SMALLK>(r[4 * j4 + 0], r[4 * j4 + 1]);
                    const float2 a1 = i2f_pair<SMALLK>(r[4 * j4 + 2], r[4 * j4 + 3]);
                    if constexpr (HAS_B) {
                        const float4 bv = *reinterpret_cast<const float4*>(cm + BN + cl + 4 * j4);
                        y[2 * j4] = f2_fma(a0, make_float2(mv.x, mv.y), make_float2(bv.x, bv.y));
                        y[2 * j4 + 1] = f2_fma(a1, make_float2(mv.z, mv.w), make_float2(bv.z, bv.w));
                    } else {
                        y[2 * j4] = f2_mul(a0, make_float2(mv.x, mv.y));
                        y[2 * j4 + 1] = f2_mul(a1, make_float2(mv.z, mv.w));
                    }
                }
            };
            auto tap_acc = [&](const uint32_t (&r)[16], int col) {
                if (p.acc_tap && valid) {
                    int32_t* trow = p.acc_tap + row * (int64_t)p.ldo + col;
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4)
                        st_v4(trow + 4 * j4, make_int4((int)r[4 * j4], (int)r[4 * j4 + 1], (int)r[4 * j4 + 2],
                                                       (int)r[4 * j4 + 3]));
                }
            };
            // chunk loop; op #5 keeps the next tcgen05.ld in flight while processing
            auto for_chunks = [&](auto&& fn) {
                if constexpr (IS_LN && !LN_PREFETCH) {
                    for (int ch = ch_lo; ch < ch_hi; ++ch) {
                        uint32_t ra[16];
                        tmem_ld16(tb + (uint32_t)(ch * kChunk), ra);
                        tmem_wait_ld_dep(ra);
                        fn(ra, ch);
                    }
                } else {
                    uint32_t ra[16], rb[16];
                    int ch = ch_lo;
                    if (ch < ch_hi) tmem_ld16(tb + (uint32_t)(ch * kChunk), ra);
                    while (ch < ch_hi) {
                        tmem_wait_ld_dep(ra);
                        if (ch + 1 < ch_hi) tmem_ld16(tb + (uint32_t)((ch + 1) * kChunk), rb);
                        fn(ra, ch);
                        if (++ch >= ch_hi) break;
                        tmem_wait_ld_dep(rb);
                        if (ch + 1 < ch_hi) tmem_ld16(tb + (uint32_t)((ch + 1) * kChunk), ra);
                        fn(rb, ch);
                        ++ch;
                    }
                }
            };

            if constexpr (EPI == EP_ACC) {
                // A1 = raw dot - z_x * wsum1[n], straight to global (64 contiguous bytes of
                // this thread's row per chunk): the round trip the unfused plan measures
                for_chunks([&](uint32_t (&r)[16], int ch) {
                    const int cl = ch * kChunk;
                    if constexpr (HAS_ZC) {
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4) {
                            const int4 zv = *reinterpret_cast<const int4*>(cm + 2 * BN + cl + 4 * j4);
                            r[4 * j4 + 0] -= (uint32_t)zv.x; r[4 * j4 + 1] -= (uint32_t)zv.y;
                            r[4 * j4 + 2] -= (uint32_t)zv.z; r[4 * j4 + 3] -= (uint32_t)zv.w;
                        }
                    }
                    if (valid) {
                        int32_t* orow = p.acc_out + row * (int64_t)p.ldo + n0 + cl;
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4)
                            st_v4(orow + 4 * j4, make_int4((int)r[4 * j4], (int)r[4 * j4 + 1], (int)r[4 * j4 + 2],
                                                           (int)r[4 * j4 + 3]));
                    }
                });
            } else if constexpr (!IS_LN) {
                for_chunks([&](uint32_t (&r)[16], int ch) {
                    const int cl = ch * kChunk;
                    float2 y[8];
                    dequant16(r, cl, y);
                    tap_acc(r, n0 + cl);
                    float v[16];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float2 t;
                        if constexpr (EPI == EP5_RELU) t = f2_mul(y[j], inv2);   // ReLU folds into the pack
                        else if constexpr (EPI == EP2_QKV)   // op #2: fl(y * fl(1/s_q|k|v)) per column
                            t = f2_mul(y[j], *reinterpret_cast<const float2*>(cm + 3 * BN + cl + 2 * j));
                        else t = f2_mul(make_float2(gelu_erf_f32(y[j].x), gelu_erf_f32(y[j].y)), inv2);
                        v[2 * j] = t.x;
                        v[2 * j + 1] = t.y;
                    }
                    uint32_t w[4];
                    quant_pack16<EPI == EP5_RELU, ZQNZ>(v, p.zq, w);
                    if (dst) {
                        if (valid) st_v4(p.out + row * (int64_t)p.ldo + n0 + cl,
                                         make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]));
                    } else {
                        st_shared_v4(sbuf + gran(ch), w[0], w[1], w[2], w[3]);
                    }
                });
            } else {
                // ---------------- fused op #6: dQ, bias, +residual, LayerNorm, Q ----------------
                const int C = p.ldo;
                const bool x_res = (p.resid == nullptr);
                const bool x_smem = x_res && p.xstage;
                const uint32_t xtile = base + L.xres + xbuf_of(it) * tile_bytes;
                if (x_smem) mbar_wait(bar_xfull + 8u * xbuf_of(it), xph_of(it));   // residual x tile landed
                if (KS > 1u) mbar_wait(bar_kfull, 0);   // split-K reducer: the partners' sums staged in smem
                if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 6] = gtimer();
                const float2 sx2 = make_float2(p.s_x, p.s_x);
                const float2 one2 = make_float2(p.one, p.one);
                const float xoff = 8388608.0f + 128.0f + (float)p.z_x;   // exact: |z_x| <= 128
                const float2 xoff2 = make_float2(xoff, xoff);
                // pass 1: z = fl(fl(fmaf(fl(A2), m2, b2)) + r); park z in TMEM; row statistics:
                // fp64 the plain sum (two-pass, O5 order); fp32 shifted sums (S1, S2) about
                // K = mean of this warp's first 16 columns (R15)
                double s1d = 0.0;
                float2 s1f = make_float2(0.f, 0.f), s2f = make_float2(0.f, 0.f), Kv = make_float2(0.f, 0.f);
                float K = 0.f;
                for_chunks([&](uint32_t (&r)[16], int ch) {
                    const int cl = ch * kChunk;
                    float2 rr[8];
                    if (!x_res) {
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4) {
                            const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(p.resid + row * C + n0 + cl) + j4)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                            rr[2 * j4] = make_float2(v.x, v.y);
                            rr[2 * j4 + 1] = make_float2(v.z, v.w);
                        }
                    } else {
                        // x - z_x as float (then z = fl(d + fl((x - z_x) * s_x))).  Exact int8 -> float without the
                        // 1/8-rate I2F.S8: with u = x ^ 0x80 (offset binary) the bits
                        // 0x4B0000uu are the float 2^23 + u, and
                        // (2^23 + u) - (2^23 + 128 + z_x) = x - z_x exactly.
                        uint32_t xw[4];
                        if (x_smem) {
                            ld_shared_v4(xtile + gran(ch), xw);
                        } else {
                            const int4 xv = valid ? ld_nc_v4(p.x + row * C + n0 + cl) : make_int4(0, 0, 0, 0);
                            xw[0] = (uint32_t)xv.x; xw[1] = (uint32_t)xv.y; xw[2] = (uint32_t)xv.z; xw[3] = (uint32_t)xv.w;
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t ob = xw[q] ^ 0x80808080u;
                            const float2 f01 = make_float2(__uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7650)),
                                                           __uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7651)));
                            const float2 f23 = make_float2(__uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7652)),
                                                           __uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7653)));
                            rr[2 * q] = f2_sub(f01, xoff2);      // x - z_x, exact
                            rr[2 * q + 1] = f2_sub(f23, xoff2);
                        }
                    }
                    if (KS > 1u && valid) {   // + the other splits' partial sums (exact int32)
                        const uint32_t kp = base + L.a + rit * ksplit_row_bytes(BN) + (uint32_t)cl * 4u;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint32_t v[4];
                            ld_shared_v4(kp + 16u * q, v);
                            r[4 * q] += v[0]; r[4 * q + 1] += v[1]; r[4 * q + 2] += v[2]; r[4 * q + 3] += v[3];
                        }
                    }
                    float2 z[8];
                    dequant16(r, cl, z);
                    tap_acc(r, n0 + cl);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        // z = fl(d + R), or fl(d + fl((x - z_x) * s_x)): dQ(x) then Add (R3)
                        z[j] = x_res ? f2_fma(f2_mul(rr[j], sx2), one2, z[j]) : f2_add(z[j], rr[j]);   // (see GemmArgs::one)
                        if constexpr (STATS64) {
                            s1d = __dadd_rn(s1d, (double)z[j].x);
                            s1d = __dadd_rn(s1d, (double)z[j].y);
                        }
                        r[2 * j] = __float_as_uint(z[j].x);
                        r[2 * j + 1] = __float_as_uint(z[j].y);
                    }
                    if constexpr (!STATS64) {
                        if (ch == ch_lo) {
                            float2 t = z[0];
#pragma unroll
                            for (int j = 1; j < 8; ++j) t = f2_add(t, z[j]);
                            K = __fmul_rn(__fadd_rn(t.x, t.y), 0.0625f);
                            Kv = make_float2(K, K);
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float2 d = f2_sub(z[j], Kv);
                            s1f = f2_add(s1f, d);
                            s2f = f2_fma(d, d, s2f);
                        }
                    }
                    if (p.resid_out && valid) {
                        float* zrow = p.resid_out + row * (int64_t)C + n0 + cl;
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4)
                            *reinterpret_cast<float4*>(zrow + 4 * j4) =
                                make_float4(z[2 * j4].x, z[2 * j4].y, z[2 * j4 + 1].x, z[2 * j4 + 1].y);
                    }
                    tmem_st16(tb + (uint32_t)cl, r);
                });
                tmem_wait_st();
                if (x_smem && !yin) {   // the x tile has been consumed: let the loader prefetch the next one
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_xfree + 8u * xbuf_of(it));
                }
                if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 3] = gtimer();

                // row statistics: column parts via smem (named barrier of the group's
                // threads), the CS CTAs of the cluster via DSMEM; always summed in the
                // same (part, rank) order so every thread / CTA derives identical stats
                // (pairs of sums travel together: one smem round and one DSMEM round per pass)
                auto row_sum2 = [&](acc_t v0, acc_t v1, uint32_t pass, acc_t& o1) -> acc_t {
                    acc_t t0 = v0, t1 = v1;
                    if (P > 1) {
                        const uint32_t slot = ((buf * 2u + pass) * P) * 2u;   // [G][pass][part][val]
                        red[(slot + part * 2u) * kBM + rit] = v0;
                        red[(slot + part * 2u + 1u) * kBM + rit] = v1;
                        named_bar_sync(1u + buf, 32u * tile_warps);
                        t0 = (acc_t)red[slot * kBM + rit];
                        t1 = (acc_t)red[(slot + 1u) * kBM + rit];
                        for (uint32_t q = 1; q < P; ++q) {   // parts in order
                            t0 = t0 + (acc_t)red[(slot + 2u * q) * kBM + rit];
                            t1 = t1 + (acc_t)red[(slot + 2u * q + 1u) * kBM + rit];
                        }
                    }
                    if (CS == 1) { o1 = t1; return t0; }
                    const uint32_t sid = buf * 2u + pass;
                    const uint32_t xb = bar_xst + 8u * sid;
                    if (part == 0) {
                        if (grp_leader) mbar_arrive_expect_tx(xb, CS * kBM * 2u * (uint32_t)sizeof(acc_t));
                        const uint32_t d0 = smem_u32(xbuf + (((size_t)sid * CS + rank) * 2u) * kBM + rit);
                        for (uint32_t r = 0; r < CS; ++r) {
                            st_async_val(mapa(d0, r), t0, mapa(xb, r));
                            st_async_val(mapa(d0 + kBM * (uint32_t)sizeof(acc_t), r), t1, mapa(xb, r));
                        }
                    }
                    mbar_wait_cluster(xb, aph);
                    acc_t S0 = 0, S1 = 0;
                    for (uint32_t r = 0; r < CS; ++r) {
                        S0 = S0 + (acc_t)xbuf[(((size_t)sid * CS + r) * 2u) * kBM + rit];
                        S1 = S1 + (acc_t)xbuf[(((size_t)sid * CS + r) * 2u + 1u) * kBM + rit];
                    }
                    o1 = S1;
                    return S0;
                };
                double mu_d64 = 0.0;
                acc_t rstd;
                float2 mu2c;
                if constexpr (STATS64) {
                    acc_t unused;
                    const acc_t mu = row_sum2(s1d, (acc_t)0, 0, unused) / (acc_t)C;
                    if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 4] = gtimer();
                    // pass 2: centred sum of squares
                    double s2d = 0.0;
                    for_chunks([&](uint32_t (&r)[16], int) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const double d0 = __dsub_rn((double)__uint_as_float(r[j]), (double)mu);
                            s2d = __dadd_rn(s2d, __dmul_rn(d0, d0));
                        }
                    });
                    double dummy;
                    const double SS = row_sum2(s2d, 0.0, 1, dummy);
                    rstd = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(SS, (double)C), (double)p.eps)));
                    mu2c = make_float2((float)mu, (float)mu);
                    mu_d64 = (double)mu;
                } else {
                    // one round of statistics exchange: per warp (mean, M2) of its columns,
                    // combined pairwise (Chan) over the column parts (smem), then over the CS
                    // CTAs of the cluster (DSMEM), in the same order everywhere
                    const float S1 = __fadd_rn(s1f.x, s1f.y), S2 = __fadd_rn(s2f.x, s2f.y);
                    const float nw = (float)((ch_hi - ch_lo) * kChunk);
                    const float q1 = nw > 0.f ? __fdiv_rn(S1, nw) : 0.f;
                    float m = __fadd_rn(K, q1), M2 = __fsub_rn(S2, __fmul_rn(S1, q1)), n = nw;
                    if (P > 1) {
                        const uint32_t slot = (buf * NPASS * P) * 2u;   // [G][pass 0][part][val]
                        red[(slot + part * 2u) * kBM + rit] = m;
                        red[(slot + part * 2u + 1u) * kBM + rit] = M2;
                        named_bar_sync(1u + buf, 32u * tile_warps);
                        // pairwise (Chan) combine of the parts, in part order
                        float ma = red[slot * kBM + rit], qa = red[(slot + 1u) * kBM + rit];
                        float na = (float)(min(per, nch) * kChunk);
                        for (uint32_t q = 1; q < P; ++q) {
                            const int lo = min((int)q * per, nch), hi = min(lo + per, nch);
                            if (hi <= lo) continue;
                            const float nb = (float)((hi - lo) * kChunk);
                            const float mb = red[(slot + 2u * q) * kBM + rit], qb = red[(slot + 2u * q + 1u) * kBM + rit];
                            const float nt = __fadd_rn(na, nb);
                            const float dm = __fsub_rn(mb, ma);
                            ma = __fadd_rn(ma, __fmul_rn(dm, __fdiv_rn(nb, nt)));
                            qa = __fadd_rn(__fadd_rn(qa, qb), __fmul_rn(__fmul_rn(dm, dm), __fdiv_rn(__fmul_rn(na, nb), nt)));
                            na = nt;
                        }
                        m = ma;
                        M2 = qa;
                        n = na;
                    }
                    if (CS > 1) {
                        const uint32_t sid = buf * 2u, sidd = buf * NPASS;   // barrier / data slot
                        const uint32_t xb = bar_xst + 8u * sid;
                        if (part == 0) {
                            if (grp_leader) mbar_arrive_expect_tx(xb, CS * kBM * 2u * (uint32_t)sizeof(acc_t));
                            const uint32_t d0 = smem_u32(xbuf + (((size_t)sidd * CS + rank) * 2u) * kBM + rit);
                            for (uint32_t r = 0; r < CS; ++r) {
                                st_async_val(mapa(d0, r), (acc_t)m, mapa(xb, r));
                                st_async_val(mapa(d0 + kBM * (uint32_t)sizeof(acc_t), r), (acc_t)M2, mapa(xb, r));
                            }
                        }
                        mbar_wait_cluster(xb, aph);
                        float msum = 0.f, qsum = 0.f;
                        for (uint32_t r = 0; r < CS; ++r) {
                            msum = __fadd_rn(msum, (float)xbuf[(((size_t)sidd * CS + r) * 2u) * kBM + rit]);
                            qsum = __fadd_rn(qsum, (float)xbuf[(((size_t)sidd * CS + r) * 2u + 1u) * kBM + rit]);
                        }
                        const float mean = __fdiv_rn(msum, (float)CS);
                        float dsq = 0.f;
                        for (uint32_t r = 0; r < CS; ++r) {
                            const float dr = __fsub_rn((float)xbuf[(((size_t)sidd * CS + r) * 2u) * kBM + rit], mean);
                            dsq = __fmaf_rn(dr, dr, dsq);
                        }
                        m = mean;
                        M2 = __fmaf_rn(dsq, n, qsum);
                    }
                    if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 4] = gtimer();
                    const float var = fmaxf(__fdiv_rn(M2, (float)C), 0.0f);
                    rstd = (acc_t)__fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
                    mu2c = make_float2(m, m);
                }
                const float2 rstd2 = make_float2((float)rstd, (float)rstd);
                if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 5] = gtimer();

                // pass 3: yhat = fl(((z-mu)*rstd)*gamma + beta); Y = Q_y(yhat)
                const float* cg = cm + 3 * BN;
                const float* cbt = cm + 4 * BN;
                for_chunks([&](uint32_t (&r)[16], int ch) {
                    const int cl = ch * kChunk;
                    float yh[16];
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4) {
                        const float4 gv = *reinterpret_cast<const float4*>(cg + cl + 4 * j4);
                        const float4 bv = *reinterpret_cast<const float4*>(cbt + cl + 4 * j4);
                        if constexpr (STATS64) {
                            const float gg[4] = {gv.x, gv.y, gv.z, gv.w};
                            const float bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const double xh = __dmul_rn(__dsub_rn((double)__uint_as_float(r[4 * j4 + j]), mu_d64), rstd);
                                yh[4 * j4 + j] = __double2float_rn(__dadd_rn(__dmul_rn(xh, (double)gg[j]), (double)bb[j]));
                            }
                        } else {
                            const float2 z0 = make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]));
                            const float2 z1 = make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3]));
                            const float2 y0 = f2_fma(f2_mul(f2_sub(z0, mu2c), rstd2), make_float2(gv.x, gv.y), make_float2(bv.x, bv.y));
                            const float2 y1 = f2_fma(f2_mul(f2_sub(z1, mu2c), rstd2), make_float2(gv.z, gv.w), make_float2(bv.z, bv.w));
                            yh[4 * j4] = y0.x; yh[4 * j4 + 1] = y0.y; yh[4 * j4 + 2] = y1.x; yh[4 * j4 + 3] = y1.y;
                        }
                    }
                    float v[16];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float2 t = f2_mul(make_float2(yh[2 * j], yh[2 * j + 1]), inv2);
                        v[2 * j] = t.x;
                        v[2 * j + 1] = t.y;
                    }
                    uint32_t w[4];
                    quant_pack16<false, ZQNZ>(v, p.zq, w);
                    st_shared_v4(sbuf + gran(ch), w[0], w[1], w[2], w[3]);
                    if (p.ln_tap && valid) {
                        float* lrow = p.ln_tap + row * (int64_t)C + n0 + cl;
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4)
                            *reinterpret_cast<float4*>(lrow + 4 * j4) =
                                make_float4(yh[4 * j4], yh[4 * j4 + 1], yh[4 * j4 + 2], yh[4 * j4 + 3]);
                    }
                });
            }
            tc_fence_before();
            fence_proxy_async_smem();   // staged bytes visible to the TMA (async proxy)
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(bar_tempty + 8u * buf);   // TMEM free: the next MMA may start
                if constexpr (PAIR) {                 // (pair: the leader's MMA waits on both CTAs)
                    if (rank == 0) mbar_arrive(bar_ptempty + 8u * buf);
                    else mbar_arrive_cluster_relaxed(mapa(bar_ptempty + 8u * buf, 0));
                }
                if (!dst) mbar_arrive(bar_sfull + 8u * buf);    // this warp's part of the tile is staged
            }
            if (trc && grp_leader && it < 64) trc[2048 + 16 * it + 7] = gtimer();
        }
    }

    // teardown: no CTA leaves while a peer may still address its shared memory
    if (trc && lane == 0) trc[2048 + 16 * 60 + warp] = gtimer();   // (debug: role done)
    tc_fence_before();
    cluster_sync_all();
    if (trc && threadIdx.x == 0) trc[2048 + 16 * 62] = gtimer();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (PAIR) tmem_dealloc_pair(tmem_base, tmem_cols);
        else tmem_dealloc(tmem_base, tmem_cols);
    }
    if (p.cta_stamps && threadIdx.x == 0) p.cta_stamps[2 * blockIdx.x + 1] = gtimer();
}

}  // namespace swinmlp
