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
//
// Roles (384 threads, 1 CTA per SM):
//   warp 0      TMA producer (one lane): A (activations) and B (weights) K-blocks
//               of 128 B into a `stages`-deep ring; A is multicast across the
//               CS CTAs of a cluster, which all work on the same 128-row m-tile.
//   warp 1      MMA issuer (one lane): tcgen05.mma.kind::i8, M=128, N=BN, K=32 per
//               instruction, int32 accumulators in TMEM, 2 accumulator buffers so
//               the epilogue of tile i overlaps the MMAs of tile i+1.
//   warp 2      TMEM allocator.
//   warp 3      column-constant loader: per tile, copies the tile's per-column
//               constants (dequant multiplier, bias, zero-point correction,
//               LN gamma/beta) from global into a 2-deep shared-memory ring.
//   warps 4-11  epilogue: warp w drains TMEM lane quadrant (w % 4) — thread = one
//               token row — over half of the tile's columns ((w-4)/4 picks the half),
//               16 columns per tcgen05.ld, next load in flight while the current
//               chunk is processed.  Each warp stages its int8 output chunk
//               [32 rows][16 B] in a private smem ring and writes it with a TMA
//               bulk tensor store (rows >= T are clipped by the TMA unit).
//
// EP6 row statistics: each thread owns one row of its half; the two halves are
// combined through shared memory, the CS CTAs of the cluster (which split the
// C columns of the same rows) exchange partial sums through DSMEM with
// st.async + mbarrier complete_tx, always summed in rank order, so every CTA
// of the cluster derives bit-identical mean and rstd.  z is parked in TMEM
// between the three passes (sum, centred sum of squares, normalise).
// Template flags F (so the hot loop carries no predicated-off work):
//   kHasB  bias present, kHasZc activation zero point != 0 (int32 correction),
//   kZqNz  output zero point != 0, kS64 LayerNorm in fp64.
// kS64 = true computes the statistics and the normalisation in fp64 in the
// oracle's operation order (bit-exact up to summation order); false uses fp32
// (cheaper; the <= 1 LSB on <= 0.01 % tier).
#pragma once
#include <cuda.h>
#include <cstdint>
#include <type_traits>

#include "sm100_ptx.cuh"

namespace swinmlp {

enum Epi : int { EP5_RELU = 0, EP5_GELU = 1, EP6_LN = 2 };

constexpr int kBM = 128;             // rows per tile (UMMA M, TMEM lanes)
constexpr int kBK = 128;             // K bytes per pipeline stage (one 128-B swizzle row)
constexpr int kEpiWarp0 = 4;
// Epilogue width per kernel: the op-#5 epilogue is light (few registers), so it
// runs 16 warps (4 per SMSP, 4 column parts per TMEM lane quadrant); op #6 keeps
// 8 warps (2 parts) for its register-heavy LayerNorm passes.
__host__ __device__ constexpr int epi_warps(int epi) { return 16; }
__host__ __device__ constexpr int kernel_threads(int epi) { return 32 * (kEpiWarp0 + epi_warps(epi)); }
constexpr int kChunk = 16;           // columns per tcgen05.ld (32x32b.x16)
constexpr int kChunkBytes = 32 * kChunk;        // [32 rows][16 B] = one warp's output chunk

constexpr int kHasB = 1, kHasZc = 2, kZqNz = 4, kS64 = 8;
constexpr int kNConst = 5;           // m, b, zc, gamma, beta

struct GemmArgs {
    int64_t M;             // token rows
    int32_t K;             // reduction length (bytes of int8)
    int32_t BN;            // columns per CTA tile (UMMA N)
    int32_t CS;            // CTAs per cluster (share one m-tile, A multicast)
    int32_t stages;        // smem ring depth
    int32_t nbuf;          // output staging tiles (1 or 2)
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
    const int8_t* x;       // [M][ldo] layer input (residual = dQ(x) when resid == nullptr)
    float s_x;
    int32_t z_x;
    const float* resid;    // [M][ldo] fp32 residual or nullptr
    float* resid_out;      // [M][ldo] fp32 z or nullptr
    const float* gamma;
    const float* beta;
    float eps;
    // debug taps
    int32_t* acc_tap;      // [M][ldo] int32 accumulators (incl. zero-point term)
    float* ln_tap;         // [M][ldo] fp32 yhat (EP6)
    // pipeline trace (debug): when non-null, CTA `trace_cta` records %globaltimer
    // stamps: trace[role*1024 + 2*i + {0,1}] for its i-th tile, roles 0 producer
    // (first stage acquired, last k-block issued), 1 MMA (accumulator acquired,
    // tile committed), 2 epilogue warp 4 (accumulator ready, tile stored), 3 the
    // constant loader (buffer acquired, constants published).
    unsigned long long* trace;
    int32_t trace_cta;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct SmemLayout {
    uint32_t a, b, ring, xres, consts, bars, tmem_slot, red, xbuf, total;
};

// nbuf: output staging buffers per epilogue warp (1 or 2 tiles in flight)
__host__ __device__ inline SmemLayout smem_layout(int epi, int BN, int CS, int stages, int nbuf) {
    SmemLayout L;
    L.a = 0;
    L.b = L.a + (uint32_t)stages * kBM * kBK;
    L.ring = L.b + (uint32_t)stages * (uint32_t)BN * kBK;
    L.xres = L.ring + (uint32_t)nbuf * (uint32_t)BN * kBM;            // op #6: residual x tiles [2]
    L.consts = L.xres + (epi == 2 ? 2u : 0u) * (uint32_t)BN * kBM;
    L.bars = L.consts + 2u * kNConst * (uint32_t)BN * 4u;
    const uint32_t nbars = 2u * stages + 2 + 2 + 4 + 2 + 2 + 2 + 2 + 2;
    L.tmem_slot = L.bars + 8u * nbars;
    L.red = (L.tmem_slot + 8 + 15) & ~15u;
    L.xbuf = L.red + 2u * 2u * 2u * kBM * 8u;
    L.total = L.xbuf + 4u * (uint32_t)CS * kBM * 8u;   // [group][pass][rank][row] doubles
    return L;
}

__host__ __device__ inline uint32_t tmem_cols_for(int BN) {
    uint32_t need = 2u * (uint32_t)BN, c = 32;
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

template <int EPI, int F>
__global__ void __launch_bounds__(kernel_threads(EPI), 1)
mlp_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ GemmArgs p) {
    using namespace sm100;
    constexpr bool HAS_B = (F & kHasB) != 0, HAS_ZC = (F & kHasZc) != 0, ZQNZ = (F & kZqNz) != 0;
    constexpr bool STATS64 = (F & kS64) != 0;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);

    const int BN = p.BN;
    const uint32_t CS = (uint32_t)p.CS;
    const int stages = p.stages;
    constexpr int kEpiWarps = epi_warps(EPI), kParts = kEpiWarps / 4;
    // warps that work on one tile: all epilogue warps (op #5), one ping-pong group (op #6)
    constexpr int kTileWarps = (EPI == EP6_LN) ? 8 : kEpiWarps;
    const SmemLayout L = smem_layout(EPI, BN, p.CS, stages, p.nbuf);
    const uint32_t sA = base + L.a, sB = base + L.b;
    const uint32_t bar_full = base + L.bars;
    const uint32_t bar_empty = bar_full + 8u * stages;
    const uint32_t bar_tfull = bar_empty + 8u * stages;
    const uint32_t bar_tempty = bar_tfull + 16u;
    const uint32_t bar_x = bar_tempty + 16u;
    const uint32_t bar_cfull = bar_x + 32u;         // bar_x: [group][pass] DSMEM row-stat exchange
    const uint32_t bar_sfull = bar_cfull + 16u;     // output tile staged (count: epilogue warps)
    const uint32_t bar_sfree = bar_sfull + 16u;     // staging buffer reusable (count 1)
    const uint32_t bar_xfull = bar_sfree + 16u;     // op #6 residual x tile landed (count 1 + tx)
    const uint32_t bar_xfree = bar_xfull + 16u;     // op #6 pass 1 done with the x tile (tile warps)
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gbase + L.tmem_slot);
    float* consts = reinterpret_cast<float*>(gbase + L.consts);   // [2][kNConst][BN]
    double* red = reinterpret_cast<double*>(gbase + L.red);   // [group][pass][half][row] partial row sums
    double* xbuf = reinterpret_cast<double*>(gbase + L.xbuf);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    unsigned long long* trc = (p.trace && (int)blockIdx.x == p.trace_cta) ? p.trace : nullptr;
    const uint32_t tmem_cols = tmem_cols_for(BN);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmO);
        if (EPI == EP6_LN) tma_prefetch_desc(&tmX);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(bar_full + 8u * s, 1);
            mbar_init(bar_empty + 8u * s, CS);   // one tcgen05.commit from every CTA of the cluster
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_tfull + 8u * i, 1);
            mbar_init(bar_tempty + 8u * i, kTileWarps);
            mbar_init(bar_x + 8u * i, 1);
            mbar_init(bar_x + 16u + 8u * i, 1);
            mbar_init(bar_cfull + 8u * i, 32);
            mbar_init(bar_sfull + 8u * i, kTileWarps);
            mbar_init(bar_sfree + 8u * i, 1);
            mbar_init(bar_xfull + 8u * i, 1);
            mbar_init(bar_xfree + 8u * i, kTileWarps);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(const_cast<uint32_t*>(tmem_slot)), tmem_cols);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const uint32_t cid = blockIdx.x / CS, nclus = gridDim.x / CS;
    const int num_kb = (p.K + kBK - 1) / kBK;
    const uint32_t a_bytes = kBM * kBK, b_bytes = (uint32_t)BN * kBK;
    const uint16_t cmask = (uint16_t)((1u << CS) - 1u);

    // Producer, MMA and store roles run on the whole warp with warp-uniform control
    // flow (so addresses and descriptors live in uniform registers); one elected
    // lane issues the TMA / tcgen05 instructions.
    if (warp == 0) {
        // ============================ TMA producer ============================
        int s = 0;
        uint32_t ph = 0, tu = 0;
        const int a_rows = kBM / (int)CS;
        for (uint32_t u = cid; u < (uint32_t)p.num_units; u += nclus) {
            const uint32_t m_tile = u / (uint32_t)p.n_groups;
            const int ng = (int)(u % (uint32_t)p.n_groups);
            const int n0 = (ng * (int)CS + (int)rank) * BN;
            const int row0 = (int)(m_tile * kBM);
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(bar_empty + 8u * s, ph ^ 1u);
                if (elect_one()) {
                    if (trc && kb == 0 && tu < 512) trc[2 * tu] = gtimer();
                    mbar_arrive_expect_tx(bar_full + 8u * s, a_bytes + b_bytes);
                    tma_load_2d(&tmB, sB + (uint32_t)s * b_bytes, bar_full + 8u * s, kb * kBK, n0);
                    if (CS == 1)
                        tma_load_2d(&tmA, sA + (uint32_t)s * a_bytes, bar_full + 8u * s, kb * kBK, row0);
                    else
                        tma_load_2d_mc(&tmA, sA + (uint32_t)s * a_bytes + rank * (uint32_t)a_rows * kBK,
                                       bar_full + 8u * s, kb * kBK, row0 + (int)rank * a_rows, cmask);
                }
                __syncwarp();
                if (++s == stages) { s = 0; ph ^= 1u; }
            }
            if (trc && lane == 0 && tu < 512) trc[2 * tu + 1] = gtimer();
            ++tu;
        }
        // Drain: every stage's last fill released by all consumers of the cluster,
        // so no multicast commit can still target this CTA after it exits.
        for (int i = 0; i < stages; ++i) {
            mbar_wait(bar_empty + 8u * s, ph ^ 1u);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ==============================
        const uint32_t idesc = idesc_i8(kBM, (uint32_t)BN);
        int s = 0;
        uint32_t ph = 0, it = 0;
        for (uint32_t u = cid; u < (uint32_t)p.num_units; u += nclus, ++it) {
            const uint32_t buf = it & 1u, aph = (it >> 1) & 1u;
            mbar_wait(bar_tempty + 8u * buf, aph ^ 1u);
            tc_fence_after();
            if (trc && lane == 0 && it < 256) trc[1024 + 4 * it] = gtimer();
            const uint32_t d = tmem_base + buf * (uint32_t)BN;
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(bar_full + 8u * s, ph);
                tc_fence_after();
                if (trc && lane == 0 && it < 256 && kb == 0) trc[1024 + 4 * it + 1] = gtimer();
                const uint64_t ad = umma_desc_k128(sA + (uint32_t)s * a_bytes);
                const uint64_t bd = umma_desc_k128(sB + (uint32_t)s * b_bytes);
                const int rem = p.K - kb * kBK;
                const int nk = rem >= kBK ? 4 : rem / 32;
                if (elect_one()) {
                    for (int k = 0; k < nk; ++k)
                        mma_i8(d, ad + 2u * k, bd + 2u * k, idesc, (kb | k) != 0);
                    if (trc && it < 256 && kb == 0) trc[1024 + 4 * it + 2] = gtimer();
                    if (CS == 1) mma_commit(bar_empty + 8u * s);
                    else mma_commit_mc(bar_empty + 8u * s, cmask);
                }
                __syncwarp();
                if (++s == stages) { s = 0; ph ^= 1u; }
            }
            if (elect_one()) mma_commit(bar_tfull + 8u * buf);
            __syncwarp();
            if (trc && lane == 0 && it < 256) trc[1024 + 4 * it + 3] = gtimer();
        }
    } else if (warp == 2) {
        // ============================ output store warp =========================
        // Writes each staged output tile with BN/W TMA tensor stores, and re-arms
        // the staging buffer (sfree): for op #6 with the int8 residual it first
        // TMA-loads the residual tile x[rows][cols] into the buffer (the epilogue
        // reads x there in pass 1 and overwrites it in place with Y in pass 3).
        {
            const uint32_t W = (uint32_t)p.out_w;
            const uint32_t nb = (uint32_t)p.nbuf;
            const bool load_x = false;   // (op #6 residual tiles are loaded by warp 3 into xres)
            auto make_ready = [&](uint32_t u, uint32_t sbuf) {   // called by one elected lane
                const uint32_t bar = bar_sfree + 8u * sbuf;
                if (load_x) {
                    const uint32_t m_tile = u / (uint32_t)p.n_groups;
                    const int ng = (int)(u % (uint32_t)p.n_groups);
                    const int n0 = (ng * (int)CS + (int)rank) * BN;
                    const uint32_t dst = base + L.ring + sbuf * (uint32_t)BN * kBM;
                    mbar_arrive_expect_tx(bar, (uint32_t)BN * kBM);
                    for (uint32_t sub = 0; sub < (uint32_t)BN / W; ++sub)
                        tma_load_2d(&tmX, dst + sub * (kBM * W), bar, n0 + (int)(sub * W), (int32_t)(m_tile * kBM));
                } else {
                    mbar_arrive(bar);
                }
            };
            if (lane == 0)
                for (uint32_t j = 0; j < nb && cid + j * nclus < (uint32_t)p.num_units; ++j)
                    make_ready(cid + j * nclus, j);
            __syncwarp();
            uint32_t it = 0;
            for (uint32_t u = cid; u < (uint32_t)p.num_units; u += nclus, ++it) {
                const uint32_t m_tile = u / (uint32_t)p.n_groups;
                const int ng = (int)(u % (uint32_t)p.n_groups);
                const int n0 = (ng * (int)CS + (int)rank) * BN;
                const uint32_t sbuf = nb == 2 ? (it & 1u) : 0u;
                const uint32_t sph = nb == 2 ? ((it >> 1) & 1u) : (it & 1u);
                mbar_wait(bar_sfull + 8u * sbuf, sph);
                const uint32_t src = base + L.ring + sbuf * (uint32_t)BN * kBM;
                if (lane == 0) {
                    for (uint32_t sub = 0; sub < (uint32_t)BN / W; ++sub)
                        tma_store_2d(&tmO, src + sub * (kBM * W), n0 + (int)(sub * W), (int32_t)(m_tile * kBM));
                    bulk_commit();
                    bulk_wait_read<0>();              // smem read: the buffer may be refilled
                    const uint32_t nxt = u + nb * nclus;
                    if (nxt < (uint32_t)p.num_units) make_ready(nxt, sbuf);
                }
                __syncwarp();
            }
            if (lane == 0) bulk_wait_all();           // output writes complete before the CTA retires
            __syncwarp();
        }
    } else if (warp == 3) {
        // ============================ column constants ========================
        // Per tile: (op #6) TMA the residual x[rows][cols] tile into xres[buf] as soon
        // as the previous user of that buffer finished pass 1 (xfree), then copy the
        // per-column constants once the buffer's previous tile is fully drained (tempty).
        const bool load_x = (EPI == EP6_LN) && (p.resid == nullptr);
        uint32_t it = 0;
        for (uint32_t u = cid; u < (uint32_t)p.num_units; u += nclus, ++it) {
            const int ng = (int)(u % (uint32_t)p.n_groups);
            const int n0 = (ng * (int)CS + (int)rank) * BN;
            const uint32_t buf = it & 1u, aph = (it >> 1) & 1u;
            if (load_x) {
                mbar_wait(bar_xfree + 8u * buf, aph ^ 1u);
                if (lane == 0) {
                    const uint32_t W = (uint32_t)p.out_w;
                    const uint32_t m_tile = u / (uint32_t)p.n_groups;
                    const uint32_t dst = base + L.xres + buf * (uint32_t)BN * kBM;
                    mbar_arrive_expect_tx(bar_xfull + 8u * buf, (uint32_t)BN * kBM);
                    for (uint32_t sub = 0; sub < (uint32_t)BN / W; ++sub)
                        tma_load_2d(&tmX, dst + sub * (kBM * W), bar_xfull + 8u * buf, n0 + (int)(sub * W),
                                    (int32_t)(m_tile * kBM));
                }
                __syncwarp();
            }
            mbar_wait(bar_tempty + 8u * buf, aph ^ 1u);     // epilogue done with this buffer
            if (trc && lane == 0 && it < 512) trc[3072 + 2 * it] = gtimer();
            float* cb = consts + (size_t)buf * kNConst * BN;
            for (int c = (int)lane; c < BN; c += 32) {
                const int n = n0 + c;
                cb[0 * BN + c] = __ldg(p.m + n);
                cb[1 * BN + c] = p.b ? __ldg(p.b + n) : 0.0f;
                cb[2 * BN + c] = p.zc ? __int_as_float(__ldg(p.zc + n)) : __int_as_float(0);
                if (EPI == EP6_LN) {
                    cb[3 * BN + c] = __ldg(p.gamma + n);
                    cb[4 * BN + c] = __ldg(p.beta + n);
                }
            }
            if (trc && lane == 0 && it < 512) trc[3072 + 2 * it + 1] = gtimer();
            mbar_arrive(bar_cfull + 8u * buf);
        }
    } else if (warp >= kEpiWarp0) {
        // ============================ epilogue ================================
        // op #5: 16 warps; warp w drains TMEM lane quadrant (w % 4) over column part
        //        (w-4)/4 of every tile.
        // op #6: two ping-pong groups of 4 warps; group g = (w-4)/4 takes the tiles
        //        with local index it % 2 == g (accumulator buffer g) and each thread
        //        owns a whole row of its CTA's columns, so row statistics are
        //        thread-local (plus the cluster exchange when C spans CTAs).
        const uint32_t ew = warp - kEpiWarp0;
        const uint32_t quad = warp & 3u;          // TMEM lane quadrant this warp may access
        const uint32_t grp = ew >> 2;             // column part (op #5) / ping-pong group (op #6)
        const uint32_t rit = quad * 32u + lane;   // row in tile
        const int nch = BN / kChunk;
        constexpr bool kPingPong = (EPI == EP6_LN);
        // op #6: group = (w-4)/8 (ping-pong), column half = ((w-4)/4) & 1
        const uint32_t pgrp = kPingPong ? (ew >> 3) : 0u;
        const uint32_t part = kPingPong ? ((ew >> 2) & 1u) : grp;
        const int nparts = kPingPong ? 2 : kParts;
        const int per = (nch + nparts - 1) / nparts;
        const int ch_lo = min((int)part * per, nch);
        const int ch_hi = min(ch_lo + per, nch);
        // Output staging: the whole tile [128 rows][BN] in sub-boxes of W bytes
        // ([BN/W][128][W], 16-byte granules XOR-swizzled exactly like the TMA
        // SWIZZLE_{W}B mode, so the 16-B writes of a warp are bank-conflict free).
        // The store warp (warp 2) writes it with BN/W TMA tensor stores of [128][W]
        // once the tile's epilogue warps arrived on sfull[buf]; it re-arms
        // sfree[buf] when the stores have read the buffer.
        const uint32_t W = (uint32_t)p.out_w;
        const uint32_t tile_bytes = (uint32_t)BN * kBM;
        const uint32_t swz_shift = W == 128 ? 0u : W == 64 ? 1u : 2u;
        const uint32_t swz_mask = W == 128 ? 7u : W == 64 ? 3u : W == 32 ? 1u : 0u;
        const uint32_t row_swz = (rit >> swz_shift) & swz_mask;
        uint32_t ubuf = base + L.ring;
        const bool elected = (ew == 0 && lane == 0);
        const bool grp_leader = ((ew & 7u) == 0 && lane == 0);
        const float2 inv2 = make_float2(p.inv_q, p.inv_q);
        uint32_t it = 0;

        // W is a power of two: chunk ch (16 columns = one 16-B granule) lives in
        // sub-box ch >> lg, granule ch & gm of this row
        const uint32_t lgW = 31u - (uint32_t)__clz((int)W);            // log2(W)
        const uint32_t lg = lgW - 4u, gm = (W >> 4) - 1u;
        const uint32_t row_base = rit << lgW;
        auto granule = [&](int ch) -> uint32_t {   // smem address of this row's 16-B granule of chunk ch
            const uint32_t c = (uint32_t)ch;
            return ubuf + ((c >> lg) << (lgW + 7u)) + row_base + (((c & gm) ^ row_swz) << 4);
        };

        for (uint32_t u = cid; u < (uint32_t)p.num_units; u += nclus, ++it) {
            if (kPingPong && (it & 1u) != pgrp) continue;
            const uint32_t m_tile = u / (uint32_t)p.n_groups;
            const int ng = (int)(u % (uint32_t)p.n_groups);
            const int n0 = (ng * (int)CS + (int)rank) * BN;
            const uint32_t buf = it & 1u, aph = (it >> 1) & 1u;
            const uint32_t sbuf = p.nbuf == 2 ? buf : 0u, sph = p.nbuf == 2 ? aph : (it & 1u);
            ubuf = base + L.ring + sbuf * tile_bytes;
            if (trc && elected && it < 64) trc[2048 + 16 * it + 0] = gtimer();
            mbar_wait(bar_sfree + 8u * sbuf, sph);   // staging buffer free (and residual x tile landed)
            if (trc && elected && it < 64) trc[2048 + 16 * it + 1] = gtimer();
            mbar_wait(bar_cfull + 8u * buf, aph);
            if (trc && elected && it < 64) trc[2048 + 16 * it + 8] = gtimer();
            mbar_wait(bar_tfull + 8u * buf, aph);
            if (trc && elected && it < 64) trc[2048 + 16 * it + 2] = gtimer();
            tc_fence_after();
            const int64_t row = (int64_t)m_tile * kBM + rit;
            const bool valid = row < p.M;
            const uint32_t tb = tmem_base + ((quad * 32u) << 16) + buf * (uint32_t)BN;
            const float* cm = consts + (size_t)buf * kNConst * BN;
            const float* cbias = cm + BN;
            const int32_t* czc = reinterpret_cast<const int32_t*>(cm + 2 * BN);

            // dQ (+bias) of one 16-column chunk, two columns per f32x2 op:
            // y = fl(fmaf(fl(acc - zc), m, b))  (bit-identical to the scalar form)
            auto dequant16 = [&](uint32_t (&r)[16], int cl, float2 (&y)[8]) {
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) {
                    const float4 mv = *reinterpret_cast<const float4*>(cm + cl + 4 * j4);
                    float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
                    if constexpr (HAS_B) bv = *reinterpret_cast<const float4*>(cbias + cl + 4 * j4);
                    if constexpr (HAS_ZC) {
                        const int4 zv = *reinterpret_cast<const int4*>(czc + cl + 4 * j4);
                        r[4 * j4 + 0] -= (uint32_t)zv.x; r[4 * j4 + 1] -= (uint32_t)zv.y;
                        r[4 * j4 + 2] -= (uint32_t)zv.z; r[4 * j4 + 3] -= (uint32_t)zv.w;
                    }
                    const float2 a0 = make_float2(__int2float_rn((int32_t)r[4 * j4 + 0]), __int2float_rn((int32_t)r[4 * j4 + 1]));
                    const float2 a1 = make_float2(__int2float_rn((int32_t)r[4 * j4 + 2]), __int2float_rn((int32_t)r[4 * j4 + 3]));
                    if constexpr (HAS_B) {
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
            // chunk loop with the next tcgen05.ld in flight while the current chunk is processed
            // (op #6, register-bound at 16 warps, issues one load at a time and relies
            // on its 4 warps per SMSP for latency hiding)
            auto for_chunks = [&](auto&& fn) {
                if constexpr (EPI == EP6_LN) {
                    for (int ch = ch_lo; ch < ch_hi; ++ch) {
                        uint32_t ra[16];
                        tmem_ld16(tb + (uint32_t)(ch * kChunk), ra);
                        tmem_wait_ld_dep(ra);
                        fn(ra, ch);
                    }
                    return;
                }
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
            };

            if constexpr (EPI == EP5_RELU || EPI == EP5_GELU) {
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
                        else t = f2_mul(make_float2(gelu_erf_f32(y[j].x), gelu_erf_f32(y[j].y)), inv2);
                        v[2 * j] = t.x;
                        v[2 * j + 1] = t.y;
                    }
                    uint32_t w[4];
                    quant_pack16<EPI == EP5_RELU, ZQNZ>(v, p.zq, w);
                    st_shared_v4(granule(ch), w[0], w[1], w[2], w[3]);
                });
            } else {
                // ---------------- fused op #6: dQ, bias, +residual, LayerNorm, Q ----------------
                const int C = p.ldo;
                using acc_t = typename std::conditional<STATS64, double, float>::type;
                if (!p.resid) mbar_wait(bar_xfull + 8u * buf, aph);   // residual x tile landed
                const float2 sx2 = make_float2(p.s_x, p.s_x);
                const float xoff = 8388608.0f + 128.0f + (float)p.z_x;   // exact: |z_x| <= 128
                const float2 xoff2 = make_float2(xoff, xoff);
                // pass 1: z = fl(fl(fmaf(fl(A2), m2, b2)) + r); park z in TMEM; row sum
                double s1d = 0.0;
                float2 s1f = make_float2(0.f, 0.f);
                for_chunks([&](uint32_t (&r)[16], int ch) {
                    const int cl = ch * kChunk;
                    float2 rr[8];
                    if (p.resid) {
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4) {
                            const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(p.resid + row * C + n0 + cl) + j4)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                            rr[2 * j4] = make_float2(v.x, v.y);
                            rr[2 * j4 + 1] = make_float2(v.z, v.w);
                        }
                    } else {
                        // r = fl(fl(x - z_x) * s_x); the x tile was TMA-staged in this tile's buffer
                        uint32_t xw[4];
#ifndef SWIN_EXP_NO_X
                        ld_shared_v4(granule(ch) - ubuf + base + L.xres + buf * tile_bytes, xw);
#else
                        xw[0] = xw[1] = xw[2] = xw[3] = 0x01020304u;
#endif
                        // exact int8 -> float without the 1/8-rate I2F.S8: with u = x ^ 0x80
                        // (offset binary), bits 0x4B0000uu are the float 2^23 + u, and
                        // (2^23 + u) - (2^23 + 128 + z_x) = x - z_x exactly (small integers).
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t ob = xw[q] ^ 0x80808080u;
                            const float2 f01 = make_float2(__uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7650)),
                                                           __uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7651)));
                            const float2 f23 = make_float2(__uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7652)),
                                                           __uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7653)));
                            rr[2 * q] = f2_mul(f2_sub(f01, xoff2), sx2);
                            rr[2 * q + 1] = f2_mul(f2_sub(f23, xoff2), sx2);
                        }
                    }
                    float2 z[8];
                    dequant16(r, cl, z);
                    tap_acc(r, n0 + cl);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        z[j] = f2_add(z[j], rr[j]);
                        if constexpr (STATS64) {
                            s1d = __dadd_rn(s1d, (double)z[j].x);
                            s1d = __dadd_rn(s1d, (double)z[j].y);
                        } else {
                            s1f = f2_add(s1f, z[j]);
                        }
                        r[2 * j] = __float_as_uint(z[j].x);
                        r[2 * j + 1] = __float_as_uint(z[j].y);
                    }
                    if (p.resid_out && valid) {
                        float* zrow = p.resid_out + row * (int64_t)C + n0 + cl;
#pragma unroll
                        for (int j4 = 0; j4 < 4; ++j4)
                            *reinterpret_cast<float4*>(zrow + 4 * j4) =
                                make_float4(z[2 * j4].x, z[2 * j4].y, z[2 * j4 + 1].x, z[2 * j4 + 1].y);
                    }
#ifndef SWIN_EXP_NO_STTM
                    tmem_st16(tb + (uint32_t)cl, r);
#endif
                });
                tmem_wait_st();
                if (!p.resid) {   // the x tile has been consumed: let warp 3 prefetch the next one
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_xfree + 8u * buf);
                }
                if (trc && elected && it < 64) trc[2048 + 16 * it + 3] = gtimer();

                // row statistics across the CS CTAs of the cluster (DSMEM, summed in rank order)
                // row statistics: the two column halves via smem (named barrier of the
                // group's 256 threads), the CS CTAs of the cluster via DSMEM, always
                // summed in the same order so every thread/CTA derives identical stats
                auto cluster_sum = [&](acc_t v, int pass) -> acc_t {
                    const uint32_t slot_id = pgrp * 2u + (uint32_t)pass;
                    red[(slot_id * 2u + part) * kBM + rit] = (double)v;
                    named_bar_sync(1u + pgrp, 256);
                    const acc_t t = (acc_t)red[(slot_id * 2u + 0u) * kBM + rit] + (acc_t)red[(slot_id * 2u + 1u) * kBM + rit];
                    if (CS == 1) return t;
                    const uint32_t xb = bar_x + 8u * slot_id;
                    if (part == 0) {
                        if (grp_leader) mbar_arrive_expect_tx(xb, CS * kBM * 8u);
                        const uint32_t slot = smem_u32(xbuf + ((size_t)slot_id * CS + rank) * kBM + rit);
                        for (uint32_t r = 0; r < CS; ++r) st_async_f64(mapa(slot, r), (double)t, mapa(xb, r));
                    }
                    mbar_wait_cluster(xb, (it >> 1) & 1u);
                    acc_t S = 0;
                    for (uint32_t r = 0; r < CS; ++r) S = S + (acc_t)xbuf[((size_t)slot_id * CS + r) * kBM + rit];
                    return S;
                };
                acc_t s1;
                if constexpr (STATS64) s1 = s1d; else s1 = __fadd_rn(s1f.x, s1f.y);
                const acc_t S = cluster_sum(s1, 0);
                const acc_t mu = S / (acc_t)C;
                if (trc && elected && it < 64) trc[2048 + 16 * it + 4] = gtimer();

                // pass 2: centred sum of squares
                double s2d = 0.0;
                float2 s2f = make_float2(0.f, 0.f);
                const float2 mu2 = make_float2((float)mu, (float)mu);
                for_chunks([&](uint32_t (&r)[16], int) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float2 zz = make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
                        if constexpr (STATS64) {
                            const double d0 = __dsub_rn((double)zz.x, (double)mu), d1 = __dsub_rn((double)zz.y, (double)mu);
                            s2d = __dadd_rn(s2d, __dmul_rn(d0, d0));
                            s2d = __dadd_rn(s2d, __dmul_rn(d1, d1));
                        } else {
                            const float2 dz = f2_sub(zz, mu2);
                            s2f = f2_fma(dz, dz, s2f);
                        }
                    }
                });
                acc_t s2;
                if constexpr (STATS64) s2 = s2d; else s2 = __fadd_rn(s2f.x, s2f.y);
                const acc_t SS = cluster_sum(s2, 1);
                acc_t rstd;
                if constexpr (STATS64) rstd = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(SS, (double)C), (double)p.eps)));
                else rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(SS, (float)C), p.eps)));
                const float2 rstd2 = make_float2((float)rstd, (float)rstd);
                if (trc && elected && it < 64) trc[2048 + 16 * it + 5] = gtimer();

                // pass 3: yhat = fl(((z-mu)*rstd)*gamma + beta); Y = Q_y(yhat), staged over x in place
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
                                const double xh = __dmul_rn(__dsub_rn((double)__uint_as_float(r[4 * j4 + j]), mu), rstd);
                                yh[4 * j4 + j] = __double2float_rn(__dadd_rn(__dmul_rn(xh, (double)gg[j]), (double)bb[j]));
                            }
                        } else {
                            const float2 z0 = make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]));
                            const float2 z1 = make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3]));
                            const float2 y0 = f2_fma(f2_mul(f2_sub(z0, mu2), rstd2), make_float2(gv.x, gv.y), make_float2(bv.x, bv.y));
                            const float2 y1 = f2_fma(f2_mul(f2_sub(z1, mu2), rstd2), make_float2(gv.z, gv.w), make_float2(bv.z, bv.w));
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
                    st_shared_v4(granule(ch), w[0], w[1], w[2], w[3]);
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
                mbar_arrive(bar_tempty + 8u * buf);   // TMEM free: next MMA may start
                mbar_arrive(bar_sfull + 8u * sbuf);   // this warp's part of the tile is staged
            }
            if (trc && elected && it < 64) trc[2048 + 16 * it + 7] = gtimer();
        }
    }

    // teardown: no CTA leaves while a peer may still address its shared memory
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, tmem_cols);
    }
}

}  // namespace swinmlp
