// small_mlp.cuh — the whole MLP sub-layer in ONE launch for runs of at most 64 tokens
// (BASELINE configs[0]: one 7x7 window, T = 49), two-kernel channel widths (C >= 384).
//
// At T <= 64 the layer is a chain of latencies, not of bandwidth: the
// two-kernel plan pays two launches, the programmatic-dependent hand-off, FC2's K = 4C on a
// few SMs and a one-tile LayerNorm.  Here the hidden dimension is split over P = H / 128 CTAs
// (one per SM, all co-resident), in clusters of Q CTAs (S = P / Q slices of Q * 128 hidden
// columns), and nothing but int32 FC2 partials leaves the cluster:
//
//   CTA j = Q s + g (cluster s, rank g):
//           acc1_j = X . W1[128 j .. 128 j + 127]^T            (tcgen05, TMEM cols [0, 128))
//           Hq_j   = op #5(acc1_j)                              (smem slot g of the cluster's Hq
//                    tile, SW128 K-major; bulk-copied into slot g of the Q - 1 peers: DSMEM)
//           part   = Hq_s . W2[g PR .. g PR + PR - 1, slice s]^T (tcgen05, PR = C / Q columns,
//                    K = Q * 128), staged in smem and bulk-reduce-added (cp.reduce.async.bulk
//                    .add.s32) into acc[T][C]: S-way sums instead of P-way ones
//   all:    arrival counter == P (release / acquire at gpu scope)
//           rows r = j, j + P, ...: A2 = acc[r] - z_h wsum2 (int32 sums: exact in any order),
//           then op #6 (dQ, bias, residual, LayerNorm, Q) with the row in registers of one
//           warp; the row of acc is zeroed again after it is read, and the last CTA to leave
//           resets the counters: acc and the counters are all zero between runs (handle-owned,
//           so runs of one handle must be stream-ordered).
// The L2's reduction throughput (≈ 0.65 TB/s for these many-way int32 sums) set the pace of the
// P-way version (3.6 MB at C = 768, T = 49); the cluster split divides those bytes by Q.
//
// Same arithmetic as the other plans: A1, Hq, A2 and z bit-exact; the LayerNorm statistics
// are the fp32 two-pass of the row held by one warp (Y within the R15 tier).
//
// Weights never wait on the previous kernel: the producer issues the W1 K-blocks of the
// first ring slots before griddepcontrol.wait and only the X boxes after it.
//
// CTA = 320 threads: warp 0 TMA producer, warp 1 MMA issuer (and TMEM allocator),
// warps 2-9 epilogue (two per TMEM lane quadrant, column halves; quadrants 2-3 hold rows
// 64-127 of the M = 128 tiles, which carry no tokens).
#pragma once
#include "mlp_kernels.cuh"

namespace swinmlp {

constexpr int kSThreads = 32 * 10;
constexpr int kSMaxT = 64;
constexpr int kSStages = 4;
constexpr int kSMaxQ = 8;                          // cluster size (portable maximum)
constexpr uint32_t kSSlot = 32768;                 // FC1 {A 16 KB (64 rows loaded), B 16 KB} | W2 K-block
// C <= 768 (at most 6 K-blocks): FC1's operands resident at once, each landed by ONE 3-D TMA op
// (the per-op cost of the TMA unit, not the bytes, paces small boxes):
//   A  [K-blocks][64 rows][128 B] at 8 KB steps (+ 8 KB: the M = 128 MMA's rows 64-127 of a K-block
//      are the next one's rows, TMEM lanes without tokens)            base .. base + 56 KB
//   W1 [K-blocks][128 rows][128 B]                                    base + 56 KB .. base + 152 KB
// and after FC1 the cluster slice's W2 K-blocks [Q][PR rows][128 B] (C * 128 bytes) over W1, again
// one op.
constexpr int kSResKB = 6;
constexpr uint32_t kSResW1 = 57344;
constexpr uint32_t kSHq = kSResW1 + kSResKB * 16384;   // Hq: Q K-blocks of [64 rows][128 B] SW128, 8 KB apart
                                                   // (+ 8 KB: the M = 128 MMA's rows 64-127 of the last one,
                                                   // which land in TMEM lanes that carry no tokens)
constexpr uint32_t kSHqSlot = 8192;
constexpr uint32_t kSStageRow = 256 * 4 + 16;      // one int32 partial row (+16 B: bank shift)
constexpr uint32_t kSStage = 0;                    // [64 rows][kSStageRow] partial staging, over the
                                                   // operand ring (free once FC2's MMAs completed)
constexpr uint32_t kSConst = kSHq + (kSMaxQ + 1) * kSHqSlot;   // m1, b1, zc1 of the CTA's 128 columns
constexpr uint32_t kSBars = kSConst + 3 * 128 * 4;
constexpr uint32_t kSSmem = kSBars + 256 + 1024;   // + barriers/TMEM slot + alignment slack

struct SmallArgs {
    int32_t T, C, H, P;    // tokens (<= 64), channels, hidden, CTAs (= H / 128)
    int32_t Q, PR;         // cluster size (P % Q == 0) and FC2 columns per CTA (Q * PR == C, PR <= 256,
                           // PR % 32 == 0)
    int32_t act;           // 0 ReLU, 1 GELU (exact erf)
    const float* m1; const float* b1; const int32_t* zc1;   // [H]
    const float* m2; const float* b2; const int32_t* zc2;   // [C]
    const float* gamma; const float* beta;
    float inv_h; int32_t z_h; float inv_y; int32_t z_y; float s_x; int32_t z_x; float eps;
    const int8_t* x; int8_t* y; const float* resid; float* resid_out;
    int32_t* acc;          // [64][C] int32 FC2 sums (handle-owned; 0 between runs)
    int32_t* cnt;          // [2] arrival / departure counters (handle-owned; 0 between runs)
    int32_t* acc1_tap; int8_t* hid_tap; int32_t* acc2_tap; float* ln_tap;   // debug (rows < T)
    unsigned long long* trace;   // debug: per CTA 16 %globaltimer stamps (swin_mlp_int8_set_trace)
};

__device__ __forceinline__ float s_warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// G = C / 128: the float4 groups of a LayerNorm row per lane
template <int G, int ACT>
__global__ void __launch_bounds__(kSThreads, 1)
small_mlp_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                 const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ SmallArgs p) {
    // (resident mode, G <= kSResKB: tmX / tmW1 / tmW2 are the 3-D maps {128 B, rows, K-blocks})
    using namespace sm100;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t j = blockIdx.x;
    constexpr bool RES = G <= kSResKB;   // (G = C / 128 = FC1's K-blocks)
    const uint32_t bar_full = base + kSBars, bar_empty = bar_full + 8u * 8u;   // [8] FC1 K-block / ring slot
    const uint32_t bar_acc1 = bar_empty + 8u * kSStages, bar_hq = bar_acc1 + 8u;
    const uint32_t bar_tfull = bar_hq + 8u, bar_peer = bar_tfull + 8u;   // FC2 done; [Q] slot kk landed
    const uint32_t bar_w2 = bar_peer + 8u * kSMaxQ;                     // [Q] resident mode: W2 K-block i landed
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (base - raw) + kSBars + 248);
    const int C = p.C, NKB = (C + kBK - 1) / kBK;
    const uint32_t Q = (uint32_t)p.Q, g = Q > 1 ? cluster_ctarank() : 0u, s_slice = j / Q;
    unsigned long long* trc = p.trace ? p.trace + 16 * blockIdx.x : nullptr;
    if (trc && threadIdx.x == 0) trc[0] = gtimer();

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmW1);
        tma_prefetch_desc(&tmW2);
    }
    if (warp == 1) {
        if (lane == 0) {
            for (int s = 0; s < 8; ++s) {
                mbar_init(bar_full + 8u * s, 1);
                mbar_init(bar_w2 + 8u * s, 1);
                if (s < kSStages) mbar_init(bar_empty + 8u * s, 1);
            }
            mbar_init(bar_acc1, 1);
            mbar_init(bar_hq, 8);
            mbar_init(bar_tfull, 1);
            for (uint32_t r = 0; r < Q; ++r) {   // one barrier per peer's Hq slot
                if (r == g) continue;
                mbar_init(bar_peer + 8u * r, 1);
                mbar_arrive_expect_tx(bar_peer + 8u * r, kSHqSlot);
            }
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc(smem_u32(const_cast<uint32_t*>(tmem_slot)), 512);
    }
    tc_fence_before();
    if (Q > 1) cluster_sync_all();   // every peer's barriers exist before any copy signals them
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (trc && threadIdx.x == 0) trc[1] = gtimer();
    pdl_launch_dependents();   // (all P CTAs are resident by now: the next kernel cannot starve them)

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (RES && elect_one()) {
            // the W1 slice before the wait (a constant), X after it; one op each
            mbar_arrive_expect_tx(bar_full, (uint32_t)NKB * 128u * kBK);
            tma_load_3d(&tmW1, base + kSResW1, bar_full, 0, (int)(j * 128), 0);
            pdl_wait();   // X: the previous kernel's output
            if (trc) trc[2] = gtimer();
            mbar_arrive_expect_tx(bar_full + 8u, (uint32_t)NKB * 64u * kBK);
            tma_load_3d(&tmX, base, bar_full + 8u, 0, 0, 0);
            mbar_wait(bar_acc1, 0);   // FC1's MMAs have read W1: the slice's W2 K-blocks replace it
            mbar_arrive_expect_tx(bar_w2, (uint32_t)C * kBK);
            tma_load_3d(&tmW2, base + kSResW1, bar_w2, 0, (int)g * p.PR, (int)(s_slice * Q));
        } else if (!RES && elect_one()) {
            const int n_pre = NKB < kSStages ? NKB : kSStages;
            // W1 K-blocks of the first slots: constants, issued before the wait on the previous kernel
            for (int kb = 0; kb < n_pre; ++kb) {
                const uint32_t slot = base + (uint32_t)kb * kSSlot;
                mbar_arrive_expect_tx(bar_full + 8u * kb, 64u * kBK + 128u * kBK);
                tma_load_2d(&tmW1, slot + 16384u, bar_full + 8u * kb, kb * kBK, (int)(j * 128));
            }
            pdl_wait();   // X: the previous kernel's output
            if (trc) trc[2] = gtimer();
            for (int kb = 0; kb < n_pre; ++kb)
                tma_load_2d(&tmX, base + (uint32_t)kb * kSSlot, bar_full + 8u * kb, kb * kBK, 0);
            int s = n_pre % kSStages;
            uint32_t ph = n_pre == kSStages ? 1u : 0u;
            for (int kb = n_pre; kb < NKB; ++kb) {
                mbar_wait(bar_empty + 8u * s, ph ^ 1u);
                const uint32_t slot = base + (uint32_t)s * kSSlot;
                mbar_arrive_expect_tx(bar_full + 8u * s, 64u * kBK + 128u * kBK);
                tma_load_2d(&tmW1, slot + 16384u, bar_full + 8u * s, kb * kBK, (int)(j * 128));
                tma_load_2d(&tmX, slot, bar_full + 8u * s, kb * kBK, 0);
                if (++s == kSStages) { s = 0; ph ^= 1u; }
            }
            // FC2: the W2 K-blocks [PR rows of group g][128 hidden columns] of the cluster's slice
            for (uint32_t i = 0; i < Q; ++i) {   // the MMA's order: own slot first, then the peers'
                const uint32_t kk = (g + i) % Q;
                mbar_wait(bar_empty + 8u * s, ph ^ 1u);
                mbar_arrive_expect_tx(bar_full + 8u * s, (uint32_t)p.PR * kBK);
                tma_load_2d(&tmW2, base + (uint32_t)s * kSSlot, bar_full + 8u * s, (int)((s_slice * Q + kk) * 128),
                            (int)g * p.PR);
                if (++s == kSStages) { s = 0; ph ^= 1u; }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ============================ MMA issuer ==============================
        int s = 0;
        uint32_t ph = 0;
        const uint32_t id1 = idesc_i8(kBM, 128), id2 = idesc_i8(kBM, (uint32_t)p.PR);
        if constexpr (RES) {
            mbar_wait(bar_full, 0);        // W1
            mbar_wait(bar_full + 8u, 0);   // X
            tc_fence_after();
            for (int kb = 0; kb < NKB; ++kb) {
                const uint32_t xa = base + (uint32_t)kb * 8192u, wb = base + kSResW1 + (uint32_t)kb * 16384u;
                const int rem = C - kb * kBK, nk = rem >= kBK ? 4 : rem / 32;
                if (elect_one()) {
                    for (int k = 0; k < nk; ++k)
                        mma_i8(tmem, umma_desc_k128(xa) + 2u * k, umma_desc_k128(wb) + 2u * k, id1, (kb | k) != 0);
                    if (kb == NKB - 1) mma_commit(bar_acc1);
                }
                __syncwarp();
            }
        }
        for (int kb = 0; kb < (RES ? 0 : NKB); ++kb) {
            mbar_wait(bar_full + 8u * s, ph);
            tc_fence_after();
            const uint32_t slot = base + (uint32_t)s * kSSlot;
            const int rem = C - kb * kBK, nk = rem >= kBK ? 4 : rem / 32;
            if (elect_one()) {
                for (int k = 0; k < nk; ++k)
                    mma_i8(tmem, umma_desc_k128(slot) + 2u * k, umma_desc_k128(slot + 16384u) + 2u * k, id1,
                           (kb | k) != 0);
                mma_commit(bar_empty + 8u * s);
                if (kb == NKB - 1) mma_commit(bar_acc1);
            }
            __syncwarp();
            if (++s == kSStages) { s = 0; ph ^= 1u; }
        }
        mbar_wait(bar_hq, 0);                // this CTA's Hq slot staged
        tc_fence_after();
        if (trc && lane == 0) trc[4] = gtimer();
        for (uint32_t i = 0; i < Q; ++i) {   // K = Q * 128: own slot, then each peer's as it lands
            const uint32_t kk = (g + i) % Q;
            if (i > 0) mbar_wait(bar_peer + 8u * kk, 0);   // (DSMEM bulk copy from peer kk)
            if constexpr (RES) mbar_wait(bar_w2, 0);
            else mbar_wait(bar_full + 8u * s, ph);
            tc_fence_after();
            const uint32_t slot = RES ? base + kSResW1 + kk * (uint32_t)p.PR * kBK : base + (uint32_t)s * kSSlot;
            if (elect_one()) {
                for (int k = 0; k < 4; ++k)
                    mma_i8(tmem + 256u, umma_desc_k128(base + kSHq + kk * kSHqSlot) + 2u * k,
                           umma_desc_k128(slot) + 2u * k, id2, (i | (uint32_t)k) != 0u);
                if (!RES) mma_commit(bar_empty + 8u * s);
                if (i + 1u == Q) mma_commit(bar_tfull);
            }
            __syncwarp();
            if (!RES && ++s == kSStages) { s = 0; ph ^= 1u; }
        }
    } else {
        // ============================ epilogue ================================
        const uint32_t ew = warp - 2, quad = warp & 3u, half = ew >> 2;
        const uint32_t row = quad * 32u + lane;          // TMEM lane = token row of the tile
        const bool live = quad < 2;                      // rows 0-63 (token rows < T among them)
        const bool valid = (int)row < p.T;
        pdl_wait();   // partials / counters / outputs: the previous kernel must be done with them
        // ---- the CTA's 128 columns of m1 / b1 / zc1 -> smem (quadrant 2-3 warps: no token rows)
        float* cm = reinterpret_cast<float*>(smem_raw + (base - raw) + kSConst);
        if (!live) {
            const uint32_t t = ((ew & 1u) + 2u * (ew >> 2)) * 32u + lane;   // ew 0, 1, 4, 5 -> 0..127
            cm[t] = __ldg(p.m1 + j * 128 + t);
            cm[128 + t] = p.b1 ? __ldg(p.b1 + j * 128 + t) : 0.0f;
            cm[256 + t] = p.zc1 ? __int_as_float(__ldg(p.zc1 + j * 128 + t)) : 0.0f;
        }
        named_bar_sync(2, 256);
        // ---- op #5: acc1 (128 hidden columns) -> Hq tile (SW128 K-major, FC2's A operand)
        mbar_wait(bar_acc1, 0);
        tc_fence_after();
        if (trc && ew == 0 && lane == 0) trc[3] = gtimer();
        if (live) {
            const uint32_t hrow = base + kSHq + g * kSHqSlot + row * 128u;   // slot g, rows 0-63
            uint32_t r[4][16];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)   // this warp's 64 columns in one round trip
                tmem_ld16(tmem + ((quad * 32u) << 16) + (uint32_t)((half * 4 + c4) * 16), r[c4]);
            tmem_wait_ld();
            if (trc && ew == 0 && lane == 0) trc[10] = gtimer();
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                reg_fence16(r[c4]);
                const int ch = (int)half * 4 + c4, cl = ch * 16, n0 = (int)j * 128 + cl;
                float v[16];
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) {   // four columns per 16-B constant load
                    const float4 mv = *reinterpret_cast<const float4*>(cm + cl + 4 * e4);
                    const float4 bv = *reinterpret_cast<const float4*>(cm + 128 + cl + 4 * e4);
                    const int4 zv = *reinterpret_cast<const int4*>(cm + 256 + cl + 4 * e4);
                    const int32_t a[4] = {(int32_t)r[c4][4 * e4] - zv.x, (int32_t)r[c4][4 * e4 + 1] - zv.y,
                                          (int32_t)r[c4][4 * e4 + 2] - zv.z, (int32_t)r[c4][4 * e4 + 3] - zv.w};
                    if (p.acc1_tap && valid)
                        *reinterpret_cast<int4*>(p.acc1_tap + (int64_t)row * p.H + n0 + 4 * e4) = make_int4(a[0], a[1], a[2], a[3]);
                    float2 y0 = f2_fma(make_float2(__int2float_rn(a[0]), __int2float_rn(a[1])), make_float2(mv.x, mv.y),
                                       make_float2(bv.x, bv.y));
                    float2 y1 = f2_fma(make_float2(__int2float_rn(a[2]), __int2float_rn(a[3])), make_float2(mv.z, mv.w),
                                       make_float2(bv.z, bv.w));
                    if (ACT) {
                        y0 = make_float2(gelu_erf_f32(y0.x), gelu_erf_f32(y0.y));
                        y1 = make_float2(gelu_erf_f32(y1.x), gelu_erf_f32(y1.y));
                    }
                    const float2 ih = make_float2(p.inv_h, p.inv_h);   // (ReLU: the max folds into Q)
                    const float2 t0 = f2_mul(y0, ih), t1 = f2_mul(y1, ih);
                    v[4 * e4] = t0.x; v[4 * e4 + 1] = t0.y; v[4 * e4 + 2] = t1.x; v[4 * e4 + 3] = t1.y;
                }
                uint32_t w[4];
                if (ACT) {
                    if (p.z_h) quant_pack16<false, true>(v, p.z_h, w);
                    else quant_pack16<false, false>(v, p.z_h, w);
                } else {
                    if (p.z_h) quant_pack16<true, true>(v, p.z_h, w);
                    else quant_pack16<true, false>(v, p.z_h, w);
                }
                st_shared_v4(hrow + ((((uint32_t)ch) ^ (row & 7u)) << 4), w[0], w[1], w[2], w[3]);
                if (p.hid_tap && valid)
                    *reinterpret_cast<int4*>(p.hid_tap + (int64_t)row * p.H + n0) =
                        make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
            }
        }
        if (trc && ew == 0 && lane == 0) trc[11] = gtimer();
        fence_proxy_async_smem();   // Hq visible to the tensor core and the bulk copies (async proxy)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_hq);
        if (Q > 1) {   // the slot to the Q - 1 peers (rows 0-63; their MMA waits on bar_peer)
            named_bar_sync(2, 256);
            if (ew == 0 && lane == 0) {
                const uint32_t src = base + kSHq + g * kSHqSlot;
                for (uint32_t r = 1; r < Q; ++r) {
                    const uint32_t peer = (g + r) % Q;
                    bulk_copy_s2cluster(mapa(src, peer), src, kSHqSlot, mapa(bar_peer + 8u * g, peer));
                }
            }
        }
        // ---- FC2: TMEM -> smem staging -> bulk reduce-add into acc[rows < T][g PR .. g PR + PR)
        const int hc = p.PR / 2;   // columns per warp half
        const uint32_t srow = base + kSStage + row * kSStageRow;
        mbar_wait(bar_tfull, 0);
        tc_fence_after();
        if (live) {
            uint32_t r[8][16];   // the warp half's <= 128 columns, one round trip
            const int nch = hc / 16;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < nch) tmem_ld16(tmem + ((quad * 32u) << 16) + 256u + (uint32_t)((int)half * hc + 16 * k), r[k]);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k >= nch) break;
                reg_fence16(r[k]);
                const int c0 = (int)half * hc + 16 * k;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    st_shared_v4(srow + (uint32_t)(c0 + 4 * q) * 4u, r[k][4 * q], r[k][4 * q + 1], r[k][4 * q + 2],
                                 r[k][4 * q + 3]);
            }
            fence_proxy_async_smem();
            if (valid) {
                bulk_reduce_add_s32(p.acc + (int64_t)row * C + (int)g * p.PR + (int)half * hc,
                                    srow + (uint32_t)((int)half * hc) * 4u, (uint32_t)hc * 4u);
                bulk_commit();
            }
        }
        if (trc && ew == 0 && lane == 0) trc[6] = gtimer();
        if (live && valid) {
            bulk_wait_all();             // this thread's reduce-adds have been performed
            fence_proxy_async_global();  // ... and are ordered before its generic-proxy release below
        }
        __threadfence();
        named_bar_sync(1, 256);
        if (ew == 0 && lane == 0) red_release_gpu_add(p.cnt, 1);
        if (trc && ew == 0 && lane == 0) trc[5] = gtimer();
        // ---- op #6 for rows j, j + P, ... (one warp per row; the row's C values in registers)
        const int r = (int)j + (int)ew * p.P;
        if (r < p.T) {
            if (lane == 0)
                while (ld_acquire_gpu(p.cnt) < p.P) __nanosleep(32);
            __syncwarp();
            (void)ld_acquire_gpu(p.cnt);
            if (trc && lane == 0 && ew == 0) trc[9] = gtimer();
            // all of the row's loads first (one round trip), then the arithmetic
            int4 a4[G];
            uint32_t xw[G];
            float4 m4[G], b4[G], r4[G];
            constexpr bool PRE = G <= 8;   // gamma / beta in the same round trip (register budget)
            float4 g4[PRE ? G : 1], t4[PRE ? G : 1];
#pragma unroll
            for (int v = 0; v < G; ++v) {
                const int c = 4 * (int)lane + 128 * v;
                a4[v] = __ldcg(reinterpret_cast<const int4*>(p.acc + (int64_t)r * C + c));   // the P partials' exact sum
                m4[v] = __ldg(reinterpret_cast<const float4*>(p.m2 + c));
                b4[v] = p.b2 ? __ldg(reinterpret_cast<const float4*>(p.b2 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (p.resid) r4[v] = __ldg(reinterpret_cast<const float4*>(p.resid + (int64_t)r * C + c));
                else xw[v] = __ldg(reinterpret_cast<const uint32_t*>(p.x + (int64_t)r * C + c));
                if constexpr (PRE) {
                    g4[v] = __ldg(reinterpret_cast<const float4*>(p.gamma + c));
                    t4[v] = __ldg(reinterpret_cast<const float4*>(p.beta + c));
                }
            }
#pragma unroll
            for (int v = 0; v < G; ++v)   // zero again for the next run
                __stcg(reinterpret_cast<int4*>(p.acc + (int64_t)r * C + 4 * (int)lane + 128 * v), make_int4(0, 0, 0, 0));
            float z[G][4];
            float s = 0.f;
#pragma unroll
            for (int v = 0; v < G; ++v) {
                const int c = 4 * (int)lane + 128 * v;
                int4 a = a4[v];
                if (p.zc2) {
                    const int4 zc = __ldg(reinterpret_cast<const int4*>(p.zc2 + c));
                    a.x -= zc.x; a.y -= zc.y; a.z -= zc.z; a.w -= zc.w;
                }
                if (p.acc2_tap) *reinterpret_cast<int4*>(p.acc2_tap + (int64_t)r * C + c) = a;
                const int ai[4] = {a.x, a.y, a.z, a.w};
                const float mm[4] = {m4[v].x, m4[v].y, m4[v].z, m4[v].w}, bb[4] = {b4[v].x, b4[v].y, b4[v].z, b4[v].w};
                float rr[4];
                if (p.resid) {
                    rr[0] = r4[v].x; rr[1] = r4[v].y; rr[2] = r4[v].z; rr[3] = r4[v].w;
                } else {   // dQ(x) = fl(fl(x - z_x) * s_x), then the Add (reading R3)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        rr[e] = __fmul_rn((float)((int)(int8_t)(xw[v] >> (8 * e)) - p.z_x), p.s_x);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float d = __fmaf_rn(__int2float_rn(ai[e]), mm[e], bb[e]);
                    z[v][e] = __fadd_rn(d, rr[e]);
                    s = __fadd_rn(s, z[v][e]);
                }
                if (p.resid_out)
                    *reinterpret_cast<float4*>(p.resid_out + (int64_t)r * C + c) = make_float4(z[v][0], z[v][1], z[v][2], z[v][3]);
            }
            const float Cf = (float)C;
            const float mu = __fdiv_rn(s_warp_sum(s), Cf);
            float ss = 0.f;
#pragma unroll
            for (int v = 0; v < G; ++v) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float dz = __fsub_rn(z[v][e], mu);
                    ss = __fmaf_rn(dz, dz, ss);
                }
            }
            const float var = __fdiv_rn(s_warp_sum(ss), Cf);
            const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
#pragma unroll
            for (int v = 0; v < G; ++v) {
                const int c = 4 * (int)lane + 128 * v;
                float4 gv, bv;
                if constexpr (PRE) {
                    gv = g4[PRE ? v : 0]; bv = t4[PRE ? v : 0];
                } else {
                    gv = __ldg(reinterpret_cast<const float4*>(p.gamma + c));
                    bv = __ldg(reinterpret_cast<const float4*>(p.beta + c));
                }
                const float gg[4] = {gv.x, gv.y, gv.z, gv.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
                float yh[4];
                int q[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    yh[e] = __fmaf_rn(__fmul_rn(__fsub_rn(z[v][e], mu), rstd), gg[e], bb[e]);
                    const float t = __fmul_rn(yh[e], p.inv_y);
                    q[e] = __float2int_rn(fminf(fmaxf(t, -1024.f), 1024.f)) + p.z_y;
                }
                if (p.ln_tap)
                    *reinterpret_cast<float4*>(p.ln_tap + (int64_t)r * C + c) = make_float4(yh[0], yh[1], yh[2], yh[3]);
                *reinterpret_cast<uint32_t*>(p.y + (int64_t)r * C + c) = pack_sat_s8(q[1], q[0], pack_sat_s8(q[3], q[2], 0u));
            }
        }
        // ---- departure: the last CTA out resets the counters for the next run
        named_bar_sync(1, 256);
        if (ew == 0 && lane == 0) {
            __threadfence();
            const int old = atomicAdd(p.cnt + 1, 1);
            if (old == p.P - 1) {
                atomicExch(p.cnt, 0);
                atomicExch(p.cnt + 1, 0);
            }
        }
    }
    if (trc && warp == 2 && lane == 0) trc[14] = gtimer();
    tc_fence_before();
    if (Q > 1) cluster_sync_all();   // no CTA leaves while a peer's copy may still read its Hq slot
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
    if (trc && threadIdx.x == 0) trc[15] = gtimer();
}

}  // namespace swinmlp
