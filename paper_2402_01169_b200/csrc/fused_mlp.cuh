// fused_mlp.cuh — the whole MLP sub-layer in ONE sm_100a kernel for C <= 384:
// FC1 -> op #5 -> FC2 -> op #6 per 128-token tile, with the hidden activation
// Hq never leaving the SM.
//
// The paper fuses each elementwise op into the GEMM that produces its input
// and still round-trips every GEMM output through global
// memory; on B200 the 4C-wide int8 hidden tile of a 128-token tile is at most
// 128 KB, so it can live in shared memory and feed FC2 directly:
//
//   for each hidden chunk j of 128 columns (H = 128 * NJ):
//       acc1_j  = X_tile . W1[j]^T                   (tcgen05, TMEM buffer j % NB1)
//       Hq_j    = op #5(acc1_j)                      (epilogue warps -> smem, SW128 K-major:
//                                                     exactly FC2's A-operand layout)
//       acc2   += Hq_j . W2[:, j]^T                  (tcgen05, TMEM columns [0, C))
//   Y_tile = op #6(acc2, X_tile)                     (LayerNorm rows on chip; Y staged in
//                                                     smem, then TMA-stored)
//
// Same arithmetic, in the same order, as the two-kernel path (mlp_kernels.cuh) and
// the oracle; HBM traffic falls to the algorithmic 2C bytes per token (X in, Y out).
//
// CTA = 640 threads, one per SM, persistent over m-tiles cid, cid + grid, ...:
//   warp 0       TMA producer: X tiles (2 slots) and, unless resident, the W1 / W2
//                chunks through a `stages`-deep ring in the MMA's consumption order
//   warp 1       FC1 MMA issuer
//   warp 3       loads the per-channel constants once, then issues the FC2 MMAs
//   warp 2       TMEM allocator, then the Y store warp
//   warps 4-11   op #5: warp = (lane quadrant, 64-column half) of each acc1 chunk
//   warps 12-19  op #6: warp = (lane quadrant, column half); a thread owns half a
//                token row, the two halves combine their statistics pairwise
#pragma once
#include "mlp_kernels.cuh"

namespace swinmlp {

constexpr int kFEp5W0 = 4, kFEp6W0 = 12;
constexpr int kFThreads = 32 * 20;          // 4 control + 8 op #5 + 8 op #6 warps (96 regs each; a 21st
                                            // warp would cost 16 registers per thread: measured slower)
constexpr int kFHc = 128;                    // hidden chunk = one 128-B K-block of FC2
constexpr int kFMaxNB1 = 3, kFMaxNH = 4, kFMaxStages = 8;
constexpr uint32_t kKB = (uint32_t)kBM * kBK;   // one [128 rows][128 B] box
// flags
constexpr int kFGelu = 1, kFZh = 2, kFB1 = 4, kFS64 = 8, kFSmallK = 16, kFTaps = 32;
constexpr int kFReg = 64;   // op #6 register path (C <= 32 * kFRegCh; not with kFS64 / kFTaps)
// CTA pair (cta_group::2): two CTAs of a cluster take m-tiles 2u and 2u + 1; the leader
// issues M = 256 MMAs whose B operand (the weight chunk) is split between the two CTAs'
// shared memory, so each SM streams half of every weight chunk (streamed weights only)
constexpr int kFPair = 128;
constexpr int kFNumVariants = 96;   // flags 0..95 (kFReg only without kFTaps), and 128..191 (kFPair)

struct FusedArgs {
    int64_t M;          // tokens
    int32_t C, H;
    int32_t NJ;         // H / 128 hidden chunks
    int32_t KBC;        // ceil(C / 128): K-blocks of the X tile and of a W1 chunk
    int32_t NB1;        // acc1 TMEM buffers (128 columns each)
    int32_t NH;         // Hq smem buffers
    int32_t stages;     // W1 ring depth (16 KB K-block items); 0 = W1 and W2 resident in smem
    int32_t stages2;    // W2 ring depth, streamed mode: items of [C rows][128 B] (one per chunk),
                        // or of [C/2 rows][128 B] when C > 256 (two per chunk, one per FC2 MMA half)
    int32_t a1_col;     // TMEM column of acc1 buffer 0 (acc2 buffers live below it)
    int32_t NA2;        // acc2 TMEM buffers (2: op #6 of tile i overlaps FC2 of tile i + 1)
    int32_t NX;         // X tile slots (2..4)
    int32_t y_inplace;  // 1: Y is staged over its tile's X slot (no separate Y buffer; the
                        //    slot is released by the Y store) -- frees smem for the weight ring
    int32_t a2_stride;  // TMEM columns between acc2 buffers
    const float* m1; const float* b1; const int32_t* zc1;   // [H]
    const float* m2; const float* b2; const int32_t* zc2;   // [C]
    const float* gamma; const float* beta;                  // [C]
    float inv_h; int32_t z_h;
    float inv_y; int32_t z_y;
    float s_x; int32_t z_x; float eps;
    float one;                                              // 1.0f (host-set), see GemmArgs::one
    const int8_t* x;                                        // [M][C] layer input (op #6 residual dQ(x))
    const float* resid; float* resid_out;                   // [M][C] fp32 or nullptr
    int32_t* acc1_tap; int8_t* hid_tap; int32_t* acc2_tap; float* ln_tap;   // debug taps
    // pipeline trace (debug): CTA trace_cta stamps %globaltimer into trace[8192]:
    // [q] FC1(q) issued, [512+u] FC2(u) issued, [1024+q] / [1536+q] FC1(q) before /
    // after its waits, [2048+2u+{0,1}] op #5 chunk u start / end, [4096+4i+{0..3}] op #6
    // tile i start / stats done / pass 1 done / end, [6144+i] Y tile i stored (reads
    // done), [6656+u] / [7168+u] FC2(u) before / after its waits
    unsigned long long* trace;
    int32_t trace_cta;
    unsigned long long* cta_stamps;   // debug: per CTA %globaltimer at entry / exit ([2 * blockIdx.x + {0,1}])
    int32_t rotate;                   // 1: per-CTA rotated hidden-chunk order (A/B switch SWIN_MLP_FUSED_ROT)
};

struct FusedLayout {
    uint32_t x, y, hq, w, w2, consts, red, bars, tmem_slot, total;
};
constexpr int kFMaxNX = 4;
// op #6 holds a thread's whole half row in registers when it has at most this many
// 16-column chunks (C <= 128): acc2 is released right after its TMEM loads and z is
// never parked back in TMEM (no tcgen05.st / second tcgen05.ld per value)
constexpr int kFRegCh = 3;
constexpr int kFMaxStages2 = 4;
constexpr uint32_t kFNumBars = 4 + 4 + 2 * kFMaxStages + 2 * kFMaxStages2 + 1 + 2 * kFMaxNB1 + 2 * kFMaxNH + 4 + 2 + 1 + 1 +
                               kFMaxNX;   // + pair: peer X landed

// Streamed ring items: W1 = one [128 (pair: 64) rows][128 B] K-block box; W2 = [rows][128 B]
// with rows = C (C > 256: C/2, one item per FC2 MMA half), halved in a CTA pair.
__host__ __device__ inline uint32_t fused_w1_item(int pair) { return (uint32_t)kBM * kBK >> (pair ? 1 : 0); }
__host__ __device__ inline uint32_t fused_w2_rows(int C, int pair) {
    return (uint32_t)(C > 256 ? C / 2 : C) >> (pair ? 1 : 0);
}
__host__ __device__ inline FusedLayout fused_layout(int C, int H, int NH, int stages, int ebytes, int NX,
                                                    int y_inplace = 0, int stages2 = 0, int pair = 0) {
    FusedLayout L;
    const uint32_t kbc = (uint32_t)((C + kBK - 1) / kBK), nj = (uint32_t)(H / kFHc);
    L.x = 0;                                             // [NX][KBC][128 rows][128 B] X tiles
    L.y = L.x + (uint32_t)NX * kbc * kKB;                // [KBC][128 rows][128 B] Y staging
    L.hq = L.y + (y_inplace ? 0u : kbc * kKB);           // [NH][128 rows][128 B]
    L.w = L.hq + (uint32_t)NH * kKB;                     // resident: W1 chunks then W2 chunks; else ring
    if (stages == 0) {
        L.w2 = L.w + nj * kbc * kKB;
        L.consts = L.w2 + nj * (uint32_t)C * kBK;
    } else {   // two rings: W1 K-blocks, W2 chunks (each consumed in its own order)
        L.w2 = L.w + (uint32_t)stages * fused_w1_item(pair);
        L.consts = L.w2 + (uint32_t)stages2 * fused_w2_rows(C, pair) * kBK;
    }
    L.red = L.consts + (3u * (uint32_t)H + 5u * (uint32_t)C) * 4u;   // m1 b1 mg1 [H]; m2 b2 zc2 g b [C]
    L.red = (L.red + 15u) & ~15u;
    L.bars = L.red + 2u * 2u * kBM * (uint32_t)ebytes;              // op #6 halves: [part][val][row]
    L.tmem_slot = L.bars + 8u * kFNumBars;
    L.total = L.tmem_slot + 16u;
    return L;
}

template <int F>
__global__ void __launch_bounds__(kFThreads, 1)
fused_mlp_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                 const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmY,
                 const __grid_constant__ FusedArgs p) {
    using namespace sm100;
    constexpr bool GELU = (F & kFGelu) != 0, ZH = (F & kFZh) != 0, B1 = (F & kFB1) != 0;
    constexpr bool TAPS = (F & kFTaps) != 0;   // debug taps compiled in (run_debug only)
    constexpr bool STATS64 = (F & kFS64) != 0, SMALLK = (F & kFSmallK) != 0;
    constexpr bool REG = (F & kFReg) != 0 && !STATS64 && !TAPS;   // op #6 half rows in registers
    constexpr bool PAIR = (F & kFPair) != 0;
    using acc_t = typename std::conditional<STATS64, double, float>::type;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* gbase = smem_raw + (base - raw);
    if (p.cta_stamps && threadIdx.x == 0) p.cta_stamps[2 * blockIdx.x] = gtimer();

    const int C = p.C, H = p.H;
    const uint32_t NJ = (uint32_t)p.NJ, KBC = (uint32_t)p.KBC, NB1 = (uint32_t)p.NB1, NH = (uint32_t)p.NH;
    const uint32_t stages = (uint32_t)p.stages;
    const bool resident = stages == 0;
    const FusedLayout L = fused_layout(C, H, p.NH, p.stages, (int)sizeof(acc_t), p.NX, p.y_inplace, p.stages2,
                                       PAIR ? 1 : 0);
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;         // pair: 0 = leader (issues the MMAs)
    const uint32_t w1item = fused_w1_item(PAIR ? 1 : 0);         // streamed W1 ring item bytes
    const uint32_t w2rows_it = fused_w2_rows(C, PAIR ? 1 : 0);   // rows of a streamed W2 ring item
    const uint32_t stages2 = (uint32_t)p.stages2;
    const bool yin = p.y_inplace != 0;
    const uint32_t NX = (uint32_t)p.NX;
    const uint32_t sX = base + L.x, sY = base + L.y, sHq = base + L.hq, sW = base + L.w, sW2 = base + L.w2;
    const uint32_t xslot = KBC * kKB;
    float* cm1 = reinterpret_cast<float*>(gbase + L.consts);
    float* cb1 = cm1 + H;
    uint32_t* cmg1 = reinterpret_cast<uint32_t*>(cb1 + H);
    float* cm2 = reinterpret_cast<float*>(cmg1 + H);
    float* cb2 = cm2 + C;
    int32_t* czc2 = reinterpret_cast<int32_t*>(cb2 + C);
    float* cg = reinterpret_cast<float*>(czc2 + C);
    float* cbt = cg + C;

    const uint32_t bar0 = base + L.bars;
    const uint32_t bar_xfull = bar0;                          // [NX]  X tile landed (1 + tx)
    const uint32_t bar_xempty = bar_xfull + 8u * kFMaxNX;     // [NX]  X tile consumed (op #6 pass 1, 8 warps)
    const uint32_t bar_wfull = bar_xempty + 8u * kFMaxNX;     // [S]   weight chunk landed (1 + tx)
    const uint32_t bar_wempty = bar_wfull + 8u * kFMaxStages; // [S]   weight chunk consumed (commit)
    const uint32_t bar_w2full = bar_wempty + 8u * kFMaxStages;   // [S2] W2 chunk landed (1 + tx)
    const uint32_t bar_w2empty = bar_w2full + 8u * kFMaxStages2; // [S2] W2 chunk consumed (commit)
    const uint32_t bar_wres = bar_w2empty + 8u * kFMaxStages2;   //       resident weights landed
    const uint32_t bar_a1full = bar_wres + 8u;                // [NB1] acc1 ready (commit)
    const uint32_t bar_a1empty = bar_a1full + 8u * kFMaxNB1;  // [NB1] acc1 drained (8 warps)
    const uint32_t bar_hqfull = bar_a1empty + 8u * kFMaxNB1;  // [NH]  Hq chunk written (8 warps)
    const uint32_t bar_hqempty = bar_hqfull + 8u * kFMaxNH;   // [NH]  Hq chunk consumed by FC2 (commit)
    const uint32_t bar_a2full = bar_hqempty + 8u * kFMaxNH;   // [NA2] acc2 complete (commit)
    const uint32_t bar_a2empty = bar_a2full + 16u;            // [NA2] acc2 drained (8 warps)
    const uint32_t bar_yfull = bar_a2empty + 16u;             //       Y tile staged (8 warps)
    const uint32_t bar_yempty = bar_yfull + 8u;               //       Y staging read by its stores (1)
    const uint32_t bar_cfull = bar_yempty + 16u;              //       constants loaded (32)
    const uint32_t bar_xpeer = bar_cfull + 8u;                // [NX]  pair (leader): the peer's X landed (1)
    // pair: barriers the leader's MMAs wait on that the peer's warps also arrive on
    auto arrive_leader = [&](uint32_t bar) {   // (the leader's own warps arrive locally)
        if (PAIR && rank != 0) mbar_arrive_cluster(mapa(bar, 0));
        else mbar_arrive(bar);
    };
    auto wait_pc = [&](uint32_t bar, uint32_t parity) {   // (cluster-scope acquire in a pair)
        if constexpr (PAIR) mbar_wait_cluster(bar, parity);
        else mbar_wait(bar, parity);
    };
    constexpr uint32_t kArrive = PAIR ? 16u : 8u;             // 8 epilogue warps per CTA
    volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(gbase + L.tmem_slot);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* trc = (p.trace && (int)blockIdx.x == p.trace_cta) ? p.trace : nullptr;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmW1);
        tma_prefetch_desc(&tmW2);
        tma_prefetch_desc(&tmY);
    }
    if (warp == 1 && lane == 0) {
        for (int i = 0; i < kFMaxNX; ++i) {
            mbar_init(bar_xfull + 8u * i, 1);
            mbar_init(bar_xempty + 8u * i, p.y_inplace ? 1u : 8u);   // Y store, or op #6 pass 1
        }
        mbar_init(bar_yfull, 8);
        mbar_init(bar_yempty, 1);
        for (int s = 0; s < kFMaxStages; ++s) {
            mbar_init(bar_wfull + 8u * s, 1);
            mbar_init(bar_wempty + 8u * s, 1);
            if (s < kFMaxStages2) {
                mbar_init(bar_w2full + 8u * s, 1);
                mbar_init(bar_w2empty + 8u * s, 1);
            }
        }
        mbar_init(bar_wres, 1);
        for (int b = 0; b < kFMaxNB1; ++b) {
            mbar_init(bar_a1full + 8u * b, 1);
            mbar_init(bar_a1empty + 8u * b, kArrive);
        }
        for (int b = 0; b < kFMaxNH; ++b) {
            mbar_init(bar_hqfull + 8u * b, kArrive);
            mbar_init(bar_hqempty + 8u * b, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_a2full + 8u * b, 1);
            mbar_init(bar_a2empty + 8u * b, kArrive);
        }
        mbar_init(bar_cfull, 32);
        for (int i = 0; i < kFMaxNX; ++i) mbar_init(bar_xpeer + 8u * i, 1);
        fence_mbar_init();
    }
    if (warp == 2) {
        if constexpr (PAIR) tmem_alloc_pair(smem_u32(const_cast<uint32_t*>(tmem_slot)), 512);
        else tmem_alloc(smem_u32(const_cast<uint32_t*>(tmem_slot)), 512);
    }
    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all();   // the peer's barriers exist before any remote arrive
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_launch_dependents();   // PDL: see mlp_kernels.cuh

    const uint32_t m_tiles = (uint32_t)((p.M + kBM - 1) / kBM);
    // work units: m-tiles, or (pair) m-tile pairs 2u (leader), 2u + 1 (peer)
    const uint32_t cid = PAIR ? blockIdx.x >> 1 : blockIdx.x, grid = PAIR ? gridDim.x >> 1 : gridDim.x;
    const uint32_t units = PAIR ? (m_tiles + 1u) >> 1 : m_tiles;
    const uint32_t n_my = cid < units ? (units - cid + grid - 1) / grid : 0u;
    const uint32_t U = n_my * NJ;                 // hidden chunks this CTA processes
    auto row0_of = [&](uint32_t i) -> int32_t {
        const uint32_t u = cid + i * grid;
        return (int32_t)((PAIR ? 2u * u + rank : u) * kBM);
    };
    // Hidden-chunk order rotated per CTA: position jj of a tile is chunk (jj + rot) mod NJ.
    // FC2 sums exact int32 partial products, so the order changes no result; it spreads
    // the CTAs' streamed weight reads over different chunks (different L2 lines) instead
    // of every SM requesting the same chunk at the same time.
    const uint32_t rot = p.rotate ? cid % NJ : 0u;
    // producer lookahead (chunks): the W1 items of FC1(q) are issued before the W2 items of
    // FC2(q - LA); LA <= NB1 - 1 keeps every wait satisfiable by earlier work, LA <= NJ keeps
    // the X-slot wait of the next tile behind the W2 loads it depends on
    const uint32_t LA = min(NB1 - 1u, NJ);
    auto chunk_of = [&](uint32_t jj) -> uint32_t { const uint32_t c = jj + rot; return c >= NJ ? c - NJ : c; };

    if (warp == 0) {
        // ============================ TMA producer ============================
        uint32_t s = 0, ph = 0;
        // a W2 chunk [C rows][128 B]: one box, or two of C/2 rows when C > 256 (TMA boxes
        // span at most 256 rows; FC2 then runs as two N = C/2 MMAs)
        const uint32_t w2rows = C > 256 ? (uint32_t)C / 2u : (uint32_t)C;
        auto load_w2 = [&](uint32_t dst, uint32_t bar, uint32_t j) {
            tma_load_2d(&tmW2, dst, bar, (int)(j * kFHc), 0);
            if (C > 256) tma_load_2d(&tmW2, dst + w2rows * kBK, bar, (int)(j * kFHc), (int)w2rows);
        };
        auto load_w1 = [&](uint32_t j, uint32_t dst, uint32_t bar) {
            for (uint32_t kb = 0; kb < KBC; ++kb)
                tma_load_2d(&tmW1, dst + kb * kKB, bar, (int)(kb * kBK), (int)(j * kFHc));
        };
        if (resident) {
            if (elect_one()) {
                mbar_arrive_expect_tx(bar_wres, NJ * (KBC * kKB + (uint32_t)C * kBK));
                for (uint32_t j = 0; j < NJ; ++j) {
                    load_w1(j, sW + j * KBC * kKB, bar_wres);
                    load_w2(sW2 + j * (uint32_t)C * kBK, bar_wres, j);
                }
            }
            __syncwarp();
        }
        pdl_wait();   // X: produced by the previous kernel
        // cursors advance incrementally (no runtime division in the role loops)
        uint32_t i = 0, j = 0, j2 = 0;     // FC1 tile / chunk of q; FC2 chunk position of q - LA
        uint32_t xs = 0, xph = 0;          // X slot of tile i, its phase
        uint32_t s2 = 0, ph2 = 0;          // W2 ring
        const uint32_t w2items = C > 256 ? 2u : 1u;
        for (uint32_t q = 0; q < U + LA; ++q) {
            if (q < U) {                       // operands of FC1(q)
                if (j == 0) {
                    mbar_wait(bar_xempty + 8u * xs, xph ^ 1u);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(bar_xfull + 8u * xs, xslot);
                        for (uint32_t kb = 0; kb < KBC; ++kb)
                            tma_load_2d(&tmX, sX + xs * xslot + kb * kKB, bar_xfull + 8u * xs, (int)(kb * kBK),
                                        row0_of(i));
                    }
                    __syncwarp();
                }
                if (!resident) {
                    for (uint32_t kb = 0; kb < KBC; ++kb) {   // one ring item per K-block
                        mbar_wait(bar_wempty + 8u * s, ph ^ 1u);
                        if (elect_one()) {
                            if constexpr (PAIR) {   // this CTA's 64 rows; bytes complete on the leader
                                if (rank == 0) mbar_arrive_expect_tx(bar_wfull + 8u * s, 2u * w1item);
                                tma_load_2d_pair(&tmW1, sW + s * w1item, mapa(bar_wfull + 8u * s, 0), (int)(kb * kBK),
                                                 (int)(chunk_of(j) * kFHc + rank * 64u));
                            } else {
                                mbar_arrive_expect_tx(bar_wfull + 8u * s, kKB);
                                tma_load_2d(&tmW1, sW + s * kKB, bar_wfull + 8u * s, (int)(kb * kBK),
                                            (int)(chunk_of(j) * kFHc));
                            }
                        }
                        __syncwarp();
                        if (++s == stages) { s = 0; ph ^= 1u; }
                    }
                }
                if (++j == NJ) {
                    j = 0;
                    ++i;
                    if (++xs == NX) { xs = 0; xph ^= 1u; }
                }
            }
            if (q >= LA && !resident) {        // operands of FC2(q - LA), in FC2's order
                for (uint32_t h = 0; h < w2items; ++h) {   // one ring item per FC2 MMA half
                    mbar_wait(bar_w2empty + 8u * s2, ph2 ^ 1u);
                    if (elect_one()) {
                        const uint32_t dst = sW2 + s2 * w2rows_it * kBK;
                        const int c0 = (int)(chunk_of(j2) * kFHc), r0 = (int)(h * w2rows + rank * w2rows_it);
                        if constexpr (PAIR) {   // this CTA's half of the MMA's B rows
                            if (rank == 0) mbar_arrive_expect_tx(bar_w2full + 8u * s2, 2u * w2rows_it * kBK);
                            tma_load_2d_pair(&tmW2, dst, mapa(bar_w2full + 8u * s2, 0), c0, r0);
                        } else {
                            mbar_arrive_expect_tx(bar_w2full + 8u * s2, w2rows_it * kBK);
                            tma_load_2d(&tmW2, dst, bar_w2full + 8u * s2, c0, r0);
                        }
                    }
                    __syncwarp();
                    if (++s2 == stages2) { s2 = 0; ph2 ^= 1u; }
                }
                if (++j2 == NJ) j2 = 0;
            }
        }
    } else if (warp == 1) {
        // ============================ FC1 issuer ==============================
        // FC1 and FC2 are issued by two warps (this one and warp 3 after the constants):
        // a tcgen05.mma issue can stall while earlier MMAs execute, and in one in-order
        // warp FC1 of the next chunk would queue behind FC2's wait for op #5.  Each
        // warp's tcgen05.commit tracks its own MMAs.  Descriptors are base + offset (the
        // 14-bit start-address field never carries: smem < 256 KB).
        if (PAIR && rank != 0) {
            // pair peer: no MMAs here; relay "my X tile landed" to the leader's FC1
            uint32_t xs = 0, xph = 0;
            for (uint32_t i = 0; i < n_my; ++i) {
                mbar_wait(bar_xfull + 8u * xs, xph);
                if (lane == 0) mbar_arrive_cluster(mapa(bar_xpeer + 8u * xs, 0));
                __syncwarp();
                if (++xs == NX) { xs = 0; xph ^= 1u; }
            }
            goto fc1_done;
        }
        {
        const uint32_t idesc1 = idesc_i8(PAIR ? 2u * kBM : kBM, kFHc);
        const uint64_t dX = umma_desc_k128(sX), dW = umma_desc_k128(sW);
        const uint32_t xslot16 = xslot >> 4, stage16 = w1item >> 4;
        const uint32_t kb16 = kKB >> 4;
        const int nk_last = (C - (int)((KBC - 1u) * kBK)) / 32;   // MMAs (K = 32) in the last K-block
        const uint32_t a1_tm = tmem_base + (uint32_t)p.a1_col;
        uint32_t s = 0, ph = 0;
        if (resident) mbar_wait(bar_wres, 0);
        uint32_t i = 0, j = 0, b = 0, bph = 0;           // tile, chunk, acc1 buffer, its phase
        uint32_t xs = 0, xph = 0;                        // X slot, its phase
        for (uint32_t q = 0; q < U; ++q) {               // FC1(q): acc1[b] = X_i . W1[j]^T
            if (trc && lane == 0 && q < 512) trc[1024 + q] = gtimer();
            if (j == 0) {
                mbar_wait(bar_xfull + 8u * xs, xph);
                if constexpr (PAIR) mbar_wait_cluster(bar_xpeer + 8u * xs, xph);
            }
            wait_pc(bar_a1empty + 8u * b, bph ^ 1u);
            if (trc && lane == 0 && q < 512) trc[1536 + q] = gtimer();
            const uint32_t d = a1_tm + b * (uint32_t)kFHc;
            const uint64_t ad0 = dX + xs * xslot16;
            for (uint32_t kb = 0; kb < KBC; ++kb) {
                if (!resident) wait_pc(bar_wfull + 8u * s, ph);
                if (trc && lane == 0 && q < 512 && kb + 1 == KBC) trc[7680 + q] = gtimer();   // weights in
                tc_fence_after();
                const uint64_t ad = ad0 + kb * kb16;
                const uint64_t bd = resident ? dW + (chunk_of(j) * KBC + kb) * kb16 : dW + s * stage16;
                const int nk = kb + 1u == KBC ? nk_last : 4;
                if (elect_one()) {
                    if constexpr (PAIR) {
                        for (int k = 0; k < nk; ++k) mma_i8_pair(d, ad + 2u * k, bd + 2u * k, idesc1, (kb | k) != 0);
                        mma_commit_pair_mc(bar_wempty + 8u * s, 3);   // both CTAs' ring slots
                    } else {
                        mma_i8(d, ad, bd, idesc1, kb);
                        if (nk > 1) mma_i8(d, ad + 2u, bd + 2u, idesc1, 1u);
                        if (nk > 2) mma_i8(d, ad + 4u, bd + 4u, idesc1, 1u);
                        if (nk > 3) mma_i8(d, ad + 6u, bd + 6u, idesc1, 1u);
                        if (!resident) mma_commit(bar_wempty + 8u * s);
                    }
                }
                __syncwarp();
                if (!resident && ++s == stages) { s = 0; ph ^= 1u; }
            }
            if (elect_one()) {
                if constexpr (PAIR) mma_commit_pair_mc(bar_a1full + 8u * b, 3);
                else mma_commit(bar_a1full + 8u * b);
                if (trc && q < 512) trc[q] = gtimer();
            }
            __syncwarp();
            if (++j == NJ) {
                j = 0;
                ++i;
                if (++xs == NX) { xs = 0; xph ^= 1u; }
            }
            if (++b == NB1) { b = 0; bph ^= 1u; }
        }
        }
    fc1_done:;
    } else if (warp == 2) {
        // ============================ Y store warp ============================
        pdl_wait();   // Y may overwrite what the previous kernel still reads
        uint32_t xs = 0;
        for (uint32_t i = 0; i < n_my; ++i) {
            mbar_wait_backoff(bar_yfull, i & 1u);
            if (lane == 0) {
                const uint32_t src = yin ? sX + xs * xslot : sY;
                for (uint32_t kb = 0; kb < KBC; ++kb)
                    tma_store_2d(&tmY, src + kb * kKB, (int)(kb * kBK), row0_of(i));
                bulk_commit();
                bulk_wait_read<0>();           // Y read out of the staging buffer
                if (yin) mbar_arrive(bar_xempty + 8u * xs);   // the X slot (Y staged over it) is free
                else mbar_arrive(bar_yempty);
                if (trc && i < 512) trc[6144 + i] = gtimer();
            }
            __syncwarp();
            if (++xs == NX) xs = 0;
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    } else if (warp == 3) {
        // ============================ constants ===============================
        for (int n = (int)lane; n < H; n += 32) {
            cm1[n] = __ldg(p.m1 + n);
            cb1[n] = p.b1 ? __ldg(p.b1 + n) : 0.0f;
            const int32_t zc = p.zc1 ? __ldg(p.zc1 + n) : 0;
            cmg1[n] = SMALLK ? 0x4B400000u - (uint32_t)zc : (uint32_t)zc;   // magic - zc, or zc
        }
        for (int c = (int)lane; c < C; c += 32) {
            cm2[c] = __ldg(p.m2 + c);
            cb2[c] = p.b2 ? __ldg(p.b2 + c) : 0.0f;
            czc2[c] = p.zc2 ? __ldg(p.zc2 + c) : 0;
            cg[c] = __ldg(p.gamma + c);
            cbt[c] = __ldg(p.beta + c);
        }
        mbar_arrive(bar_cfull);

        // ============================ FC2 issuer ==============================
        if (PAIR && rank != 0) goto fc2_done;   // the leader issues for the pair
        {
        const uint32_t n2 = C > 256 ? (uint32_t)C / 2u : (uint32_t)C;   // N per FC2 MMA (<= 256)
        const uint32_t idesc2 = idesc_i8(PAIR ? 2u * kBM : kBM, n2);
        const uint32_t it16 = (w2rows_it * kBK) >> 4;                    // streamed ring item stride
        const uint32_t n2off16 = (n2 * kBK) >> 4;                        // bytes/16 of N2 B rows
        const uint32_t w2n = C > 256 ? 2u : 1u;
        const uint64_t dW2 = umma_desc_k128(sW2), dHq = umma_desc_k128(sHq);
        const uint32_t w2c16 = ((uint32_t)C * kBK) >> 4, kb16 = kKB >> 4;
        uint32_t s2 = 0, ph2 = 0;
        if (resident) mbar_wait(bar_wres, 0);
        uint32_t j2 = 0, hb = 0, hph = 0, ab = 0, aph = 0;   // chunk, Hq buffer, acc2 buffer (+ phases)
        for (uint32_t u = 0; u < U; ++u) {                    // FC2(u): acc2 += Hq_u . W2[:, j2]^T
            if (trc && lane == 0 && u < 512) trc[6656 + u] = gtimer();
            wait_pc(bar_hqfull + 8u * hb, hph);
            if (j2 == 0) wait_pc(bar_a2empty + 8u * ab, aph ^ 1u);
            if (trc && lane == 0 && u < 512) trc[7168 + u] = gtimer();
            const uint64_t ad = dHq + hb * kb16;
            const uint32_t d2 = tmem_base + ab * (uint32_t)p.a2_stride;
            // C > 256: two MMA halves of N = C/2 (W2 rows [h C/2, (h+1) C/2) -> TMEM columns
            // h C/2 ..), each on its own streamed ring item
            for (uint32_t h = 0; h < w2n; ++h) {
                if (!resident) wait_pc(bar_w2full + 8u * s2, ph2);
                tc_fence_after();
                const uint64_t bd = resident ? dW2 + chunk_of(j2) * w2c16 + h * n2off16 : dW2 + s2 * it16;
                const uint32_t dh = d2 + h * n2;
                if (elect_one()) {
                    if constexpr (PAIR) {
                        for (int k = 0; k < 4; ++k) mma_i8_pair(dh, ad + 2u * k, bd + 2u * k, idesc2, (j2 | k) != 0);
                        mma_commit_pair_mc(bar_w2empty + 8u * s2, 3);
                    } else {
                        mma_i8(dh, ad, bd, idesc2, j2);
                        mma_i8(dh, ad + 2u, bd + 2u, idesc2, 1u);
                        mma_i8(dh, ad + 4u, bd + 4u, idesc2, 1u);
                        mma_i8(dh, ad + 6u, bd + 6u, idesc2, 1u);
                        if (!resident) mma_commit(bar_w2empty + 8u * s2);
                    }
                }
                __syncwarp();
                if (!resident && ++s2 == stages2) { s2 = 0; ph2 ^= 1u; }
            }
            if (elect_one()) {
                if constexpr (PAIR) {
                    mma_commit_pair_mc(bar_hqempty + 8u * hb, 3);
                    if (j2 + 1u == NJ) mma_commit_pair_mc(bar_a2full + 8u * ab, 3);
                } else {
                    mma_commit(bar_hqempty + 8u * hb);
                    if (j2 + 1u == NJ) mma_commit(bar_a2full + 8u * ab);
                }
                if (trc && u < 512) trc[512 + u] = gtimer();
            }
            __syncwarp();
            if (++j2 == NJ) {
                j2 = 0;
                if (++ab == (uint32_t)p.NA2) { ab = 0; aph ^= 1u; }
            }
            if (++hb == NH) { hb = 0; hph ^= 1u; }
        }
        }
    fc2_done:;
    } else if (warp < (uint32_t)kFEp6W0) {
        // ============================ op #5 ===================================
        // acc1 chunk (128 hidden columns) -> Hq chunk in smem, 128-B swizzled K-major
        // rows (16-B granule g of row r at ((g ^ (r & 7)) << 4)): FC2's A operand.
        const uint32_t ew = warp - (uint32_t)kFEp5W0;
        const uint32_t quad = warp & 3u, half = ew >> 2;
        const uint32_t rit = quad * 32u + lane;
        const uint32_t row_off = rit * (uint32_t)kBK, rsw = rit & 7u;
        const float2 inv2 = make_float2(p.inv_h, p.inv_h);
        const bool zx0 = p.z_x == 0;
        pdl_wait();   // (taps)
        mbar_wait(bar_cfull, 0);
        uint32_t i = 0, j = 0, b = 0, bph = 0, hb = 0, hph = 0;
        for (uint32_t u = 0; u < U; ++u) {
            mbar_wait_backoff(bar_a1full + 8u * b, bph);
            mbar_wait_backoff(bar_hqempty + 8u * hb, hph ^ 1u);
            tc_fence_after();
            const bool stamp = trc && ew == 0 && lane == 0 && u < 1024;
            if (stamp) trc[2048 + 2 * u] = gtimer();
            const int64_t row = (int64_t)row0_of(i) + rit;
            const bool valid = row < p.M;
            const uint32_t tb = tmem_base + ((quad * 32u) << 16) + (uint32_t)p.a1_col + b * (uint32_t)kFHc + half * 64u;
            const uint32_t hq = sHq + hb * kKB + row_off;
            const int n_base = (int)(chunk_of(j) * kFHc + half * 64u);
            auto chunk_t = [&](auto zx0_c, uint32_t (&r)[16], int ch) {
                constexpr bool ZX0 = decltype(zx0_c)::value;   // z_x == 0: plain I2FP, no correction
                const int n0 = n_base + ch * 16;
                float v[16];
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) {
                    const float4 mv = *reinterpret_cast<const float4*>(cm1 + n0 + 4 * j4);
                    const float4 bv = B1 ? *reinterpret_cast<const float4*>(cb1 + n0 + 4 * j4)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                    const uint4 gv = ZX0 ? make_uint4(0x4B400000u, 0x4B400000u, 0x4B400000u, 0x4B400000u)
                                         : *reinterpret_cast<const uint4*>(cmg1 + n0 + 4 * j4);
                    float2 a0, a1;
                    if constexpr (ZX0) {
                        // one I2FP per value (a conversion-pipe op, ~25 % busy here) instead of
                        // the magic add + subtract (1.5 issue slots): the epilogue is issue-bound
                        a0 = make_float2(__int2float_rn((int32_t)r[4 * j4]), __int2float_rn((int32_t)r[4 * j4 + 1]));
                        a1 = make_float2(__int2float_rn((int32_t)r[4 * j4 + 2]), __int2float_rn((int32_t)r[4 * j4 + 3]));
                    } else if constexpr (SMALLK) {
                        // bits (0x4B400000 - zc) + acc = float 1.5*2^23 + (acc - zc), exact
                        const float2 mg = make_float2(12582912.0f, 12582912.0f);
                        a0 = f2_sub(make_float2(__uint_as_float(r[4 * j4] + gv.x), __uint_as_float(r[4 * j4 + 1] + gv.y)), mg);
                        a1 = f2_sub(make_float2(__uint_as_float(r[4 * j4 + 2] + gv.z), __uint_as_float(r[4 * j4 + 3] + gv.w)), mg);
                    } else {
                        a0 = make_float2(__int2float_rn((int32_t)(r[4 * j4] - gv.x)), __int2float_rn((int32_t)(r[4 * j4 + 1] - gv.y)));
                        a1 = make_float2(__int2float_rn((int32_t)(r[4 * j4 + 2] - gv.z)), __int2float_rn((int32_t)(r[4 * j4 + 3] - gv.w)));
                    }
                    if (TAPS && p.acc1_tap && valid) {
                        const uint32_t o = SMALLK ? 0x4B400000u : 0u;
                        int4 t;
                        if (ZX0) t = make_int4((int)r[4 * j4], (int)r[4 * j4 + 1], (int)r[4 * j4 + 2], (int)r[4 * j4 + 3]);
                        else if (SMALLK) t = make_int4((int)(r[4 * j4] + gv.x - o), (int)(r[4 * j4 + 1] + gv.y - o),
                                                  (int)(r[4 * j4 + 2] + gv.z - o), (int)(r[4 * j4 + 3] + gv.w - o));
                        else t = make_int4((int)(r[4 * j4] - gv.x), (int)(r[4 * j4 + 1] - gv.y),
                                           (int)(r[4 * j4 + 2] - gv.z), (int)(r[4 * j4 + 3] - gv.w));
                        st_v4(p.acc1_tap + row * (int64_t)H + n0 + 4 * j4, t);
                    }
                    // y = fl(fmaf(a, m1, b1))  (b1 = 0 without bias: bit-identical to fl(a*m1))
                    float2 y0 = f2_fma(a0, make_float2(mv.x, mv.y), make_float2(bv.x, bv.y));
                    float2 y1 = f2_fma(a1, make_float2(mv.z, mv.w), make_float2(bv.z, bv.w));
                    if constexpr (GELU) {
                        y0 = make_float2(gelu_erf_f32(y0.x), gelu_erf_f32(y0.y));
                        y1 = make_float2(gelu_erf_f32(y1.x), gelu_erf_f32(y1.y));
                    }
                    const float2 t0 = f2_mul(y0, inv2), t1 = f2_mul(y1, inv2);
                    v[4 * j4] = t0.x; v[4 * j4 + 1] = t0.y; v[4 * j4 + 2] = t1.x; v[4 * j4 + 3] = t1.y;
                }
                uint32_t w[4];
                quant_pack16<!GELU, ZH>(v, p.z_h, w);
                const uint32_t g = half * 4u + (uint32_t)ch;
                st_shared_v4(hq + ((g ^ rsw) << 4), w[0], w[1], w[2], w[3]);
                if (TAPS && p.hid_tap && valid)
                    st_v4(p.hid_tap + row * (int64_t)H + n0, make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]));
            };
            auto chunk = [&](uint32_t (&r)[16], int ch) {
                if (zx0) chunk_t(std::true_type{}, r, ch);
                else chunk_t(std::false_type{}, r, ch);
            };
            uint32_t ra[16], rb[16];
            tmem_ld16(tb, ra);
            tmem_wait_ld_dep(ra);
            tmem_ld16(tb + 16u, rb);
            chunk(ra, 0);
            tmem_wait_ld_dep(rb);
            tmem_ld16(tb + 32u, ra);
            chunk(rb, 1);
            tmem_wait_ld_dep(ra);
            tmem_ld16(tb + 48u, rb);
            chunk(ra, 2);
            tmem_wait_ld_dep(rb);
            chunk(rb, 3);
            tc_fence_before();
            fence_proxy_async_smem();          // Hq visible to the tensor core (async proxy)
            __syncwarp();
            if (lane == 0) {   // (pair: on the leader, whose MMAs read both CTAs' Hq)
                arrive_leader(bar_a1empty + 8u * b);
                arrive_leader(bar_hqfull + 8u * hb);
            }
            if (stamp) trc[2048 + 2 * u + 1] = gtimer();
            if (++j == NJ) { j = 0; ++i; }
            if (++b == NB1) { b = 0; bph ^= 1u; }
            if (++hb == NH) { hb = 0; hph ^= 1u; }
        }
    } else {
        // ============================ op #6 ===================================
        // One thread per token row, the whole row: dQ + bias + residual -> z (parked
        // back in TMEM), row statistics in-thread (no cross-warp exchange), then
        // LayerNorm + Q into the Y staging tile.
        //   fp32: one pass of shifted sums, shift K = mean of the row's first 16 z
        //         (any K gives the exact statistics; K near the mean keeps the
        //         S2/C - (S1/C)^2 cancellation small): mu = K + S1/C,
        //         var = S2/C - (S1/C)^2   (reading R15)
        //   fp64: the oracle's two passes, ascending columns (O5)
        const uint32_t quad = warp & 3u, part = (warp - (uint32_t)kFEp6W0) >> 2;
        const uint32_t rit = quad * 32u + lane;
        const uint32_t row_off = rit * (uint32_t)kBK, rsw = rit & 7u;
        const int hc = C >> 1;                     // columns of this half: [cb, cb + hc)
        const int cb = (int)part * hc;
        const int nch = hc >> 4;                   // chunks of 16 (C % 32 == 0)
        const float inv_nh = 1.0f / (float)hc, inv_c = 1.0f / (float)C;
        // pairwise combine of the two halves' statistics through smem; both halves
        // combine in the same (part 0, part 1) order, so they agree bit for bit
        using acc_t2 = typename std::conditional<STATS64, double, float>::type;
        acc_t2* red = reinterpret_cast<acc_t2*>(gbase + L.red);
        auto exchange = [&](acc_t2 v0, acc_t2 v1, acc_t2 (&o)[2][2]) {
            red[(part * 2u) * kBM + rit] = v0;
            red[(part * 2u + 1u) * kBM + rit] = v1;
            named_bar_sync(1u + quad, 64u);       // the two warps of this lane quadrant
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                o[q][0] = red[((uint32_t)q * 2u) * kBM + rit];
                o[q][1] = red[((uint32_t)q * 2u + 1u) * kBM + rit];
            }
            named_bar_sync(1u + quad, 64u);       // reads done before the next tile's writes
        };
        const float2 inv2 = make_float2(p.inv_y, p.inv_y);
        const float2 sx2 = make_float2(p.s_x, p.s_x);
        const float2 one2 = make_float2(p.one, p.one);
        const float xoff = 8388608.0f + 128.0f + (float)p.z_x;   // exact: |z_x| <= 128
        const float2 xoff2 = make_float2(xoff, xoff);
        auto goff = [&](int c) -> uint32_t {       // this row's granule of column c (multiple of 16)
            const uint32_t kb = (uint32_t)c >> 7, g = ((uint32_t)c >> 4) & 7u;
            return kb * kKB + row_off + ((g ^ rsw) << 4);
        };
        constexpr bool regpath = REG;   // (host: only when nch <= kFRegCh)
        pdl_wait();   // (global residual, residual_out, taps)
        mbar_wait(bar_cfull, 0);
        uint32_t ab = 0, aph = 0, xs = 0, xph = 0;
        for (uint32_t i = 0; i < n_my; ++i) {
            mbar_wait_backoff(bar_a2full + 8u * ab, aph);
            mbar_wait(bar_xfull + 8u * xs, xph);     // (complete since FC1: visibility of X)
            tc_fence_after();
            const bool stamp = trc && quad == 0 && lane == 0 && i < 512;
            if (stamp) trc[4096 + 4 * i] = gtimer();
            const int64_t row = (int64_t)row0_of(i) + rit;
            const bool valid = row < p.M;
            const uint32_t tb = tmem_base + ((quad * 32u) << 16) + ab * (uint32_t)p.a2_stride + (uint32_t)cb;
            const uint32_t xt = sX + xs * xslot;

            // chunk loop for the passes over parked z: pairs of chunks behind one wait
            // (chunk index ch is local to this half; column = cb + 16 ch)
            auto for_chunks = [&](auto&& fn) {
                int ch = 0;
                for (; ch + 1 < nch; ch += 2) {
                    uint32_t ra[16], rb[16];
                    tmem_ld16(tb + (uint32_t)(ch * 16), ra);
                    tmem_ld16(tb + (uint32_t)((ch + 1) * 16), rb);
                    tmem_wait_ld_dep(ra);
                    reg_fence16(rb);
                    fn(ra, ch);
                    fn(rb, ch + 1);
                }
                if (ch < nch) {
                    uint32_t ra[16];
                    tmem_ld16(tb + (uint32_t)(ch * 16), ra);
                    tmem_wait_ld_dep(ra);
                    fn(ra, ch);
                }
            };
            // pass 1: z = fl(fl(fmaf(fl(A2), m2, b2)) + r), back into TMEM; statistics.
            // Pairs of chunks behind one TMEM wait, branch-free bodies (residual source
            // and taps resolved outside) so the two chunks' arithmetic interleaves.
            float K = 0.f;
            float2 s1f = make_float2(0.f, 0.f), s2f = make_float2(0.f, 0.f), Kv = make_float2(0.f, 0.f);
            double s1d = 0.0;
            // z of one 16-column chunk (r: raw accumulators, modified in place)
            auto chunk_z = [&](auto resid_c, uint32_t (&r)[16], int c0, float2 (&z)[8]) {
                constexpr bool RESID = decltype(resid_c)::value;
                float2 rr[8];
                if constexpr (RESID) {
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4) {
                        const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(p.resid + row * C + c0) + j4)
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
                        rr[2 * j4] = make_float2(v.x, v.y);
                        rr[2 * j4 + 1] = make_float2(v.z, v.w);
                    }
                } else {
                    // x - z_x as float, exactly, by offset binary: bits 0x4B0000uu =
                    // 2^23 + u, u = x ^ 0x80 = x + 128
                    const uint4 xv = *reinterpret_cast<const uint4*>(gbase + (xt - base) + goff(c0));
                    const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t ob = xw[q] ^ 0x80808080u;
                        const float2 f01 = make_float2(__uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7650)),
                                                       __uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7651)));
                        const float2 f23 = make_float2(__uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7652)),
                                                       __uint_as_float(__byte_perm(ob, 0x4B000000u, 0x7653)));
                        rr[2 * q] = f2_sub(f01, xoff2);          // x - z_x, exact
                        rr[2 * q + 1] = f2_sub(f23, xoff2);
                    }
                }
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) {
                    const float4 mv = *reinterpret_cast<const float4*>(cm2 + c0 + 4 * j4);
                    const float4 bv = *reinterpret_cast<const float4*>(cb2 + c0 + 4 * j4);
                    if constexpr (ZH) {
                        const int4 zv = *reinterpret_cast<const int4*>(czc2 + c0 + 4 * j4);
                        r[4 * j4 + 0] -= (uint32_t)zv.x; r[4 * j4 + 1] -= (uint32_t)zv.y;
                        r[4 * j4 + 2] -= (uint32_t)zv.z; r[4 * j4 + 3] -= (uint32_t)zv.w;
                    }
                    const float2 a0 = make_float2(__int2float_rn((int32_t)r[4 * j4]), __int2float_rn((int32_t)r[4 * j4 + 1]));
                    const float2 a1 = make_float2(__int2float_rn((int32_t)r[4 * j4 + 2]), __int2float_rn((int32_t)r[4 * j4 + 3]));
                    const float2 d0 = f2_fma(a0, make_float2(mv.x, mv.y), make_float2(bv.x, bv.y));
                    const float2 d1 = f2_fma(a1, make_float2(mv.z, mv.w), make_float2(bv.z, bv.w));
                    if constexpr (RESID) {       // z = fl(d + R)
                        z[2 * j4] = f2_add(d0, rr[2 * j4]);
                        z[2 * j4 + 1] = f2_add(d1, rr[2 * j4 + 1]);
                    } else {                     // z = fl(d + fl((x - z_x) * s_x))
                        // dQ(x), then Add (R3): fl(fl(r * s_x) * 1 + d), see GemmArgs::one
                        z[2 * j4] = f2_fma(f2_mul(rr[2 * j4], sx2), one2, d0);
                        z[2 * j4 + 1] = f2_fma(f2_mul(rr[2 * j4 + 1], sx2), one2, d1);
                    }
                }
            };
            auto stats = [&](const float2 (&z)[8]) {
                if constexpr (STATS64) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        s1d = __dadd_rn(s1d, (double)z[j].x);
                        s1d = __dadd_rn(s1d, (double)z[j].y);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float2 d = f2_sub(z[j], Kv);
                        s1f = f2_add(s1f, d);
                        s2f = f2_fma(d, d, s2f);
                    }
                }
            };
            auto park = [&](const float2 (&z)[8], const uint32_t (&r)[16], int c0) {   // z -> TMEM (+ taps)
                if (TAPS && p.acc2_tap && valid) {
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4)
                        st_v4(p.acc2_tap + row * (int64_t)C + cb + c0 + 4 * j4,
                              make_int4((int)r[4 * j4], (int)r[4 * j4 + 1], (int)r[4 * j4 + 2], (int)r[4 * j4 + 3]));
                }
                uint32_t zu[16];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    zu[2 * j] = __float_as_uint(z[j].x);
                    zu[2 * j + 1] = __float_as_uint(z[j].y);
                }
                tmem_st16(tb + (uint32_t)c0, zu);
            };
            auto set_shift = [&](const float2 (&z)[8]) {   // K = mean of this half's first 16 values
                float2 t = z[0];
#pragma unroll
                for (int j = 1; j < 8; ++j) t = f2_add(t, z[j]);
                K = __fmul_rn(__fadd_rn(t.x, t.y), 0.0625f);
                Kv = make_float2(K, K);
            };
            auto store_z = [&](const float2 (&z)[8], int c0) {
                if (p.resid_out && valid) {
                    float* zrow = p.resid_out + row * (int64_t)C + c0;
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4)
                        *reinterpret_cast<float4*>(zrow + 4 * j4) =
                            make_float4(z[2 * j4].x, z[2 * j4].y, z[2 * j4 + 1].x, z[2 * j4 + 1].y);
                }
            };
            auto pass1 = [&](auto resid_c) {
                int ch = 0;
                for (; ch + 1 < nch; ch += 2) {
                    uint32_t ra[16], rb[16];
                    tmem_ld16(tb + (uint32_t)(ch * 16), ra);
                    tmem_ld16(tb + (uint32_t)((ch + 1) * 16), rb);
                    tmem_wait_ld_dep(ra);
                    reg_fence16(rb);
                    float2 za[8], zb[8];
                    chunk_z(resid_c, ra, cb + ch * 16, za);
                    chunk_z(resid_c, rb, cb + ch * 16 + 16, zb);
                    if (!STATS64 && ch == 0) set_shift(za);
                    stats(za);
                    stats(zb);
                    store_z(za, cb + ch * 16);
                    store_z(zb, cb + ch * 16 + 16);
                    park(za, ra, ch * 16);
                    park(zb, rb, ch * 16 + 16);
                }
                if (ch < nch) {
                    uint32_t ra[16];
                    tmem_ld16(tb + (uint32_t)(ch * 16), ra);
                    tmem_wait_ld_dep(ra);
                    float2 za[8];
                    chunk_z(resid_c, ra, cb + ch * 16, za);
                    if (!STATS64 && ch == 0) set_shift(za);
                    stats(za);
                    store_z(za, cb + ch * 16);
                    park(za, ra, ch * 16);
                }
            };
            // register path: all of this half row's A2 chunks in one batch of TMEM loads,
            // acc2 released at once (FC2 of the next tile may start), z kept in registers
            uint32_t r[REG ? kFRegCh : 1][16];   // A2, then z (fp32 bits) in place
            auto pass1_reg = [&](auto resid_c) {
#pragma unroll
                for (int ch = 0; ch < (REG ? kFRegCh : 1); ++ch)
                    if (ch < nch) tmem_ld16(tb + (uint32_t)(ch * 16), r[ch]);
                tmem_wait_ld_dep(r[0]);
#pragma unroll
                for (int ch = 1; ch < (REG ? kFRegCh : 1); ++ch) reg_fence16(r[ch]);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive_leader(bar_a2empty + 8u * ab);   // acc2 drained
#pragma unroll
                for (int ch = 0; ch < (REG ? kFRegCh : 1); ++ch) {
                    if (ch < nch) {
                        float2 z[8];
                        chunk_z(resid_c, r[ch], cb + ch * 16, z);
                        if (ch == 0) set_shift(z);
                        stats(z);
                        store_z(z, cb + ch * 16);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            r[ch][2 * j] = __float_as_uint(z[j].x);
                            r[ch][2 * j + 1] = __float_as_uint(z[j].y);
                        }
                    }
                }
            };
            if constexpr (regpath) {
                if (p.resid) pass1_reg(std::true_type{});
                else pass1_reg(std::false_type{});
            } else {
                if (p.resid) pass1(std::true_type{});
                else pass1(std::false_type{});
                tmem_wait_st();
            }
            __syncwarp();
            if (lane == 0 && !yin) mbar_arrive(bar_xempty + 8u * xs);   // X tile consumed
            if (stamp) trc[4096 + 4 * i + 2] = gtimer();

            float mu_f = 0.f, rstd_f = 0.f;
            double mu_d = 0.0, rstd_d = 0.0;
            if constexpr (STATS64) {
                acc_t2 o[2][2];
                exchange(s1d, 0.0, o);
                mu_d = __dadd_rn(o[0][0], o[1][0]) / (double)C;
                double s2d = 0.0;
                for_chunks([&](uint32_t (&r)[16], int) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const double d = __dsub_rn((double)__uint_as_float(r[j]), mu_d);
                        s2d = __dadd_rn(s2d, __dmul_rn(d, d));
                    }
                });
                exchange(s2d, 0.0, o);
                const double SS = __dadd_rn(o[0][0], o[1][0]);
                rstd_d = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(SS, (double)C), (double)p.eps)));
            } else {
                // each half: mean m_h = K + S1/n, M2_h = S2 - S1^2/n (n = C/2); combined
                // (Chan): mean = (m_0 + m_1)/2, M2 = M2_0 + M2_1 + (m_1 - m_0)^2 n/2
                const float nh = (float)hc;
                const float S1 = __fadd_rn(s1f.x, s1f.y), S2 = __fadd_rn(s2f.x, s2f.y);
                const float q1 = __fmul_rn(S1, inv_nh);   // (fp32 LN tier: reciprocal multiplies, rsqrt)
                acc_t2 o[2][2];
                exchange(__fadd_rn(K, q1), __fsub_rn(S2, __fmul_rn(S1, q1)), o);
                const float dm = __fsub_rn(o[1][0], o[0][0]);
                mu_f = __fmul_rn(__fadd_rn(o[0][0], o[1][0]), 0.5f);
                const float M2 = __fadd_rn(__fadd_rn(o[0][1], o[1][1]), __fmul_rn(__fmul_rn(dm, dm), __fmul_rn(nh, 0.5f)));
                const float var = fmaxf(__fmul_rn(M2, inv_c), 0.0f);
                rstd_f = rsqrtf(__fadd_rn(var, p.eps));
            }
            const float2 mu2 = make_float2(mu_f, mu_f), rstd2 = make_float2(rstd_f, rstd_f);
            if (stamp) trc[4096 + 4 * i + 1] = gtimer();

            // pass 2: yhat = fl(((z - mu) * rstd) * gamma + beta); Y = Q_y(yhat) into the staging
            // buffer once the previous tile's stores have read it
            if (!yin) mbar_wait_backoff(bar_yempty, (i & 1u) ^ 1u);
            const uint32_t sYt = yin ? xt : sY;   // Y staging: own X slot, or the Y buffer
            auto ln_chunk = [&](const uint32_t (&r)[16], int ch) {
                const int c0 = cb + ch * 16;
                float v[16];
#pragma unroll
                for (int j4 = 0; j4 < 4; ++j4) {
                    const float4 gv = *reinterpret_cast<const float4*>(cg + c0 + 4 * j4);
                    const float4 bv = *reinterpret_cast<const float4*>(cbt + c0 + 4 * j4);
                    float yh[4];
                    if constexpr (STATS64) {
                        const float gg[4] = {gv.x, gv.y, gv.z, gv.w};
                        const float bb[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const double xh = __dmul_rn(__dsub_rn((double)__uint_as_float(r[4 * j4 + jj]), mu_d), rstd_d);
                            yh[jj] = __double2float_rn(__dadd_rn(__dmul_rn(xh, (double)gg[jj]), (double)bb[jj]));
                        }
                    } else {
                        const float2 z0 = make_float2(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]));
                        const float2 z1 = make_float2(__uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3]));
                        const float2 y0 = f2_fma(f2_mul(f2_sub(z0, mu2), rstd2), make_float2(gv.x, gv.y), make_float2(bv.x, bv.y));
                        const float2 y1 = f2_fma(f2_mul(f2_sub(z1, mu2), rstd2), make_float2(gv.z, gv.w), make_float2(bv.z, bv.w));
                        yh[0] = y0.x; yh[1] = y0.y; yh[2] = y1.x; yh[3] = y1.y;
                    }
                    if (TAPS && p.ln_tap && valid)
                        *reinterpret_cast<float4*>(p.ln_tap + row * (int64_t)C + c0 + 4 * j4) =
                            make_float4(yh[0], yh[1], yh[2], yh[3]);
                    const float2 t0 = f2_mul(make_float2(yh[0], yh[1]), inv2), t1 = f2_mul(make_float2(yh[2], yh[3]), inv2);
                    v[4 * j4] = t0.x; v[4 * j4 + 1] = t0.y; v[4 * j4 + 2] = t1.x; v[4 * j4 + 3] = t1.y;
                }
                uint32_t w[4];
                if (p.z_y) quant_pack16<false, true>(v, p.z_y, w);
                else quant_pack16<false, false>(v, 0, w);
                st_shared_v4(sYt + goff(c0), w[0], w[1], w[2], w[3]);
            };
            if constexpr (regpath) {
#pragma unroll
                for (int ch = 0; ch < (REG ? kFRegCh : 1); ++ch)
                    if (ch < nch) ln_chunk(r[ch], ch);
            } else {
                for_chunks([&](uint32_t (&r)[16], int ch) { ln_chunk(r, ch); });
            }
            tc_fence_before();
            fence_proxy_async_smem();          // Y visible to the TMA store
            __syncwarp();
            if (lane == 0) {
                if (!regpath) arrive_leader(bar_a2empty + 8u * ab);
                mbar_arrive(bar_yfull);
            }
            if (stamp) trc[4096 + 4 * i + 3] = gtimer();
            if (++ab == (uint32_t)p.NA2) { ab = 0; aph ^= 1u; }
            if (++xs == NX) { xs = 0; xph ^= 1u; }
        }
    }

    tc_fence_before();
    if constexpr (PAIR) cluster_sync_all();   // no CTA leaves while its peer may still signal it
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (PAIR) tmem_dealloc_pair(tmem_base, 512);
        else tmem_dealloc(tmem_base, 512);
    }
    if (p.cta_stamps && threadIdx.x == 0) p.cta_stamps[2 * blockIdx.x + 1] = gtimer();
}

}  // namespace swinmlp
