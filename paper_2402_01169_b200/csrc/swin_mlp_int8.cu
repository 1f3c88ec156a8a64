// swin_mlp_int8.cu — host side of the C ABI declared in include/swin_mlp_int8.h:
// validation, constant folding, weight upload, tile/cluster planning, TMA
// descriptor encoding and stream-ordered launches of the sm_100a kernels in
// mlp_kernels.cuh.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// (tcgen05.mma.kind::i8 exists only on sm_100a).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <utility>
#include <mutex>
#include <tuple>
#include <vector>

#include "../../include/swin_mlp_int8.h"
#include "../../include/swin_attn_int8.h"
#include "mlp_kernels.cuh"
#include "attn_kernels.cuh"
#include "small_mlp.cuh"
#include "fused_mlp.cuh"
#include "op5_unfused.cuh"

using namespace swinmlp;

namespace swinmlp {
using FusedFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, FusedArgs);
FusedFn fused_kernel_part0(int flags);   // fused_mlp.cu, -DFUSED_PART=0..3 (flags >> 4)
FusedFn fused_kernel_part1(int flags);
FusedFn fused_kernel_part2(int flags);
FusedFn fused_kernel_part3(int flags);
inline FusedFn fused_kernel_for(int flags) {
    switch (flags >> 4) {
        case 0: return fused_kernel_part0(flags);
        case 1: return fused_kernel_part1(flags);
        case 2: return fused_kernel_part2(flags);
        default: return fused_kernel_part3(flags);
    }
}
}  // namespace swinmlp

namespace {

thread_local std::string g_last_error;

swin_mlp_status_t fail(swin_mlp_status_t st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(e_ == cudaErrorMemoryAllocation ? SWIN_MLP_ENOMEM : SWIN_MLP_ECUDA,     \
                        "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)


// One GEMM+epilogue launch plan.
struct Plan {
    void (*fn)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, GemmArgs) = nullptr;
    int epi = 0, threads = 0;
    int BN = 0, CS = 1, stages = 0, n_groups = 1, G = 2, out_w = 16, ebytes = 4, xstage = 1, resb = 0, yin = 0, dst = 0, wsl = 0;
    int eg = 2;     // epilogue groups: G ping-pong groups, or 1 (all 16 warps drain every tile)
    int pair = 0;   // CTA pair (cta_group::2): clusters of 2 CTAs on m-tiles 2u, 2u+1 (CS == 1)
    int one_group = 0;   // few-tile plans: every CTA drains ONE tile, so all 16 epilogue warps take it
    uint32_t smem = 0;
    int max_clusters = 0;
};

// One-kernel plan (fused_mlp.cuh): C <= 256, H % 128 == 0.
struct FusedPlan {
    bool on = false;
    FusedFn fn = nullptr;
    int NJ = 0, KBC = 0, NB1 = 0, NH = 0, stages = 0, a1_col = 0, NA2 = 1, a2_stride = 0, NX = 2, y_inplace = 0,
        stages2 = 0;
    int pair = 0;   // CTA pair (cta_group::2): clusters of 2 on m-tiles 2u, 2u+1, weights split
    uint32_t smem = 0;
};

// Programmatic dependent launch between consecutive kernels (SWIN_MLP_NO_PDL=1 disables).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SWIN_MLP_NO_PDL");
        return !(e && *e && *e != '0');
    }();
    return on;
}

bool normal_positive(float v) { return std::isfinite(v) && std::fpclassify(v) == FP_NORMAL && v > 0.0f; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// 2-D int8 tensor [rows][cols] (row stride `ld` bytes) as a TMA map with a
// {128 B along K, box_rows} box and 128-byte swizzle; out-of-range rows and
// columns read as zero (ragged T and K tails).
swin_mlp_status_t encode_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                            uint32_t box_rows, uint32_t box_cols = kBK,
                            CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto fn = encode_fn();
    if (!fn) return fail(SWIN_MLP_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(SWIN_MLP_ECUDA, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld box_rows=%u", (int)r,
                    (long long)rows, (long long)cols, box_rows);
    return SWIN_MLP_OK;
}

// 3-D view {128 B of K, rows, K-blocks} (strides ld, 128) of an int8 [rows][ld] matrix, 128-byte
// swizzle: one box {128, box_rows, box_kb} lands box_kb consecutive K-blocks as [box_kb][box_rows][128 B]
swin_mlp_status_t encode_3dk(CUtensorMap* map, const void* ptr, int64_t rows, int64_t ld, int64_t nkb, uint32_t box_rows,
                             uint32_t box_kb) {
    auto fn = encode_fn();
    if (!fn) return fail(SWIN_MLP_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    cuuint64_t dims[3] = {(cuuint64_t)kBK, (cuuint64_t)rows, (cuuint64_t)nkb};
    cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)kBK};
    cuuint32_t box[3] = {(cuuint32_t)kBK, box_rows, box_kb};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(ptr), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(SWIN_MLP_ECUDA, "cuTensorMapEncodeTiled (3-D) failed (%d) rows=%lld nkb=%lld box=%u x %u", (int)r,
                    (long long)rows, (long long)nkb, box_rows, box_kb);
    return SWIN_MLP_OK;
}

constexpr uint32_t kSmemBudget = 227 * 1024;

using KernelFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, GemmArgs);

// table index bit 3 means kSmallK for op #5 and kS64 for op #6; bit 4 (op #5) the CTA pair
template <int EPI, int I>
constexpr int flags_of() {
    return (I & 7) | ((I & 8) ? (EPI == EP6_LN ? kS64 : kSmallK) : 0) | ((I & 16) ? kPair : 0);
}
template <int EPI, int... Is>
KernelFn pick(int f, std::integer_sequence<int, Is...>, bool) {
    static const KernelFn table[] = {mlp_gemm_kernel<EPI, flags_of<EPI, Is>()>...};
    return table[f];
}

// The kernel specialised for one layer's flags (bias present, activation zero
// point, output zero point, LN precision) — no predicated-off work in the hot loop.
KernelFn kernel_for(int epi, int flags) {
    switch (epi) {
        // op #5: bias, zero points, small-K conversion (no fp64 LN); op #6: bias, zero
        // points, fp64 LN (its K = H is never small)
        case EP5_RELU: return pick<EP5_RELU>((flags & 7) | ((flags & kSmallK) ? 8 : 0) | ((flags & kPair) ? 16 : 0),
                                             std::make_integer_sequence<int, 32>{}, true);
        case EP5_GELU: return pick<EP5_GELU>((flags & 7) | ((flags & kSmallK) ? 8 : 0) | ((flags & kPair) ? 16 : 0),
                                             std::make_integer_sequence<int, 32>{}, true);
        case EP_ACC: {   // the unfused plan's FC1: only the zero-point correction and the pair matter
            static const KernelFn t[4] = {mlp_gemm_kernel<EP_ACC, 0>, mlp_gemm_kernel<EP_ACC, kHasZc>,
                                          mlp_gemm_kernel<EP_ACC, kPair>, mlp_gemm_kernel<EP_ACC, kHasZc | kPair>};
            return t[((flags & kHasZc) ? 1 : 0) | ((flags & kPair) ? 2 : 0)];
        }
        case EP2_QKV: {   // op #2: bias, input zero point, small-K conversion, CTA pair
            static const KernelFn t[16] = {
#define Q2(f) mlp_gemm_kernel<EP2_QKV, (f)>
                Q2(0), Q2(kHasB), Q2(kHasZc), Q2(kHasB | kHasZc),
                Q2(kSmallK), Q2(kSmallK | kHasB), Q2(kSmallK | kHasZc), Q2(kSmallK | kHasB | kHasZc),
                Q2(kPair), Q2(kPair | kHasB), Q2(kPair | kHasZc), Q2(kPair | kHasB | kHasZc),
                Q2(kPair | kSmallK), Q2(kPair | kSmallK | kHasB), Q2(kPair | kSmallK | kHasZc),
                Q2(kPair | kSmallK | kHasB | kHasZc)
#undef Q2
            };
            return t[((flags & kHasB) ? 1 : 0) | ((flags & kHasZc) ? 2 : 0) | ((flags & kSmallK) ? 4 : 0) |
                     ((flags & kPair) ? 8 : 0)];
        }
        default: return pick<EP6_LN>((flags & 15) | ((flags & kPair) ? 16 : 0), std::make_integer_sequence<int, 32>{},
                                     false);
    }
}

using Op5Fn = void (*)(Op5Args);
// The separate op #5 kernel of the unfused plan, specialised like the fused epilogue.
Op5Fn op5_kernel_for(bool gelu, bool has_b, bool zh) {
    static const Op5Fn t[8] = {
        op5_unfused_kernel<false, false, false>, op5_unfused_kernel<false, false, true>,
        op5_unfused_kernel<false, true, false>,  op5_unfused_kernel<false, true, true>,
        op5_unfused_kernel<true, false, false>,  op5_unfused_kernel<true, false, true>,
        op5_unfused_kernel<true, true, false>,   op5_unfused_kernel<true, true, true>};
    return t[(gelu ? 4 : 0) | (has_b ? 2 : 0) | (zh ? 1 : 0)];
}

swin_mlp_status_t prepare(Plan& pl, int num_sms) {
    // The attribute is per kernel function (process-wide), shared by every handle:
    // always grant the full budget so one layer's plan never shrinks another's.
    CUDA_TRY(cudaFuncSetAttribute(pl.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
    cudaLaunchConfig_t cfg = {};
    const int cl = pl.pair ? 2 : pl.CS;
    cfg.gridDim = dim3((unsigned)cl);
    cfg.blockDim = dim3((unsigned)pl.threads);
    cfg.dynamicSmemBytes = pl.smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, pl.fn, &cfg);
    if (e != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = num_sms / cl;
    }
    pl.max_clusters = n;
    return SWIN_MLP_OK;
}

// Columns per CTA tile, CTAs per cluster, ring depth for one GEMM.
// full_row: the epilogue needs whole rows (LayerNorm) -> the cluster must
// cover all N columns (CS * BN == N); otherwise column groups are independent.
// The first candidate whose shared-memory plan fits wins.
// Epilogue groups: G ping-pong groups, one per accumulator buffer.  (Round 1 measured one
// group of all 16 warps per tile: no gain for op #5, its drain is issue-bound at the same
// SM-wide rate, and op #6 ~1 us slower from the 4-part statistics combine; removed.)
int epilogue_groups(int, int G) { return G; }

bool fit_smem(int epi, Plan& pl, int min_stages, int K) {
    // output TMA box width: widest swizzle span dividing BN (full 128-B lines when possible)
    pl.out_w = pl.BN % 128 == 0 ? 128 : pl.BN % 64 == 0 ? 64 : pl.BN % 32 == 0 ? 32 : 16;
    const int num_kb = (K + kBK - 1) / kBK;
    // Resident B: the CTA's whole weight slice stays in smem and the ring streams
    // A (activations) only -- 2x deeper prefetch per byte of smem, and the weights
    // are read from L2 once per CTA instead of once per tile.  Tried first.
    // Weight-stationary slice (op #5, mode 2): each cluster keeps only ITS column group's
    // weights resident (half of them per CTA of a pair) and streams A tiles only -- half the
    // operand bytes per MAC of the streamed plan.  Tried after whole-B residency.
    // (Round 1 also measured weight-stationary column slices -- each cluster keeping its W1
    // slice resident: C = 512 FC1 40.0 vs 41.0 us, C = 384 22.4 vs 20.7 us, no faster because
    // FC1's tiles are gated by the op #5 drain, DESIGN.md §2.3 -- so that mode is not planned.)
    const bool no_resb = false, no_wsl = true;
    for (int mode : {1, 2, 0}) {   // 1: whole B resident, 2: this cluster's B slice, 0: streamed
    const int rb = mode != 0;
    if (mode == 1 && (no_resb || pl.pair)) continue;   // pair: B halves (mode 2 or streamed)
    if (mode == 2 && (no_wsl || epi == EP6_LN || epi == EP_ACC || pl.CS != 1 || (pl.pair && pl.BN > 256))) continue;
    const int bn_rows = pl.pair ? pl.BN / 2 : pl.BN;
    const uint32_t resb_bytes = mode == 1 ? (uint32_t)pl.n_groups * (uint32_t)num_kb * (uint32_t)pl.BN * kBK
                                          : (uint32_t)num_kb * (uint32_t)bn_rows * kBK;
    // output staging: G ping-pong groups / accumulator buffers / staging tiles, 4 when
    // 4*BN TMEM columns fit (more tiles in flight), else 2; op #6 also prefers its
    // residual x tiles staged in smem
    const int xs_max = 4;
    for (int xs : {4, 2, 1, 0}) {   // op #6 x tile buffers: one per group, one shared, none
    if (epi != EP6_LN && xs != 0) continue;
    if (xs > xs_max) continue;
    // (op #6 prefers two accumulator buffers: at C = 512 G = 4 with a 3-deep ring measured
    // 54.7 us vs 51.7 us for G = 2 with 4 stages)
    static const int kGOrderLn[3] = {2, 4, 1}, kGOrder[3] = {4, 2, 1};
    for (int gi = 0; gi < 3; ++gi) {
        const int G = epi == EP6_LN ? kGOrderLn[gi] : kGOrder[gi];
        if (G * pl.BN > 512) continue;
        if (G == 1 && (!pl.pair || epi != EP6_LN)) continue;   // (one accumulator buffer: the pair op #6 plan only)
        if (xs > 1 && xs != G) continue;
        const uint32_t rbb = rb ? resb_bytes : 0u;
        const int bn_b = pl.pair ? pl.BN / 2 : pl.BN;   // B rows per stage in one CTA
        // op #6 with one x tile per group: Y staged over its x tile (yin) frees G output tiles of
        // smem for ring stages; SWIN_MLP_NO_YIN=1 keeps separate staging (A/B switch)
        const bool no_yin = std::getenv("SWIN_MLP_NO_YIN") != nullptr;   // (read per create)
        // (op #5 storing Hq from registers to free the staging tiles for ring stages measured
        // slower in round 1 -- C = 512 FC1 43.7 us with 6 stages vs 39.2 us staged with 4 -- and is
        // not planned)
        const bool no_dst = true;
        for (int dst : {1, 0}) {
        if (dst && (epi == EP6_LN || epi == EP_ACC || no_dst)) continue;
        for (int yin : {1, 0}) {
        if (yin && (epi != EP6_LN || xs != G || no_yin)) continue;
        for (int eg : {pl.one_group ? 1 : epilogue_groups(epi, G), G}) {
        pl.eg = eg;
        pl.yin = yin;
        pl.dst = dst;
        const uint32_t stage = (uint32_t)(kBM * kBK) + (rb ? 0u : (uint32_t)bn_b * kBK);
        const int csh = epi == EP6_LN && pl.n_groups == 1;
        const uint32_t extra = smem_layout(epi, pl.BN, pl.CS, 0, G, pl.ebytes, xs, rbb, bn_b, pl.eg, yin, csh, dst).total + 1024;
        if (extra >= kSmemBudget) continue;
        int stages = (int)((kSmemBudget - extra - 64u * 8u) / stage);
        if (stages > 8) stages = 8;
        int need = min_stages;
        if (mode == 1) need = std::max(need, pl.n_groups > 1 ? num_kb + 2 : 3);   // an m-tile's k-blocks stay resident
        if (mode == 2) need = std::max(need, 3);
        if (stages < need) continue;
        pl.stages = stages;
        pl.G = G;
        pl.xstage = xs;
        pl.resb = mode == 1;
        pl.wsl = mode == 2;
        pl.smem = smem_layout(epi, pl.BN, pl.CS, stages, G, pl.ebytes, xs, rbb, bn_b, pl.eg, yin, csh, dst).total + 1024;
        if (pl.smem <= kSmemBudget) return true;
        }
        }
        }
    }
    }
    }
    return false;
}

// few-tile plans drain with one group of all 16 epilogue warps (SWIN_MLP_ONE_GROUP=0: G groups; A/B)
static int one_group_env() {
    const char* e = std::getenv("SWIN_MLP_ONE_GROUP");   // (read per create)
    return (e && *e == '0') ? 0 : 1;
}

// The one-launch plan's P / Q clusters must all be co-resident (its CTAs wait on each other).
template <class F>
static bool tiny_clusters_fit(F fn, int P, int Q) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSSmem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P);
    cfg.blockDim = dim3((unsigned)kSThreads);
    cfg.dynamicSmemBytes = kSSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)Q;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return n >= P / Q;
}

// ln_pair: -1 = the SWIN_MLP_LN_PAIR switch, 1 = only the CTA-pair op #6 plan, 0 = never it
// small_bn > 0: the few-tile plan for runs of one or two m-tiles (a 7x7 window, T = 49):
// FC1 single-CTA tiles of small_bn columns (more CTAs on the same few rows), op #6 the
// widest cluster that covers the row (CS = 8 first), so more SMs share each weight stream.
bool make_plan(int epi, int N, int K, bool full_row, Plan& pl, int ebytes = 4, int ln_pair_mode = -1,
               int small_bn = 0) {
    pl = Plan();
    pl.epi = epi;
    pl.ebytes = ebytes;
    pl.threads = kernel_threads(epi);
    if (full_row) {
        // op #6 on a CTA pair (cta_group::2, M = 256): the whole row (BN = N <= 512, two
        // N/2 MMAs past 256) in each CTA's TMEM, each CTA streaming half of every W2
        // K-block -- fewer operand bytes per MAC than the column-split cluster, but one
        // accumulator buffer (the LayerNorm drain is exposed) and a 2-deep ring.  Measured
        // slower (Swin-B b128 stack 2.03 ms vs 1.87 ms; C = 512: 27 us per tile pair), so
        // opt-in: SWIN_MLP_LN_PAIR=1 (read per create).
        const char* lp = std::getenv("SWIN_MLP_LN_PAIR");
        const bool ln_pair = ln_pair_mode < 0 ? (lp && *lp == '1') : ln_pair_mode == 1;
        if (ln_pair && N <= 512 && N > 256 && N % 64 == 0) {
            pl.BN = N; pl.CS = 1; pl.n_groups = 1; pl.pair = 1;
            if (fit_smem(epi, pl, 2, K)) return true;
            pl.pair = 0;
        }
        if (ln_pair_mode == 1) return false;
        if (small_bn > 0) {
            for (int cs : {8, 4}) {
                if (N % cs || N / cs > 256 || (N / cs) % 16) continue;
                pl.BN = N / cs; pl.CS = cs; pl.n_groups = 1; pl.one_group = one_group_env();
                if (fit_smem(epi, pl, 3, K) || fit_smem(epi, pl, 2, K)) return true;
            }
            return false;
        }
        // SWIN_MLP_LN_CS forces the op #6 cluster size (A/B switch)
        const char* cs_env = std::getenv("SWIN_MLP_LN_CS");   // (read per create)
        const int cs_force = cs_env && *cs_env ? atoi(cs_env) : 0;
        for (int cs : {1, 2, 4, 8}) {
            if (N % cs || (cs_force && cs != cs_force)) continue;
            const int bn = N / cs;
            if (bn > 256 || bn % 16) continue;
            pl.BN = bn; pl.CS = cs; pl.n_groups = 1;
            if (fit_smem(epi, pl, 3, K)) return true;   // prefer a >= 3-deep operand ring
        }
        for (int cs : {1, 2, 4, 8}) {
            if (N % cs) continue;
            const int bn = N / cs;
            if (bn > 256 || bn % 16) continue;
            pl.BN = bn; pl.CS = cs; pl.n_groups = 1;
            if (fit_smem(epi, pl, 2, K)) return true;
        }
        return false;
    }
    // op #5 with K >= 512: a CTA pair (cta_group::2, 256 x 256 tiles: each CTA streams
    // its A rows and half of B, 2/3 of the single-CTA operand bytes per MAC in a 4-deep
    // ring).  Measured on the Swin-T stages: FC1 at C = 768 2 us faster, at C = 384
    // 0.5 us slower (there the single-CTA ring already holds a whole tile's K).
    if (small_bn > 0) {
        if (N % small_bn) return false;
        pl.BN = small_bn; pl.CS = 1; pl.n_groups = N / small_bn; pl.one_group = one_group_env();
        return fit_smem(epi, pl, 3, K) || fit_smem(epi, pl, 2, K);
    }
    const bool want_pair = K >= 512;
    const int pbn = 256;   // (128-wide pair tiles with 4 accumulator buffers measured slower: 50.5 vs 36.7 us)
    if (epi != EP6_LN && want_pair && (pbn == 128 || pbn == 192 || pbn == 256) && N % pbn == 0) {
        pl.BN = pbn; pl.CS = 1; pl.n_groups = N / pbn; pl.pair = 1;
        if (fit_smem(epi, pl, 3, K)) return true;
        pl.pair = 0;
    }
    for (int bn : {256, 128, 192, 96, 64, 32}) {
        if (N % bn) continue;
        pl.BN = bn; pl.CS = 1; pl.n_groups = N / bn;
        if (fit_smem(epi, pl, 3, K) || fit_smem(epi, pl, 2, K)) return true;
    }
    return false;
}

// The one-kernel plan: weights resident in smem when they fit (W1 and W2 each
// 4C^2 bytes: C <= 128), else streamed through a ring; Hq buffers 2..4.
// (A CTA-pair one-kernel plan measured slower in round 1 -- C = 192 41.7 us vs 30.2 us
// single-CTA, C = 384 40.6 vs 35.1: halving each SM's weight stream does not pay for the
// per-chunk cross-CTA handshakes -- and is not built.)
int fused_pair_for(int) { return 0; }

bool make_fused(int C, int H, int ebytes, FusedPlan& fp, int pair) {
    fp = FusedPlan();
    fp.pair = pair;
    const char* no = std::getenv("SWIN_MLP_NO_FUSED");   // A/B switch (read per create)
    if (no && *no && *no != '0') return false;
    // C <= 256 (256 < C <= 384 -- a single acc1, FC2 as two N = C/2 MMAs -- measured at
    // C = 384, T = 12544: 35.1 us vs 33.4 us for the two-kernel plan, so not planned)
    const int maxc = 256;
    if (C > maxc || H % kFHc) return false;
    fp.KBC = (C + kBK - 1) / kBK;
    fp.NJ = H / kFHc;
    // TMEM (512 columns): acc2 buffers, then 128-column acc1 buffers.  C <= 128: two of
    // each (op #6 of one tile overlaps FC2 of the next); else one acc2 (C or 256 columns).
    //   C <= 128:  2 acc2 (128-column stride) + 2 acc1
    //   C <= 256:  1 acc2 + 2 acc1 (measured: 2 acc2 + 1 acc1 at C = 192 is slower, the
    //              single acc1 serialises FC1 and op #5)
    //   C <= 384:  1 acc2 + 1 acc1 (FC1 of chunk j+1 waits for op #5 to drain chunk j; at
    //              C = 384 the alternative is the two-kernel plan, whose GEMM tiles are
    //              bound by operand ingest and an exposed LayerNorm drain)
    if (C <= 128) { fp.NA2 = 2; fp.a2_stride = 128; fp.a1_col = 256; }
    else if (C <= 256) { fp.NA2 = 1; fp.a2_stride = 0; fp.a1_col = 256; }
    else { fp.NA2 = 1; fp.a2_stride = 0; fp.a1_col = 384; }
    fp.NB1 = (512 - fp.a1_col) / kFHc;
    // resident weights first (X slots 4..2, Hq buffers 3..2), else a weight ring
    for (int nx : {4, 3, 2}) {
        if (pair) break;   // (a pair streams its weights)
        for (int nh : {3, 2}) {
            const uint32_t need = fused_layout(C, H, nh, 0, ebytes, nx).total + 1024;
            if (need <= kSmemBudget) {
                fp.NX = nx; fp.NH = nh; fp.stages = 0; fp.smem = need; fp.on = true;
                return true;
            }
        }
    }
    // streamed weights: two rings (W1 K-blocks, W2 chunks) so the W1 items of the next
    // chunks load while FC2 still holds W2 items; Y staged over its X slot (frees a Y
    // buffer); the W1 ring as deep as fits (measured at C = 192: a 2-CTA cluster
    // multicasting the weight items, or W2 split in two items, did not help)
    const int yin = 1;
    // C > 256: one X slot (a CTA gets about one tile) so the weight rings get the smem
    for (int nx : {C > 256 ? 1 : 2, C > 256 ? 2 : 1}) {
    // W2 ring: up to two chunks of items (C > 256: two half-chunk items per chunk), then the
    // deepest W1 ring that fits
    const int w2n = C > 256 ? 2 : 1;
    for (int st2 = std::min(kFMaxStages2, 2 * w2n); st2 >= 1; --st2) {
        for (int st = kFMaxStages; st >= (fp.NB1 > 1 ? 2 * fp.KBC : 2); --st) {
            const uint32_t need = fused_layout(C, H, 2, st, ebytes, nx, yin, st2, pair).total + 1024;
            if (need <= kSmemBudget) {
                fp.NX = nx; fp.NH = 2; fp.stages = st; fp.stages2 = st2; fp.smem = need; fp.on = true;
                fp.y_inplace = yin;
                return true;
            }
        }
    }
    }
    return false;
}

swin_mlp_status_t launch(const Plan& pl, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to,
                         const CUtensorMap& tx, const GemmArgs& a, cudaStream_t stream) {
    // independent work items: m-tiles in m-major order, (m, n) units otherwise
    const int64_t units = a.mt_major ? a.num_units / a.n_groups : a.num_units;
    int64_t clusters = units < pl.max_clusters ? units : pl.max_clusters;
    // weight-stationary slices: the same number of clusters on every column group
    if (a.wsl && clusters > a.n_groups) clusters -= clusters % a.n_groups;
    if (clusters < 1) clusters = 1;
    cudaLaunchConfig_t cfg = {};
    const int cl = pl.pair ? 2 : pl.CS;   // CTAs per cluster
    cfg.gridDim = dim3((unsigned)(clusters * cl));
    cfg.blockDim = dim3((unsigned)pl.threads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (see the kernels)
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, pl.fn, ta, tb, to, tx, a));
    static const bool sync_check = std::getenv("SWIN_MLP_SYNC_CHECK") != nullptr;
    if (sync_check) {   // debug: surface asynchronous kernel faults at the launch that caused them
        CUDA_TRY(cudaStreamSynchronize(stream));
        CUDA_TRY(cudaGetLastError());
    }
    return SWIN_MLP_OK;
}

}  // namespace

struct swin_mlp_int8_s {
    swin_mlp_int8_desc_t d;   // scalars; pointers not retained
    int device = 0, num_sms = 0;
    Plan p1, p2;
    FusedPlan fp;          // one-kernel plan (used when fp.on)
    FusedFn fp_dbg = nullptr;   // its tap-writing variant (run_debug)
    bool unfused = false;       // desc.op5_unfused: FC1 (EP_ACC) -> op5_fn -> FC2 + op #6
    Op5Fn op5_fn = nullptr;
    int op5_grid = 0;
    // the shift-GELU control (act == SWIN_MLP_ACT_SHIFT_GELU, always unfused): row-max op #5 kernel
    void (*sg_fn)(ShiftGeluArgs) = nullptr;
    ShiftGeluArgs sg = {};
    int sg_grid = 0;
    CUtensorMap tm_fw1, tm_fw2;
    // device copies (handle-owned)
    int8_t *w1 = nullptr, *w2 = nullptr;
    float *m1 = nullptr, *b1 = nullptr, *m2 = nullptr, *b2 = nullptr, *gamma = nullptr, *beta = nullptr;
    int32_t *zc1 = nullptr, *zc2 = nullptr;
    // host copies of the folded constants (debug getter)
    std::vector<float> hm1, hm2;
    std::vector<int32_t> hws1, hws2;
    float inv_h = 0.f, inv_y = 0.f;
    CUtensorMap tm_w1, tm_w2;
    // few-tile alternative for op #6 (256 < C <= 512): the CTA-pair whole-row plan, used when
    // the run has at most 2 * p2b.max_clusters m-tiles (one wave of pairs) -- measured faster
    // there (C = 384, T = 12544: 22.7 vs 25.4 us; C = 512, T = 12544: 28.8 vs 30.9 us) and
    // slower for more tiles (C = 512, T = 25088: 47.2 vs 39.9 us)
    Plan p2b;
    bool has_p2b = false;
    CUtensorMap tm_w2b;
    // few-tile plans (make_plan small_bn): used when the default plans would put both
    // GEMMs of the run on fewer than num_sms / 4 CTAs (configs[0]: one 7x7 window, T = 49,
    // C = 768 -- FC1 12 CTA pairs, op #6 one cluster of 4).  SWIN_MLP_SMALL=0 disables,
    // SWIN_MLP_SMALL_BN picks the FC1 tile width (default 64).
    Plan p1s, p2s;
    bool has_small = false;
    CUtensorMap tm_w1s, tm_w2s;
    // one-launch plan for runs of at most kSMaxT tokens (small_mlp.cuh): P = H / 128 CTAs
    bool has_tiny = false;
    int tiny_P = 0, tiny_Q = 0, tiny_PR = 0;   // CTAs, cluster size, FC2 columns per CTA (Q * PR == C)
    CUtensorMap tm_w1t, tm_w2t;
    int32_t* tiny_cnt = nullptr;   // [2] arrival / departure counters (zero between runs)
    int32_t* tiny_acc = nullptr;   // [64][C] int32 FC2 sums (zero between runs)
    void (*tiny_fn)(CUtensorMap, CUtensorMap, CUtensorMap, SmallArgs) = nullptr;
    std::vector<void*> allocs;
    // native profiling (bench roofline): event triples per recorded run
    bool prof_on = false;
    int prof_max = 0, prof_n = 0;
    std::vector<cudaEvent_t> prof_ev;
    unsigned long long* trace = nullptr;
    int trace_cta = 0;
    // activation tensor maps of recent runs (encoding costs microseconds of host time per
    // map; a serving loop reuses the same buffers): key -> map, small linear cache
    struct MapKey {
        const void* ptr; int64_t rows, cols, ld; uint32_t box_rows, box_cols; int swz;
        bool operator==(const MapKey& o) const {
            return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows &&
                   box_cols == o.box_cols && swz == o.swz;
        }
    };
    std::vector<std::pair<MapKey, CUtensorMap>> map_cache;
    size_t map_next = 0;
    std::mutex map_mu;
    // run_host pipeline: copy-in and copy-out streams + per-chunk events (created lazily)
    cudaStream_t io_in = nullptr, io_out = nullptr;
    std::vector<cudaEvent_t> io_ev;
    // plan hint (swin_mlp_int8_set_plan_hint): > 0 = runs choose their launch plans as a run of
    // plan_hint tokens would, so shards / chunks of one batch run the batch's plan
    int64_t plan_hint = 0;
    // op #6 split-K for runs of few m-tiles (SWIN_MLP_KSPLIT=0 disables; A/B switch read per create)
    bool ksplit_on = true;
    ~swin_mlp_int8_s() {
        for (void* p : allocs) cudaFree(p);
        for (cudaEvent_t e : prof_ev) cudaEventDestroy(e);
        for (cudaEvent_t e : io_ev) cudaEventDestroy(e);
        if (io_in) cudaStreamDestroy(io_in);
        if (io_out) cudaStreamDestroy(io_out);
    }
};

// Which plan pair a run of T tokens takes (two-kernel path): 0 = the default plans,
// 1 = the CTA-pair op #6 (p2b, at most one wave of pairs), 2 = the few-tile plans
// (p1s/p2s: the defaults would put both GEMMs on fewer than num_sms / 4 CTAs).
static int plan_choice(const swin_mlp_int8_s* h, int64_t T) {
    if (h->has_tiny && T <= kSMaxT) return 3;   // one launch (small_mlp.cuh)
    const int64_t m_tiles = (T + kBM - 1) / kBM;
    const int64_t units1 = (h->p1.pair ? (m_tiles + 1) / 2 * 2 : m_tiles) * h->p1.n_groups;
    const int64_t units2 = (h->p2.pair ? (m_tiles + 1) / 2 * 2 : m_tiles) * h->p2.CS;
    if (h->has_small && units1 + units2 < h->num_sms / 4) return 2;
    if (h->has_p2b && m_tiles <= 2 * (int64_t)h->p2b.max_clusters) return 1;
    return 0;
}

namespace {

// encode_2d through the handle's cache of activation maps
swin_mlp_status_t encode_cached(swin_mlp_int8_s* h, CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols,
                                int64_t ld, uint32_t box_rows, uint32_t box_cols = kBK,
                                CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    const swin_mlp_int8_s::MapKey key{ptr, rows, cols, ld, box_rows, box_cols, (int)swz};
    {
        std::lock_guard<std::mutex> lk(h->map_mu);
        for (auto& e : h->map_cache)
            if (e.first == key) { *map = e.second; return SWIN_MLP_OK; }
    }
    const swin_mlp_status_t st = (int)swz < 0 ? encode_3dk(map, ptr, rows, ld, cols, box_rows, box_cols)
                                              : encode_2d(map, ptr, rows, cols, ld, box_rows, box_cols, swz);
    if (st != SWIN_MLP_OK) return st;
    std::lock_guard<std::mutex> lk(h->map_mu);
    constexpr size_t kCap = 64;
    if (h->map_cache.size() < kCap) h->map_cache.emplace_back(key, *map);
    else { h->map_cache[h->map_next] = {key, *map}; h->map_next = (h->map_next + 1) % kCap; }
    return SWIN_MLP_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename T>
swin_mlp_status_t fetch(const T* src, size_t n, std::vector<T>& out, const char* name) {
    if (!src) return fail(SWIN_MLP_EINVAL, "%s is NULL", name);
    out.resize(n);
    CUDA_TRY(cudaMemcpy(out.data(), src, n * sizeof(T), cudaMemcpyDefault));
    return SWIN_MLP_OK;
}

template <typename T>
swin_mlp_status_t upload(swin_mlp_int8_s* h, const std::vector<T>& v, T** dst) {
    void* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, v.size() * sizeof(T) + 16));
    h->allocs.push_back(p);
    CUDA_TRY(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    *dst = static_cast<T*>(p);
    return SWIN_MLP_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

#define ST_TRY(...)                                 \
    do {                                            \
        swin_mlp_status_t s_ = (__VA_ARGS__);       \
        if (s_ != SWIN_MLP_OK) return s_;           \
    } while (0)

extern "C" {

const char* swin_mlp_int8_last_error(void) { return g_last_error.c_str(); }

swin_mlp_status_t swin_mlp_int8_create(const swin_mlp_int8_desc_t* desc, swin_mlp_int8_t* out) {
    g_last_error.clear();
    if (!desc || !out) return fail(SWIN_MLP_EINVAL, "desc and out must be non-NULL");
    const swin_mlp_int8_desc_t& d = *desc;
    if (d.C < 32 || d.C % 32) return fail(SWIN_MLP_EINVAL, "C=%d must be a multiple of 32 and >= 32", d.C);
    if (d.H < d.C || d.H % 32) return fail(SWIN_MLP_EINVAL, "H=%d must be a multiple of 32 and >= C", d.H);
    if (d.C > 1536 || d.H > 6144) return fail(SWIN_MLP_EUNSUPPORTED, "C=%d H=%d exceed 1536/6144", d.C, d.H);
    if (d.act != SWIN_MLP_ACT_RELU && d.act != SWIN_MLP_ACT_GELU_ERF && d.act != SWIN_MLP_ACT_SHIFT_GELU)
        return fail(SWIN_MLP_EINVAL, "unknown activation %d", (int)d.act);
    if (d.act == SWIN_MLP_ACT_SHIFT_GELU) {
        if (!normal_positive(d.gelu_in_scale)) return fail(SWIN_MLP_EINVAL, "gelu_in_scale must be finite, normal and > 0");
        volatile float S = 1.702f * d.gelu_in_scale;
        if (!(1.0 / (double)S < (double)(1 << 26))) return fail(SWIN_MLP_EINVAL, "gelu_in_scale too small (1/(1.702 s_g) >= 2^26)");
    }
    if (d.op5_unfused != 0 && d.op5_unfused != 1) return fail(SWIN_MLP_EINVAL, "op5_unfused=%d must be 0 or 1", d.op5_unfused);
    if (!normal_positive(d.x_scale) || !normal_positive(d.h_scale) || !normal_positive(d.y_scale))
        return fail(SWIN_MLP_EINVAL, "activation scales must be finite, normal and > 0");
    if (!(d.ln_eps > 0.0f) || !std::isfinite(d.ln_eps)) return fail(SWIN_MLP_EINVAL, "ln_eps must be > 0");
    for (int32_t z : {d.x_zero_point, d.h_zero_point, d.y_zero_point})
        if (z < -128 || z > 127) return fail(SWIN_MLP_EINVAL, "zero point %d outside [-128, 127]", z);
    if (!d.w1 || !d.w2 || !d.w1_scale || !d.w2_scale || !d.ln_gamma || !d.ln_beta)
        return fail(SWIN_MLP_EINVAL, "w1, w2, w1_scale, w2_scale, ln_gamma, ln_beta are required");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (d.device < 0 || d.device >= ndev) return fail(SWIN_MLP_EINVAL, "device %d of %d", d.device, ndev);
    DeviceGuard guard(d.device);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(SWIN_MLP_EUNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", d.device,
                    prop.major, prop.minor);

    const int C = d.C, H = d.H;
    std::vector<int8_t> w1, w2;
    std::vector<float> sw1, sw2, b1, b2, g, bt;
    ST_TRY(fetch(d.w1, (size_t)H * C, w1, "w1"));
    ST_TRY(fetch(d.w2, (size_t)C * H, w2, "w2"));
    ST_TRY(fetch(d.w1_scale, (size_t)H, sw1, "w1_scale"));
    ST_TRY(fetch(d.w2_scale, (size_t)C, sw2, "w2_scale"));
    ST_TRY(fetch(d.ln_gamma, (size_t)C, g, "ln_gamma"));
    ST_TRY(fetch(d.ln_beta, (size_t)C, bt, "ln_beta"));
    if (d.b1) ST_TRY(fetch(d.b1, (size_t)H, b1, "b1"));
    if (d.b2) ST_TRY(fetch(d.b2, (size_t)C, b2, "b2"));

    auto h = new swin_mlp_int8_s();
    h->d = d;
    h->d.w1 = h->d.w2 = nullptr;
    h->d.w1_scale = h->d.w2_scale = h->d.b1 = h->d.b2 = h->d.ln_gamma = h->d.ln_beta = nullptr;
    h->device = d.device;
    h->num_sms = prop.multiProcessorCount;
    auto bail = [&](swin_mlp_status_t st) {
        delete h;
        return st;
    };

    // O0: folded constants, literal fp32 formulas (one rounding each).
    h->hm1.resize(H);
    h->hm2.resize(C);
    for (int n = 0; n < H; ++n) {
        if (!normal_positive(sw1[n])) return bail(fail(SWIN_MLP_EINVAL, "w1_scale[%d] not finite/normal/positive", n));
        volatile float m = d.x_scale * sw1[n];
        h->hm1[n] = m;
        if (!normal_positive(h->hm1[n])) return bail(fail(SWIN_MLP_EINVAL, "x_scale*w1_scale[%d] not normal", n));
    }
    for (int c = 0; c < C; ++c) {
        if (!normal_positive(sw2[c])) return bail(fail(SWIN_MLP_EINVAL, "w2_scale[%d] not finite/normal/positive", c));
        volatile float m = d.h_scale * sw2[c];
        h->hm2[c] = m;
        if (!normal_positive(h->hm2[c])) return bail(fail(SWIN_MLP_EINVAL, "h_scale*w2_scale[%d] not normal", c));
    }
    {
        volatile float one = 1.0f;
        h->inv_h = one / d.h_scale;
        h->inv_y = one / d.y_scale;
    }
    if (!normal_positive(h->inv_h) || !normal_positive(h->inv_y))
        return bail(fail(SWIN_MLP_EINVAL, "1/h_scale or 1/y_scale not normal"));
    // int32 zero-point corrections z * sum_k W[n][k]
    h->hws1.assign(H, 0);
    h->hws2.assign(C, 0);
    std::vector<int32_t> zc1(H), zc2(C);
    for (int n = 0; n < H; ++n) {
        int64_t s = 0;
        for (int k = 0; k < C; ++k) {
            if (w1[(size_t)n * C + k] == -128) return bail(fail(SWIN_MLP_EINVAL, "w1 must be symmetric (-128 not allowed)"));
            s += w1[(size_t)n * C + k];
        }
        h->hws1[n] = (int32_t)s;
        zc1[n] = (int32_t)(s * d.x_zero_point);
    }
    for (int c = 0; c < C; ++c) {
        int64_t s = 0;
        for (int k = 0; k < H; ++k) {
            if (w2[(size_t)c * H + k] == -128) return bail(fail(SWIN_MLP_EINVAL, "w2 must be symmetric (-128 not allowed)"));
            s += w2[(size_t)c * H + k];
        }
        h->hws2[c] = (int32_t)s;
        zc2[c] = (int32_t)(s * d.h_zero_point);
    }

    // tile / cluster plans
    h->unfused = d.op5_unfused != 0 || d.act == SWIN_MLP_ACT_SHIFT_GELU;   // (shift-GELU: the row max)
    const int epi1 = h->unfused ? EP_ACC : d.act == SWIN_MLP_ACT_RELU ? EP5_RELU : EP5_GELU;
    if (!make_plan(epi1, H, C, false, h->p1)) return bail(fail(SWIN_MLP_EUNSUPPORTED, "no FC1 tile plan for H=%d", H));
    if (!make_plan(EP6_LN, C, H, true, h->p2, d.ln_fp64 ? 8 : 4))
        return bail(fail(SWIN_MLP_EUNSUPPORTED, "no FC2 tile plan for C=%d (needs C = CS*BN, BN%%16==0, BN<=256, CS in 1,2,4,8)", C));

    swin_mlp_status_t st;
#define H_TRY(expr)                                   \
    do {                                              \
        if ((st = (expr)) != SWIN_MLP_OK) return bail(st); \
    } while (0)
    H_TRY(upload(h, w1, &h->w1));
    H_TRY(upload(h, w2, &h->w2));
    H_TRY(upload(h, h->hm1, &h->m1));
    H_TRY(upload(h, h->hm2, &h->m2));
    H_TRY(upload(h, g, &h->gamma));
    H_TRY(upload(h, bt, &h->beta));
    if (d.b1) H_TRY(upload(h, b1, &h->b1));
    if (d.b2) H_TRY(upload(h, b2, &h->b2));
    if (d.x_zero_point) H_TRY(upload(h, zc1, &h->zc1));
    if (d.h_zero_point) H_TRY(upload(h, zc2, &h->zc2));
    H_TRY(encode_2d(&h->tm_w1, h->w1, H, C, C, (uint32_t)(h->p1.pair ? h->p1.BN / 2 : h->p1.BN)));
    // W2 boxes: BN rows, or (pair) the BN/4 or BN/2 rows a CTA holds per MMA half
    H_TRY(encode_2d(&h->tm_w2, h->w2, C, H, H,
                    (uint32_t)(h->p2.pair ? (h->p2.BN > 256 ? h->p2.BN / 4 : h->p2.BN / 2) : h->p2.BN)));
    // |A1[t][n]| = |sum_k (X - z_x) W1[n][k]| <= (128 + |z_x|) * max_n sum_k |W1[n][k]| (a rigorous
    // bound from the actual weights, tighter than 127 * C): below 2^22 the exact magic-number
    // int->float applies (for max-abs-quantised Gaussian weights this holds up to C ~ 768)
    int64_t w1_rowabs = 0;
    for (int n = 0; n < H; ++n) {
        int64_t s = 0;
        for (int k = 0; k < C; ++k) s += std::abs((int)w1[(size_t)n * C + k]);
        w1_rowabs = std::max(w1_rowabs, s);
    }
    const bool small_k1 = (int64_t)(128 + std::abs(d.x_zero_point)) * w1_rowabs < (int64_t(1) << 22);
    h->p1.fn = kernel_for(epi1,
                          (d.b1 ? kHasB : 0) | (d.x_zero_point ? kHasZc : 0) | (d.h_zero_point ? kZqNz : 0) |
                          (small_k1 ? kSmallK : 0) | (h->p1.pair ? kPair : 0));
    h->p2.fn = kernel_for(EP6_LN, (d.b2 ? kHasB : 0) | (d.h_zero_point ? kHasZc : 0) |
                                      (d.y_zero_point ? kZqNz : 0) | (d.ln_fp64 ? kS64 : 0) |
                                      (h->p2.pair ? kPair : 0));
    H_TRY(prepare(h->p1, h->num_sms));
    H_TRY(prepare(h->p2, h->num_sms));
    {
        const char* lp = std::getenv("SWIN_MLP_LN_PAIR");   // '0': never the pair plan
        if (!h->p2.pair && !(lp && *lp == '0') && make_plan(EP6_LN, C, H, true, h->p2b, d.ln_fp64 ? 8 : 4, 1)) {
            H_TRY(encode_2d(&h->tm_w2b, h->w2, C, H, H, (uint32_t)(h->p2b.BN > 256 ? h->p2b.BN / 4 : h->p2b.BN / 2)));
            h->p2b.fn = kernel_for(EP6_LN, (d.b2 ? kHasB : 0) | (d.h_zero_point ? kHasZc : 0) |
                                               (d.y_zero_point ? kZqNz : 0) | (d.ln_fp64 ? kS64 : 0) | kPair);
            H_TRY(prepare(h->p2b, h->num_sms));
            h->has_p2b = true;
        }
    }
    {
        const char* ke = std::getenv("SWIN_MLP_KSPLIT");      // (read per create)
        h->ksplit_on = !(ke && *ke == '0');
    }
    {
        const char* se = std::getenv("SWIN_MLP_SMALL");       // (read per create)
        const int sbn = 64;   // (BN = 32 / 128 measured no better at the layer level)
        if (!h->unfused && !(se && *se == '0') && sbn >= 16 && sbn % 16 == 0 &&
            make_plan(epi1, H, C, false, h->p1s, 4, -1, sbn) &&
            make_plan(EP6_LN, C, H, true, h->p2s, d.ln_fp64 ? 8 : 4, 0, sbn)) {
            H_TRY(encode_2d(&h->tm_w1s, h->w1, H, C, C, (uint32_t)h->p1s.BN));
            H_TRY(encode_2d(&h->tm_w2s, h->w2, C, H, H, (uint32_t)h->p2s.BN));
            h->p1s.fn = kernel_for(epi1, (d.b1 ? kHasB : 0) | (d.x_zero_point ? kHasZc : 0) |
                                             (d.h_zero_point ? kZqNz : 0) | (small_k1 ? kSmallK : 0));
            h->p2s.fn = kernel_for(EP6_LN, (d.b2 ? kHasB : 0) | (d.h_zero_point ? kHasZc : 0) |
                                               (d.y_zero_point ? kZqNz : 0) | (d.ln_fp64 ? kS64 : 0));
            H_TRY(prepare(h->p1s, h->num_sms));
            H_TRY(prepare(h->p2s, h->num_sms));
            h->has_small = true;
        }
    }
    {
        // one-launch plan for T <= 64: fp32 LayerNorm, C % 128 == 0 (the row's float4 groups per
        // lane), H / 128 CTAs all co-resident, FC2 output in pieces of <= 256 columns
        const char* te = std::getenv("SWIN_MLP_TINY");   // '0': never (A/B switch, read per create)
        const int P = H / 128;
        // the smallest cluster size Q (P % Q == 0, Q <= 8) whose column group PR = C / Q fits one
        // MMA (<= 256) and splits into two warp halves of 16-column chunks
        const char* qe = std::getenv("SWIN_MLP_TINY_Q");   // A/B: the smallest valid Q >= this (read per create)
        int Q = (qe && *qe) ? std::max(1, std::atoi(qe)) : 1;
        while (Q <= kSMaxQ && (P % Q || C % Q || C / Q > 256 || (C / Q) % 32)) ++Q;
        const int PR = Q <= kSMaxQ ? C / Q : 0;
        void (*tfn)(CUtensorMap, CUtensorMap, CUtensorMap, SmallArgs) = nullptr;
        const bool gl = d.act == SWIN_MLP_ACT_GELU_ERF;
        switch (C / 128) {   // the LayerNorm row groups per lane (C % 128 == 0)
#define TINY(g) case g: tfn = gl ? small_mlp_kernel<g, 1> : small_mlp_kernel<g, 0>; break;
            TINY(3) TINY(4) TINY(5) TINY(6) TINY(8) TINY(10) TINY(12)
#undef TINY
            default: break;
        }
        if (!(te && *te == '0') && tfn && !h->unfused && !d.ln_fp64 && C >= 384 && C % 128 == 0 && H % 128 == 0 &&
            P <= h->num_sms && Q <= kSMaxQ && PR * Q == C && PR % 32 == 0 && PR <= 256 &&
            tiny_clusters_fit(tfn, P, Q)) {
            h->tiny_fn = tfn;
            if (C / 128 <= kSResKB) {   // resident mode: one 3-D op per operand (small_mlp.cuh)
                H_TRY(encode_3dk(&h->tm_w1t, h->w1, H, C, C / 128, 128, (uint32_t)(C / 128)));
                H_TRY(encode_3dk(&h->tm_w2t, h->w2, C, H, H / 128, (uint32_t)PR, (uint32_t)Q));
            } else {
                H_TRY(encode_2d(&h->tm_w1t, h->w1, H, C, C, 128));
                H_TRY(encode_2d(&h->tm_w2t, h->w2, C, H, H, (uint32_t)PR));
            }
            void* cp = nullptr;
            const size_t acc_bytes = (size_t)kSMaxT * C * 4;
            CUDA_TRY(cudaMalloc(&cp, acc_bytes + 256));
            h->allocs.push_back(cp);
            CUDA_TRY(cudaMemset(cp, 0, acc_bytes + 256));
            h->tiny_acc = static_cast<int32_t*>(cp);
            h->tiny_cnt = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(cp) + acc_bytes);
            CUDA_TRY(cudaFuncSetAttribute(tfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSSmem));
            h->tiny_P = P; h->tiny_Q = Q; h->tiny_PR = PR;
            h->has_tiny = true;
        }
    }
    if (h->unfused && d.act == SWIN_MLP_ACT_SHIFT_GELU) {
        static void (*const sgt[4])(ShiftGeluArgs) = {op5_shiftgelu_kernel<false, false>, op5_shiftgelu_kernel<false, true>,
                                                      op5_shiftgelu_kernel<true, false>, op5_shiftgelu_kernel<true, true>};
        h->sg_fn = sgt[(d.b1 ? 2 : 0) | (d.h_zero_point ? 1 : 0)];
        volatile float one = 1.0f;
        volatile float inv_g = one / d.gelu_in_scale;
        volatile float S = 1.702f * d.gelu_in_scale;
        volatile float sgih = d.gelu_in_scale * h->inv_h;
        volatile float k_g = sgih * 0.0078125f;
        h->sg.inv_g = inv_g; h->sg.k_g = k_g;
        h->sg.x0 = (int32_t)std::floor(-1.0 / (double)S);
        h->sg.divx0 = make_fastdiv((uint32_t)(-h->sg.x0));
        h->sg.z_h = d.h_zero_point;
        int per_sm = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h->sg_fn, kOp5Threads, 0));
        h->sg_grid = std::max(1, per_sm) * h->num_sms;
    } else if (h->unfused) {
        h->op5_fn = op5_kernel_for(d.act == SWIN_MLP_ACT_GELU_ERF, d.b1 != nullptr, d.h_zero_point != 0);
        int per_sm = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h->op5_fn, kOp5Threads, 0));
        h->op5_grid = std::max(1, per_sm) * h->num_sms;   // persistent grid-stride: whole waves
    } else if (make_fused(C, H, d.ln_fp64 ? 8 : 4, h->fp, fused_pair_for(C))) {
        const int ff = (d.act == SWIN_MLP_ACT_GELU_ERF ? kFGelu : 0) | (d.h_zero_point ? kFZh : 0) |
                       (d.b1 ? kFB1 : 0) | (d.ln_fp64 ? kFS64 : 0) | (small_k1 ? kFSmallK : 0);
        const int fpair = h->fp.pair ? kFPair : 0;
        h->fp.fn = fused_kernel_for(ff | fpair);
        h->has_small = false;   // (the one-kernel plan serves every T: no per-run plans)
        h->fp_dbg = fused_kernel_for(ff | kFTaps | fpair);
        H_TRY(encode_2d(&h->tm_fw1, h->w1, H, C, C, (uint32_t)(h->fp.pair ? kFHc / 2 : kFHc)));
        H_TRY(encode_2d(&h->tm_fw2, h->w2, C, H, H, fused_w2_rows(C, h->fp.pair)));
        CUDA_TRY(cudaFuncSetAttribute(h->fp.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
        CUDA_TRY(cudaFuncSetAttribute(h->fp_dbg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
    }
#undef H_TRY
    *out = h;
    return SWIN_MLP_OK;
}

// op #6 split-K region of the workspace: int32 partial sums [rows][C] + counters [m_tiles][CS],
// for runs of at most two m-tiles (the only runs ksplit_for splits)
static int64_t split_rows_cap(const swin_mlp_int8_s*) { return 2 * (int64_t)kBM; }
static size_t split_region_bytes(const swin_mlp_int8_s* h, int64_t T) {
    const int64_t rows = std::min<int64_t>(T, split_rows_cap(h));
    const int64_t words = (rows * h->d.C + 3) / 4 * 4 + ((rows + kBM - 1) / kBM * 8 + 3) / 4 * 4;
    return (size_t)((words * 4 + 127) / 128 * 128);
}

// Split-K factor of op #6 for a run of T tokens on plan P2 (1 = none): only when the unsplit grid
// fills at most half the SMs, with every (m-tile, split) unit on its own co-resident cluster (the
// reducer waits for its partners) and the int32 partial tile fitting the operand ring.
static int ksplit_for(const swin_mlp_int8_s* h, const Plan& P2, int64_t T, int& kb_per) {
    kb_per = 0;
    if (!h->ksplit_on || h->unfused || P2.pair || P2.resb) return 1;
    const int64_t m_tiles = (T + kBM - 1) / kBM;
    // (measured: a win for one m-tile -- C = 768 / 1024 / 1536 at T = 49: 31.6 -> 29.7, 37.9 -> 31.7,
    // 48.2 -> 35.9 us per layer -- a loss from 13 m-tiles on: C = 768, T = 1568 36 -> 42 us, the
    // partials' global reduce-add and the reducer's wait outweigh the shorter K loops)
    if (m_tiles > 2 || m_tiles * P2.CS * 2 > h->num_sms) return 1;
    const int num_kb = (h->d.H + kBK - 1) / kBK;
    int64_t S = std::min<int64_t>(num_kb, P2.max_clusters / std::max<int64_t>(m_tiles, 1));
    if (S < 2) return 1;
    kb_per = (int)((num_kb + S - 1) / S);
    S = (num_kb + kb_per - 1) / kb_per;
    if ((uint64_t)P2.stages * ((uint64_t)kBM * kBK + (uint64_t)P2.BN * kBK) < (uint64_t)kBM * ksplit_row_bytes(P2.BN)) return 1;
    return (int)S;
}

size_t swin_mlp_int8_workspace_bytes(swin_mlp_int8_t h, int64_t T) {
    if (!h || T <= 0) return 0;
    if (h->fp.on) return 0;   // one kernel: the hidden tile never leaves the SM
    const size_t hq = (size_t)(((T * h->d.H) + 127) / 128 * 128);
    if (h->unfused) return hq + (size_t)T * h->d.H * 4;   // unfused plan: + A1 int32 [T][H]
    const size_t two = hq + split_region_bytes(h, T);      // + op #6 split-K partials (small T)
    return two;   // (the one-launch plan, T <= 64, uses handle-owned buffers only)
}

// plan_T: the token count the launch plans are chosen for (the run's own T, the handle's plan
// hint, or -- run_host / run_host_batch -- the whole call's T, so every chunk of one call runs
// one plan and the result does not depend on the chunking; R20)
static swin_mlp_status_t run_impl(swin_mlp_int8_t h, const int8_t* x, const float* residual, int8_t* y,
                                  float* residual_out, int64_t T, void* workspace, size_t ws_bytes, void* stream,
                                  int32_t* acc1, int8_t* hidden, int32_t* acc2, float* ln_out, bool dbg,
                                  int64_t plan_T = 0) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (T < 0) return fail(SWIN_MLP_EINVAL, "T=%lld < 0", (long long)T);
    if (T == 0) return SWIN_MLP_OK;
    if (T > (int64_t)1 << 31) return fail(SWIN_MLP_EUNSUPPORTED, "T=%lld too large", (long long)T);
    const size_t ws_need = swin_mlp_int8_workspace_bytes(h, T);
    if (!x || !y || (ws_need && !workspace)) return fail(SWIN_MLP_EINVAL, "x, y and workspace are required");
    if (!aligned16(x) || !aligned16(y) || (residual && !aligned16(residual)) ||
        (residual_out && !aligned16(residual_out)) || (reinterpret_cast<uintptr_t>(workspace) & 127u))
        return fail(SWIN_MLP_EINVAL, "x/y/residual/residual_out must be 16-byte aligned, workspace 128-byte aligned");
    if (ws_bytes < ws_need) return fail(SWIN_MLP_EINVAL, "workspace %zu < %zu bytes", ws_bytes, ws_need);
    if ((const void*)x == (const void*)y) return fail(SWIN_MLP_EINVAL, "y may not alias x");
    const int C = h->d.C, H = h->d.H;
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int8_t* hq = static_cast<int8_t*>(workspace);

    if (h->fp.on) {
        CUtensorMap fx, fy;
        ST_TRY(encode_cached(h, &fx, x, T, C, C, kBM));
        ST_TRY(encode_cached(h, &fy, y, T, C, C, kBM));
        FusedArgs a = {};
        a.M = T; a.C = C; a.H = H;
        a.NJ = h->fp.NJ; a.KBC = h->fp.KBC; a.NB1 = h->fp.NB1; a.NH = h->fp.NH; a.stages = h->fp.stages;
        a.a1_col = h->fp.a1_col; a.NA2 = h->fp.NA2; a.a2_stride = h->fp.a2_stride; a.NX = h->fp.NX;
        a.y_inplace = h->fp.y_inplace; a.stages2 = h->fp.stages2;
        a.m1 = h->m1; a.b1 = h->b1; a.zc1 = h->zc1;
        a.m2 = h->m2; a.b2 = h->b2; a.zc2 = h->zc2;
        a.gamma = h->gamma; a.beta = h->beta;
        a.inv_h = h->inv_h; a.z_h = h->d.h_zero_point; a.inv_y = h->inv_y; a.z_y = h->d.y_zero_point;
        a.s_x = h->d.x_scale; a.z_x = h->d.x_zero_point; a.eps = h->d.ln_eps; a.one = 1.0f;
        a.x = x; a.resid = residual; a.resid_out = residual_out;
        a.rotate = 1;
        if (dbg) { a.acc1_tap = acc1; a.hid_tap = hidden; a.acc2_tap = acc2; a.ln_tap = ln_out; }
        a.trace = h->trace; a.trace_cta = h->trace_cta;
        a.cta_stamps = h->trace ? h->trace + 8192 : nullptr;
        const int64_t m_tiles = (T + kBM - 1) / kBM;
        cudaLaunchConfig_t cfg = {};
        if (h->fp.pair)   // clusters of 2 CTAs on m-tile pairs
            cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>((m_tiles + 1) / 2, h->num_sms / 2)));
        else
            cfg.gridDim = dim3((unsigned)std::min<int64_t>(m_tiles, h->num_sms));
        cfg.blockDim = dim3((unsigned)kFThreads);
        cfg.dynamicSmemBytes = h->fp.smem;
        cfg.stream = s;
        cudaLaunchAttribute fat[2];
        fat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        fat[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        fat[1].id = cudaLaunchAttributeClusterDimension;
        fat[1].val.clusterDim.x = h->fp.pair ? 2 : 1;
        fat[1].val.clusterDim.y = 1;
        fat[1].val.clusterDim.z = 1;
        cfg.attrs = fat;
        cfg.numAttrs = 2;
        cudaEvent_t* ev = nullptr;
        if (h->prof_on && h->prof_n < h->prof_max) ev = &h->prof_ev[3 * (size_t)h->prof_n++];
        if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
        CUDA_TRY(cudaLaunchKernelEx(&cfg, dbg ? h->fp_dbg : h->fp.fn, fx, h->tm_fw1, h->tm_fw2, fy, a));
        if (ev) {
            CUDA_TRY(cudaEventRecord(ev[1], s));
            CUDA_TRY(cudaEventRecord(ev[2], s));
        }
        static const bool sync_check = std::getenv("SWIN_MLP_SYNC_CHECK") != nullptr;
        if (sync_check) {
            CUDA_TRY(cudaStreamSynchronize(s));
            CUDA_TRY(cudaGetLastError());
        }
        return SWIN_MLP_OK;
    }

    const int64_t m_tiles = (T + kBM - 1) / kBM;
    const int run_plan = plan_choice(h, plan_T > 0 ? plan_T : h->plan_hint > 0 ? h->plan_hint : T);
    if (run_plan == 3 && T <= kSMaxT) {   // one launch for the whole layer (small_mlp.cuh)
        CUtensorMap tmx;
        if (C / 128 <= kSResKB)   // 3-D: all K-blocks of the <= 64 rows in one op (a negative swizzle tags it)
            ST_TRY(encode_cached(h, &tmx, x, T, C / 128, C, (uint32_t)kSMaxT, (uint32_t)(C / 128),
                                 (CUtensorMapSwizzle)-1));
        else
            ST_TRY(encode_cached(h, &tmx, x, T, C, C, (uint32_t)kSMaxT));
        SmallArgs a = {};
        a.T = (int32_t)T; a.C = C; a.H = H; a.P = h->tiny_P; a.Q = h->tiny_Q; a.PR = h->tiny_PR;
        a.act = h->d.act == SWIN_MLP_ACT_GELU_ERF ? 1 : 0;
        a.m1 = h->m1; a.b1 = h->b1; a.zc1 = h->zc1; a.m2 = h->m2; a.b2 = h->b2; a.zc2 = h->zc2;
        a.gamma = h->gamma; a.beta = h->beta;
        a.inv_h = h->inv_h; a.z_h = h->d.h_zero_point; a.inv_y = h->inv_y; a.z_y = h->d.y_zero_point;
        a.s_x = h->d.x_scale; a.z_x = h->d.x_zero_point; a.eps = h->d.ln_eps;
        a.x = x; a.y = y; a.resid = residual; a.resid_out = residual_out;
        a.acc = h->tiny_acc; a.cnt = h->tiny_cnt;
        if (dbg) { a.acc1_tap = acc1; a.hid_tap = hidden; a.acc2_tap = acc2; a.ln_tap = ln_out; }
        a.trace = h->trace;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)h->tiny_P);
        cfg.blockDim = dim3((unsigned)kSThreads);
        cfg.dynamicSmemBytes = kSSmem;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = (unsigned)h->tiny_Q;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        cudaEvent_t* ev = nullptr;
        if (h->prof_on && h->prof_n < h->prof_max) ev = &h->prof_ev[3 * (size_t)h->prof_n++];
        if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
        CUDA_TRY(cudaLaunchKernelEx(&cfg, h->tiny_fn, tmx, h->tm_w1t, h->tm_w2t, a));
        if (ev) {
            CUDA_TRY(cudaEventRecord(ev[1], s));
            CUDA_TRY(cudaEventRecord(ev[2], s));
        }
        return SWIN_MLP_OK;
    }
    const bool use_s = run_plan == 2, use_b = run_plan == 1;
    const Plan& P1 = use_s ? h->p1s : h->p1;
    const CUtensorMap& tmw1 = use_s ? h->tm_w1s : h->tm_w1;
    const Plan& P2 = use_s ? h->p2s : use_b ? h->p2b : h->p2;
    const CUtensorMap& tmw2 = use_s ? h->tm_w2s : use_b ? h->tm_w2b : h->tm_w2;
    CUtensorMap tm_x, tm_h, tm_ho, tm_y, tm_xr;
    ST_TRY(encode_cached(h, &tm_x, x, T, C, C, (uint32_t)(kBM / P1.CS)));
    ST_TRY(encode_cached(h, &tm_h, hq, T, H, H, (uint32_t)(kBM / P2.CS)));
    // epilogue output maps: [128 rows][W B] boxes with the W-byte swizzle the staging uses
    auto swz = [](int w) {
        return w == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : w == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
             : w == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    };
    ST_TRY(encode_cached(h, &tm_ho, hq, T, H, H, kBM, (uint32_t)P1.out_w, swz(P1.out_w)));
    ST_TRY(encode_cached(h, &tm_y, y, T, C, C, kBM, (uint32_t)P2.out_w, swz(P2.out_w)));
    // op #6 residual source x, staged by TMA with the output tile's box and swizzle
    ST_TRY(encode_cached(h, &tm_xr, x, T, C, C, kBM, (uint32_t)P2.out_w, swz(P2.out_w)));

    GemmArgs a1 = {};
    a1.M = T; a1.K = C; a1.BN = P1.BN; a1.CS = P1.CS; a1.stages = P1.stages; a1.G = P1.G; a1.resb = P1.resb;
    a1.mt_major = P1.resb ? 1 : 0;   // resident B needs the m-major order; otherwise deal (m, n) units
    a1.out_w = P1.out_w;
    a1.n_groups = P1.n_groups; a1.num_units = (P1.pair ? (m_tiles + 1) / 2 : m_tiles) * P1.n_groups;
    a1.eg = P1.eg; a1.ldo = H;
    a1.m = h->m1; a1.b = h->b1; a1.zc = h->zc1; a1.inv_q = h->inv_h; a1.zq = h->d.h_zero_point;
    a1.acc_tap = dbg ? acc1 : nullptr;
    int32_t* a1ws = h->unfused ? reinterpret_cast<int32_t*>(hq + ((T * H + 127) / 128 * 128)) : nullptr;
    a1.acc_out = a1ws;
    a1.dst = P1.dst; a1.out = hq; a1.wsl = P1.wsl;
    if (P1.wsl) a1.mt_major = 0;
    a1.trace = h->trace; a1.trace_cta = h->trace_cta;
    a1.cta_stamps = h->trace ? h->trace + 8192 : nullptr;

    GemmArgs a2 = {};
    a2.M = T; a2.K = H; a2.BN = P2.BN; a2.CS = P2.CS; a2.stages = P2.stages; a2.G = P2.G; a2.eg = P2.eg;
    a2.xstage = P2.xstage; a2.yin = P2.yin; a2.x = x;
    a2.out_w = P2.out_w;
    a2.resb = P2.resb; a2.mt_major = P2.pair ? 0 : 1;   // op #6: one n-group per cluster
    a2.n_groups = 1; a2.num_units = P2.pair ? (m_tiles + 1) / 2 : m_tiles; a2.ldo = C;
    a2.m = h->m2; a2.b = h->b2; a2.zc = h->zc2; a2.inv_q = h->inv_y; a2.zq = h->d.y_zero_point;
    a2.s_x = h->d.x_scale; a2.z_x = h->d.x_zero_point; a2.one = 1.0f;
    a2.resid = residual; a2.resid_out = residual_out;
    a2.gamma = h->gamma; a2.beta = h->beta; a2.eps = h->d.ln_eps;
    a2.acc_tap = dbg ? acc2 : nullptr; a2.ln_tap = dbg ? ln_out : nullptr;
    a2.trace = h->trace ? h->trace + 4096 : nullptr; a2.trace_cta = h->trace_cta;
    a2.cta_stamps = h->trace ? h->trace + 8192 + 512 : nullptr;
    // op #6 split-K for runs of few m-tiles: partial sums + counters after Hq in the workspace,
    // cleared by this run's FC1 launch
    int kb_per = 0;
    const int ks = ksplit_for(h, P2, T, kb_per);
    if (ks > 1) {
        int32_t* kacc = reinterpret_cast<int32_t*>(hq + ((T * H + 127) / 128 * 128));
        const int64_t acc_words = (T * C + 3) / 4 * 4;
        a2.ksplit = ks; a2.kb_per = kb_per; a2.kacc = kacc; a2.kcnt = kacc + acc_words;
        a2.mt_major = 0;
        a2.num_units = m_tiles * ks;
        a1.zero_ptr = kacc;
        a1.zero_words = acc_words + (m_tiles * P2.CS + 3) / 4 * 4;
    }

    cudaEvent_t* ev = nullptr;
    if (h->prof_on && h->prof_n < h->prof_max) ev = &h->prof_ev[3 * (size_t)h->prof_n++];
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    ST_TRY(launch(P1, tm_x, tmw1, tm_ho, tm_ho, a1, s));
    if (h->unfused && h->sg_fn) {   // the shift-GELU control's row-max op #5 kernel
        if (dbg && acc1) CUDA_TRY(cudaMemcpyAsync(acc1, a1ws, (size_t)T * H * 4, cudaMemcpyDeviceToDevice, s));
        ShiftGeluArgs o = h->sg;
        o.a1 = a1ws; o.hq = hq; o.m1 = h->m1; o.b1 = h->b1; o.H = H; o.T = T;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((T + kOp5Threads / 32 - 1) / (kOp5Threads / 32), h->sg_grid)));
        cfg.blockDim = dim3((unsigned)kOp5Threads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CUDA_TRY(cudaLaunchKernelEx(&cfg, h->sg_fn, o));
    } else if (h->unfused) {   // the separate op #5 kernel (PDL-chained like the GEMMs)
        if (dbg && acc1) CUDA_TRY(cudaMemcpyAsync(acc1, a1ws, (size_t)T * H * 4, cudaMemcpyDeviceToDevice, s));
        Op5Args o = {};
        o.a1 = a1ws; o.hq = hq; o.m1 = h->m1; o.b1 = h->b1; o.inv_h = h->inv_h; o.z_h = h->d.h_zero_point;
        o.H = H; o.quads = T * (int64_t)H / 4;
        cudaLaunchConfig_t cfg = {};
        const int64_t need = (o.quads + kOp5Threads * kOp5Unroll - 1) / (kOp5Threads * kOp5Unroll);
        cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(need, h->op5_grid)));
        cfg.blockDim = dim3((unsigned)kOp5Threads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CUDA_TRY(cudaLaunchKernelEx(&cfg, h->op5_fn, o));
    }
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], s));
    if (dbg && hidden) CUDA_TRY(cudaMemcpyAsync(hidden, hq, (size_t)T * H, cudaMemcpyDeviceToDevice, s));
    ST_TRY(launch(P2, tm_h, tmw2, tm_y, tm_xr, a2, s));
    if (ev) CUDA_TRY(cudaEventRecord(ev[2], s));
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_mlp_int8_run(swin_mlp_int8_t h, const int8_t* x, const float* residual, int8_t* y,
                                    float* residual_out, int64_t T, void* workspace, size_t workspace_bytes,
                                    void* stream) {
    return run_impl(h, x, residual, y, residual_out, T, workspace, workspace_bytes, stream, nullptr, nullptr,
                    nullptr, nullptr, false);
}

swin_mlp_status_t swin_mlp_int8_set_plan_hint(swin_mlp_int8_t h, int64_t T_hint) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (T_hint < 0) return fail(SWIN_MLP_EINVAL, "T_hint=%lld < 0", (long long)T_hint);
    h->plan_hint = T_hint;
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_mlp_int8_run_debug(swin_mlp_int8_t h, const int8_t* x, const float* residual, int8_t* y,
                                          float* residual_out, int64_t T, void* workspace, size_t workspace_bytes,
                                          void* stream, int32_t* acc1, int8_t* hidden, int32_t* acc2,
                                          float* ln_out) {
    return run_impl(h, x, residual, y, residual_out, T, workspace, workspace_bytes, stream, acc1, hidden, acc2,
                    ln_out, true);
}

static size_t align128(size_t v) { return (v + 127) / 128 * 128; }

size_t swin_mlp_int8_host_workspace_bytes(swin_mlp_int8_t h, int64_t T, int32_t with_residual) {
    if (!h || T <= 0) return 0;
    const size_t tc = (size_t)T * h->d.C;
    return swin_mlp_int8_workspace_bytes(h, T) + align128(tc) + align128(tc) + (with_residual ? align128(tc * 4) : 0);
}

swin_mlp_status_t swin_mlp_int8_run_host(swin_mlp_int8_t h, const int8_t* x_host, const float* residual_host,
                                         int8_t* y_host, int64_t T, void* workspace, size_t workspace_bytes,
                                         void* stream) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (T < 0) return fail(SWIN_MLP_EINVAL, "T=%lld < 0", (long long)T);
    if (T == 0) return SWIN_MLP_OK;
    if (!x_host || !y_host || !workspace) return fail(SWIN_MLP_EINVAL, "x_host, y_host and workspace are required");
    const size_t need = swin_mlp_int8_host_workspace_bytes(h, T, residual_host != nullptr);
    if (workspace_bytes < need) return fail(SWIN_MLP_EINVAL, "workspace %zu < %zu bytes", workspace_bytes, need);
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int C = h->d.C;
    const size_t tc = (size_t)T * C;
    uint8_t* w = static_cast<uint8_t*>(workspace);
    const size_t ws = swin_mlp_int8_workspace_bytes(h, T);
    int8_t* xd = reinterpret_cast<int8_t*>(w + ws);
    int8_t* yd = reinterpret_cast<int8_t*>(w + ws + align128(tc));
    float* rd = residual_host ? reinterpret_cast<float*>(w + ws + 2 * align128(tc)) : nullptr;

    // Pipeline over token chunks (rows are independent): copy-in of chunk k+1 and
    // copy-out of chunk k-1 overlap the kernels of chunk k (PCIe is full duplex).
    // Kernels run on the caller's stream; the copies on two handle-owned streams,
    // ordered by events; the caller's stream finally waits for the last copy-out.
    constexpr int kMaxChunks = 8;
    int64_t rows = (T + kMaxChunks - 1) / kMaxChunks;
    rows = std::max<int64_t>((rows + kBM - 1) / kBM * kBM, 4096);
    const int nch = (int)((T + rows - 1) / rows);
    if (!h->io_in) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->io_in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&h->io_out, cudaStreamNonBlocking));
    }
    while (h->io_ev.size() < 2 * kMaxChunks + 2) {   // (run_host_batch may have created fewer)
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->io_ev.push_back(e);
    }
    cudaEvent_t ev_start = h->io_ev[2 * kMaxChunks], ev_done = h->io_ev[2 * kMaxChunks + 1];
    CUDA_TRY(cudaEventRecord(ev_start, s));
    CUDA_TRY(cudaStreamWaitEvent(h->io_in, ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(h->io_out, ev_start, 0));
    for (int k = 0; k < nch; ++k) {
        const int64_t r0 = (int64_t)k * rows, n = std::min<int64_t>(rows, T - r0);
        const size_t off = (size_t)r0 * C, bytes = (size_t)n * C;
        cudaEvent_t ev_in = h->io_ev[2 * k], ev_out = h->io_ev[2 * k + 1];
        CUDA_TRY(cudaMemcpyAsync(xd + off, x_host + off, bytes, cudaMemcpyHostToDevice, h->io_in));
        if (rd) CUDA_TRY(cudaMemcpyAsync(rd + off, residual_host + off, bytes * 4, cudaMemcpyHostToDevice, h->io_in));
        CUDA_TRY(cudaEventRecord(ev_in, h->io_in));
        CUDA_TRY(cudaStreamWaitEvent(s, ev_in, 0));
        ST_TRY(run_impl(h, xd + off, rd ? rd + off : nullptr, yd + off, nullptr, n, w, ws, stream, nullptr, nullptr,
                        nullptr, nullptr, false, h->plan_hint > 0 ? h->plan_hint : T));
        CUDA_TRY(cudaEventRecord(ev_out, s));
        CUDA_TRY(cudaStreamWaitEvent(h->io_out, ev_out, 0));
        CUDA_TRY(cudaMemcpyAsync(y_host + off, yd + off, bytes, cudaMemcpyDeviceToHost, h->io_out));
    }
    CUDA_TRY(cudaEventRecord(ev_done, h->io_out));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
    return SWIN_MLP_OK;
}

size_t swin_mlp_int8_host_batch_workspace_bytes(int32_t n, const swin_mlp_int8_t* hs, const int64_t* Ts) {
    if (n <= 0 || !hs || !Ts) return 0;
    size_t ws = 0, stage = 0;
    for (int32_t l = 0; l < n; ++l) {
        if (!hs[l] || Ts[l] < 0) return 0;
        ws = std::max(ws, swin_mlp_int8_workspace_bytes(hs[l], Ts[l]));
        stage += 2 * align128((size_t)Ts[l] * hs[l]->d.C);
    }
    return align128(ws) + stage;
}

swin_mlp_status_t swin_mlp_int8_run_host_batch(int32_t n, const swin_mlp_int8_t* hs, const int8_t* const* x_hosts,
                                               int8_t* const* y_hosts, const int64_t* Ts, void* workspace,
                                               size_t workspace_bytes, void* stream) {
    if (n <= 0 || !hs || !x_hosts || !y_hosts || !Ts || !workspace)
        return fail(SWIN_MLP_EINVAL, "n > 0 and non-NULL arrays and workspace are required");
    for (int32_t l = 0; l < n; ++l) {
        if (!hs[l]) return fail(SWIN_MLP_EINVAL, "handle %d is NULL", l);
        if (Ts[l] < 0) return fail(SWIN_MLP_EINVAL, "T[%d] < 0", l);
        if (Ts[l] > 0 && (!x_hosts[l] || !y_hosts[l])) return fail(SWIN_MLP_EINVAL, "x/y of layer %d NULL", l);
        if (hs[l]->device != hs[0]->device) return fail(SWIN_MLP_EINVAL, "all handles must live on one device");
    }
    const size_t need = swin_mlp_int8_host_batch_workspace_bytes(n, hs, Ts);
    if (workspace_bytes < need) return fail(SWIN_MLP_EINVAL, "workspace %zu < %zu bytes", workspace_bytes, need);
    swin_mlp_int8_t h0 = hs[0];
    DeviceGuard guard(h0->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint8_t* w = static_cast<uint8_t*>(workspace);
    size_t ws = 0;
    for (int32_t l = 0; l < n; ++l) ws = std::max(ws, swin_mlp_int8_workspace_bytes(hs[l], Ts[l]));
    ws = align128(ws);

    // one pipeline over the chunks of all layers (see run_host): copy-in on one stream,
    // kernels on `stream`, copy-out on another, chunk by chunk in layer order
    constexpr int64_t kRows = 16384;
    std::vector<std::tuple<int32_t, int64_t, int64_t>> chunks;   // (layer, first row, rows)
    for (int32_t l = 0; l < n; ++l)
        for (int64_t r0 = 0; r0 < Ts[l]; r0 += kRows) chunks.emplace_back(l, r0, std::min<int64_t>(kRows, Ts[l] - r0));
    if (!h0->io_in) {
        CUDA_TRY(cudaStreamCreateWithFlags(&h0->io_in, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&h0->io_out, cudaStreamNonBlocking));
    }
    while (h0->io_ev.size() < 2 * chunks.size() + 2) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h0->io_ev.push_back(e);
    }
    const size_t nev = h0->io_ev.size();
    cudaEvent_t ev_start = h0->io_ev[nev - 2], ev_done = h0->io_ev[nev - 1];
    CUDA_TRY(cudaEventRecord(ev_start, s));
    CUDA_TRY(cudaStreamWaitEvent(h0->io_in, ev_start, 0));
    CUDA_TRY(cudaStreamWaitEvent(h0->io_out, ev_start, 0));
    std::vector<size_t> stage_off(n);
    size_t off = ws;
    for (int32_t l = 0; l < n; ++l) {
        stage_off[l] = off;
        off += 2 * align128((size_t)Ts[l] * hs[l]->d.C);
    }
    for (size_t k = 0; k < chunks.size(); ++k) {
        const int32_t l = std::get<0>(chunks[k]);
        const int64_t r0 = std::get<1>(chunks[k]), rows = std::get<2>(chunks[k]);
        const int C = hs[l]->d.C;
        const size_t tc = (size_t)Ts[l] * C, o = (size_t)r0 * C, bytes = (size_t)rows * C;
        int8_t* xd = reinterpret_cast<int8_t*>(w + stage_off[l]);
        int8_t* yd = reinterpret_cast<int8_t*>(w + stage_off[l] + align128(tc));
        cudaEvent_t ev_in = h0->io_ev[2 * k], ev_out = h0->io_ev[2 * k + 1];
        CUDA_TRY(cudaMemcpyAsync(xd + o, x_hosts[l] + o, bytes, cudaMemcpyHostToDevice, h0->io_in));
        CUDA_TRY(cudaEventRecord(ev_in, h0->io_in));
        CUDA_TRY(cudaStreamWaitEvent(s, ev_in, 0));
        ST_TRY(run_impl(hs[l], xd + o, nullptr, yd + o, nullptr, rows, w, ws, stream, nullptr, nullptr, nullptr,
                        nullptr, false, hs[l]->plan_hint > 0 ? hs[l]->plan_hint : Ts[l]));
        CUDA_TRY(cudaEventRecord(ev_out, s));
        CUDA_TRY(cudaStreamWaitEvent(h0->io_out, ev_out, 0));
        CUDA_TRY(cudaMemcpyAsync(y_hosts[l] + o, yd + o, bytes, cudaMemcpyDeviceToHost, h0->io_out));
    }
    CUDA_TRY(cudaEventRecord(ev_done, h0->io_out));
    CUDA_TRY(cudaStreamWaitEvent(s, ev_done, 0));
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_mlp_int8_get_constants(swin_mlp_int8_t h, float* m1, float* inv_h, float* m2, float* inv_y,
                                              int32_t* wsum1, int32_t* wsum2) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (m1) std::memcpy(m1, h->hm1.data(), h->hm1.size() * sizeof(float));
    if (m2) std::memcpy(m2, h->hm2.data(), h->hm2.size() * sizeof(float));
    if (wsum1) std::memcpy(wsum1, h->hws1.data(), h->hws1.size() * sizeof(int32_t));
    if (wsum2) std::memcpy(wsum2, h->hws2.data(), h->hws2.size() * sizeof(int32_t));
    if (inv_h) *inv_h = h->inv_h;
    if (inv_y) *inv_y = h->inv_y;
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_mlp_int8_profile_begin(swin_mlp_int8_t h, int32_t max_runs) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (max_runs < 0) return fail(SWIN_MLP_EINVAL, "max_runs < 0");
    DeviceGuard guard(h->device);
    while ((int)h->prof_ev.size() < 3 * max_runs) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        h->prof_ev.push_back(e);
    }
    h->prof_max = max_runs;
    h->prof_n = 0;
    h->prof_on = true;
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_mlp_int8_profile_end(swin_mlp_int8_t h, float* fc1_ms, float* fc2_ms, int32_t* runs) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    DeviceGuard guard(h->device);
    float t1 = 0.f, t2 = 0.f;
    for (int i = 0; i < h->prof_n; ++i) {
        cudaEvent_t* ev = &h->prof_ev[3 * (size_t)i];
        CUDA_TRY(cudaEventSynchronize(ev[2]));
        float a = 0.f, b = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&a, ev[0], ev[1]));
        CUDA_TRY(cudaEventElapsedTime(&b, ev[1], ev[2]));
        t1 += a;
        t2 += b;
    }
    if (fc1_ms) *fc1_ms = t1;
    if (fc2_ms) *fc2_ms = t2;
    if (runs) *runs = h->prof_n;
    h->prof_on = false;
    h->prof_n = 0;
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_mlp_int8_set_trace(swin_mlp_int8_t h, void* trace, int32_t cta) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (cta < 0) return fail(SWIN_MLP_EINVAL, "cta < 0");
    h->trace = static_cast<unsigned long long*>(trace);
    h->trace_cta = cta;
    return SWIN_MLP_OK;
}

int32_t swin_mlp_int8_launches_per_run(swin_mlp_int8_t h) { return h ? (h->fp.on ? 1 : h->unfused ? 3 : 2) : 0; }

swin_mlp_status_t swin_mlp_int8_destroy(swin_mlp_int8_t h) {
    if (!h) return SWIN_MLP_OK;
    {
        DeviceGuard guard(h->device);
        delete h;
    }
    return SWIN_MLP_OK;
}

// ---------------------------------------------------------------------------------------
// NEXT-2: Proj GEMM + fused op #4 (+ LN2), Fig. 1 lines 63-70.  Kernel 2 of the
// two-kernel plan (mlp_gemm_kernel<EP6_LN>) with K = C: the handle is an MLP handle whose
// FC2 slot holds W_proj and whose "hidden" quantizer is the attention-output quantizer.
struct swin_proj_int8_s {
    swin_mlp_int8_s m;
};

swin_mlp_status_t swin_proj_int8_create(const swin_proj_int8_desc_t* desc, swin_proj_int8_t* out) {
    g_last_error.clear();
    if (!desc || !out) return fail(SWIN_MLP_EINVAL, "desc and out must be non-NULL");
    const swin_proj_int8_desc_t& d = *desc;
    if (d.C < 32 || d.C % 32) return fail(SWIN_MLP_EINVAL, "C=%d must be a multiple of 32 and >= 32", d.C);
    if (d.C > 1536) return fail(SWIN_MLP_EUNSUPPORTED, "C=%d exceeds 1536", d.C);
    if (!normal_positive(d.a_scale) || !normal_positive(d.y_scale))
        return fail(SWIN_MLP_EINVAL, "activation scales must be finite, normal and > 0");
    if (!(d.ln_eps > 0.0f) || !std::isfinite(d.ln_eps)) return fail(SWIN_MLP_EINVAL, "ln_eps must be > 0");
    for (int32_t z : {d.a_zero_point, d.y_zero_point})
        if (z < -128 || z > 127) return fail(SWIN_MLP_EINVAL, "zero point %d outside [-128, 127]", z);
    if (!d.w || !d.w_scale || !d.ln_gamma || !d.ln_beta)
        return fail(SWIN_MLP_EINVAL, "w, w_scale, ln_gamma, ln_beta are required");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (d.device < 0 || d.device >= ndev) return fail(SWIN_MLP_EINVAL, "device %d of %d", d.device, ndev);
    DeviceGuard guard(d.device);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(SWIN_MLP_EUNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", d.device,
                    prop.major, prop.minor);
    const int C = d.C;
    std::vector<int8_t> w;
    std::vector<float> sw, b, g, bt;
    ST_TRY(fetch(d.w, (size_t)C * C, w, "w"));
    ST_TRY(fetch(d.w_scale, (size_t)C, sw, "w_scale"));
    ST_TRY(fetch(d.ln_gamma, (size_t)C, g, "ln_gamma"));
    ST_TRY(fetch(d.ln_beta, (size_t)C, bt, "ln_beta"));
    if (d.b) ST_TRY(fetch(d.b, (size_t)C, b, "b"));

    auto ph = new swin_proj_int8_s();
    swin_mlp_int8_s* h = &ph->m;
    auto bail = [&](swin_mlp_status_t st) {
        delete ph;
        return st;
    };
    h->d = swin_mlp_int8_desc_t{};
    h->d.C = C; h->d.H = C; h->d.act = SWIN_MLP_ACT_RELU;
    h->d.x_scale = 1.0f; h->d.x_zero_point = 0;                       // (no FC1 / no dQ(x) residual)
    h->d.h_scale = d.a_scale; h->d.h_zero_point = d.a_zero_point;     // the GEMM input quantizer
    h->d.ln_eps = d.ln_eps; h->d.y_scale = d.y_scale; h->d.y_zero_point = d.y_zero_point;
    h->d.device = d.device; h->d.ln_fp64 = d.ln_fp64;
    h->device = d.device;
    h->num_sms = prop.multiProcessorCount;
    // O0 for op #4: m[c] = fl(a_scale * w_scale[c]), inv_y = fl(1/y_scale); zero-point correction
    h->hm2.resize(C);
    for (int c = 0; c < C; ++c) {
        if (!normal_positive(sw[c])) return bail(fail(SWIN_MLP_EINVAL, "w_scale[%d] not finite/normal/positive", c));
        volatile float m = d.a_scale * sw[c];
        h->hm2[c] = m;
        if (!normal_positive(h->hm2[c])) return bail(fail(SWIN_MLP_EINVAL, "a_scale*w_scale[%d] not normal", c));
    }
    {
        volatile float one = 1.0f;
        h->inv_y = one / d.y_scale;
    }
    if (!normal_positive(h->inv_y)) return bail(fail(SWIN_MLP_EINVAL, "1/y_scale not normal"));
    h->hws2.assign(C, 0);
    std::vector<int32_t> zc(C);
    for (int c = 0; c < C; ++c) {
        int64_t s = 0;
        for (int k = 0; k < C; ++k) {
            if (w[(size_t)c * C + k] == -128) return bail(fail(SWIN_MLP_EINVAL, "w must be symmetric (-128 not allowed)"));
            s += w[(size_t)c * C + k];
        }
        h->hws2[c] = (int32_t)s;
        zc[c] = (int32_t)(s * d.a_zero_point);
    }
    if (!make_plan(EP6_LN, C, C, true, h->p2, d.ln_fp64 ? 8 : 4))
        return bail(fail(SWIN_MLP_EUNSUPPORTED, "no proj tile plan for C=%d", C));
    swin_mlp_status_t st;
#define H_TRY(expr)                                   \
    do {                                              \
        if ((st = (expr)) != SWIN_MLP_OK) return bail(st); \
    } while (0)
    H_TRY(upload(h, w, &h->w2));
    H_TRY(upload(h, h->hm2, &h->m2));
    H_TRY(upload(h, g, &h->gamma));
    H_TRY(upload(h, bt, &h->beta));
    if (d.b) H_TRY(upload(h, b, &h->b2));
    if (d.a_zero_point) H_TRY(upload(h, zc, &h->zc2));
    H_TRY(encode_2d(&h->tm_w2, h->w2, C, C, C,
                    (uint32_t)(h->p2.pair ? (h->p2.BN > 256 ? h->p2.BN / 4 : h->p2.BN / 2) : h->p2.BN)));
    h->p2.fn = kernel_for(EP6_LN, (d.b ? kHasB : 0) | (d.a_zero_point ? kHasZc : 0) | (d.y_zero_point ? kZqNz : 0) |
                                      (d.ln_fp64 ? kS64 : 0) | (h->p2.pair ? kPair : 0));
    H_TRY(prepare(h->p2, h->num_sms));
#undef H_TRY
    *out = ph;
    return SWIN_MLP_OK;
}

static swin_mlp_status_t proj_run_impl(swin_proj_int8_t ph, const int8_t* a, const float* residual, int8_t* y,
                                       float* residual_out, int64_t T, void* stream, int32_t* acc, float* ln_out,
                                       bool dbg) {
    if (!ph) return fail(SWIN_MLP_EINVAL, "NULL handle");
    swin_mlp_int8_s* h = &ph->m;
    if (T < 0) return fail(SWIN_MLP_EINVAL, "T=%lld < 0", (long long)T);
    if (T == 0) return SWIN_MLP_OK;
    if (T > (int64_t)1 << 31) return fail(SWIN_MLP_EUNSUPPORTED, "T=%lld too large", (long long)T);
    if (!a || !y || !residual) return fail(SWIN_MLP_EINVAL, "a, residual and y are required");
    if (!aligned16(a) || !aligned16(y) || !aligned16(residual) || (residual_out && !aligned16(residual_out)))
        return fail(SWIN_MLP_EINVAL, "a/y/residual/residual_out must be 16-byte aligned");
    if ((const void*)a == (const void*)y) return fail(SWIN_MLP_EINVAL, "y may not alias a");
    const int C = h->d.C;
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto swz = [](int w) {
        return w == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : w == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
             : w == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    };
    CUtensorMap tm_a, tm_y;
    ST_TRY(encode_cached(h, &tm_a, a, T, C, C, (uint32_t)(kBM / h->p2.CS)));
    ST_TRY(encode_cached(h, &tm_y, y, T, C, C, kBM, (uint32_t)h->p2.out_w, swz(h->p2.out_w)));
    const int64_t m_tiles = (T + kBM - 1) / kBM;
    GemmArgs a2 = {};
    a2.M = T; a2.K = C; a2.BN = h->p2.BN; a2.CS = h->p2.CS; a2.stages = h->p2.stages; a2.G = h->p2.G; a2.eg = h->p2.eg;
    a2.xstage = h->p2.xstage; a2.yin = h->p2.yin; a2.x = nullptr;
    a2.out_w = h->p2.out_w;
    a2.resb = h->p2.resb; a2.mt_major = h->p2.pair ? 0 : 1;
    a2.n_groups = 1; a2.num_units = h->p2.pair ? (m_tiles + 1) / 2 : m_tiles; a2.ldo = C;
    a2.m = h->m2; a2.b = h->b2; a2.zc = h->zc2; a2.inv_q = h->inv_y; a2.zq = h->d.y_zero_point;
    a2.s_x = 1.0f; a2.z_x = 0; a2.one = 1.0f;
    a2.resid = residual; a2.resid_out = residual_out;
    a2.gamma = h->gamma; a2.beta = h->beta; a2.eps = h->d.ln_eps;
    a2.acc_tap = dbg ? acc : nullptr; a2.ln_tap = dbg ? ln_out : nullptr;
    return launch(h->p2, tm_a, h->tm_w2, tm_y, tm_y, a2, s);
}

swin_mlp_status_t swin_proj_int8_run(swin_proj_int8_t h, const int8_t* a, const float* residual, int8_t* y,
                                     float* residual_out, int64_t T, void* stream) {
    return proj_run_impl(h, a, residual, y, residual_out, T, stream, nullptr, nullptr, false);
}

swin_mlp_status_t swin_proj_int8_run_debug(swin_proj_int8_t h, const int8_t* a, const float* residual, int8_t* y,
                                           float* residual_out, int64_t T, void* stream, int32_t* acc,
                                           float* ln_out) {
    return proj_run_impl(h, a, residual, y, residual_out, T, stream, acc, ln_out, true);
}

int32_t swin_proj_int8_plan(swin_proj_int8_t h, int32_t* out4) {
    if (!h || !out4) return -1;
    out4[0] = h->m.p2.BN; out4[1] = h->m.p2.CS; out4[2] = h->m.p2.stages; out4[3] = h->m.p2.pair;
    return 0;
}

swin_mlp_status_t swin_proj_int8_destroy(swin_proj_int8_t h) {
    if (!h) return SWIN_MLP_OK;
    {
        DeviceGuard guard(h->m.device);
        delete h;
    }
    return SWIN_MLP_OK;
}

// Test/bench introspection: the launch plan chosen for this layer.
int32_t swin_mlp_int8_plan(swin_mlp_int8_t h, int32_t* out10) {
    if (!h || !out10) return -1;  // out10 holds 20 entries
    out10[0] = h->p1.BN; out10[1] = h->p1.CS; out10[2] = h->p1.stages; out10[3] = h->p1.max_clusters;
    out10[4] = h->p2.BN; out10[5] = h->p2.CS; out10[6] = h->p2.stages; out10[7] = h->p2.max_clusters;
    out10[8] = h->p1.G; out10[9] = h->p2.G;
    out10[10] = h->p1.resb ? 1 : h->p1.wsl ? 2 : 0; out10[11] = h->p2.resb;
    out10[12] = h->fp.on ? 1 : 0; out10[13] = h->fp.stages; out10[14] = h->fp.NH; out10[15] = h->fp.NB1;
    out10[16] = h->p1.pair; out10[17] = h->fp.NX; out10[18] = h->fp.stages2; out10[19] = h->unfused ? 1 : 0;
    return 0;
}

int32_t swin_mlp_int8_plan_for(swin_mlp_int8_t h, int64_t T, int32_t* out20) {
    if (!h || !out20 || T < 0) return -1;
    swin_mlp_int8_plan(h, out20);
    if (h->fp.on) return 0;   // the one-kernel plan: the same launch for every T
    const int c = plan_choice(h, h->plan_hint > 0 ? h->plan_hint : T);
    if (c == 3) {   // the one-launch plan: out20[0] = CTAs, [4] = FC2 piece columns, [5] = pieces
        for (int i = 0; i < 12; ++i) out20[i] = 0;
        out20[0] = h->tiny_P; out20[4] = h->tiny_PR; out20[5] = h->tiny_Q; out20[13] = 1; out20[16] = 0;
        out20[19] = (h->unfused ? 1 : 0) | (c << 1);
        return 0;
    }
    const Plan& P1 = c == 2 ? h->p1s : h->p1;
    const Plan& P2 = c == 2 ? h->p2s : c == 1 ? h->p2b : h->p2;
    out20[0] = P1.BN; out20[1] = P1.CS; out20[2] = P1.stages; out20[3] = P1.max_clusters;
    out20[4] = P2.BN; out20[5] = P2.CS; out20[6] = P2.stages; out20[7] = P2.max_clusters;
    out20[8] = P1.G; out20[9] = P2.G;
    out20[10] = P1.resb ? 1 : P1.wsl ? 2 : 0; out20[11] = P2.resb; out20[16] = P1.pair;
    out20[19] = (h->unfused ? 1 : 0) | (c << 1);
    int kb_per = 0;   // op #6 split-K factor of this run (two-kernel handles only; 1 = none)
    out20[13] = ksplit_for(h, P2, T, kb_per);
    return 0;
}

// ---------------------------------------------------------------------------------------
// NEXT-4: fused op #1 (LayerNorm -> window shift -> Q), Fig. 1 lines 39-43.
struct swin_op1_int8_s {
    swin_op1_int8_desc_t d;
    int device = 0, num_sms = 0, blocks_per_sm = 1, U = 1, L = 32;
    void (*fn)(Op1Args) = nullptr;
    float* gamma = nullptr;
    float* beta = nullptr;
    float inv_s = 0.f;
    ~swin_op1_int8_s() {
        if (gamma) cudaFree(gamma);
        if (beta) cudaFree(beta);
    }
};

swin_mlp_status_t swin_op1_int8_create(const swin_op1_int8_desc_t* desc, swin_op1_int8_t* out) {
    g_last_error.clear();
    if (!desc || !out) return fail(SWIN_MLP_EINVAL, "desc and out must be non-NULL");
    const swin_op1_int8_desc_t& d = *desc;
    if (d.C < 4 || d.C % 4) return fail(SWIN_MLP_EINVAL, "C=%d must be a positive multiple of 4", d.C);
    if (d.C > 1536) return fail(SWIN_MLP_EUNSUPPORTED, "C=%d exceeds 1536", d.C);
    if (d.M < 1 || d.M > 16) return fail(SWIN_MLP_EINVAL, "window M=%d outside [1, 16]", d.M);
    if (d.shift < 0 || d.shift >= d.M) return fail(SWIN_MLP_EINVAL, "shift=%d outside [0, M)", d.shift);
    if (d.Hs < d.M || d.Ws < d.M || d.Hs % d.M || d.Ws % d.M)
        return fail(SWIN_MLP_EINVAL, "Hs=%d, Ws=%d must be positive multiples of M=%d", d.Hs, d.Ws, d.M);
    if (!normal_positive(d.y_scale)) return fail(SWIN_MLP_EINVAL, "y_scale must be finite, normal and > 0");
    if (!(d.ln_eps > 0.0f) || !std::isfinite(d.ln_eps)) return fail(SWIN_MLP_EINVAL, "ln_eps must be > 0");
    if (d.y_zero_point < -128 || d.y_zero_point > 127) return fail(SWIN_MLP_EINVAL, "zero point outside [-128, 127]");
    if (!d.ln_gamma || !d.ln_beta) return fail(SWIN_MLP_EINVAL, "ln_gamma and ln_beta are required");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (d.device < 0 || d.device >= ndev) return fail(SWIN_MLP_EINVAL, "device %d of %d", d.device, ndev);
    DeviceGuard guard(d.device);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(SWIN_MLP_EUNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", d.device,
                    prop.major, prop.minor);
    std::vector<float> g, b;
    ST_TRY(fetch(d.ln_gamma, (size_t)d.C, g, "ln_gamma"));
    ST_TRY(fetch(d.ln_beta, (size_t)d.C, b, "ln_beta"));
    auto h = new swin_op1_int8_s();
    h->d = d;
    h->d.ln_gamma = h->d.ln_beta = nullptr;
    h->device = d.device;
    h->num_sms = prop.multiProcessorCount;
    auto bail = [&](swin_mlp_status_t st) { delete h; return st; };
    {
        volatile float one = 1.0f;
        h->inv_s = one / d.y_scale;
    }
    if (!normal_positive(h->inv_s)) return bail(fail(SWIN_MLP_EINVAL, "1/y_scale not normal"));
    // a row on L lanes (8, 16 or 32: 32 / L rows per warp instruction), VPL float4 per lane, U row
    // groups per warp in flight (~8 float4 loads per lane)
    const int c4 = d.C / 4;
    const int L = c4 <= 32 ? 8 : c4 <= 64 ? 16 : 32;
    const int vpl = (c4 + L - 1) / L;
#define OP1(LL, V, UU) do { h->fn = op1_kernel<LL, V, UU>; h->U = UU; h->L = LL; } while (0)
    if (L == 8) {
        if (vpl == 1) OP1(8, 1, 8); else if (vpl == 2) OP1(8, 2, 4); else if (vpl == 3) OP1(8, 3, 2); else OP1(8, 4, 2);
    } else if (L == 16) {
        if (vpl == 3) OP1(16, 3, 2); else OP1(16, 4, 2);   // (c4 in 33..64)
    } else {
        if (vpl <= 3) OP1(32, 3, 2); else if (vpl == 4) OP1(32, 4, 2); else if (vpl <= 6) OP1(32, 6, 1);
        else if (vpl <= 8) OP1(32, 8, 1); else OP1(32, 12, 1);
    }
#undef OP1
    cudaError_t e = cudaMalloc(&h->gamma, sizeof(float) * d.C);
    if (e == cudaSuccess) e = cudaMalloc(&h->beta, sizeof(float) * d.C);
    if (e == cudaSuccess) e = cudaMemcpy(h->gamma, g.data(), sizeof(float) * d.C, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->beta, b.data(), sizeof(float) * d.C, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->blocks_per_sm, h->fn, 256, 0);
    if (e != cudaSuccess) return bail(fail(SWIN_MLP_ECUDA, "op1 create: %s", cudaGetErrorString(e)));
    h->blocks_per_sm = std::max(1, h->blocks_per_sm);
    *out = h;
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_op1_int8_run(swin_op1_int8_t h, const float* x, int64_t B, int8_t* y, void* stream) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (B < 0) return fail(SWIN_MLP_EINVAL, "B=%lld < 0", (long long)B);
    if (B == 0) return SWIN_MLP_OK;
    if (!x || !y) return fail(SWIN_MLP_EINVAL, "x and y are required");
    if ((reinterpret_cast<uintptr_t>(x) & 15u) || (reinterpret_cast<uintptr_t>(y) & 3u))
        return fail(SWIN_MLP_EINVAL, "x must be 16-byte and y 4-byte aligned");
    const int64_t rows = B * (int64_t)h->d.Hs * h->d.Ws;
    if (rows >= ((int64_t)1 << 31)) return fail(SWIN_MLP_EUNSUPPORTED, "B=%lld too large", (long long)B);
    DeviceGuard guard(h->device);
    Op1Args a = {};
    a.x = x; a.y = y; a.rows = rows;
    a.C = h->d.C; a.Hs = h->d.Hs; a.Ws = h->d.Ws; a.M = h->d.M; a.shift = h->d.shift;
    a.gamma = h->gamma; a.beta = h->beta; a.eps = h->d.ln_eps; a.inv_s = h->inv_s; a.z = h->d.y_zero_point;
    a.divN = make_fastdiv((uint32_t)(h->d.M * h->d.M));
    a.divNW = make_fastdiv((uint32_t)((h->d.Hs / h->d.M) * (h->d.Ws / h->d.M)));
    a.divNWx = make_fastdiv((uint32_t)(h->d.Ws / h->d.M));
    a.divM = make_fastdiv((uint32_t)h->d.M);
    const int64_t per_warp = (int64_t)h->U * (32 / h->L);
    const int64_t warps = (rows + per_warp - 1) / per_warp;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)h->num_sms * h->blocks_per_sm));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, h->fn, a));
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_op1_int8_destroy(swin_op1_int8_t h) {
    if (!h) return SWIN_MLP_OK;
    DeviceGuard guard(h->device);
    delete h;
    return SWIN_MLP_OK;
}

// ---------------------------------------------------------------------------------------
// NEXT-3: QKV GEMM + op #2 -> Q.K + op #3 -> V.att, Fig. 1 lines 45-62.  The QKV GEMM
// is the MLP's GEMM skeleton with the op #2 epilogue (mlp_gemm_kernel<EP2_QKV>); the attention
// core is attn_core_kernel<M> (attn_kernels.cuh).
struct swin_attn_int8_s {
    swin_mlp_int8_s m;          // the QKV GEMM: p1 / tm_w1 / w1 (Wqkv) / m1 / b1 / zc1, map cache
    swin_attn_int8_desc_t d;
    float* inv_cols = nullptr;  // [3C] fl(1/s_q | 1/s_k | 1/s_v) per column
    float* bias = nullptr;      // [heads][MT*16][NT*8] padded (-inf at columns >= N, 0 at rows >= N)
    std::vector<float> hbias;   // [heads][N][N] (get_constants)
    float m3 = 0.f, inv_p = 0.f, m_o = 0.f;
    int N = 0, nW = 0, core_smem = 0, core_blocks_per_sm = 1, qrows = 0, np = 0;
    void (*core)(AttnArgs) = nullptr;
};

swin_mlp_status_t swin_attn_int8_create(const swin_attn_int8_desc_t* desc, swin_attn_int8_t* out) {
    g_last_error.clear();
    if (!desc || !out) return fail(SWIN_MLP_EINVAL, "desc and out must be non-NULL");
    const swin_attn_int8_desc_t& d = *desc;
    if (d.heads < 1 || d.C != 32 * d.heads) return fail(SWIN_MLP_EINVAL, "C=%d must be 32 * heads (heads=%d)", d.C, d.heads);
    if (d.C < 64) return fail(SWIN_MLP_EINVAL, "C=%d < 64", d.C);
    if (d.C > 1536) return fail(SWIN_MLP_EUNSUPPORTED, "C=%d exceeds 1536", d.C);
    if (d.M != 7 && d.M != 12) return fail(SWIN_MLP_EUNSUPPORTED, "window M=%d (built: 7, 12)", d.M);
    if (d.shift < 0 || d.shift >= d.M) return fail(SWIN_MLP_EINVAL, "shift=%d outside [0, M)", d.shift);
    if (d.Hs < d.M || d.Ws < d.M || d.Hs % d.M || d.Ws % d.M)
        return fail(SWIN_MLP_EINVAL, "Hs=%d, Ws=%d must be positive multiples of M=%d", d.Hs, d.Ws, d.M);
    if (!normal_positive(d.x_scale) || !normal_positive(d.q_scale) || !normal_positive(d.k_scale) ||
        !normal_positive(d.v_scale) || !normal_positive(d.a_scale))
        return fail(SWIN_MLP_EINVAL, "scales must be finite, normal and > 0");
    for (int32_t z : {d.x_zero_point, d.a_zero_point})
        if (z < -128 || z > 127) return fail(SWIN_MLP_EINVAL, "zero point %d outside [-128, 127]", z);
    if (!d.w_qkv || !d.w_qkv_scale || !d.rel_bias_table)
        return fail(SWIN_MLP_EINVAL, "w_qkv, w_qkv_scale and rel_bias_table are required");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (d.device < 0 || d.device >= ndev) return fail(SWIN_MLP_EINVAL, "device %d of %d", d.device, ndev);
    DeviceGuard guard(d.device);
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(SWIN_MLP_EUNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", d.device,
                    prop.major, prop.minor);
    const int C = d.C, N3 = 3 * d.C, M = d.M, N = M * M, heads = d.heads;
    const int nW = (d.Hs / M) * (d.Ws / M);
    std::vector<int8_t> w;
    std::vector<float> sw, b, table;
    ST_TRY(fetch(d.w_qkv, (size_t)N3 * C, w, "w_qkv"));
    ST_TRY(fetch(d.w_qkv_scale, (size_t)N3, sw, "w_qkv_scale"));
    ST_TRY(fetch(d.rel_bias_table, (size_t)(2 * M - 1) * (2 * M - 1) * heads, table, "rel_bias_table"));
    if (d.b_qkv) ST_TRY(fetch(d.b_qkv, (size_t)N3, b, "b_qkv"));

    auto ah = new swin_attn_int8_s();
    swin_mlp_int8_s* h = &ah->m;
    auto bail = [&](swin_mlp_status_t st) {
        delete ah;
        return st;
    };
    ah->d = d;
    ah->d.w_qkv = nullptr; ah->d.w_qkv_scale = ah->d.b_qkv = ah->d.rel_bias_table = nullptr;
    ah->N = N; ah->nW = nW;
    h->d = swin_mlp_int8_desc_t{};
    h->d.C = C; h->d.H = N3; h->d.x_scale = d.x_scale; h->d.x_zero_point = d.x_zero_point;
    h->d.device = d.device;
    h->device = d.device;
    h->num_sms = prop.multiProcessorCount;
    // op #2 folded constants: m[n] = fl(s_x * s_w[n]), inv per column; zero-point correction
    h->hm1.resize(N3);
    std::vector<float> inv(N3);
    float inv3[3];
    {
        volatile float one = 1.0f;
        inv3[0] = one / d.q_scale; inv3[1] = one / d.k_scale; inv3[2] = one / d.v_scale;
    }
    std::vector<int32_t> zc(N3);
    int64_t rowabs = 0;
    for (int n = 0; n < N3; ++n) {
        if (!normal_positive(sw[n])) return bail(fail(SWIN_MLP_EINVAL, "w_qkv_scale[%d] not finite/normal/positive", n));
        volatile float m = d.x_scale * sw[n];
        h->hm1[n] = m;
        if (!normal_positive(h->hm1[n])) return bail(fail(SWIN_MLP_EINVAL, "x_scale*w_qkv_scale[%d] not normal", n));
        inv[n] = inv3[n / C];
        int64_t s = 0, sa = 0;
        for (int k = 0; k < C; ++k) {
            const int8_t v = w[(size_t)n * C + k];
            if (v == -128) return bail(fail(SWIN_MLP_EINVAL, "w_qkv must be symmetric (-128 not allowed)"));
            s += v;
            sa += std::abs((int)v);
        }
        zc[n] = (int32_t)(s * d.x_zero_point);
        rowabs = std::max(rowabs, sa);
    }
    for (float v : inv3)
        if (!normal_positive(v)) return bail(fail(SWIN_MLP_EINVAL, "1/q|k|v_scale not normal"));
    // op #3 and V.att constants (one fp32 rounding each, as written in the header)
    {
        volatile float rs = (float)(1.0 / std::sqrt(32.0));
        volatile float sqk = d.q_scale * d.k_scale;
        volatile float m3 = sqk * rs;
        volatile float one = 1.0f;
        volatile float s_p = one / 127.0f;
        volatile float inv_p = one / s_p;
        volatile float spv = s_p * d.v_scale;
        volatile float inv_a = one / d.a_scale;
        volatile float m_o = spv * inv_a;
        ah->m3 = m3; ah->inv_p = inv_p; ah->m_o = m_o;
    }
    if (!normal_positive(ah->m3) || !normal_positive(ah->m_o)) return bail(fail(SWIN_MLP_EINVAL, "folded op #3 constants not normal"));
    // relative position bias [heads][N][N] and the shifted-window mask [nW][N][N]
    ah->hbias.resize((size_t)heads * N * N);
    for (int hh = 0; hh < heads; ++hh)
        for (int i = 0; i < N; ++i)
            for (int j = 0; j < N; ++j) {
                const int dy = i / M - j / M + M - 1, dx = i % M - j % M + M - 1;
                ah->hbias[((size_t)hh * N + i) * N + j] = table[(size_t)(dy * (2 * M - 1) + dx) * heads + hh];
            }
    // the kernel's padded tile per head: [MT*16][NT*8], -inf beyond column N (those logits vanish
    // in the softmax), 0 on the padding rows (finite, discarded)
    ah->qrows = M == 7 ? AttnGeom<7>::QROWS : AttnGeom<12>::QROWS;
    ah->np = M == 7 ? AttnGeom<7>::NP : AttnGeom<12>::NP;
    std::vector<float> pbias((size_t)heads * ah->qrows * ah->np, 0.0f);
    for (int hh = 0; hh < heads; ++hh)
        for (int i = 0; i < ah->qrows; ++i)
            for (int j = 0; j < ah->np; ++j)
                pbias[((size_t)hh * ah->qrows + i) * ah->np + j] =
                    j >= N ? -INFINITY : i >= N ? 0.0f : ah->hbias[((size_t)hh * N + i) * N + j];
    // QKV GEMM plan (op #2 epilogue)
    if (!make_plan(EP2_QKV, N3, C, false, h->p1)) return bail(fail(SWIN_MLP_EUNSUPPORTED, "no QKV GEMM plan for C=%d", C));
    swin_mlp_status_t st;
#define A_TRY(expr)                                        \
    do {                                                   \
        if ((st = (expr)) != SWIN_MLP_OK) return bail(st); \
    } while (0)
    A_TRY(upload(h, w, &h->w1));
    A_TRY(upload(h, h->hm1, &h->m1));
    A_TRY(upload(h, inv, &ah->inv_cols));   // (device copies are owned by h->allocs)
    if (d.b_qkv) A_TRY(upload(h, b, &h->b1));
    if (d.x_zero_point) A_TRY(upload(h, zc, &h->zc1));
    A_TRY(upload(h, pbias, &ah->bias));
    A_TRY(encode_2d(&h->tm_w1, h->w1, N3, C, C, (uint32_t)(h->p1.pair ? h->p1.BN / 2 : h->p1.BN)));
    const bool small_k = (int64_t)(128 + std::abs(d.x_zero_point)) * rowabs < (int64_t(1) << 22);
    h->p1.fn = kernel_for(EP2_QKV, (d.b_qkv ? kHasB : 0) | (d.x_zero_point ? kHasZc : 0) | (small_k ? kSmallK : 0) |
                                       (h->p1.pair ? kPair : 0));
    A_TRY(prepare(h->p1, h->num_sms));
    // attention core: one warp per (window, head), kAttnWarps warps per CTA
    ah->core = M == 7 ? attn_core_kernel<7> : attn_core_kernel<12>;
    ah->core_smem = M == 7 ? AttnGeom<7>::SMEM : AttnGeom<12>::SMEM;
    CUDA_TRY(cudaFuncSetAttribute(ah->core, cudaFuncAttributeMaxDynamicSharedMemorySize, ah->core_smem));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ah->core_blocks_per_sm, ah->core, 32 * kAttnWarps,
                                                           ah->core_smem));
    ah->core_blocks_per_sm = std::max(1, ah->core_blocks_per_sm);
#undef A_TRY
    *out = ah;
    return SWIN_MLP_OK;
}

size_t swin_attn_int8_workspace_bytes(swin_attn_int8_t h, int64_t B) {
    if (!h || B <= 0) return 0;
    const int64_t T = B * (int64_t)h->d.Hs * h->d.Ws;
    return (size_t)((T * 3 * h->d.C + 127) / 128 * 128);
}

static swin_mlp_status_t attn_run_impl(swin_attn_int8_t ah, const int8_t* xw, int64_t B, int8_t* aout, void* workspace,
                                       size_t ws_bytes, void* stream, int8_t* qkv_tap, int32_t* acc_tap, int8_t* p_tap) {
    if (!ah) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (B < 0) return fail(SWIN_MLP_EINVAL, "B=%lld < 0", (long long)B);
    if (B == 0) return SWIN_MLP_OK;
    swin_mlp_int8_s* h = &ah->m;
    const int C = ah->d.C, N3 = 3 * C;
    const int64_t T = B * (int64_t)ah->d.Hs * ah->d.Ws;
    if (T > ((int64_t)1 << 31)) return fail(SWIN_MLP_EUNSUPPORTED, "B=%lld too large", (long long)B);
    const size_t need = swin_attn_int8_workspace_bytes(ah, B);
    if (!xw || !aout || !workspace) return fail(SWIN_MLP_EINVAL, "xw, a and workspace are required");
    if (ws_bytes < need) return fail(SWIN_MLP_EINVAL, "workspace %zu < %zu bytes", ws_bytes, need);
    if (!aligned16(xw) || !aligned16(aout) || (reinterpret_cast<uintptr_t>(workspace) & 127u))
        return fail(SWIN_MLP_EINVAL, "xw and a 16-byte, workspace 128-byte aligned");
    DeviceGuard guard(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int8_t* qkv = static_cast<int8_t*>(workspace);
    const Plan& P1 = h->p1;
    auto swz = [](int w) {
        return w == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : w == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
             : w == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    };
    CUtensorMap tm_x, tm_o;
    ST_TRY(encode_cached(h, &tm_x, xw, T, C, C, (uint32_t)(kBM / P1.CS)));
    ST_TRY(encode_cached(h, &tm_o, qkv, T, N3, N3, kBM, (uint32_t)P1.out_w, swz(P1.out_w)));
    const int64_t m_tiles = (T + kBM - 1) / kBM;
    GemmArgs a1 = {};
    a1.M = T; a1.K = C; a1.BN = P1.BN; a1.CS = P1.CS; a1.stages = P1.stages; a1.G = P1.G; a1.resb = P1.resb;
    a1.mt_major = P1.resb ? 1 : 0;
    a1.out_w = P1.out_w;
    a1.n_groups = P1.n_groups; a1.num_units = (P1.pair ? (m_tiles + 1) / 2 : m_tiles) * P1.n_groups;
    a1.eg = P1.eg; a1.ldo = N3;
    a1.m = h->m1; a1.b = h->b1; a1.zc = h->zc1; a1.inv_q = 1.0f; a1.zq = 0;
    a1.gamma = ah->inv_cols;
    a1.acc_tap = acc_tap;
    a1.out = qkv;
    cudaEvent_t* ev = nullptr;
    if (h->prof_on && h->prof_n < h->prof_max) ev = &h->prof_ev[3 * (size_t)h->prof_n++];
    if (ev) CUDA_TRY(cudaEventRecord(ev[0], s));
    ST_TRY(launch(P1, tm_x, h->tm_w1, tm_o, tm_o, a1, s));
    if (ev) CUDA_TRY(cudaEventRecord(ev[1], s));
    if (qkv_tap) CUDA_TRY(cudaMemcpyAsync(qkv_tap, qkv, (size_t)T * N3, cudaMemcpyDeviceToDevice, s));

    AttnArgs c = {};
    c.qkv = qkv; c.out = aout;
    c.n_win = T / ah->N;
    c.C = C; c.heads = ah->d.heads; c.Hs = ah->d.Hs; c.Ws = ah->d.Ws; c.shift = ah->d.shift; c.nW = ah->nW;
    c.bias = ah->bias;
    c.m3 = ah->m3; c.inv_p = ah->inv_p; c.m_o = ah->m_o; c.z_a = ah->d.a_zero_point;
    c.p_tap = p_tap;
    // CTAs come in groups of `heads` (CTA c serves head c % heads): as many groups as the windows
    // need (kAttnWarps per CTA) or as fit resident
    const int64_t groups = std::max<int64_t>(
        1, std::min<int64_t>((c.n_win + kAttnWarps - 1) / kAttnWarps,
                             std::max<int64_t>(1, (int64_t)h->num_sms * ah->core_blocks_per_sm / ah->d.heads)));
    const int64_t blocks = groups * ah->d.heads;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(32 * kAttnWarps);
    cfg.dynamicSmemBytes = (size_t)ah->core_smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (pdl_enabled() && !qkv_tap) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, ah->core, c));
    if (ev) CUDA_TRY(cudaEventRecord(ev[2], s));
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_attn_int8_profile_begin(swin_attn_int8_t h, int32_t max_runs) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    return swin_mlp_int8_profile_begin(&h->m, max_runs);
}

swin_mlp_status_t swin_attn_int8_profile_end(swin_attn_int8_t h, float* qkv_ms, float* core_ms, int32_t* runs) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    return swin_mlp_int8_profile_end(&h->m, qkv_ms, core_ms, runs);
}

swin_mlp_status_t swin_attn_int8_run(swin_attn_int8_t h, const int8_t* xw, int64_t B, int8_t* a, void* workspace,
                                     size_t workspace_bytes, void* stream) {
    return attn_run_impl(h, xw, B, a, workspace, workspace_bytes, stream, nullptr, nullptr, nullptr);
}

swin_mlp_status_t swin_attn_int8_run_debug(swin_attn_int8_t h, const int8_t* xw, int64_t B, int8_t* a,
                                           void* workspace, size_t workspace_bytes, void* stream, int8_t* qkv,
                                           int32_t* acc, int8_t* p) {
    return attn_run_impl(h, xw, B, a, workspace, workspace_bytes, stream, qkv, acc, p);
}

swin_mlp_status_t swin_attn_int8_get_constants(swin_attn_int8_t h, float* m3_invp_mo, float* bias) {
    if (!h) return fail(SWIN_MLP_EINVAL, "NULL handle");
    if (m3_invp_mo) { m3_invp_mo[0] = h->m3; m3_invp_mo[1] = h->inv_p; m3_invp_mo[2] = h->m_o; }
    if (bias) std::memcpy(bias, h->hbias.data(), h->hbias.size() * sizeof(float));
    return SWIN_MLP_OK;
}

swin_mlp_status_t swin_attn_int8_destroy(swin_attn_int8_t h) {
    if (!h) return SWIN_MLP_OK;
    DeviceGuard guard(h->m.device);
    delete h;
    return SWIN_MLP_OK;
}

}  // extern "C"
