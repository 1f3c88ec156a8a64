// attn_kernels.cuh — sm_100a kernels of the attention half of the quantized Swin block
// (Fig. 1 lines 39-62):
//
//   op1_kernel        fused op #1: LayerNorm -> window shift -> Q.  HBM-bound
//                     gather: one warp per output (window-ordered) row, reading its source
//                     token's fp32 row (4C bytes, 16-B loads) and writing C int8 bytes; U rows
//                     per warp in flight.  Row statistics: a two-pass mean / centred sum of
//                     squares over the row held in registers, reduced by xor butterflies (every
//                     lane derives the identical value).
//   attn_core_kernel  Q.K GEMM -> fused op #3 (dQ with the folded attention scale, relative
//                     position bias, shifted-window mask, softmax, Q) -> V.att GEMM with its
//                     int8 requant, per (window, head).  One warp per item;
//                     the head's q / k rows and the transposed v slice staged in the warp's
//                     shared memory; the 16 x N score tile of one m-tile lives in mma
//                     accumulators; P goes through shared memory to become the A operand of the
//                     P.V product; the output rows are scattered back to raster order (window
//                     reverse + inverse shift) so the Proj GEMM and op #4's residual add see
//                     the residual stream's token order.
//
// The per-window GEMMs are tiny (S: N x N x 32, O: N x 32 x N, N = 49 or 144): 4 * N^2 * 32
// int8 ops per (window, head) against 4 * N * 32 bytes of q / k / v / output, ~98 ops/B at
// N = 49 -- far under the int8 ridge (~500 ops/B), so the core is bound by HBM (and the softmax
// ALU work), not by the tensor pipe: they run on warp-level mma.sync.m16n8k32 (s8), whose
// operand fragments come straight from row-major q / k and the transposed v in shared memory.
// tcgen05 tiles (M >= 64 per CTA, TMEM allocation, descriptor setup) buy nothing at this
// intensity.
#pragma once
#include <cstdint>
#include <type_traits>

#include "sm100_ptx.cuh"

namespace swinmlp {

// ------------------------------------------------------------------------------- op #1
// Unsigned division by a runtime constant d >= 1 for n < 2^31: q = (umulhi(n, mul) + n) >> sh
// with sh = ceil(log2 d), mul = floor(2^32 (2^sh - d) / d) + 1 (exact for every such n).
struct FastDiv {
    uint32_t d, mul, sh;
};
__host__ inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t sh = 0;
    while ((1ull << sh) < d) ++sh;
    const uint64_t mul = ((1ull << 32) * ((1ull << sh) - d)) / d + 1;
    return FastDiv{d, (uint32_t)mul, sh};
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (__umulhi(n, f.mul) + n) >> f.sh;
}

struct Op1Args {
    const float* x;        // [B][Hs][Ws][C] fp32 (raster)
    int8_t* y;             // [B*Hs*Ws][C] int8 (window order)
    int64_t rows;          // B*Hs*Ws (< 2^31)
    int32_t C, Hs, Ws, M, shift;
    FastDiv divN, divNW, divNWx, divM;   // by M*M, windows per image, windows per row, M
    const float* gamma;
    const float* beta;
    float eps, inv_s;      // inv_s = fl(1/s) of the output quantizer
    int32_t z;
};

// Raster row of window-ordered row r (R21/R22): window w = (r / M^2) mod nW of image
// b, token p = r mod M^2; source pixel ((wy M + iy + s) mod Hs, (wx M + ix + s) mod Ws).
__device__ __forceinline__ uint32_t window_src_row(uint32_t r, const Op1Args& a) {
    const uint32_t wi = fdiv(r, a.divN), p = r - wi * a.divN.d;
    const uint32_t b = fdiv(wi, a.divNW), w = wi - b * a.divNW.d;
    const uint32_t wy = fdiv(w, a.divNWx), wx = w - wy * a.divNWx.d;
    const uint32_t iy = fdiv(p, a.divM), ix = p - iy * (uint32_t)a.M;
    uint32_t y = wy * a.M + iy + a.shift, x = wx * a.M + ix + a.shift;
    if (y >= (uint32_t)a.Hs) y -= a.Hs;
    if (x >= (uint32_t)a.Ws) x -= a.Ws;
    return (b * a.Hs + y) * (uint32_t)a.Ws + x;
}

template <int L>
__device__ __forceinline__ float group_sum(float v) {   // butterfly over the L lanes of a row
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ uint32_t q4_pack(float4 v, int32_t z) {
    const int a = min(max(__float2int_rn(fminf(fmaxf(v.x, -1024.f), 1024.f)) + z, -128), 127);
    const int b = min(max(__float2int_rn(fminf(fmaxf(v.y, -1024.f), 1024.f)) + z, -128), 127);
    const int c = min(max(__float2int_rn(fminf(fmaxf(v.z, -1024.f), 1024.f)) + z, -128), 127);
    const int d = min(max(__float2int_rn(fminf(fmaxf(v.w, -1024.f), 1024.f)) + z, -128), 127);
    return (uint32_t)(a & 0xff) | ((uint32_t)(b & 0xff) << 8) | ((uint32_t)(c & 0xff) << 16) | ((uint32_t)d << 24);
}

// A row of C = 4 L VPL channels on a group of L lanes (32 / L rows per warp instruction), VPL
// float4 per lane, U row groups per warp in flight.  fp32 statistics:
//   mu = fl(S / C), S the butterfly sum of the row; var = fl(SS / C), SS the butterfly sum of
//   fl(x - mu)^2 (fmaf); rstd = fl(1 / fl(sqrt(fl(var + eps))));
//   yhat = fmaf(fl(fl(x - mu) * rstd), gamma, beta);  Y = clamp(rne(fl(yhat * inv_s)) + z)
// (the oracle's statistics are in double: Y within 1 LSB on <= 0.01 %).
template <int L, int VPL, int U>
__global__ void __launch_bounds__(256) op1_kernel(const Op1Args a) {
    using namespace sm100;
    constexpr int RPW = 32 / L;   // rows per warp instruction
    pdl_wait();   // x may be the previous kernel's output
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31, sub = lane / L, gl = lane % L;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int C4 = a.C >> 2;
    float4 g[VPL], bt[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int idx = gl + L * v;
        g[v] = idx < C4 ? __ldg(reinterpret_cast<const float4*>(a.gamma) + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
        bt[v] = idx < C4 ? __ldg(reinterpret_cast<const float4*>(a.beta) + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float Cf = (float)a.C;
    for (int64_t r0 = warp * (U * RPW); r0 < a.rows; r0 += nwarps * (U * RPW)) {
        float4 xv[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + u * RPW + sub;
            const float4* src = reinterpret_cast<const float4*>(
                a.x + (r < a.rows ? (int64_t)window_src_row((uint32_t)r, a) : 0) * (int64_t)a.C);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int idx = gl + L * v;
                xv[u][v] = (r < a.rows && idx < C4) ? __ldcs(src + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + u * RPW + sub;
            float s = 0.f;
#pragma unroll
            for (int v = 0; v < VPL; ++v)
                s = __fadd_rn(__fadd_rn(s, __fadd_rn(xv[u][v].x, xv[u][v].y)), __fadd_rn(xv[u][v].z, xv[u][v].w));
            const float mu = __fdiv_rn(group_sum<L>(s), Cf);
            float ss = 0.f;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                if (gl + L * v >= C4) continue;
                const float d0 = __fsub_rn(xv[u][v].x, mu), d1 = __fsub_rn(xv[u][v].y, mu);
                const float d2 = __fsub_rn(xv[u][v].z, mu), d3 = __fsub_rn(xv[u][v].w, mu);
                ss = __fmaf_rn(d0, d0, ss); ss = __fmaf_rn(d1, d1, ss);
                ss = __fmaf_rn(d2, d2, ss); ss = __fmaf_rn(d3, d3, ss);
            }
            const float var = __fdiv_rn(group_sum<L>(ss), Cf);
            const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, a.eps)));
            if (r >= a.rows) continue;
            uint32_t* dst = reinterpret_cast<uint32_t*>(a.y + r * (int64_t)a.C);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int idx = gl + L * v;
                if (idx >= C4) continue;
                const float4 xx = xv[u][v];
                float4 yh;
                yh.x = __fmaf_rn(__fmul_rn(__fsub_rn(xx.x, mu), rstd), g[v].x, bt[v].x);
                yh.y = __fmaf_rn(__fmul_rn(__fsub_rn(xx.y, mu), rstd), g[v].y, bt[v].y);
                yh.z = __fmaf_rn(__fmul_rn(__fsub_rn(xx.z, mu), rstd), g[v].z, bt[v].z);
                yh.w = __fmaf_rn(__fmul_rn(__fsub_rn(xx.w, mu), rstd), g[v].w, bt[v].w);
                const float4 q = make_float4(__fmul_rn(yh.x, a.inv_s), __fmul_rn(yh.y, a.inv_s),
                                             __fmul_rn(yh.z, a.inv_s), __fmul_rn(yh.w, a.inv_s));
                dst[idx] = q4_pack(q, a.z);
            }
        }
    }
}

// ------------------------------------------------------------------------ attention core
struct AttnArgs {
    const int8_t* qkv;     // [T][3C] window order: q | k | v, head h at columns h*32 .. h*32+31
    int8_t* out;           // [T][C] raster order
    int64_t n_win;         // windows (B * nW)
    int32_t C, heads, Hs, Ws, shift, nW;
    const float* bias;     // [heads][MT*16][NT*8] relative position bias, -inf at columns >= N
    float m3, inv_p, m_o;  // folded: fl(fl(s_q s_k) / sqrt(32)), fl(1/s_p), fl(fl(s_p s_v) / s_a)
    int32_t z_a;
    int8_t* p_tap;         // debug: [windows][heads][N][N] Pq, or nullptr
};

constexpr int kAttnWarps = 8;

__device__ __forceinline__ void mma_s8_16832(int32_t (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// rne(v) saturated to [0, 255] (v >= 0 here: a probability times 127)
__device__ __forceinline__ uint32_t f2u8_rn_sat(float v) {
    uint32_t q;
    asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(q) : "f"(v));
    return q;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int M>
struct AttnGeom {
    static constexpr int N = M * M;                  // tokens per window
    static constexpr int MT = (N + 15) / 16;         // m-tiles of the score / output rows
    static constexpr int NT = (N + 7) / 8;           // n-tiles of the score columns
    static constexpr int KP = (N + 31) / 32 * 32;    // P.V reduction length (zero padded)
    static constexpr int QROWS = MT * 16, KROWS = NT * 8, NP = NT * 8;
    static constexpr int Q_OFF = 0, K_OFF = QROWS * 32, VT_OFF = K_OFF + KROWS * 32, P_OFF = VT_OFF + 32 * KP;
    static constexpr int BYTES = P_OFF + 16 * KP;    // per warp
    static constexpr bool BIAS_SMEM = M <= 8;        // the head's padded bias tile staged per CTA
    static constexpr int BIAS_BYTES = BIAS_SMEM ? QROWS * NP * 4 : 0;
    static constexpr int SMEM = BIAS_BYTES + kAttnWarps * BYTES;
};

// Shifted-window region of a token (reading R25): 3 x 3 regions split at Hs - M and Hs - s.
__device__ __forceinline__ int shift_region(int y, int x, int Hs, int Ws, int M, int s) {
    const int ry = y < Hs - M ? 0 : y < Hs - s ? 1 : 2;
    const int rx = x < Ws - M ? 0 : x < Ws - s ? 1 : 2;
    return ry * 3 + rx;
}

// Per (window, head), with i, j tokens of the window and d < 32:
//   S[i][j] = sum_d q[i][d] k[j][d]                                   (mma, int32, exact)
//   l = fmaf(fl(S), m3, bias[h][i][j]) (+ -100 across shifted regions, another rounding)
//   e = ex2(fmaf(l, log2 e, -fl(max_j l * log2 e))),  Pq = rne_sat(fl(e * fl(inv_p * rcp(sum_j e))))
//   (the oracle rounds S m3 and + bias separately and divides in double: every GPU deviation
//   is a few fp32 ulps of p, far inside the 1-LSB tier)
//   O[i][n] = sum_j Pq[i][j] v[j][n]                                  (mma, int32, exact)
//   out[raster(i)][h*32 + n] = clamp(rne(fl(fl(O) * m_o)) + z_a, -128, 127)
// (the oracle's softmax is in double: Pq within 1 LSB on <= 0.01 %).
// CTA = kAttnWarps warps on ONE head (blockIdx.x % heads): the head's bias tile is staged once;
// warp w takes windows (blockIdx.x / heads) * kAttnWarps + w, + (gridDim.x / heads) * kAttnWarps, ...
template <int M>
__global__ void __launch_bounds__(32 * kAttnWarps) attn_core_kernel(const AttnArgs a) {
    using namespace sm100;
    using G = AttnGeom<M>;
    constexpr int N = G::N, MT = G::MT, NT = G::NT, KP = G::KP, NP = G::NP;
    extern __shared__ __align__(16) uint8_t attn_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int h = (int)(blockIdx.x % (unsigned)a.heads);
    const int64_t cg = blockIdx.x / (unsigned)a.heads, ncg = gridDim.x / (unsigned)a.heads;
    float* sBias = reinterpret_cast<float*>(attn_smem);
    uint8_t* sm = attn_smem + G::BIAS_BYTES + wid * G::BYTES;
    uint8_t* sQ = sm + G::Q_OFF;
    uint8_t* sK = sm + G::K_OFF;
    uint8_t* sVt = sm + G::VT_OFF;
    uint8_t* sP = sm + G::P_OFF;
    // zero this warp's region once: the pads (rows >= N of q / k, columns >= N of v^T and P)
    // are never written again
    for (int i = lane * 16; i < G::BYTES; i += 32 * 16) *reinterpret_cast<int4*>(sm + i) = make_int4(0, 0, 0, 0);
    const float* gbias = a.bias + (int64_t)h * G::QROWS * NP;
    if constexpr (G::BIAS_SMEM) {   // (a constant of the layer: no wait on the previous kernel)
        for (int i = threadIdx.x; i < G::QROWS * NP / 4; i += 32 * kAttnWarps)
            reinterpret_cast<float4*>(sBias)[i] = __ldg(reinterpret_cast<const float4*>(gbias) + i);
        __syncthreads();
    } else {
        __syncwarp();
    }
    const float* bias_h = G::BIAS_SMEM ? sBias : gbias;
    pdl_wait();   // qkv: the QKV GEMM's output
    pdl_launch_dependents();
    const int g = lane >> 2, tq = lane & 3;
    const int C = a.C, C3 = 3 * a.C;
    const float L2E = 1.4426950408889634f;
    const int nWx = a.Ws / M, nWy = a.Hs / M;
    for (int64_t win = cg * kAttnWarps + wid; win < a.n_win; win += ncg * kAttnWarps) {
        const int8_t* base = a.qkv + win * (int64_t)N * C3 + h * 32;
        // ---- stage q, k (row-major, 16-B granules) and v^T of this head (4 x 4 byte blocks: 4
        // tokens x 4 dims read as 4 words, transposed with 8 PRMT, written as 4 words of v^T)
        for (int idx = lane; idx < 2 * N; idx += 32) {
            const int i = idx >> 1, half = idx & 1;
            const int8_t* rp = base + (int64_t)i * C3 + half * 16;
            *reinterpret_cast<int4*>(sQ + i * 32 + half * 16) = ld_nc_v4(rp);
            *reinterpret_cast<int4*>(sK + i * 32 + half * 16) = ld_nc_v4(rp + C);
        }
        for (int idx = lane; idx < ((N + 3) / 4) * 8; idx += 32) {
            const int i4 = idx >> 3, d4 = idx & 7;   // tokens 4 i4 .. 4 i4 + 3, dims 4 d4 .. 4 d4 + 3
            uint32_t w[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = 4 * i4 + r;
                w[r] = i < N ? __ldg(reinterpret_cast<const uint32_t*>(base + (int64_t)i * C3 + 2 * C + 4 * d4)) : 0u;
            }
            const uint32_t t0 = __byte_perm(w[0], w[1], 0x5140), t1 = __byte_perm(w[0], w[1], 0x7362);
            const uint32_t t2 = __byte_perm(w[2], w[3], 0x5140), t3 = __byte_perm(w[2], w[3], 0x7362);
            uint32_t* vt = reinterpret_cast<uint32_t*>(sVt + (4 * d4) * KP + 4 * i4);
            vt[0] = __byte_perm(t0, t2, 0x5410);
            vt[KP / 4] = __byte_perm(t0, t2, 0x7632);
            vt[2 * (KP / 4)] = __byte_perm(t1, t3, 0x5410);
            vt[3 * (KP / 4)] = __byte_perm(t1, t3, 0x7632);
        }
        __syncwarp();
        const int w_in = (int)(win % a.nW);
        const int64_t b_img = win / a.nW;
        const int wy = w_in / nWx, wx = w_in - wy * nWx;
        // shifted blocks: only windows on the last window row / column straddle regions
        const bool masked = a.shift > 0 && (wy == nWy - 1 || wx == nWx - 1);
        auto region = [&](int i) { return shift_region(wy * M + i / M, wx * M + i % M, a.Hs, a.Ws, M, a.shift); };
        // raster row of window token i (the inverse of op #1's gather)
        auto raster = [&](int i) -> int64_t {
            const int iy = i / M, ix = i - iy * M;
            int y = wy * M + iy + a.shift, x = wx * M + ix + a.shift;
            if (y >= a.Hs) y -= a.Hs;
            if (x >= a.Ws) x -= a.Ws;
            return (b_img * a.Hs + y) * (int64_t)a.Ws + x;
        };
        // per-lane column regions of the shifted block (4-bit codes, n-tile nt at bits 4 nt of
        // creg[e] for column nt*8 + 2 tq + e); only windows on the last window row / column
        constexpr int CW = (NT + 7) / 8;   // 32-bit words of 8 nibbles
        uint32_t creg[2][CW];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int k = 0; k < CW; ++k) creg[e][k] = 0u;
        if (masked) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int jj = nt * 8 + tq * 2 + e;
                    creg[e][nt / 8] |= (uint32_t)(jj < N ? region(jj) : 15) << (4 * (nt % 8));
                }
        }
        // N = 16 k + 1 (M = 7: 49 tokens): the last token row is done on its own below (dp4a,
        // lane-parallel over keys), not as an m-tile of 15 empty rows
        constexpr int MTM = (N % 16 == 1) ? MT - 1 : MT;
#pragma unroll 1
        for (int mt = 0; mt < MTM; ++mt) {
            const int i0 = mt * 16 + g, i1 = i0 + 8;
            uint32_t af[4];
            af[0] = *reinterpret_cast<const uint32_t*>(sQ + i0 * 32 + tq * 4);
            af[1] = *reinterpret_cast<const uint32_t*>(sQ + i1 * 32 + tq * 4);
            af[2] = *reinterpret_cast<const uint32_t*>(sQ + i0 * 32 + 16 + tq * 4);
            af[3] = *reinterpret_cast<const uint32_t*>(sQ + i1 * 32 + 16 + tq * 4);
            float l[NT][4];
            // logits l = fma(fl(S), m3, bias) (+ -100 across shifted regions); padded columns -inf
            auto logits = [&](auto mk) {
                constexpr bool MK = decltype(mk)::value;
                const uint32_t r0 = MK && i0 < N ? (uint32_t)region(i0) : 0u, r1 = MK && i1 < N ? (uint32_t)region(i1) : 0u;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    int32_t c[4] = {0, 0, 0, 0};
                    const uint32_t b0 = *reinterpret_cast<const uint32_t*>(sK + (nt * 8 + g) * 32 + tq * 4);
                    const uint32_t b1 = *reinterpret_cast<const uint32_t*>(sK + (nt * 8 + g) * 32 + 16 + tq * 4);
                    mma_s8_16832(c, af, b0, b1);
                    const int j = nt * 8 + tq * 2;
                    const float2 bv0 = *reinterpret_cast<const float2*>(bias_h + i0 * NP + j);
                    const float2 bv1 = *reinterpret_cast<const float2*>(bias_h + i1 * NP + j);
                    l[nt][0] = __fmaf_rn((float)c[0], a.m3, bv0.x);
                    l[nt][1] = __fmaf_rn((float)c[1], a.m3, bv0.y);
                    l[nt][2] = __fmaf_rn((float)c[2], a.m3, bv1.x);
                    l[nt][3] = __fmaf_rn((float)c[3], a.m3, bv1.y);
                    if constexpr (MK) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint32_t rj = (creg[e & 1][nt / 8] >> (4 * (nt % 8))) & 15u;
                            l[nt][e] = __fadd_rn(l[nt][e], rj == (e < 2 ? r0 : r1) ? 0.0f : -100.0f);
                        }
                    }
                }
            };
            if (masked) logits(std::true_type{});
            else logits(std::false_type{});
            // row max / sum over the quad (4 lanes share a row; butterflies give every lane the
            // same value), then probabilities and their quantization
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                mx0 = fmaxf(mx0, fmaxf(l[nt][0], l[nt][1]));
                mx1 = fmaxf(mx1, fmaxf(l[nt][2], l[nt][3]));
            }
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
            }
            // e = 2^(l log2e - max log2e): one fma per element (padded columns: ex2(-inf) = 0)
            const float nm0 = -__fmul_rn(mx0, L2E), nm1 = -__fmul_rn(mx1, L2E);
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                l[nt][0] = ex2_approx(__fmaf_rn(l[nt][0], L2E, nm0));
                l[nt][1] = ex2_approx(__fmaf_rn(l[nt][1], L2E, nm0));
                l[nt][2] = ex2_approx(__fmaf_rn(l[nt][2], L2E, nm1));
                l[nt][3] = ex2_approx(__fmaf_rn(l[nt][3], L2E, nm1));
                s0 = __fadd_rn(s0, __fadd_rn(l[nt][0], l[nt][1]));
                s1 = __fadd_rn(s1, __fadd_rn(l[nt][2], l[nt][3]));
            }
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                s0 = __fadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
                s1 = __fadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
            }
            // Pq = rne(e * fl(inv_p / sum)) in [0, 127] (one product per element)
            const float q0 = __fmul_rn(a.inv_p, rcp_approx(s0)), q1 = __fmul_rn(a.inv_p, rcp_approx(s1));
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int j = nt * 8 + tq * 2;
                const uint32_t p0 = f2u8_rn_sat(__fmul_rn(l[nt][0], q0)), p1 = f2u8_rn_sat(__fmul_rn(l[nt][1], q0));
                const uint32_t p2 = f2u8_rn_sat(__fmul_rn(l[nt][2], q1)), p3 = f2u8_rn_sat(__fmul_rn(l[nt][3], q1));
                *reinterpret_cast<uint16_t*>(sP + g * KP + j) = (uint16_t)__byte_perm(p0, p1, 0x0040);
                *reinterpret_cast<uint16_t*>(sP + (g + 8) * KP + j) = (uint16_t)__byte_perm(p2, p3, 0x0040);
            }
            if (a.p_tap) {   // (debug) the valid rows of this m-tile's Pq
                __syncwarp();
                int8_t* pt = a.p_tap + (win * a.heads + h) * (int64_t)N * N;
                for (int k = lane; k < 16 * N; k += 32) {
                    const int r = k / N, jj = k - r * N, i = mt * 16 + r;
                    if (i < N) pt[i * N + jj] = (int8_t)sP[r * KP + jj];
                }
            }
            __syncwarp();
            // O = Pq . V for this m-tile: 4 n-tiles of 8 head dims, KP / 32 k-steps
            int32_t o[4][4];
#pragma unroll
            for (int n2 = 0; n2 < 4; ++n2) o[n2][0] = o[n2][1] = o[n2][2] = o[n2][3] = 0;
#pragma unroll
            for (int ks = 0; ks < KP / 32; ++ks) {
                uint32_t pa[4];
                pa[0] = *reinterpret_cast<const uint32_t*>(sP + g * KP + ks * 32 + tq * 4);
                pa[1] = *reinterpret_cast<const uint32_t*>(sP + (g + 8) * KP + ks * 32 + tq * 4);
                pa[2] = *reinterpret_cast<const uint32_t*>(sP + g * KP + ks * 32 + 16 + tq * 4);
                pa[3] = *reinterpret_cast<const uint32_t*>(sP + (g + 8) * KP + ks * 32 + 16 + tq * 4);
#pragma unroll
                for (int n2 = 0; n2 < 4; ++n2) {
                    const uint32_t b0 = *reinterpret_cast<const uint32_t*>(sVt + (n2 * 8 + g) * KP + ks * 32 + tq * 4);
                    const uint32_t b1 = *reinterpret_cast<const uint32_t*>(sVt + (n2 * 8 + g) * KP + ks * 32 + 16 + tq * 4);
                    mma_s8_16832(o[n2], pa, b0, b1);
                }
            }
            __syncwarp();   // (P is rewritten by the next m-tile)
            // requant into the (now free) P tile as a 16 x 32 int8 row block, then one 16-B store per
            // lane (row lane / 2, half lane % 2) to the token's raster row
#pragma unroll
            for (int half = 0; half < 2; ++half) {
#pragma unroll
                for (int n2 = 0; n2 < 4; ++n2) {   // clamp(rne(fl(fl(O) m_o)) + z_a), saturating pack
                    const int q0 = __float2int_rn(__fmul_rn((float)o[n2][2 * half], a.m_o)) + a.z_a;
                    const int q1 = __float2int_rn(__fmul_rn((float)o[n2][2 * half + 1], a.m_o)) + a.z_a;
                    *reinterpret_cast<uint16_t*>(sP + (g + 8 * half) * 32 + n2 * 8 + tq * 2) =
                        (uint16_t)pack_sat_s8(q1, q0, 0u);
                }
            }
            __syncwarp();
            {
                const int r = lane >> 1, i = mt * 16 + r;
                if (i < N)
                    *reinterpret_cast<int4*>(a.out + raster(i) * C + h * 32 + (lane & 1) * 16) =
                        *reinterpret_cast<const int4*>(sP + r * 32 + (lane & 1) * 16);
            }
            __syncwarp();   // (the P tile is rewritten by the next m-tile)
        }
        if constexpr (N % 16 == 1) {
            // ---- the last token row r = N - 1: S[r][j] by dp4a for keys j = lane, lane + 32, the
            // same fp32 softmax steps as the m-tiles (one fma per logit and per exponent,
            // e * fl(inv_p * rcp(sum))), Pq into smem, O[r][n] = Pq . v^T[n] by dp4a for n = lane
            constexpr int r = N - 1;
            uint32_t qw[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) qw[k] = reinterpret_cast<const uint32_t*>(sQ + r * 32)[k];
            const int rr = masked ? region(r) : 0;
            float lv[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int j = (int)lane + 32 * t;
                float l = -INFINITY;
                if (j < N) {
                    const uint32_t* kr = reinterpret_cast<const uint32_t*>(sK + j * 32);
                    int acc = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc = __dp4a((int)qw[k], (int)kr[k], acc);
                    l = __fmaf_rn((float)acc, a.m3, bias_h[r * NP + j]);
                    if (masked && region(j) != rr) l = __fadd_rn(l, -100.0f);
                }
                lv[t] = l;
            }
            float mx = fmaxf(lv[0], lv[1]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float nm = -__fmul_rn(mx, L2E);
            const float e0 = ex2_approx(__fmaf_rn(lv[0], L2E, nm)), e1 = ex2_approx(__fmaf_rn(lv[1], L2E, nm));
            float sm = __fadd_rn(e0, e1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sm = __fadd_rn(sm, __shfl_xor_sync(0xffffffffu, sm, o));
            const float qs = __fmul_rn(a.inv_p, rcp_approx(sm));
            const uint32_t p0 = f2u8_rn_sat(__fmul_rn(e0, qs)), p1 = f2u8_rn_sat(__fmul_rn(e1, qs));
            sP[lane] = (uint8_t)p0;
            if ((int)lane + 32 < KP) sP[lane + 32] = (int)lane + 32 < N ? (uint8_t)p1 : (uint8_t)0;
            if (a.p_tap) {
                int8_t* pt = a.p_tap + (win * a.heads + h) * (int64_t)N * N + (int64_t)r * N;
                pt[lane] = (int8_t)p0;
                if ((int)lane + 32 < N) pt[lane + 32] = (int8_t)p1;
            }
            __syncwarp();
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(sP);
            const uint32_t* vw = reinterpret_cast<const uint32_t*>(sVt + lane * KP);
            int ov = 0;
#pragma unroll
            for (int w = 0; w < KP / 4; ++w) ov = __dp4a((int)pw[w], (int)vw[w], ov);
            const int qo = min(max(__float2int_rn(__fmul_rn((float)ov, a.m_o)) + a.z_a, -128), 127);
            a.out[raster(r) * C + h * 32 + lane] = (int8_t)qo;
            __syncwarp();   // (the P row is rewritten by the next window)
        }
        __syncwarp();   // (q / k / v^T are restaged by the next window)
    }
}

}  // namespace swinmlp
