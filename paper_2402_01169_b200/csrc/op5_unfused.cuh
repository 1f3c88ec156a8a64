// op5_unfused.cuh — fused op #5 as its own kernel: the layout of the paper's
// starting point (FasterTransformer's quantized Swin), where FC1's int32
// accumulators go to global memory and a separate kernel dequantises, adds the
// FC1 bias, applies GELU (or ReLU) and requantises (Fig. 1 op #5,
// lines 74-78; "each fused operation ... dominated by the global memory
// accesses", 239-241).  SURVEY.md §8(f) NEXT-1: with desc.op5_unfused the
// library runs FC1 (EP_ACC) -> this kernel -> FC2 + op #6, so the bench can
// measure on B200 what the paper's change (delete this kernel, fold ReLU into
// the GEMM drain) saves against both this baseline and the fused-GELU control.
//
// Arithmetic is the fused epilogue's, operation for operation:
//   a = fl(A1) (RNE), y = fmaf(a, m1[n], b1[n]) (fl(a*m1[n]) without bias),
//   v = fl(act(y) * inv_h), Hq = clamp(rne(v) + z_h, -128, 127).
//
// HBM-bound (4 B read + 1 B written per element).  Grid-stride over quads of 4
// consecutive elements of one row (H % 32 == 0): a warp reads 512 contiguous
// bytes and writes 128 per instruction; the column index advances incrementally
// (one 64-bit modulo per thread); UNROLL quads are loaded before any is used.
#pragma once
#include <cstdint>

#include "mlp_kernels.cuh"
#include "attn_kernels.cuh"   // (FastDiv)

namespace swinmlp {

constexpr int kOp5Threads = 256, kOp5Unroll = 4;

struct Op5Args {
    const int32_t* a1;   // [T][H]
    int8_t* hq;          // [T][H]
    const float* m1;     // [H]
    const float* b1;     // [H] or nullptr (HAS_B)
    float inv_h;
    int32_t z_h;
    int32_t H;
    int64_t quads;       // T * H / 4
};

template <bool GELU, bool HAS_B, bool ZH>
__global__ void __launch_bounds__(kOp5Threads) op5_unfused_kernel(const __grid_constant__ Op5Args p) {
    using namespace sm100;
    pdl_wait();   // A1 is the previous kernel's output (programmatic dependent launch)
    const int64_t stride = (int64_t)gridDim.x * kOp5Threads;
    int64_t q = (int64_t)blockIdx.x * kOp5Threads + threadIdx.x;
    const uint32_t H = (uint32_t)p.H;
    uint32_t n = (uint32_t)((q * 4) % H);                  // column of this quad's first element
    const uint32_t dn = (uint32_t)((stride * 4) % H);      // column advance per grid stride
    const int4* a4 = reinterpret_cast<const int4*>(p.a1);
    uint32_t* h4 = reinterpret_cast<uint32_t*>(p.hq);
    for (; q < p.quads; q += kOp5Unroll * stride) {
        int4 av[kOp5Unroll];
        uint32_t nn[kOp5Unroll];
#pragma unroll
        for (int u = 0; u < kOp5Unroll; ++u) {
            const int64_t qu = q + u * stride;
            av[u] = qu < p.quads ? __ldcs(a4 + qu) : make_int4(0, 0, 0, 0);   // streamed once
            nn[u] = n;
            n += dn;
            if (n >= H) n -= H;
        }
#pragma unroll
        for (int u = 0; u < kOp5Unroll; ++u) {
            const int64_t qu = q + u * stride;
            if (qu >= p.quads) break;
            const float4 mv = __ldg(reinterpret_cast<const float4*>(p.m1 + nn[u]));
            const float2 a0 = make_float2(__int2float_rn(av[u].x), __int2float_rn(av[u].y));
            const float2 a1 = make_float2(__int2float_rn(av[u].z), __int2float_rn(av[u].w));
            float2 y0, y1;
            if constexpr (HAS_B) {
                const float4 bv = __ldg(reinterpret_cast<const float4*>(p.b1 + nn[u]));
                y0 = f2_fma(a0, make_float2(mv.x, mv.y), make_float2(bv.x, bv.y));
                y1 = f2_fma(a1, make_float2(mv.z, mv.w), make_float2(bv.z, bv.w));
            } else {
                y0 = f2_mul(a0, make_float2(mv.x, mv.y));
                y1 = f2_mul(a1, make_float2(mv.z, mv.w));
            }
            if constexpr (GELU) {
                y0 = make_float2(gelu_erf_f32(y0.x), gelu_erf_f32(y0.y));
                y1 = make_float2(gelu_erf_f32(y1.x), gelu_erf_f32(y1.y));
            }
            const float2 inv2 = make_float2(p.inv_h, p.inv_h);
            const float2 t0 = f2_mul(y0, inv2), t1 = f2_mul(y1, inv2);
            const float v[4] = {t0.x, t0.y, t1.x, t1.y};
            int32_t qv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if constexpr (ZH) {   // zero point added after rounding (reading R5)
                    qv[j] = f2i_rn_sat16(v[j]) + p.z_h;
                    if (!GELU) qv[j] = max(qv[j], p.z_h);
                } else {
                    qv[j] = __float2int_rn(GELU ? v[j] : fmaxf(v[j], 0.0f));
                }
            }
            __stcs(h4 + qu, pack_sat_s8(qv[1], qv[0], pack_sat_s8(qv[3], qv[2], 0u)));
        }
    }
}

// ---- the I-ViT shift-GELU control (reading R28) ------------
// Needs the max of each token's FC1 row before any of its outputs: one
// warp per token row, two passes over A1 (the second from L2); integer arithmetic after the
// two fp32 quantizer products, so Hq is bit-exact with the oracle.
struct ShiftGeluArgs {
    const int32_t* a1;   // [T][H]
    int8_t* hq;          // [T][H]
    const float* m1;     // [H]
    const float* b1;     // [H] or nullptr
    float inv_g;         // fl(1/s_g)
    float k_g;           // fl(fl(s_g * inv_h) * 2^-7)
    int32_t x0;          // floor(-1 / fl(1.702 s_g)) < 0
    FastDiv divx0;       // by |x0| (ShiftExp's q = floor(p / x0) = |p| / |x0| for p <= 0)
    int32_t z_h;
    int32_t H;
    int64_t T;
};

__device__ __forceinline__ int32_t sg_quant_in(int32_t a, float m, float b, float inv_g) {
    const float y = __fmaf_rn(__int2float_rn(a), m, b);
    return (int32_t)fminf(fmaxf(rintf(__fmul_rn(y, inv_g)), -32767.f), 32767.f);   // rne, clamp
}

// ShiftExp(x <= 0) with n = 15 (see swin_mlp_int8.h): 2^(x S log2 e) on the scale 2^15 |x0|.
__device__ __forceinline__ int64_t sg_shift_exp(int32_t x, int32_t x0, const FastDiv& dx0) {
    int32_t p = x + (x >> 1) - (x >> 4);             // arithmetic shifts: floor(x/2), floor(x/16)
    p = max(p, 15 * x0);
    const int32_t q = (int32_t)fdiv((uint32_t)(-p), dx0);   // p <= 0, x0 < 0: floor(p / x0) = |p| / |x0|
    const int32_t m = p - q * x0 - 2 * x0;           // r - 2 x0 > 0
    const int64_t e = 14 - q >= 0 ? (int64_t)m << (14 - q) : (int64_t)(m >> 1);
    return e > 0 ? e : 0;
}

template <bool HAS_B, bool ZH>
__global__ void __launch_bounds__(kOp5Threads) op5_shiftgelu_kernel(const __grid_constant__ ShiftGeluArgs p) {
    using namespace sm100;
    pdl_wait();   // A1 is the previous kernel's output
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kOp5Threads + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kOp5Threads) >> 5;
    const int H4 = p.H >> 2;
    for (int64_t t = warp; t < p.T; t += nwarps) {
        const int4* row = reinterpret_cast<const int4*>(p.a1 + t * p.H);
        int32_t im = -32768;
#pragma unroll 2
        for (int k = lane; k < H4; k += 32) {   // pass 1: the row max of I
            const int4 a = __ldg(row + k);
            const float4 mv = __ldg(reinterpret_cast<const float4*>(p.m1) + k);
            const float4 bv = HAS_B ? __ldg(reinterpret_cast<const float4*>(p.b1) + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            im = max(im, max(max(sg_quant_in(a.x, mv.x, bv.x, p.inv_g), sg_quant_in(a.y, mv.y, bv.y, p.inv_g)),
                             max(sg_quant_in(a.z, mv.z, bv.z, p.inv_g), sg_quant_in(a.w, mv.w, bv.w, p.inv_g))));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) im = max(im, __shfl_xor_sync(0xffffffffu, im, o));
        const int64_t e_m = sg_shift_exp(im > 0 ? -im : 0, p.x0, p.divx0);
        uint32_t* out = reinterpret_cast<uint32_t*>(p.hq + t * p.H);
#pragma unroll 2
        for (int k = lane; k < H4; k += 32) {   // pass 2 (A1 from L2)
            const int4 a = __ldg(row + k);
            const float4 mv = __ldg(reinterpret_cast<const float4*>(p.m1) + k);
            const float4 bv = HAS_B ? __ldg(reinterpret_cast<const float4*>(p.b1) + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            const int32_t I[4] = {sg_quant_in(a.x, mv.x, bv.x, p.inv_g), sg_quant_in(a.y, mv.y, bv.y, p.inv_g),
                                  sg_quant_in(a.z, mv.z, bv.z, p.inv_g), sg_quant_in(a.w, mv.w, bv.w, p.inv_g)};
            int32_t qv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t e_x = sg_shift_exp(I[j] - im, p.x0, p.divx0);
                const int64_t sum = min(e_x + e_m, (int64_t)2147483647);
                // floor((2^31 - 1) / sum): an fp32 reciprocal estimate (relative error < 2^-21, so
                // off by at most 2^10 / sum + 1), corrected to the exact floor with integer products;
                // small sums (rare: both exponentials tiny) take the double quotient
                int64_t f = 0;
                if (sum >= 4096) {
                    f = (int64_t)__fmul_rn(2147483647.0f, __frcp_rn((float)sum));
                    while (f * sum > 2147483647LL) --f;
                    while ((f + 1) * sum <= 2147483647LL) ++f;
                } else if (sum > 0) {
                    f = (int64_t)(2147483647.0 / (double)sum);
                    if (f * sum > 2147483647LL) --f;
                    else if ((f + 1) * sum <= 2147483647LL) ++f;
                }
                const int32_t sig = (int32_t)((e_x * f) >> 24);
                const float v = __fmul_rn((float)(I[j] * sig), p.k_g);
                qv[j] = ZH ? f2i_rn_sat16(v) + p.z_h : __float2int_rn(fminf(fmaxf(v, -1024.f), 1024.f));
            }
            out[k] = pack_sat_s8(qv[1], qv[0], pack_sat_s8(qv[3], qv[2], 0u));
        }
    }
}

}  // namespace swinmlp
