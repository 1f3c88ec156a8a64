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

}  // namespace swinmlp
