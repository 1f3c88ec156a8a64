// Probe: per-SM issue throughput of the epilogue's instruction mix on sm_100a.
// Each kernel runs 148 CTAs x 512 threads, a long unrolled loop of independent ops.
#include <cstdio>
#include <cstdint>
#define N_IT 4096
__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2*>(&a); }

__global__ void k_i2fp(int* out, int seed) {
    int a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    float s = 0;
    for (int i = 0; i < N_IT; ++i) {
        float f0 = __int2float_rn(a0), f1 = __int2float_rn(a1), f2 = __int2float_rn(a2), f3 = __int2float_rn(a3);
        float f4 = __int2float_rn(a4), f5 = __int2float_rn(a5), f6 = __int2float_rn(a6), f7 = __int2float_rn(a7);
        a0 ^= __float_as_int(f0); a1 ^= __float_as_int(f1); a2 ^= __float_as_int(f2); a3 ^= __float_as_int(f3);
        a4 ^= __float_as_int(f4); a5 ^= __float_as_int(f5); a6 ^= __float_as_int(f6); a7 ^= __float_as_int(f7);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + (int)s;
}
__global__ void k_i2f_s8(int* out, int seed) {
    int a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < N_IT; ++i) {
        float f0 = (float)(int8_t)(a0 >> 8), f1 = (float)(int8_t)(a1 >> 8), f2 = (float)(int8_t)(a2 >> 8), f3 = (float)(int8_t)(a3 >> 8);
        float f4 = (float)(int8_t)(a4 >> 8), f5 = (float)(int8_t)(a5 >> 8), f6 = (float)(int8_t)(a6 >> 8), f7 = (float)(int8_t)(a7 >> 8);
        a0 ^= __float_as_int(f0); a1 ^= __float_as_int(f1); a2 ^= __float_as_int(f2); a3 ^= __float_as_int(f3);
        a4 ^= __float_as_int(f4); a5 ^= __float_as_int(f5); a6 ^= __float_as_int(f6); a7 ^= __float_as_int(f7);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_f2ip(int* out, float seed) {
    float a0 = threadIdx.x * seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    uint32_t acc = 0;
    for (int i = 0; i < N_IT; ++i) {
        uint32_t d0, d1, d2, d3;
        asm volatile("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(d0) : "r"(__float2int_rn(a0)), "r"(__float2int_rn(a1)));
        asm volatile("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(d1) : "r"(__float2int_rn(a2)), "r"(__float2int_rn(a3)));
        asm volatile("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(d2) : "r"(__float2int_rn(a4)), "r"(__float2int_rn(a5)));
        asm volatile("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(d3) : "r"(__float2int_rn(a6)), "r"(__float2int_rn(a7)));
        acc ^= d0 ^ d1 ^ d2 ^ d3;
        a0 += 1.f; a1 += 1.f; a2 += 1.f; a3 += 1.f; a4 += 1.f; a5 += 1.f; a6 += 1.f; a7 += 1.f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_fmul2(int* out, float seed) {
    float2 a0 = make_float2(seed, seed + 1), a1 = make_float2(seed + 2, seed), a2 = a0, a3 = a1, a4 = a0, a5 = a1, a6 = a0, a7 = a1;
    const float2 m = make_float2(1.0001f, 0.9999f);
    for (int i = 0; i < N_IT; ++i) {
        uint64_t r0, r1, r2, r3, r4, r5, r6, r7;
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r0) : "l"(f2u(a0)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r1) : "l"(f2u(a1)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r2) : "l"(f2u(a2)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r3) : "l"(f2u(a3)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r4) : "l"(f2u(a4)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r5) : "l"(f2u(a5)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r6) : "l"(f2u(a6)), "l"(f2u(m)));
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r7) : "l"(f2u(a7)), "l"(f2u(m)));
        a0 = u2f(r0); a1 = u2f(r1); a2 = u2f(r2); a3 = u2f(r3); a4 = u2f(r4); a5 = u2f(r5); a6 = u2f(r6); a7 = u2f(r7);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_int(a0.x + a1.y + a2.x + a3.y + a4.x + a5.y + a6.x + a7.y);
}
__global__ void k_prmt(int* out, int seed) {
    uint32_t a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < N_IT; ++i) {
        a0 = __byte_perm(a0, 0x4B000000u, 0x7650); a1 = __byte_perm(a1, 0x4B000000u, 0x7651);
        a2 = __byte_perm(a2, 0x4B000000u, 0x7652); a3 = __byte_perm(a3, 0x4B000000u, 0x7653);
        a4 = __byte_perm(a4, 0x4B000000u, 0x7650); a5 = __byte_perm(a5, 0x4B000000u, 0x7651);
        a6 = __byte_perm(a6, 0x4B000000u, 0x7652); a7 = __byte_perm(a7, 0x4B000000u, 0x7653);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
template <typename K, typename A>
void run(const char* name, K k, A arg, int ops_per_iter_per_thread, int* d) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<148, 512>>>(d, arg);
    cudaEventRecord(e0);
    k<<<148, 512>>>(d, arg);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = 148.0 * 512 * N_IT * ops_per_iter_per_thread;
    double per_sm_clk = ops / (ms * 1e-3) / 148 / 1.9e9;
    printf("%-10s %8.3f ms  %7.1f thread-ops/clk/SM (@1.9GHz)\n", name, ms, per_sm_clk);
}
int main() {
    int* d; cudaMalloc(&d, 148 * 512 * 4);
    run("i2fp", k_i2fp, 3, 8, d);
    run("i2f_s8", k_i2f_s8, 3, 8, d);
    run("f2ip(x2)", k_f2ip, 0.5f, 8, d);
    run("fmul2(x2)", k_fmul2, 1.0f, 16, d);
    run("prmt", k_prmt, 3, 8, d);
    return 0;
}
