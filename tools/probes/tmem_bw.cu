// TMEM read / write throughput probe (sm_100a): W warps each issue N tcgen05.ld
// (32x32b.xR) + wait::ld; reports bytes per SM clock.  Build:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tools/probes/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld16(uint32_t a, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
__device__ __forceinline__ void st16(uint32_t a, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}

template <int MODE>   // 0: ld + wait each, 1: 4 lds then wait, 2: st, 3: 4 lds then wait, rotating over all 512 columns
__global__ void __launch_bounds__(640, 1) probe(int iters, int nwarps, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t slot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = slot + (((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    if ((int)warp < nwarps) {
        const uint32_t col0 = (warp >> 2) * 64;
        for (int i = 0; i < iters; ++i) {
            uint32_t r[16];
            if (MODE == 0) {
                ld16(tb + col0 + (i & 3) * 16, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                acc ^= r[0] ^ r[15];
            } else if (MODE == 1) {
                uint32_t a[16], b[16], c[16];
                ld16(tb + col0, r); ld16(tb + col0 + 16, a); ld16(tb + col0 + 32, b); ld16(tb + col0 + 48, c);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                acc ^= r[0] ^ a[3] ^ b[7] ^ c[15];
            } else if (MODE == 3) {
                uint32_t a[16], b[16], c[16];
                const uint32_t cb = ((uint32_t)(i * 64 + warp * 128)) & 511u;
                ld16(tb + cb, r); ld16(tb + cb + 16, a); ld16(tb + cb + 32, b); ld16(tb + cb + 48, c);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                acc ^= r[0] ^ a[3] ^ b[7] ^ c[15] ^ r[9] ^ a[11];
            } else {
                for (int k = 0; k < 16; ++k) r[k] = acc + k;
                st16(tb + col0 + (i & 3) * 16, r);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                acc += 1;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
}

int main() {
    unsigned long long* out; uint32_t* sink;
    cudaMalloc(&out, 8 * 148); cudaMalloc(&sink, 4 * 640);
    const int iters = 4096;
    for (int mode = 0; mode < 4; ++mode) {
        for (int nw : {1, 4, 8, 16, 20}) {
            auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : probe<3>;
            k<<<1, 640>>>(iters, nw, out, sink);
            cudaDeviceSynchronize();
            unsigned long long c = 0;
            cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
            const double per = (mode == 1 || mode == 3) ? 4.0 : 1.0;
            const double bytes = (double)iters * nw * 32 * 16 * 4 * per;
            printf("mode %d (%s) warps %2d: %8llu clk  %.1f B/clk  %.1f clk/instr/warp\n", mode,
                   mode == 0 ? "ld16+wait" : mode == 1 ? "4xld16+wait" : mode == 2 ? "st16+wait" : "4xld16 rot", nw, c, bytes / c,
                   (double)c / iters / per);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
