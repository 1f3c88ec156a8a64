// TMA ring throughput probe: every CTA streams a [rows][128 B] int8 matrix (L2
// resident after the first pass) through an S-stage ring of 16 KB boxes; the
// consumer only waits and releases.  Reports bytes / ns per SM and per GPU.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../../paper_2402_01169_b200/csrc/sm100_ptx.cuh"
using namespace sm100;

__global__ void __launch_bounds__(64, 1) ring(const __grid_constant__ CUtensorMap tm, int S, int items, int rows_total,
                                               unsigned long long* out, int cs) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t bars = base + (uint32_t)S * 16384u;
    const uint32_t warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(bars + 8u * s, 1); mbar_init(bars + 8u * (S + s), (uint32_t)cs); }
        fence_mbar_init();
    }
    cluster_sync_all();
    const uint32_t rank = cluster_ctarank();
    unsigned long long t0 = clock64();
    if (warp == 0) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * (S + s), ph ^ 1u);
            if (elect_one()) {
                mbar_arrive_expect_tx(bars + 8u * s, 16384u);
                const int row = (int)(((unsigned)it * 128u + (blockIdx.x / cs) * 1024u) % (unsigned)rows_total);
                if (cs == 1) tma_load_2d(&tm, base + (uint32_t)s * 16384u, bars + 8u * s, 0, row);
                else {
                    const uint32_t hr = 128u / (uint32_t)cs;
                    tma_load_2d_mc(&tm, base + (uint32_t)s * 16384u + rank * hr * 128u, bars + 8u * s, 0,
                                   row + (int)(rank * hr), (uint16_t)((1u << cs) - 1u));
                }
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    } else {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * s, ph);
            __syncwarp();
            if (elect_one()) {
                if (cs == 1) mbar_arrive(bars + 8u * (S + s));
                else for (int r = 0; r < cs; ++r)   // release the slot in every CTA of the cluster
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa(bars + 8u * (S + s), (uint32_t)r)) : "memory");
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    }
    cluster_sync_all();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    const int rows_total = 2304;   // 288 KB of weights (C = 192 stage: W1 + W2)
    int8_t* w; cudaMalloc(&w, (size_t)rows_total * 128);
    cudaMemset(w, 1, (size_t)rows_total * 128);
    unsigned long long* out; cudaMalloc(&out, 148 * 8);
    void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows_total}; cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {128, 128}; cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int items = 4000;
    for (int cs : {1, 2, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(64);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        for (int grid : {cs, 148 / cs * cs}) {
            for (int S : {3, 8}) {
                const int smem = S * 16384 + 1024 + 16 * S + 64;
                cfg.gridDim = dim3(grid); cfg.dynamicSmemBytes = smem;
                int itemsv = items, rt = rows_total, csv = cs, Sv = S;
                void* args[] = {(void*)&tm, (void*)&Sv, (void*)&itemsv, (void*)&rt, (void*)&out, (void*)&csv};
                printf("launch cs %d grid %d S %d\n", cs, grid, S); fflush(stdout);
                cudaError_t e = cudaLaunchKernelExC(&cfg, (const void*)ring, args);
                if (e != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(e)); return 1; }
                e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("sync error %s\n", cudaGetErrorString(e)); return 1; }
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a);
                cudaLaunchKernelExC(&cfg, (const void*)ring, args);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                const double bytes = (double)items * 16384.0;
                printf("cs %d grid %3d S %2d: %.1f us  %.1f B/ns received per SM  %.0f GB/s received total\n", cs, grid, S,
                       ms * 1e3, bytes / (ms * 1e6), bytes * grid / (ms * 1e6));
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
