// TMA ingest-rate probe: CTAs stream an L2-resident [rows][128 B] int8 matrix into smem through
// P independent rings (one producer warp each, S stages of box_rows x 128 B boxes); consumers
// only wait and release.  Reports bytes received per SM per ns for box sizes and producer counts.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../../paper_2402_01169_b200/csrc/sm100_ptx.cuh"
using namespace sm100;

__global__ void __launch_bounds__(256, 1) ring(const __grid_constant__ CUtensorMap tm, int S, int items, int rows_total,
                                                int box_rows, int P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t box = (uint32_t)box_rows * 128u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t ring_id = warp >> 1;   // warps 2r (producer), 2r+1 (consumer)
    const uint32_t rbase = base + ring_id * (uint32_t)S * box;
    const uint32_t bars = base + (uint32_t)P * (uint32_t)S * box + ring_id * 16u * (uint32_t)S;
    if ((warp & 1u) == 0 && (int)ring_id < P && (threadIdx.x & 31) == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(bars + 8u * s, 1); mbar_init(bars + 8u * (S + s), 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if ((int)ring_id >= P) return;
    if ((warp & 1u) == 0) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * (S + s), ph ^ 1u);
            if (elect_one()) {
                mbar_arrive_expect_tx(bars + 8u * s, box);
                const int row = (int)(((unsigned)it * (unsigned)box_rows + (blockIdx.x * 4 + ring_id) * 1024u) % (unsigned)rows_total);
                tma_load_2d(&tm, rbase + (uint32_t)s * box, bars + 8u * s, 0, row);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    } else {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * s, ph);
            __syncwarp();
            if (elect_one()) mbar_arrive(bars + 8u * (S + s));
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    }
}

// P rings in lockstep driven by ONE producer warp (lane r issues ring r's box) and one consumer warp
__global__ void __launch_bounds__(64, 1) ring_lanes(const __grid_constant__ CUtensorMap tm, int S, int items, int rows_total,
                                                     int box_rows, int P) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t box = (uint32_t)box_rows * 128u;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bars = base + (uint32_t)P * (uint32_t)S * box;   // full[S] (count 1, P boxes of tx), empty[S]
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(bars + 8u * s, 1); mbar_init(bars + 8u * (S + s), 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * (S + s), ph ^ 1u);
            if (lane == 0) mbar_arrive_expect_tx(bars + 8u * s, box * (uint32_t)(P < 0 ? -P : P));
            __syncwarp();
            if (P > 0 && (int)lane < P) {   // P boxes from P lanes
                const int row = (int)(((unsigned)it * (unsigned)box_rows + (blockIdx.x * 4 + lane) * 1024u) % (unsigned)rows_total);
                tma_load_2d(&tm, base + (lane * (uint32_t)S + (uint32_t)s) * box, bars + 8u * s, 0, row);
            }
            if (P < 0 && lane == 0) {       // -P boxes, all from lane 0
                for (int q = 0; q < -P; ++q) {
                    const int row = (int)(((unsigned)it * (unsigned)box_rows + (blockIdx.x * 4 + q) * 1024u) % (unsigned)rows_total);
                    tma_load_2d(&tm, base + ((uint32_t)q * (uint32_t)S + (uint32_t)s) * box, bars + 8u * s, 0, row);
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
            if (elect_one()) mbar_arrive(bars + 8u * (S + s));
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    }
}

// one ring, one box per stage, the issuing lane rotating over NL lanes (it % NL)
__global__ void __launch_bounds__(64, 1) ring_rot(const __grid_constant__ CUtensorMap tm, int S, int items, int rows_total,
                                                   int box_rows, int NL, int spin) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t box = (uint32_t)box_rows * 128u;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bars = base + (uint32_t)S * box;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(bars + 8u * s, 1); mbar_init(bars + 8u * (S + s), 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * (S + s), ph ^ 1u);
            if ((int)lane == it % NL) {
                mbar_arrive_expect_tx(bars + 8u * s, box);
                const int row = (int)(((unsigned)it * (unsigned)box_rows + blockIdx.x * 1024u) % (unsigned)rows_total);
                tma_load_2d(&tm, base + (uint32_t)s * box, bars + 8u * s, 0, row);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    } else {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            if (spin) {   // non-blocking test_wait spin
                uint32_t done = 0;
                while (!done)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bars + 8u * s), "r"(ph) : "memory");
            } else {
                mbar_wait(bars + 8u * s, ph);
            }
            __syncwarp();
            if (elect_one()) mbar_arrive(bars + 8u * (S + s));
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    }
}

// Row-strided source: a [rows][ld] int8 matrix read as {128 B x box_rows} boxes (the GEMM operand
// pattern: K-blocks of 128 B out of rows of C or H bytes), one ring, one box per stage.
__global__ void __launch_bounds__(64, 1) ring_ld(const __grid_constant__ CUtensorMap tm, int S, int items, int rows_total,
                                                  int box_rows, int nkb) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t box = (uint32_t)box_rows * 128u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t bars = base + (uint32_t)S * box;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(bars + 8u * s, 1); mbar_init(bars + 8u * (S + s), 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * (S + s), ph ^ 1u);
            if (elect_one()) {
                mbar_arrive_expect_tx(bars + 8u * s, box);
                const int kb = it % nkb;
                const int row = (int)(((unsigned)(it / nkb) * (unsigned)box_rows + blockIdx.x * 512u) % (unsigned)rows_total);
                tma_load_2d(&tm, base + (uint32_t)s * box, bars + 8u * s, kb * 128, row);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    } else {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * s, ph);
            __syncwarp();
            if (elect_one()) mbar_arrive(bars + 8u * (S + s));
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    }
}

// 3-D boxes: {128 B of K, 128 rows, KB K-blocks} of a [rows][ld] matrix seen as dims {128, rows, ld/128}
// (strides ld, 128): one TMA op lands KB consecutive K-blocks as [KB][128 rows][128 B] (SW128 K-major)
__device__ __forceinline__ void tma_load_3d(const void* tmap, uint32_t dst, uint32_t bar, int32_t c0, int32_t c1, int32_t c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__global__ void __launch_bounds__(64, 1) ring_3d(const __grid_constant__ CUtensorMap tm, int S, int items, int rows_total,
                                                  int KB, int nkb) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t box = 128u * 128u * (uint32_t)KB;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t bars = base + (uint32_t)S * box;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(bars + 8u * s, 1); mbar_init(bars + 8u * (S + s), 1); }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * (S + s), ph ^ 1u);
            if (elect_one()) {
                mbar_arrive_expect_tx(bars + 8u * s, box);
                const int kb = (it * KB) % nkb;
                const int row = (int)(((unsigned)(it * KB / nkb) * 128u + blockIdx.x * 512u) % (unsigned)rows_total);
                tma_load_3d(&tm, base + (uint32_t)s * box, bars + 8u * s, 0, row, kb);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    } else {
        int s = 0; uint32_t ph = 0;
        for (int it = 0; it < items; ++it) {
            mbar_wait(bars + 8u * s, ph);
            __syncwarp();
            if (elect_one()) mbar_arrive(bars + 8u * (S + s));
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1u; }
        }
    }
}

int main() {
    const int rows_total = 8192;   // 1 MB, L2 resident
    int8_t* w; cudaMalloc(&w, (size_t)rows_total * 128);
    cudaMemset(w, 1, (size_t)rows_total * 128);
    void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int box_rows : {64, 128, 256}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {128, (cuuint64_t)rows_total}; cuuint64_t str[1] = {128};
        cuuint32_t bx[2] = {128, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int P : {1, 2, 4}) {
            const int box = box_rows * 128;
            const int S = (196 * 1024) / (P * box) < 8 ? (196 * 1024) / (P * box) : 8;
            if (S < 2) continue;
            const int items = (64 << 20) / box / P / 8;   // 8 MB per ring total... per CTA
            const int smem = P * S * box + 1024 + 16 * S * P + 64;
            for (int grid : {1, 148}) {
                int a0 = S, a1 = items, a2 = rows_total, a3 = box_rows, a4 = P;
                void* args[] = {(void*)&tm, (void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4};
                cudaLaunchKernel((const void*)ring, dim3(grid), dim3(256), args, smem, 0);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaLaunchKernel((const void*)ring, dim3(grid), dim3(256), args, smem, 0);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)items * box * P;
                printf("box %3d rows (%2d KB) rings %d S %d grid %3d: %.1f B/ns per SM, %.0f GB/s total\n", box_rows,
                       box / 1024, P, S, grid, bytes / (ms * 1e6), bytes * grid / (ms * 1e6));
            }
        }
    }
    {
        cudaFuncSetAttribute(ring_ld, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        int8_t* w2; cudaMalloc(&w2, (size_t)16 << 20);
        cudaMemset(w2, 1, (size_t)16 << 20);
        for (int ld : {128, 512, 2048}) for (int box_rows : {128, 256}) {
            const int rows = (8 << 20) / ld;   // 8 MB matrix, L2 resident
            CUtensorMap tm;
            cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)ld};
            cuuint32_t bx[2] = {128, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
            enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w2, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int box = box_rows * 128, S = box_rows == 128 ? 8 : 6, items = (64 << 20) / box / 8;
            const int smem = S * box + 1024 + 16 * S + 64;
            for (int grid : {1, 148}) {
                int a0 = S, a1 = items, a2 = rows, a3 = box_rows, a4 = ld / 128;
                void* args[] = {(void*)&tm, (void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4};
                cudaLaunchKernel((const void*)ring_ld, dim3(grid), dim3(64), args, smem, 0);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaLaunchKernel((const void*)ring_ld, dim3(grid), dim3(64), args, smem, 0);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)items * box;
                printf("STRIDE ld %4d box %3d rows S %d grid %3d: %.1f B/ns per SM, %.0f GB/s total\n", ld, box_rows, S,
                       grid, bytes / (ms * 1e6), bytes * grid / (ms * 1e6));
            }
        }
    }
    {
        cudaFuncSetAttribute(ring_3d, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        int8_t* w3; cudaMalloc(&w3, (size_t)16 << 20);
        cudaMemset(w3, 1, (size_t)16 << 20);
        const int ld = 2048, rows = (8 << 20) / ld, nkb = ld / 128;
        for (int KB : {1, 2, 4}) {
            CUtensorMap tm;
            cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)nkb};
            cuuint64_t str[2] = {(cuuint64_t)ld, 128};
            cuuint32_t bx[3] = {128, 128, (cuuint32_t)KB}; cuuint32_t es[3] = {1, 1, 1};
            CUresult er = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, w3, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (er != CUDA_SUCCESS) { printf("3D encode failed %d (KB %d)\n", (int)er, KB); continue; }
            const int box = 16384 * KB, S = KB == 1 ? 8 : KB == 2 ? 6 : 3, items = (64 << 20) / box / 8;
            const int smem = S * box + 1024 + 16 * S + 64;
            for (int grid : {1, 148}) {
                int a0 = S, a1 = items, a2 = rows, a3 = KB, a4 = nkb;
                void* args[] = {(void*)&tm, (void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4};
                cudaLaunchKernel((const void*)ring_3d, dim3(grid), dim3(64), args, smem, 0);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf("error 3d\n"); return 1; }
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaLaunchKernel((const void*)ring_3d, dim3(grid), dim3(64), args, smem, 0);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)items * box;
                printf("BOX3D 128 rows x %d K-blocks (%d KB) S %d grid %3d: %.1f B/ns per SM, %.0f GB/s total\n", KB, box / 1024,
                       S, grid, bytes / (ms * 1e6), bytes * grid / (ms * 1e6));
            }
        }
    }
    cudaFuncSetAttribute(ring_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    {
        CUtensorMap tm;
        cuuint64_t dims[2] = {128, (cuuint64_t)rows_total}; cuuint64_t str[1] = {128};
        cuuint32_t bx[2] = {128, 128}; cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int spin : {0, 1}) for (int NL : {1}) for (int S : {4, 8}) {
            const int box = 128 * 128, items = (64 << 20) / box / 8;
            const int smem = S * box + 1024 + 16 * S + 64;
            for (int grid : {1, 148}) {
                int a0 = S, a1 = items, a2 = rows_total, a3 = 128, a4 = NL, a5 = spin;
                void* args[] = {(void*)&tm, (void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4, (void*)&a5};
                cudaLaunchKernel((const void*)ring_rot, dim3(grid), dim3(64), args, smem, 0);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaLaunchKernel((const void*)ring_rot, dim3(grid), dim3(64), args, smem, 0);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)items * box;
                printf("ROT spin %d 16KB boxes, issuing lanes %d S %2d grid %3d: %.1f B/ns per SM, %.0f GB/s total\n", spin, NL, S, grid,
                       bytes / (ms * 1e6), bytes * grid / (ms * 1e6));
            }
        }
    }
    cudaFuncSetAttribute(ring_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int box_rows : {128, 256}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {128, (cuuint64_t)rows_total}; cuuint64_t str[1] = {128};
        cuuint32_t bx[2] = {128, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int PP : {1, 2, 3, -2, -3}) {
            const int P = PP < 0 ? -PP : PP;
            const int box = box_rows * 128;
            const int S = (196 * 1024) / (P * box) < 8 ? (196 * 1024) / (P * box) : 8;
            if (S < 2) continue;
            const int items = (64 << 20) / box / P / 8;
            const int smem = P * S * box + 1024 + 16 * S + 64;
            for (int grid : {1, 148}) {
                int a0 = S, a1 = items, a2 = rows_total, a3 = box_rows, a4 = PP;
                void* args[] = {(void*)&tm, (void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4};
                cudaLaunchKernel((const void*)ring_lanes, dim3(grid), dim3(64), args, smem, 0);
                if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaLaunchKernel((const void*)ring_lanes, dim3(grid), dim3(64), args, smem, 0);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                const double bytes = (double)items * box * P;
                printf("LANES box %3d rows (%2d KB) boxes/stage %d (one lane: %d) S %d grid %3d: %.1f B/ns per SM, %.0f GB/s total\n", box_rows,
                       box / 1024, P, PP < 0, S, grid, bytes / (ms * 1e6), bytes * grid / (ms * 1e6));
            }
        }
    }
    return 0;
}
