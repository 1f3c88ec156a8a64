// Probe: semantics of cvt.pack.sat.s8.s32.b32 and cvt.rni.sat.s8/s16.f32 on sm_100a.
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out, int* o2) {
    int a = 0x11, b = 0x22, c = 0x7766;
    uint32_t d;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    out[0] = d;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(300), "r"(-300), "r"(0));
    out[1] = d;
    int q;
    float vs[6] = {0.5f, 1.5f, 2.5f, -2.5f, 1e10f, -1e10f};
    for (int i = 0; i < 6; ++i) { asm("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(q) : "f"(vs[i])); o2[i] = q; }
    for (int i = 0; i < 6; ++i) { asm("cvt.rni.sat.s16.f32 %0, %1;" : "=r"(q) : "f"(vs[i])); o2[6 + i] = q; }
    asm("cvt.sat.s8.s32 %0, %1;" : "=r"(q) : "r"(200)); o2[12] = q;
    asm("cvt.sat.s8.s32 %0, %1;" : "=r"(q) : "r"(-200)); o2[13] = q;
}
int main() {
    uint32_t* d; int* e;
    cudaMallocManaged(&d, 8); cudaMallocManaged(&e, 64);
    k<<<1, 1>>>(d, e);
    cudaDeviceSynchronize();
    printf("pack(0x11,0x22,0x7766)=%08x pack(300,-300,0)=%08x\n", d[0], d[1]);
    for (int i = 0; i < 14; ++i) printf("%d ", e[i]);
    printf("\n");
}
