// Microbenchmark (sm_100a): issue rate of FFMA2 operand forms that a lifted DWT
// would use — immediate broadcast coefficient vs register / constant-bank pair —
// against scalar FFMA (reg and imm) and FADD2.  8 independent chains per thread,
// full occupancy; prints warp-instructions per clock per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ float2 c_pair[4] = {{0.3222f, 0.3222f}, {-1.117f, -1.117f}, {0.54f, 0.54f}, {1.6889f, 1.6889f}};
__device__ __forceinline__ unsigned long long u64(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 f2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
template <int MODE>
__global__ void k(float* out, int n, float x) {
    float a[8];
    float2 p[8];
    for (int i = 0; i < 8; ++i) { a[i] = x + threadIdx.x + i; p[i] = make_float2(a[i], a[i] + 1.f); }
    const float y = x * 0.5f + 1e-3f * threadIdx.x;
    const float2 yy = make_float2(y, y * 1.1f);
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                unsigned long long q;
                if (MODE == 0) { asm("{.reg .b64 kk; mov.b64 kk, {%1,%1}; fma.rn.f32x2 %0, kk, %2, %3;}" : "=l"(q) : "f"(0.99991f), "l"(u64(p[i])), "l"(u64(p[(i + 1) & 7]))); p[i] = f2(q); }
                if (MODE == 1) { asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(q) : "l"(u64(c_pair[i & 3])), "l"(u64(p[i])), "l"(u64(p[(i + 1) & 7]))); p[i] = f2(q); }
                if (MODE == 2) { asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(q) : "l"(u64(yy)), "l"(u64(p[i])), "l"(u64(p[(i + 1) & 7]))); p[i] = f2(q); }
                if (MODE == 3) a[i] = fmaf(a[i], y, a[(i + 1) & 7]);
                if (MODE == 4) a[i] = fmaf(a[i], 0.99991f, a[(i + 1) & 7]);
                if (MODE == 5) { asm("add.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(u64(p[i])), "l"(u64(p[(i + 1) & 7]))); p[i] = f2(q); }
                if (MODE == 6) { asm("{.reg .b64 kk; mov.b64 kk, {%1,%1}; mul.rn.f32x2 %0, kk, %2;}" : "=l"(q) : "f"(0.99991f), "l"(u64(p[i]))); p[i] = f2(q); }
                if (MODE == 7) a[i] = a[i] + a[(i + 1) & 7];
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + p[i].x + p[i].y;
    if (s == 12345.678f) out[threadIdx.x] = s;
}
template <int MODE>
void run(const char* name) {
    float* out;
    cudaMalloc(&out, 4096);
    const int blocks = 148 * 8, threads = 256, n = 4000;
    k<MODE><<<blocks, threads>>>(out, 10, 1.f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, n, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_inst = (double)blocks * threads / 32 * n * 64;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-34s %8.3f ms  warp-inst/clk/SMSP %.3f (at the %d MHz attribute clock)\n", name, ms, warp_inst / cyc / 148 / 4, clk / 1000);
    cudaFree(out);
}
int main() {
    run<0>("FFMA2 imm broadcast");
    run<1>("FFMA2 const-bank pair");
    run<2>("FFMA2 register pair");
    run<3>("FFMA reg,reg,reg");
    run<4>("FFMA reg,imm,reg");
    run<5>("FADD2 reg,reg");
    run<6>("FMUL2 imm broadcast");
    run<7>("FADD reg,reg");
    return 0;
}
