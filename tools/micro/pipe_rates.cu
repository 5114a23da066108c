// Microbenchmark: issue/throughput of fp32 instruction forms on sm_100a.
// 8 independent accumulator chains per thread, N iterations, full occupancy.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ float2 c_pair[2] = {{1.0001f, 0.9999f}, {0.5f, 0.25f}};
__constant__ float c_s[2] = {1.0001f, 0.9999f};

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
                if (MODE == 0) a[i] = fmaf(a[i], y, yy.y);         // FFMA r,r,r
                if (MODE == 1) a[i] = fmaf(a[i], 1.0001f, 0.5f);                          // FFMA imm
                if (MODE == 2) a[i] = fmaf(a[i], c_s[0], c_s[1]);                         // FFMA const
                if (MODE == 3) { unsigned long long r_; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r_) : "l"(u64(p[i])), "l"(u64(yy)), "l"(u64(p[(i+1)&7]))); p[i] = f2(r_); }
                if (MODE == 4) { unsigned long long r_; asm("{.reg .b64 aa; mov.b64 aa, {%1, %1}; fma.rn.f32x2 %0, aa, %2, %3;}" : "=l"(r_) : "f"(a[i]), "l"(u64(c_pair[0])), "l"(u64(p[i]))); p[i] = f2(r_); }
                if (MODE == 5) a[i] = a[i] + y;                                           // FADD r,r
                if (MODE == 6) { unsigned long long r_; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r_) : "l"(u64(p[i])), "l"(u64(yy))); p[i] = f2(r_); }
                if (MODE == 7) a[i] = fminf(a[i] + 0.f, (i & 1) ? y : yy.y);                              // FMNMX
                if (MODE == 8) a[i] = a[i] * y;                                           // FMUL r,r
                if (MODE == 9) { unsigned long long r_; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r_) : "l"(u64(p[i])), "l"(u64(yy))); p[i] = f2(r_); }
                if (MODE == 10) a[i] = a[i] + 1.5f;                                       // FADD imm
                if (MODE == 11) { a[i] = a[i] + y; p[i].x = p[i].x * y; }                 // FADD + FMUL mix
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + p[i].x + p[i].y;
    if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int ops_per_inner) {
    float* out;
    cudaMalloc(&out, 4096);
    const int blocks = 148 * 8, threads = 256, n = 2000;
    k<MODE><<<blocks, threads>>>(out, 10, 1.f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, n, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_inst = (double)blocks * threads / 32 * n * 64 * ops_per_inner;
    const double cyc = ms * 1e-3 * clk * 1e3;   // at the nominal clock
    printf("%-28s %8.3f ms  warp-inst/cycle/SM %.3f  (per SMSP %.3f)\n", name, ms, warp_inst / cyc / 148, warp_inst / cyc / 148 / 4);
    cudaFree(out);
}
int main() {
    run<0>("FFMA r,r,r", 1);
    run<1>("FFMA r,imm,imm", 1);
    run<2>("FFMA r,c,c", 1);
    run<3>("FFMA2 r,r,r", 1);
    run<4>("FFMA2 bcast,c,r", 1);
    run<5>("FADD r,r", 1);
    run<6>("FADD2 r,r", 1);
    run<7>("FMNMX+FADD (2 inst)", 2);
    run<8>("FMUL r,r", 1);
    run<9>("FMUL2 r,r", 1);
    run<10>("FADD r,imm", 1);
    run<11>("FADD+FMUL (2 inst)", 2);
    return 0;
}
