// common.cuh — shared device/host helpers of libprnu.so (sm_100a).
// Product code: never includes or links anything under oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <atomic>
#include <string>
#include <algorithm>

#include "../../include/prnu.h"

// Device-side bounds checks, compiled in only for PRNU_DEBUG builds
// (PRNU_DEBUG=1 python paper_1909_04573_b200/_build.py --force).
#ifdef PRNU_DEBUG
#include <cstdio>
#define PRNU_DCHECK(c)                                                                          \
    do {                                                                                        \
        if (!(c)) {                                                                             \
            printf("PRNU_DCHECK %s:%d %s blk(%d,%d,%d) thr %d\n", __FILE__, __LINE__, #c,        \
                   blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);                            \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define PRNU_DCHECK(c) \
    do {               \
    } while (0)
#endif

// Race stress (debug builds: PRNU_NVCC_DEFS=PRNU_RACE_STRESS): at the phase boundaries
// of the shared-memory kernels a pseudo-random quarter of the warps sleeps up to ~4 us,
// reshuffling the interleaving of warps; a missing barrier or mbarrier wait then changes
// the results, which tools/gpu_race_stress.sh compares bit for bit with the release
// build (compute-sanitizer is not available on the GPU pool).
#ifdef PRNU_RACE_STRESS
__device__ __forceinline__ void prnu_race_stress(uint32_t tag) {
    uint32_t h = (blockIdx.x * 73856093u) ^ (blockIdx.y * 19349663u) ^ (blockIdx.z * 83492791u) ^
                 ((threadIdx.x >> 5) * 2654435761u) ^ (tag * 40503u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    if ((h & 3u) == 0u) __nanosleep(64u + (h >> 20) % 4096u);
}
#define PRNU_STRESS(tag) prnu_race_stress(tag)
#else
#define PRNU_STRESS(tag) \
    do {                 \
    } while (0)
#endif

namespace prnu {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void count_launch(int n = 1);
int check_launch(const char* what);   // PRNU_OK or PRNU_CUDA_ERROR (cudaGetLastError)

// Optional per-kernel CUDA-event timing (prnu_profile_begin/end): when
// enabled, a KTimer records an event pair around one launch on its stream.
struct KTimer {
    int slot;
    cudaStream_t st;
    KTimer(const char* name, cudaStream_t s);
    ~KTimer();
};

bool profiling_active();

// Per-device "done" flags (bit d = device d), for one-time per-device setup such
// as cudaFuncSetAttribute, which applies to the current device only.
struct DeviceFlags {
    std::atomic<uint64_t> bits{0};
};
// Raise fn's dynamic shared-memory limit to `bytes` on the current device, once
// per device (a failed call is reported and retried on the next launch).
int set_smem_attr(const void* fn, size_t bytes, DeviceFlags& done);
// Streaming multiprocessors of the current device (cudaDevAttrMultiProcessorCount, cached per device).
int device_sm_count();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- packed fp32 (f32x2)
// Two fp32 lanes per instruction (FADD2 / FMUL2 / FFMA2): half the issue slots of
// the scalar forms at the same lane throughput (broadcast-scalar forms: ffma2 /
// fmul2s below).
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&a);
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&a);
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&a);
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {   // a * b + c
    unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&a);
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long rc = *reinterpret_cast<const unsigned long long*>(&c);
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(ra), "l"(rb), "l"(rc));
    return *reinterpret_cast<float2*>(&r);
}

// 8 consecutive floats with one 256-bit store (STG.E.256, sm_100; p 32-byte aligned).
// The L1 data pipe spends one wavefront per 32-byte sector a store instruction touches:
// two STG.128 of a lane's 8 outputs touch its sector twice, one STG.256 once.
__device__ __forceinline__ void st_global_v8(float* p, const float (&v)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// 4 consecutive doubles with one 256-bit load / store (p 32-byte aligned): whole sectors.
__device__ __forceinline__ void ld_global_v4d(const double* p, double (&v)[4]) {
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st_global_v4d(double* p, const double (&v)[4]) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}

// ---------------------------------------------------------------- reductions
// Deterministic warp-shuffle sums (the fingerprint / NCC / PCE / WDFT block
// reductions): an xor butterfly inside each warp (lane i and lane i^o add the
// same two operands, so every lane ends with the same bits), then every thread
// adds the NW warp totals in warp order.  A fixed shape => bit-reproducible.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// Sums N values per thread across the block (NW = blockDim.x / 32 warps);
// sh holds N * NW doubles.  Result in v[] on every thread.
template <int N, int NW = 8>
__device__ __forceinline__ void block_sum(double (&v)[N], double* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < N; ++j) v[j] = warp_sum(v[j]);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < N; ++j) sh[j * NW + w] = v[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < N; ++j) {
        double t = sh[j * NW];
#pragma unroll
        for (int k = 1; k < NW; ++k) t += sh[j * NW + k];
        v[j] = t;
    }
    __syncthreads();   // sh may be reused at once
}

// ---------------------------------------------------------------- wavelet
// 8-tap Daubechies (4 vanishing moments) in minimum-phase order (R-2, R-5):
// analysis   a[c] = sum_i H_[i] x[2c-6+i],   d[c] = sum_i G_[i] x[2c-6+i]
// synthesis  x[2s+e] = sum_{m=0..3} a[s+m] H_[6-2m+e] + d[s+m] G_[6-2m+e]
// with G_[i] = (-1)^i H_[7-i].  (Equivalent to the analysis/synthesis pair of
// DESIGN.md §3 R-5; perfect reconstruction is tested on the GPU.)
#define PRNU_H0 0.2303778133088965f
#define PRNU_H1 0.7148465705529157f
#define PRNU_H2 0.6308807679298589f
#define PRNU_H3 (-0.027983769416859854f)
#define PRNU_H4 (-0.18703481171909309f)
#define PRNU_H5 0.030841381835560764f
#define PRNU_H6 0.0328830116668852f
#define PRNU_H7 (-0.010597401785069032f)

__host__ __device__ __forceinline__ constexpr float wl_h(int i) {
    return i == 0 ? PRNU_H0 : i == 1 ? PRNU_H1 : i == 2 ? PRNU_H2 : i == 3 ? PRNU_H3
         : i == 4 ? PRNU_H4 : i == 5 ? PRNU_H5 : i == 6 ? PRNU_H6 : PRNU_H7;
}
__host__ __device__ __forceinline__ constexpr float wl_g(int i) {
    return (i & 1) ? -wl_h(7 - i) : wl_h(7 - i);
}

// Packed fp32 FMA (sm_100a FFMA2): lane-wise RN fma, bit-identical to two fmaf.
// The scalar first operand is broadcast inside the asm (mov.b64 {a, a}), which
// ptxas folds into the instruction's .F32 broadcast operand: no MOVs.
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long rc = *reinterpret_cast<const unsigned long long*>(&c);
    unsigned long long r;
    asm("{.reg .b64 aa; mov.b64 aa, {%1, %1}; fma.rn.f32x2 %0, aa, %2, %3;}" : "=l"(r) : "f"(a), "l"(rb), "l"(rc));
    return *reinterpret_cast<float2*>(&r);
}
// Packed product of a broadcast scalar and a pair (FMUL2), == ffma2(a, b, 0).
__device__ __forceinline__ float2 fmul2s(float a, float2 b) {
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long r;
    asm("{.reg .b64 aa; mov.b64 aa, {%1, %1}; mul.rn.f32x2 %0, aa, %2;}" : "=l"(r) : "f"(a), "l"(rb));
    return *reinterpret_cast<float2*>(&r);
}

// subband length of the expansive symmetric DWT: floor((N + 7) / 2)
__host__ __device__ __forceinline__ int sub_len(int N) { return (N + 7) >> 1; }

// half-sample symmetric index map e_N (R-4), valid for any integer i.
__host__ __device__ __forceinline__ int mirror(int i, int N) {
    int P2 = 2 * N;
    int r = i % P2;
    if (r < 0) r += P2;
    return r < N ? r : P2 - 1 - r;
}

constexpr int kMaxLevels = 6;
constexpr int kHalo = 4;  // max window radius (9x9)

// Geometry of one decomposition: level 0 is the input plane.
struct Pyramid {
    int levels;
    int nH[kMaxLevels + 1], nW[kMaxLevels + 1];
    int pitch[kMaxLevels + 1];        // floats per row of each subband plane (level >= 1)
    size_t plane[kMaxLevels + 1];     // floats per subband plane (nH * pitch)
};

Pyramid make_pyramid(int H, int W, int levels);

// SDA frames from exact group sums (a1, R-11): S = RN(sum / d) with sum an integer
// < 2^24.  d and r = RN(1/d) as fp32; d = 1 for plain frames.
struct SdaDiv {
    float d = 1.0f, r = 1.0f;
};
// u16 in the low (hi = 0) or high (hi = 1) half of w -> its exact fp32 value
// (2^23 + u as a bit pattern, minus 2^23).
__device__ __forceinline__ float u16_to_f32(uint32_t w, int hi) {
    return __fadd_rn(__uint_as_float(__byte_perm(w, 0x4B000000u, hi ? 0x7632u : 0x7610u)), -8388608.0f);
}
// SDA pairs (depth d = 2, R-11): the two u8 frames of a group staged together by one
// TMA box of depth 2 ([frame][row][x] in shared memory), S = (b0 + b1) / 2 formed where
// it is consumed (exact in fp32: no sum pass, no u16 plane).  A tag type: 2 bytes per
// pixel, like the u16 sums it replaces at d = 2.
struct u8pair {
    uint8_t b[2];
};
// (2^22 + b/2) as a float bit pattern from byte b (ulp 0.5 at 2^22): the half of a u8
// exactly, so S = ((h(b0) - 2^22) + h(b1)) - 2^22 = (b0 + b1) / 2 with two exact adds.
__device__ __forceinline__ float u8_half_bias(uint32_t w, int byte) {
    return __uint_as_float(__byte_perm(w, 0x4A800000u, 0x7640u | (uint32_t)byte));
}
// RN_fp32(s / d): reciprocal product plus one FMA correction.  Equal to the correctly
// rounded quotient for every integer s <= 255 d and 2 <= d <= 257 (and the config
// depths 300..3600): exhaustive check in tools/sda_div_check.py / tests/test_capi_cpu.py.
__device__ __forceinline__ float sda_div(float s, float d, float r) {
    const float q0 = __fmul_rn(s, r);
    const float rem = __fmaf_rn(-q0, d, s);
    return __fmaf_rn(rem, r, q0);
}

// Shrink constants passed by value to kernels.
struct ShrinkParams {
    float sigma0_sq;
    int wmask;            // bit k set <=> window (2k+3) enabled, k = 0..3
};

int validate_params(const prnu_denoise_params* p, int H, int W, ShrinkParams* sp);

// shrink.cu: the streaming shrink of detail planes held in HBM (variants, WDFT)
int launch_shrink_strip(const float* const src[3], float* const dst[3], long long bstride, int pitch, int nH, int nW,
                        const ShrinkParams& sp, int nb, cudaStream_t st, int nsub = 3, const float* s0_dev = nullptr);


// analysis.cu: column-streaming analysis (lifting) + shrink of one level
int launch_analysis_lift_u8(const uint8_t* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                            float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                            const ShrinkParams& sp, int nb, cudaStream_t st);
int launch_analysis_lift_u16(const uint16_t* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                             float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                             const ShrinkParams& sp, const SdaDiv& div, int nb, cudaStream_t st);
// prnu_check_results (mle.cu): synchronous status of results already written on st
int check_results(int kind, const double* v, long long n, cudaStream_t st);
// SDA pairs (d = 2): groups of two u8 frames (frame_stride apart; group b = frames 2b, 2b+1)
int launch_analysis_lift_pair(const uint8_t* in, long long frame_stride, int in_pitch, int NH, int NW, float* ll,
                              float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                              const ShrinkParams& sp, int nb, cudaStream_t st);
int launch_analysis_lift_f32(const float* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                             float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                             const ShrinkParams& sp, int nb, cudaStream_t st);

}  // namespace prnu
