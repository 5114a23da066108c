// strip.cu — column-streaming DWT analysis + local-variance shrink (a2 + a3).
//
// One DWT level (rows then columns, R-6) with the local-variance MAP/Wiener
// shrink of the three detail subbands (R-7) fused, like
// k_analysis_shrink in wavelet.cu, but organised so that the vertical
// direction never leaves registers:
//
//   * A CTA of 128 threads owns a vertical STRIP of the subband: O <= 120
//     output coefficient columns plus a 4-column halo on each side (the 9x9
//     windows), one thread per region column, and walks down a SEGMENT of SH
//     output rows in blocks of 8 coefficient rows.
//   * Per block, 16 new input rows arrive in shared memory (TMA box loads,
//     double-buffered one block ahead; border blocks whose rows mirror are
//     loaded by the threads).  A cooperative row pass (along x) writes lo/hi
//     rows to shared memory.
//   * Each thread then runs the column pass (along y) of ITS column over a
//     22-row register window (6 rows carried from the previous block), so
//     the coefficient rows of a column come out in order; the squares c^2 of
//     the three detail subbands stay in a 16-row register ring from which the
//     vertical window sums (3, 5, 7, 9 rows, nested) of 8 output rows are
//     formed without any shared-memory traffic or vertical halo recompute.
//   * The vertical sums (float4 per coefficient) and the coefficients go
//     through shared memory once for the horizontal sums (sliding, 8 outputs
//     per thread), the Wiener factor and the store of c - F(c) (R-10).
//
// Subband borders (R-4): region columns / rows outside the subband are
// copies of the mirrored ones (the row pass computes mirrored columns; the
// register ring copies mirrored rows), exactly as the oracle's e_N windows.
// Arithmetic per coefficient is the same sequence of fp32 operations as
// k_analysis_shrink (FFMA2 taps in the same order, nested sums in the same
// order), so both kernels produce the same bits.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tma.cuh"

namespace prnu {

// Phase-time probes (build with -DPRNU_STRIP_PROFILE; read with prnu_debug_strip_profile):
// per warp, clock64 cycles spent in each phase of a block, summed over warps and CTAs.
#ifdef PRNU_STRIP_PROFILE
__device__ unsigned long long g_strip_prof[16];
#define SPROBE(i)                                         \
    do {                                                  \
        const long long now_ = clock64();                 \
        pacc[i] += (unsigned long long)(now_ - plast);    \
        plast = now_;                                     \
    } while (0)
#else
#define SPROBE(i) \
    do {          \
    } while (0)
#endif

constexpr int SR_NT = 128;                  // threads per CTA == region columns
constexpr int SR_RW = 128;                  // region width (O + 8 <= 128)
constexpr int SR_BK = 8;                    // coefficient rows per block
constexpr int SR_IR = 2 * SR_BK;            // input rows per block
// Filter tap pairs (H_[i], G_[i]) and window scales in constant memory: FFMA2 /
// FMUL2 read them as uniform operands (no per-use MOVs of immediate pairs).
__constant__ float2 c_st_hg[8] = {{PRNU_H0, PRNU_H7}, {PRNU_H1, -PRNU_H6}, {PRNU_H2, PRNU_H5}, {PRNU_H3, -PRNU_H4},
                                  {PRNU_H4, PRNU_H3}, {PRNU_H5, -PRNU_H2}, {PRNU_H6, PRNU_H1}, {PRNU_H7, -PRNU_H0}};
__constant__ float2 c_st_ws[2] = {{1.0f / 9.0f, 1.0f / 25.0f}, {1.0f / 49.0f, 1.0f / 81.0f}};

constexpr int SR_RBP = 132;                 // row-buffer pitch (== 4 mod 32: conflict-free STS.128, lanes over rows)
constexpr int SR_RB_FLOATS = 2 * SR_IR * SR_RBP;
// Per input type: strip width, V/c plane pitches, staging buffers.  u8: 3 staging
// buffers (TMA two blocks ahead), 112 output columns; fp32 (levels >= 2, SDA
// frames): a single staging buffer and 104 output columns, so that both variants
// fit 3 CTAs/SM (<= 75 KB shared memory).
template <typename T>
struct StripCfg;
#ifndef PRNU_U8_OMAX   // build-time A/B knobs of the u8 configuration (defaults: measured best)
#define PRNU_U8_OMAX 112
#define PRNU_U8_P2 121
#define PRNU_U8_CP 124
#define PRNU_U8_NSTG 3
#define PRNU_U8_MINB 3
#endif
template <>
struct StripCfg<uint8_t> {
    static constexpr int OMAX = PRNU_U8_OMAX;   // max output columns per strip
    static constexpr int P2 = PRNU_U8_P2;       // float2 pitch of the vertical-sum planes (== 1 mod 8: conflict-free LDS.64)
    static constexpr int CP = PRNU_U8_CP;       // float pitch of the coefficient planes (== 28 mod 32: conflict-free LDS.128)
    static constexpr int NSTG = PRNU_U8_NSTG;
    static constexpr int MINB = PRNU_U8_MINB;   // CTAs per SM the register budget targets
};
template <>
struct StripCfg<float> {
    static constexpr int OMAX = 104;
    static constexpr int P2 = 113;
    static constexpr int CP = 116;     // == 20 mod 32
    static constexpr int NSTG = 1;
    static constexpr int MINB = 3;
};
// V/c buffer of one subband: (v3, v5) plane [8][P2] float2, (v7, v9) plane, c plane [8][CP]
template <typename T>
__host__ __device__ constexpr int sr_vc_floats() { return 2 * SR_BK * StripCfg<T>::P2 * 2 + SR_BK * StripCfg<T>::CP; }
template <typename T>
__host__ __device__ constexpr int sr_a_floats() { return SR_RB_FLOATS > sr_vc_floats<T>() ? SR_RB_FLOATS : sr_vc_floats<T>(); }
static_assert(StripCfg<uint8_t>::OMAX + 8 <= StripCfg<uint8_t>::P2 && StripCfg<uint8_t>::OMAX + 8 <= StripCfg<uint8_t>::CP &&
                  StripCfg<float>::OMAX + 8 <= StripCfg<float>::P2 && StripCfg<float>::OMAX + 8 <= StripCfg<float>::CP,
              "V/c planes hold every region column");
#ifndef PRNU_H_UNROLL
#define PRNU_H_UNROLL 3
#endif
constexpr int kStripHUnroll = PRNU_H_UNROLL;   // subband items of the H pass unrolled (A/B knob)                  // staging buffers: TMA two blocks ahead
static_assert(8 * 16 <= SR_RBP, "row-buffer columns of the 16 row-pass groups");

// Staging: two TMA boxes per block, box 0 = logical columns [0, BOXW), box 1 =
// [128, 128 + BOXW), each [16 rows][BOXW] dense.  A row-pass group g reads
// logical columns [16g, 16g + 24) (u8) / [16g + 2, 16g + 24) (fp32): box 0
// for g < 8, box 1 for g >= 8.  Logical column x is input column xs + x,
// xs = 2 cx0 - 16 (16-byte aligned for u8: cx0 is a multiple of 8).
template <typename T>
struct StripStage;
template <>
struct StripStage<uint8_t> {
    static constexpr int BOXW = 144;   // bytes (36 words == 4 mod 32: conflict-free, lanes over rows)
    static constexpr int LOGW = 272;
};
template <>
struct StripStage<float> {
#ifndef PRNU_F32_BOXW
#define PRNU_F32_BOXW 140
#endif
    // floats (a 16-B multiple); 140 == 12 mod 32 words: the row pass's LDS.128 over 8 rows
    // is conflict-free (136 == 8 mod 32 was 2-way)
    static constexpr int BOXW = PRNU_F32_BOXW;
    static constexpr int LOGW = 128 + PRNU_F32_BOXW;
};

template <typename T>
__host__ __device__ constexpr int strip_stage_elems() { return 2 * SR_IR * StripStage<T>::BOXW; }   // one buffer

template <typename T>
constexpr size_t strip_smem_bytes() {
    return StripCfg<T>::NSTG * strip_stage_elems<T>() * sizeof(T) + sizeof(float) * (sr_a_floats<T>() + 2 * sr_vc_floats<T>()) +
           32;
}

struct StripArgs {
    const void* in;
    long long in_bstride;   // elements between frames
    int in_pitch;           // elements per row
    int NH, NW;             // input plane
    float* ll;              // approximation out (nullable: coarsest level)
    float* d0;              // da = lo_y(hi_x)
    float* d1;              // ad = hi_y(lo_x)
    float* d2;              // dd = hi_y(hi_x)
    long long out_bstride;
    int out_pitch;
    int nH, nW;             // subband
    ShrinkParams sp;
    int O;                  // output columns per strip (multiple of 8, <= SR_OMAX)
    int SH;                 // output rows per segment (multiple of 8)
    int use_tma;
};


template <typename T>
__device__ __forceinline__ float stg_at(const T* s, int r, int x) {
    constexpr int BW = StripStage<T>::BOXW;
    PRNU_DCHECK(r >= 0 && r < SR_IR && x >= 0 && x < StripStage<T>::LOGW);
    return x < BW ? (float)s[r * BW + x] : (float)s[SR_IR * BW + r * BW + x - 128];
}

// 22 consecutive staged values of group g, row r: v[i] = logical column 16g + 2 + i.
__device__ __forceinline__ void stg_row22(const uint8_t* s, int r, int g, float (&v)[24]) {
    constexpr int BW = StripStage<uint8_t>::BOXW;
    const uint8_t* src = s + (g < 8 ? r * BW + 16 * g : SR_IR * BW + r * BW + 16 * g - 128);
    const uint4 w0 = *reinterpret_cast<const uint4*>(src);
    const uint2 w1 = *reinterpret_cast<const uint2*>(src + 16);   // (a 16-byte load here: +0.3%)
    const uint32_t w[6] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y};
#pragma unroll
    for (int k = 0; k < 22; k += 2) {   // exact byte -> float (2^23 trick), two at a time (FADD2)
        const float2 p = make_float2(
            __uint_as_float(__byte_perm(w[(k + 2) >> 2], 0x4B000000u, 0x7540u | (uint32_t)((k + 2) & 3))),
            __uint_as_float(__byte_perm(w[(k + 3) >> 2], 0x4B000000u, 0x7540u | (uint32_t)((k + 3) & 3))));
        unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&p), r;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(0xCB000000CB000000ull));   // - (2^23, 2^23)
        const float2 q = *reinterpret_cast<const float2*>(&r);
        v[k] = q.x;
        v[k + 1] = q.y;
    }
    v[22] = v[23] = 0.f;
}
__device__ __forceinline__ void stg_row22(const float* s, int r, int g, float (&v)[24]) {
    constexpr int BW = StripStage<float>::BOXW;
    const float* src = s + (g < 8 ? r * BW + 16 * g : SR_IR * BW + r * BW + 16 * g - 128) + 2;
    const float2 a = *reinterpret_cast<const float2*>(src);
    v[0] = a.x;
    v[1] = a.y;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const float4 b = *reinterpret_cast<const float4*>(src + 2 + 4 * k);
        v[2 + 4 * k] = b.x;
        v[3 + 4 * k] = b.y;
        v[4 + 4 * k] = b.z;
        v[5 + 4 * k] = b.w;
    }
    v[22] = v[23] = 0.f;
}

// Group 0 of the first strip (xs = -16, plane at least 16 columns wide): logical
// columns x < 16 are the mirrored input columns 15 - (x - 16) (R-4), i.e. logical
// 31 - x, so v[k] (column 2 + k) = S[29 - k] for k < 14 and S[k + 2] otherwise: all
// from S[16 .. 29], read as one 16-byte chunk — no fix-up of the staged row needed.
__device__ __forceinline__ void stg_row22_left(const uint8_t* s, int r, float (&v)[24]) {
    const uint4 w = *reinterpret_cast<const uint4*>(s + r * StripStage<uint8_t>::BOXW + 16);
    const uint32_t b[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 22; k += 2) {
        const int i0 = k < 14 ? 13 - k : k - 14, i1 = k + 1 < 14 ? 12 - k : k - 13;   // byte index in S[16 ..]
        const float2 p = make_float2(__uint_as_float(__byte_perm(b[i0 >> 2], 0x4B000000u, 0x7540u | (uint32_t)(i0 & 3))),
                                     __uint_as_float(__byte_perm(b[i1 >> 2], 0x4B000000u, 0x7540u | (uint32_t)(i1 & 3))));
        unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&p), rr;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(ra), "l"(0xCB000000CB000000ull));
        const float2 q = *reinterpret_cast<const float2*>(&rr);
        v[k] = q.x;
        v[k + 1] = q.y;
    }
    v[22] = v[23] = 0.f;
}
__device__ __forceinline__ void stg_row22_left(const float* s, int r, float (&v)[24]) {
    const float4* src = reinterpret_cast<const float4*>(s + r * StripStage<float>::BOXW + 16);
    const float4 a0 = src[0], a1 = src[1], a2 = src[2], a3 = src[3];
    const float S[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
#pragma unroll
    for (int k = 0; k < 22; ++k) v[k] = k < 14 ? S[13 - k] : S[k - 14];
    v[22] = v[23] = 0.f;
}

__device__ __forceinline__ float pick16(const float (&q)[16][3], int sl, int s) {
    float r = q[0][s];
#pragma unroll
    for (int i = 1; i < 16; ++i) r = (sl == i) ? q[i][s] : r;
    return r;
}

__device__ __forceinline__ void stg_put(uint8_t* s, int r, int x, float v) {
    constexpr int BW = StripStage<uint8_t>::BOXW;
    const uint8_t u = (uint8_t)v;
    if (x < BW) s[r * BW + x] = u;
    if (x >= 128) s[SR_IR * BW + r * BW + x - 128] = u;
}
__device__ __forceinline__ void stg_put(float* s, int r, int x, float v) {
    constexpr int BW = StripStage<float>::BOXW;
    if (x < BW) s[r * BW + x] = v;
    if (x >= 128) s[SR_IR * BW + r * BW + x - 128] = v;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&a);
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&b);
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&r);
}

// Edge fix-up slots per thread: out-of-plane logical columns of a staged row
// (left: x < -xs, right: input columns NW .. NW+23) receive their mirrored
// in-plane values (R-4), so every row-pass group reads plain staged rows.
constexpr int SR_FIX = 5;   // ceil(16 rows * 40 columns / 128 threads)

template <typename T, int MINB, bool ALL4>
__global__ void __launch_bounds__(SR_NT, MINB) k_analysis_strip(const __grid_constant__ CUtensorMap map, StripArgs a) {
    constexpr int BW = StripStage<T>::BOXW;
    constexpr int LOGW = StripStage<T>::LOGW;
    constexpr int STG = strip_stage_elems<T>();
    constexpr int SR_NSTG = StripCfg<T>::NSTG, SR_P2 = StripCfg<T>::P2, SR_CP = StripCfg<T>::CP;
    constexpr int SR_VC_FLOATS = sr_vc_floats<T>(), SR_A_FLOATS = sr_a_floats<T>();
    extern __shared__ __align__(128) unsigned char smem[];
    T* stg0 = reinterpret_cast<T*>(smem);
    float* regA = reinterpret_cast<float*>(smem + SR_NSTG * STG * sizeof(T));   // row buffer, later V/c buffer A
    float* regB = regA + SR_A_FLOATS;                                      // V/c buffer of subband 0
    float* regC = regB + SR_VC_FLOATS;                                     // V/c buffer of subband 2
    uint64_t* bar = reinterpret_cast<uint64_t*>(regC + SR_VC_FLOATS);

    const int t = threadIdx.x;
    const int cx0 = blockIdx.x * a.O;
    const int ky0 = blockIdx.y * a.SH;
    const int ky1 = min(ky0 + a.SH, a.nH);
    const int b = blockIdx.z;
    const int xs = 2 * cx0 - 16;
    const int K0 = ky0 - 4;
    const int nblk = 1 + (ky1 - ky0 + SR_BK - 1) / SR_BK;
    const int ncols = a.O + 8;
    const int ngroups = ncols / 8;
    const T* in = reinterpret_cast<const T*>(a.in) + (size_t)b * a.in_bstride;
    const int gc = cx0 - 4 + t;   // this thread's coefficient column
    // column-pass source: in-plane columns read their own row-pass column; the
    // mirrored halo columns outside the subband read their partner (R-4)
    const int src_t = (gc < 0 || gc >= a.nW) ? min(max(mirror(gc, a.nW) - cx0 + 4, 0), SR_RW - 1) : t;
    const int pos = src_t;   // row-buffer column (plain layout)
    PRNU_DCHECK(pos >= 0 && pos < SR_RW);
    const bool inner = (t >= 4) && (t < 4 + a.O) && (gc < a.nW);
    // row-pass items of this thread: row rr of groups ga and ga + 8 (skipped when
    // every column of the group lies beyond the subband)
    const int rr = t & 15, ga = t >> 4;
    const bool doA = ga < ngroups && cx0 - 4 + 8 * ga < a.nW;
    const bool doB = ga + 8 < ngroups && cx0 - 4 + 8 * (ga + 8) < a.nW;
    // H-pass item: output row j of the block, outputs 8g .. 8g+7
    const int hj = t & 7, hg = t >> 3;
    const int hx = cx0 + 8 * hg;
    const bool hv = (t < a.O) && (hx < a.nW);
    const bool hfull = hx + 8 <= a.nW;

    if (t == 0) {
        for (int k = 0; k < SR_NSTG; ++k) mbar_init(&bar[k], 1);
        fence_mbar_init();
    }

    // edge fix-up slots (TMA-staged blocks of the first / last strip)
    // the first strip's left mirror is read directly by its group 0 (stg_row22_left):
    // fp32 levels only (measured: levels 2-3 -6% / -10%; the u8 level 1 +1%)
    const bool left_fast = sizeof(T) == 4 && xs < 0 && a.NW >= 16;
    const bool edge = a.use_tma && ((xs < 0 && !left_fast) || xs + LOGW > a.NW);
    int fix_dst[SR_FIX], fix_src[SR_FIX];
    {
        const int nleft = (xs < 0 && !left_fast) ? min(-xs, LOGW) : 0;
        const int xr0 = max(a.NW - xs, nleft), xr1 = min(LOGW, a.NW - xs + 24);
        const int nright = max(xr1 - xr0, 0);
        const int ncnt = nleft + nright;
#pragma unroll
        for (int k = 0; k < SR_FIX; ++k) {
            const int e = t + k * SR_NT;
            fix_dst[k] = -1;
            fix_src[k] = 0;
            if (ncnt > 0 && e < SR_IR * ncnt) {
                const int r = e / ncnt, idx = e - r * ncnt;
                const int x = idx < nleft ? idx : xr0 + idx - nleft;
                fix_dst[k] = r * 512 + x;   // row in bits 9.., logical column in bits 0..8
                fix_src[k] = min(max(mirror(xs + x, a.NW) - xs, 0), LOGW - 1);
            }
        }
    }

    // block i (i = -1: the prologue) is staged in buffer (i + 3) % 3; blocks need input
    // rows 2K .. 2K+15, the prologue rows 2K0-6 .. 2K0-1
    auto stg_of = [&](int i) { return (i + SR_NSTG) % SR_NSTG; };
    // block i needs input rows y0(i) .. y0(i) + nrows(i) - 1 (mirrored into the plane, R-4);
    // they all lie in one 16-row window [box_y, box_y + 16) of the plane unless the plane
    // is shorter than 16 rows: the window is staged by TMA and the row pass reads
    // physical row mirror(y) - box_y (so mirrored blocks are staged asynchronously too)
    auto y0_of = [&](int i) { return i < 0 ? 2 * K0 - 6 : 2 * (K0 + SR_BK * i); };
    // rows y in [-16, NH + 32) mirror by one reflection when NH >= 32 (no integer modulo)
    const bool refl1 = a.NH >= 32;
    auto mirror_row = [&](int y) {
        return refl1 ? (y < 0 ? -1 - y : (y >= a.NH ? 2 * a.NH - 1 - y : y)) : mirror(y, a.NH);
    };
    auto inside = [&](int i) { const int y0 = y0_of(i); return y0 >= 0 && y0 + SR_IR <= a.NH; };
    auto box_y = [&](int i) {
        const int y0 = y0_of(i);
        if (inside(i)) return y0;
        const int y1 = y0 + (i < 0 ? 6 : SR_IR) - 1;
        int lo = min(mirror_row(y0), mirror_row(y1));
        if (y0 < 0 && y1 >= 0) lo = 0;   // the range folds at the top edge
        return min(lo, a.NH - SR_IR);
    };
    // every block is staged by TMA (a 16-row box pair at box_y) when the plane has at
    // least 16 rows; otherwise (and without a tensor map) the threads load the rows
    // planes of 32+ rows: every block's mirrored rows lie in one 16-row window (one
    // reflection, rows -14 .. NH + 28); shorter planes stage their mirrored blocks by
    // threads (the mirrored span can wrap through both edges)
    auto tma_ok = [&](int i) { return a.use_tma && (refl1 || (a.NH >= SR_IR && inside(i))); };
    auto issue = [&](int i) {   // thread 0 only
        const int k = stg_of(i);
        T* s = stg0 + k * STG;
        const int y = box_y(i);
        mbar_arrive_expect_tx(&bar[k], (uint32_t)(2 * SR_IR * BW * sizeof(T)));
        tma_load_3d(s, &map, xs, y, b, &bar[k]);
        tma_load_3d(s + SR_IR * BW, &map, xs + 128, y, b, &bar[k]);
    };
    if (t == 0) {   // prologue and blocks 0, 1 in flight before anything else
        for (int i = -1; i < SR_NSTG - 1 && i < nblk; ++i)
            if (tma_ok(i)) issue(i);
    }
    __syncthreads();   // mbarrier initialisation visible to every thread before any wait
    // Thread loads of nr rows starting at input row y0, rows and columns
    // mirrored (R-4), 16-byte chunks, all of a thread's chunks in flight first.
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && ((a.in_pitch * sizeof(T)) % 16 == 0);
    auto manual = [&](T* s, int y0, int nr) {
        constexpr int CE = 16 / sizeof(T);                         // elements per chunk
        constexpr int NCH = LOGW / CE;                             // chunks per row
        constexpr int PER = (SR_IR * NCH + SR_NT - 1) / SR_NT;     // chunks per thread (max)
        uint4 v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = t + k * SR_NT;
            v[k] = make_uint4(0u, 0u, 0u, 0u);
            if (e < nr * NCH) {
                const int r = e / NCH, ch = e - r * NCH;
                const int gx = xs + ch * CE;
                const T* row = in + (size_t)mirror(y0 + r, a.NH) * a.in_pitch;
                if (vec_ok && gx >= 0 && gx + CE <= a.NW) {
                    v[k] = __ldg(reinterpret_cast<const uint4*>(row + gx));
                } else {
                    T tmp[CE];
#pragma unroll
                    for (int i = 0; i < CE; ++i) tmp[i] = row[mirror(gx + i, a.NW)];
                    memcpy(&v[k], tmp, 16);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = t + k * SR_NT;
            if (e < nr * NCH) {
                const int r = e / NCH, x = (e - r * NCH) * CE;
                if (x < BW) *reinterpret_cast<uint4*>(s + r * BW + x) = v[k];
                if (x >= 128) *reinterpret_cast<uint4*>(s + SR_IR * BW + r * BW + x - 128) = v[k];
            }
        }
    };
    // Row pass (along x) of row rr < nr of the staged rows into the row buffer
    // (regA): lo plane rows [0, 16), hi plane rows [16, 32), columns permuted.
    auto rowpass = [&](const T* s, int prow, int nr) {   // prow: physical staged row of row rr
        PRNU_DCHECK(rr >= nr || (prow >= 0 && prow < SR_IR));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = ga + 8 * h;
            if ((h == 0 ? doA : doB) && rr < nr) {
                float v[24];
                if (h == 0 && left_fast && ga == 0) stg_row22_left(s, prow, v);
                else stg_row22(s, prow, g, v);
                float lo[8], hi[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float2 lh = fmul2s(v[2 * q], c_st_hg[0]);
#pragma unroll
                    for (int i = 1; i < 8; ++i) lh = ffma2(v[2 * q + i], c_st_hg[i], lh);
                    lo[q] = lh.x;
                    hi[q] = lh.y;
                }
                float* dl = regA + rr * SR_RBP + 8 * g;
                float* dh = dl + SR_IR * SR_RBP;
                *reinterpret_cast<float4*>(dl) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                *reinterpret_cast<float4*>(dl + 4) = make_float4(lo[4], lo[5], lo[6], lo[7]);
                *reinterpret_cast<float4*>(dh) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4*>(dh + 4) = make_float4(hi[4], hi[5], hi[6], hi[7]);
            }
        }
    };

    float lo_c[6], hi_c[6], q_c[8][3], c_c[4][3];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int s2 = 0; s2 < 3; ++s2) q_c[k][s2] = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int s2 = 0; s2 < 3; ++s2) c_c[k][s2] = 0.f;
#pragma unroll
    for (int r = 0; r < 6; ++r) lo_c[r] = hi_c[r] = 0.f;

    const float s0 = a.sp.sigma0_sq;
    const int wm = a.sp.wmask;
    uint32_t phase = 0;
    float* const llb = a.ll ? a.ll + (size_t)b * a.out_bstride + gc : nullptr;
    const size_t dst_off = (size_t)b * a.out_bstride + hx;

#ifdef PRNU_STRIP_PROFILE
    unsigned long long pacc[16] = {};
    long long plast = clock64();
#endif
    // i = -1: prologue (the 6 row-pass rows preceding block 0: input rows 2K0-6 .. 2K0-1)
#pragma unroll 1
    for (int i = -1; i < nblk; ++i) {
        const bool pro = i < 0;
        const int K = K0 + SR_BK * i;
        const int sk = stg_of(i);
        T* s = stg0 + sk * STG;
        int prow = -1;   // physical staged row of this thread's row-pass row (TMA blocks)
        if (tma_ok(i)) {
            SPROBE(10);   // carries of the previous block, loop head
            mbar_wait(&bar[sk], (phase >> sk) & 1);
            SPROBE(11);   // TMA wait
            phase ^= 1u << sk;
            prow = inside(i) ? rr : mirror_row(y0_of(i) + rr) - box_y(i);
            PRNU_DCHECK(rr >= (pro ? 6 : SR_IR) || (prow >= 0 && prow < SR_IR));
            if (edge) {   // sources in the plane, destinations outside it: no hazard inside the pass
#pragma unroll
                for (int k = 0; k < SR_FIX; ++k) {
                    const float v = fix_dst[k] >= 0 ? stg_at(s, fix_dst[k] >> 9, fix_src[k]) : 0.f;
                    if (fix_dst[k] >= 0) stg_put(s, fix_dst[k] >> 9, fix_dst[k] & 511, v);
                }
                __syncthreads();
            }
            SPROBE(13);   // edge fix-ups
        } else {
            SPROBE(12);   // carries of the previous block, loop head (thread-loaded block)
            manual(s, pro ? 2 * K0 - 6 : 2 * K, pro ? 6 : SR_IR);
            prow = rr;
            __syncthreads();
        }
        SPROBE(0);        // thread loads of mirrored rows
        rowpass(s, prow, pro ? 6 : SR_IR);
        fence_proxy_async();
        SPROBE(1);
        __syncthreads();   // B1: row buffer complete, staging buffer s consumed
        SPROBE(2);
        if (t == 0 && i + SR_NSTG < nblk && tma_ok(i + SR_NSTG)) issue(i + SR_NSTG);   // into the buffer just consumed
        if (pro) {
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                lo_c[r] = regA[r * SR_RBP + pos];
                hi_c[r] = regA[SR_IR * SR_RBP + r * SR_RBP + pos];
            }
            __syncthreads();
            continue;
        }

        // ---- column pass of this thread's column: coefficient rows K .. K+7
        float q[16][3], cc[8][3];
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int s2 = 0; s2 < 3; ++s2) q[k][s2] = q_c[k][s2];
        {
            float lo[22], hi[22];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                lo[r] = lo_c[r];
                hi[r] = hi_c[r];
            }
#pragma unroll
            for (int r = 0; r < SR_IR; ++r) {
                lo[6 + r] = regA[r * SR_RBP + pos];
                hi[6 + r] = regA[SR_IR * SR_RBP + r * SR_RBP + pos];
            }
            const int kmin = inner ? max(ky0 - K, 0) : SR_BK, kmax = min(ky1 - K, SR_BK);
            float* llp = llb ? llb + (ptrdiff_t)K * a.out_pitch : nullptr;
#pragma unroll
            for (int k = 0; k < SR_BK; ++k) {
                float2 p_l = fmul2s(lo[2 * k], c_st_hg[0]);   // (aa, ad)
                float2 p_h = fmul2s(hi[2 * k], c_st_hg[0]);   // (da, dd)
#pragma unroll
                for (int j = 1; j < 8; ++j) {
                    p_l = ffma2(lo[2 * k + j], c_st_hg[j], p_l);
                    p_h = ffma2(hi[2 * k + j], c_st_hg[j], p_h);
                }
                cc[k][0] = p_h.x;   // da
                cc[k][1] = p_l.y;   // ad
                cc[k][2] = p_h.y;   // dd
                if (llp != nullptr && k >= kmin && k < kmax) llp[(ptrdiff_t)k * a.out_pitch] = p_l.x;
#pragma unroll
                for (int s2 = 0; s2 < 3; ++s2) q[8 + k][s2] = __fmul_rn(cc[k][s2], cc[k][s2]);
            }
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                lo_c[r] = lo[16 + r];
                hi_c[r] = hi[16 + r];
            }
        }
        // rows beyond the subband are mirrored copies (R-4): row r >= nH <- 2nH-1-r
        if (K + SR_BK > a.nH) {
#pragma unroll
            for (int k = 0; k < SR_BK; ++k) {
                const int row = K + k;
                if (row >= a.nH) {
                    const int sl = (2 * a.nH - 1 - row) - K + 8;
#pragma unroll
                    for (int s2 = 0; s2 < 3; ++s2) q[8 + k][s2] = pick16(q, sl, s2);
                }
            }
        }
        // rows -4..-1 (top segment, K == -4) <- rows 3..0
        if (K < 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int s2 = 0; s2 < 3; ++s2) q[8 + k][s2] = q[15 - k][s2];
        }

        if (i > 0) {
            // output rows K-4 .. K+3: vertical sums (nested 3/5/7/9) of subband sb -> buf
            auto write_vc = [&](float* buf, int sb) {
                if (t >= ncols) return;
                float2* P35 = reinterpret_cast<float2*>(buf);
                float2* P79 = P35 + SR_BK * SR_P2;
                float* C = buf + 4 * SR_BK * SR_P2;
#pragma unroll
                for (int j = 0; j < SR_BK; ++j) {
                    const float v3 = q[j + 3][sb] + q[j + 4][sb] + q[j + 5][sb];
                    const float v5 = v3 + q[j + 2][sb] + q[j + 6][sb];
                    const float v7 = v5 + q[j + 1][sb] + q[j + 7][sb];
                    const float v9 = v7 + q[j][sb] + q[j + 8][sb];
                    P35[j * SR_P2 + t] = make_float2(v3, v5);
                    P79[j * SR_P2 + t] = make_float2(v7, v9);
                    C[j * SR_CP + t] = j < 4 ? c_c[j][sb] : cc[j - 4][sb];
                }
            };
            SPROBE(3);
            write_vc(regB, 0);
            write_vc(regC, 2);
            SPROBE(4);
            __syncthreads();   // B2: every thread is done reading the row buffer
            SPROBE(5);
            write_vc(regA, 1);
            SPROBE(6);
            __syncthreads();   // B3: V/c of all three subbands ready
            SPROBE(7);
            if (hv && K - 4 + hj < ky1) {
#pragma unroll kStripHUnroll
                for (int sb = 0; sb < 3; ++sb) {
                    // horizontal sums (sliding), Wiener factor, store: outputs 8hg .. 8hg+7 of row hj
                    const float* buf = sb == 0 ? regB : sb == 1 ? regA : regC;
                    const float2* P35 = reinterpret_cast<const float2*>(buf) + hj * SR_P2 + 8 * hg;
                    const float2* P79 = P35 + SR_BK * SR_P2;
                    const float* crow = buf + 4 * SR_BK * SR_P2 + hj * SR_CP + 4 + 8 * hg;
                    float m[8];
                    {
                        float2 u[12];   // (v3, v5) of columns 2 .. 13
#pragma unroll
                        for (int k = 0; k < 12; ++k) u[k] = P35[2 + k];
                        float s3 = u[1].x + u[2].x + u[3].x;
                        float s5 = u[0].y + u[1].y + u[2].y + u[3].y + u[4].y;
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) {   // slide one column right
                                s3 += u[x + 3].x - u[x].x;
                                s5 += u[x + 4].y - u[x - 1].y;
                            }
                            const float2 r = fmul2(make_float2(s3, s5), c_st_ws[0]);
                            if (ALL4) m[x] = fminf(r.x, r.y);
                            else m[x] = fminf((wm & 1) ? r.x : 3.402823466e38f, (wm & 2) ? r.y : 3.402823466e38f);
                        }
                    }
                    {
                        float2 u[16];   // (v7, v9) of columns 0 .. 15
#pragma unroll
                        for (int k = 0; k < 16; ++k) u[k] = P79[k];
                        float s7 = u[1].x + u[2].x + u[3].x + u[4].x + u[5].x + u[6].x + u[7].x;
                        float s9 = u[0].y + u[1].y + u[2].y + u[3].y + u[4].y + u[5].y + u[6].y + u[7].y + u[8].y;
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) {
                                s7 += u[x + 7].x - u[x].x;
                                s9 += u[x + 8].y - u[x - 1].y;
                            }
                            const float2 r = fmul2(make_float2(s7, s9), c_st_ws[1]);
                            if (ALL4) m[x] = fminf(m[x], fminf(r.x, r.y));
                            else m[x] = fminf(m[x], fminf((wm & 4) ? r.x : 3.402823466e38f,
                                                          (wm & 8) ? r.y : 3.402823466e38f));
                        }
                    }
                    const float4 c0 = *reinterpret_cast<const float4*>(crow);
                    const float4 c1 = *reinterpret_cast<const float4*>(crow + 4);
                    const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
                    float o[8];
#pragma unroll
                    for (int x = 0; x < 8; ++x)   // c - F(c) = c s0 / (max(m - s0, 0) + s0) = c s0 / max(m, s0)
                        o[x] = cv[x] * s0 * rcp_approx(fmaxf(m[x], s0));
                    float* drow = (sb == 0 ? a.d0 : sb == 1 ? a.d1 : a.d2) + dst_off + (size_t)(K - 4 + hj) * a.out_pitch;
                    if (hfull) {
                        reinterpret_cast<float4*>(drow)[0] = make_float4(o[0], o[1], o[2], o[3]);
                        reinterpret_cast<float4*>(drow)[1] = make_float4(o[4], o[5], o[6], o[7]);
                    } else {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if (hx + x < a.nW) drow[x] = o[x];
                    }
                }
            }
        }
        SPROBE(8);
        __syncthreads();   // B4: V/c buffers and the row buffer free for the next block
        SPROBE(9);
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int s2 = 0; s2 < 3; ++s2) q_c[k][s2] = q[8 + k][s2];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int s2 = 0; s2 < 3; ++s2) c_c[k][s2] = cc[4 + k][s2];
    }
#ifdef PRNU_STRIP_PROFILE
    if ((t & 31) == 0)
        for (int k = 0; k < 14; ++k) atomicAdd(&g_strip_prof[k], pacc[k]);
#endif
}

// ------------------------------------------------------------------ host
bool encode_tensor_map_3d(CUtensorMap* map, CUtensorMapDataType dt, size_t elem_bytes, const void* base, uint64_t cols,
                          uint64_t rows, uint64_t depth, uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t box_w,
                          uint32_t box_h);

static bool g_strip_attr = false;
// A/B experiment knob: extra dynamic shared memory per CTA (lowers occupancy)
static int smem_pad() {
    static const int p = getenv("PRNU_STRIP_SMEM_PAD") ? atoi(getenv("PRNU_STRIP_SMEM_PAD")) : 0;
    return p;
}

template <typename T>
static int strip_launch(const T* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll, float* d0,
                        float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                        const ShrinkParams& sp, int nb, cudaStream_t st) {
    if (!g_strip_attr) {
        cudaError_t e[4] = {
            cudaFuncSetAttribute(k_analysis_strip<uint8_t, StripCfg<uint8_t>::MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)strip_smem_bytes<uint8_t>() + smem_pad()),
            cudaFuncSetAttribute(k_analysis_strip<uint8_t, StripCfg<uint8_t>::MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)strip_smem_bytes<uint8_t>() + smem_pad()),
            cudaFuncSetAttribute(k_analysis_strip<float, StripCfg<float>::MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)strip_smem_bytes<float>() + smem_pad()),
            cudaFuncSetAttribute(k_analysis_strip<float, StripCfg<float>::MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)strip_smem_bytes<float>() + smem_pad())};
        for (cudaError_t x : e)
            if (x != cudaSuccess)
                return fail(PRNU_CUDA_ERROR, std::string("cudaFuncSetAttribute(strip): ") + cudaGetErrorString(x));
        g_strip_attr = true;
    }
    StripArgs a{};
    a.in = in;
    a.in_bstride = in_bstride;
    a.in_pitch = in_pitch;
    a.NH = NH;
    a.NW = NW;
    a.ll = ll;
    a.d0 = d0;
    a.d1 = d1;
    a.d2 = d2;
    a.out_bstride = out_bstride;
    a.out_pitch = out_pitch;
    a.nH = nH;
    a.nW = nW;
    a.sp = sp;
    const int S0 = (nW + StripCfg<T>::OMAX - 1) / StripCfg<T>::OMAX;
    a.O = (int)align_up((size_t)((nW + S0 - 1) / S0), 8);
    const int S = (nW + a.O - 1) / a.O;
    static const int sh_env = getenv("PRNU_STRIP_SH") ? atoi(getenv("PRNU_STRIP_SH")) : 0;
    // segments of <= 300 rows (prologue overhead <= 3%), more of them while the grid
    // holds fewer than 6 (u8, level 1) / 1 (fp32, levels >= 2 and SDA frames) waves of
    // 3 CTAs/SM: the fp32 levels of one wave overlap the other streams' work, so fewer,
    // longer segments win there (interleaved A/B, tools/ab_repeat.sh: -0.9% per step)
    static const int seg_rows = getenv("PRNU_STRIP_SEGROWS") ? atoi(getenv("PRNU_STRIP_SEGROWS")) : 300;
    static const int waves_u8 = getenv("PRNU_STRIP_WAVES_U8") ? atoi(getenv("PRNU_STRIP_WAVES_U8")) : 6;
    static const int waves_f32 = getenv("PRNU_STRIP_WAVES_F32") ? atoi(getenv("PRNU_STRIP_WAVES_F32")) : 1;
    const long long waves = sizeof(T) == 1 ? waves_u8 : waves_f32;
    int nseg = (nH + seg_rows - 1) / seg_rows;
    while ((long long)S * nseg * nb < waves * 148 * StripCfg<T>::MINB && (nH + nseg) / (nseg + 1) >= 32) ++nseg;
    a.SH = sh_env > 0 ? (int)align_up((size_t)sh_env, 8) : (int)align_up((size_t)((nH + nseg - 1) / nseg), 8);
    nseg = (nH + a.SH - 1) / a.SH;
    CUtensorMap map{};
    const size_t es = sizeof(T);
    const CUtensorMapDataType dt = sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    a.use_tma = ((in_pitch * es) % 16 == 0) && ((in_bstride * es) % 16 == 0) && ((uintptr_t)in % 16 == 0) &&
                encode_tensor_map_3d(&map, dt, es, in, (uint64_t)NW, (uint64_t)NH, (uint64_t)nb, (uint64_t)in_pitch * es,
                                     (uint64_t)in_bstride * es, StripStage<T>::BOXW, SR_IR);
    static const bool no_tma = getenv("PRNU_STRIP_NO_TMA") != nullptr;
    if (no_tma) a.use_tma = 0;
    dim3 grid(S, nseg, nb);
    if (sp.wmask == 15)
        k_analysis_strip<T, StripCfg<T>::MINB, true><<<grid, SR_NT, strip_smem_bytes<T>() + smem_pad(), st>>>(map, a);
    else
        k_analysis_strip<T, StripCfg<T>::MINB, false><<<grid, SR_NT, strip_smem_bytes<T>() + smem_pad(), st>>>(map, a);
    return PRNU_OK;
}

// Debug: phase cycle counters of k_analysis_strip (all zero unless built with
// -DPRNU_STRIP_PROFILE).  out[0..15]; reset != 0 clears them afterwards.
extern "C" int prnu_debug_strip_profile(unsigned long long* out, int reset) {
#ifdef PRNU_STRIP_PROFILE
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_strip_prof, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_strip_prof, z, sizeof(z));
    }
#else
    for (int k = 0; k < 16; ++k) out[k] = 0;
    (void)reset;
#endif
    return 0;
}

int launch_analysis_strip_u8(const uint8_t* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                             float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                             const ShrinkParams& sp, int nb, cudaStream_t st) {
    return strip_launch<uint8_t>(in, in_bstride, in_pitch, NH, NW, ll, d0, d1, d2, out_bstride, out_pitch, nH, nW, sp,
                                 nb, st);
}
int launch_analysis_strip_f32(const float* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                              float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                              const ShrinkParams& sp, int nb, cudaStream_t st) {
    return strip_launch<float>(in, in_bstride, in_pitch, NH, NW, ll, d0, d1, d2, out_bstride, out_pitch, nH, nW, sp,
                               nb, st);
}

}  // namespace prnu
