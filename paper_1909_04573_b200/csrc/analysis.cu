// analysis.cu — one DWT analysis level (a2) with the local-variance MAP/Wiener
// shrink of its three detail subbands fused (a3): the column-streaming strip
// kernel, with the 8-tap Daubechies filter pair applied as a LIFTING cascade.
//
// Operation (R-2, R-4..R-7): for one level,
//   a[k] = sum_i H_[i] x[2k-6+i],  d[k] = sum_i G_[i] x[2k-6+i]   along rows,
// then along columns (R-6), on the half-sample symmetric extension of the
// plane (R-4); the detail subbands da, ad, dd are then shrunk in the noise
// domain: c - F(c) = c s0 / max(min_w mean_w(c^2), s0) (R-7, R-10).
//
// Lifting.  With e[m] = x[2m], o[m] = x[2m+1] (polyphase components), the
// polyphase matrix of (H_, G_) factors (Daubechies-Sweldens; constants from the
// factorisation in fp64, tools/lifting.py) into
//   e1[m] = e[m]  - C1  o[m]
//   o1[m] = o[m]  + C2A e1[m]   - C2B e1[m+1]
//   e2[m] = e1[m] + C3A o1[m-1] - C3B o1[m]
//   o2[m] = o1[m] + C4A e2[m]   + C4B e2[m+1]
//   e3[m] = e2[m] - C5  o2[m-1]
//   a[k]  = KA o2[k-2],   d[k] = KD e3[k-1]          (KA KD = 1)
// i.e. 8 multiply-adds per (a, d) pair instead of 16: the FP32 pipe (not HBM)
// bounds this kernel, so halving the filter's lane-operations is
// the lever.  The KA/KD scales are folded: rows store (o2, e3) unscaled; after
// the column pass aa = KA^2 A.x, da = A.y, ad = D.x, dd = KD^2 D.y (A = column
// o2, D = column e3), so only LL takes one multiply; the dd scale enters the
// shrink through per-subband window / sigma constants.
//
// Organisation (per CTA of 128 threads = one vertical strip of <= O output
// coefficient columns plus a 4-column halo each side, one thread per region
// column, walking down a segment of output rows in blocks of 8 coefficient rows):
//   * 16 input rows per block arrive by TMA (two boxes, a ring of staging
//     buffers two blocks ahead); mirrored border rows through a row remap,
//     out-of-plane columns through an in-smem fix-up (R-4);
//   * row pass (cooperative; u8: pairs of outputs (k, k+4) through packed
//     FFMA2 with immediate coefficients, the u8 -> fp32 conversion building the
//     pairs directly; fp32: scalar lifting) -> row buffer, (k, k+4) adjacent;
//   * column pass (per thread, streaming): the lifting recurrences along y on
//     the (lo, hi) pair of the thread's column, carrying 4 pairs of state
//     between rows; coefficient rows come out in order;
//   * squares of the details in a 16-row register ring (da scalar, (ad, dd) as
//     a pair), nested vertical window sums 3/5/7/9 -> shared memory;
//   * H pass (cooperative, 8 outputs of one row per thread): sliding horizontal
//     sums ((ad, dd) packed FADD2), window means, Wiener factor, store.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tma.cuh"

namespace prnu {

// ---- lifting constants (fp64 factorisation of R-2's filter, rounded to fp32)
#define LF_C1 0.3222758880002811f
#define LF_C2A 0.29195312600347534f
#define LF_C2B 1.117123605116217f
#define LF_C3A 0.5400282834197139f
#define LF_C3B 1.6889170665560485f
#define LF_C4A 0.5547946968043377f
#define LF_C4B 0.006617338010625356f
#define LF_C5 0.31909219261386207f
#define LF_KA 2.6337752658977225f
#define LF_KD 0.3796831160760221f
#define LF_KA2 6.936772151254619f      // KA^2
#define LF_KD2 0.14415926863319808f    // KD^2
#define LF_KD4 0.02078189473285857f    // KD^4

constexpr int AL_NT = 128;   // threads per CTA == region columns
constexpr int AL_BK = 8;     // coefficient rows per block
constexpr int AL_IR = 16;    // input rows per block
constexpr int AL_RBP = 122;  // row-buffer pitch (floats, == 2 mod 4: conflict-free STS.64, lanes over rows)

template <typename T>
struct AlCfg;
template <>
struct AlCfg<uint8_t> {
    using E = uint8_t;                 // staged element
    static constexpr int DEP = 1;      // frames per staged box (u8pair: 2)
    static constexpr int OMAX = 112;   // output columns per strip (region 120)
    static constexpr int P1 = 124;     // da planes pitch (floats, == 28 mod 32: LDS.128 over 8 rows conflict-free)
    static constexpr int P2 = 122;     // (ad, dd) planes pitch (float2; 2 P2 == 20 mod 32)
    static constexpr int NSTG = 3;     // staging buffers (TMA two blocks ahead)
    static constexpr int BOXW = 144;   // staged bytes per row and box
    // SPLITV = true (one V buffer used by (ad, dd) then da: 52.9 KB, 4 CTAs/SM at 128 registers)
    // measured 8% slower at FHD (11.26 vs 10.46 ms/step): the L1 data pipe, not latency, binds
    static constexpr bool SPLITV = false;
    static constexpr int MINB = 3;
};
template <>
struct AlCfg<uint16_t> {   // exact SDA group sums (level 1 at 3 <= d <= 257)
    using E = uint16_t;
    static constexpr int DEP = 1;
    static constexpr int OMAX = 112;
    static constexpr int P1 = 124;
    static constexpr int P2 = 122;
    static constexpr int NSTG = 1;
    static constexpr int BOXW = 152;   // elements (304 B = 76 words == 12 mod 32)
    static constexpr bool SPLITV = false;
    static constexpr int MINB = 3;
};
template <>
struct AlCfg<float> {
    using E = float;
    static constexpr int DEP = 1;
    static constexpr int OMAX = 104;   // region 112
    static constexpr int P1 = 116;     // == 20 mod 32
    static constexpr int P2 = 114;     // 2 P2 == 4 mod 32
    static constexpr int NSTG = 1;
    static constexpr int BOXW = 140;   // floats (12 mod 32 words)
    static constexpr bool SPLITV = false;
    static constexpr int MINB = 3;
};
template <>
struct AlCfg<u8pair> {   // SDA pairs (level 1 at d = 2): both u8 frames of a group in one depth-2 box
    using E = uint8_t;
    static constexpr int DEP = 2;
    static constexpr int OMAX = 112;
    static constexpr int P1 = 124;
    static constexpr int P2 = 122;
    // a stage holds 2 boxes x 2 frames x 16 rows (9.2 KB, as the u16 sums); measured: 2 stages at
    // 104-column strips (to fit 3 CTAs/SM) 5.37 vs 5.11 ms per 900 FHD pairs, slower
    static constexpr int NSTG = 1;
    static constexpr int BOXW = 144;
    static constexpr bool SPLITV = false;
    static constexpr int MINB = 3;
};
template <typename T>
__host__ __device__ constexpr int al_logw() { return 128 + AlCfg<T>::BOXW; }
// staged elements per stage: [box 0: DEP frames x 16 rows x BOXW][box 1: likewise]
template <typename T>
__host__ __device__ constexpr int al_stage_elems() { return 2 * AlCfg<T>::DEP * AL_IR * AlCfg<T>::BOXW; }
template <typename T>
__host__ __device__ constexpr int al_da_floats() { return 5 * AL_BK * AlCfg<T>::P1; }
template <typename T>
__host__ __device__ constexpr int al_pr_floats() { return 2 * 5 * AL_BK * AlCfg<T>::P2; }
// V buffer: da and (ad, dd) planes side by side, or (SPLITV) one buffer used by both in turn;
// the row buffer (2 x 16 x AL_RBP floats) lives at its start
template <typename T>
__host__ __device__ constexpr int al_v_floats() {
    return AlCfg<T>::SPLITV ? (al_pr_floats<T>() > al_da_floats<T>() ? al_pr_floats<T>() : al_da_floats<T>())
                            : al_da_floats<T>() + al_pr_floats<T>();
}
template <typename T>
constexpr size_t al_smem_bytes() {
    return AlCfg<T>::NSTG * al_stage_elems<T>() * sizeof(typename AlCfg<T>::E) + sizeof(float) * al_v_floats<T>() + 32;
}
static_assert(2 * AL_IR * AL_RBP <= 5 * AL_BK * AlCfg<float>::P1, "row buffer inside the da planes");
static_assert(AlCfg<uint8_t>::OMAX + 8 <= AlCfg<uint8_t>::P2 && AlCfg<float>::OMAX + 8 <= AlCfg<float>::P2, "V planes");
template <typename T>
constexpr bool al_fits() {   // MINB CTAs per SM in 228 KB (1 KB reserved per CTA)
    return AlCfg<T>::MINB * (al_smem_bytes<T>() + 1024) <= 228 * 1024;
}
static_assert(al_fits<uint8_t>() && al_fits<uint16_t>() && al_fits<float>() && al_fits<u8pair>(), "CTAs per SM");

struct AlArgs {
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
    int O;                  // output columns per strip (multiple of 8)
    int SH;                 // output rows per segment (multiple of 8)
    int use_tma;
    float div_d, div_r;     // u16 SDA sums: S = RN(sum / d) (R-11)
};

__device__ __forceinline__ float al_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// per-subband constants of the (ad, dd) pair: window means (1/w^2, KD^4/w^2), sigma (s0, KD^2 s0) set per launch
__constant__ float2 c_al_w[4] = {{1.0f / 9.0f, LF_KD4 / 9.0f},
                                 {1.0f / 25.0f, LF_KD4 / 25.0f},
                                 {1.0f / 49.0f, LF_KD4 / 49.0f},
                                 {1.0f / 81.0f, LF_KD4 / 81.0f}};

// staged row r (< DEP * 16: frame r / 16, row r % 16), logical column x (box 0: x < BOXW, box 1: x >= 128)
template <typename T>
__device__ __forceinline__ typename AlCfg<T>::E al_stg_at(const typename AlCfg<T>::E* s, int r, int x) {
    constexpr int BW = AlCfg<T>::BOXW, BOFF = AlCfg<T>::DEP * AL_IR * BW;
    return x < BW ? s[r * BW + x] : s[BOFF + r * BW + x - 128];
}
template <typename T>
__device__ __forceinline__ void al_stg_put(typename AlCfg<T>::E* s, int r, int x, typename AlCfg<T>::E v) {
    constexpr int BW = AlCfg<T>::BOXW, BOFF = AlCfg<T>::DEP * AL_IR * BW;
    if (x < BW) s[r * BW + x] = v;
    if (x >= 128) s[BOFF + r * BW + x - 128] = v;
}

// ---- row pass of one item (staged row r, group g: region columns 8g .. 8g+7):
// lo/hi (unscaled o2 / e3) of the 8 coefficient columns as pairs (i, i+4), i < 4.
// Inputs v[k] = logical staged column 16g + 2 + k (k < 22) = x[2 gc0 - 6 + k].
// lifting of the 14 input pairs E[j] = (v[2j], v[2j+8]), O[j] = (v[2j+1], v[2j+9]), j < 7
__device__ __forceinline__ void al_lift_pairs(const float2 (&E)[7], const float2 (&O)[7], float2 (&L)[4], float2 (&Hh)[4]) {
    float2 E1[7], O1[6], E2[6], O2[5];
#pragma unroll
    for (int j = 0; j < 7; ++j) E1[j] = ffma2(-LF_C1, O[j], E[j]);
#pragma unroll
    for (int j = 0; j < 6; ++j) O1[j] = ffma2(-LF_C2B, E1[j + 1], ffma2(LF_C2A, E1[j], O[j]));
#pragma unroll
    for (int j = 1; j < 6; ++j) E2[j] = ffma2(-LF_C3B, O1[j], ffma2(LF_C3A, O1[j - 1], E1[j]));
#pragma unroll
    for (int j = 1; j < 5; ++j) O2[j] = ffma2(LF_C4B, E2[j + 1], ffma2(LF_C4A, E2[j], O1[j]));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        L[i] = O2[i + 1];                          // o2 at k = i, i + 4
        Hh[i] = ffma2(-LF_C5, O2[i + 1], E2[i + 2]);  // e3 at k = i, i + 4 (e3[j] = e2[j] - C5 o2[j-1])
    }
}
__device__ __forceinline__ void al_rowpass(const uint8_t* s, int r, int g, float, float, float2 (&L)[4],
                                           float2 (&Hh)[4]) {
    constexpr int BW = AlCfg<uint8_t>::BOXW;
    const uint8_t* src = s + (g < 8 ? r * BW + 16 * g : AL_IR * BW + r * BW + 16 * g - 128);
    const uint4 w0 = *reinterpret_cast<const uint4*>(src);
    const uint2 w1 = *reinterpret_cast<const uint2*>(src + 16);
    const uint32_t w[6] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y};
    // byte b (logical 16g + b) -> 2^23 + byte as a float bit pattern
    auto bf = [&](int b) { return __uint_as_float(__byte_perm(w[b >> 2], 0x4B000000u, 0x7540u | (uint32_t)(b & 3))); };
    const float2 m23 = make_float2(-8388608.f, -8388608.f);
    float2 E[7], O[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) {   // E[j] = (v[2j], v[2j+8]), O[j] = (v[2j+1], v[2j+9]) exactly
        E[j] = add2(make_float2(bf(2 * j + 2), bf(2 * j + 10)), m23);
        O[j] = add2(make_float2(bf(2 * j + 3), bf(2 * j + 11)), m23);
    }
    al_lift_pairs(E, O, L, Hh);
}
// exact SDA group sums: v[k] = RN(sum / d) (R-11), then the same lifting
__device__ __forceinline__ void al_rowpass(const uint16_t* s, int r, int g, float dv, float rv, float2 (&L)[4],
                                           float2 (&Hh)[4]) {
    constexpr int BW = AlCfg<uint16_t>::BOXW;
    const uint16_t* src = s + (g < 8 ? r * BW + 16 * g : AL_IR * BW + r * BW + 16 * g - 128);
    const uint4 w0 = *reinterpret_cast<const uint4*>(src);
    const uint4 w1 = *reinterpret_cast<const uint4*>(src + 8);
    const uint4 w2 = *reinterpret_cast<const uint4*>(src + 16);
    const uint32_t w[12] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w, w2.x, w2.y, w2.z, w2.w};
    // element e (logical 16g + e) -> 2^23 + sum as a float bit pattern
    auto bf = [&](int e) {
        return __uint_as_float(__byte_perm(w[e >> 1], 0x4B000000u, (e & 1) ? 0x7632u : 0x7610u));
    };
    const float2 m23 = make_float2(-8388608.f, -8388608.f);
    float2 E[7], O[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) {   // sums exactly, then q = RN(sum / d) lane-wise (sda_div, packed)
        const float2 se = add2(make_float2(bf(2 * j + 2), bf(2 * j + 10)), m23);
        const float2 so = add2(make_float2(bf(2 * j + 3), bf(2 * j + 11)), m23);
        const float2 qe = mul2(se, make_float2(rv, rv)), qo = mul2(so, make_float2(rv, rv));
        E[j] = ffma2(rv, ffma2(-dv, qe, se), qe);
        O[j] = ffma2(rv, ffma2(-dv, qo, so), qo);
    }
    al_lift_pairs(E, O, L, Hh);
}
// SDA pairs (d = 2): S = (b0 + b1) / 2 exactly (u8_half_bias, R-11), then the same lifting
__device__ __forceinline__ void al_rowpass_pair(const uint8_t* s, int r, int g, float2 (&L)[4], float2 (&Hh)[4]) {
    constexpr int BW = AlCfg<u8pair>::BOXW;
    const uint8_t* src = s + (g < 8 ? r * BW + 16 * g : 2 * AL_IR * BW + r * BW + 16 * g - 128);
    const uint8_t* src1 = src + AL_IR * BW;   // the group's second frame, same row
    const uint4 a0 = *reinterpret_cast<const uint4*>(src);
    const uint2 a1 = *reinterpret_cast<const uint2*>(src + 16);
    const uint4 b0 = *reinterpret_cast<const uint4*>(src1);
    const uint2 b1 = *reinterpret_cast<const uint2*>(src1 + 16);
    const uint32_t wa[6] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y};
    const uint32_t wb[6] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y};
    auto ha = [&](int b) { return u8_half_bias(wa[b >> 2], b & 3); };
    auto hb = [&](int b) { return u8_half_bias(wb[b >> 2], b & 3); };
    const float2 m22 = make_float2(-4194304.f, -4194304.f);
    auto sv = [&](int b0_, int b1_) {   // (S[b0_], S[b1_]) = ((h(a) - 2^22) + h(b)) - 2^22, exact
        return add2(add2(add2(make_float2(ha(b0_), ha(b1_)), m22), make_float2(hb(b0_), hb(b1_))), m22);
    };
    float2 E[7], O[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        E[j] = sv(2 * j + 2, 2 * j + 10);
        O[j] = sv(2 * j + 3, 2 * j + 11);
    }
    al_lift_pairs(E, O, L, Hh);
}
__device__ __forceinline__ void al_rowpass(const float* s, int r, int g, float, float, float2 (&L)[4],
                                           float2 (&Hh)[4]) {
    constexpr int BW = AlCfg<float>::BOXW;
    const float* src = s + (g < 8 ? r * BW + 16 * g : AL_IR * BW + r * BW + 16 * g - 128) + 2;
    float v[22];
    {
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
    }
    float e1[11], o1[10], e2[10], o2[9];
#pragma unroll
    for (int j = 0; j < 11; ++j) e1[j] = fmaf(-LF_C1, v[2 * j + 1], v[2 * j]);
#pragma unroll
    for (int j = 0; j < 10; ++j) o1[j] = fmaf(-LF_C2B, e1[j + 1], fmaf(LF_C2A, e1[j], v[2 * j + 1]));
#pragma unroll
    for (int j = 1; j < 10; ++j) e2[j] = fmaf(-LF_C3B, o1[j], fmaf(LF_C3A, o1[j - 1], e1[j]));
#pragma unroll
    for (int j = 1; j < 9; ++j) o2[j] = fmaf(LF_C4B, e2[j + 1], fmaf(LF_C4A, e2[j], o1[j]));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        L[i] = make_float2(o2[i + 1], o2[i + 5]);
        Hh[i] = make_float2(fmaf(-LF_C5, o2[i + 1], e2[i + 2]), fmaf(-LF_C5, o2[i + 5], e2[i + 6]));
    }
}

__device__ __forceinline__ float al_pick16(const float (&q)[16], int sl) {
    float r = q[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) r = (sl == i) ? q[i] : r;
    return r;
}
__device__ __forceinline__ float2 al_pick16(const float2 (&q)[16], int sl) {
    float2 r = q[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) r = (sl == i) ? q[i] : r;
    return r;
}


template <typename T, int MINB, bool ALL4>
__global__ void __launch_bounds__(AL_NT, MINB) k_analysis_lift(const __grid_constant__ CUtensorMap map, AlArgs a) {
    constexpr int BW = AlCfg<T>::BOXW;
    constexpr int LOGW = al_logw<T>();
    constexpr int STG = al_stage_elems<T>();
    constexpr int NSTG = AlCfg<T>::NSTG, P1 = AlCfg<T>::P1, P2 = AlCfg<T>::P2;
    constexpr bool SPLITV = AlCfg<T>::SPLITV;
    constexpr int DEP = AlCfg<T>::DEP;
    using E = typename AlCfg<T>::E;
    extern __shared__ __align__(128) unsigned char smem[];
    E* stg0 = reinterpret_cast<E*>(smem);
    float* V0 = reinterpret_cast<float*>(smem + NSTG * STG * sizeof(E));
    float* DA = V0;                                                         // da planes v3 v5 v7 v9 c [8][P1]; row buffer
    float2* PR = reinterpret_cast<float2*>(SPLITV ? V0 : V0 + al_da_floats<T>());   // (ad, dd) planes [8][P2]
    uint64_t* bar = reinterpret_cast<uint64_t*>(V0 + al_v_floats<T>());
    float* RBlo = DA;                    // row buffer: lo [16][AL_RBP], hi [16][AL_RBP] (overlaps the da planes)
    float* RBhi = DA + AL_IR * AL_RBP;

    const int t = threadIdx.x;
    const int cx0 = blockIdx.x * a.O;
    const int ky0 = blockIdx.y * a.SH;
    const int ky1 = min(ky0 + a.SH, a.nH);
    const int b = blockIdx.z;
    const int xs = 2 * cx0 - 16;
    const int K0 = ky0 - 4;
    const int nblk = 1 + (ky1 - ky0 + AL_BK - 1) / AL_BK;
    const int ncols = a.O + 8;
    const int ngroups = ncols / 8;
    const E* in = reinterpret_cast<const E*>(a.in) + (size_t)b * a.in_bstride;
    const int gc = cx0 - 4 + t;   // this thread's coefficient column
    // column-pass source column: in-plane columns read their own row-pass column; mirrored
    // halo columns outside the subband read their partner's (R-4); idle threads a valid one
    int src = (gc < 0 || gc >= a.nW) ? mirror(gc, a.nW) - cx0 + 4 : t;
    src = min(max(src, 0), ncols - 1);
    const int slot = 8 * (src >> 3) + 2 * (src & 3) + ((src >> 2) & 1);   // (k, k+4) adjacent
    PRNU_DCHECK(slot >= 0 && slot < AL_RBP && ncols <= P2 && ncols <= P1 && (ncols & 7) == 0);
    const bool inner = (t >= 4) && (t < 4 + a.O) && (gc < a.nW);
    const int rr = t & 15, ga = t >> 4;
    const bool doA = ga < ngroups && cx0 - 4 + 8 * ga < a.nW;
    const bool doB = ga + 8 < ngroups && cx0 - 4 + 8 * (ga + 8) < a.nW;
    const int hj = t & 7, hg = t >> 3;
    const int hx = cx0 + 8 * hg;
    const bool hv = (t < a.O) && (hx < a.nW);
    const bool hfull = hx + 8 <= a.nW;   // 8 outputs in the plane: one 256-bit store (32-byte aligned, host-checked)

    if (t == 0) {
        for (int k = 0; k < NSTG; ++k) mbar_init(&bar[k], 1);
        fence_mbar_init();
    }
    const bool edge = a.use_tma && (xs < 0 || xs + LOGW > a.NW);
    // edge fix-up (TMA-staged blocks of the first / last strip): out-of-plane logical columns
    // of the staged rows receive their mirrored in-plane values (R-4).  At most 16 + 24
    // columns (xs >= -16; input columns NW .. NW+23): thread t handles column slot t % 40
    // of staged rows t / 40 + 3k (DEP x 16 rows); sources in the plane, destinations outside
    // it (no hazard).
    int fx = -1, fs = 0;
    const int fr0 = t / 40;
    if (edge) {
        const int nleft = xs < 0 ? min(-xs, LOGW) : 0;
        const int xr0 = max(a.NW - xs, nleft), xr1 = min(LOGW, a.NW - xs + 24);
        const int ncnt = nleft + max(xr1 - xr0, 0);
        const int idx = t - 40 * fr0;
        if (t < 120 && idx < ncnt) {
            fx = idx < nleft ? idx : xr0 + idx - nleft;
            fs = min(max(mirror(xs + fx, a.NW) - xs, 0), LOGW - 1);
        }
    }
    auto fixup = [&](E* s) {
        if (fx < 0) return;
        constexpr int FR = (DEP * AL_IR + 2) / 3;
        E v[FR];
#pragma unroll
        for (int k = 0; k < FR; ++k)
            if (fr0 + 3 * k < DEP * AL_IR) v[k] = al_stg_at<T>(s, fr0 + 3 * k, fs);
#pragma unroll
        for (int k = 0; k < FR; ++k)
            if (fr0 + 3 * k < DEP * AL_IR) al_stg_put<T>(s, fr0 + 3 * k, fx, v[k]);
    };
    auto stg_of = [&](int i) { return (i + NSTG) % NSTG; };
    auto y0_of = [&](int i) { return i < 0 ? 2 * K0 - 6 : 2 * (K0 + AL_BK * i); };
    const bool refl1 = a.NH >= 32;
    auto mirror_row = [&](int y) {
        return refl1 ? (y < 0 ? -1 - y : (y >= a.NH ? 2 * a.NH - 1 - y : y)) : mirror(y, a.NH);
    };
    auto inside = [&](int i) { const int y0 = y0_of(i); return y0 >= 0 && y0 + AL_IR <= a.NH; };
    auto box_y = [&](int i) {
        const int y0 = y0_of(i);
        if (inside(i)) return y0;
        const int y1 = y0 + (i < 0 ? 6 : AL_IR) - 1;
        int lo = min(mirror_row(y0), mirror_row(y1));
        if (y0 < 0 && y1 >= 0) lo = 0;
        return min(lo, a.NH - AL_IR);
    };
    // (u8pair: TMA only; the host takes the u16-sum path where the pair boxes do not apply)
    auto tma_ok = [&](int i) { return a.use_tma && (refl1 || (a.NH >= AL_IR && inside(i))); };
    auto issue = [&](int i) {
        const int k = stg_of(i);
        E* s = stg0 + k * STG;
        const int y = box_y(i);
        PRNU_DCHECK(y >= 0 && y + AL_IR <= a.NH);
        mbar_arrive_expect_tx(&bar[k], (uint32_t)(2 * DEP * AL_IR * BW * sizeof(E)));
        tma_load_3d(s, &map, xs, y, DEP * b, &bar[k]);
        tma_load_3d(s + DEP * AL_IR * BW, &map, xs + 128, y, DEP * b, &bar[k]);
    };
    if (t == 0) {
        for (int i = -1; i < NSTG - 1 && i < nblk; ++i)
            if (tma_ok(i)) issue(i);
    }
    __syncthreads();
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && ((a.in_pitch * sizeof(E)) % 16 == 0);
    auto manual = [&](E* s, int y0, int nr) {
        if (DEP != 1) {   // unreachable: pairs are staged by TMA only
            __trap();
            return;
        }
        constexpr int CE = 16 / sizeof(E);
        constexpr int NCH = LOGW / CE;
        constexpr int PER = (AL_IR * NCH + AL_NT - 1) / AL_NT;
        uint4 v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = t + k * AL_NT;
            v[k] = make_uint4(0u, 0u, 0u, 0u);
            if (e < nr * NCH) {
                const int r = e / NCH, ch = e - r * NCH;
                const int gx = xs + ch * CE;
                const E* row = in + (size_t)mirror(y0 + r, a.NH) * a.in_pitch;
                if (vec_ok && gx >= 0 && gx + CE <= a.NW) {
                    v[k] = __ldg(reinterpret_cast<const uint4*>(row + gx));
                } else {
                    E tmp[CE];
#pragma unroll
                    for (int i = 0; i < CE; ++i) tmp[i] = row[mirror(gx + i, a.NW)];
                    memcpy(&v[k], tmp, 16);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = t + k * AL_NT;
            if (e < nr * NCH) {
                const int r = e / NCH, x = (e - r * NCH) * CE;
                if (x < BW) *reinterpret_cast<uint4*>(s + r * BW + x) = v[k];
                if (x >= 128) *reinterpret_cast<uint4*>(s + AL_IR * BW + r * BW + x - 128) = v[k];
            }
        }
    };
    auto rowpass = [&](const E* s, int prow, int nr) {
        if (rr >= nr) return;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int g = ga + 8 * h;
            if (h == 0 ? doA : doB) {
                float2 L[4], Hh[4];
                if constexpr (DEP == 2)
                    al_rowpass_pair(s, prow, g, L, Hh);
                else
                    al_rowpass(s, prow, g, a.div_d, a.div_r, L, Hh);
                PRNU_DCHECK(rr < AL_IR && 8 * g + 8 <= AL_RBP && prow >= 0 && prow < AL_IR);
                float2* dl = reinterpret_cast<float2*>(RBlo + rr * AL_RBP + 8 * g);
                float2* dh = reinterpret_cast<float2*>(RBhi + rr * AL_RBP + 8 * g);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    dl[i] = L[i];
                    dh[i] = Hh[i];
                }
            }
        }
    };

    // column-pass lifting state (pairs over (lo, hi) of this column): o[m-1], e1[m-1], o1[m-2], e2[m-2]
    float2 so = make_float2(0.f, 0.f), se1 = so, so1 = so, se2 = so;
    float qd_c[8], cd_c[4];       // da: squares of the last 8 coefficient rows, c of the last 4
    float2 qp_c[8], cp_c[4];      // (ad, dd) likewise
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        qd_c[k] = 0.f;
        qp_c[k] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        cd_c[k] = 0.f;
        cp_c[k] = make_float2(0.f, 0.f);
    }
    const float s0 = a.sp.sigma0_sq;
    const float2 s0p = make_float2(s0, s0 * LF_KD2);
    // ALL4 (windows 3, 5, 7, 9): the window means are kept scaled by 81 (the 9x9 sum needs no
    // multiply; the 7 and 9 minima go through one 3-input min), and the Wiener factor
    // c s0 / max(m, s0) = c (81 s0) / max(81 m, 81 s0) takes the scaled thresholds; for the
    // (ad, dd) pair the dd lane's KD^4 / KD^2 factors move from the window weights into them
    const float t81 = 81.0f * s0;
    const float2 t81p = make_float2(t81, t81 / LF_KD4);   // thresholds (da / ad lane, dd lane)
    const float2 c81p = make_float2(t81, t81 / LF_KD2);   // numerators
    // the 7x7 term kept live for a 3-input min only where it does not spill (fp32 levels;
    // measured: the u8 / u16 / pair instances spill at the 168-register cap and run slower)
    constexpr bool MIN3 = ALL4 && std::is_same<T, float>::value;
    const int wm = a.sp.wmask;
    uint32_t phase = 0;
    const long long ll_off = (long long)b * a.out_bstride + gc;   // LL element offset of row 0 (a.ll may be null)
    const size_t dst_off = (size_t)b * a.out_bstride + hx;

#pragma unroll 1
    for (int i = -1; i < nblk; ++i) {
        const bool pro = i < 0;
        const int K = K0 + AL_BK * i;
        const int sk = stg_of(i);
        E* s = stg0 + sk * STG;
        int prow;
        PRNU_STRESS(1);
        if (tma_ok(i)) {
            mbar_wait(&bar[sk], (phase >> sk) & 1);
            phase ^= 1u << sk;
            prow = inside(i) ? rr : mirror_row(y0_of(i) + rr) - box_y(i);
            if (edge) {
                fixup(s);
                __syncthreads();
            }
        } else {
            manual(s, pro ? 2 * K0 - 6 : 2 * K, pro ? 6 : AL_IR);
            prow = rr;
            __syncthreads();
        }
        rowpass(s, prow, pro ? 6 : AL_IR);
        fence_proxy_async();
        __syncthreads();   // B1: row buffer complete, staging buffer s consumed
        PRNU_STRESS(2);
        if (t == 0 && i + NSTG < nblk && tma_ok(i + NSTG)) issue(i + NSTG);

        // ---- column pass: (e, o) row pairs j of the block = coefficient rows m = K + j;
        // squares straight into the ring (slots 8..15), LL stored as it comes out
        auto lift_y = [&](int j, float2& o2, float2& e3) {
            const float2 pe = make_float2(RBlo[(2 * j) * AL_RBP + slot], RBhi[(2 * j) * AL_RBP + slot]);
            const float2 po = make_float2(RBlo[(2 * j + 1) * AL_RBP + slot], RBhi[(2 * j + 1) * AL_RBP + slot]);
            const float2 e1 = ffma2(-LF_C1, po, pe);                              // e1[m]
            const float2 o1 = ffma2(-LF_C2B, e1, ffma2(LF_C2A, se1, so));           // o1[m-1]
            const float2 e2 = ffma2(-LF_C3B, o1, ffma2(LF_C3A, so1, se1));          // e2[m-1]
            o2 = ffma2(LF_C4B, e2, ffma2(LF_C4A, se2, so1));                        // o2[m-2] = a[m] / KA
            e3 = ffma2(-LF_C5, o2, e2);                                           // e3[m-1] = d[m] / KD
            so = po;
            se1 = e1;
            so1 = o1;
            se2 = e2;
        };
        if (pro) {   // input rows 2K0-6 .. 2K0-1: lifting state only
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                float2 o2, e3;
                lift_y(j, o2, e3);
            }
            __syncthreads();   // row buffer free for block 0
            continue;
        }
        float qd[16], cn[8];
        float2 qp[16], cpn[8];
        // LL rows of this block inside the segment (bit j: row K + j), interior columns only
        const uint32_t llmask = (a.ll != nullptr && inner)
                                    ? ((0xFFu >> (8 - min(max(ky1 - K, 0), 8))) & (0xFFu << min(max(ky0 - K, 0), 8)))
                                    : 0u;
        float* llp = a.ll + ll_off + K * a.out_pitch;
#pragma unroll
        for (int j = 0; j < AL_BK; ++j) {
            float2 o2, e3;
            lift_y(j, o2, e3);
            const float llv = LF_KA2 * o2.x;
            PRNU_DCHECK(!(llmask & (1u << j)) || (K + j >= 0 && K + j < a.nH && gc >= 0 && gc < a.nW));
            if (llmask & (1u << j)) *llp = llv;
            llp += a.out_pitch;
            cn[j] = o2.y;                  // da
            cpn[j] = e3;                   // (ad, dd / KD^2)
            qd[8 + j] = __fmul_rn(o2.y, o2.y);
            qp[8 + j] = mul2(e3, e3);
        }
        float cd[8];
        float2 cp[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            qd[k] = qd_c[k];
            qp[k] = qp_c[k];
        }
        // rows beyond the subband are mirrored copies (R-4): row r >= nH <- 2nH-1-r
        if (K + AL_BK > a.nH) {
#pragma unroll
            for (int k = 0; k < AL_BK; ++k) {
                const int row = K + k;
                if (row >= a.nH) {
                    const int sl = (2 * a.nH - 1 - row) - K + 8;
                    qd[8 + k] = al_pick16(qd, sl);
                    qp[8 + k] = al_pick16(qp, sl);
                }
            }
        }
        if (K < 0) {   // rows -4..-1 (top segment) <- rows 3..0
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                qd[8 + k] = qd[15 - k];
                qp[8 + k] = qp[15 - k];
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // c of output rows K-4 .. K+3
            cd[j] = j < 4 ? cd_c[j] : cn[j - 4];
            cp[j] = j < 4 ? cp_c[j] : cpn[j - 4];
        }
        if (i > 0) {
            // output rows K-4 .. K+3: nested vertical sums over ring rows j .. j+8 -> V planes,
            // then the H pass.  SPLITV (4 CTAs/SM configurations): the (ad, dd) and the da planes
            // share one buffer, written and consumed one after the other.
            const bool hon = hv && K - 4 + hj < ky1;
            PRNU_DCHECK(!hon || (K - 4 + hj >= 0 && K - 4 + hj < a.nH && hx < a.nW && 8 * hg + 16 <= P2 &&
                                 (!hfull || hx + 8 <= a.out_pitch)));
            const size_t roff = dst_off + (size_t)(K - 4 + hj) * a.out_pitch;
            auto write_pair = [&]() {
                if (t < ncols) {
#pragma unroll
                    for (int j = 0; j < AL_BK; ++j) {
                        const float2 v3 = add2(add2(qp[j + 3], qp[j + 4]), qp[j + 5]);
                        const float2 v5 = add2(v3, add2(qp[j + 2], qp[j + 6]));
                        const float2 v7 = add2(v5, add2(qp[j + 1], qp[j + 7]));
                        const float2 v9 = add2(v7, add2(qp[j], qp[j + 8]));
                        PR[(0 * AL_BK + j) * P2 + t] = v3;
                        PR[(1 * AL_BK + j) * P2 + t] = v5;
                        PR[(2 * AL_BK + j) * P2 + t] = v7;
                        PR[(3 * AL_BK + j) * P2 + t] = v9;
                        PR[(4 * AL_BK + j) * P2 + t] = cp[j];
                    }
                }
            };
            auto write_da = [&]() {
                if (t < ncols) {
#pragma unroll
                    for (int j = 0; j < AL_BK; ++j) {
                        const float v3 = qd[j + 3] + qd[j + 4] + qd[j + 5];
                        const float v5 = v3 + qd[j + 2] + qd[j + 6];
                        const float v7 = v5 + qd[j + 1] + qd[j + 7];
                        const float v9 = v7 + qd[j] + qd[j + 8];
                        DA[(0 * AL_BK + j) * P1 + t] = v3;
                        DA[(1 * AL_BK + j) * P1 + t] = v5;
                        DA[(2 * AL_BK + j) * P1 + t] = v7;
                        DA[(3 * AL_BK + j) * P1 + t] = v9;
                        DA[(4 * AL_BK + j) * P1 + t] = cd[j];
                    }
                }
            };
            auto h_da = [&]() {
                // ---- da: region columns 8hg .. 8hg+15 of row hj
                {
                    const float* base = DA + hj * P1 + 8 * hg;
                    float m[8], r7[8];
                    {
                        float u[16];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 0 * AL_BK * P1 + 4 * q4);
                            u[4 * q4] = x.x; u[4 * q4 + 1] = x.y; u[4 * q4 + 2] = x.z; u[4 * q4 + 3] = x.w;
                        }
                        float s3 = u[3] + u[4] + u[5];
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s3 += u[x + 5] - u[x + 2];
                            m[x] = ALL4 ? s3 * 9.0f : (wm & 1) ? s3 * (1.0f / 9.0f) : 3.402823466e38f;
                        }
                    }
                    {
                        float u[16];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 1 * AL_BK * P1 + 4 * q4);
                            u[4 * q4] = x.x; u[4 * q4 + 1] = x.y; u[4 * q4 + 2] = x.z; u[4 * q4 + 3] = x.w;
                        }
                        float s5 = u[2] + u[3] + u[4] + u[5] + u[6];
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s5 += u[x + 6] - u[x + 1];
                            if (ALL4 || (wm & 2)) m[x] = fminf(m[x], s5 * (ALL4 ? 3.24f : 1.0f / 25.0f));
                        }
                    }
                    {
                        float u[16];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 2 * AL_BK * P1 + 4 * q4);
                            u[4 * q4] = x.x; u[4 * q4 + 1] = x.y; u[4 * q4 + 2] = x.z; u[4 * q4 + 3] = x.w;
                        }
                        float s7 = u[1] + u[2] + u[3] + u[4] + u[5] + u[6] + u[7];
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s7 += u[x + 7] - u[x];
                            if (MIN3) r7[x] = s7 * (81.0f / 49.0f);
                            else if (ALL4) m[x] = fminf(m[x], s7 * (81.0f / 49.0f));
                            else if (wm & 4) m[x] = fminf(m[x], s7 * (1.0f / 49.0f));
                        }
                    }
                    {
                        float u[16];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 3 * AL_BK * P1 + 4 * q4);
                            u[4 * q4] = x.x; u[4 * q4 + 1] = x.y; u[4 * q4 + 2] = x.z; u[4 * q4 + 3] = x.w;
                        }
                        float s9 = u[0] + u[1] + u[2] + u[3] + u[4] + u[5] + u[6] + u[7] + u[8];
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s9 += u[x + 8] - u[x - 1];
                            if (MIN3) m[x] = fminf(fminf(m[x], r7[x]), s9);   // FMNMX3
                            else if (ALL4) m[x] = fminf(m[x], s9);
                            else if (wm & 8) m[x] = fminf(m[x], s9 * (1.0f / 81.0f));
                        }
                    }
                    const float4 c0 = *reinterpret_cast<const float4*>(base + 4 * AL_BK * P1 + 4);
                    const float4 c1 = *reinterpret_cast<const float4*>(base + 4 * AL_BK * P1 + 8);
                    const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
                    float o[8];
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        o[x] = ALL4 ? (cv[x] * t81) * al_rcp(fmaxf(m[x], t81)) : (cv[x] * s0) * al_rcp(fmaxf(m[x], s0));
                    float* drow = a.d0 + roff;
                    if (hfull) {
                        st_global_v8(drow, o);
                    } else {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if (hx + x < a.nW) drow[x] = o[x];
                    }
                }
            };
            auto h_pair = [&]() {
                // ---- (ad, dd): float2 region columns 8hg .. 8hg+15 of row hj
                {
                    const float2* base = PR + hj * P2 + 8 * hg;
                    float2 m[8], r7[8];
                    {
                        float2 u[12];   // columns 2 .. 13
#pragma unroll
                        for (int q2 = 0; q2 < 6; ++q2) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 0 * AL_BK * P2 + 2 + 2 * q2);
                            u[2 * q2] = make_float2(x.x, x.y);
                            u[2 * q2 + 1] = make_float2(x.z, x.w);
                        }
                        float2 s3 = add2(add2(u[1], u[2]), u[3]);
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s3 = add2(s3, sub2(u[x + 3], u[x]));
                            m[x] = ALL4 ? mul2(s3, make_float2(9.0f, 9.0f))
                                   : (wm & 1) ? mul2(s3, c_al_w[0]) : make_float2(3.402823466e38f, 3.402823466e38f);
                        }
                    }
                    {
                        float2 u[12];   // columns 2 .. 13
#pragma unroll
                        for (int q2 = 0; q2 < 6; ++q2) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 1 * AL_BK * P2 + 2 + 2 * q2);
                            u[2 * q2] = make_float2(x.x, x.y);
                            u[2 * q2 + 1] = make_float2(x.z, x.w);
                        }
                        float2 s5 = add2(add2(add2(u[0], u[1]), add2(u[2], u[3])), u[4]);
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s5 = add2(s5, sub2(u[x + 4], u[x - 1]));
                            if (ALL4 || (wm & 2)) {
                                const float2 r = ALL4 ? mul2(s5, make_float2(3.24f, 3.24f)) : mul2(s5, c_al_w[1]);
                                m[x] = make_float2(fminf(m[x].x, r.x), fminf(m[x].y, r.y));
                            }
                        }
                    }
                    {
                        float2 u[16];   // columns 0 .. 15
#pragma unroll
                        for (int q2 = 0; q2 < 8; ++q2) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 2 * AL_BK * P2 + 2 * q2);
                            u[2 * q2] = make_float2(x.x, x.y);
                            u[2 * q2 + 1] = make_float2(x.z, x.w);
                        }
                        float2 s7 = add2(add2(add2(u[1], u[2]), add2(u[3], u[4])), add2(add2(u[5], u[6]), u[7]));
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s7 = add2(s7, sub2(u[x + 7], u[x]));
                            if (MIN3) {
                                r7[x] = mul2(s7, make_float2(81.0f / 49.0f, 81.0f / 49.0f));
                            } else if (ALL4) {
                                const float2 r = mul2(s7, make_float2(81.0f / 49.0f, 81.0f / 49.0f));
                                m[x] = make_float2(fminf(m[x].x, r.x), fminf(m[x].y, r.y));
                            } else if (wm & 4) {
                                const float2 r = mul2(s7, c_al_w[2]);
                                m[x] = make_float2(fminf(m[x].x, r.x), fminf(m[x].y, r.y));
                            }
                        }
                    }
                    {
                        float2 u[16];   // columns 0 .. 15
#pragma unroll
                        for (int q2 = 0; q2 < 8; ++q2) {
                            const float4 x = *reinterpret_cast<const float4*>(base + 3 * AL_BK * P2 + 2 * q2);
                            u[2 * q2] = make_float2(x.x, x.y);
                            u[2 * q2 + 1] = make_float2(x.z, x.w);
                        }
                        float2 s9 = add2(add2(add2(add2(u[0], u[1]), add2(u[2], u[3])), add2(add2(u[4], u[5]), add2(u[6], u[7]))), u[8]);
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            if (x > 0) s9 = add2(s9, sub2(u[x + 8], u[x - 1]));
                            if (MIN3) {   // FMNMX3 per lane
                                m[x] = make_float2(fminf(fminf(m[x].x, r7[x].x), s9.x), fminf(fminf(m[x].y, r7[x].y), s9.y));
                            } else if (ALL4) {
                                m[x] = make_float2(fminf(m[x].x, s9.x), fminf(m[x].y, s9.y));
                            } else if (wm & 8) {
                                const float2 r = mul2(s9, c_al_w[3]);
                                m[x] = make_float2(fminf(m[x].x, r.x), fminf(m[x].y, r.y));
                            }
                        }
                    }
                    float oa[8], od[8];
#pragma unroll
                    for (int q2 = 0; q2 < 4; ++q2) {
                        const float4 x = *reinterpret_cast<const float4*>(base + 4 * AL_BK * P2 + 4 + 2 * q2);
                        const float2 cs = ALL4 ? c81p : s0p;
                        const float2 th = ALL4 ? t81p : make_float2(s0, s0);
                        const float2 c0 = mul2(make_float2(x.x, x.y), cs), c1 = mul2(make_float2(x.z, x.w), cs);
                        oa[2 * q2] = c0.x * al_rcp(fmaxf(m[2 * q2].x, th.x));
                        od[2 * q2] = c0.y * al_rcp(fmaxf(m[2 * q2].y, th.y));
                        oa[2 * q2 + 1] = c1.x * al_rcp(fmaxf(m[2 * q2 + 1].x, th.x));
                        od[2 * q2 + 1] = c1.y * al_rcp(fmaxf(m[2 * q2 + 1].y, th.y));
                    }
                    float* arow = a.d1 + roff;
                    float* drow = a.d2 + roff;
                    if (hfull) {
                        st_global_v8(arow, oa);
                        st_global_v8(drow, od);
                    } else {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if (hx + x < a.nW) {
                                arow[x] = oa[x];
                                drow[x] = od[x];
                            }
                    }
                }
            };
            if (SPLITV) {
                __syncthreads();   // B2: every thread is done reading the row buffer (inside the V buffer)
                PRNU_STRESS(3);
                write_pair();
                __syncthreads();   // B3: (ad, dd) V/c ready
                PRNU_STRESS(4);
                if (hon) h_pair();
                __syncthreads();   // B3b: (ad, dd) planes consumed
                PRNU_STRESS(6);
                write_da();
                __syncthreads();   // B3c: da V/c ready
                PRNU_STRESS(7);
                if (hon) h_da();
            } else {
                write_pair();      // (the (ad, dd) planes do not overlap the row buffer)
                __syncthreads();   // B2: every thread is done reading the row buffer (overlaps the da planes)
                PRNU_STRESS(3);
                write_da();
                __syncthreads();   // B3: V/c of all three subbands ready
                PRNU_STRESS(4);
                if (hon) {
                    h_da();
                    h_pair();
                }
            }
        }
        __syncthreads();   // B4: V buffers and the row buffer free for the next block
        PRNU_STRESS(5);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            qd_c[k] = qd[8 + k];
            qp_c[k] = qp[8 + k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {   // c of rows K+4 .. K+7 (output rows of the next block)
            cd_c[k] = cn[4 + k];
            cp_c[k] = cpn[4 + k];
        }
    }
}

// ------------------------------------------------------------------ host

template <typename T>
static int lift_launch(const typename AlCfg<T>::E* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll, float* d0,
                       float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                       const ShrinkParams& sp, const SdaDiv& div, int nb, cudaStream_t st) {
    static DeviceFlags done[2];
    int rc;
    if ((rc = set_smem_attr((const void*)k_analysis_lift<T, AlCfg<T>::MINB, true>, al_smem_bytes<T>(), done[0])))
        return rc;
    if ((rc = set_smem_attr((const void*)k_analysis_lift<T, AlCfg<T>::MINB, false>, al_smem_bytes<T>(), done[1])))
        return rc;
    if (nb > 65535) return fail(PRNU_INVALID_ARG, "analysis: more than 65535 planes in one launch");
    // the H pass stores 8 outputs per thread with one 256-bit store: 32-byte aligned subband rows
    if ((((uintptr_t)d0 | (uintptr_t)d1 | (uintptr_t)d2) & 31) || (out_pitch & 7) || (out_bstride & 7))
        return fail(PRNU_INVALID_ARG, "analysis: subband planes must have 32-byte aligned rows");
    AlArgs a{};
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
    a.div_d = div.d;
    a.div_r = div.r;
    const int S0 = (nW + AlCfg<T>::OMAX - 1) / AlCfg<T>::OMAX;
    a.O = (int)align_up((size_t)((nW + S0 - 1) / S0), 8);
    const int S = (nW + a.O - 1) / a.O;
    // segments of <= 300 rows (prologue overhead <= 3%), more of them while the grid holds
    // fewer than 6 (u8, level 1) / 1 (fp32) waves of MINB CTAs per SM
    const long long waves = sizeof(typename AlCfg<T>::E) == 1 ? 6 : 1;
    const long long slots = (long long)device_sm_count() * AlCfg<T>::MINB;
    int nseg = (nH + 299) / 300;
    while ((long long)S * nseg * nb < waves * slots && (nH + nseg) / (nseg + 1) >= 32) ++nseg;
    a.SH = (int)align_up((size_t)((nH + nseg - 1) / nseg), 8);
    nseg = (nH + a.SH - 1) / a.SH;
    CUtensorMap map{};
    constexpr int DEP = AlCfg<T>::DEP;
    const size_t es = sizeof(typename AlCfg<T>::E);
    const CUtensorMapDataType dt = es == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    a.use_tma = ((in_pitch * es) % 16 == 0) && ((in_bstride * es) % 16 == 0) && ((uintptr_t)in % 16 == 0) &&
                encode_tensor_map_3d(&map, dt, es, in, (uint64_t)NW, (uint64_t)NH, (uint64_t)nb * DEP,
                                     (uint64_t)in_pitch * es, (uint64_t)in_bstride * es, AlCfg<T>::BOXW, AL_IR, DEP);
    // pairs: in_bstride is the frame stride, group b = frames DEP b, DEP b + 1 (TMA only, >= 32 rows)
    if (DEP != 1 && (!a.use_tma || NH < 32)) return fail(PRNU_INVALID_ARG, "analysis: SDA pairs need TMA-stageable frames");
    dim3 grid(S, nseg, nb);
    if (sp.wmask == 15)
        k_analysis_lift<T, AlCfg<T>::MINB, true><<<grid, AL_NT, al_smem_bytes<T>(), st>>>(map, a);
    else
        k_analysis_lift<T, AlCfg<T>::MINB, false><<<grid, AL_NT, al_smem_bytes<T>(), st>>>(map, a);
    return PRNU_OK;
}

int launch_analysis_lift_u8(const uint8_t* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                            float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                            const ShrinkParams& sp, int nb, cudaStream_t st) {
    return lift_launch<uint8_t>(in, in_bstride, in_pitch, NH, NW, ll, d0, d1, d2, out_bstride, out_pitch, nH, nW, sp,
                                SdaDiv{}, nb, st);
}
int launch_analysis_lift_u16(const uint16_t* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                             float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                             const ShrinkParams& sp, const SdaDiv& div, int nb, cudaStream_t st) {
    return lift_launch<uint16_t>(in, in_bstride, in_pitch, NH, NW, ll, d0, d1, d2, out_bstride, out_pitch, nH, nW,
                                 sp, div, nb, st);
}
int launch_analysis_lift_pair(const uint8_t* in, long long frame_stride, int in_pitch, int NH, int NW, float* ll,
                              float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                              const ShrinkParams& sp, int nb, cudaStream_t st) {
    return lift_launch<u8pair>(in, frame_stride, in_pitch, NH, NW, ll, d0, d1, d2, out_bstride, out_pitch, nH, nW, sp,
                               SdaDiv{}, nb, st);
}
int launch_analysis_lift_f32(const float* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll,
                             float* d0, float* d1, float* d2, long long out_bstride, int out_pitch, int nH, int nW,
                             const ShrinkParams& sp, int nb, cudaStream_t st) {
    return lift_launch<float>(in, in_bstride, in_pitch, NH, NW, ll, d0, d1, d2, out_bstride, out_pitch, nH, nW, sp,
                              SdaDiv{}, nb, st);
}

}  // namespace prnu
