// wavelet.cu — the denoiser F of the SDA/PRNU hot path on sm_100a.
//
// a2+a3  k_analysis_shrink : one DWT level (rows then columns, R-6) of a tile
//        of 32x32 subband coefficients plus a 4-coefficient halo, computed in
//        shared memory from a mirrored input tile (R-4), followed by the local
//        variance MAP/Wiener shrink of the three detail subbands (R-7)
//        on the same tile.  Writes the approximation (for the next level) and
//        the NOISE-DOMAIN details c * sigma0^2 / (v + sigma0^2) = c - F(c).
// a4     k_synthesis       : one inverse level (columns then rows) in the
//        noise domain (approximation of the coarsest level = 0, R-10).
// a4+a5  k_synthesis_accumulate : the last inverse level fused with the MLE
//        accumulation (Eq. 2, P:151-155 / P:200-203): one CTA owns a pixel
//        tile for every frame of the batch and adds W*I and I^2 to registers
//        in ascending frame order, so NUM/DEN are read and written once per
//        batch and the per-pixel summation order is the sequential one.
//
// Filters are compile-time immediates (FFMA-imm).  fp32 arithmetic; the
// accumulators are fp64.
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace prnu {

// ============================================================== analysis
// Tile: AT x AT output coefficients per subband, computed over an AR x AR
// region (halo kHalo for the 9x9 windows) from an AIN x AIN input tile.
constexpr int AT = 32;                  // output coefficient tile (square)
#ifndef PRNU_ANALYSIS_THREADS
#define PRNU_ANALYSIS_THREADS 256
#endif
constexpr int A_NT = PRNU_ANALYSIS_THREADS;   // threads per analysis CTA (8 warps x 4 CTAs/SM: measured best, profiles/r01)
constexpr int A_NW = A_NT / 32;
constexpr int AR = AT + 2 * kHalo;      // 40: computed coefficient region
constexpr int AIN = 2 * AR + 6;         // 86: input rows / columns of the region
constexpr int IN_P = 92;                // input tile pitch (== 28 mod 32: conflict-free LDS.128, row-major lanes)
constexpr int RW_P = 44;                // row-pass plane pitch (== 12 mod 32)
constexpr int RW_PLANE = AIN * RW_P + 48;   // one row-pass plane incl. the row-block skew (<= 8*5)
constexpr int DT_P = AR + 1;            // detail plane pitch (odd: conflict-free column walks)
constexpr int V_P4 = AR + 1;            // vertical-sum plane pitch in float4 (41*4 == 4 mod 32)
constexpr int V_PLANE4 = AT * V_P4;     // float4 per vertical-sum buffer
constexpr int A_SMEM_IN = AIN * IN_P;             // input tile; later the 3 detail planes
constexpr int A_SMEM_ROW = 2 * V_PLANE4 * 4;      // row-pass lo/hi; later two vertical-sum buffers
static_assert(3 * AR * DT_P <= A_SMEM_IN, "detail planes must fit in the input tile");
static_assert(2 * RW_PLANE <= A_SMEM_ROW, "row-pass planes must fit");

// Row r of a row-pass plane starts at r*RW_P plus a skew of 8 floats per block
// of 16 rows (monotonic: rows never overlap), so column walks of different row groups (16 rows apart) fall in
// different banks; the 16-byte alignment of row-pass stores is kept.
__device__ __forceinline__ int rw_off(int r) { return r * RW_P + 8 * (r >> 4); }

struct AnalysisArgs {
    const void* in;
    long long in_bstride;   // elements between frames
    int in_pitch;           // elements per row
    int NH, NW;             // input plane size
    float* ll;              // approximation out (nullable: coarsest level)
    float* d0;              // da = lo_y(hi_x)
    float* d1;              // ad = hi_y(lo_x)
    float* d2;              // dd = hi_y(hi_x)
    long long out_bstride;
    int out_pitch;
    int nH, nW;             // subband size
    ShrinkParams sp;
};

// Filter pairs in constant memory: FFMA2 takes them as c[][] / uniform-register
// operands instead of re-materialising immediate pairs with MOVs at every use.
__constant__ float2 c_hg[8] = {{PRNU_H0, PRNU_H7}, {PRNU_H1, -PRNU_H6}, {PRNU_H2, PRNU_H5}, {PRNU_H3, -PRNU_H4},
                               {PRNU_H4, PRNU_H3}, {PRNU_H5, -PRNU_H2}, {PRNU_H6, PRNU_H1}, {PRNU_H7, -PRNU_H0}};
// synthesis: (H(6-2m), H(7-2m)) and (G(6-2m), G(7-2m)), m = 0..3
__constant__ float2 c_sh[4] = {{PRNU_H6, PRNU_H7}, {PRNU_H4, PRNU_H5}, {PRNU_H2, PRNU_H3}, {PRNU_H0, PRNU_H1}};
__constant__ float2 c_sg[4] = {{PRNU_H1, -PRNU_H0}, {PRNU_H3, -PRNU_H2}, {PRNU_H5, -PRNU_H4}, {PRNU_H7, -PRNU_H6}};

// Analysis (lo, hi) tap pairs: immediates (default) or constant-memory pairs.
// (immediates measured faster than constant-memory pairs in this kernel, profiles/r01)
#ifdef PRNU_HG_CONST
#define PRNU_HG(i) c_hg[i]
#else
#define PRNU_HG(i) make_float2(wl_h(i), wl_g(i))
#endif

// Geometry of one analysis tile.
struct ATile {
    int b, y0, x0, cy0, cx0;
    bool bx, by;   // the window region crosses a subband border (mirrored reads)
};

__device__ __forceinline__ ATile analysis_tile(const AnalysisArgs& a, int b, int ty, int tx) {
    ATile g;
    g.b = b;
    g.y0 = ty * AT;
    g.x0 = tx * AT;
    g.cy0 = g.y0 - kHalo;
    g.cx0 = g.x0 - kHalo;
    g.bx = (g.cx0 < 0) || (g.cx0 + AR > a.nW);
    g.by = (g.cy0 < 0) || (g.cy0 + AR > a.nH);
    return g;
}

// Mirror tables of a tile (R-4): input rows/cols of the AIN x AIN tile and the
// region rows/cols the shrink windows read.  Window rows/cols of every output
// inside the plane mirror into the region; indices that only feed discarded
// outputs (beyond the plane) are clamped.  Caller synchronises.
__device__ __forceinline__ void analysis_tables(const AnalysisArgs& a, const ATile& g, int* s_iy, int* s_ix,
                                                int* s_rmap, int* s_cmap, int tid = threadIdx.x, int nthr = A_NT) {
    for (int i = tid; i < AIN; i += nthr) {
        s_iy[i] = mirror(2 * g.cy0 - 6 + i, a.NH);
        s_ix[i] = mirror(2 * g.cx0 - 6 + i, a.NW);
    }
    for (int i = tid; i < AR; i += nthr) {
        const int mr = mirror(g.cy0 + i, a.nH) - g.cy0;
        const int mc = mirror(g.cx0 + i, a.nW) - g.cx0;
        s_rmap[i] = (mr >= 0 && mr < AR) ? mr : i;
        s_cmap[i] = (mc >= 0 && mc < AR) ? mc : i;
    }
}

// Row pass (along x) of the 8 coefficient columns 8cg..8cg+7 of input row r,
// from 24 consecutive input values v (only v[0..21] contribute).
__device__ __forceinline__ void rowpass_item(const float (&v)[24], float* s_row, int r, int cg) {
    float lo[8], hi[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        float2 lh = fmul2s(v[2 * q], PRNU_HG(0));   // (lo, hi) in one FFMA2 per tap
#pragma unroll
        for (int i = 1; i < 8; ++i) lh = ffma2(v[2 * q + i], PRNU_HG(i), lh);
        lo[q] = lh.x;
        hi[q] = lh.y;
    }
    float4* dl = reinterpret_cast<float4*>(s_row + rw_off(r) + 8 * cg);
    float4* dh = reinterpret_cast<float4*>(s_row + RW_PLANE + rw_off(r) + 8 * cg);
    dl[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
    dl[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
    dh[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
    dh[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
}

// fp32 input tile [AIN][IN_P]: item = (row, 8 coefficient columns), 6 LDS.128
__device__ __forceinline__ void rowpass_f32(const float* s_in, float* s_row, int tid = threadIdx.x,
                                            int nthr = A_NT) {
    for (int it = tid; it < AIN * (AR / 8); it += nthr) {
        const int r = it % AIN, cg = it / AIN;
        const float4* src = reinterpret_cast<const float4*>(s_in + r * IN_P + 16 * cg);
        float v[24];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const float4 t = src[k];
            v[4 * k] = t.x;
            v[4 * k + 1] = t.y;
            v[4 * k + 2] = t.z;
            v[4 * k + 3] = t.w;
        }
        rowpass_item(v, s_row, r, cg);
    }
}

// u8 input tile [AIN][U8_P] bytes: one LDS.128 + one LDS.64 per item; bytes are
// widened exactly with the 2^23 trick: float(0x4B0000bb) - 2^23 = bb.
constexpr int U8_P = 112;   // 28 words == 28 mod 32: conflict-free LDS.128 for row-major lanes
__device__ __forceinline__ float u8_to_f32(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | (uint32_t)k)) - 8388608.0f;
}
// The u8 tile row starts U8_OFF bytes before input column 2*cx0-6: u8 TMA boxes
// must start on a 16-byte boundary (measured: other x offsets fault).
constexpr int U8_OFF = 2;
__device__ __forceinline__ void rowpass_u8(const uint8_t* s_in8, float* s_row, int tid = threadIdx.x,
                                           int nthr = A_NT) {
    for (int it = tid; it < AIN * (AR / 8); it += nthr) {
        const int r = it % AIN, cg = it / AIN;
        const uint8_t* src = s_in8 + r * U8_P + 16 * cg;
        const uint4 w0 = *reinterpret_cast<const uint4*>(src);
        const uint2 w1 = *reinterpret_cast<const uint2*>(src + 16);
        const uint32_t w[6] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y};
        float v[24];
#pragma unroll
        for (int k = 0; k < 22; ++k) v[k] = u8_to_f32(w[(k + U8_OFF) >> 2], (k + U8_OFF) & 3);
        v[22] = v[23] = 0.f;
        rowpass_item(v, s_row, r, cg);
    }
}

// Column pass (along y): 4 subbands for the AR x AR region; item = (column,
// 8 coefficient rows) from 22 rows of lo and hi.  Details -> s_det, the inner
// approximation -> global (next level's input).
__device__ __forceinline__ void colpass(const AnalysisArgs& a, const ATile& g, const float* s_row, float* s_det,
                                        int tid = threadIdx.x, int nthr = A_NT) {
    for (int it = tid; it < AR * (AR / 8); it += nthr) {
        // warps cover 32 consecutive columns of one row group (no bank-shifted wrap)
        const int c = it < 32 * (AR / 8) ? (it & 31) : 32 + ((it - 32 * (AR / 8)) % (AR - 32));
        const int rg = it < 32 * (AR / 8) ? (it >> 5) : (it - 32 * (AR / 8)) / (AR - 32);
        float lo[22], hi[22];
        // rw_off(16 rg + k) = (16 RW_P + 8) rg + RW_P k + 8 (k >> 4) for k < 32
        const float* lo_base = s_row + (16 * RW_P + 8) * rg + c;
#pragma unroll
        for (int k = 0; k < 22; ++k) {
            lo[k] = lo_base[RW_P * k + 8 * (k >> 4)];
            hi[k] = lo_base[RW_PLANE + RW_P * k + 8 * (k >> 4)];
        }
        const bool inner_c = (c >= kHalo) && (c < kHalo + AT) && (g.x0 + c - kHalo < a.nW);
        // approximation of region row rr goes to plane row y0 + rr - kHalo
        float* llc = a.ll ? a.ll + (size_t)g.b * a.out_bstride + (ptrdiff_t)(g.y0 - kHalo) * a.out_pitch + g.x0 + c -
                                kHalo
                          : nullptr;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float2 p_l = fmul2s(lo[2 * q], PRNU_HG(0)), p_h = fmul2s(hi[2 * q], PRNU_HG(0));   // (aa, ad), (da, dd)
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                p_l = ffma2(lo[2 * q + i], PRNU_HG(i), p_l);
                p_h = ffma2(hi[2 * q + i], PRNU_HG(i), p_h);
            }
            const float aa = p_l.x, ad = p_l.y, da = p_h.x, dd = p_h.y;
            const int rr = 8 * rg + q;
            s_det[0 * AR * DT_P + rr * DT_P + c] = da;
            s_det[1 * AR * DT_P + rr * DT_P + c] = ad;
            s_det[2 * AR * DT_P + rr * DT_P + c] = dd;
            if (llc != nullptr && inner_c && rr >= kHalo && rr < kHalo + AT && g.y0 + rr - kHalo < a.nH)
                llc[(ptrdiff_t)rr * a.out_pitch] = aa;
        }
    }
}

// Shrink of the three detail subbands (R-7): separable window sums of
// c^2 — vertical (per column, 8 rows per item, nested 3/5/7/9) into a float4
// plane, then horizontal (per row, 8 columns per item, sliding sums) — and the
// Wiener factor; writes the noise-domain coefficients c sigma0^2/(v+sigma0^2).
// Two vertical-sum buffers pipeline the subbands: phases V0 | H0+V1 | H1+V2 | H2.
// Starts after a barrier that made s_det complete; ends with a barrier.
template <bool BY>
__device__ __forceinline__ void shrink_v_t(const ATile& g, const float* det, float4* s_v, const int* s_rmap,
                                           const int* s_cmap, int it) {
    const int x = it < 32 * (AT / 8) ? (it & 31) : 32 + ((it - 32 * (AT / 8)) % (AR - 32));
    const int ig = it < 32 * (AT / 8) ? (it >> 5) : (it - 32 * (AT / 8)) / (AR - 32);
    if (g.bx && s_cmap[x] != x) return;
    float q[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int rr = BY ? s_rmap[8 * ig + k] : 8 * ig + k;
        const float c = det[rr * DT_P + x];
        q[k] = __fmul_rn(c, c);   // no contraction into the sums: identical in every kernel
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const float v3 = q[t + 3] + q[t + 4] + q[t + 5];
        const float v5 = v3 + q[t + 2] + q[t + 6];
        const float v7 = v5 + q[t + 1] + q[t + 7];
        const float v9 = v7 + q[t] + q[t + 8];
        s_v[(8 * ig + t) * V_P4 + x] = make_float4(v3, v5, v7, v9);
    }
}

__device__ __forceinline__ void shrink_v(const ATile& g, const float* det, float4* s_v, const int* s_rmap,
                                         const int* s_cmap, int it) {
    if (g.by) shrink_v_t<true>(g, det, s_v, s_rmap, s_cmap, it);
    else shrink_v_t<false>(g, det, s_v, s_rmap, s_cmap, it);
}

template <bool BX, bool ALL4>
__device__ __forceinline__ void shrink_h_t(const AnalysisArgs& a, const ATile& g, const float* det,
                                           const float4* s_v, const int* s_cmap, float* dst, int it) {
    const float s0 = a.sp.sigma0_sq;
    const int wm = a.sp.wmask;
    const int i = it % AT, jg = it / AT;
    const int gy = g.y0 + i;
    float4 u[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int xx = BX ? s_cmap[8 * jg + k] : 8 * jg + k;
        u[k] = s_v[i * V_P4 + xx];
    }
    const float* crow = det + (i + kHalo) * DT_P + 8 * jg + kHalo;
    float s3 = u[3].x + u[4].x + u[5].x;
    float s5 = u[2].y + u[3].y + u[4].y + u[5].y + u[6].y;
    float s7 = u[1].z + u[2].z + u[3].z + u[4].z + u[5].z + u[6].z + u[7].z;
    float s9 = u[0].w + u[1].w + u[2].w + u[3].w + u[4].w + u[5].w + u[6].w + u[7].w + u[8].w;
    float o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        if (t > 0) {   // slide the windows one column right
            s3 += u[t + 5].x - u[t + 2].x;
            s5 += u[t + 6].y - u[t + 1].y;
            s7 += u[t + 7].z - u[t].z;
            s9 += u[t + 8].w - u[t - 1].w;
        }
        float m;
        if (ALL4) {   // the default window set {3,5,7,9}: no per-window selects
            m = fminf(fminf(s3 * (1.0f / 9.0f), s5 * (1.0f / 25.0f)), fminf(s7 * (1.0f / 49.0f), s9 * (1.0f / 81.0f)));
        } else {
            m = 3.402823466e38f;
            if (wm & 1) m = fminf(m, s3 * (1.0f / 9.0f));
            if (wm & 2) m = fminf(m, s5 * (1.0f / 25.0f));
            if (wm & 4) m = fminf(m, s7 * (1.0f / 49.0f));
            if (wm & 8) m = fminf(m, s9 * (1.0f / 81.0f));
        }
        // noise-domain coefficient c - F(c) = c s0 / (max(m - s0, 0) + s0) = c s0 / max(m, s0)
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(m, s0)));
        o[t] = crow[t] * s0 * r;
    }
    if (gy < a.nH) {
        const int gx = g.x0 + 8 * jg;
        float* drow = dst + (size_t)gy * a.out_pitch + gx;
        if (gx + 8 <= a.nW) {
            reinterpret_cast<float4*>(drow)[0] = make_float4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<float4*>(drow)[1] = make_float4(o[4], o[5], o[6], o[7]);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (gx + t < a.nW) drow[t] = o[t];
        }
    }
}

__device__ __forceinline__ void shrink_h(const AnalysisArgs& a, const ATile& g, const float* det, const float4* s_v,
                                         const int* s_cmap, float* dst, int it) {
    const bool all4 = a.sp.wmask == 15;
    if (g.bx) {
        if (all4) shrink_h_t<true, true>(a, g, det, s_v, s_cmap, dst, it);
        else shrink_h_t<true, false>(a, g, det, s_v, s_cmap, dst, it);
    } else {
        if (all4) shrink_h_t<false, true>(a, g, det, s_v, s_cmap, dst, it);
        else shrink_h_t<false, false>(a, g, det, s_v, s_cmap, dst, it);
    }
}

// CTA-wide barrier, or a named barrier over a warp group (bar.sync id, count).
struct CtaBar {
    __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct NamedBar {
    int id, count;
    __device__ __forceinline__ void sync() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
    }
};

template <class Bar>
__device__ __forceinline__ void shrink3(const AnalysisArgs& a, const ATile& g, const float* s_det, float4* s_v,
                                        const int* s_rmap, const int* s_cmap, Bar bar, int tid = threadIdx.x,
                                        int nthr = A_NT) {
    constexpr int VI = AR * (AT / 8);   // 160 vertical items per subband
    constexpr int HI = AT * (AT / 8);   // 128 horizontal items per subband
    for (int it = tid; it < VI; it += nthr) shrink_v(g, s_det, s_v, s_rmap, s_cmap, it);
    bar.sync();
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
        // H of subband s (buffer s&1) together with V of subband s+1 (buffer (s+1)&1)
        const int n = HI + (s < 2 ? VI : 0);
        for (int it = tid; it < n; it += nthr) {
            if (it < HI)
                shrink_h(a, g, s_det + s * AR * DT_P, s_v + (s & 1) * V_PLANE4, s_cmap,
                         (s == 0 ? a.d0 : s == 1 ? a.d1 : a.d2) + (size_t)g.b * a.out_bstride, it);
            else
                shrink_v(g, s_det + (s + 1) * AR * DT_P, s_v + ((s + 1) & 1) * V_PLANE4, s_rmap, s_cmap, it - HI);
        }
        bar.sync();
    }
}

// One vertical-sum buffer: V0 | H0 | V1 | H1 | V2 | H2 (smaller footprint).
__device__ __forceinline__ void shrink3_single(const AnalysisArgs& a, const ATile& g, const float* s_det, float4* s_v,
                                               const int* s_rmap, const int* s_cmap, int tid = threadIdx.x,
                                               int nthr = A_NT) {
    constexpr int VI = AR * (AT / 8);
    constexpr int HI = AT * (AT / 8);
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
        for (int it = tid; it < VI; it += nthr) shrink_v(g, s_det + s * AR * DT_P, s_v, s_rmap, s_cmap, it);
        __syncthreads();
        for (int it = tid; it < HI; it += nthr)
            shrink_h(a, g, s_det + s * AR * DT_P, s_v, s_cmap,
                     (s == 0 ? a.d0 : s == 1 ? a.d1 : a.d2) + (size_t)g.b * a.out_bstride, it);
        __syncthreads();
    }
}

__device__ __forceinline__ bool fast_f32(const AnalysisArgs& a, const ATile& g);

// Input tile of one analysis tile into s_in [AIN][IN_P] (fp32), by NWARPS warps
// (warp = 0..NWARPS-1).  Interior u8 tiles: each row is 22 aligned words covering
// input columns ix0-2 .. ix0+85, widened exactly (2^23 trick); otherwise mirrored
// element loads via the tables (which the caller computed and synchronised).
// Returns nothing; the caller synchronises before the row pass.
template <typename TIn, int NWARPS>
__device__ __forceinline__ void load_tile(const AnalysisArgs& a, const ATile& g, bool fast_u8, float* s_in,
                                          const int* s_iy, const int* s_ix, int warp, int lane) {
    const TIn* in = reinterpret_cast<const TIn*>(a.in) + (size_t)g.b * a.in_bstride;
    constexpr int RPW = (AIN + NWARPS - 1) / NWARPS;   // rows per warp
    if (fast_u8) {
        const int ix0 = 2 * g.cx0 - 6, iy0 = 2 * g.cy0 - 6;
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(in) +
                                                               (size_t)(iy0 + warp) * a.in_pitch + ix0 - 2) +
                             min(lane, 21);
        const size_t wstep = (size_t)NWARPS * a.in_pitch / 4;   // NWARPS rows, in 32-bit words
        uint32_t wv[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) wv[k] = (warp + NWARPS * k < AIN) ? __ldg(wp + k * wstep) : 0u;
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int r = warp + NWARPS * k;
            if (r < AIN && lane < 22) {
                const int c0 = 4 * lane - 2;   // tile column of byte 0
                const float f0 = __uint_as_float(__byte_perm(wv[k], 0x4B000000u, 0x7540u)) - 8388608.0f;
                const float f1 = __uint_as_float(__byte_perm(wv[k], 0x4B000000u, 0x7541u)) - 8388608.0f;
                const float f2 = __uint_as_float(__byte_perm(wv[k], 0x4B000000u, 0x7542u)) - 8388608.0f;
                const float f3 = __uint_as_float(__byte_perm(wv[k], 0x4B000000u, 0x7543u)) - 8388608.0f;
                float* row = s_in + r * IN_P;
                if (lane > 0) *reinterpret_cast<float2*>(row + c0) = make_float2(f0, f1);
                *reinterpret_cast<float2*>(row + c0 + 2) = make_float2(f2, f3);   // c0 + 3 <= 85
            }
        }
    } else if (sizeof(TIn) == 4 && fast_f32(a, g)) {
        // interior fp32 tile: each row is 43 aligned float2 (input columns ix0 .. ix0+85)
        const int ix0 = 2 * g.cx0 - 6, iy0 = 2 * g.cy0 - 6;
        const float2* rp = reinterpret_cast<const float2*>(reinterpret_cast<const float*>(in) +
                                                           (size_t)(iy0 + warp) * a.in_pitch + ix0);
        const size_t rstep = (size_t)NWARPS * a.in_pitch / 2;   // NWARPS rows, in float2
        float2 v0[RPW], v1[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const bool ok = warp + NWARPS * k < AIN;
            v0[k] = ok ? __ldg(rp + k * rstep + lane) : make_float2(0.f, 0.f);
            v1[k] = (ok && lane < AIN / 2 - 32) ? __ldg(rp + k * rstep + 32 + lane) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int r = warp + NWARPS * k;
            if (r < AIN) {
                float2* row = reinterpret_cast<float2*>(s_in + r * IN_P);
                row[lane] = v0[k];
                if (lane < AIN / 2 - 32) row[32 + lane] = v1[k];
            }
        }
    } else {
        float v[RPW][3];
        int ixs[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) ixs[j] = s_ix[min(lane + 32 * j, AIN - 1)];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const TIn* row = in + (size_t)s_iy[min(warp + NWARPS * k, AIN - 1)] * a.in_pitch;
#pragma unroll
            for (int j = 0; j < 3; ++j) v[k][j] = (float)__ldg(row + ixs[j]);
        }
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int r = warp + NWARPS * k;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int c = lane + 32 * j;
                if (r < AIN && c < AIN) s_in[r * IN_P + c] = v[k][j];
            }
        }
    }
}

// interior fp32 tile whose rows can be read as aligned float2 (no mirroring)
__device__ __forceinline__ bool fast_f32(const AnalysisArgs& a, const ATile& g) {
    const int ix0 = 2 * g.cx0 - 6, iy0 = 2 * g.cy0 - 6;
    const float* in = reinterpret_cast<const float*>(a.in) + (size_t)g.b * a.in_bstride;
    return ix0 >= 0 && iy0 >= 0 && ix0 + AIN <= a.NW && iy0 + AIN <= a.NH && (ix0 & 1) == 0 &&
           (a.in_pitch & 1) == 0 && ((reinterpret_cast<uintptr_t>(in) & 7) == 0);
}

template <typename TIn>
__device__ __forceinline__ bool tile_fast_u8(const AnalysisArgs& a, const ATile& g) {
    const TIn* in = reinterpret_cast<const TIn*>(a.in) + (size_t)g.b * a.in_bstride;
    const int ix0 = 2 * g.cx0 - 6, iy0 = 2 * g.cy0 - 6;
    return sizeof(TIn) == 1 && ix0 >= 2 && iy0 >= 0 && ix0 - 2 + 88 <= a.NW && iy0 + AIN <= a.NH &&
           ((reinterpret_cast<uintptr_t>(in) + (size_t)ix0 - 2) & 3) == 0 && (a.in_pitch & 3) == 0;
}

// Generic analysis kernel: one tile per CTA.
// u8 input tile kept as bytes [AIN][U8_P] (row = input columns 2*cx0-6-U8_OFF ..):
// interior tiles store the 22 aligned words of each row as loaded (one STS.32
// per lane); border tiles store mirrored bytes through the tables.
template <int NWARPS>
__device__ __forceinline__ void load_tile_u8(const AnalysisArgs& a, const ATile& g, bool fast_u8, uint8_t* s_in8,
                                             const int* s_iy, const int* s_ix, int warp, int lane) {
    const uint8_t* in = reinterpret_cast<const uint8_t*>(a.in) + (size_t)g.b * a.in_bstride;
    constexpr int RPW = (AIN + NWARPS - 1) / NWARPS;
    if (fast_u8) {
        const int ix0 = 2 * g.cx0 - 6, iy0 = 2 * g.cy0 - 6;
        const uint32_t* wp =
            reinterpret_cast<const uint32_t*>(in + (size_t)(iy0 + warp) * a.in_pitch + ix0 - U8_OFF) + min(lane, 21);
        const size_t wstep = (size_t)NWARPS * a.in_pitch / 4;
        uint32_t wv[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) wv[k] = (warp + NWARPS * k < AIN) ? __ldg(wp + k * wstep) : 0u;
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int r = warp + NWARPS * k;
            if (r < AIN && lane < 22) reinterpret_cast<uint32_t*>(s_in8 + r * U8_P)[lane] = wv[k];
        }
    } else {
        uint8_t v[RPW][3];
        int ixs[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) ixs[j] = s_ix[min(lane + 32 * j, AIN - 1)];
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const uint8_t* row = in + (size_t)s_iy[min(warp + NWARPS * k, AIN - 1)] * a.in_pitch;
#pragma unroll
            for (int j = 0; j < 3; ++j) v[k][j] = __ldg(row + ixs[j]);
        }
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int r = warp + NWARPS * k;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int c = lane + 32 * j;
                if (r < AIN && c < AIN) s_in8[r * U8_P + U8_OFF + c] = v[k][j];
            }
        }
    }
}

// Shared-memory layout of the generic analysis kernel per input type: the
// input tile (fp32 [AIN][IN_P], or u8 [AIN][U8_P] bytes when PRNU_U8_FLOAT_TILE
// is not set) later holds the detail planes; the row-pass planes later hold the
// vertical-sum buffer(s).
#ifndef PRNU_U8_FLOAT_TILE
constexpr bool kU8Bytes = true;
#else
constexpr bool kU8Bytes = false;
#endif
#ifdef PRNU_DOUBLE_V
constexpr bool kDoubleV = true;    // two vertical-sum buffers (pipelined V/H phases, 3 CTAs/SM)
#else
constexpr bool kDoubleV = false;   // one buffer: u8 kernel fits 4 CTAs/SM (measured faster)
#endif
template <typename TIn>
__host__ __device__ constexpr int a_in_floats() {
    return (sizeof(TIn) == 1 && kU8Bytes) ? (3 * AR * DT_P > (AIN * U8_P + 3) / 4 ? 3 * AR * DT_P : (AIN * U8_P + 3) / 4)
                                          : A_SMEM_IN;
}
__host__ __device__ constexpr int a_row_floats() {
    return kDoubleV ? A_SMEM_ROW : (2 * RW_PLANE > V_PLANE4 * 4 ? 2 * RW_PLANE : V_PLANE4 * 4);
}
template <typename TIn>
constexpr size_t a_smem_bytes() {
    return sizeof(float) * (a_in_floats<TIn>() + a_row_floats()) + sizeof(int) * (2 * AIN + 2 * AR);
}
#ifndef PRNU_ANALYSIS_MINB
#define PRNU_ANALYSIS_MINB 4
#endif

template <typename TIn>
__global__ void __launch_bounds__(A_NT, PRNU_ANALYSIS_MINB) k_analysis_shrink(AnalysisArgs a) {
    extern __shared__ __align__(128) float smem[];
    float* s_in = smem;                              // input tile; later details [3][AR][DT_P]
    float* s_row = smem + a_in_floats<TIn>();        // [2][AIN][RW_P]; later vertical sums
    int* s_iy = reinterpret_cast<int*>(s_row + a_row_floats());
    int* s_ix = s_iy + AIN;
    int* s_rmap = s_ix + AIN;
    int* s_cmap = s_rmap + AR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const ATile g = analysis_tile(a, blockIdx.z, blockIdx.y, blockIdx.x);
    const bool fast_u8 = tile_fast_u8<TIn>(a, g);
    const bool fast = fast_u8 || (sizeof(TIn) == 4 && fast_f32(a, g));
    if (!fast || g.bx || g.by) {   // mirror tables: only tiles that read mirrored samples need them
        analysis_tables(a, g, s_iy, s_ix, s_rmap, s_cmap);
        __syncthreads();
    }
    if (sizeof(TIn) == 1 && kU8Bytes) {
        load_tile_u8<A_NW>(a, g, fast_u8, reinterpret_cast<uint8_t*>(s_in), s_iy, s_ix, warp, lane);
        __syncthreads();
        rowpass_u8(reinterpret_cast<const uint8_t*>(s_in), s_row);
    } else {
        load_tile<TIn, A_NW>(a, g, fast_u8, s_in, s_iy, s_ix, warp, lane);
        __syncthreads();
        rowpass_f32(s_in, s_row);
    }
    __syncthreads();
    float* s_det = s_in;
    colpass(a, g, s_row, s_det);
    __syncthreads();
    if (kDoubleV) shrink3(a, g, s_det, reinterpret_cast<float4*>(s_row), s_rmap, s_cmap, CtaBar{});
    else shrink3_single(a, g, s_det, reinterpret_cast<float4*>(s_row), s_rmap, s_cmap);
}

// ============================================================== synthesis
// Output tile ST_Y x ST_X; its coefficients (rows ky0 .. ky0+SC_Y, cols kx0 ..
// kx0+SC_X of the four subband planes) arrive by TMA into a double-buffered
// shared tile: thread 0 issues frame f+1's four box loads on an mbarrier while
// the CTA reconstructs frame f.  TMA zero-fills coefficients beyond the plane;
// only outputs beyond the plane depend on them (t < N uses k <= (N+5)/2 < n).
constexpr int ST_Y = 32, ST_X = 64;     // output tile
constexpr int SC_Y = ST_Y / 2 + 3;      // 19 coefficient rows
constexpr int SC_X = ST_X / 2 + 3;      // 35 coefficient cols
constexpr int SC_BW = 36;               // TMA box width (144 B, multiple of 16)
constexpr int SC_PS = 704;              // plane stride in floats (>= 19*36, 128-B multiple)
constexpr int SC_TILE = 4 * SC_PS;      // one frame's 4 planes (128-B multiple)
constexpr int SL_P = SC_X + 2;          // 37 (odd) pitch of the column-pass planes
constexpr int SO_P = ST_X + 1;          // 65 pitch of the output staging tile
constexpr size_t S_SMEM_BYTES = sizeof(float) * (2 * SC_TILE + 2 * ST_Y * SL_P + ST_Y * SO_P) + 2 * sizeof(uint64_t);
static_assert(SC_Y * SC_BW <= SC_PS && (SC_PS * 4) % 128 == 0, "TMA plane tile layout");
static_assert(((2 * SC_TILE + 2 * ST_Y * SL_P + ST_Y * SO_P) * 4) % 8 == 0, "mbarrier alignment");
constexpr int ACC_PER_THREAD = (ST_Y * ST_X) / 256;

struct SynthMaps {
    CUtensorMap A, d0, d1, d2;   // approximation (unused if !has_A), da, ad, dd
};

struct SynthArgs {
    int has_A;
    int NH, NW;                  // output plane size
    int nb;                      // frames
    int frames_per_cta;          // MODE 0: frames per CTA along grid.z
    float* out;                  // MODE 0 output [nb][NH][out_pitch]
    long long out_bstride;
    int out_pitch;
    const void* I;               // MODE 1/2: frames the residuals come from
    long long i_bstride;
    int i_pitch;
    double* num;                 // MODE 1/2: fp64 accumulators [NH][acc_pitch]
    double* den;
    int acc_pitch;
};

// Column pass (along y) then row pass (along x) of one frame's tile in `c`
// into s_out[ST_Y][SO_P].  Ends with a barrier (s_out complete).
__device__ __forceinline__ void synth_compute(const float* c, float* s_L, float* s_out) {
    const int tid = threadIdx.x;
    // Lx = synth(A, ad), Hx = synth(da, dd); item = (coefficient column k, 4 output rows)
    for (int it = tid; it < SC_X * (ST_Y / 4); it += 256) {
        // warps 0..7: columns 0..31 of one row group each; the last items take
        // columns 32..34 of every group (no bank-shifted wrap inside a warp)
        const int k = it < 32 * (ST_Y / 4) ? (it & 31) : 32 + (it - 32 * (ST_Y / 4)) % (SC_X - 32);
        const int sg = it < 32 * (ST_Y / 4) ? (it >> 5) : (it - 32 * (ST_Y / 4)) / (SC_X - 32);
        float va[5], vda[5], vad[5], vdd[5];
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            const int r = (2 * sg + m) * SC_BW + k;
            va[m] = c[0 * SC_PS + r];
            vda[m] = c[1 * SC_PS + r];
            vad[m] = c[2 * SC_PS + r];
            vdd[m] = c[3 * SC_PS + r];
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            // outputs t = 2s (e = 0) and 2s+1 (e = 1) as one FFMA2 pair
            float2 l = make_float2(0.f, 0.f), h = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                l = ffma2(va[q + m], c_sh[m], l);
                l = ffma2(vad[q + m], c_sg[m], l);
                h = ffma2(vda[q + m], c_sh[m], h);
                h = ffma2(vdd[q + m], c_sg[m], h);
            }
            const int t = 4 * sg + 2 * q;
            s_L[t * SL_P + k] = l.x;
            s_L[(t + 1) * SL_P + k] = l.y;
            s_L[ST_Y * SL_P + t * SL_P + k] = h.x;
            s_L[ST_Y * SL_P + (t + 1) * SL_P + k] = h.y;
        }
    }
    __syncthreads();
    // row pass: item = (output row t, 8 output columns)
    for (int it = tid; it < ST_Y * (ST_X / 8); it += 256) {
        const int t = it % ST_Y, g = it / ST_Y;
        float vl[7], vh[7];
#pragma unroll
        for (int m = 0; m < 7; ++m) {
            vl[m] = s_L[t * SL_P + 4 * g + m];
            vh[m] = s_L[ST_Y * SL_P + t * SL_P + 4 * g + m];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 x = make_float2(0.f, 0.f);   // outputs 2q (e = 0) and 2q+1 (e = 1)
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                x = ffma2(vl[q + m], c_sh[m], x);
                x = ffma2(vh[q + m], c_sg[m], x);
            }
            s_out[t * SO_P + 8 * g + 2 * q] = x.x;
            s_out[t * SO_P + 8 * g + 2 * q + 1] = x.y;
        }
    }
    __syncthreads();
}

// MODE 0: write the reconstruction (grid.z = frame chunks).
// MODE 1: level-1 reconstruction fused with the MLE accumulation over all nb
//         frames (grid.z = 1), I of type TI; NUM/DEN read once, written once,
//         per-pixel sums in ascending frame order.
template <int MODE, typename TI>
#ifndef PRNU_SYNTH_ACC_MINB
#define PRNU_SYNTH_ACC_MINB 3
#endif
__global__ void __launch_bounds__(256, MODE == 0 ? 3 : PRNU_SYNTH_ACC_MINB) k_synth_tma(const __grid_constant__ SynthMaps maps, SynthArgs a) {
    extern __shared__ __align__(128) float smem[];
    float* cbuf0 = smem;
    float* s_L = smem + 2 * SC_TILE;
    float* s_out = s_L + 2 * ST_Y * SL_P;
    uint64_t* bar = reinterpret_cast<uint64_t*>(s_out + ST_Y * SO_P);
    const int tid = threadIdx.x;
    const int ty0 = blockIdx.y * ST_Y, tx0 = blockIdx.x * ST_X;
    const int ky0 = ty0 >> 1, kx0 = tx0 >> 1;
    int f0 = 0, f1 = a.nb;
    if (MODE == 0) {
        f0 = blockIdx.z * a.frames_per_cta;
        f1 = min(a.nb, f0 + a.frames_per_cta);
    }
    const uint32_t tx_bytes = (a.has_A ? 4u : 3u) * SC_BW * SC_Y * 4u;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (!a.has_A) {   // coarsest level: the approximation of the noise domain is 0 (R-10)
        for (int i = tid; i < SC_PS; i += 256) {
            cbuf0[i] = 0.f;
            cbuf0[SC_TILE + i] = 0.f;
        }
    }
    __syncthreads();
    auto issue = [&](int f, int buf) {
        float* c = cbuf0 + buf * SC_TILE;
        mbar_arrive_expect_tx(&bar[buf], tx_bytes);
        if (a.has_A) tma_load_3d(c, &maps.A, kx0, ky0, f, &bar[buf]);
        tma_load_3d(c + 1 * SC_PS, &maps.d0, kx0, ky0, f, &bar[buf]);
        tma_load_3d(c + 2 * SC_PS, &maps.d1, kx0, ky0, f, &bar[buf]);
        tma_load_3d(c + 3 * SC_PS, &maps.d2, kx0, ky0, f, &bar[buf]);
    };
    if (tid == 0 && f0 < f1) issue(f0, 0);

    // accumulate mapping: thread owns column cc of rows r0, r0+4, ..., r0+28 of the tile
    static_assert(ST_X == 64 && ACC_PER_THREAD * 4 == ST_Y, "accumulate mapping");
    const int r0 = tid >> 6, cc = tid & 63;
    const int gx = tx0 + cc;
    const int gxc = min(gx, a.NW - 1);
    double an[ACC_PER_THREAD], ad[ACC_PER_THREAD];
    if (MODE == 1) {
#pragma unroll
        for (int k = 0; k < ACC_PER_THREAD; ++k) {
            const int gy = ty0 + r0 + 4 * k;
            const bool ok = gy < a.NH && gx < a.NW;
            an[k] = ok ? a.num[(size_t)gy * a.acc_pitch + gx] : 0.0;
            ad[k] = ok ? a.den[(size_t)gy * a.acc_pitch + gx] : 0.0;
        }
    }

    for (int f = f0; f < f1; ++f) {
        const int it = f - f0, buf = it & 1;
        if (tid == 0 && f + 1 < f1) {
            fence_proxy_async();
            issue(f + 1, buf ^ 1);   // buffer buf^1 was released by the barrier ending iteration it-1
        }
        float iv[ACC_PER_THREAD];
        if (MODE == 1) {   // this frame's I values, in flight during the reconstruction
            const TI* Ib = reinterpret_cast<const TI*>(a.I) + (size_t)f * a.i_bstride;
#pragma unroll   // rows clamped into the plane: values of pixels beyond it are read, never stored
            for (int k = 0; k < ACC_PER_THREAD; ++k)
                iv[k] = (float)__ldg(Ib + min(ty0 + r0 + 4 * k, a.NH - 1) * a.i_pitch + gxc);
        }
        mbar_wait(&bar[buf], (it >> 1) & 1);
        synth_compute(cbuf0 + buf * SC_TILE, s_L, s_out);
        if (MODE == 0) {
            float* out = a.out + (size_t)f * a.out_bstride;
            if (gx < a.NW) {
#pragma unroll
                for (int k = 0; k < ACC_PER_THREAD; ++k) {
                    const int gy = ty0 + r0 + 4 * k;
                    if (gy < a.NH) out[(size_t)gy * a.out_pitch + gx] = s_out[(r0 + 4 * k) * SO_P + cc];
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < ACC_PER_THREAD; ++k) {
                const double w = (double)s_out[(r0 + 4 * k) * SO_P + cc];
                const double x = (double)iv[k];
                an[k] += w * x;   // exact product (fp32 x fp32 fits fp64), fp64 sum
                ad[k] += x * x;
            }
        }
        __syncthreads();   // s_L / s_out / cbuf[buf] free for the next frame
    }
    if (MODE == 1) {
#pragma unroll
        for (int k = 0; k < ACC_PER_THREAD; ++k) {
            const int gy = ty0 + r0 + 4 * k;
            if (gy < a.NH && gx < a.NW) {
                a.num[(size_t)gy * a.acc_pitch + gx] = an[k];
                a.den[(size_t)gy * a.acc_pitch + gx] = ad[k];
            }
        }
    }
}

// ============================================================== synthesis + accumulate, v2
// Level-1 inverse fused with the MLE accumulation (a4 + a5):
// one CTA owns a 32 x 64 pixel tile for every frame of the wave.  Per frame:
//   * the four coefficient tiles AND the frame's I tile arrive by TMA into a
//     two-stage ring (frame f+1 lands while f is reconstructed);
//   * column pass (along y) into a double-buffered pair of L/H planes;
//   * ONE barrier; the row pass (along x) of 8 pixels per thread feeds the
//     accumulation straight from registers: NUM += W I (fp64 FMA of the exact
//     fp32 x fp32 product), DEN += I^2 — for u8 frames an exact integer
//     sum added to the fp64 accumulator at the end (bit-identical to the
//     sequential fp64 sum, every partial sum being an integer < 2^53).
// Per-pixel order is ascending frame order, as in k_synth_tma<1>.
constexpr int SA_STAGE_COEF = 4 * SC_PS;           // floats per stage (4 planes)
#ifndef PRNU_SACC_VEC
#define PRNU_SACC_VEC 1   // row pass reads its 7 L/H values with two LDS.128 (pitch 40); 0: scalar, pitch 37
#endif
// L/H plane pitch: 40 == 8 mod 32 makes the row pass's LDS.128 (8 lanes: rows 4w+(l&3),
// columns 4 (l>>2)) conflict-free; the column pass stores consecutive columns (any pitch)
constexpr int SA_LP = PRNU_SACC_VEC ? 40 : SL_P;
template <int TY, typename TI, int MODE = 1>
constexpr size_t sacc_smem_bytes() {
    return 2 * SA_STAGE_COEF * sizeof(float) + (MODE ? 3 * TY * ST_X * sizeof(TI) : 0) +
           2 * 2 * TY * SA_LP * sizeof(float) + 2 * sizeof(uint64_t);
}

// MODE 1: accumulate (frames 0 .. nb-1, one CTA per tile); MODE 0: plain inverse
// level written to a.out (frames [z * frames_per_cta, ...) per CTA, no I tiles).
template <int TY, typename TI, int MODE = 1>
#ifndef PRNU_SACC_MINB
#define PRNU_SACC_MINB 4
#endif
__global__ void __launch_bounds__(256, PRNU_SACC_MINB) k_synth_acc2(const __grid_constant__ SynthMaps maps,
                                                       const __grid_constant__ CUtensorMap imap, SynthArgs a) {
    constexpr int CY = TY / 2 + 3;   // coefficient rows of a TY-row tile
    static_assert(TY % 4 == 0 && TY <= 32, "tile height");
    extern __shared__ __align__(128) float smem[];
    // coefficient ring of 2 stages (frame f in stage f & 1, released after its
    // column pass), I-tile ring of 3 (frame f in f % 3, released after its row
    // pass): frame f+2 is issued at the barrier of frame f, two frames ahead.
    float* coef0 = smem;                                                      // [2][4][SC_PS]
    TI* itile0 = reinterpret_cast<TI*>(smem + 2 * SA_STAGE_COEF);             // [3][TY][ST_X] (MODE 1)
    float* sL0 = reinterpret_cast<float*>(itile0 + (MODE ? 3 * TY * ST_X : 0));   // [2][2][TY][SA_LP]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sL0 + 2 * 2 * TY * SA_LP);
    const int tid = threadIdx.x;
    const int ty0 = blockIdx.y * TY, tx0 = blockIdx.x * ST_X;
    const int ky0 = ty0 >> 1, kx0 = tx0 >> 1;
    const int f0 = MODE ? 0 : blockIdx.z * a.frames_per_cta;
    const int nb = MODE ? a.nb : min(a.nb - f0, a.frames_per_cta);   // frames of this CTA: f0 .. f0+nb-1
    const uint32_t tx_bytes = (a.has_A ? 4u : 3u) * SC_BW * CY * 4u + (MODE ? (uint32_t)(TY * ST_X * sizeof(TI)) : 0u);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    if (!a.has_A) {   // coarsest level: the approximation of the noise domain is 0 (R-10)
        for (int i = tid; i < SC_PS; i += 256) {
            coef0[i] = 0.f;
            coef0[SA_STAGE_COEF + i] = 0.f;
        }
    }
    __syncthreads();
    auto issue = [&](int f) {
        const int st = f & 1;
        float* c = coef0 + st * SA_STAGE_COEF;
        mbar_arrive_expect_tx(&bar[st], tx_bytes);
        if (a.has_A) tma_load_3d(c, &maps.A, kx0, ky0, f0 + f, &bar[st]);
        tma_load_3d(c + 1 * SC_PS, &maps.d0, kx0, ky0, f0 + f, &bar[st]);
        tma_load_3d(c + 2 * SC_PS, &maps.d1, kx0, ky0, f0 + f, &bar[st]);
        tma_load_3d(c + 3 * SC_PS, &maps.d2, kx0, ky0, f0 + f, &bar[st]);
        if (MODE) tma_load_3d(itile0 + (f % 3) * TY * ST_X, &imap, tx0, ty0, f, &bar[st]);
    };
    if (tid == 0) {
        if (nb > 0) issue(0);
        if (nb > 1) issue(1);
    }

    // row pass / accumulate mapping: warp w rows 4w .. 4w+3, lane -> (row 4w + (lane & 3), 8 columns at 8 (lane >> 2))
    const int lane = tid & 31, warp = tid >> 5;
    const int rt = 4 * warp + (lane & 3), rg = lane >> 2;
    const int gy = ty0 + rt, gx = tx0 + 8 * rg;
    const bool rowact = rt < TY;            // warp-uniform: the last warp idles in the row pass when TY = 28
    const bool rowok = rowact && gy < a.NH;
    double num[8];
    uint32_t den_i[8];
    double den_d[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        num[k] = (MODE && rowok && gx + k < a.NW) ? a.num[(size_t)gy * a.acc_pitch + gx + k] : 0.0;
        den_i[k] = 0u;
        den_d[k] = 0.0;
    }
    if (MODE && sizeof(TI) == 4) {
#pragma unroll
        for (int k = 0; k < 8; ++k) den_d[k] = (rowok && gx + k < a.NW) ? a.den[(size_t)gy * a.acc_pitch + gx + k] : 0.0;
    }
    // column-pass items (frame-invariant): item it = (coefficient column k, output rows 4 sg .. 4 sg + 3);
    // with at most one item per thread (TY <= 28) it is computed once here
    constexpr int NITEM = SC_X * (TY / 4);
    auto item_k = [](int it) { return it < 32 * (TY / 4) ? (it & 31) : 32 + (it - 32 * (TY / 4)) % (SC_X - 32); };
    auto item_sg = [](int it) { return it < 32 * (TY / 4) ? (it >> 5) : (it - 32 * (TY / 4)) / (SC_X - 32); };
    const int ck = item_k(tid), csg = item_sg(tid);

    for (int f = 0; f < nb; ++f) {
        const int st = f & 1;
        mbar_wait(&bar[st], (f >> 1) & 1);
        const float* c = coef0 + st * SA_STAGE_COEF;
        float* sLo = sL0 + (f & 1) * 2 * TY * SA_LP;
        float* sHi = sLo + TY * SA_LP;
        // column pass: Lx = synth_y(A, ad), Hx = synth_y(da, dd); item = (coefficient column k, 4 output rows)
        for (int it = tid; it < NITEM; it += 256) {
            const int k = NITEM <= 256 ? ck : item_k(it), sg = NITEM <= 256 ? csg : item_sg(it);
            PRNU_DCHECK(k < SC_X && 2 * sg + 4 < CY && 4 * sg + 3 < TY);
            float va[5], vda[5], vad[5], vdd[5];
#pragma unroll
            for (int m = 0; m < 5; ++m) {
                const int r = (2 * sg + m) * SC_BW + k;
                va[m] = c[0 * SC_PS + r];
                vda[m] = c[1 * SC_PS + r];
                vad[m] = c[2 * SC_PS + r];
                vdd[m] = c[3 * SC_PS + r];
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                float2 l = fmul2s(va[q], c_sh[0]), h = fmul2s(vda[q], c_sh[0]);
                l = ffma2(vad[q], c_sg[0], l);
                h = ffma2(vdd[q], c_sg[0], h);
#pragma unroll
                for (int m = 1; m < 4; ++m) {
                    l = ffma2(va[q + m], c_sh[m], l);
                    l = ffma2(vad[q + m], c_sg[m], l);
                    h = ffma2(vda[q + m], c_sh[m], h);
                    h = ffma2(vdd[q + m], c_sg[m], h);
                }
                const int t = 4 * sg + 2 * q;
                sLo[t * SA_LP + k] = l.x;
                sLo[(t + 1) * SA_LP + k] = l.y;
                sHi[t * SA_LP + k] = h.x;
                sHi[(t + 1) * SA_LP + k] = h.y;
            }
        }
        __syncthreads();   // L/H planes of frame f complete; every thread is past frame f-1
        if (tid == 0 && f + 2 < nb) {
            fence_proxy_async();
            issue(f + 2);   // coefficient stage of frame f, I stage of frame f-1: both consumed
        }
        if (!rowact) continue;
        // row pass of 8 pixels + accumulation
        float vl[8], vh[8];
#if PRNU_SACC_VEC
        {   // columns 4 rg .. 4 rg + 7 (the 8th unused): two LDS.128 per plane
            const float4* pl = reinterpret_cast<const float4*>(sLo + rt * SA_LP + 4 * rg);
            const float4* ph = reinterpret_cast<const float4*>(sHi + rt * SA_LP + 4 * rg);
            const float4 l0 = pl[0], l1 = pl[1], h0 = ph[0], h1 = ph[1];
            vl[0] = l0.x; vl[1] = l0.y; vl[2] = l0.z; vl[3] = l0.w; vl[4] = l1.x; vl[5] = l1.y; vl[6] = l1.z; vl[7] = l1.w;
            vh[0] = h0.x; vh[1] = h0.y; vh[2] = h0.z; vh[3] = h0.w; vh[4] = h1.x; vh[5] = h1.y; vh[6] = h1.z; vh[7] = h1.w;
        }
#else
#pragma unroll
        for (int m = 0; m < 7; ++m) {
            vl[m] = sLo[rt * SA_LP + 4 * rg + m];
            vh[m] = sHi[rt * SA_LP + 4 * rg + m];
        }
#endif
        float w[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 x = fmul2s(vl[q], c_sh[0]);
            x = ffma2(vh[q], c_sg[0], x);
#pragma unroll
            for (int m = 1; m < 4; ++m) {
                x = ffma2(vl[q + m], c_sh[m], x);
                x = ffma2(vh[q + m], c_sg[m], x);
            }
            w[2 * q] = x.x;
            w[2 * q + 1] = x.y;
        }
        if (MODE == 0) {   // plain inverse level: write this thread's 8 outputs
            if (rowok) {
                float* orow = a.out + (size_t)(f0 + f) * a.out_bstride + (size_t)gy * a.out_pitch + gx;
                if (gx + 8 <= a.NW && ((a.out_pitch & 3) == 0)) {
                    reinterpret_cast<float4*>(orow)[0] = make_float4(w[0], w[1], w[2], w[3]);
                    reinterpret_cast<float4*>(orow)[1] = make_float4(w[4], w[5], w[6], w[7]);
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (gx + k < a.NW) orow[k] = w[k];
                }
            }
            continue;
        }
        const TI* irow = itile0 + (f % 3) * TY * ST_X + rt * ST_X + 8 * rg;
        if (sizeof(TI) == 1) {
            const uint2 iv = *reinterpret_cast<const uint2*>(irow);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t xb = __byte_perm(k < 4 ? iv.x : iv.y, 0, 0x4440u | (uint32_t)(k & 3));
                den_i[k] += xb * xb;
                // exact integer -> double: (2^52 + x) - 2^52
                const double xd = __hiloint2double(0x43300000, (int)xb) - 4503599627370496.0;
                num[k] = fma((double)w[k], xd, num[k]);   // exact product, one fp64 rounding
            }
        } else {
            const float4 i0 = *reinterpret_cast<const float4*>(irow);
            const float4 i1 = *reinterpret_cast<const float4*>(irow + 4);
            const float iv[8] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double xd = (double)iv[k];
                num[k] = fma((double)w[k], xd, num[k]);
                den_d[k] = fma(xd, xd, den_d[k]);
            }
        }
    }
    if (MODE && rowok) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (gx + k < a.NW) {
                a.num[(size_t)gy * a.acc_pitch + gx + k] = num[k];
                double* dp = a.den + (size_t)gy * a.acc_pitch + gx + k;
                *dp = sizeof(TI) == 1 ? *dp + (double)den_i[k] : den_d[k];
            }
        }
    }
}

// ============================================================== host side
Pyramid make_pyramid(int H, int W, int levels) {
    Pyramid p{};
    p.levels = levels;
    p.nH[0] = H;
    p.nW[0] = W;
    p.pitch[0] = W;
    p.plane[0] = (size_t)H * W;
    for (int l = 1; l <= levels; ++l) {
        p.nH[l] = sub_len(p.nH[l - 1]);
        p.nW[l] = sub_len(p.nW[l - 1]);
        p.pitch[l] = (int)align_up((size_t)p.nW[l], 32);
        p.plane[l] = (size_t)p.nH[l] * p.pitch[l];
    }
    return p;
}

// floats of pyramid workspace per frame: per level, approximation/synthesis
// plane + 3 detail planes.
size_t pyramid_floats_per_frame(const Pyramid& p) {
    size_t f = 0;
    for (int l = 1; l <= p.levels; ++l) f += 4 * p.plane[l];
    return f + 3 * p.plane[1];   // + raw detail scratch of the split analysis (level-1 size, reused by every level)
}

struct PyramidBuffers {
    float* approx[kMaxLevels + 1];   // level-l approximation, reused for the synthesis output of level l+1
    float* det[kMaxLevels + 1][3];
    size_t bstride[kMaxLevels + 1];  // floats between frames within a level buffer
    float* raw[3];                   // raw detail scratch (split analysis), batch x plane[1] floats each
};

PyramidBuffers carve_pyramid(const Pyramid& p, float* base, int batch) {
    PyramidBuffers pb{};
    float* cur = base;
    for (int l = 1; l <= p.levels; ++l) {
        pb.bstride[l] = p.plane[l];
        pb.approx[l] = cur;
        cur += (size_t)batch * p.plane[l];
        for (int s = 0; s < 3; ++s) {
            pb.det[l][s] = cur;
            cur += (size_t)batch * p.plane[l];
        }
    }
    for (int s = 0; s < 3; ++s) {
        pb.raw[s] = cur;
        cur += (size_t)batch * p.plane[1];
    }
    return pb;
}

static const char* kAnalysisName[kMaxLevels + 1] = {"", "analysis_l1", "analysis_l2", "analysis_l3",
                                                    "analysis_l4", "analysis_l5", "analysis_l6"};
static const char* kSynthName[kMaxLevels + 1] = {"", "synthesis_l1", "synthesis_l2", "synthesis_l3",
                                                 "synthesis_l4", "synthesis_l5", "synthesis_l6"};

bool encode_tensor_map_3d(CUtensorMap* map, CUtensorMapDataType dt, size_t elem_bytes, const void* base, uint64_t cols,
                          uint64_t rows, uint64_t depth, uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t box_w,
                          uint32_t box_h) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return false;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    (void)elem_bytes;
    cuuint64_t dims[3] = {cols, rows, depth};
    cuuint64_t strides[2] = {pitch_bytes, plane_bytes};
    cuuint32_t box[3] = {box_w, box_h, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static bool g_attr_done = false;

static int setup_attributes() {
    if (g_attr_done) return PRNU_OK;
    cudaError_t e1 = cudaFuncSetAttribute(k_analysis_shrink<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)a_smem_bytes<float>());
    cudaError_t e2 = cudaFuncSetAttribute(k_analysis_shrink<uint8_t>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a_smem_bytes<uint8_t>());
    cudaError_t e3 = cudaFuncSetAttribute(k_synth_tma<0, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)S_SMEM_BYTES);
    cudaError_t e4 = cudaFuncSetAttribute(k_synth_tma<1, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)S_SMEM_BYTES);
    cudaError_t e5 = cudaFuncSetAttribute(k_synth_tma<1, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)S_SMEM_BYTES);
    cudaError_t e = e1 ? e1 : e2 ? e2 : e3 ? e3 : e4 ? e4 : e5;
    if (e != cudaSuccess) return fail(PRNU_CUDA_ERROR, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    g_attr_done = true;
    return PRNU_OK;
}

// Tensor maps over the four level-l planes of `nb` frames, box SC_BW x SC_Y.
static int synth_maps(const Pyramid& p, const PyramidBuffers& pb, int l, int nb, bool has_A, SynthMaps* m) {
    const uint64_t pitch = (uint64_t)p.pitch[l] * 4, plane = (uint64_t)pb.bstride[l] * 4;
    const float* src[4] = {pb.approx[l], pb.det[l][0], pb.det[l][1], pb.det[l][2]};
    CUtensorMap* dst[4] = {&m->A, &m->d0, &m->d1, &m->d2};
    for (int i = 0; i < 4; ++i) {
        if (i == 0 && !has_A) {
            *dst[0] = CUtensorMap{};
            continue;
        }
        if (!encode_tensor_map_3d(dst[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src[i], p.nW[l], p.nH[l], nb, pitch,
                                  plane, SC_BW, SC_Y))
            return fail(PRNU_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    }
    return PRNU_OK;
}

// Column-streaming strip analysis (strip.cu) unless PRNU_STRIP=0 (A/B switch
// back to the tile kernel k_analysis_shrink).
static bool use_strip() {
    static const bool on = !(getenv("PRNU_STRIP") && getenv("PRNU_STRIP")[0] == '0');
    return on;
}

// Split analysis (split.cu: streaming DWT + streaming shrink) when PRNU_SPLIT=1:
// measured slower than the fused strip kernel at levels 1-3 once the fp32 strip
// variant fits 3 CTAs/SM (level 2: 3.65 vs 3.90 ms/step, profiles/r01).
static bool use_split() {
    static const bool on = getenv("PRNU_SPLIT") && getenv("PRNU_SPLIT")[0] == '1';
    return on;
}
// First level analysed by the split kernels (PRNU_SPLIT_MINL, default 2): level 1
// stays with the fused strip kernel (12.0 vs 13.6 ms/step split, profiles/r01).
static int split_min_level() {
    static const int l = getenv("PRNU_SPLIT_MINL") ? atoi(getenv("PRNU_SPLIT_MINL")) : 2;
    return l;
}
// Last level analysed by the split kernels (PRNU_SPLIT_MAXL, default 2): on the
// small coarse planes the tile kernel is faster (profiles/r01).
static int split_max_level() {
    static const int l = getenv("PRNU_SPLIT_MAXL") ? atoi(getenv("PRNU_SPLIT_MAXL")) : 2;
    return l;
}
static const char* kDwtName[kMaxLevels + 1] = {"", "dwt_l1", "dwt_l2", "dwt_l3", "dwt_l4", "dwt_l5", "dwt_l6"};
static const char* kShrinkName[kMaxLevels + 1] = {"", "shrink_l1", "shrink_l2", "shrink_l3",
                                                  "shrink_l4", "shrink_l5", "shrink_l6"};

// Deepest level analysed by the strip kernel (PRNU_STRIP_MAXL, default: all).  With
// the fp32 strips' fill rule (fewer, longer segments; 1 wave) and the direct left
// mirror, the strip kernel also wins at level 4 (step 22.70 -> 22.55 ms, interleaved
// A/B); the tile kernel k_analysis_shrink stays as the PRNU_STRIP=0 / A/B path.
// A/B during development: PRNU_ANALYSIS=strip selects the direct-filter strip kernel
static bool use_lift() {
    static const bool on = !(getenv("PRNU_ANALYSIS") && std::string(getenv("PRNU_ANALYSIS")) == "strip");
    return on;
}
static int strip_max_level() {
    static const int l = getenv("PRNU_STRIP_MAXL") ? atoi(getenv("PRNU_STRIP_MAXL")) : 6;   // every level
    return l;
}

// Analysis of all levels, then synthesis of levels L..2 (the level-1
// synthesis is launched by the caller, fused or not with the accumulation).
template <typename TIn>
static int denoise_front(const TIn* in, long long in_bstride, int in_pitch, int nb, const Pyramid& p,
                         const PyramidBuffers& pb, const ShrinkParams& sp, cudaStream_t st) {
    int rc = setup_attributes();
    if (rc) return rc;
    const int L = p.levels;
    for (int l = 1; l <= L; ++l) {
        AnalysisArgs a{};
        a.NH = p.nH[l - 1];
        a.NW = p.nW[l - 1];
        a.ll = (l < L) ? pb.approx[l] : nullptr;
        a.d0 = pb.det[l][0];
        a.d1 = pb.det[l][1];
        a.d2 = pb.det[l][2];
        a.out_bstride = (long long)pb.bstride[l];
        a.out_pitch = p.pitch[l];
        a.nH = p.nH[l];
        a.nW = p.nW[l];
        a.sp = sp;
        dim3 grid((p.nW[l] + AT - 1) / AT, (p.nH[l] + AT - 1) / AT, nb);
        if (use_split() && l >= split_min_level() && l <= split_max_level()) {   // streaming DWT kernel + streaming shrink kernel (split.cu)
            {
                KTimer kt(l == 1 ? (sizeof(TIn) == 1 ? "dwt_l1_u8" : "dwt_l1_f32") : kDwtName[l], st);
                if (l == 1 && sizeof(TIn) == 1)
                    rc = launch_dwt_strip_u8(reinterpret_cast<const uint8_t*>(in), in_bstride, in_pitch, a.NH, a.NW,
                                             a.ll, pb.raw[0], pb.raw[1], pb.raw[2], a.out_bstride, a.out_pitch, a.nH,
                                             a.nW, nb, st);
                else
                    rc = launch_dwt_strip_f32(l == 1 ? reinterpret_cast<const float*>(in) : pb.approx[l - 1],
                                              l == 1 ? in_bstride : (long long)pb.bstride[l - 1],
                                              l == 1 ? in_pitch : p.pitch[l - 1], a.NH, a.NW, a.ll, pb.raw[0],
                                              pb.raw[1], pb.raw[2], a.out_bstride, a.out_pitch, a.nH, a.nW, nb, st);
                if (rc) return rc;
            }
            count_launch();
            if ((rc = check_launch("k_dwt_strip"))) return rc;
            {
                KTimer kt(kShrinkName[l], st);
                const float* src[3] = {pb.raw[0], pb.raw[1], pb.raw[2]};
                float* dst[3] = {a.d0, a.d1, a.d2};
                rc = launch_shrink_strip(src, dst, a.out_bstride, a.out_pitch, a.nH, a.nW, sp, nb, st);
                if (rc) return rc;
            }
            count_launch();
            if ((rc = check_launch("k_shrink_strip"))) return rc;
            continue;
        }
        KTimer kt(l == 1 ? (sizeof(TIn) == 1 ? "analysis_l1_u8" : "analysis_l1_f32") : kAnalysisName[l], st);
        if (l == 1) {
            a.in = in;
            a.in_bstride = in_bstride;
            a.in_pitch = in_pitch;
            if (use_lift()) {
                rc = sizeof(TIn) == 1
                         ? launch_analysis_lift_u8(reinterpret_cast<const uint8_t*>(in), in_bstride, in_pitch, a.NH,
                                                   a.NW, a.ll, a.d0, a.d1, a.d2, a.out_bstride, a.out_pitch, a.nH,
                                                   a.nW, sp, nb, st)
                         : launch_analysis_lift_f32(reinterpret_cast<const float*>(in), in_bstride, in_pitch, a.NH,
                                                    a.NW, a.ll, a.d0, a.d1, a.d2, a.out_bstride, a.out_pitch, a.nH,
                                                    a.nW, sp, nb, st);
                if (rc) return rc;
            } else if (use_strip()) {
                rc = sizeof(TIn) == 1
                         ? launch_analysis_strip_u8(reinterpret_cast<const uint8_t*>(in), in_bstride, in_pitch, a.NH,
                                                    a.NW, a.ll, a.d0, a.d1, a.d2, a.out_bstride, a.out_pitch, a.nH,
                                                    a.nW, sp, nb, st)
                         : launch_analysis_strip_f32(reinterpret_cast<const float*>(in), in_bstride, in_pitch, a.NH,
                                                     a.NW, a.ll, a.d0, a.d1, a.d2, a.out_bstride, a.out_pitch, a.nH,
                                                     a.nW, sp, nb, st);
                if (rc) return rc;
            } else {   // PRNU_STRIP=0: the tile kernel
                k_analysis_shrink<TIn><<<grid, A_NT, a_smem_bytes<TIn>(), st>>>(a);
            }
        } else {
            a.in = pb.approx[l - 1];
            a.in_bstride = (long long)pb.bstride[l - 1];
            a.in_pitch = p.pitch[l - 1];
            if (use_lift()) {
                rc = launch_analysis_lift_f32(pb.approx[l - 1], a.in_bstride, a.in_pitch, a.NH, a.NW, a.ll, a.d0,
                                              a.d1, a.d2, a.out_bstride, a.out_pitch, a.nH, a.nW, sp, nb, st);
                if (rc) return rc;
            } else if (use_strip() && l <= strip_max_level()) {
                rc = launch_analysis_strip_f32(pb.approx[l - 1], a.in_bstride, a.in_pitch, a.NH, a.NW, a.ll, a.d0,
                                               a.d1, a.d2, a.out_bstride, a.out_pitch, a.nH, a.nW, sp, nb, st);
                if (rc) return rc;
            } else {
                k_analysis_shrink<float><<<grid, A_NT, a_smem_bytes<float>(), st>>>(a);
            }
        }
        count_launch();
        if ((rc = check_launch(l == 1 ? "k_analysis_strip" : "k_analysis_shrink"))) return rc;
    }
    for (int l = L; l >= 2; --l) {
        SynthMaps m;
        if ((rc = synth_maps(p, pb, l, nb, l < L, &m))) return rc;
        SynthArgs s{};
        s.has_A = l < L;
        s.NH = p.nH[l - 1];
        s.NW = p.nW[l - 1];
        s.nb = nb;
        s.out = pb.approx[l - 1];
        s.out_bstride = (long long)pb.bstride[l - 1];
        s.out_pitch = p.pitch[l - 1];
        static const bool synth2 = !(getenv("PRNU_SYNTH2") && getenv("PRNU_SYNTH2")[0] == '0');
        if (synth2) {   // v2 pipeline (2-frame-deep TMA prefetch, one barrier per frame), 32-row tiles
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_synth_acc2<32, float, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sacc_smem_bytes<32, float, 0>());
                attr = true;
            }
            const int tiles = ((s.NW + ST_X - 1) / ST_X) * ((s.NH + 31) / 32);
            // frames per CTA: enough CTAs for ~4 waves of 4 CTAs/SM, at least 4 frames to amortise the pipeline
            static const int waves = getenv("PRNU_SYNTH_WAVES") ? atoi(getenv("PRNU_SYNTH_WAVES")) : 4;
            static const int fmin = getenv("PRNU_SYNTH_FMIN") ? atoi(getenv("PRNU_SYNTH_FMIN")) : 4;
            s.frames_per_cta = std::max(fmin, std::min(nb, (int)((long long)tiles * nb / (148 * 4 * waves))));
            dim3 grid((s.NW + ST_X - 1) / ST_X, (s.NH + 31) / 32, (nb + s.frames_per_cta - 1) / s.frames_per_cta);
            KTimer kt(kSynthName[l], st);
            k_synth_acc2<32, float, 0><<<grid, 256, sacc_smem_bytes<32, float, 0>(), st>>>(m, CUtensorMap{}, s);
        } else {
            const int tiles = ((s.NW + ST_X - 1) / ST_X) * ((s.NH + ST_Y - 1) / ST_Y);
            s.frames_per_cta = std::max(1, std::min(4, tiles * nb / (148 * 6)));
            dim3 grid((s.NW + ST_X - 1) / ST_X, (s.NH + ST_Y - 1) / ST_Y, (nb + s.frames_per_cta - 1) / s.frames_per_cta);
            KTimer kt(kSynthName[l], st);
            k_synth_tma<0, float><<<grid, 256, S_SMEM_BYTES, st>>>(m, s);
        }
        count_launch();
        if ((rc = check_launch("k_synth_tma"))) return rc;
    }
    return PRNU_OK;
}

template <typename TIn>
int run_residual(const TIn* in, int nb, int H, int W, const Pyramid& p, const ShrinkParams& sp, float* W_out,
                 float* ws_pyr, cudaStream_t st, int in_pitch) {
    if (in_pitch <= 0) in_pitch = W;
    PyramidBuffers pb = carve_pyramid(p, ws_pyr, nb);
    int rc = denoise_front<TIn>(in, (long long)H * in_pitch, in_pitch, nb, p, pb, sp, st);
    if (rc) return rc;
    SynthMaps m;
    if ((rc = synth_maps(p, pb, 1, nb, p.levels > 1, &m))) return rc;
    SynthArgs s{};
    s.has_A = p.levels > 1;
    s.NH = H;
    s.NW = W;
    s.nb = nb;
    s.out = W_out;
    s.out_bstride = (long long)H * W;
    s.out_pitch = W;
    static const bool synth2 = !(getenv("PRNU_SYNTH2") && getenv("PRNU_SYNTH2")[0] == '0');
    if (synth2) {   // the v2 pipeline of the levels above (MODE 0: W written, no accumulation)
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_synth_acc2<32, float, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sacc_smem_bytes<32, float, 0>());
            attr = true;
        }
        const int tiles = ((W + ST_X - 1) / ST_X) * ((H + 31) / 32);
        s.frames_per_cta = std::max(4, std::min(nb, (int)((long long)tiles * nb / (148 * 4 * 4))));
        dim3 grid((W + ST_X - 1) / ST_X, (H + 31) / 32, (nb + s.frames_per_cta - 1) / s.frames_per_cta);
        KTimer kt("synthesis_l1", st);
        k_synth_acc2<32, float, 0><<<grid, 256, sacc_smem_bytes<32, float, 0>(), st>>>(m, CUtensorMap{}, s);
    } else {
        const int tiles = ((W + ST_X - 1) / ST_X) * ((H + ST_Y - 1) / ST_Y);
        s.frames_per_cta = std::max(1, std::min(4, tiles * nb / (148 * 6)));
        dim3 grid((W + ST_X - 1) / ST_X, (H + ST_Y - 1) / ST_Y, (nb + s.frames_per_cta - 1) / s.frames_per_cta);
        KTimer kt("synthesis_l1", st);
        k_synth_tma<0, float><<<grid, 256, S_SMEM_BYTES, st>>>(m, s);
    }
    count_launch();
    return check_launch("k_synth (level 1)");
}

// acc_wait (optional): event the accumulating launch must wait for (the previous
// wave's accumulation on another stream); acc_done (optional): recorded after it.
// frame_stride: elements between consecutive frames of `in`/`I` (H*W for a
// contiguous stack; k*H*W selects every k-th frame, f4 stride emulation).
template <typename TIn>
int run_residual_accumulate(const TIn* in, const TIn* I, int nb, int H, int W, const Pyramid& p,
                            const ShrinkParams& sp, double* num, double* den, float* ws_pyr, cudaStream_t st,
                            cudaEvent_t acc_wait, cudaEvent_t acc_done, long long frame_stride, int in_pitch) {
    if (in_pitch <= 0) in_pitch = W;   // elements between the rows of `in` and `I`
    PyramidBuffers pb = carve_pyramid(p, ws_pyr, nb);
    int rc = denoise_front<TIn>(in, frame_stride, in_pitch, nb, p, pb, sp, st);
    if (rc) return rc;
    SynthMaps m;
    if ((rc = synth_maps(p, pb, 1, nb, p.levels > 1, &m))) return rc;
    SynthArgs s{};
    s.has_A = p.levels > 1;
    s.NH = H;
    s.NW = W;
    s.nb = nb;
    s.I = I;
    s.i_bstride = frame_stride;
    s.i_pitch = in_pitch;
    s.num = num;
    s.den = den;
    s.acc_pitch = W;
    dim3 grid((W + ST_X - 1) / ST_X, (H + ST_Y - 1) / ST_Y, 1);
    if (acc_wait && cudaStreamWaitEvent(st, acc_wait, 0) != cudaSuccess)
        return fail(PRNU_CUDA_ERROR, "cudaStreamWaitEvent");
    // v2 (TMA-staged I tiles, one barrier per frame) unless PRNU_SACC2=0 or the
    // frames violate the TMA stride/alignment rules.  Tile height 32 or 28 rows,
    // whichever fills the last wave of 4 CTAs/SM better.
    static const bool sacc2 = !(getenv("PRNU_SACC2") && getenv("PRNU_SACC2")[0] == '0');
    const int slots = 148 * 4;
    auto waste = [&](int ty) {
        const long n = (long)((W + ST_X - 1) / ST_X) * ((H + ty - 1) / ty);
        return (double)((n + slots - 1) / slots) * ty / ((double)n * ty / slots);   // waves rounded up / exact
    };
    static const int ty_env = getenv("PRNU_SACC_TY") ? atoi(getenv("PRNU_SACC_TY")) : 0;
    const int TYsel = ty_env == 28 || ty_env == 32 ? ty_env : (waste(28) < waste(32) - 1e-9 ? 28 : 32);
    CUtensorMap imap;
    SynthMaps m2;
    const size_t es = sizeof(TIn);
    bool v2 = sacc2 && ((size_t)in_pitch * es) % 16 == 0 && ((size_t)frame_stride * es) % 16 == 0 &&
              ((uintptr_t)I % 16) == 0 &&
              encode_tensor_map_3d(&imap, sizeof(TIn) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                   es, I, (uint64_t)W, (uint64_t)H, (uint64_t)nb, (uint64_t)in_pitch * es,
                                   (uint64_t)frame_stride * es, ST_X, TYsel);
    if (v2) {
        const uint64_t pitch = (uint64_t)p.pitch[1] * 4, plane = (uint64_t)pb.bstride[1] * 4;
        const float* src[4] = {pb.approx[1], pb.det[1][0], pb.det[1][1], pb.det[1][2]};
        CUtensorMap* dst[4] = {&m2.A, &m2.d0, &m2.d1, &m2.d2};
        for (int i = 0; i < 4 && v2; ++i) {
            if (i == 0 && !s.has_A) {
                *dst[0] = CUtensorMap{};
                continue;
            }
            v2 = encode_tensor_map_3d(dst[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src[i], p.nW[1], p.nH[1], nb, pitch,
                                      plane, SC_BW, TYsel / 2 + 3);
        }
    }
    {
        KTimer kt(sizeof(TIn) == 1 ? "synth_acc_l1_u8" : "synth_acc_l1_f32", st);
        if (v2) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_synth_acc2<32, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sacc_smem_bytes<32, uint8_t>());
                cudaFuncSetAttribute(k_synth_acc2<32, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sacc_smem_bytes<32, float>());
                cudaFuncSetAttribute(k_synth_acc2<28, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sacc_smem_bytes<28, uint8_t>());
                cudaFuncSetAttribute(k_synth_acc2<28, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sacc_smem_bytes<28, float>());
                attr = true;
            }
            dim3 g2((W + ST_X - 1) / ST_X, (H + TYsel - 1) / TYsel, 1);
            if (TYsel == 28)
                k_synth_acc2<28, TIn><<<g2, 256, sacc_smem_bytes<28, TIn>(), st>>>(m2, imap, s);
            else
                k_synth_acc2<32, TIn><<<g2, 256, sacc_smem_bytes<32, TIn>(), st>>>(m2, imap, s);
        } else {
            k_synth_tma<1, TIn><<<grid, 256, S_SMEM_BYTES, st>>>(m, s);
        }
    }
    count_launch();
    if ((rc = check_launch("k_synth_tma(accumulate)"))) return rc;
    if (acc_done && cudaEventRecord(acc_done, st) != cudaSuccess) return fail(PRNU_CUDA_ERROR, "cudaEventRecord");
    return PRNU_OK;
}

template int run_residual<float>(const float*, int, int, int, const Pyramid&, const ShrinkParams&, float*, float*,
                                 cudaStream_t, int);
template int run_residual<uint8_t>(const uint8_t*, int, int, int, const Pyramid&, const ShrinkParams&, float*,
                                   float*, cudaStream_t, int);
template int run_residual_accumulate<float>(const float*, const float*, int, int, int, const Pyramid&,
                                            const ShrinkParams&, double*, double*, float*, cudaStream_t, cudaEvent_t,
                                            cudaEvent_t, long long, int);
template int run_residual_accumulate<uint8_t>(const uint8_t*, const uint8_t*, int, int, int, const Pyramid&,
                                              const ShrinkParams&, double*, double*, float*, cudaStream_t,
                                              cudaEvent_t, cudaEvent_t, long long, int);

}  // namespace prnu
