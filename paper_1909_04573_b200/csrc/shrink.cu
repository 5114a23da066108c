// shrink.cu — the local-variance MAP/Wiener shrink (a3, R-7) of detail
// planes held in HBM, c -> c - F(c) = c s0 / max(min_w mean_w(c^2), s0) (the
// noise domain, R-10), as a column-streaming kernel.  Used where the shrink is
// not fused into the analysis: the f3 denoiser variants (variant.cu, on the raw
// detail planes of the generic DWT passes) and the f2 Wiener-in-DFT clean-up
// (wdft.cu, the Wiener gain on the magnitude spectrum, sigma0^2 per plane read
// from device memory).
//
// A CTA of 128 threads owns a vertical strip of the plane (one thread per
// region column, <= 120 output columns plus the 4-column window halo each side)
// and walks down a segment of rows in blocks of 8 rows.  Borders (R-4): the
// shrink reads the mirrored subband row / column directly, so its windows hold
// exactly the oracle's e_N samples.
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace prnu {
namespace shrinkk {

constexpr int NT = 128;      // threads per CTA
constexpr int BK = 8;        // rows per block
__constant__ float2 c_ws[2] = {{1.0f / 9.0f, 1.0f / 25.0f}, {1.0f / 49.0f, 1.0f / 81.0f}};

// (a, b) * w lane-wise (FMUL2)
__device__ __forceinline__ float2 fmul2s_pair(float a, float b, float2 w) {
    const float2 v = make_float2(a, b);
    unsigned long long ra = *reinterpret_cast<const unsigned long long*>(&v);
    unsigned long long rb = *reinterpret_cast<const unsigned long long*>(&w);
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&r);
}

constexpr int SO_MAX = NT - 8;       // output columns per strip (4-column window halo each side)

struct ShrinkArgs {
    const float* src[3];   // raw detail planes
    float* dst[3];         // c - F(c)
    long long bstride;
    int pitch;
    int nH, nW;
    int nb;
    ShrinkParams sp;
    int O;                 // output columns per strip (multiple of 8, <= SO_MAX)
    int SH;                // output rows per segment (multiple of BK)
    int nsub;              // planes per frame (3 detail subbands; 1 for the WDFT magnitude)
    const float* s0_dev;   // per-frame sigma0^2 on the device (nullable: sp.sigma0_sq)
};

// ---------------------------------------------------------------- shrink, horizontal-first
// The separable window sums horizontal-first: the squares c^2 of 8 rows go through shared memory once (one float per
// coefficient); each output thread forms the nested horizontal sums h3..h9 of
// its column from its 8 neighbours, and the vertical sums of h_w over 3..9 rows
// slide down per-window register rings (re-initialised every block of 8 rows,
// so no rounding drifts across blocks).  One barrier per block (double-buffered
// square planes).  Shared traffic per coefficient: 4 B written + 32 B read.
constexpr int QP = NT;   // square-plane pitch (threads read consecutive columns: conflict-free)

template <bool ALL4>
__global__ void __launch_bounds__(NT, 4) k_shrink_hfirst(ShrinkArgs a) {
    __shared__ __align__(16) float qb[2][BK][QP];
    const int t = threadIdx.x;
    const int sb = blockIdx.z % a.nsub, b = blockIdx.z / a.nsub;
    const int cx0 = blockIdx.x * a.O;
    const int ky0 = blockIdx.y * a.SH;
    const int ky1 = min(ky0 + a.SH, a.nH);
    const int gc = cx0 - 4 + t;
    const int nW = a.nW, nH = a.nH;
    const int mc = mirror(gc, nW);   // the column whose values this region column holds (R-4)
    const float* src = (sb == 0 ? a.src[0] : sb == 1 ? a.src[1] : a.src[2]) + (size_t)b * a.bstride + mc;
    float* const dst = (sb == 0 ? a.dst[0] : sb == 1 ? a.dst[1] : a.dst[2]) + (size_t)b * a.bstride + gc;
    const int nblk = 1 + (ky1 - ky0 + BK - 1) / BK;   // block 0 = prologue (rows ky0-4 .. ky0+3)
    const int K0 = ky0 - 4;
    const bool outc = t >= 4 && t < 4 + a.O && gc < nW;   // this thread's column is an output column
    const float s0 = a.s0_dev ? a.s0_dev[b] : a.sp.sigma0_sq;
    const int wm = a.sp.wmask;

    float pf[BK], pf2[BK];
    auto rowm = [&](int r) {
        if (nH >= 8) return r < 0 ? -1 - r : (r >= nH ? 2 * nH - 1 - r : r);
        return mirror(r, nH);
    };
    auto load_block = [&](int i, float (&dv)[BK]) {
        const int K = K0 + BK * i;
        if (K >= 0 && K + BK <= nH) {
            const float* p = src + (size_t)K * a.pitch;
#pragma unroll
            for (int k = 0; k < BK; ++k) dv[k] = __ldg(p + (size_t)k * a.pitch);
        } else {
#pragma unroll
            for (int k = 0; k < BK; ++k) dv[k] = __ldg(src + (size_t)rowm(K + k) * a.pitch);
        }
    };
    // rings (slot s = row K-8+s): h_w of rows K-8 .. K+7, coefficients of rows K-4 .. K+7
    float h3[16], h5[16], h7[16], h9[16], c[12];
#pragma unroll
    for (int k = 0; k < 16; ++k) h3[k] = h5[k] = h7[k] = h9[k] = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k) c[k] = 0.f;
    load_block(0, pf);
    if (nblk > 1) load_block(1, pf2);
#pragma unroll 1
    for (int i = 0; i < nblk; ++i) {
        const int K = K0 + BK * i;
        float (&qs)[BK][QP] = qb[i & 1];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h3[k] = h3[8 + k];
            h5[k] = h5[8 + k];
            h7[k] = h7[8 + k];
            h9[k] = h9[8 + k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = c[8 + k];
        float q[BK];
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            c[4 + k] = pf[k];
            q[k] = __fmul_rn(pf[k], pf[k]);
            qs[k][t] = q[k];
            pf[k] = pf2[k];
        }
        if (i + 2 < nblk) load_block(i + 2, pf2);
        __syncthreads();
        PRNU_STRESS(21);   // squares of rows K .. K+7 visible (the other plane is free)
        if (!outc) continue;
        // nested horizontal sums of this column, rows K .. K+7 -> ring slots 8 .. 15
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float* row = &qs[k][t];
            const float x3 = row[-1] + q[k] + row[1];
            const float x5 = x3 + row[-2] + row[2];
            const float x7 = x5 + row[-3] + row[3];
            h3[8 + k] = x3;
            h5[8 + k] = x5;
            h7[8 + k] = x7;
            h9[8 + k] = x7 + row[-4] + row[4];
        }
        if (i == 0) continue;
        // output rows K-4 .. K+3: vertical sums over slots j+4-r .. j+4+r (sliding within the block)
        float s3 = h3[3] + h3[4] + h3[5];
        float s5 = h5[2] + h5[3] + h5[4] + h5[5] + h5[6];
        float s7 = h7[1] + h7[2] + h7[3] + h7[4] + h7[5] + h7[6] + h7[7];
        float s9 = h9[0] + h9[1] + h9[2] + h9[3] + h9[4] + h9[5] + h9[6] + h9[7] + h9[8];
        float* drow = dst + (size_t)(K - 4) * a.pitch;
#pragma unroll
        for (int j = 0; j < BK; ++j) {
            if (j > 0) {
                s3 += h3[j + 5] - h3[j + 2];
                s5 += h5[j + 6] - h5[j + 1];
                s7 += h7[j + 7] - h7[j];
                s9 += h9[j + 8] - h9[j - 1];
            }
            const float2 r35 = fmul2s_pair(s3, s5, c_ws[0]);
            const float2 r79 = fmul2s_pair(s7, s9, c_ws[1]);
            float m;
            if (ALL4) {
                m = fminf(fminf(r35.x, r35.y), fminf(r79.x, r79.y));
            } else {
                m = 3.402823466e38f;
                if (wm & 1) m = fminf(m, r35.x);
                if (wm & 2) m = fminf(m, r35.y);
                if (wm & 4) m = fminf(m, r79.x);
                if (wm & 8) m = fminf(m, r79.y);
            }
            float rc;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(fmaxf(m, s0)));
            // c - F(c) = c s0 / (max(m - s0, 0) + s0) = c s0 / max(m, s0)
            if (K - 4 + j < ky1) drow[(size_t)j * a.pitch] = c[j] * s0 * rc;
        }
    }
}

}  // namespace shrinkk

// ---------------------------------------------------------------- host
// Rows per segment: about per_seg, but small planes are cut into more segments
// so that the grid holds at least two waves of resident CTAs (min_ctas).
static int seg_rows(int nH, int per_seg, int align, long long ctas_per_seg, long long min_ctas) {
    int nseg = (nH + per_seg - 1) / per_seg;
    while (nseg * ctas_per_seg < min_ctas && (nH + nseg) / (nseg + 1) >= align) ++nseg;
    return (int)align_up((size_t)((nH + nseg - 1) / nseg), align);
}

int launch_shrink_strip(const float* const src[3], float* const dst[3], long long bstride, int pitch, int nH, int nW,
                        const ShrinkParams& sp, int nb, cudaStream_t st, int nsub, const float* s0_dev) {
    using namespace shrinkk;
    ShrinkArgs a{};
    for (int s = 0; s < 3; ++s) {
        a.src[s] = src[s];
        a.dst[s] = dst[s];
    }
    a.nsub = nsub;
    a.s0_dev = s0_dev;
    a.bstride = bstride;
    a.pitch = pitch;
    a.nH = nH;
    a.nW = nW;
    a.nb = nb;
    a.sp = sp;
    const int S0 = (nW + SO_MAX - 1) / SO_MAX;
    a.O = (int)align_up((size_t)((nW + S0 - 1) / S0), 8);
    const int S = (nW + a.O - 1) / a.O;
    a.SH = seg_rows(nH, 136, BK, (long long)nsub * S * nb, 2LL * device_sm_count() * 4);
    const int nseg = (nH + a.SH - 1) / a.SH;
    dim3 grid(S, nseg, nsub * nb);
    if (nsub * nb > 65535) return fail(PRNU_INVALID_ARG, "shrink: more than 65535 planes in one launch");
    if (sp.wmask == 15) k_shrink_hfirst<true><<<grid, NT, 0, st>>>(a);
    else k_shrink_hfirst<false><<<grid, NT, 0, st>>>(a);
    return PRNU_OK;
}

}  // namespace prnu
