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
#include "common.cuh"

namespace prnu {

// ============================================================== analysis
constexpr int AT = 32;                  // output coefficient tile (square)
constexpr int AR = AT + 2 * kHalo;      // 40: computed coefficient region
constexpr int AIN = 2 * AR + 6;         // 86: input rows / columns of the region
constexpr int AIN_P = AIN + 1;          // smem pitch of the input tile (odd)
constexpr int ROW_P = AR + 1;           // pitch of row-pass / detail planes
constexpr int HS_P = AT + 1;            // pitch of the horizontal window sums
constexpr int A_SMEM_IN = AIN * AIN_P;            // >= 3*AR*ROW_P (details alias it)
constexpr int A_SMEM_ROW = 2 * AIN * ROW_P;       // >= 4*AR*HS_P  (window sums alias it)
constexpr size_t A_SMEM_BYTES = sizeof(float) * (A_SMEM_IN + A_SMEM_ROW) + sizeof(int) * (2 * AIN + 2 * AR);
static_assert(3 * AR * ROW_P <= A_SMEM_IN, "detail planes must fit in the input tile");
static_assert(4 * AR * HS_P <= A_SMEM_ROW, "window sums must fit in the row-pass planes");

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

template <typename TIn>
__global__ void __launch_bounds__(256) k_analysis_shrink(AnalysisArgs a) {
    extern __shared__ float smem[];
    float* s_in = smem;                          // [AIN][AIN_P]; later details [3][AR][ROW_P]
    float* s_row = smem + A_SMEM_IN;             // [2][AIN][ROW_P]; later sums [4][AR][HS_P]
    int* s_iy = reinterpret_cast<int*>(s_row + A_SMEM_ROW);   // [AIN] input row index
    int* s_ix = s_iy + AIN;                                   // [AIN] input col index
    int* s_rmap = s_ix + AIN;                                 // [AR] mirrored region row
    int* s_cmap = s_rmap + AR;                                // [AR] mirrored region col

    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int b = blockIdx.z;
    const int y0 = blockIdx.y * AT, x0 = blockIdx.x * AT;
    const int cy0 = y0 - kHalo, cx0 = x0 - kHalo;
    const TIn* in = reinterpret_cast<const TIn*>(a.in) + (size_t)b * a.in_bstride;

    for (int i = tid; i < AIN; i += nthr) {
        s_iy[i] = mirror(2 * cy0 - 6 + i, a.NH);
        s_ix[i] = mirror(2 * cx0 - 6 + i, a.NW);
    }
    for (int i = tid; i < AR; i += nthr) {
        s_rmap[i] = mirror(cy0 + i, a.nH) - cy0;
        s_cmap[i] = mirror(cx0 + i, a.nW) - cx0;
    }
    __syncthreads();

    // ---- load the mirrored input tile: every thread issues all its loads
    // before the first shared-memory store, so they are in flight together.
    {
        constexpr int PER = (AIN * AIN + 255) / 256;
        float v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            int e = tid + 256 * k;
            if (e < AIN * AIN) {
                int r = e / AIN, c = e - r * AIN;
                v[k] = (float)__ldg(in + (size_t)s_iy[r] * a.in_pitch + s_ix[c]);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            int e = tid + 256 * k;
            if (e < AIN * AIN) {
                int r = e / AIN, c = e - r * AIN;
                s_in[r * AIN_P + c] = v[k];
            }
        }
    }
    __syncthreads();

    // ---- row pass (along x): lo/hi for AIN rows x AR coefficient columns
    for (int it = tid; it < AIN * (AR / 4); it += nthr) {
        int r = it % AIN, cg = it / AIN;
        const float* src = s_in + r * AIN_P + 8 * cg;
        float v[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) v[k] = src[k];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float lo = 0.f, hi = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                lo = fmaf(wl_h(i), v[2 * q + i], lo);
                hi = fmaf(wl_g(i), v[2 * q + i], hi);
            }
            s_row[r * ROW_P + 4 * cg + q] = lo;
            s_row[AIN * ROW_P + r * ROW_P + 4 * cg + q] = hi;
        }
    }
    __syncthreads();

    // ---- column pass (along y): 4 subbands for AR x AR coefficients
    float* s_det = s_in;
    for (int it = tid; it < AR * (AR / 4); it += nthr) {
        int c = it % AR, rg = it / AR;
        float lo[14], hi[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) {
            lo[k] = s_row[(8 * rg + k) * ROW_P + c];
            hi[k] = s_row[AIN * ROW_P + (8 * rg + k) * ROW_P + c];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float aa = 0.f, ad = 0.f, da = 0.f, dd = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                aa = fmaf(wl_h(i), lo[2 * q + i], aa);
                ad = fmaf(wl_g(i), lo[2 * q + i], ad);
                da = fmaf(wl_h(i), hi[2 * q + i], da);
                dd = fmaf(wl_g(i), hi[2 * q + i], dd);
            }
            int rr = 4 * rg + q;
            s_det[0 * AR * ROW_P + rr * ROW_P + c] = da;
            s_det[1 * AR * ROW_P + rr * ROW_P + c] = ad;
            s_det[2 * AR * ROW_P + rr * ROW_P + c] = dd;
            if (a.ll != nullptr && rr >= kHalo && rr < kHalo + AT && c >= kHalo && c < kHalo + AT) {
                int gy = y0 + rr - kHalo, gx = x0 + c - kHalo;
                if (gy < a.nH && gx < a.nW)
                    a.ll[(size_t)b * a.out_bstride + (size_t)gy * a.out_pitch + gx] = aa;
            }
        }
    }
    __syncthreads();

    // ---- shrink each detail subband (R-7)
    const float s0 = a.sp.sigma0_sq;
    const int wm = a.sp.wmask;
    float* s_hs = s_row;
    for (int s = 0; s < 3; ++s) {
        const float* det = s_det + s * AR * ROW_P;
        // stage A: horizontal window sums of c^2 (3,5,7,9 nested) for real region rows
        for (int it = tid; it < AR * AT; it += nthr) {
            int j = it % AT, rr = it / AT;
            if (s_rmap[rr] != rr) continue;
            float v[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                float c = det[rr * ROW_P + s_cmap[j + k]];
                v[k] = c * c;
            }
            float h3 = v[3] + v[4] + v[5];
            float h5 = h3 + v[2] + v[6];
            float h7 = h5 + v[1] + v[7];
            float h9 = h7 + v[0] + v[8];
            s_hs[0 * AR * HS_P + rr * HS_P + j] = h3;
            s_hs[1 * AR * HS_P + rr * HS_P + j] = h5;
            s_hs[2 * AR * HS_P + rr * HS_P + j] = h7;
            s_hs[3 * AR * HS_P + rr * HS_P + j] = h9;
        }
        __syncthreads();
        // stage B: vertical window sums, MAP variance, Wiener factor; 4 rows per thread
        float* dst = (s == 0 ? a.d0 : s == 1 ? a.d1 : a.d2) + (size_t)b * a.out_bstride;
        for (int it = tid; it < AT * (AT / 4); it += nthr) {
            int j = it % AT, ig = it / AT;
            float h[4][12];
#pragma unroll
            for (int k = 0; k < 12; ++k) {
                int rr = s_rmap[4 * ig + k];
#pragma unroll
                for (int w = 0; w < 4; ++w) h[w][k] = s_hs[w * AR * HS_P + rr * HS_P + j];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float s3 = 0.f, s5 = 0.f, s7 = 0.f, s9 = 0.f;
#pragma unroll
                for (int k = 3; k <= 5; ++k) s3 += h[0][q + k];
#pragma unroll
                for (int k = 2; k <= 6; ++k) s5 += h[1][q + k];
#pragma unroll
                for (int k = 1; k <= 7; ++k) s7 += h[2][q + k];
#pragma unroll
                for (int k = 0; k <= 8; ++k) s9 += h[3][q + k];
                float m = 3.402823466e38f;
                if (wm & 1) m = fminf(m, s3 * (1.0f / 9.0f));
                if (wm & 2) m = fminf(m, s5 * (1.0f / 25.0f));
                if (wm & 4) m = fminf(m, s7 * (1.0f / 49.0f));
                if (wm & 8) m = fminf(m, s9 * (1.0f / 81.0f));
                float v = fmaxf(m - s0, 0.0f);
                int i = 4 * ig + q;
                float c = det[(i + kHalo) * ROW_P + j + kHalo];
                float cn = c * __fdividef(s0, v + s0);     // noise-domain coefficient c - F(c)
                int gy = y0 + i, gx = x0 + j;
                if (gy < a.nH && gx < a.nW) dst[(size_t)gy * a.out_pitch + gx] = cn;
            }
        }
        __syncthreads();
    }
}

// ============================================================== synthesis
constexpr int ST_Y = 32, ST_X = 64;     // output tile
constexpr int SC_Y = ST_Y / 2 + 3;      // 19 coefficient rows
constexpr int SC_X = ST_X / 2 + 3;      // 35 coefficient cols
constexpr int SC_P = SC_X + 1;          // 36
constexpr int SL_P = SC_X + 2;          // 37 (odd) pitch of the column-pass planes
constexpr int SO_P = ST_X + 1;          // 65 pitch of the output staging tile
constexpr int S_SMEM_COEF = 4 * SC_Y * SC_P;          // coefficient tiles; output staging aliases it
constexpr int S_SMEM_L = 2 * ST_Y * SL_P;
constexpr size_t S_SMEM_BYTES = sizeof(float) * (S_SMEM_COEF + S_SMEM_L);
static_assert(ST_Y * SO_P <= S_SMEM_COEF, "output staging must fit in the coefficient tiles");

struct SynthArgs {
    const float* A;     // approximation (nullable = 0)
    const float* d0;    // da
    const float* d1;    // ad
    const float* d2;    // dd
    long long c_bstride;
    int c_pitch;
    int nH, nW;
    float* out;
    long long out_bstride;
    int out_pitch;
    int NH, NW;
};

// Reconstruct the ST_Y x ST_X output tile at (ty0, tx0) of frame b into
// s_out[ST_Y][SO_P] (shared).  All threads participate; ends with a barrier.
constexpr int S_LOAD_PER = (4 * SC_Y * SC_X + 255) / 256;

// Issue the loads of frame b's coefficient tile into registers (no smem write).
__device__ __forceinline__ void synth_fetch(const SynthArgs& a, int b, int ty0, int tx0, float (&v)[S_LOAD_PER]) {
    const int ky0 = ty0 >> 1, kx0 = tx0 >> 1;
    const size_t boff = (size_t)b * a.c_bstride;
#pragma unroll
    for (int k = 0; k < S_LOAD_PER; ++k) {
        int e = threadIdx.x + 256 * k;
        v[k] = 0.0f;
        if (e < 4 * SC_Y * SC_X) {
            int p = e / (SC_Y * SC_X);
            int rem = e - p * (SC_Y * SC_X);
            int r = rem / SC_X, c = rem - r * SC_X;
            int gy = min(ky0 + r, a.nH - 1), gx = min(kx0 + c, a.nW - 1);
            const float* src = p == 0 ? a.A : p == 1 ? a.d0 : p == 2 ? a.d1 : a.d2;
            if (src) v[k] = __ldg(src + boff + (size_t)gy * a.c_pitch + gx);
        }
    }
}

__device__ __forceinline__ void synth_commit(const float (&v)[S_LOAD_PER], float* smem) {
#pragma unroll
    for (int k = 0; k < S_LOAD_PER; ++k) {
        int e = threadIdx.x + 256 * k;
        if (e < 4 * SC_Y * SC_X) {
            int p = e / (SC_Y * SC_X);
            int rem = e - p * (SC_Y * SC_X);
            int r = rem / SC_X, c = rem - r * SC_X;
            smem[(p * SC_Y + r) * SC_P + c] = v[k];
        }
    }
}

// Reconstruct from the coefficient tile already committed to smem.
__device__ __forceinline__ void synth_compute(float* smem) {
    float* s_c = smem;                              // [4][SC_Y][SC_P]
    float* s_L = smem + S_SMEM_COEF;                // [2][ST_Y][SL_P]  (Lx, Hx)
    const int tid = threadIdx.x, nthr = blockDim.x;
    __syncthreads();

    // column pass (along y): Lx = synth(A, ad), Hx = synth(da, dd); 4 output rows per item
    for (int it = tid; it < SC_X * (ST_Y / 4); it += nthr) {
        int k = it % SC_X, sg = it / SC_X;
        float va[5], vad[5], vda[5], vdd[5];
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            int r = 2 * sg + m;
            va[m] = s_c[(0 * SC_Y + r) * SC_P + k];
            vda[m] = s_c[(1 * SC_Y + r) * SC_P + k];
            vad[m] = s_c[(2 * SC_Y + r) * SC_P + k];
            vdd[m] = s_c[(3 * SC_Y + r) * SC_P + k];
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float l = 0.f, h = 0.f;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    l = fmaf(wl_h(6 - 2 * m + e), va[q + m], l);
                    l = fmaf(wl_g(6 - 2 * m + e), vad[q + m], l);
                    h = fmaf(wl_h(6 - 2 * m + e), vda[q + m], h);
                    h = fmaf(wl_g(6 - 2 * m + e), vdd[q + m], h);
                }
                int t = 4 * sg + 2 * q + e;
                s_L[t * SL_P + k] = l;
                s_L[ST_Y * SL_P + t * SL_P + k] = h;
            }
        }
    }
    __syncthreads();

    // row pass (along x): 8 output columns per item; stage into s_out (aliases s_c)
    float* s_out = smem;
    for (int it = tid; it < ST_Y * (ST_X / 8); it += nthr) {
        int t = it % ST_Y, g = it / ST_Y;
        float vl[7], vh[7];
#pragma unroll
        for (int m = 0; m < 7; ++m) {
            vl[m] = s_L[t * SL_P + 4 * g + m];
            vh[m] = s_L[ST_Y * SL_P + t * SL_P + 4 * g + m];
        }
        float o[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float x = 0.f;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    x = fmaf(wl_h(6 - 2 * m + e), vl[q + m], x);
                    x = fmaf(wl_g(6 - 2 * m + e), vh[q + m], x);
                }
                o[2 * q + e] = x;
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s_out[t * SO_P + 8 * g + k] = o[k];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_synthesis(SynthArgs a) {
    extern __shared__ float smem[];
    const int b = blockIdx.z;
    const int ty0 = blockIdx.y * ST_Y, tx0 = blockIdx.x * ST_X;
    {
        float v[S_LOAD_PER];
        synth_fetch(a, b, ty0, tx0, v);
        synth_commit(v, smem);
    }
    synth_compute(smem);
    float* out = a.out + (size_t)b * a.out_bstride;
    for (int e = threadIdx.x; e < ST_Y * ST_X; e += blockDim.x) {
        int r = e / ST_X, c = e - r * ST_X;
        int gy = ty0 + r, gx = tx0 + c;
        if (gy < a.NH && gx < a.NW) out[(size_t)gy * a.out_pitch + gx] = smem[r * SO_P + c];
    }
}

// Level-1 synthesis fused with the MLE accumulation over `nb` frames.
// I: the frames the residuals come from (the SDA frames, or the u8 frames at
// depth 1), [nb][NH][NW] with pitch i_pitch.  num/den: fp64 [NH][NW] (pitch
// acc_pitch), read once before the frame loop and written once after it.
constexpr int ACC_PER_THREAD = (ST_Y * ST_X) / 256;

template <typename TI>
__global__ void __launch_bounds__(256, 2) k_synthesis_accumulate(SynthArgs a, const TI* I, long long i_bstride,
                                                              int i_pitch, int nb, double* num, double* den,
                                                              int acc_pitch) {
    extern __shared__ float smem[];
    const int ty0 = blockIdx.y * ST_Y, tx0 = blockIdx.x * ST_X;
    double an[ACC_PER_THREAD], ad[ACC_PER_THREAD];
#pragma unroll
    for (int k = 0; k < ACC_PER_THREAD; ++k) {
        int e = threadIdx.x + 256 * k;
        int r = e / ST_X, c = e - r * ST_X;
        int gy = ty0 + r, gx = tx0 + c;
        bool ok = gy < a.NH && gx < a.NW;
        an[k] = ok ? num[(size_t)gy * acc_pitch + gx] : 0.0;
        ad[k] = ok ? den[(size_t)gy * acc_pitch + gx] : 0.0;
    }
    float v[S_LOAD_PER];
    synth_fetch(a, 0, ty0, tx0, v);
    for (int b = 0; b < nb; ++b) {
        synth_commit(v, smem);
        if (b + 1 < nb) synth_fetch(a, b + 1, ty0, tx0, v);   // prefetch the next frame's tile
        // this frame's I values, issued before the reconstruction so they are in flight
        const TI* Ib = I + (size_t)b * i_bstride;
        float iv[ACC_PER_THREAD];
#pragma unroll
        for (int k = 0; k < ACC_PER_THREAD; ++k) {
            int e = threadIdx.x + 256 * k;
            int r = e / ST_X, c = e - r * ST_X;
            int gy = min(ty0 + r, a.NH - 1), gx = min(tx0 + c, a.NW - 1);
            iv[k] = (float)Ib[(size_t)gy * i_pitch + gx];
        }
        synth_compute(smem);
#pragma unroll
        for (int k = 0; k < ACC_PER_THREAD; ++k) {
            int e = threadIdx.x + 256 * k;
            int r = e / ST_X, c = e - r * ST_X;
            int gy = ty0 + r, gx = tx0 + c;
            if (gy < a.NH && gx < a.NW) {
                double w = (double)smem[r * SO_P + c];
                double x = (double)iv[k];
                an[k] += w * x;      // exact product (fp32 x fp32 fits fp64), fp64 sum
                ad[k] += x * x;
            }
        }
        __syncthreads();   // s_out is overwritten by the next frame's coefficient commit
    }
#pragma unroll
    for (int k = 0; k < ACC_PER_THREAD; ++k) {
        int e = threadIdx.x + 256 * k;
        int r = e / ST_X, c = e - r * ST_X;
        int gy = ty0 + r, gx = tx0 + c;
        if (gy < a.NH && gx < a.NW) {
            num[(size_t)gy * acc_pitch + gx] = an[k];
            den[(size_t)gy * acc_pitch + gx] = ad[k];
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
    return f;
}

struct PyramidBuffers {
    float* approx[kMaxLevels + 1];   // level-l approximation, reused for the synthesis output of level l+1
    float* det[kMaxLevels + 1][3];
    size_t bstride[kMaxLevels + 1];  // floats between frames within a level buffer
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
    return pb;
}

static const char* kAnalysisName[kMaxLevels + 1] = {"", "analysis_l1", "analysis_l2", "analysis_l3",
                                                    "analysis_l4", "analysis_l5", "analysis_l6"};
static const char* kSynthName[kMaxLevels + 1] = {"", "synthesis_l1", "synthesis_l2", "synthesis_l3",
                                                 "synthesis_l4", "synthesis_l5", "synthesis_l6"};

static bool g_attr_done = false;

static int setup_attributes() {
    if (g_attr_done) return PRNU_OK;
    cudaError_t e1 = cudaFuncSetAttribute(k_analysis_shrink<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)A_SMEM_BYTES);
    cudaError_t e2 = cudaFuncSetAttribute(k_analysis_shrink<uint8_t>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)A_SMEM_BYTES);
    if (e1 != cudaSuccess || e2 != cudaSuccess)
        return fail(PRNU_CUDA_ERROR, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e1 ? e1 : e2));
    g_attr_done = true;
    return PRNU_OK;
}

// Run the analysis of all levels and the synthesis of levels L..2 for `nb`
// frames; leaves the level-1 noise-domain subbands + the level-1 synthesis
// input ready.  Returns a SynthArgs for the final (level-1) synthesis.
template <typename TIn>
static int denoise_front(const TIn* in, long long in_bstride, int in_pitch, int nb, const Pyramid& p,
                         const PyramidBuffers& pb, const ShrinkParams& sp, cudaStream_t st, SynthArgs* last) {
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
        KTimer kt(l == 1 ? (sizeof(TIn) == 1 ? "analysis_l1_u8" : "analysis_l1_f32") : kAnalysisName[l], st);
        if (l == 1) {
            a.in = in;
            a.in_bstride = in_bstride;
            a.in_pitch = in_pitch;
            k_analysis_shrink<TIn><<<grid, 256, A_SMEM_BYTES, st>>>(a);
        } else {
            a.in = pb.approx[l - 1];
            a.in_bstride = (long long)pb.bstride[l - 1];
            a.in_pitch = p.pitch[l - 1];
            k_analysis_shrink<float><<<grid, 256, A_SMEM_BYTES, st>>>(a);
        }
        count_launch();
        if ((rc = check_launch("k_analysis_shrink"))) return rc;
    }
    for (int l = L; l >= 1; --l) {
        SynthArgs s{};
        s.A = (l < L) ? pb.approx[l] : nullptr;
        s.d0 = pb.det[l][0];
        s.d1 = pb.det[l][1];
        s.d2 = pb.det[l][2];
        s.c_bstride = (long long)pb.bstride[l];
        s.c_pitch = p.pitch[l];
        s.nH = p.nH[l];
        s.nW = p.nW[l];
        s.NH = p.nH[l - 1];
        s.NW = p.nW[l - 1];
        if (l == 1) {
            *last = s;   // out filled by the caller
            break;
        }
        s.out = pb.approx[l - 1];
        s.out_bstride = (long long)pb.bstride[l - 1];
        s.out_pitch = p.pitch[l - 1];
        dim3 grid((s.NW + ST_X - 1) / ST_X, (s.NH + ST_Y - 1) / ST_Y, nb);
        {
            KTimer kt(kSynthName[l], st);
            k_synthesis<<<grid, 256, S_SMEM_BYTES, st>>>(s);
        }
        count_launch();
        if ((rc = check_launch("k_synthesis"))) return rc;
    }
    return PRNU_OK;
}

template <typename TIn>
int run_residual(const TIn* in, int nb, int H, int W, const Pyramid& p, const ShrinkParams& sp, float* W_out,
                 float* ws_pyr, cudaStream_t st) {
    PyramidBuffers pb = carve_pyramid(p, ws_pyr, nb);
    SynthArgs s{};
    int rc = denoise_front<TIn>(in, (long long)H * W, W, nb, p, pb, sp, st, &s);
    if (rc) return rc;
    s.out = W_out;
    s.out_bstride = (long long)H * W;
    s.out_pitch = W;
    dim3 grid((W + ST_X - 1) / ST_X, (H + ST_Y - 1) / ST_Y, nb);
    {
        KTimer kt("synthesis_l1", st);
        k_synthesis<<<grid, 256, S_SMEM_BYTES, st>>>(s);
    }
    count_launch();
    return check_launch("k_synthesis(level 1)");
}

template <typename TIn>
int run_residual_accumulate(const TIn* in, const TIn* I, int nb, int H, int W, const Pyramid& p,
                            const ShrinkParams& sp, double* num, double* den, float* ws_pyr, cudaStream_t st) {
    PyramidBuffers pb = carve_pyramid(p, ws_pyr, nb);
    SynthArgs s{};
    int rc = denoise_front<TIn>(in, (long long)H * W, W, nb, p, pb, sp, st, &s);
    if (rc) return rc;
    dim3 grid((W + ST_X - 1) / ST_X, (H + ST_Y - 1) / ST_Y, 1);
    {
        KTimer kt(sizeof(TIn) == 1 ? "synth_acc_l1_u8" : "synth_acc_l1_f32", st);
        k_synthesis_accumulate<TIn><<<grid, 256, S_SMEM_BYTES, st>>>(s, I, (long long)H * W, W, nb, num, den, W);
    }
    count_launch();
    return check_launch("k_synthesis_accumulate");
}

template int run_residual<float>(const float*, int, int, int, const Pyramid&, const ShrinkParams&, float*, float*,
                                 cudaStream_t);
template int run_residual<uint8_t>(const uint8_t*, int, int, int, const Pyramid&, const ShrinkParams&, float*,
                                   float*, cudaStream_t);
template int run_residual_accumulate<float>(const float*, const float*, int, int, int, const Pyramid&,
                                            const ShrinkParams&, double*, double*, float*, cudaStream_t);
template int run_residual_accumulate<uint8_t>(const uint8_t*, const uint8_t*, int, int, int, const Pyramid&,
                                              const ShrinkParams&, double*, double*, float*, cudaStream_t);

}  // namespace prnu
