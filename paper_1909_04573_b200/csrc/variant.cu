// variant.cu — f3: the denoiser variants of Q2-Q4 (R-24..R-26).
//
//   taps = 16        db8 (8 vanishing moments) instead of the 8-tap filter (Q2)
//   boundary = 1     pad to a multiple of 2^levels by e_N, periodic DWT, crop (Q4, R-24)
//   transform = 1    undecimated (stationary) DWT, circular, dilation 2^(l-1) (Q3, R-25)
//
// Same method as the default path (decomposition, local-variance Wiener shrink of
// every detail subband with mirror windows, noise-domain reconstruction
// W = I - F(I), R-10):
//
//   decimated variants (db4 / db8, symmetric or pad + periodic): fused 2-D tile kernels,
//     k_var_ana2d<T, MODE> (one launch per analysis level: rows and columns of a tile in
//     shared memory, the four subbands written once) and k_var_syn2d<T, MODE> (one launch
//     per synthesis level);
//   undecimated variants: separable passes k_var_row_ana / k_var_ana_col and
//     k_var_row_syn / k_var_syn_col (circular, dilation s);
//   launch_shrink_strip (shrink.cu) between analysis and synthesis.
//
// Filter convention (GPU side; R-5 generalised to T taps): H_ is the
// minimum-phase lowpass in common.cuh's order (PRNU_H0..7 for T = 8),
// G_[i] = (-1)^i H_[T-1-i], and
//   decimated analysis   a[c] = sum_i H_[i] x[map(2c - (T-2) + i)]        (d with G_)
//   decimated synthesis  x[t] = sum_m H_[e+2m] a[k] + G_[e+2m] d[k],  e = t & 1,
//                        k = (t-e)/2 + (T-2)/2 - m: dropped outside [0, n) for the
//                        symmetric transform, taken mod n for the periodic one (its
//                        synthesis is the transpose of its orthogonal analysis)
//   undecimated          a[t] = sum_i H_[i] x[(t - s (T-1-i)) mod N],
//                        x[t] = 1/2 sum_i H_[i] a[(t + s (T-1-i)) mod N] + G_[i] d[...]
#include "common.cuh"

namespace prnu {

// db8: Daubechies, "Ten Lectures on Wavelets" (1992), Table 6.1, N = 8, normalised
// to sum sqrt(2), minimum-phase order.  8 taps: common.cuh's PRNU_H0..7.
#define PRNU_DB8                                                                                             \
    0.05441584224308161, 0.3128715909144659, 0.6756307362980128, 0.5853546836548691, -0.015829105256023893,  \
        -0.2840155429624281, 0.00047248457399797254, 0.128747426620186, -0.01736930100202211,               \
        -0.04408825393106472, 0.013981027917015516, 0.008746094047015655, -0.00487035299301066,             \
        -0.0003917403729959771, 0.0006754494059985568, -0.00011747678400228192
static constexpr double kDb8[16] = {PRNU_DB8};
__constant__ float c_var_h[2][16] = {
    {PRNU_H0, PRNU_H1, PRNU_H2, PRNU_H3, PRNU_H4, PRNU_H5, PRNU_H6, PRNU_H7, 0, 0, 0, 0, 0, 0, 0, 0},
    {(float)kDb8[0], (float)kDb8[1], (float)kDb8[2], (float)kDb8[3], (float)kDb8[4], (float)kDb8[5],
     (float)kDb8[6], (float)kDb8[7], (float)kDb8[8], (float)kDb8[9], (float)kDb8[10], (float)kDb8[11],
     (float)kDb8[12], (float)kDb8[13], (float)kDb8[14], (float)kDb8[15]}};

enum VarMode { VM_SYM = 0, VM_PER = 1, VM_SWT = 2 };

__device__ __forceinline__ int var_mod(int i, int n) {
    if (i >= 0 && i < n) return i;           // the common case: no division
    if (i >= n && i < 2 * n) return i - n;   // one wrap
    const int r = i % n;
    return r < 0 ? r + n : r;
}
// where analysis input sample i of a length-N axis comes from (R-4, R-24, R-25).
// Interior samples (almost all) return at once: the integer modulo of the general
// maps made the passes instruction-bound (8 FHD frames, db4 periodic: see DESIGN §6).
template <int MODE>
__device__ __forceinline__ int var_map(int i, int N, int Np) {
    if (i >= 0 && i < N) return i;
    if (MODE == VM_SYM) return mirror(i, N);
    if (MODE == VM_PER) {
        const int r = var_mod(i, Np);       // periodic over the padded length Np ...
        return r < N ? r : mirror(r, N);    // ... whose samples beyond N mirror the plane
    }
    return var_mod(i, N);
}

// ------------------------------------------------------------------ separable passes (undecimated)
// The undecimated variants (R-25) run as separable 1-D passes with circular indexing at
// dilation s = 2^(l-1): a[t] = sum_i H_[i] x[(t - s (T-1-i)) mod N] (d with G_), and the
// synthesis x[t] = 1/2 sum_i H_[i] a[(t + s (T-1-i)) mod N] + G_[i] d[...].
struct VarPass {
    const float* in[4];   // analysis: plane pl reads in[pl]; synthesis: (in[2pl], in[2pl+1]) = (a, d)
    float* out[4];        // analysis: plane pl writes (out[2pl], out[2pl+1]) = (lo, hi); synthesis: out[pl]
    long long in_bstride, out_bstride;   // floats between frames
    int in_pitch, out_pitch;             // floats between rows
    int N;         // length of the axis the pass filters (circular)
    int nout;      // outputs along the axis (== N)
    int other;     // extent along the other axis
    int s;         // dilation 2^(l-1)
    int nplanes;
};

// column passes: grid x over the columns (128 threads per CTA), y over runs of 8 outputs of
// one polyphase component, z = frame * nplanes + plane
constexpr int VAR_RY = 8;

template <int T>
__global__ void __launch_bounds__(128) k_var_ana_col(VarPass p) {
    const int pl = blockIdx.z % p.nplanes, b = blockIdx.z / p.nplanes;
    const int x = blockIdx.x * 128 + threadIdx.x;
    if (x >= p.other) return;
    const float* in = p.in[pl] + (size_t)b * p.in_bstride;
    float* lo = p.out[2 * pl] + (size_t)b * p.out_bstride;
    float* hi = p.out[2 * pl + 1] + (size_t)b * p.out_bstride;
    const float* H = c_var_h[T == 16];
    // run r = q s + ph holds the outputs t_u = 8 s q + ph + s u (one polyphase component),
    // which read input rows 8 s q + ph + s j, j = u + i - (T-1): T + 7 rows, each loaded once
    const int s_ = p.s, q = blockIdx.y / s_, ph = blockIdx.y - q * s_;
    const int tb = 8 * s_ * q + ph;
    if (tb >= p.nout) return;
    float v[T + 7];
#pragma unroll
    for (int j = 0; j < T + 7; ++j)
        v[j] = __ldg(in + (size_t)var_mod(tb + s_ * (j - (T - 1)), p.N) * p.in_pitch + x);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int t = tb + s_ * u;
        if (t >= p.nout) break;
        float a = 0.f, d = 0.f;
#pragma unroll
        for (int i = 0; i < T; ++i) {
            const float g = (i & 1) ? -H[T - 1 - i] : H[T - 1 - i];
            a = fmaf(H[i], v[u + i], a);
            d = fmaf(g, v[u + i], d);
        }
        const size_t oi = (size_t)t * p.out_pitch + x;
        lo[oi] = a;
        hi[oi] = d;
    }
}

template <int T>
__global__ void __launch_bounds__(128) k_var_syn_col(VarPass p) {
    const int pl = blockIdx.z % p.nplanes, b = blockIdx.z / p.nplanes;
    const int x = blockIdx.x * 128 + threadIdx.x;
    if (x >= p.other) return;
    const float* A = p.in[2 * pl] ? p.in[2 * pl] + (size_t)b * p.in_bstride : nullptr;   // null: zero approximation
    const float* D = p.in[2 * pl + 1] + (size_t)b * p.in_bstride;
    float* out = p.out[pl] + (size_t)b * p.out_bstride;
    const float* H = c_var_h[T == 16];
    // the polyphase run of k_var_ana_col; outputs t_u = tb + s u gather a, d rows tb + s j,
    // j = u + T-1-i in [0, T + 6]
    const int s_ = p.s, q = blockIdx.y / s_, ph = blockIdx.y - q * s_;
    const int tb = 8 * s_ * q + ph;
    if (tb >= p.nout) return;
    float ca[T + 7], cd[T + 7];
#pragma unroll
    for (int j = 0; j < T + 7; ++j) {
        const size_t at = (size_t)var_mod(tb + s_ * j, p.N) * p.in_pitch + x;
        ca[j] = A ? __ldg(A + at) : 0.f;
        cd[j] = __ldg(D + at);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int t = tb + s_ * u;
        if (t >= p.nout) break;
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < T; ++i) {
            const float g = (i & 1) ? -H[T - 1 - i] : H[T - 1 - i];
            if (A) acc = fmaf(H[i], ca[u + T - 1 - i], acc);
            acc = fmaf(g, cd[u + T - 1 - i], acc);
        }
        out[(size_t)t * p.out_pitch + x] = 0.5f * acc;
    }
}

// Row (x) passes through shared memory: a CTA stages, for one row at a time, the input
// span its 512 outputs need (each element loaded once, index map applied once per
// element), then every thread computes 4 outputs (t0 + tid + 128 j) from shared memory
// with consecutive lanes on consecutive addresses.
constexpr int VR_OUT = 512;   // outputs per CTA and row

template <int T>
__host__ __device__ inline int var_row_span(int s) { return VR_OUT + s * (T - 1); }   // staged elements per array

template <int T>
__global__ void __launch_bounds__(128) k_var_row_ana(VarPass p) {
    extern __shared__ float vr_smem[];
    const int nst = var_row_span<T>(p.s);
    float* sE = vr_smem;
    const int pl = blockIdx.z % p.nplanes, b = blockIdx.z / p.nplanes;
    const int tid = threadIdx.x;
    const int t0 = blockIdx.x * VR_OUT;
    const float* in = p.in[pl] + (size_t)b * p.in_bstride;
    float* lo = p.out[2 * pl] + (size_t)b * p.out_bstride;
    float* hi = p.out[2 * pl + 1] + (size_t)b * p.out_bstride;
    const float* H = c_var_h[T == 16];
    const int y0 = blockIdx.y * VAR_RY, y1 = min(y0 + VAR_RY, p.other);
    const int base = t0 - p.s * (T - 1);   // E[j] = x[base + j]
    for (int y = y0; y < y1; ++y) {
        const float* row = in + (size_t)y * p.in_pitch;
        __syncthreads();
        PRNU_STRESS(31);   // the previous row's staging is consumed
        for (int j = tid; j < nst; j += 128) sE[j] = __ldg(row + var_mod(base + j, p.N));
        __syncthreads();
        PRNU_STRESS(31);
        float* lrow = lo + (size_t)y * p.out_pitch;
        float* hrow = hi + (size_t)y * p.out_pitch;
#pragma unroll
        for (int q = 0; q < VR_OUT / 128; ++q) {
            const int u = tid + 128 * q, k = t0 + u;
            if (k >= p.nout) break;
            float a = 0.f, d = 0.f;
#pragma unroll
            for (int i = 0; i < T; ++i) {   // x[k - s (T-1-i)] = E[u + s i]
                PRNU_DCHECK(u + p.s * i < nst);
                const float v = sE[u + p.s * i];
                const float g = (i & 1) ? -H[T - 1 - i] : H[T - 1 - i];
                a = fmaf(H[i], v, a);
                d = fmaf(g, v, d);
            }
            lrow[k] = a;
            hrow[k] = d;
        }
    }
}

template <int T>
__global__ void __launch_bounds__(128) k_var_row_syn(VarPass p) {
    extern __shared__ float vr_smem[];
    const int nst = var_row_span<T>(p.s);
    float* sA = vr_smem;
    float* sD = vr_smem + nst;
    const int pl = blockIdx.z % p.nplanes, b = blockIdx.z / p.nplanes;
    const int tid = threadIdx.x;
    const int t0 = blockIdx.x * VR_OUT;
    const float* A = p.in[2 * pl] ? p.in[2 * pl] + (size_t)b * p.in_bstride : nullptr;
    const float* D = p.in[2 * pl + 1] + (size_t)b * p.in_bstride;
    float* out = p.out[pl] + (size_t)b * p.out_bstride;
    const float* H = c_var_h[T == 16];
    const int y0 = blockIdx.y * VAR_RY, y1 = min(y0 + VAR_RY, p.other);
    for (int y = y0; y < y1; ++y) {   // coefficients t0 + j (mod n), j < 512 + s (T-1)
        const float* arow = A ? A + (size_t)y * p.in_pitch : nullptr;
        const float* drow = D + (size_t)y * p.in_pitch;
        __syncthreads();
        PRNU_STRESS(31);
        for (int j = tid; j < nst; j += 128) {
            const int k = var_mod(t0 + j, p.N);
            sA[j] = arow ? __ldg(arow + k) : 0.f;
            sD[j] = __ldg(drow + k);
        }
        __syncthreads();
        PRNU_STRESS(31);
        float* orow = out + (size_t)y * p.out_pitch;
#pragma unroll
        for (int q = 0; q < VR_OUT / 128; ++q) {
            const int u = tid + 128 * q, t = t0 + u;
            if (t >= p.nout) break;
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < T; ++i) {
                const float g = (i & 1) ? -H[T - 1 - i] : H[T - 1 - i];
                const int j = u + p.s * (T - 1 - i);
                acc = fmaf(H[i], sA[j], acc);
                acc = fmaf(g, sD[j], acc);
            }
            orow[t] = 0.5f * acc;
        }
    }
}

// ------------------------------------------------------------------ fused 2-D tile passes
// Decimated variants (symmetric / periodic): one kernel per analysis level (rows and
// columns of a tile through shared memory: input read once, the four subbands written
// once) and one per synthesis level (four coefficient tiles in, the level's output out),
// instead of two separable passes with an HBM round trip in between (round 1; the same
// arithmetic in the same order); parity against the oracle in tests/test_gpu_variants.py.
constexpr int VT_Y = 32, VT_X = 32;   // analysis: coefficient positions per tile (64-row tiles at T = 16: slower)
constexpr int VS_X = 64;   // synthesis: output pixels per tile row
// output rows per synthesis tile: 64 for the 16-tap filter (its coefficient halo is T/2 - 1 rows)
template <int T>
__host__ __device__ constexpr int var_vs_y() { return T == 16 ? 64 : 32; }

struct VarTile {
    const float* in;          // analysis: the level's input plane;  synthesis: unused
    const float* c[4];        // synthesis: A (null: zero approximation), ad, da, dd
    float* out[4];            // analysis: A, ad, da, dd;  synthesis: out[0]
    long long in_bstride, out_bstride;
    int in_pitch, out_pitch;
    int N_y, Np_y, N_x, Np_x; // analysis: real / periodic input extents
    int nH, nW;               // analysis: subband extent;  synthesis: coefficient extent
    int oH, oW;               // synthesis: output extent
};

// analysis tile layout: even / odd input columns [IR][ECP] (ECP: a row pass item reads NLD
// float4 from column 4 u4), the odd array offset so even / odd staging lanes hit distinct banks
template <int T>
struct VaLayout {
    static constexpr int IR = 2 * VT_Y + T - 2;               // input rows of the tile
    static constexpr int EC = VT_X + T / 2 - 1;               // even / odd input columns used
    static constexpr int NLD = (T / 2 + 3 + 3) / 4;           // float4 per row pass item and array
    static constexpr int ECP = VT_X - 4 + 4 * NLD;            // row pitch (>= EC, multiple of 4)
    static constexpr int OFF = ((16 - (IR * ECP) % 32) + 32) % 32;
    static constexpr size_t floats = 2 * (size_t)IR * ECP + OFF + 2 * (size_t)IR * VT_X;
};
template <int T>
__host__ __device__ constexpr size_t var_ana2d_smem() {
    return sizeof(float) * VaLayout<T>::floats;
}
template <int T>
__host__ __device__ constexpr int var_syn_nld() { return (T / 2 + 3 + 3) / 4; }   // float4 per x-pass item
template <int T>
__host__ __device__ constexpr int var_syn_kxp() { return VS_X / 2 - 4 + 4 * var_syn_nld<T>(); }   // X pitch
template <int T>
__host__ __device__ constexpr size_t var_syn2d_smem() {
    return sizeof(float) * (4 * (size_t)(var_vs_y<T>() / 2 + T / 2 - 1) * (VS_X / 2 + T / 2 - 1) +
                            2 * (size_t)var_vs_y<T>() * var_syn_kxp<T>());
}

template <int T, int MODE>
__global__ void __launch_bounds__(256, 2) k_var_ana2d(VarTile p) {
    using LY = VaLayout<T>;
    constexpr int IR = LY::IR, EC = LY::EC, ECP = LY::ECP, NLD = LY::NLD;
    extern __shared__ __align__(16) float va_smem[];
    float* sE = va_smem;                          // [IR][ECP] x[.][base + 2j]
    float* sO = sE + IR * ECP + LY::OFF;          // [IR][ECP] x[.][base + 2j + 1]
    float* sL = sO + IR * ECP;                    // [IR][VT_X] lo_x
    float* sH = sL + IR * VT_X;                   // [IR][VT_X] hi_x
    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int ky0 = blockIdx.y * VT_Y, kx0 = blockIdx.x * VT_X;
    const int yb = 2 * ky0 - (T - 2), xb = 2 * kx0 - (T - 2);
    const float* in = p.in + (size_t)b * p.in_bstride;
    const float* H = c_var_h[T == 16];
    // stage: consecutive threads on consecutive input columns (coalesced), boundary map once per
    // element; all of a thread's loads issued before the first store (memory-level parallelism)
    {   // thread = (input column c, row group rg): the column map once, rows rg, rg + NRG, ...
        constexpr int CW = 2 * EC, NRG = 256 / CW, NI = (IR + NRG - 1) / NRG;
        const int c = tid % CW, rg = tid / CW;
        // tiles whose input region lies inside the plane (almost all): no index maps
        const bool interior = yb >= 0 && yb + IR <= p.N_y && xb >= 0 && xb + CW <= p.N_x;
        if (rg < NRG) {
            const int x = interior ? xb + c : var_map<MODE>(xb + c, p.N_x, p.Np_x);
            float* dst = (c & 1 ? sO : sE) + (c >> 1);
            float v[NI];
            if (interior) {
                const float* src = in + (size_t)(yb + rg) * p.in_pitch + x;
                const size_t step = (size_t)NRG * p.in_pitch;
#pragma unroll
                for (int k = 0; k < NI; ++k)
                    if (rg + NRG * k < IR) v[k] = __ldg(src + k * step);
            } else {
#pragma unroll
                for (int k = 0; k < NI; ++k) {
                    const int r = rg + NRG * k;
                    if (r < IR) v[k] = __ldg(in + (size_t)var_map<MODE>(yb + r, p.N_y, p.Np_y) * p.in_pitch + x);
                }
            }
#pragma unroll
            for (int k = 0; k < NI; ++k) {
                const int r = rg + NRG * k;
                if (r < IR) dst[r * ECP] = v[k];
            }
        }
    }
    __syncthreads();
    PRNU_STRESS(41);
    // (lo, hi) as one packed pair: FFMA2 of the sample with (H_[i], G_[i]), lane-wise the fmaf chain
    float2 hg[T];
#pragma unroll
    for (int i = 0; i < T; ++i) hg[i] = make_float2(H[i], (i & 1) ? -H[T - 1 - i] : H[T - 1 - i]);
    // rows: item = (staged row r, coefficient columns 4 u4 .. 4 u4 + 3), inputs by float4
    for (int e = tid; e < IR * (VT_X / 4); e += 256) {
        const int r = e / (VT_X / 4), u4 = e - r * (VT_X / 4);
        float ev[4 * NLD], ov[4 * NLD];
#pragma unroll
        for (int k = 0; k < NLD; ++k) {
            const float4 a = *reinterpret_cast<const float4*>(sE + r * ECP + 4 * u4 + 4 * k);
            const float4 c = *reinterpret_cast<const float4*>(sO + r * ECP + 4 * u4 + 4 * k);
            ev[4 * k] = a.x; ev[4 * k + 1] = a.y; ev[4 * k + 2] = a.z; ev[4 * k + 3] = a.w;
            ov[4 * k] = c.x; ov[4 * k + 1] = c.y; ov[4 * k + 2] = c.z; ov[4 * k + 3] = c.w;
        }
        float2 acc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            acc[q] = make_float2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < T; ++i) acc[q] = ffma2((i & 1) ? ov[q + i / 2] : ev[q + i / 2], hg[i], acc[q]);
        }
        *reinterpret_cast<float4*>(sL + r * VT_X + 4 * u4) = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
        *reinterpret_cast<float4*>(sH + r * VT_X + 4 * u4) = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
    }
    __syncthreads();
    PRNU_STRESS(42);
    // columns: item = (coefficient rows 4 q4 .. 4 q4 + 3, column u); (aa, ad) from lo_x, (da, dd) from hi_x
    const size_t ob = (size_t)b * p.out_bstride;
    for (int e = tid; e < (VT_Y / 4) * VT_X; e += 256) {
        const int q4 = e / VT_X, u = e - q4 * VT_X;
        const int gx = kx0 + u;
        float lv[T + 6], hv[T + 6];
#pragma unroll
        for (int j = 0; j < T + 6; ++j) {
            lv[j] = sL[(8 * q4 + j) * VT_X + u];
            hv[j] = sH[(8 * q4 + j) * VT_X + u];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int gy = ky0 + 4 * q4 + q;
            float2 la = make_float2(0.f, 0.f), ha = la;   // (aa, ad), (da, dd)
#pragma unroll
            for (int i = 0; i < T; ++i) {
                la = ffma2(lv[2 * q + i], hg[i], la);
                ha = ffma2(hv[2 * q + i], hg[i], ha);
            }
            if (gy < p.nH && gx < p.nW) {
                const size_t o = ob + (size_t)gy * p.out_pitch + gx;
                p.out[0][o] = la.x;
                p.out[1][o] = la.y;
                p.out[2][o] = ha.x;
                p.out[3][o] = ha.y;
            }
        }
    }
}

template <int T, int MODE>
__global__ void __launch_bounds__(256, 2) k_var_syn2d(VarTile p) {
    constexpr int VS_Y = var_vs_y<T>();
    constexpr int KY = VS_Y / 2 + T / 2 - 1, KX = VS_X / 2 + T / 2 - 1;   // coefficient rows / columns
    constexpr int KXP = var_syn_kxp<T>(), NLD = var_syn_nld<T>();
    extern __shared__ __align__(16) float vs_smem[];
    float* sC = vs_smem;                 // [4][KY][KX]: A, ad, da, dd
    float* sX0 = sC + 4 * KY * KX;       // [VS_Y][KXP] synthesis along y of (A, ad)
    float* sX1 = sX0 + VS_Y * KXP;       // [VS_Y][KXP] of (da, dd)
    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int ty0 = blockIdx.y * VS_Y, tx0 = blockIdx.x * VS_X;
    const int k0y = ty0 / 2, k0x = tx0 / 2;
    const int n_y = p.nH, n_x = p.nW;
    const size_t cb = (size_t)b * p.in_bstride;
    const float* H = c_var_h[T == 16];
    // coefficients k = k0 + j: dropped outside [0, n) (symmetric), mod n (periodic)
    {   // thread = (coefficient column i, row group rg): the column map once, then rows
        // rg, rg + NRG, ... of the four planes; all loads before the first store
        constexpr int NRG = 256 / KX, NJ = (KY + NRG - 1) / NRG;
        const int i = tid % KX, rg = tid / KX;
        if (rg < NRG) {
            int kx = k0x + i;
            bool okx = true;
            if (MODE == VM_SYM) okx = kx < n_x;
            else kx = var_mod(kx, n_x);
            // tiles whose coefficient region lies inside the planes (almost all): no index maps
            const bool interior = k0y + KY <= n_y && k0x + KX <= n_x;
            float v[4][NJ];
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) {
                // (no dynamic index into the parameter struct: it would copy it to local memory)
                const float* src = p.c[pl];
                if (interior) {
                    const float* q = src ? src + cb + (size_t)(k0y + rg) * p.in_pitch + kx : nullptr;
                    const size_t step = (size_t)NRG * p.in_pitch;
#pragma unroll
                    for (int k = 0; k < NJ; ++k)
                        v[pl][k] = (q && rg + NRG * k < KY) ? __ldg(q + k * step) : 0.f;
                    continue;
                }
#pragma unroll
                for (int k = 0; k < NJ; ++k) {
                    const int j = rg + NRG * k;
                    int ky = k0y + j;
                    bool ok = okx && j < KY && src != nullptr;
                    if (MODE == VM_SYM) ok = ok && ky < n_y;
                    else ky = var_mod(ky, n_y);
                    v[pl][k] = ok ? __ldg(src + cb + (size_t)ky * p.in_pitch + kx) : 0.f;
                }
            }
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
#pragma unroll
                for (int k = 0; k < NJ; ++k) {
                    const int j = rg + NRG * k;
                    if (j < KY) sC[(pl * KY + j) * KX + i] = v[pl][k];
                }
        }
    }
    __syncthreads();
    PRNU_STRESS(43);
    const float* sA = sC;
    const float* sAD = sC + KY * KX;
    const float* sDA = sC + 2 * KY * KX;
    const float* sDD = sC + 3 * KY * KX;
    // synthesis taps of the (even, odd) output pair: (H_[2m], H_[2m+1]) and (G_[2m], G_[2m+1])
    float2 hp[T / 2], gp[T / 2];
#pragma unroll
    for (int m = 0; m < T / 2; ++m) {
        hp[m] = make_float2(H[2 * m], H[2 * m + 1]);
        gp[m] = make_float2(H[T - 1 - 2 * m], -H[T - 2 - 2 * m]);
    }
    // along y: item = output rows 4 q2 .. 4 q2 + 3 (pairs q = 2 q2, 2 q2 + 1) of coefficient column i;
    // pair q: x[2q + e] = sum_m H_[e + 2m] a[q + (T-2)/2 - m] + G_[e + 2m] d[...] (compile-time taps),
    // coefficient rows 2 q2 .. 2 q2 + T/2 loaded once
    for (int e = tid; e < (VS_Y / 4) * KX; e += 256) {
        const int q2 = e / KX, i = e - q2 * KX;
        float ca[T / 2 + 1], cad[T / 2 + 1], cda[T / 2 + 1], cdd[T / 2 + 1];
#pragma unroll
        for (int j = 0; j <= T / 2; ++j) {
            const int o = (2 * q2 + j) * KX + i;
            ca[j] = sA[o];
            cad[j] = sAD[o];
            cda[j] = sDA[o];
            cdd[j] = sDD[o];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {   // q = 2 q2 + h: rows j = h + (T-2)/2 - m relative to 2 q2
            float2 x0 = make_float2(0.f, 0.f), x1 = x0;   // (even, odd) output rows
#pragma unroll
            for (int m = 0; m < T / 2; ++m) {
                const int j = h + (T - 2) / 2 - m;
                x0 = ffma2(ca[j], hp[m], x0);
                x0 = ffma2(cad[j], gp[m], x0);
                x1 = ffma2(cda[j], hp[m], x1);
                x1 = ffma2(cdd[j], gp[m], x1);
            }
            const int r = 4 * q2 + 2 * h;
            sX0[r * KXP + i] = x0.x;
            sX0[(r + 1) * KXP + i] = x0.y;
            sX1[r * KXP + i] = x1.x;
            sX1[(r + 1) * KXP + i] = x1.y;
        }
    }
    __syncthreads();
    PRNU_STRESS(44);
    // along x: item = 8 output pixels 8 q4 .. 8 q4 + 7 (pairs q = 4 q4 + h) of row u; X columns
    // 4 q4 .. 4 q4 + T/2 + 2 by float4; lanes on consecutive items
    float* out = p.out[0] + (size_t)b * p.out_bstride;
    const bool v4 = (p.out_pitch % 4 == 0) && ((uintptr_t)out % 16 == 0);
    for (int e = tid; e < VS_Y * (VS_X / 8); e += 256) {
        const int u = e / (VS_X / 8), q4 = e - u * (VS_X / 8);
        const int gy = ty0 + u, gx = tx0 + 8 * q4;
        if (gy >= p.oH || gx >= p.oW) continue;
        float x0[4 * NLD], x1[4 * NLD];
#pragma unroll
        for (int k = 0; k < NLD; ++k) {
            const float4 a = *reinterpret_cast<const float4*>(sX0 + u * KXP + 4 * q4 + 4 * k);
            const float4 c = *reinterpret_cast<const float4*>(sX1 + u * KXP + 4 * q4 + 4 * k);
            x0[4 * k] = a.x; x0[4 * k + 1] = a.y; x0[4 * k + 2] = a.z; x0[4 * k + 3] = a.w;
            x1[4 * k] = c.x; x1[4 * k + 1] = c.y; x1[4 * k + 2] = c.z; x1[4 * k + 3] = c.w;
        }
        float o8[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {   // pair q = 4 q4 + h: X columns h + (T-2)/2 - m relative to 4 q4
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int m = 0; m < T / 2; ++m) {
                acc = ffma2(x0[h + (T - 2) / 2 - m], hp[m], acc);
                acc = ffma2(x1[h + (T - 2) / 2 - m], gp[m], acc);
            }
            o8[2 * h] = acc.x;
            o8[2 * h + 1] = acc.y;
        }
        float* o = out + (size_t)gy * p.out_pitch + gx;
        if (v4 && gx + 8 <= p.oW) {
            reinterpret_cast<float4*>(o)[0] = make_float4(o8[0], o8[1], o8[2], o8[3]);
            reinterpret_cast<float4*>(o)[1] = make_float4(o8[4], o8[5], o8[6], o8[7]);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (gx + k < p.oW) o[k] = o8[k];
        }
    }
}

template <int T, int MODE>
static int var_tile_launch(bool syn, const VarTile& p, int nb, cudaStream_t st) {
    static DeviceFlags attr[2];
    int rc;
    if (syn) {
        if ((rc = set_smem_attr((const void*)k_var_syn2d<T, MODE>, var_syn2d_smem<T>(), attr[1]))) return rc;
        const dim3 g((unsigned)((p.oW + VS_X - 1) / VS_X), (unsigned)((p.oH + var_vs_y<T>() - 1) / var_vs_y<T>()),
                     (unsigned)nb);
        k_var_syn2d<T, MODE><<<g, 256, var_syn2d_smem<T>(), st>>>(p);
    } else {
        if ((rc = set_smem_attr((const void*)k_var_ana2d<T, MODE>, var_ana2d_smem<T>(), attr[0]))) return rc;
        const dim3 g((unsigned)((p.nW + VT_X - 1) / VT_X), (unsigned)((p.nH + VT_Y - 1) / VT_Y), (unsigned)nb);
        k_var_ana2d<T, MODE><<<g, 256, var_ana2d_smem<T>(), st>>>(p);
    }
    return PRNU_OK;
}

static int var_tile_dispatch(int taps, int mode, bool syn, const VarTile& p, int nb, cudaStream_t st) {
    if (nb > 65535) return fail(PRNU_INVALID_ARG, "variant: more than 65535 frames in one launch");
    if (taps == 8) return mode == VM_SYM ? var_tile_launch<8, VM_SYM>(syn, p, nb, st) : var_tile_launch<8, VM_PER>(syn, p, nb, st);
    return mode == VM_SYM ? var_tile_launch<16, VM_SYM>(syn, p, nb, st) : var_tile_launch<16, VM_PER>(syn, p, nb, st);
}

template <int T>
static void var_launch(bool syn, int ax, const VarPass& p, int nb, cudaStream_t st) {
    if (ax == 0) {   // rows: shared-memory staged
        const dim3 g((unsigned)((p.nout + VR_OUT - 1) / VR_OUT), (unsigned)((p.other + VAR_RY - 1) / VAR_RY),
                     (unsigned)(nb * p.nplanes));
        const size_t sm = 2 * sizeof(float) * var_row_span<T>(p.s);
        if (syn) k_var_row_syn<T><<<g, 128, sm, st>>>(p);
        else k_var_row_ana<T><<<g, 128, sm, st>>>(p);
        return;
    }
    // columns: polyphase runs, ceil(nout / (8 s)) blocks of 8 s rows x s phases
    const dim3 grid((unsigned)((p.other + 127) / 128), (unsigned)(((p.nout + 8 * p.s - 1) / (8 * p.s)) * p.s),
                    (unsigned)(nb * p.nplanes));
    if (syn) k_var_syn_col<T><<<grid, 128, 0, st>>>(p);
    else k_var_ana_col<T><<<grid, 128, 0, st>>>(p);
}

static void var_dispatch(int taps, bool syn, int ax, const VarPass& p, int nb, cudaStream_t st) {
    if (taps == 8) var_launch<8>(syn, ax, p, nb, st);
    else var_launch<16>(syn, ax, p, nb, st);
}

// ------------------------------------------------------------------ geometry / workspace
struct VarGeom {
    int T, mode, L;
    int H, W;
    int inH[8], inW[8];     // real input extent of level l (l = 1..L)
    int perH[8], perW[8];   // period of the level's input (== real except padded level 1)
    int nH[8], nW[8];       // subband extent of level l
    int P[8];               // row pitch of level l's planes (the tile path: a multiple of 8 floats)
    size_t sub_off[8];      // offset of level l's three noise planes (floats, per frame)
    size_t scratch, approx, noise;   // floats per frame: one scratch plane, one approximation plane, all noise
};

static VarGeom var_geom(int H, int W, int levels, int taps, int boundary, int transform) {
    VarGeom g{};
    g.T = taps;
    g.mode = transform ? VM_SWT : boundary ? VM_PER : VM_SYM;
    g.L = levels;
    g.H = H;
    g.W = W;
    const int m = 1 << levels;
    int h = H, w = W;
    size_t off = 0;
    for (int l = 1; l <= levels; ++l) {
        g.inH[l] = h;
        g.inW[l] = w;
        g.perH[l] = (g.mode == VM_PER && l == 1) ? (H + m - 1) / m * m : h;
        g.perW[l] = (g.mode == VM_PER && l == 1) ? (W + m - 1) / m * m : w;
        if (g.mode == VM_SWT) {
            g.nH[l] = h;
            g.nW[l] = w;
        } else if (g.mode == VM_PER) {
            g.nH[l] = g.perH[l] / 2;
            g.nW[l] = g.perW[l] / 2;
        } else {
            g.nH[l] = (h + taps - 1) / 2;
            g.nW[l] = (w + taps - 1) / 2;
        }
        // 32-byte rows for the tile kernels' vector accesses; dense for the separable (SWT) passes
        g.P[l] = g.mode == VM_SWT ? g.nW[l] : (int)align_up((size_t)g.nW[l], 8);
        g.sub_off[l] = off;
        off += 3 * (size_t)g.nH[l] * g.P[l];
        h = g.nH[l];
        w = g.nW[l];
    }
    g.noise = off;
    size_t sc = 0, ap = 0;
    for (int l = 1; l <= levels; ++l) {
        sc = std::max(sc, (size_t)std::max(g.inH[l], g.perH[l]) * g.nW[l]);
        ap = std::max(ap, (size_t)g.nH[l] * g.P[l]);
    }
    g.scratch = align_up(sc, 64);
    g.approx = align_up(ap, 64);
    g.noise = align_up(g.noise, 64);
    return g;
}

// per frame: 2 scratch + 2 approximation (ping-pong) + 3 raw details + all noise planes
static size_t var_floats_per_frame(const VarGeom& g) { return 2 * g.scratch + 5 * g.approx + g.noise; }

size_t variant_workspace_bytes(int batch, int H, int W, int levels, int taps, int boundary, int transform) {
    const VarGeom g = var_geom(H, W, levels, taps, boundary, transform);
    return align_up(sizeof(float) * var_floats_per_frame(g) * (size_t)batch, 256);
}

int variant_filter(int taps, double* h) {
    if (taps == 8) {
        const float h8[8] = {PRNU_H0, PRNU_H1, PRNU_H2, PRNU_H3, PRNU_H4, PRNU_H5, PRNU_H6, PRNU_H7};
        for (int i = 0; i < 8; ++i) h[i] = h8[i];
        return PRNU_OK;
    }
    if (taps == 16) {
        for (int i = 0; i < 16; ++i) h[i] = (double)(float)kDb8[i];
        return PRNU_OK;
    }
    return fail(PRNU_BAD_PARAMETER, "taps must be 8 or 16");
}

// Decimated variants through the fused tile kernels: per level one analysis launch
// (input -> A, ad, da, dd), the shrink, and per level one synthesis launch.
template <typename NoiseFn>
static int run_residual_variant_tiles(const VarGeom& g, const float* in, int nb, int H, int W, const ShrinkParams& sp,
                                      float* W_out, float* const (&A)[2], float* const (&R)[3], NoiseFn noise,
                                      cudaStream_t st) {
    int rc;
    const float* cur = in;
    long long cur_bs = (long long)H * W;
    int cur_pitch = W;
    for (int l = 1; l <= g.L; ++l) {
        const int nHl = g.nH[l], nWl = g.nW[l], Pl = g.P[l];
        {
            VarTile p{};
            p.in = cur;
            p.out[0] = A[l & 1];
            p.out[1] = R[1];   // ad = hi_y(lo_x)
            p.out[2] = R[0];   // da = lo_y(hi_x)
            p.out[3] = R[2];   // dd
            p.in_bstride = cur_bs;
            p.in_pitch = cur_pitch;
            p.out_bstride = (long long)nHl * Pl;
            p.out_pitch = Pl;
            p.N_y = g.inH[l];
            p.Np_y = g.perH[l];
            p.N_x = g.inW[l];
            p.Np_x = g.perW[l];
            p.nH = nHl;
            p.nW = nWl;
            KTimer kt("variant_ana", st);
            if ((rc = var_tile_dispatch(g.T, g.mode, false, p, nb, st))) return rc;
        }
        count_launch();
        if ((rc = check_launch("k_var_ana2d"))) return rc;
        {
            const float* src[3] = {R[0], R[1], R[2]};
            float* dst[3] = {noise(l, 0), noise(l, 1), noise(l, 2)};
            KTimer kt("variant_shrink", st);
            if ((rc = launch_shrink_strip(src, dst, (long long)nHl * Pl, Pl, nHl, nWl, sp, nb, st))) return rc;
        }
        count_launch();
        if ((rc = check_launch("k_shrink (variant)"))) return rc;
        cur = A[l & 1];
        cur_bs = (long long)nHl * Pl;
        cur_pitch = Pl;
    }
    for (int l = g.L; l >= 1; --l) {
        const int nHl = g.nH[l], nWl = g.nW[l], Pl = g.P[l];
        VarTile p{};
        p.c[0] = l == g.L ? nullptr : A[l & 1];
        p.c[1] = noise(l, 1);
        p.c[2] = noise(l, 0);
        p.c[3] = noise(l, 2);
        p.out[0] = l == 1 ? W_out : A[(l - 1) & 1];
        p.in_bstride = (long long)nHl * Pl;
        p.in_pitch = Pl;
        p.nH = nHl;
        p.nW = nWl;
        p.oH = l == 1 ? H : g.inH[l];
        p.oW = l == 1 ? W : g.inW[l];
        p.out_pitch = l == 1 ? W : g.P[l - 1];   // the level l-1 approximation plane (pitched)
        p.out_bstride = (long long)p.oH * p.out_pitch;
        {
            KTimer kt("variant_syn", st);
            if ((rc = var_tile_dispatch(g.T, g.mode, true, p, nb, st))) return rc;
        }
        count_launch();
        if ((rc = check_launch("k_var_syn2d"))) return rc;
    }
    return PRNU_OK;
}

int run_residual_variant(const float* in, int nb, int H, int W, int levels, int taps, int boundary, int transform,
                         const ShrinkParams& sp, float* W_out, float* ws, cudaStream_t st) {
    const VarGeom g = var_geom(H, W, levels, taps, boundary, transform);
    // each buffer holds nb frames; a plane of level l is stored densely, frame stride
    // nH_l nW_l (the buffers are sized for level 1, the largest)
    float* X[2] = {ws, ws + g.scratch * nb};
    float* A[2] = {ws + 2 * g.scratch * nb, ws + (2 * g.scratch + g.approx) * nb};
    float* R[3] = {A[1] + g.approx * nb, A[1] + 2 * g.approx * nb, A[1] + 3 * g.approx * nb};
    float* NZ = A[1] + 4 * g.approx * nb;
    auto noise = [&](int l, int k) { return NZ + (g.sub_off[l] + (size_t)k * g.nH[l] * g.P[l]) * nb; };
    int rc;
    if (g.mode != VM_SWT) return run_residual_variant_tiles(g, in, nb, H, W, sp, W_out, A, R, noise, st);
    const float* cur = in;
    long long cur_bs = (long long)H * W;
    int cur_pitch = W;
    for (int l = 1; l <= levels; ++l) {
        const int s = 1 << (l - 1);
        const int nHl = g.nH[l], nWl = g.nW[l];
        {   // rows: cur [inH][inW] -> X0 = lo_x, X1 = hi_x  [inH][nW]
            VarPass p{};
            p.in[0] = cur;
            p.out[0] = X[0];
            p.out[1] = X[1];
            p.in_bstride = cur_bs;
            p.in_pitch = cur_pitch;
            p.out_bstride = (long long)g.scratch;
            p.out_pitch = nWl;
            p.N = g.inW[l];
            p.nout = nWl;
            p.other = g.inH[l];
            p.s = s;
            p.nplanes = 1;
            KTimer kt("variant_ana_x", st);
            var_dispatch(taps, false, 0, p, nb, st);
        }
        count_launch();
        if ((rc = check_launch("k_var_ana (x)"))) return rc;
        {   // columns: X0 -> (aa, ad), X1 -> (da, dd)   [nH][nW]
            VarPass p{};
            p.in[0] = X[0];
            p.in[1] = X[1];
            p.out[0] = A[l & 1];
            p.out[1] = R[1];
            p.out[2] = R[0];
            p.out[3] = R[2];
            p.in_bstride = (long long)g.scratch;
            p.in_pitch = nWl;
            p.out_bstride = (long long)nHl * nWl;
            p.out_pitch = nWl;
            p.N = g.inH[l];
            p.nout = nHl;
            p.other = nWl;
            p.s = s;
            p.nplanes = 2;
            KTimer kt("variant_ana_y", st);
            var_dispatch(taps, false, 1, p, nb, st);
        }
        count_launch();
        if ((rc = check_launch("k_var_ana (y)"))) return rc;
        {   // shrink: raw (da, ad, dd) -> noise-domain planes of level l (R-10)
            const float* src[3] = {R[0], R[1], R[2]};
            float* dst[3] = {noise(l, 0), noise(l, 1), noise(l, 2)};
            KTimer kt("variant_shrink", st);
            if ((rc = launch_shrink_strip(src, dst, (long long)nHl * nWl, nWl, nHl, nWl, sp, nb, st))) return rc;
        }
        count_launch();
        if ((rc = check_launch("k_shrink (variant)"))) return rc;
        cur = A[l & 1];
        cur_bs = (long long)nHl * nWl;
        cur_pitch = nWl;
    }
    for (int l = levels; l >= 1; --l) {
        const int s = 1 << (l - 1);
        const int nHl = g.nH[l], nWl = g.nW[l];
        const int outH = l == 1 ? H : g.inH[l], outW = l == 1 ? W : g.inW[l];
        const float* approx = l == levels ? nullptr : A[l & 1];
        {   // columns: (approx, ad) -> X0, (da, dd) -> X1   [outH][nW]
            VarPass p{};
            p.in[0] = approx;
            p.in[1] = noise(l, 1);
            p.in[2] = noise(l, 0);
            p.in[3] = noise(l, 2);
            p.out[0] = X[0];
            p.out[1] = X[1];
            p.in_bstride = (long long)nHl * nWl;
            p.in_pitch = nWl;
            p.out_bstride = (long long)g.scratch;
            p.out_pitch = nWl;
            p.N = nHl;
            p.nout = outH;
            p.other = nWl;
            p.s = s;
            p.nplanes = 2;
            KTimer kt("variant_syn_y", st);
            var_dispatch(taps, true, 1, p, nb, st);
        }
        count_launch();
        if ((rc = check_launch("k_var_syn (y)"))) return rc;
        {   // rows: (X0, X1) -> approx of level l-1 (or W at l = 1)   [outH][outW]
            VarPass p{};
            p.in[0] = X[0];
            p.in[1] = X[1];
            p.out[0] = l == 1 ? W_out : A[(l - 1) & 1];
            p.in_bstride = (long long)g.scratch;
            p.in_pitch = nWl;
            p.out_bstride = l == 1 ? (long long)H * W : (long long)outH * outW;
            p.out_pitch = outW;
            p.N = nWl;
            p.nout = outW;
            p.other = outH;
            p.s = s;
            p.nplanes = 1;
            KTimer kt("variant_syn_x", st);
            var_dispatch(taps, true, 0, p, nb, st);
        }
        count_launch();
        if ((rc = check_launch("k_var_syn (x)"))) return rc;
    }
    return PRNU_OK;
}

}  // namespace prnu
