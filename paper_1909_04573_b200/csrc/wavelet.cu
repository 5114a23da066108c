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
#include <type_traits>

#include "common.cuh"
#include "tma.cuh"

namespace prnu {

// Synthesis filter pairs (H(6-2m), H(7-2m)) and (G(6-2m), G(7-2m)), m = 0..3, in
// constant memory: FFMA2 takes them as uniform operands.
__constant__ float2 c_sh[4] = {{PRNU_H6, PRNU_H7}, {PRNU_H4, PRNU_H5}, {PRNU_H2, PRNU_H3}, {PRNU_H0, PRNU_H1}};
__constant__ float2 c_sg[4] = {{PRNU_H1, -PRNU_H0}, {PRNU_H3, -PRNU_H2}, {PRNU_H5, -PRNU_H4}, {PRNU_H7, -PRNU_H6}};

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
static_assert(SC_Y * SC_BW <= SC_PS && (SC_PS * 4) % 128 == 0, "TMA plane tile layout");

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
    int out_v8;                  // MODE 0: out, out_pitch, out_bstride allow 32-byte aligned 8-float stores
    const void* I;               // MODE 1: frames the residuals come from (u8, u16 SDA sums, fp32)
    long long i_bstride;
    int i_pitch;
    double* num;                 // MODE 1: fp64 accumulators [NH][acc_pitch]
    double* den;
    int acc_pitch;
    int acc_v4;                  // num, den and acc_pitch allow 32-byte aligned 4-double accesses
    float div_d, div_r;          // u16 SDA sums: S = RN(sum / d), d and RN(1/d) (R-11)
};

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
// For u16 SDA group sums the frame is S = RN(sum / d), recomputed here with the same
// exact sequence as the analysis (sda_div), so both kernels see the oracle's fp32 S.
// Per-pixel order is ascending frame order.
constexpr int SA_STAGE_COEF = 4 * SC_PS;           // floats per stage (4 planes)
// L/H plane pitch.  The row pass maps lane l to row 4w + (l >> 3), column group l & 7, so
// its LDS.128 (8 lanes: one row, 128 contiguous bytes) and the I-tile loads (a half-warp:
// two 64-byte rows) are conflict-free at any pitch; 36 (== 4 mod 32) spreads the column
// pass's halo items (coefficient columns 32 .. 35 of 4-row groups sg, one warp: banks
// 16 sg + k) over 8 banks (4-way) where 40 put them on 4 (7-way).
constexpr int SA_LP = 36;
// Swizzled planes (u8 accumulation and the plain inverse levels, where the shared memory
// for 4 CTAs/SM allows it): pitch 52 (== 20 mod 32) and row t stored 4 ((t >> 3) & 3)
// columns to the right.  A halo item's row 4 sg + c then sits in bank
// 16 (sg & 1) + 4 ((sg >> 1) & 3) + 20 c + (k - 32) (mod 32): the 8 row groups on 8
// distinct bank quads, so the halo warp's stores are conflict-free (4-way at pitch 36);
// the main items (32 consecutive columns of one row) and the row pass's LDS.128 (8 lanes:
// 128 contiguous bytes of one row) stay conflict-free, and the shift is a per-thread
// constant (no instruction per frame).
constexpr int SA_LP_SWZ = 52;
template <typename TI, int MODE>
__host__ __device__ constexpr int sacc_lp() {
    return (MODE == 0 || (sizeof(TI) == 1 && !std::is_same<TI, u8pair>::value)) ? SA_LP_SWZ : SA_LP;
}
template <int TY, typename TI, int MODE = 1>
constexpr size_t sacc_smem_bytes() {
    return 2 * SA_STAGE_COEF * sizeof(float) + (MODE ? 3 * TY * ST_X * sizeof(TI) : 0) +
           2 * 2 * TY * sacc_lp<TI, MODE>() * sizeof(float) + 2 * sizeof(uint64_t);
}
static_assert(4 * (sacc_smem_bytes<32, uint8_t, 1>() + 1024) <= 228 * 1024 &&
              4 * (sacc_smem_bytes<32, float, 0>() + 1024) <= 228 * 1024, "4 CTAs/SM with the swizzled planes");

// MODE 1: accumulate (frames 0 .. nb-1, one CTA per tile); MODE 0: plain inverse
// level written to a.out (frames [z * frames_per_cta, ...) per CTA, no I tiles).
template <int TY, typename TI, int MODE = 1>
__global__ void __launch_bounds__(256, 4) k_synth_acc2(const __grid_constant__ SynthMaps maps,
                                                       const __grid_constant__ CUtensorMap imap, SynthArgs a) {
    constexpr int CY = TY / 2 + 3;   // coefficient rows of a TY-row tile
    static_assert(TY % 4 == 0 && TY <= 32, "tile height");
    // SDA pairs (d = 2): the I tile is both frames of the group, [2][TY][ST_X] bytes (one depth-2 box)
    constexpr bool PAIR = std::is_same<TI, u8pair>::value;
    constexpr int IDEP = PAIR ? 2 : 1;
    extern __shared__ __align__(128) float smem[];
    // coefficient ring of 2 stages (frame f in stage f & 1, released after its
    // column pass), I-tile ring of 3 (frame f in f % 3, released after its row
    // pass): frame f+2 is issued at the barrier of frame f, two frames ahead.
    float* coef0 = smem;                                                      // [2][4][SC_PS]
    TI* itile0 = reinterpret_cast<TI*>(smem + 2 * SA_STAGE_COEF);             // [3][TY][ST_X] (MODE 1)
    constexpr int LP = sacc_lp<TI, MODE>();
    constexpr bool SWZ = LP == SA_LP_SWZ;
    float* sL0 = reinterpret_cast<float*>(itile0 + (MODE ? 3 * TY * ST_X : 0));   // [2][2][TY][LP]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sL0 + 2 * 2 * TY * LP);
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
        if (MODE) tma_load_3d(itile0 + (f % 3) * TY * ST_X, &imap, tx0, ty0, IDEP * f, &bar[st]);
    };
    if (tid == 0) {
        if (nb > 0) issue(0);
        if (nb > 1) issue(1);
    }

    // row pass / accumulate mapping: warp w rows 4w .. 4w+3, lane -> (row 4w + (lane >> 3), 8 columns at 8 (lane & 7))
    const int lane = tid & 31, warp = tid >> 5;
    const int rt = 4 * warp + (lane >> 3), rg = lane & 7;
    const int gy = ty0 + rt, gx = tx0 + 8 * rg;
    const bool rowact = rt < TY;            // warp-uniform: the last warp idles in the row pass when TY = 28
    const bool rowok = rowact && gy < a.NH;
    double num[8];
    uint32_t den_i[8];
    double den_d[8];
    // NUM / DEN rows of this thread's 8 pixels: two 256-bit accesses each when 32-byte aligned
    // (scalar fp64 accesses at a 64-byte lane stride touch every sector 4 times)
    const bool acc_v = MODE && rowok && gx + 8 <= a.NW && a.acc_v4;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        num[k] = 0.0;
        den_i[k] = 0u;
        den_d[k] = 0.0;
    }
    if (acc_v) {
        const double* np = a.num + (size_t)gy * a.acc_pitch + gx;
        double t0[4], t1[4];
        ld_global_v4d(np, t0);
        ld_global_v4d(np + 4, t1);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            num[k] = t0[k];
            num[k + 4] = t1[k];
        }
        if (sizeof(TI) != 1) {   // u16 / fp32 / pairs: the fp64 DEN accumulator in registers
            const double* dp = a.den + (size_t)gy * a.acc_pitch + gx;
            ld_global_v4d(dp, t0);
            ld_global_v4d(dp + 4, t1);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                den_d[k] = t0[k];
                den_d[k + 4] = t1[k];
            }
        }
    } else if (MODE) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            num[k] = (rowok && gx + k < a.NW) ? a.num[(size_t)gy * a.acc_pitch + gx + k] : 0.0;
            if (sizeof(TI) != 1) den_d[k] = (rowok && gx + k < a.NW) ? a.den[(size_t)gy * a.acc_pitch + gx + k] : 0.0;
        }
    }
    // column-pass items (frame-invariant): item it = (coefficient column k, output rows 4 sg .. 4 sg + 3);
    // with at most one item per thread (TY <= 28) it is computed once here
    constexpr int NITEM = SC_X * (TY / 4);
    auto item_k = [](int it) { return it < 32 * (TY / 4) ? (it & 31) : 32 + (it - 32 * (TY / 4)) % (SC_X - 32); };
    auto item_sg = [](int it) { return it < 32 * (TY / 4) ? (it >> 5) : (it - 32 * (TY / 4)) / (SC_X - 32); };
    const int ck = item_k(tid), csg = item_sg(tid);
    // an item's coefficient-tile load offset (row 2 sg) and plane store offset (row 4 sg, swizzle shift)
    auto ld_off = [](int k, int sg) { return 2 * sg * SC_BW + k; };
    auto st_off = [](int k, int sg) { return 4 * sg * LP + k + (SWZ ? 4 * ((sg >> 1) & 3) : 0); };
    const int cld = ld_off(ck, csg), cst = st_off(ck, csg);
    // row-pass plane offset of this thread's 8 columns (swizzled planes: row rt shifted 4 ((rt >> 3) & 3))
    const int roff = rt * LP + (SWZ ? 4 * ((rt >> 3) & 3) : 0) + 4 * rg;

    for (int f = 0; f < nb; ++f) {
        const int st = f & 1;
        PRNU_STRESS(11);
        mbar_wait(&bar[st], (f >> 1) & 1);
        const float* c = coef0 + st * SA_STAGE_COEF;
        float* sLo = sL0 + (f & 1) * 2 * TY * LP;
        float* sHi = sLo + TY * LP;
        // column pass: Lx = synth_y(A, ad), Hx = synth_y(da, dd); item = (coefficient column k, 4 output rows)
        for (int it = tid; it < NITEM; it += 256) {
            PRNU_DCHECK(item_k(it) < SC_X && 2 * item_sg(it) + 4 < CY && 4 * item_sg(it) + 3 < TY);
            const int lo0 = NITEM <= 256 ? cld : ld_off(item_k(it), item_sg(it));
            const int so0 = NITEM <= 256 ? cst : st_off(item_k(it), item_sg(it));
            float va[5], vda[5], vad[5], vdd[5];
#pragma unroll
            for (int m = 0; m < 5; ++m) {
                const int r = lo0 + m * SC_BW;
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
                const int o = so0 + 2 * q * LP;   // output row 4 sg + 2 q
                sLo[o] = l.x;
                sLo[o + LP] = l.y;
                sHi[o] = h.x;
                sHi[o + LP] = h.y;
            }
        }
        __syncthreads();   // L/H planes of frame f complete; every thread is past frame f-1
        PRNU_STRESS(12);
        if (tid == 0 && f + 2 < nb) {
            fence_proxy_async();
            issue(f + 2);   // coefficient stage of frame f, I stage of frame f-1: both consumed
        }
        if (!rowact) continue;
        // row pass of 8 pixels + accumulation
        float vl[8], vh[8];
        {   // columns 4 rg .. 4 rg + 7 (the 8th unused): two LDS.128 per plane
            const float4* pl = reinterpret_cast<const float4*>(sLo + roff);
            const float4* ph = reinterpret_cast<const float4*>(sHi + roff);
            const float4 l0 = pl[0], l1 = pl[1], h0 = ph[0], h1 = ph[1];
            vl[0] = l0.x; vl[1] = l0.y; vl[2] = l0.z; vl[3] = l0.w; vl[4] = l1.x; vl[5] = l1.y; vl[6] = l1.z; vl[7] = l1.w;
            vh[0] = h0.x; vh[1] = h0.y; vh[2] = h0.z; vh[3] = h0.w; vh[4] = h1.x; vh[5] = h1.y; vh[6] = h1.z; vh[7] = h1.w;
        }
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
                if (gx + 8 <= a.NW && a.out_v8) {   // one 256-bit store per thread (whole sectors)
                    st_global_v8(orow, w);
                } else if (gx + 8 <= a.NW && ((a.out_pitch & 3) == 0)) {
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
        if constexpr (PAIR) {   // S = (b0 + b1) / 2 exactly; I^2 = s^2 / 4 summed as the integer s^2
            const uint8_t* ib = reinterpret_cast<const uint8_t*>(itile0 + (f % 3) * TY * ST_X) + rt * ST_X + 8 * rg;
            const uint2 i0 = *reinterpret_cast<const uint2*>(ib);
            const uint2 i1 = *reinterpret_cast<const uint2*>(ib + TY * ST_X);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t sb = __byte_perm(k < 4 ? i0.x : i0.y, 0, 0x4440u | (uint32_t)(k & 3)) +
                                    __byte_perm(k < 4 ? i1.x : i1.y, 0, 0x4440u | (uint32_t)(k & 3));
                den_i[k] += sb * sb;   // <= 8192 groups between flushes: < 2^32
                const double xd = 0.5 * (__hiloint2double(0x43300000, (int)sb) - 4503599627370496.0);
                num[k] = fma((double)w[k], xd, num[k]);   // exact product, one fp64 rounding
            }
            if ((f & 8191) == 8191) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    den_d[k] += 0.25 * (double)den_i[k];   // exact (multiples of 1/4 below 2^51)
                    den_i[k] = 0u;
                }
            }
        } else if (sizeof(TI) == 1) {
            const uint2 iv = *reinterpret_cast<const uint2*>(irow);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t xb = __byte_perm(k < 4 ? iv.x : iv.y, 0, 0x4440u | (uint32_t)(k & 3));
                den_i[k] += xb * xb;
                // exact integer -> double: (2^52 + x) - 2^52
                const double xd = __hiloint2double(0x43300000, (int)xb) - 4503599627370496.0;
                num[k] = fma((double)w[k], xd, num[k]);   // exact product, one fp64 rounding
            }
        } else if (sizeof(TI) == 2) {   // exact SDA group sums: S = RN(sum / d) (R-11)
            const uint4 iw = *reinterpret_cast<const uint4*>(irow);
            const uint32_t w4[4] = {iw.x, iw.y, iw.z, iw.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float sk = sda_div(u16_to_f32(w4[k >> 1], k & 1), a.div_d, a.div_r);
                const double xd = (double)sk;
                num[k] = fma((double)w[k], xd, num[k]);
                den_d[k] = fma(xd, xd, den_d[k]);
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
    PRNU_DCHECK(!rowok || (gy >= 0 && gy < a.NH));
    if (MODE && rowok) {
        double dv[8];
        if (sizeof(TI) == 1 && !PAIR) {   // u8: DEN += the wave's exact integer sum (read here, once)
            if (acc_v) {
                double t0[4], t1[4];
                const double* dp = a.den + (size_t)gy * a.acc_pitch + gx;
                ld_global_v4d(dp, t0);
                ld_global_v4d(dp + 4, t1);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    dv[k] = t0[k] + (double)den_i[k];
                    dv[k + 4] = t1[k] + (double)den_i[k + 4];
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    dv[k] = gx + k < a.NW ? a.den[(size_t)gy * a.acc_pitch + gx + k] + (double)den_i[k] : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) dv[k] = PAIR ? den_d[k] + 0.25 * (double)den_i[k] : den_d[k];
        }
        if (acc_v) {
            double* np = a.num + (size_t)gy * a.acc_pitch + gx;
            double* dp = a.den + (size_t)gy * a.acc_pitch + gx;
            const double n0[4] = {num[0], num[1], num[2], num[3]}, n1[4] = {num[4], num[5], num[6], num[7]};
            const double d0[4] = {dv[0], dv[1], dv[2], dv[3]}, d1[4] = {dv[4], dv[5], dv[6], dv[7]};
            st_global_v4d(np, n0);
            st_global_v4d(np + 4, n1);
            st_global_v4d(dp, d0);
            st_global_v4d(dp + 4, d1);
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (gx + k < a.NW) {
                    a.num[(size_t)gy * a.acc_pitch + gx + k] = num[k];
                    a.den[(size_t)gy * a.acc_pitch + gx + k] = dv[k];
                }
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

bool encode_tensor_map_3d(CUtensorMap* map, CUtensorMapDataType dt, size_t elem_bytes, const void* base, uint64_t cols,
                          uint64_t rows, uint64_t depth, uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t box_w,
                          uint32_t box_h, uint32_t box_d) {
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
    cuuint32_t box[3] = {box_w, box_h, box_d};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Tensor maps over the four level-l planes of `nb` frames, box SC_BW x box_rows.
static int synth_maps(const Pyramid& p, const PyramidBuffers& pb, int l, int nb, bool has_A, int box_rows,
                      SynthMaps* m) {
    const uint64_t pitch = (uint64_t)p.pitch[l] * 4, plane = (uint64_t)pb.bstride[l] * 4;
    const float* src[4] = {pb.approx[l], pb.det[l][0], pb.det[l][1], pb.det[l][2]};
    CUtensorMap* dst[4] = {&m->A, &m->d0, &m->d1, &m->d2};
    for (int i = 0; i < 4; ++i) {
        if (i == 0 && !has_A) {
            *dst[0] = CUtensorMap{};
            continue;
        }
        if (!encode_tensor_map_3d(dst[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, src[i], p.nW[l], p.nH[l], nb, pitch,
                                  plane, SC_BW, box_rows))
            return fail(PRNU_CUDA_ERROR, "cuTensorMapEncodeTiled failed (pyramid plane)");
    }
    return PRNU_OK;
}

// One inverse level (MODE 0 of k_synth_acc2, 32-row tiles) from the level-l planes
// into `out` [nb][NH][out_pitch]: frames split over grid.z, enough CTAs for about
// 4 waves of 4 CTAs per SM, at least 4 frames per CTA to amortise the TMA pipeline.
static int synth_level(const Pyramid& p, const PyramidBuffers& pb, int l, int nb, float* out, long long out_bstride,
                       int out_pitch, cudaStream_t st) {
    static DeviceFlags attr;
    int rc;
    if ((rc = set_smem_attr((const void*)k_synth_acc2<32, float, 0>, sacc_smem_bytes<32, float, 0>(), attr)))
        return rc;
    SynthMaps m;
    const bool has_A = l < p.levels;
    if ((rc = synth_maps(p, pb, l, nb, has_A, 32 / 2 + 3, &m))) return rc;
    SynthArgs s{};
    s.has_A = has_A;
    s.NH = p.nH[l - 1];
    s.NW = p.nW[l - 1];
    s.nb = nb;
    s.out = out;
    s.out_bstride = out_bstride;
    s.out_pitch = out_pitch;
    s.out_v8 = ((uintptr_t)out % 32 == 0) && (out_pitch % 8 == 0) && (out_bstride % 8 == 0);
    const long long tiles = (long long)((s.NW + ST_X - 1) / ST_X) * ((s.NH + 31) / 32);
    const long long slots = 4LL * device_sm_count();
    s.frames_per_cta = (int)std::max<long long>(4, std::min<long long>(nb, tiles * nb / (slots * 4)));
    const int nz = (nb + s.frames_per_cta - 1) / s.frames_per_cta;
    if (nz > 65535 || (s.NH + 31) / 32 > 65535) return fail(PRNU_INVALID_ARG, "synthesis grid too large");
    dim3 grid((s.NW + ST_X - 1) / ST_X, (s.NH + 31) / 32, nz);
    KTimer kt(kSynthName[l], st);
    k_synth_acc2<32, float, 0><<<grid, 256, sacc_smem_bytes<32, float, 0>(), st>>>(m, CUtensorMap{}, s);
    count_launch();
    return check_launch("k_synth_acc2 (inverse level)");
}

// Analysis of all levels (lifting kernels, analysis.cu), then synthesis of levels
// L..2 (the level-1 synthesis is launched by the caller, fused or not with the
// accumulation).  Level 1 reads `in` (u8 frames, u16 SDA sums with div, or fp32).
template <typename TIn>
static int denoise_front(const TIn* in, long long in_bstride, int in_pitch, int nb, const Pyramid& p,
                         const PyramidBuffers& pb, const ShrinkParams& sp, const SdaDiv& div, cudaStream_t st) {
    int rc;
    const int L = p.levels;
    for (int l = 1; l <= L; ++l) {
        float* ll = (l < L) ? pb.approx[l] : nullptr;
        const long long ob = (long long)pb.bstride[l];
        {
            constexpr bool PAIR = std::is_same<TIn, u8pair>::value;
            KTimer kt(l == 1 ? (PAIR ? "analysis_l1_pair" : sizeof(TIn) == 1 ? "analysis_l1_u8"
                                : sizeof(TIn) == 2 ? "analysis_l1_u16" : "analysis_l1_f32")
                             : kAnalysisName[l],
                      st);
            if (l == 1 && PAIR)
                rc = launch_analysis_lift_pair(reinterpret_cast<const uint8_t*>(in), in_bstride, in_pitch, p.nH[0],
                                               p.nW[0], ll, pb.det[1][0], pb.det[1][1], pb.det[1][2], ob, p.pitch[1],
                                               p.nH[1], p.nW[1], sp, nb, st);
            else if (l == 1 && sizeof(TIn) == 1)
                rc = launch_analysis_lift_u8(reinterpret_cast<const uint8_t*>(in), in_bstride, in_pitch, p.nH[0],
                                             p.nW[0], ll, pb.det[1][0], pb.det[1][1], pb.det[1][2], ob, p.pitch[1],
                                             p.nH[1], p.nW[1], sp, nb, st);
            else if (l == 1 && sizeof(TIn) == 2)
                rc = launch_analysis_lift_u16(reinterpret_cast<const uint16_t*>(in), in_bstride, in_pitch, p.nH[0],
                                              p.nW[0], ll, pb.det[1][0], pb.det[1][1], pb.det[1][2], ob, p.pitch[1],
                                              p.nH[1], p.nW[1], sp, div, nb, st);
            else if (l == 1 && sizeof(TIn) != 4)
                rc = fail(PRNU_INVALID_ARG, "denoise: unsupported level-1 input");
            else
                rc = launch_analysis_lift_f32(l == 1 ? reinterpret_cast<const float*>(in) : pb.approx[l - 1],
                                              l == 1 ? in_bstride : (long long)pb.bstride[l - 1],
                                              l == 1 ? in_pitch : p.pitch[l - 1], p.nH[l - 1], p.nW[l - 1], ll,
                                              pb.det[l][0], pb.det[l][1], pb.det[l][2], ob, p.pitch[l], p.nH[l],
                                              p.nW[l], sp, nb, st);
            if (rc) return rc;
        }
        count_launch();
        if ((rc = check_launch("k_analysis_lift"))) return rc;
    }
    for (int l = L; l >= 2; --l)
        if ((rc = synth_level(p, pb, l, nb, pb.approx[l - 1], (long long)pb.bstride[l - 1], p.pitch[l - 1], st)))
            return rc;
    return PRNU_OK;
}

template <typename TIn>
int run_residual(const TIn* in, int nb, int H, int W, const Pyramid& p, const ShrinkParams& sp, float* W_out,
                 float* ws_pyr, cudaStream_t st, int in_pitch) {
    if (in_pitch <= 0) in_pitch = W;
    PyramidBuffers pb = carve_pyramid(p, ws_pyr, nb);
    int rc = denoise_front<TIn>(in, (long long)H * in_pitch, in_pitch, nb, p, pb, sp, SdaDiv{}, st);
    if (rc) return rc;
    return synth_level(p, pb, 1, nb, W_out, (long long)H * W, W, st);
}

// Residuals of nb planes fused with the MLE accumulation (a4 + a5): the last inverse
// level adds W*I and I^2 to NUM/DEN in ascending frame order.  I = the planes the
// residuals come from: u8 frames (d = 1), u16 exact SDA group sums (2 <= d <= 257,
// S = RN(sum / d) recomputed in-kernel, R-11) or fp32 SDA frames (d > 257).  `in`
// and `I` rows must be TMA-stageable (16-byte pitch, frame stride and base; the
// extraction guarantees it by re-pitching).
// acc_wait (optional): event the accumulating launch must wait for (the previous
// wave's accumulation on another stream); acc_done (optional): recorded after it.
// frame_stride: elements between consecutive frames of `in`/`I` (k*H*pitch selects
// every k-th frame, f4 stride emulation).
template <typename TIn>
int run_residual_accumulate(const TIn* in, const TIn* I, int nb, int H, int W, const Pyramid& p,
                            const ShrinkParams& sp, const SdaDiv& div, double* num, double* den, float* ws_pyr,
                            cudaStream_t st, cudaEvent_t acc_wait, cudaEvent_t acc_done, long long frame_stride,
                            int in_pitch) {
    if (in_pitch <= 0) in_pitch = W;
    PyramidBuffers pb = carve_pyramid(p, ws_pyr, nb);
    int rc = denoise_front<TIn>(in, frame_stride, in_pitch, nb, p, pb, sp, div, st);
    if (rc) return rc;
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
    s.acc_v4 = ((uintptr_t)num % 32 == 0) && ((uintptr_t)den % 32 == 0) && (W % 4 == 0);
    s.div_d = div.d;
    s.div_r = div.r;
    if (acc_wait && cudaStreamWaitEvent(st, acc_wait, 0) != cudaSuccess)
        return fail(PRNU_CUDA_ERROR, "cudaStreamWaitEvent");
    // tile height 32 or 28 rows, whichever fills the last wave of 4 CTAs/SM better
    const long long slots = 4LL * device_sm_count();
    auto waste = [&](int ty) {
        const long long n = (long long)((W + ST_X - 1) / ST_X) * ((H + ty - 1) / ty);
        return (double)((n + slots - 1) / slots) * ty / ((double)n * ty / slots);   // waves rounded up / exact
    };
    const int TY = waste(28) < waste(32) - 1e-9 ? 28 : 32;
    CUtensorMap imap;
    SynthMaps m2;
    // pairs (d = 2): u8 frames frame_stride apart, group f = frames 2f, 2f+1 in one depth-2 box
    constexpr bool PAIR = std::is_same<TIn, u8pair>::value;
    constexpr int IDEP = PAIR ? 2 : 1;
    const size_t es = PAIR ? 1 : sizeof(TIn);
    const CUtensorMapDataType dt = es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    if (((size_t)in_pitch * es) % 16 || ((size_t)frame_stride * es) % 16 || ((uintptr_t)I % 16) ||
        !encode_tensor_map_3d(&imap, dt, es, I, (uint64_t)W, (uint64_t)H, (uint64_t)nb * IDEP,
                              (uint64_t)in_pitch * es, (uint64_t)frame_stride * es, ST_X, TY, IDEP))
        return fail(PRNU_CUDA_ERROR, "accumulation: frames not TMA-stageable (16-byte pitch / stride / base)");
    if ((rc = synth_maps(p, pb, 1, nb, s.has_A, TY / 2 + 3, &m2))) return rc;
    if ((H + TY - 1) / TY > 65535) return fail(PRNU_INVALID_ARG, "accumulation grid too large");
    static DeviceFlags attr[2];
    {
        KTimer kt(PAIR ? "synth_acc_l1_pair" : es == 1 ? "synth_acc_l1_u8" : es == 2 ? "synth_acc_l1_u16" : "synth_acc_l1_f32", st);
        dim3 g2((W + ST_X - 1) / ST_X, (H + TY - 1) / TY, 1);
        if (TY == 28) {
            if ((rc = set_smem_attr((const void*)k_synth_acc2<28, TIn>, sacc_smem_bytes<28, TIn>(), attr[0]))) return rc;
            k_synth_acc2<28, TIn><<<g2, 256, sacc_smem_bytes<28, TIn>(), st>>>(m2, imap, s);
        } else {
            if ((rc = set_smem_attr((const void*)k_synth_acc2<32, TIn>, sacc_smem_bytes<32, TIn>(), attr[1]))) return rc;
            k_synth_acc2<32, TIn><<<g2, 256, sacc_smem_bytes<32, TIn>(), st>>>(m2, imap, s);
        }
    }
    count_launch();
    if ((rc = check_launch("k_synth_acc2 (accumulate)"))) return rc;
    if (acc_done && cudaEventRecord(acc_done, st) != cudaSuccess) return fail(PRNU_CUDA_ERROR, "cudaEventRecord");
    return PRNU_OK;
}

template int run_residual<float>(const float*, int, int, int, const Pyramid&, const ShrinkParams&, float*, float*,
                                 cudaStream_t, int);
template int run_residual<uint8_t>(const uint8_t*, int, int, int, const Pyramid&, const ShrinkParams&, float*,
                                   float*, cudaStream_t, int);
template int run_residual_accumulate<float>(const float*, const float*, int, int, int, const Pyramid&,
                                            const ShrinkParams&, const SdaDiv&, double*, double*, float*,
                                            cudaStream_t, cudaEvent_t, cudaEvent_t, long long, int);
template int run_residual_accumulate<uint16_t>(const uint16_t*, const uint16_t*, int, int, int, const Pyramid&,
                                               const ShrinkParams&, const SdaDiv&, double*, double*, float*,
                                               cudaStream_t, cudaEvent_t, cudaEvent_t, long long, int);
template int run_residual_accumulate<u8pair>(const u8pair*, const u8pair*, int, int, int, const Pyramid&,
                                             const ShrinkParams&, const SdaDiv&, double*, double*, float*,
                                             cudaStream_t, cudaEvent_t, cudaEvent_t, long long, int);
template int run_residual_accumulate<uint8_t>(const uint8_t*, const uint8_t*, int, int, int, const Pyramid&,
                                              const ShrinkParams&, const SdaDiv&, double*, double*, float*,
                                              cudaStream_t, cudaEvent_t, cudaEvent_t, long long, int);

}  // namespace prnu
