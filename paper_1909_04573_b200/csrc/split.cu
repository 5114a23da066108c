// split.cu — one DWT level as two streaming kernels (a2, a3):
//
//   k_dwt_strip<TIn>  the 2-D analysis (rows then columns, R-6) of one level:
//                     raw detail subbands da, ad, dd and the approximation.
//   k_shrink_strip    the local-variance MAP/Wiener shrink (R-7) of one
//                     detail subband, c -> c - F(c) (the noise domain, R-10).
//
// Both are column-streaming: a CTA of 128 threads owns a vertical strip of the
// plane (one thread per column) and walks down a segment of rows in blocks of
// 8 rows, so every vertical dependency (the 8-tap column filter, the 3/5/7/9-row
// window sums) lives in a per-thread register window and nothing vertical is
// recomputed.  Compared with the fused k_analysis_strip (strip.cu) this moves
// 24 B per coefficient through HBM in addition (raw details written once and
// read once), in exchange for two small kernels with little per-thread state:
// the fused kernel is bound by latency at 3 CTAs/SM (145 registers, 72 KB
// shared memory), these run at 4-8 CTAs/SM and are bound by HBM bandwidth.
//
// Borders (R-4): input rows and columns outside the plane are the mirrored
// ones (rows at load time, columns by an in-shared-memory fix-up of the staged
// rows); the shrink reads the mirrored subband row/column directly, so its
// windows hold exactly the oracle's e_N samples.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tma.cuh"

namespace prnu {
namespace splitk {

constexpr int NT = 128;      // threads per CTA
constexpr int BK = 8;        // coefficient rows per block
constexpr int IR = 2 * BK;   // input rows per block
// Staging of one block: two TMA boxes [IR][BOXW] covering logical input
// columns [0, 144) and [128, 272); logical column x = input column xs + x,
// xs = 2 cx0 - 16 (cx0 a multiple of 128: 16-byte aligned for u8 boxes).
template <typename T>
struct Box;
template <>
struct Box<uint8_t> {
    static constexpr int W = 144;   // bytes (== 16 mod 128: lanes over rows conflict-free)
};
template <>
struct Box<float> {
    static constexpr int W = 148;   // floats (592 B == 80 mod 128: lanes over rows conflict-free)
};
constexpr int LOGW = 272;
constexpr int HALF = 80;     // row-buffer column permutation, second half (== 16 mod 32)
constexpr int RBP = 164;     // row-buffer pitch (== 4 mod 32)
constexpr int RB_FLOATS = 2 * IR * RBP;
constexpr int FIX = (IR * 24 + NT - 1) / NT;   // edge fix-up slots per thread (16 left + 8 right columns)

__constant__ float2 c_hg[8] = {{PRNU_H0, PRNU_H7}, {PRNU_H1, -PRNU_H6}, {PRNU_H2, PRNU_H5}, {PRNU_H3, -PRNU_H4},
                               {PRNU_H4, PRNU_H3}, {PRNU_H5, -PRNU_H2}, {PRNU_H6, PRNU_H1}, {PRNU_H7, -PRNU_H0}};
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

template <typename T>
__host__ __device__ constexpr int stage_elems() { return 2 * IR * Box<T>::W; }

template <typename T>
constexpr size_t dwt_smem_bytes() { return 2 * stage_elems<T>() * sizeof(T) + sizeof(float) * RB_FLOATS + 16; }

__device__ __forceinline__ int rb_pos(int c) { return ((c & 4) ? HALF : 0) + 4 * (c >> 3) + (c & 3); }

template <typename T>
__device__ __forceinline__ float stg_at(const T* s, int r, int x) {
    constexpr int BOXW = Box<T>::W;
    return x < BOXW ? (float)s[r * BOXW + x] : (float)s[IR * BOXW + r * BOXW + x - 128];
}
template <typename T>
__device__ __forceinline__ void stg_put(T* s, int r, int x, float v) {
    constexpr int BOXW = Box<T>::W;
    const T u = (T)v;
    if (x < BOXW) s[r * BOXW + x] = u;
    if (x >= 128) s[IR * BOXW + r * BOXW + x - 128] = u;
}

// 22 staged values of row-pass group g (coefficient columns cx0 + 8g ..), row r:
// v[i] = logical column 16g + 10 + i = input column 2(cx0 + 8g) - 6 + i.
__device__ __forceinline__ void row22(const uint8_t* s, int r, int g, float (&v)[24]) {
    constexpr int BOXW = Box<uint8_t>::W;
    const uint8_t* src = s + (g < 8 ? r * BOXW + 16 * g : IR * BOXW + r * BOXW + 16 * g - 128);
    const uint4 w0 = *reinterpret_cast<const uint4*>(src);
    const uint4 w1 = *reinterpret_cast<const uint4*>(src + 16);
    const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int k = 0; k < 22; ++k)   // exact byte -> float (2^23 trick)
        v[k] = __uint_as_float(__byte_perm(w[(k + 10) >> 2], 0x4B000000u, 0x7540u | (uint32_t)((k + 10) & 3))) -
               8388608.0f;
    v[22] = v[23] = 0.f;
}
__device__ __forceinline__ void row22(const float* s, int r, int g, float (&v)[24]) {
    constexpr int BOXW = Box<float>::W;
    const float* src = s + (g < 8 ? r * BOXW + 16 * g : IR * BOXW + r * BOXW + 16 * g - 128) + 10;
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

struct DwtArgs {
    const void* in;
    long long in_bstride;   // elements between frames
    int in_pitch;           // elements per row
    int NH, NW;             // input plane
    float* ll;              // approximation (nullable: coarsest level)
    float* c0;              // da = lo_y(hi_x), raw
    float* c1;              // ad = hi_y(lo_x), raw
    float* c2;              // dd = hi_y(hi_x), raw
    long long out_bstride;
    int out_pitch;
    int nH, nW;             // subband
    int SH;                 // rows per segment (multiple of BK)
    int use_tma;
};

template <typename T, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_dwt_strip(const __grid_constant__ CUtensorMap map, DwtArgs a) {
    constexpr int STG = stage_elems<T>();
    constexpr int BOXW = Box<T>::W;
    extern __shared__ __align__(128) unsigned char smem[];
    T* stg0 = reinterpret_cast<T*>(smem);
    float* rowbuf = reinterpret_cast<float*>(smem + 2 * STG * sizeof(T));
    uint64_t* bar = reinterpret_cast<uint64_t*>(rowbuf + RB_FLOATS);

    const int t = threadIdx.x;
    const int cx0 = blockIdx.x * NT;
    const int ky0 = blockIdx.y * a.SH;
    const int ky1 = min(ky0 + a.SH, a.nH);
    const int b = blockIdx.z;
    const int xs = 2 * cx0 - 16;
    const int nblk = (ky1 - ky0 + BK - 1) / BK;
    const T* in = reinterpret_cast<const T*>(a.in) + (size_t)b * a.in_bstride;
    const int gc = cx0 + t;
    const bool colok = gc < a.nW;
    const int pos = rb_pos(t);
    // row-pass items: row rr of groups ga and ga + 8 (groups wholly beyond the subband skipped)
    const int rr = t & 15, ga = t >> 4;
    const bool doA = cx0 + 8 * ga < a.nW;
    const bool doB = cx0 + 8 * (ga + 8) < a.nW;

    if (t == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    // edge fix-up (TMA-staged blocks of the first / last strip): out-of-plane
    // logical columns receive the mirrored in-plane values
    const bool edge = a.use_tma && (xs < 0 || xs + LOGW > a.NW);
    int fix_dst[FIX], fix_src[FIX];
    {
        const int nleft = xs < 0 ? min(-xs, LOGW) : 0;
        const int xr0 = max(a.NW - xs, nleft), xr1 = min(LOGW, a.NW - xs + 8);
        const int nright = max(xr1 - xr0, 0);
        const int ncnt = nleft + nright;
#pragma unroll
        for (int k = 0; k < FIX; ++k) {
            const int e = t + k * NT;
            fix_dst[k] = -1;
            fix_src[k] = 0;
            if (ncnt > 0 && e < IR * ncnt) {
                const int r = e / ncnt, idx = e - r * ncnt;
                const int x = idx < nleft ? idx : xr0 + idx - nleft;
                fix_dst[k] = r * 512 + x;
                fix_src[k] = min(max(mirror(xs + x, a.NW) - xs, 0), LOGW - 1);
            }
        }
    }
    auto tma_ok = [&](int i) {
        const int y = 2 * (ky0 + BK * i);
        return a.use_tma && y >= 0 && y + IR <= a.NH;
    };
    auto issue = [&](int i) {
        T* s = stg0 + (i & 1) * STG;
        const int y = 2 * (ky0 + BK * i);
        mbar_arrive_expect_tx(&bar[i & 1], (uint32_t)(2 * IR * BOXW * sizeof(T)));
        tma_load_3d(s, &map, xs, y, b, &bar[i & 1]);
        tma_load_3d(s + IR * BOXW, &map, xs + 128, y, b, &bar[i & 1]);
    };
    // issue block 0 before the prologue so its latency overlaps it
    if (t == 0 && nblk > 0 && tma_ok(0)) issue(0);
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && ((a.in_pitch * sizeof(T)) % 16 == 0);
    // thread loads of nr rows from input row y0 (rows and columns mirrored), 16-byte chunks
    auto manual = [&](T* s, int y0, int nr) {
        constexpr int CE = 16 / sizeof(T);
        constexpr int NCH = LOGW / CE;
        constexpr int PER = (IR * NCH + NT - 1) / NT;
        uint4 v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = t + k * NT;
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
            const int e = t + k * NT;
            if (e < nr * NCH) {
                const int r = e / NCH, x = (e - r * NCH) * CE;
                if (x < BOXW) *reinterpret_cast<uint4*>(s + r * BOXW + x) = v[k];
                if (x >= 128) *reinterpret_cast<uint4*>(s + IR * BOXW + r * BOXW + x - 128) = v[k];
            }
        }
    };
    auto rowpass = [&](const T* s, int nr) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int g = ga + 8 * h;
            if ((h == 0 ? doA : doB) && rr < nr) {
                float v[24];
                row22(s, rr, g, v);
                float lo[8], hi[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float2 lh = fmul2s(v[2 * q], c_hg[0]);
#pragma unroll
                    for (int j = 1; j < 8; ++j) lh = ffma2(v[2 * q + j], c_hg[j], lh);
                    lo[q] = lh.x;
                    hi[q] = lh.y;
                }
                float* dl = rowbuf + rr * RBP + 4 * g;
                float* dh = dl + IR * RBP;
                *reinterpret_cast<float4*>(dl) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                *reinterpret_cast<float4*>(dl + HALF) = make_float4(lo[4], lo[5], lo[6], lo[7]);
                *reinterpret_cast<float4*>(dh) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4*>(dh + HALF) = make_float4(hi[4], hi[5], hi[6], hi[7]);
            }
        }
    };

    // ---- prologue: row-pass rows 2ky0-6 .. 2ky0-1, staged in buffer 1 while block 0's
    //      TMA (issued above) is in flight; block 1 is issued once buffer 1 is consumed
    float lo_c[6], hi_c[6];
    {
        T* ps = stg0 + STG;
        manual(ps, 2 * ky0 - 6, 6);
        __syncthreads();
        rowpass(ps, 6);
        fence_proxy_async();
        __syncthreads();
        if (t == 0 && nblk > 1 && tma_ok(1)) issue(1);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            lo_c[r] = rowbuf[r * RBP + pos];
            hi_c[r] = rowbuf[IR * RBP + r * RBP + pos];
        }
        __syncthreads();
    }

    uint32_t phase = 0;
    const size_t obase = (size_t)b * a.out_bstride + gc;
#pragma unroll 1
    for (int i = 0; i < nblk; ++i) {
        const int K = ky0 + BK * i;
        T* s = stg0 + (i & 1) * STG;
        if (tma_ok(i)) {
            mbar_wait(&bar[i & 1], (phase >> (i & 1)) & 1);
            phase ^= 1u << (i & 1);
            if (edge) {
#pragma unroll
                for (int k = 0; k < FIX; ++k) {
                    const float v = fix_dst[k] >= 0 ? stg_at(s, fix_dst[k] >> 9, fix_src[k]) : 0.f;
                    __syncwarp();
                    if (fix_dst[k] >= 0) stg_put(s, fix_dst[k] >> 9, fix_dst[k] & 511, v);
                }
                __syncthreads();
            }
        } else {
            manual(s, 2 * K, IR);
            __syncthreads();
        }
        rowpass(s, IR);
        fence_proxy_async();
        __syncthreads();   // row buffer complete, staging buffer s consumed
        if (t == 0 && i + 2 < nblk && tma_ok(i + 2)) issue(i + 2);
        // column pass of this thread's column, coefficient rows K .. K+7
        float lo[22], hi[22];
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            lo[r] = lo_c[r];
            hi[r] = hi_c[r];
        }
#pragma unroll
        for (int r = 0; r < IR; ++r) {
            lo[6 + r] = rowbuf[r * RBP + pos];
            hi[6 + r] = rowbuf[IR * RBP + r * RBP + pos];
        }
        __syncthreads();   // row buffer free for the next block's row pass
        const int kmax = min(ky1 - K, BK);
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            float2 p_l = fmul2s(lo[2 * k], c_hg[0]);   // (aa, ad)
            float2 p_h = fmul2s(hi[2 * k], c_hg[0]);   // (da, dd)
#pragma unroll
            for (int j = 1; j < 8; ++j) {
                p_l = ffma2(lo[2 * k + j], c_hg[j], p_l);
                p_h = ffma2(hi[2 * k + j], c_hg[j], p_h);
            }
            if (colok && k < kmax) {
                const size_t o = obase + (size_t)(K + k) * a.out_pitch;
                if (a.ll) a.ll[o] = p_l.x;
                a.c0[o] = p_h.x;
                a.c1[o] = p_l.y;
                a.c2[o] = p_h.y;
            }
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            lo_c[r] = lo[IR + r];
            hi_c[r] = hi[IR + r];
        }
    }
}

// ---------------------------------------------------------------- shrink
constexpr int SO_MAX = NT - 8;       // output columns per shrink strip (4-column window halo each side)
constexpr int P2 = 129;              // float2 pitch of the (v3,v5) / (v7,v9) planes (8 B mod 128 B)
constexpr int CP = 132;              // float pitch of the coefficient plane (16 B mod 128 B)
constexpr int VC_FLOATS = 2 * BK * P2 * 2 + BK * CP;

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

template <bool ALL4>
__global__ void __launch_bounds__(NT, 5) k_shrink_strip(ShrinkArgs a) {
    __shared__ __align__(16) float vc[VC_FLOATS];
    float2* const P35 = reinterpret_cast<float2*>(vc);
    float2* const P79 = P35 + BK * P2;
    float* const C = vc + 4 * BK * P2;

    const int t = threadIdx.x;
    const int sb = blockIdx.z % a.nsub, b = blockIdx.z / a.nsub;
    const int cx0 = blockIdx.x * a.O;
    const int ky0 = blockIdx.y * a.SH;
    const int ky1 = min(ky0 + a.SH, a.nH);
    const int ncols = a.O + 8;
    const int gc = cx0 - 4 + t;
    const int mc = mirror(gc, a.nW);   // the column whose values this region column holds (R-4)
    const float* src = (sb == 0 ? a.src[0] : sb == 1 ? a.src[1] : a.src[2]) + (size_t)b * a.bstride + mc;
    const int nblk = 1 + (ky1 - ky0 + BK - 1) / BK;   // block 0 = prologue (rows ky0-4 .. ky0+3)
    const int K0 = ky0 - 4;
    // H item: output row hj of the block, outputs 8hg .. 8hg+7
    const int hj = t & 7, hg = t >> 3;
    const int hx = cx0 + 8 * hg;
    const bool hv = t < a.O && hx < a.nW;
    const bool hfull = hx + 8 <= a.nW;
    float* const dst = (sb == 0 ? a.dst[0] : sb == 1 ? a.dst[1] : a.dst[2]) + (size_t)b * a.bstride + hx;
    const float s0 = a.s0_dev ? a.s0_dev[b] : a.sp.sigma0_sq;
    const int wm = a.sp.wmask;

    // prefetch: the coefficients of the next two blocks in flight (rows mirrored, R-4;
    // a single reflection suffices when nH >= 8, the general map otherwise)
    float pf[BK], pf2[BK];
    const int nH = a.nH;
    auto rowm = [&](int r) {
        if (nH >= 8) return r < 0 ? -1 - r : (r >= nH ? 2 * nH - 1 - r : r);
        return mirror(r, nH);
    };
    auto load_block = [&](int i, float (&dstv)[BK]) {
        const int K = K0 + BK * i;
#pragma unroll
        for (int k = 0; k < BK; ++k) dstv[k] = __ldg(src + (size_t)rowm(K + k) * a.pitch);
    };
    float q[16], c[12];   // squares of rows K-8 .. K+7; coefficients of rows K-4 .. K+7
#pragma unroll
    for (int k = 0; k < 16; ++k) q[k] = 0.f;
#pragma unroll
    for (int k = 0; k < 12; ++k) c[k] = 0.f;
    load_block(0, pf);
    if (nblk > 1) load_block(1, pf2);
#pragma unroll 1
    for (int i = 0; i < nblk; ++i) {
        const int K = K0 + BK * i;
        // shift the ring by one block (rows K-8 .. K-1 were K .. K+7)
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = q[8 + k];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] = c[8 + k];
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            c[4 + k] = pf[k];
            q[8 + k] = __fmul_rn(pf[k], pf[k]);
        }
#pragma unroll
        for (int k = 0; k < BK; ++k) pf[k] = pf2[k];
        if (i + 2 < nblk) load_block(i + 2, pf2);
        if (i == 0) continue;
        // output rows K-4 .. K+3: vertical window sums (ring slots j .. j+8)
        if (t < ncols) {
#pragma unroll
            for (int j = 0; j < BK; ++j) {
                const float v3 = q[j + 3] + q[j + 4] + q[j + 5];
                const float v5 = v3 + q[j + 2] + q[j + 6];
                const float v7 = v5 + q[j + 1] + q[j + 7];
                const float v9 = v7 + q[j] + q[j + 8];
                P35[j * P2 + t] = make_float2(v3, v5);
                P79[j * P2 + t] = make_float2(v7, v9);
                C[j * CP + t] = c[j];
            }
        }
        __syncthreads();
        if (hv && K - 4 + hj < ky1) {
            const float2* p35 = P35 + hj * P2 + 8 * hg;
            const float2* p79 = P79 + hj * P2 + 8 * hg;
            float m[8];
            {
                float2 u[12];   // (v3, v5) of columns 2 .. 13
#pragma unroll
                for (int k = 0; k < 12; ++k) u[k] = p35[2 + k];
                float s3 = u[1].x + u[2].x + u[3].x;
                float s5 = u[0].y + u[1].y + u[2].y + u[3].y + u[4].y;
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    if (x > 0) {   // slide one column right
                        s3 += u[x + 3].x - u[x].x;
                        s5 += u[x + 4].y - u[x - 1].y;
                    }
                    float2 r;
                    {
                        unsigned long long ra, rb = *reinterpret_cast<const unsigned long long*>(&c_ws[0]), rr;
                        const float2 sv = make_float2(s3, s5);
                        ra = *reinterpret_cast<const unsigned long long*>(&sv);
                        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(ra), "l"(rb));
                        r = *reinterpret_cast<float2*>(&rr);
                    }
                    if (ALL4) m[x] = fminf(r.x, r.y);
                    else m[x] = fminf((wm & 1) ? r.x : 3.402823466e38f, (wm & 2) ? r.y : 3.402823466e38f);
                }
            }
            {
                float2 u[16];   // (v7, v9) of columns 0 .. 15
#pragma unroll
                for (int k = 0; k < 16; ++k) u[k] = p79[k];
                float s7 = u[1].x + u[2].x + u[3].x + u[4].x + u[5].x + u[6].x + u[7].x;
                float s9 = u[0].y + u[1].y + u[2].y + u[3].y + u[4].y + u[5].y + u[6].y + u[7].y + u[8].y;
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    if (x > 0) {
                        s7 += u[x + 7].x - u[x].x;
                        s9 += u[x + 8].y - u[x - 1].y;
                    }
                    float2 r;
                    {
                        unsigned long long ra, rb = *reinterpret_cast<const unsigned long long*>(&c_ws[1]), rr;
                        const float2 sv = make_float2(s7, s9);
                        ra = *reinterpret_cast<const unsigned long long*>(&sv);
                        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(ra), "l"(rb));
                        r = *reinterpret_cast<float2*>(&rr);
                    }
                    if (ALL4) m[x] = fminf(m[x], fminf(r.x, r.y));
                    else m[x] = fminf(m[x], fminf((wm & 4) ? r.x : 3.402823466e38f, (wm & 8) ? r.y : 3.402823466e38f));
                }
            }
            const float* crow = C + hj * CP + 4 + 8 * hg;
            const float4 c0 = *reinterpret_cast<const float4*>(crow);
            const float4 c1 = *reinterpret_cast<const float4*>(crow + 4);
            const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            float o[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {   // c - F(c) = c s0 / (max(m - s0, 0) + s0) = c s0 / max(m, s0)
                float r;
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(m[x], s0)));
                o[x] = cv[x] * s0 * r;
            }
            float* drow = dst + (size_t)(K - 4 + hj) * a.pitch;
            if (hfull) {
                reinterpret_cast<float4*>(drow)[0] = make_float4(o[0], o[1], o[2], o[3]);
                reinterpret_cast<float4*>(drow)[1] = make_float4(o[4], o[5], o[6], o[7]);
            } else {
#pragma unroll
                for (int x = 0; x < 8; ++x)
                    if (hx + x < a.nW) drow[x] = o[x];
            }
        }
        __syncthreads();   // planes free for the next block
    }
}

// ---------------------------------------------------------------- shrink, horizontal-first
// Same operation as k_shrink_strip with the separable window sums in the other
// order: the squares c^2 of 8 rows go through shared memory once (one float per
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
        __syncthreads();   // squares of rows K .. K+7 visible (the other plane is free)
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

}  // namespace splitk

// ---------------------------------------------------------------- host
bool encode_tensor_map_3d(CUtensorMap* map, CUtensorMapDataType dt, size_t elem_bytes, const void* base, uint64_t cols,
                          uint64_t rows, uint64_t depth, uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t box_w,
                          uint32_t box_h);

// Rows per segment: about per_seg, but small planes are cut into more segments
// so that the grid holds at least two waves of resident CTAs (min_ctas).
static int seg_rows(int nH, int per_seg, int align, long long ctas_per_seg, long long min_ctas) {
    int nseg = (nH + per_seg - 1) / per_seg;
    while (nseg * ctas_per_seg < min_ctas && (nH + nseg) / (nseg + 1) >= align) ++nseg;
    return (int)align_up((size_t)((nH + nseg - 1) / nseg), align);
}

template <typename T>
static int dwt_launch(const T* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll, float* c0, float* c1,
                      float* c2, long long out_bstride, int out_pitch, int nH, int nW, int nb, cudaStream_t st) {
    using namespace splitk;
    constexpr int MINB = sizeof(T) == 1 ? 6 : 3;
    static bool attr = false;
    if (!attr) {
        cudaError_t e1 = cudaFuncSetAttribute(k_dwt_strip<uint8_t, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)dwt_smem_bytes<uint8_t>());
        cudaError_t e2 = cudaFuncSetAttribute(k_dwt_strip<float, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)dwt_smem_bytes<float>());
        if (e1 != cudaSuccess || e2 != cudaSuccess)
            return fail(PRNU_CUDA_ERROR, std::string("cudaFuncSetAttribute(dwt): ") +
                                             cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
        attr = true;
    }
    DwtArgs a{};
    a.in = in;
    a.in_bstride = in_bstride;
    a.in_pitch = in_pitch;
    a.NH = NH;
    a.NW = NW;
    a.ll = ll;
    a.c0 = c0;
    a.c1 = c1;
    a.c2 = c2;
    a.out_bstride = out_bstride;
    a.out_pitch = out_pitch;
    a.nH = nH;
    a.nW = nW;
    static const int sh_env = getenv("PRNU_DWT_SH") ? atoi(getenv("PRNU_DWT_SH")) : 0;
    const int S = (nW + NT - 1) / NT;
    a.SH = sh_env > 0 ? (int)align_up((size_t)sh_env, BK) : seg_rows(nH, 136, BK, (long long)S * nb, 2LL * 148 * MINB);
    const int nseg = (nH + a.SH - 1) / a.SH;
    CUtensorMap map{};
    const size_t es = sizeof(T);
    a.use_tma = ((in_pitch * es) % 16 == 0) && ((in_bstride * es) % 16 == 0) && ((uintptr_t)in % 16 == 0) &&
                encode_tensor_map_3d(&map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                     es, in, (uint64_t)NW, (uint64_t)NH, (uint64_t)nb, (uint64_t)in_pitch * es,
                                     (uint64_t)in_bstride * es, Box<T>::W, IR);
    dim3 grid(S, nseg, nb);
    k_dwt_strip<T, MINB><<<grid, NT, dwt_smem_bytes<T>(), st>>>(map, a);
    return PRNU_OK;
}

int launch_dwt_strip_u8(const uint8_t* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll, float* c0,
                        float* c1, float* c2, long long out_bstride, int out_pitch, int nH, int nW, int nb,
                        cudaStream_t st) {
    return dwt_launch<uint8_t>(in, in_bstride, in_pitch, NH, NW, ll, c0, c1, c2, out_bstride, out_pitch, nH, nW, nb,
                               st);
}
int launch_dwt_strip_f32(const float* in, long long in_bstride, int in_pitch, int NH, int NW, float* ll, float* c0,
                         float* c1, float* c2, long long out_bstride, int out_pitch, int nH, int nW, int nb,
                         cudaStream_t st) {
    return dwt_launch<float>(in, in_bstride, in_pitch, NH, NW, ll, c0, c1, c2, out_bstride, out_pitch, nH, nW, nb,
                             st);
}

int launch_shrink_strip(const float* const src[3], float* const dst[3], long long bstride, int pitch, int nH, int nW,
                        const ShrinkParams& sp, int nb, cudaStream_t st, int nsub, const float* s0_dev) {
    using namespace splitk;
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
    static const int sh_env = getenv("PRNU_SHRINK_SH") ? atoi(getenv("PRNU_SHRINK_SH")) : 0;
    a.SH = sh_env > 0 ? (int)align_up((size_t)sh_env, BK) : seg_rows(nH, 136, BK, (long long)nsub * S * nb, 2LL * 148 * 5);
    const int nseg = (nH + a.SH - 1) / a.SH;
    dim3 grid(S, nseg, nsub * nb);
    static const bool vfirst = getenv("PRNU_SHRINK_VFIRST") != nullptr;   // A/B: vertical-sums-first variant
    if (vfirst) {
        if (sp.wmask == 15) k_shrink_strip<true><<<grid, NT, 0, st>>>(a);
        else k_shrink_strip<false><<<grid, NT, 0, st>>>(a);
    } else {
        if (sp.wmask == 15) k_shrink_hfirst<true><<<grid, NT, 0, st>>>(a);
        else k_shrink_hfirst<false><<<grid, NT, 0, st>>>(a);
    }
    return PRNU_OK;
}

}  // namespace prnu
