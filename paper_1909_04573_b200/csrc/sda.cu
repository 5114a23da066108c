// sda.cu — a1: SDA averaging.
//
// S_i[p] = RN_fp32( sum_{j = i d}^{(i+1) d - 1} u8_j[p] / d ).
// The sum is an exact uint32 (max 255 * d < 2^24 for d <= 65793, so the
// int -> float conversion is exact too) and the division is one IEEE
// correctly-rounded fp32 divide (__fdiv_rn; never a reciprocal multiply,
// R-11).  Each thread owns 16 consecutive pixels (one 16-byte load per
// frame), loops over the d frames of its group with 8 loads in flight, and
// writes four float4.  HBM-bound: (d + 4) bytes per output pixel.
#include "common.cuh"

namespace prnu {

constexpr int SDA_VEC = 16;

// Packed accumulation: each 32-bit word holds two 16-bit partial sums (bytes
// 0,2 and bytes 1,3 of a 4-pixel word), exact for up to 257 frames; every 256
// frames the packed sums are flushed into 32-bit per-pixel totals.
__device__ __forceinline__ void sda_add_packed(const uint4& v, uint32_t (&pe)[4], uint32_t (&po)[4]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        pe[q] += w[q] & 0x00ff00ffu;
        po[q] += (w[q] >> 8) & 0x00ff00ffu;
    }
}

__global__ void __launch_bounds__(256) k_sda_average_vec(const uint4* __restrict__ frames, long long P16, int d,
                                                          float4* __restrict__ out) {
    const int g = blockIdx.y;   // SDA group
    const float fd = (float)d;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P16;
         i += (long long)gridDim.x * blockDim.x) {
        const uint4* src = frames + (size_t)g * d * P16 + i;
        uint32_t s[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) s[k] = 0;
        for (int j0 = 0; j0 < d; j0 += 256) {
            const int j1 = min(d, j0 + 256);
            uint32_t pe[4] = {0, 0, 0, 0}, po[4] = {0, 0, 0, 0};
            int j = j0;
            for (; j + 8 <= j1; j += 8) {
                uint4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + (size_t)(j + u) * P16);
#pragma unroll
                for (int u = 0; u < 8; ++u) sda_add_packed(v[u], pe, po);
            }
            for (; j < j1; ++j) sda_add_packed(__ldcs(src + (size_t)j * P16), pe, po);
#pragma unroll
            for (int q = 0; q < 4; ++q) {   // pixel 4q+0 = low half of pe, 4q+2 = high half, etc.
                s[4 * q + 0] += pe[q] & 0xffffu;
                s[4 * q + 2] += pe[q] >> 16;
                s[4 * q + 1] += po[q] & 0xffffu;
                s[4 * q + 3] += po[q] >> 16;
            }
        }
        float4* dst = out + ((size_t)g * P16 + i) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float4 o;
            o.x = __fdiv_rn((float)s[4 * q + 0], fd);
            o.y = __fdiv_rn((float)s[4 * q + 1], fd);
            o.z = __fdiv_rn((float)s[4 * q + 2], fd);
            o.w = __fdiv_rn((float)s[4 * q + 3], fd);
            dst[q] = o;   // plain store: the SDA frame is re-read by the denoiser (keep in L2)
        }
    }
}

// Generic path (P not a multiple of 16 or unaligned): one pixel per thread.
__global__ void __launch_bounds__(256) k_sda_average_scalar(const uint8_t* __restrict__ frames, long long P, int d,
                                                             float* __restrict__ out) {
    const int g = blockIdx.y;
    const float fd = (float)d;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P;
         i += (long long)gridDim.x * blockDim.x) {
        const uint8_t* src = frames + (size_t)g * d * P + i;
        uint32_t s = 0;
        for (int j = 0; j < d; ++j) s += src[(size_t)j * P];
        out[(size_t)g * P + i] = __fdiv_rn((float)s, fd);
    }
}

// SDA group sums for the fused extraction (2 <= d <= 257, R-11): the exact sum of the
// d frames of each group as u16 (255 * 257 = 65535), rows written with a pitch of Wp
// elements (a multiple of 8: 16-byte rows, TMA-stageable; pad columns 0).  The
// analysis and the accumulation form S = RN(sum / d) themselves (sda_div), so the
// fp32 SDA frame never goes through HBM: 2 B per pixel written and read instead of 4.
// Vector path (W % 8 == 0, 8-byte aligned frames): 8 pixels per thread, packed 16-bit
// lane sums (even / odd bytes) stored interleaved as 8 u16.
__global__ void __launch_bounds__(256) k_sda_sum_u16_vec(const uint2* __restrict__ frames, long long P8, int d,
                                                          uint4* __restrict__ out) {
    const int g = blockIdx.y;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P8;
         i += (long long)gridDim.x * blockDim.x) {
        const uint2* src = frames + (size_t)g * d * P8 + i;
        uint32_t pe[2] = {0, 0}, po[2] = {0, 0};
        int j = 0;
        for (; j + 8 <= d; j += 8) {
            uint2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + (size_t)(j + u) * P8);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                pe[0] += v[u].x & 0x00ff00ffu;
                po[0] += (v[u].x >> 8) & 0x00ff00ffu;
                pe[1] += v[u].y & 0x00ff00ffu;
                po[1] += (v[u].y >> 8) & 0x00ff00ffu;
            }
        }
        for (; j < d; ++j) {
            const uint2 v = __ldcs(src + (size_t)j * P8);
            pe[0] += v.x & 0x00ff00ffu;
            po[0] += (v.x >> 8) & 0x00ff00ffu;
            pe[1] += v.y & 0x00ff00ffu;
            po[1] += (v.y >> 8) & 0x00ff00ffu;
        }
        // pixel 4q+0 = low half of pe[q], 4q+1 = low half of po[q], 4q+2 / 4q+3 = high halves
        out[(size_t)g * P8 + i] = make_uint4(__byte_perm(pe[0], po[0], 0x5410), __byte_perm(pe[0], po[0], 0x7632),
                                             __byte_perm(pe[1], po[1], 0x5410), __byte_perm(pe[1], po[1], 0x7632));
    }
}

// Generic path: one pixel per thread, any width / alignment, rows re-pitched to Wp.
template <typename TO>
__global__ void __launch_bounds__(256) k_sda_rows(const uint8_t* __restrict__ frames, int H, int W, int d, int Wp,
                                                   TO* __restrict__ out) {
    const int g = blockIdx.y;
    const long long P = (long long)H * W, Pp = (long long)H * Wp;
    const float fd = (float)d;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < Pp;
         i += (long long)gridDim.x * blockDim.x) {
        const long long y = i / Wp, x = i - y * Wp;
        uint32_t s = 0;
        if (x < W) {
            const uint8_t* src = frames + (size_t)g * d * P + y * W + x;
            for (int j = 0; j < d; ++j) s += src[(size_t)j * P];
        }
        if (sizeof(TO) == 2) out[(size_t)g * Pp + i] = (TO)s;                  // exact sum (d <= 257)
        else out[(size_t)g * Pp + i] = (TO)__fdiv_rn((float)s, fd);           // RN(sum / d) (d > 257)
    }
}

int launch_sda_sum_u16(const uint8_t* frames, long long n_groups, int H, int W, int d, uint16_t* out, int Wp,
                       cudaStream_t st) {
    if (n_groups <= 0) return PRNU_OK;
    if (d < 1 || d > 257) return fail(PRNU_BAD_PARAMETER, "u16 SDA sums need 1 <= d <= 257");
    const long long P = (long long)H * W;
    const bool vec = Wp == W && W % 8 == 0 && ((uintptr_t)frames % 8 == 0) && ((uintptr_t)out % 16 == 0);
    const long long cap = 8LL * device_sm_count();
    for (long long g0 = 0; g0 < n_groups; g0 += 65535) {
        const int ng = (int)std::min<long long>(65535, n_groups - g0);
        KTimer kt("sda_sum", st);
        if (vec) {
            const long long P8 = P / 8;
            dim3 grid((unsigned)std::min<long long>((P8 + 255) / 256, cap), ng);
            k_sda_sum_u16_vec<<<grid, 256, 0, st>>>(reinterpret_cast<const uint2*>(frames + g0 * d * P), P8, d,
                                                    reinterpret_cast<uint4*>(out + g0 * (long long)H * Wp));
        } else {
            dim3 grid((unsigned)std::min<long long>(((long long)H * Wp + 255) / 256, cap), ng);
            k_sda_rows<uint16_t><<<grid, 256, 0, st>>>(frames + g0 * d * P, H, W, d, Wp, out + g0 * (long long)H * Wp);
        }
        count_launch();
        int rc = check_launch("k_sda_sum_u16");
        if (rc) return rc;
    }
    return PRNU_OK;
}

// Pitched copy of u8 frames (rows of W bytes -> rows of Wp bytes, Wp a multiple of 16)
// so that unaligned frame widths can still be TMA-staged; one CTA per (frame, row).
__global__ void __launch_bounds__(256) k_pad_rows_u8(const uint8_t* __restrict__ src, int H, int W,
                                                      long long src_stride, uint8_t* __restrict__ dst, int Wp) {
    const long long row = blockIdx.x;   // frame * H + y
    const long long f = row / H, y = row - f * H;
    const uint8_t* s = src + f * src_stride + y * W;
    uint8_t* d = dst + row * Wp;
    for (int x = threadIdx.x; x < Wp; x += 256) d[x] = x < W ? s[x] : 0;
}

int launch_pad_rows_u8(const uint8_t* src, long long nb, int H, int W, long long src_stride, uint8_t* dst, int Wp,
                       cudaStream_t st) {
    k_pad_rows_u8<<<(unsigned)(nb * H), 256, 0, st>>>(src, H, W, src_stride, dst, Wp);
    count_launch();
    return check_launch("k_pad_rows_u8");
}

int launch_sda_average(const uint8_t* frames, long long n_groups, long long P, int d, float* out, cudaStream_t st);

// fp32 SDA frames with rows of Wp floats (Wp >= W; the extraction uses a multiple of 4
// so that the frames are TMA-stageable)
int launch_sda_average_pitched(const uint8_t* frames, long long n_groups, int H, int W, int d, float* out, int Wp,
                               cudaStream_t st) {
    if (Wp == W) return launch_sda_average(frames, n_groups, (long long)H * W, d, out, st);
    if (n_groups <= 0) return PRNU_OK;
    const long long cap = 8LL * device_sm_count();
    for (long long g0 = 0; g0 < n_groups; g0 += 65535) {
        const int ng = (int)std::min<long long>(65535, n_groups - g0);
        KTimer kt("sda_average", st);
        dim3 grid((unsigned)std::min<long long>(((long long)H * Wp + 255) / 256, cap), ng);
        k_sda_rows<float><<<grid, 256, 0, st>>>(frames + g0 * d * (long long)H * W, H, W, d, Wp,
                                                 out + g0 * (long long)H * Wp);
        count_launch();
        int rc = check_launch("k_sda_average (pitched)");
        if (rc) return rc;
    }
    return PRNU_OK;
}

int launch_sda_average(const uint8_t* frames, long long n_groups, long long P, int d, float* out,
                       cudaStream_t st) {
    if (n_groups <= 0) return PRNU_OK;
    const bool vec = (P % SDA_VEC == 0) && ((uintptr_t)frames % 16 == 0) && ((uintptr_t)out % 16 == 0);
    for (long long g0 = 0; g0 < n_groups; g0 += 65535) {
        int ng = (int)std::min<long long>(65535, n_groups - g0);
        KTimer kt("sda_average", st);
        if (vec) {
            long long P16 = P / SDA_VEC;
            long long blocks = std::min<long long>((P16 + 255) / 256, 8LL * device_sm_count());
            dim3 grid((unsigned)blocks, ng);
            k_sda_average_vec<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(frames + g0 * d * P), P16, d,
                                                    reinterpret_cast<float4*>(out + g0 * P));
        } else {
            long long blocks = std::min<long long>((P + 255) / 256, 8LL * device_sm_count());
            dim3 grid((unsigned)blocks, ng);
            k_sda_average_scalar<<<grid, 256, 0, st>>>(frames + g0 * d * P, P, d, out + g0 * P);
        }
        count_launch();
        int rc = check_launch("k_sda_average");
        if (rc) return rc;
    }
    return PRNU_OK;
}

}  // namespace prnu

// ---------------------------------------------------------------- f4: RGB -> luma
// Y = 0.299 R + 0.587 G + 0.114 B (the BT.601 weights BASELINE
// config 3 names), from the exact integer s = 299 R + 587 G + 114 B:
//   rounding 0: fp32 Y = RN_fp32(s / 1000)  (one IEEE divide, s < 2^24 exact)
//   rounding 1: u8   Y = s / 1000 rounded half to even (exact integer rule).
// layout 0: planar [n][3][H][W]; layout 1: interleaved [n][H][W][3].
// HBM-bound: 3 bytes in, 4 (or 1) out per pixel; 4 pixels per thread-iteration.
namespace prnu {

__device__ __forceinline__ uint32_t luma_s(uint32_t r, uint32_t g, uint32_t b) { return 299u * r + 587u * g + 114u * b; }

template <int LAYOUT, int ROUND>
__global__ void __launch_bounds__(256) k_rgb_to_luma(const uint8_t* __restrict__ rgb, long long n, long long P,
                                                     void* __restrict__ out) {
    const long long P4 = P / 4;   // P % 4 == 0 on this path
    const long long total = n * P4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long f = i / P4, q = i - f * P4;
        uint32_t r[4], g[4], b[4];
        if (LAYOUT == 0) {
            const uint8_t* base = rgb + (size_t)f * 3 * P + 4 * q;
            const uint32_t wr = __ldg(reinterpret_cast<const uint32_t*>(base));
            const uint32_t wg = __ldg(reinterpret_cast<const uint32_t*>(base + P));
            const uint32_t wb = __ldg(reinterpret_cast<const uint32_t*>(base + 2 * P));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                r[k] = (wr >> (8 * k)) & 0xffu;
                g[k] = (wg >> (8 * k)) & 0xffu;
                b[k] = (wb >> (8 * k)) & 0xffu;
            }
        } else {
            const uint32_t* base = reinterpret_cast<const uint32_t*>(rgb + ((size_t)f * P + 4 * q) * 3);
            const uint32_t w0 = __ldg(base), w1 = __ldg(base + 1), w2 = __ldg(base + 2);
            const uint32_t by[12] = {w0 & 0xffu, (w0 >> 8) & 0xffu, (w0 >> 16) & 0xffu, w0 >> 24,
                                     w1 & 0xffu, (w1 >> 8) & 0xffu, (w1 >> 16) & 0xffu, w1 >> 24,
                                     w2 & 0xffu, (w2 >> 8) & 0xffu, (w2 >> 16) & 0xffu, w2 >> 24};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                r[k] = by[3 * k];
                g[k] = by[3 * k + 1];
                b[k] = by[3 * k + 2];
            }
        }
        if (ROUND == 0) {
            float y[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) y[k] = __fdiv_rn((float)luma_s(r[k], g[k], b[k]), 1000.0f);
            reinterpret_cast<float4*>(out)[i] = make_float4(y[0], y[1], y[2], y[3]);
        } else {
            uint32_t w = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t s = luma_s(r[k], g[k], b[k]);
                uint32_t qv = s / 1000u;
                const uint32_t rem = s - 1000u * qv;
                if (rem > 500u || (rem == 500u && (qv & 1u))) ++qv;   // half to even
                w |= qv << (8 * k);
            }
            reinterpret_cast<uint32_t*>(out)[i] = w;
        }
    }
}

// 16 pixels per thread-iteration: 16-byte loads of each plane (planar) or three
// 16-byte loads of 48 interleaved bytes, 16-byte stores.  Requires P % 16 == 0
// (else the 4-pixel kernel below runs).
template <int LAYOUT, int ROUND>
__global__ void __launch_bounds__(256) k_rgb_to_luma16(const uint8_t* __restrict__ rgb, long long n, long long P,
                                                       void* __restrict__ out) {
    const long long P16 = P / 16;
    const long long total = n * P16;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long f = i / P16, q = i - f * P16;
        uint32_t w[12];
        if (LAYOUT == 0) {
            const uint8_t* base = rgb + (size_t)f * 3 * P + 16 * q;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + c * P));
                w[4 * c] = v.x;
                w[4 * c + 1] = v.y;
                w[4 * c + 2] = v.z;
                w[4 * c + 3] = v.w;
            }
        } else {
            const uint4* base = reinterpret_cast<const uint4*>(rgb + ((size_t)f * P + 16 * q) * 3);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const uint4 v = __ldg(base + c);
                w[4 * c] = v.x;
                w[4 * c + 1] = v.y;
                w[4 * c + 2] = v.z;
                w[4 * c + 3] = v.w;
            }
        }
        uint32_t s[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            uint32_t r, g, b;
            if (LAYOUT == 0) {
                r = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
                g = (w[4 + (k >> 2)] >> (8 * (k & 3))) & 0xffu;
                b = (w[8 + (k >> 2)] >> (8 * (k & 3))) & 0xffu;
            } else {
                const int o = 3 * k;
                r = (w[o >> 2] >> (8 * (o & 3))) & 0xffu;
                g = (w[(o + 1) >> 2] >> (8 * ((o + 1) & 3))) & 0xffu;
                b = (w[(o + 2) >> 2] >> (8 * ((o + 2) & 3))) & 0xffu;
            }
            s[k] = luma_s(r, g, b);
        }
        if (ROUND == 0) {
            float4* o4 = reinterpret_cast<float4*>(out) + 4 * i;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                o4[k] = make_float4(__fdiv_rn((float)s[4 * k], 1000.0f), __fdiv_rn((float)s[4 * k + 1], 1000.0f),
                                    __fdiv_rn((float)s[4 * k + 2], 1000.0f), __fdiv_rn((float)s[4 * k + 3], 1000.0f));
        } else {
            uint32_t ow[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                uint32_t qv = s[k] / 1000u;
                const uint32_t rem = s[k] - 1000u * qv;
                if (rem > 500u || (rem == 500u && (qv & 1u))) ++qv;   // half to even
                ow[k >> 2] |= qv << (8 * (k & 3));
            }
            reinterpret_cast<uint4*>(out)[i] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
    }
}

int launch_rgb_to_luma(const uint8_t* rgb, long long n, long long P, int layout, int rounding, void* out,
                       cudaStream_t st) {
    if (P % 16 == 0 && ((uintptr_t)rgb & 15) == 0 && ((uintptr_t)out & 15) == 0) {
        const long long total = n * (P / 16);
        const int blocks = (int)std::max(1LL, std::min((total + 255) / 256, 16LL * device_sm_count()));
        if (layout == 0 && rounding == 0) k_rgb_to_luma16<0, 0><<<blocks, 256, 0, st>>>(rgb, n, P, out);
        else if (layout == 0) k_rgb_to_luma16<0, 1><<<blocks, 256, 0, st>>>(rgb, n, P, out);
        else if (rounding == 0) k_rgb_to_luma16<1, 0><<<blocks, 256, 0, st>>>(rgb, n, P, out);
        else k_rgb_to_luma16<1, 1><<<blocks, 256, 0, st>>>(rgb, n, P, out);
        count_launch();
        return check_launch("k_rgb_to_luma16");
    }
    const long long total = n * (P / 4);
    const int blocks = (int)std::max(1LL, std::min((total + 255) / 256, 16LL * device_sm_count()));
    if (layout == 0 && rounding == 0) k_rgb_to_luma<0, 0><<<blocks, 256, 0, st>>>(rgb, n, P, out);
    else if (layout == 0) k_rgb_to_luma<0, 1><<<blocks, 256, 0, st>>>(rgb, n, P, out);
    else if (rounding == 0) k_rgb_to_luma<1, 0><<<blocks, 256, 0, st>>>(rgb, n, P, out);
    else k_rgb_to_luma<1, 1><<<blocks, 256, 0, st>>>(rgb, n, P, out);
    count_launch();
    return check_launch("k_rgb_to_luma");
}

}  // namespace prnu
