// pcefft.cu — the column stage of the PCE correlation surface (sm_100a).
//
// a8: C = IFFT2(FFT2(R) . conj(FFT2(T))) with the DC bin
// zeroed (the mean removal of both inputs), unnormalised as cuFFT's R2C/C2R.
// The rows are cuFFT 1-D C2C transforms of length M = W/2 applied to the real
// planes viewed as packed complex rows z[m] = x[2m] + i x[2m+1] (no copy); this
// file does everything between the forward and the inverse row transforms in
// ONE kernel per block of columns, entirely in shared memory / registers:
//   untangle the packed rows into the real-input spectrum X[y][k], k = 0..M
//   (X[0] and X[M] are real per row and travel packed as one complex column),
//   forward FFT along y (mixed-radix Stockham, radix-R codelets in registers),
//   [match] P = R^ . conj(T^) (R^ cached by a forward-only launch), the packed
//   column separated into its two Hermitian halves and the DC bin zeroed,
//   inverse FFT along y, re-tangle into the packed rows the inverse C2C wants.
// The 2-D cuFFT path this replaces runs ~9 HBM passes per pair (3 per 2-D real
// transform + conj-mul); this path runs 4 (rows, columns, rows, + the template
// and the reductions as before).  Spectrum layout (the cached residual
// spectrum): [b][v][m], m = 0..M-1, column 0 = X[.][0] + i X[.][M] transformed.
#include "common.cuh"


namespace prnu {
namespace fft {

// ---------------------------------------------------------------- compile-time trig
constexpr double kPi = 3.14159265358979323846264338327950288;
__host__ __device__ constexpr double cx_sin_r(double x) {   // |x| <= pi: Taylor series to double precision
    double t = x, s = x;
    for (int n = 1; n < 30; ++n) {
        t *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double cx_cos_r(double x) {
    double t = 1.0, s = 1.0;
    for (int n = 1; n < 30; ++n) {
        t *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
        s += t;
    }
    return s;
}
__host__ __device__ constexpr double cx_angle(int m, int R) {   // 2 pi m / R reduced to (-pi, pi]
    int r = ((m % R) + R) % R;
    double x = 2.0 * kPi * r / R;
    return x > kPi ? x - 2.0 * kPi : x;
}
__host__ __device__ constexpr double cx_cos2pi(int m, int R) { return cx_cos_r(cx_angle(m, R)); }
__host__ __device__ constexpr double cx_sin2pi(int m, int R) { return cx_sin_r(cx_angle(m, R)); }

template <int V>
struct Ic {   // a compile-time index usable in device code
    static constexpr int value = V;
    __host__ __device__ constexpr operator int() const { return V; }
};
template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f) {
    if constexpr (B < E) {
        f(Ic<B>{});
        sfor<B + 1, E>(f);
    }
}

// ---------------------------------------------------------------- scalar complex (global phases)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
template <int S>   // a * (S i), S = +-1
__device__ __forceinline__ float2 muli(float2 a) {
    return S > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// ---------------------------------------------------------------- column-pair complex (the passes)
// One complex value of two adjacent columns: re = (re_c, re_c+1), im = (im_c, im_c+1).
// Every real operation is one f32x2 instruction for both columns (FADD2 / FMUL2 /
// FFMA2, scalar coefficients broadcast inside the instruction).
struct Cp {
    float2 re, im;
};
__device__ __forceinline__ Cp padd(Cp a, Cp b) { return {add2(a.re, b.re), add2(a.im, b.im)}; }
__device__ __forceinline__ Cp psub(Cp a, Cp b) { return {sub2(a.re, b.re), sub2(a.im, b.im)}; }
__device__ __forceinline__ Cp pscale(float k, Cp a) { return {fmul2s(k, a.re), fmul2s(k, a.im)}; }
__device__ __forceinline__ Cp pfma(float k, Cp a, Cp c) { return {ffma2(k, a.re, c.re), ffma2(k, a.im, c.im)}; }
template <int S>   // b + S i e
__device__ __forceinline__ Cp paddi(Cp b, Cp e) {
    return S > 0 ? Cp{sub2(b.re, e.im), add2(b.im, e.re)} : Cp{add2(b.re, e.im), sub2(b.im, e.re)};
}
template <int S>   // b - S i e
__device__ __forceinline__ Cp psubi(Cp b, Cp e) {
    return S > 0 ? Cp{add2(b.re, e.im), sub2(b.im, e.re)} : Cp{sub2(b.re, e.im), add2(b.im, e.re)};
}
template <int S>   // S i a
__device__ __forceinline__ Cp pmuli(Cp a) {
    return S > 0 ? Cp{fmul2s(-1.f, a.im), a.re} : Cp{a.im, fmul2s(-1.f, a.re)};
}
// a * (c + i s) with scalar c, s broadcast
__device__ __forceinline__ Cp pcmul(Cp a, float c, float s) {
    return {ffma2(-s, a.im, fmul2s(c, a.re)), ffma2(s, a.re, fmul2s(c, a.im))};
}
// a * exp(S 2 pi i m / R), exact for the multiples of pi/2
template <int R, int S, int M>
__device__ __forceinline__ Cp twmul(Cp a) {
    constexpr int m = ((M % R) + R) % R;
    if constexpr (m == 0) {
        return a;
    } else if constexpr (4 * m == R) {
        return pmuli<S>(a);
    } else if constexpr (2 * m == R) {
        return pscale(-1.f, a);
    } else if constexpr (4 * m == 3 * R) {
        return pmuli<-S>(a);
    } else {
        constexpr float c = (float)cx_cos2pi(m, R);
        constexpr float s = (float)(S * cx_sin2pi(m, R));
        return pcmul(a, c, s);
    }
}

// ---------------------------------------------------------------- radix-R DFT codelets
// X[k] = sum_n v[n] exp(S 2 pi i n k / R), in place, registers only.
template <int R, int S>
struct Dft;

template <int S>
struct Dft<2, S> {
    static __device__ __forceinline__ void run(Cp* v) {
        Cp a = v[0], b = v[1];
        v[0] = padd(a, b);
        v[1] = psub(a, b);
    }
};
template <int S>
struct Dft<3, S> {
    static __device__ __forceinline__ void run(Cp* v) {
        constexpr float h = 0.86602540378443864676f;   // sin(2 pi / 3)
        Cp t = padd(v[1], v[2]), d = pscale(h, psub(v[1], v[2]));
        Cp m = pfma(-0.5f, t, v[0]);
        v[0] = padd(v[0], t);
        v[1] = paddi<S>(m, d);
        v[2] = psubi<S>(m, d);
    }
};
template <int S>
struct Dft<4, S> {
    static __device__ __forceinline__ void run(Cp* v) {
        Cp a = padd(v[0], v[2]), b = psub(v[0], v[2]);
        Cp c = padd(v[1], v[3]), d = psub(v[1], v[3]);
        v[0] = padd(a, c);
        v[2] = psub(a, c);
        v[1] = paddi<S>(b, d);
        v[3] = psubi<S>(b, d);
    }
};
template <int S>
struct Dft<5, S> {
    static __device__ __forceinline__ void run(Cp* v) {
        constexpr float c1 = (float)cx_cos2pi(1, 5), c2 = (float)cx_cos2pi(2, 5);
        constexpr float s1 = (float)cx_sin2pi(1, 5), s2 = (float)cx_sin2pi(2, 5);
        Cp t1 = padd(v[1], v[4]), t2 = padd(v[2], v[3]);
        Cp d1 = psub(v[1], v[4]), d2 = psub(v[2], v[3]);
        Cp a1 = pfma(c1, t1, pfma(c2, t2, v[0]));
        Cp a2 = pfma(c2, t1, pfma(c1, t2, v[0]));
        Cp b1 = pfma(s1, d1, pscale(s2, d2));
        Cp b2 = pfma(s2, d1, pscale(-s1, d2));
        v[0] = padd(v[0], padd(t1, t2));
        v[1] = paddi<S>(a1, b1);
        v[4] = psubi<S>(a1, b1);
        v[2] = paddi<S>(a2, b2);
        v[3] = psubi<S>(a2, b2);
    }
};
// R = P Q by Cooley-Tukey in registers: n = Q n1 + n2, k = k1 + P k2.
template <int P, int Q, int S>
struct DftCT {
    static __device__ __forceinline__ void run(Cp* v) {
        Cp y[Q][P];
        sfor<0, Q>([&](auto n2) {
            Cp a[P];
            sfor<0, P>([&](auto n1) { a[n1] = v[Q * n1 + n2]; });
            Dft<P, S>::run(a);
            sfor<0, P>([&](auto k1) { y[n2][k1] = twmul<P * Q, S, decltype(n2)::value * decltype(k1)::value>(a[k1]); });
        });
        sfor<0, P>([&](auto k1) {
            Cp b[Q];
            sfor<0, Q>([&](auto n2) { b[n2] = y[n2][k1]; });
            Dft<Q, S>::run(b);
            sfor<0, Q>([&](auto k2) { v[k1 + P * k2] = b[k2]; });
        });
    }
};
template <int S> struct Dft<6, S> : DftCT<2, 3, S> {};
template <int S> struct Dft<8, S> : DftCT<2, 4, S> {};
template <int S> struct Dft<9, S> : DftCT<3, 3, S> {};
template <int S> struct Dft<10, S> : DftCT<2, 5, S> {};
template <int S> struct Dft<12, S> : DftCT<3, 4, S> {};
template <int S> struct Dft<15, S> : DftCT<3, 5, S> {};
template <int S> struct Dft<16, S> : DftCT<4, 4, S> {};

// exp(2 pi i m / N) for m < N, evaluated at compile time (fp64 series, rounded once)
template <int N>
struct TwTable {
    float2 v[N];
    constexpr TwTable() : v() {
        for (int m = 0; m < N; ++m) {
            v[m].x = (float)cx_cos2pi(m, N);
            v[m].y = (float)cx_sin2pi(m, N);
        }
    }
};
template <int N>
__device__ const TwTable<N> kTw = TwTable<N>();

// ---------------------------------------------------------------- column block geometry
constexpr int NCOL = 8;      // columns per CTA: 4 (k, M-k) pairs = 4 SIMD column pairs
// Threads per CTA: every pass has 4 N / R tasks and each thread holds at most one
// (the passes run in place: load, barrier, store), so NT >= 4 N / min(R).
template <int N, int R1, int R2, int R3>
constexpr int threads() {
    int r = R1 < R2 ? R1 : R2;
    r = r < R3 ? r : R3;
    int t = (4 * N / r + 31) / 32 * 32;
    return t < 128 ? 128 : t;
}
// Shared memory: A = the transform buffer, two planes (re, im) of [N][NCOL] floats
// (a column pair's value at row y is one 8-byte word: a half-warp of a pass touches
// 4 rows x 4 pairs = 128 contiguous bytes; the first pass stores with row stride
// R1, conflict-free because every radix plan starts with an odd radix).
// B = the cached spectrum tile R^[y][pair s: (k, M-k)] (match) fetched by
// cp.async at kernel start, so its DRAM latency hides behind the forward FFT.
// tw = exp(2 pi i m / N).
template <int N>
constexpr size_t smem_bytes() {
    return sizeof(float) * 4 * (size_t)NCOL * N + sizeof(float2) * N;
}

// One Stockham pass of radix R, in place over the 4 column pairs: L = product of
// the radices already applied.  Twiddle exp(S 2 pi i j k / (L R)) = tw[j k N/(L R)].
template <int N, int R, int L, int S, int NT>
__device__ __forceinline__ void pass(float* __restrict__ re, float* __restrict__ im, const float2* __restrict__ tw) {
    constexpr int NTASK = N / R;
    static_assert(4 * NTASK <= NT, "one task per thread");
    const int tau = threadIdx.x, pp = 2 * (tau & 3), t = tau >> 2;
    const bool act = tau < 4 * NTASK;
    Cp v[R];
    if (act) {
        sfor<0, R>([&](auto j) {
            const int o = (t + decltype(j)::value * NTASK) * NCOL + pp;
            v[j] = {*reinterpret_cast<const float2*>(re + o), *reinterpret_cast<const float2*>(im + o)};
        });
    }
    __syncthreads();
    if (act) {
        if constexpr (L > 1) {
            const int step = (t % L) * (N / (L * R));
            sfor<1, R>([&](auto j) {
                const float2 w = tw[decltype(j)::value * step];
                v[j] = pcmul(v[j], w.x, S * w.y);
            });
        }
        Dft<R, S>::run(v);
        const int base = (t / L) * L * R + (t % L);
        sfor<0, R>([&](auto r) {
            const int o = (base + decltype(r)::value * L) * NCOL + pp;
            *reinterpret_cast<float2*>(re + o) = v[r].re;
            *reinterpret_cast<float2*>(im + o) = v[r].im;
        });
    }
    __syncthreads();
}

template <int N, int R1, int R2, int R3, int S, int NT>
__device__ __forceinline__ void fft3(float* re, float* im, const float2* tw) {
    pass<N, R1, 1, S, NT>(re, im, tw);
    pass<N, R2, R1, S, NT>(re, im, tw);
    pass<N, R3, R1 * R2, S, NT>(re, im, tw);
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

// MODE 0: Z (rows FFT of R) -> spectrum out;  MODE 1: Z (rows FFT of T), spectrum Rs
// -> packed rows of P = R^ conj(T^) after the inverse column FFT, written to out.
// grid (ncta_main + 1, batch): CTA a < ncta_main owns the pairs k = 4a+1 .. 4a+4,
// pair s in columns 2s (k) and 2s+1 (M-k), so the global phases move a pair as one
// 8-byte word per plane; CTA ncta_main owns column 0.  The global phases map
// task = 4 y + s and issue all of a thread's loads before using them.
template <int N, int R1, int R2, int R3, int MODE, int NT>
__global__ void __launch_bounds__(NT, (NT <= 384 ? 2 : 1))
    k_pce_cols(const float2* __restrict__ Z, const float2* __restrict__ Rs, float2* __restrict__ out, int M, int W,
               int ncta_main) {
    static_assert(R1 * R2 * R3 == N, "radix plan");
    static_assert(R1 % 2 == 1 || (R1 & (R1 - 1)) == 0, "first radix odd (or a power-of-two plan)");
    constexpr int KQ = (4 * N + NT - 1) / NT;   // (y, pair) tasks per thread
    constexpr int KP = (N + NT - 1) / NT;       // column-0 tasks per thread
    constexpr int PL = NCOL * N;                // floats per plane
    extern __shared__ float sm[];
    float *Ar = sm, *Ai = sm + PL;
    float2* Bt = reinterpret_cast<float2*>(sm + 2 * PL);   // [N][NCOL] complex
    float2* tw = reinterpret_cast<float2*>(sm + 4 * PL);
    __shared__ float2 wk[4];   // exp(-2 pi i k / W) of the 4 pairs
    const int tid = threadIdx.x;
    const size_t plane = (size_t)N * M;
    const float2* Zb = Z + (size_t)blockIdx.y * plane;
    float2* Ob = out + (size_t)blockIdx.y * plane;
    const bool packed = (int)blockIdx.x == ncta_main;
    const int npair = M / 2, k0 = 4 * blockIdx.x + 1;
    // pair access: (value at k, value at M-k) of pair s, row y
    auto put2 = [&](int y, int s, float2 vk, float2 vm) {
        *reinterpret_cast<float2*>(Ar + y * NCOL + 2 * s) = make_float2(vk.x, vm.x);
        *reinterpret_cast<float2*>(Ai + y * NCOL + 2 * s) = make_float2(vk.y, vm.y);
    };
    auto get2 = [&](int y, int s, float2& vk, float2& vm) {
        const float2 r = *reinterpret_cast<const float2*>(Ar + y * NCOL + 2 * s);
        const float2 i = *reinterpret_cast<const float2*>(Ai + y * NCOL + 2 * s);
        vk = make_float2(r.x, i.x);
        vm = make_float2(r.y, i.y);
    };
    auto put0 = [&](int y, float2 v) {
        Ar[y * NCOL] = v.x;
        Ai[y * NCOL] = v.y;
    };
    auto get0 = [&](int y) { return make_float2(Ar[y * NCOL], Ai[y * NCOL]); };

    if constexpr (MODE == 1) {   // prefetch the R^ tile: Bt[y][2s] = R^[y][k], Bt[y][2s+1] = R^[y][M-k]
        const float2* Rb = Rs + (size_t)blockIdx.y * plane;
        if (!packed) {
            for (int task = tid; task < 8 * N; task += NT) {
                const int c = task & 7, y = task >> 3, s = c >> 1, k = k0 + s;
                if (k <= npair) cp_async8(Bt + y * NCOL + c, Rb + (size_t)y * M + ((c & 1) ? M - k : k));
            }
        } else {
            for (int y = tid; y < N; y += NT) cp_async8(Bt + y * NCOL, Rb + (size_t)y * M);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int m = tid; m < N; m += NT) tw[m] = kTw<N>.v[m];

    // untangle: X[k] = (Z[k] + conj Z[M-k])/2 - (i/2) w_k (Z[k] - conj Z[M-k]),
    // X[M-k] likewise with w_{M-k} = -conj(w_k); X[0], X[M] packed as X[0] + i X[M]
    if (!packed) {
        float2 zk[KQ], zm[KQ];
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
            const int task = tid + q * NT, s = task & 3, y = task >> 2, k = k0 + s;
            zk[q] = zm[q] = make_float2(0.f, 0.f);
            if (task < 4 * N && k <= npair) {
                zk[q] = Zb[(size_t)y * M + k];
                zm[q] = Zb[(size_t)y * M + (M - k)];
            }
        }
        if (tid < 4) {
            double sn, cs;
            sincospi(-2.0 * (k0 + tid) / W, &sn, &cs);
            wk[tid] = make_float2((float)cs, (float)sn);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
            const int task = tid + q * NT, s = task & 3, y = task >> 2;
            if (task < 4 * N) {
                const float2 w = wk[s], wm = make_float2(-w.x, w.y);
                const float2 sk = cadd(zk[q], conjf2(zm[q])), dk = csub(zk[q], conjf2(zm[q]));
                const float2 sm_ = cadd(zm[q], conjf2(zk[q])), dm = csub(zm[q], conjf2(zk[q]));
                const float2 ek = muli<-1>(cmul(w, dk)), em = muli<-1>(cmul(wm, dm));
                put2(y, s, make_float2(0.5f * (sk.x + ek.x), 0.5f * (sk.y + ek.y)),
                     make_float2(0.5f * (sm_.x + em.x), 0.5f * (sm_.y + em.y)));
            }
        }
    } else {
        float2 z0[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) {
            const int y = tid + q * NT;
            if (y < N) z0[q] = Zb[(size_t)y * M];
        }
#pragma unroll
        for (int q = 0; q < KP; ++q) {
            const int y = tid + q * NT;
            if (y < N) put0(y, make_float2(z0[q].x + z0[q].y, z0[q].x - z0[q].y));
        }
    }
    __syncthreads();
    fft3<N, R1, R2, R3, -1, NT>(Ar, Ai, tw);

    if constexpr (MODE == 0) {
        if (!packed) {
#pragma unroll 4
            for (int task = tid; task < 4 * N; task += NT) {
                const int s = task & 3, y = task >> 2, k = k0 + s;
                if (k > npair) continue;
                float2 vk, vm;
                get2(y, s, vk, vm);
                Ob[(size_t)y * M + k] = vk;
                if (M - k != k) Ob[(size_t)y * M + (M - k)] = vm;
            }
        } else {
            for (int y = tid; y < N; y += NT) Ob[(size_t)y * M] = get0(y);
        }
        return;
    } else {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (!packed) {
#pragma unroll 4
            for (int task = tid; task < 4 * N; task += NT) {
                const int s = task & 3, y = task >> 2;
                if (k0 + s > npair) continue;
                const float4 r = *reinterpret_cast<const float4*>(Bt + y * NCOL + 2 * s);
                float2 tk, tm;
                get2(y, s, tk, tm);
                put2(y, s, cmul(make_float2(r.x, r.y), conjf2(tk)), cmul(make_float2(r.z, r.w), conjf2(tm)));
            }
            __syncthreads();
        } else {
            // the packed column C = F(X0) + i F(XM): F(X0)[v] = (C[v] + conj C[-v])/2,
            // F(XM)[v] = -(i/2)(C[v] - conj C[-v]); P = PA + i PB, PA[0] = 0 (DC).
            // Reads A[y] and A[-y]: all reads before any write.
            float2 pv[KP];
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const int y = tid + q * NT;
                if (y < N) {
                    const int ym = y ? N - y : 0;
                    const float2 t = get0(y), tm = conjf2(get0(ym));
                    const float2 r = Bt[y * NCOL], rm = conjf2(Bt[ym * NCOL]);
                    const float2 ta = cadd(t, tm), tb = muli<-1>(csub(t, tm));
                    const float2 ra = cadd(r, rm), rb = muli<-1>(csub(r, rm));
                    float2 pa = cmul(ra, conjf2(ta)), pb = cmul(rb, conjf2(tb));
                    if (y == 0) pa = make_float2(0.f, 0.f);
                    const float2 p = cadd(pa, muli<1>(pb));
                    pv[q] = make_float2(0.25f * p.x, 0.25f * p.y);
                }
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const int y = tid + q * NT;
                if (y < N) put0(y, pv[q]);
            }
            __syncthreads();
        }
        fft3<N, R1, R2, R3, 1, NT>(Ar, Ai, tw);
        // re-tangle: Z'[k] = (X[k] + conj X[M-k]) + i e_k (X[k] - conj X[M-k]),
        // e_k = exp(2 pi i k / W) = conj(w_k), e_{M-k} = -w_k
        if (!packed) {
#pragma unroll 4
            for (int task = tid; task < 4 * N; task += NT) {
                const int s = task & 3, y = task >> 2, k = k0 + s;
                if (k > npair) continue;
                float2 xk, xm;
                get2(y, s, xk, xm);
                const float2 w = wk[s], ek = conjf2(w), em = make_float2(-w.x, -w.y);
                const float2 zk = cadd(cadd(xk, conjf2(xm)), muli<1>(cmul(ek, csub(xk, conjf2(xm)))));
                Ob[(size_t)y * M + k] = zk;
                if (M - k != k) {
                    const float2 zm = cadd(cadd(xm, conjf2(xk)), muli<1>(cmul(em, csub(xm, conjf2(xk)))));
                    Ob[(size_t)y * M + (M - k)] = zm;
                }
            }
        } else {
            for (int y = tid; y < N; y += NT) {
                const float2 x = get0(y);   // X0 + i XM, both real
                Ob[(size_t)y * M] = make_float2(x.x + x.y, x.x - x.y);
            }
        }
    }
}

template <int N, int R1, int R2, int R3>
static int launch_cols(int mode, const float2* Z, const float2* Rs, float2* out, int M, int W, int batch,
                       cudaStream_t st) {
    constexpr int NT = threads<N, R1, R2, R3>();
    static DeviceFlags done0, done1;
    const size_t sm = smem_bytes<N>();
    const void* fn = mode ? (const void*)k_pce_cols<N, R1, R2, R3, 1, NT> : (const void*)k_pce_cols<N, R1, R2, R3, 0, NT>;
    if (int rc = set_smem_attr(fn, sm, mode ? done1 : done0)) return rc;
    const int ncta_main = (M / 2 + 3) / 4;
    dim3 grid(ncta_main + 1, batch);
    {
        KTimer kt(mode ? "pce_cols_match" : "pce_cols_fwd", st);
        if (mode)
            k_pce_cols<N, R1, R2, R3, 1, NT><<<grid, NT, sm, st>>>(Z, Rs, out, M, 2 * M, ncta_main);
        else
            k_pce_cols<N, R1, R2, R3, 0, NT><<<grid, NT, sm, st>>>(Z, Rs, out, M, 2 * M, ncta_main);
    }
    count_launch();
    return check_launch("k_pce_cols");
}

}  // namespace fft

// Heights with a compiled radix plan (the PCE plan uses the 2-D cuFFT path otherwise).
#define PRNU_PCE_COL_PLANS(X) \
    X(720, 9, 8, 10)          \
    X(1080, 15, 8, 9)         \
    X(500, 5, 10, 10)         \
    X(480, 5, 6, 16)          \
    X(128, 8, 4, 4)           \
    X(125, 5, 5, 5)           \
    X(96, 3, 4, 8)            \
    X(64, 4, 4, 4)            \
    X(48, 3, 4, 4)            \
    X(45, 3, 3, 5)            \
    X(27, 3, 3, 3)

bool pce_cols_supported(int H) {
#define PRNU_X(n, a, b, c) \
    if (H == n) return true;
    PRNU_PCE_COL_PLANS(PRNU_X)
#undef PRNU_X
    return false;
}

int launch_pce_cols(int mode, const void* Z, const void* Rs, void* out, int H, int W, int batch, cudaStream_t st) {
    const int M = W / 2;
    const float2* z = reinterpret_cast<const float2*>(Z);
    const float2* r = reinterpret_cast<const float2*>(Rs);
    float2* o = reinterpret_cast<float2*>(out);
#define PRNU_X(n, a, b, c) \
    if (H == n) return fft::launch_cols<n, a, b, c>(mode, z, r, o, M, W, batch, st);
    PRNU_PCE_COL_PLANS(PRNU_X)
#undef PRNU_X
    return fail(PRNU_INVALID_ARG, "pce columns: no radix plan for this height");
}

}  // namespace prnu
