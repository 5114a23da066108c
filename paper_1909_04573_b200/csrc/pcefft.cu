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
#include "pce.cuh"


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
// Threads per CTA: the in-place pass (forward pass 2) needs one task per thread,
// 4 N / R2 tasks; every other pass loops.  Plans put their largest radix second.
template <int N, int R1, int R2, int R3>
constexpr int threads() {
    int t = (4 * N / R2 + 31) / 32 * 32;
    return t < 128 ? 128 : t;
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

// ---------------------------------------------------------------- fused kernel (all pairs but column 0)
// Pair layout: one float4 per (row, pair s) = (re_k, re_{M-k}, im_k, im_{M-k}), a
// row of 4 pairs = 64 bytes; a quarter-warp's LDS.128 / STS.128 covers 2 rows.
// Shared-memory round trips per element: 5 (the untangle is fused into the first
// forward pass, which reads Z from global; the conjugate product into the last
// forward pass; the re-tangle and the global store into the last inverse pass).
__device__ __forceinline__ Cp ld4(const float4* A, int i) {
    const float4 q = A[i];
    return {make_float2(q.x, q.y), make_float2(q.z, q.w)};
}
__device__ __forceinline__ void st4(float4* A, int i, Cp v) { A[i] = make_float4(v.re.x, v.re.y, v.im.x, v.im.y); }

template <int N, int R, int L, int S>
__device__ __forceinline__ void twiddle(Cp* v, int t, const float2* __restrict__ tw) {
    if constexpr (L > 1) {
        const int step = (t % L) * (N / (L * R));
        sfor<1, R>([&](auto j) {
            const float2 w = tw[decltype(j)::value * step];
            v[j] = pcmul(v[j], w.x, S * w.y);
        });
    }
}

// in-place Stockham pass over the float4 pair layout
template <int N, int R, int L, int S, int NT>
__device__ __forceinline__ void pass4(float4* __restrict__ A, const float2* __restrict__ tw) {
    constexpr int NTASK = N / R;
    static_assert(4 * NTASK <= NT, "one task per thread");
    const int tau = threadIdx.x, s = tau & 3, t = tau >> 2;
    const bool act = tau < 4 * NTASK;
    Cp v[R];
    if (act) sfor<0, R>([&](auto j) { v[j] = ld4(A, (t + decltype(j)::value * NTASK) * 4 + s); });
    __syncthreads(); PRNU_STRESS(41);
    if (act) {
        twiddle<N, R, L, S>(v, t, tw);
        Dft<R, S>::run(v);
        const int base = (t / L) * L * R + (t % L);
        sfor<0, R>([&](auto r) { st4(A, (base + decltype(r)::value * L) * 4 + s, v[r]); });
    }
    __syncthreads(); PRNU_STRESS(42);
}

// out-of-place variant (no barrier between the loads and the stores)
template <int N, int R, int L, int S, int NT>
__device__ __forceinline__ void pass4o(const float4* __restrict__ A, float4* __restrict__ B,
                                       const float2* __restrict__ tw) {
    constexpr int NTASK = N / R;
    for (int tau = threadIdx.x; tau < 4 * NTASK; tau += NT) {
        const int s = tau & 3, t = tau >> 2;
        Cp v[R];
        sfor<0, R>([&](auto j) { v[j] = ld4(A, (t + decltype(j)::value * NTASK) * 4 + s); });
        twiddle<N, R, L, S>(v, t, tw);
        Dft<R, S>::run(v);
        const int base = (t / L) * L * R + (t % L);
        sfor<0, R>([&](auto r) { st4(B, (base + decltype(r)::value * L) * 4 + s, v[r]); });
    }
    __syncthreads(); PRNU_STRESS(43);
}

template <int N>
constexpr size_t smem_bytes_f() {
    return sizeof(float4) * 8 * (size_t)N + sizeof(float2) * ((N + 1) & ~1);
}

// Column 0 (the packed X[0] + i X[M]): lane k of pair 0, the other lanes zero; its
// conjugate product separates the two Hermitian halves, which needs rows v and -v:
// F(X0)[v] = (C[v] + conj C[-v])/2, F(XM)[v] = -(i/2)(C[v] - conj C[-v]);
// P = PA + i PB with PA[0] = 0 (the DC bin).
template <int N, int R1, int R2, int R3, int MODE, int NT>
__device__ __forceinline__ void packed_column(const float2* __restrict__ Zb, const float2* __restrict__ Rb,
                                              float2* __restrict__ Ob, int M, float4* A, float4* B,
                                              const float2* tw) {
    const int tid = threadIdx.x;
    for (int y = tid; y < N; y += NT) {
        const float2 z0 = Zb[(size_t)y * M];
        A[y * 4] = make_float4(z0.x + z0.y, 0.f, z0.x - z0.y, 0.f);
        A[y * 4 + 1] = A[y * 4 + 2] = A[y * 4 + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads(); PRNU_STRESS(44);
    pass4o<N, R1, 1, -1, NT>(A, B, tw);
    pass4o<N, R2, R1, -1, NT>(B, A, tw);
    pass4o<N, R3, R1 * R2, -1, NT>(A, B, tw);
    if constexpr (MODE == 0) {
        for (int y = tid; y < N; y += NT) Ob[(size_t)y * M] = make_float2(B[y * 4].x, B[y * 4].z);
        return;
    } else {
        for (int y = tid; y < N; y += NT) {
            const int ym = y ? N - y : 0;
            const float2 t = make_float2(B[y * 4].x, B[y * 4].z), tm = make_float2(B[ym * 4].x, -B[ym * 4].z);
            const float2 r = Rb[(size_t)y * M], rm = conjf2(Rb[(size_t)ym * M]);
            const float2 ta = cadd(t, tm), tb = muli<-1>(csub(t, tm));
            const float2 ra = cadd(r, rm), rb = muli<-1>(csub(r, rm));
            float2 pa = cmul(ra, conjf2(ta)), pb = cmul(rb, conjf2(tb));
            if (y == 0) pa = make_float2(0.f, 0.f);
            const float2 p = cadd(pa, muli<1>(pb));
            A[y * 4] = make_float4(0.25f * p.x, 0.f, 0.25f * p.y, 0.f);
            A[y * 4 + 1] = A[y * 4 + 2] = A[y * 4 + 3] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads(); PRNU_STRESS(45);
        pass4o<N, R1, 1, 1, NT>(A, B, tw);
        pass4o<N, R2, R1, 1, NT>(B, A, tw);
        pass4o<N, R3, R1 * R2, 1, NT>(A, B, tw);
        for (int y = tid; y < N; y += NT) {
            const float x0 = B[y * 4].x, xm = B[y * 4].z;   // X0 + i XM, both real
            Ob[(size_t)y * M] = make_float2(x0 + xm, x0 - xm);
        }
    }
}

// grid (ncta_main + 1, batch): CTA a < ncta_main owns the pairs k = 4a+1 .. 4a+4
// (k <= M/2) and their mirrors M-k; the last CTA owns column 0.
template <int N, int R1, int R2, int R3, int MODE, int NT>
__global__ void __launch_bounds__(NT, (NT <= 384 ? 2 : 1))
    k_pce_cols_f(const float2* __restrict__ Z, const float2* __restrict__ Rs, float2* __restrict__ out, int M,
                 int W) {
    static_assert(R1 * R2 * R3 == N, "radix plan");
    static_assert(R1 % 2 == 1 || (R1 & (R1 - 1)) == 0, "first radix odd (or a power-of-two plan)");
    extern __shared__ float4 sm4[];
    float4* A = sm4;                                          // [N][4 pairs]
    float4* B4 = sm4 + 4 * N;                                 // [N][4 pairs]: the R^ tile, then the P / inverse buffer
    float2* Bt = reinterpret_cast<float2*>(B4);               // R^ (k, M-k) of pair s at [y][2s], [y][2s+1]
    float2* tw = reinterpret_cast<float2*>(sm4 + 8 * N);      // exp(2 pi i m / N)
    __shared__ float2 wk[4];                                  // exp(-2 pi i k / W) of the 4 pairs
    const int tid = threadIdx.x;
    const size_t plane = (size_t)N * M;
    const float2* Zb = Z + (size_t)blockIdx.y * plane;
    const float2* Rb = Rs + (size_t)blockIdx.y * plane;
    float2* Ob = out + (size_t)blockIdx.y * plane;
    const int npair = M / 2, k0 = 4 * blockIdx.x + 1;
    const bool packed = blockIdx.x == gridDim.x - 1;

    // async copies: group 0 = the twiddle table (waited for before forward pass 2),
    // group 1 = the R^ tile (match; waited for before the conjugate product)
    for (int m = tid; m < N; m += NT) cp_async8(tw + m, &kTw<N>.v[m]);
    asm volatile("cp.async.commit_group;" ::: "memory");
    if constexpr (MODE == 1) {
        if (!packed) {
            for (int task = tid; task < 8 * N; task += NT) {
                const int c = task & 7, y = task >> 3, k = k0 + (c >> 1);
                if (k <= npair) cp_async8(Bt + y * NCOL + c, Rb + (size_t)y * M + ((c & 1) ? M - k : k));
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (packed) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        packed_column<N, R1, R2, R3, MODE, NT>(Zb, Rb, Ob, M, A, B4, tw);
        return;
    }
    if (tid < 4) {
        double sn, cs;
        sincospi(-2.0 * (k0 + tid) / W, &sn, &cs);
        wk[tid] = make_float2((float)cs, (float)sn);
    }
    __syncthreads(); PRNU_STRESS(46);

    const int s = tid & 3, k = k0 + s;   // NT % 4 == 0: a thread keeps its pair in every pass
    const bool kv = k <= npair;
    // forward pass 1 + untangle: X[k] = (Z[k] + conj Z[M-k])/2 - (i/2) w_k (Z[k] - conj Z[M-k]),
    // X[M-k] likewise with w_{M-k} = -conj(w_k).  All of a thread's loads are issued first.
    {
        constexpr int NTASK = N / R1, KT = (4 * NTASK + NT - 1) / NT;
        float2 zk[KT][R1], zm[KT][R1];
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            const int tau = tid + q * NT, t = tau >> 2;
            const bool ld = kv && tau < 4 * NTASK;
            sfor<0, R1>([&](auto j) {
                const int y = t + decltype(j)::value * NTASK;
                zk[q][j] = ld ? Zb[(size_t)y * M + k] : make_float2(0.f, 0.f);
                zm[q][j] = ld ? Zb[(size_t)y * M + (M - k)] : make_float2(0.f, 0.f);
            });
        }
        const float2 w = wk[s], wm = make_float2(-w.x, w.y);
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            const int tau = tid + q * NT, t = tau >> 2;
            if (tau < 4 * NTASK) {
                Cp v[R1];
                sfor<0, R1>([&](auto j) {
                    const float2 a = zk[q][j], c = zm[q][j];
                    const float2 sk = cadd(a, conjf2(c)), dk = csub(a, conjf2(c));
                    const float2 sm_ = cadd(c, conjf2(a)), dm = csub(c, conjf2(a));
                    const float2 ek = muli<-1>(cmul(w, dk)), em = muli<-1>(cmul(wm, dm));
                    v[j] = {make_float2(0.5f * (sk.x + ek.x), 0.5f * (sm_.x + em.x)),
                            make_float2(0.5f * (sk.y + ek.y), 0.5f * (sm_.y + em.y))};
                });
                Dft<R1, -1>::run(v);
                sfor<0, R1>([&](auto r) { st4(A, (t * R1 + decltype(r)::value) * 4 + s, v[r]); });
            }
        }
        if constexpr (MODE == 1)
            asm volatile("cp.async.wait_group 1;" ::: "memory");   // the twiddles (the R^ tile may still fly)
        else
            asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads(); PRNU_STRESS(47);
    }
    pass4<N, R2, R1, -1, NT>(A, tw);
    // forward pass 3 + (MODE 0) the spectrum store / (MODE 1) P = R^ conj(T^) in natural
    // order, written over the R^ tile (each (row, pair) read and written by one thread)
    {
        constexpr int NTASK = N / R3, L = R1 * R2;
        if constexpr (MODE == 1) {
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads(); PRNU_STRESS(48);
        }
        for (int tau = tid; tau < 4 * NTASK; tau += NT) {
            const int t = tau >> 2;
            Cp v[R3];
            sfor<0, R3>([&](auto j) { v[j] = ld4(A, (t + decltype(j)::value * NTASK) * 4 + s); });
            twiddle<N, R3, L, -1>(v, t, tw);
            Dft<R3, -1>::run(v);
            const int base = (t / L) * L * R3 + (t % L);
            if constexpr (MODE == 0) {
                if (kv) {
                    sfor<0, R3>([&](auto r) {
                        const int y = base + decltype(r)::value * L;
                        Ob[(size_t)y * M + k] = make_float2(v[r].re.x, v[r].im.x);
                        if (M - k != k) Ob[(size_t)y * M + (M - k)] = make_float2(v[r].re.y, v[r].im.y);
                    });
                }
            } else {
                sfor<0, R3>([&](auto r) {
                    const int y = base + decltype(r)::value * L;
                    const float4 q = B4[y * 4 + s];   // (R^k, R^{M-k})
                    const float2 pk = cmul(make_float2(q.x, q.y), make_float2(v[r].re.x, -v[r].im.x));
                    const float2 pm = cmul(make_float2(q.z, q.w), make_float2(v[r].re.y, -v[r].im.y));
                    st4(B4, y * 4 + s, Cp{make_float2(pk.x, pm.x), make_float2(pk.y, pm.y)});
                });
            }
        }
        if constexpr (MODE == 0) return;
        __syncthreads(); PRNU_STRESS(49);
    }
    // inverse passes 1, 2 out of place: B4 -> A -> B4
    pass4o<N, R1, 1, 1, NT>(B4, A, tw);
    pass4o<N, R2, R1, 1, NT>(A, B4, tw);
    // inverse pass 3 + re-tangle + global store:
    // Z'[k] = (X[k] + conj X[M-k]) + i e_k (X[k] - conj X[M-k]), e_k = conj(w_k), e_{M-k} = -w_k
    {
        constexpr int NTASK = N / R3, L = R1 * R2;
        const float2 w = wk[s], ek = conjf2(w), em = make_float2(-w.x, -w.y);
        for (int tau = tid; tau < 4 * NTASK; tau += NT) {
            const int t = tau >> 2;
            Cp v[R3];
            sfor<0, R3>([&](auto j) { v[j] = ld4(B4, (t + decltype(j)::value * NTASK) * 4 + s); });
            twiddle<N, R3, L, 1>(v, t, tw);
            Dft<R3, 1>::run(v);
            const int base = (t / L) * L * R3 + (t % L);
            if (kv) {
                sfor<0, R3>([&](auto r) {
                    const int y = base + decltype(r)::value * L;
                    const float2 xk = make_float2(v[r].re.x, v[r].im.x), xm = make_float2(v[r].re.y, v[r].im.y);
                    Ob[(size_t)y * M + k] = cadd(cadd(xk, conjf2(xm)), muli<1>(cmul(ek, csub(xk, conjf2(xm)))));
                    if (M - k != k)
                        Ob[(size_t)y * M + (M - k)] =
                            cadd(cadd(xm, conjf2(xk)), muli<1>(cmul(em, csub(xm, conjf2(xk)))));
                });
            }
        }
    }
}

// ---------------------------------------------------------------- row kernel
// The row transforms of length M = W/2 (complex) over packed real rows.  CTA: 8
// rows as 4 row pairs (the SIMD pairs), in the same [n][4 pairs] float4 layout
// as the column kernel.  Pass 1 reads global memory (and may loop over tasks),
// pass 2 runs in place (one task per thread), pass 3 writes global memory.
//   ROW_FWD_REAL  X [b][H][W] real        -> Z [b][H][M] = FFT_M(x[2m] + i x[2m+1])
//   ROW_FWD_TPL   K (.) Iq, formed on load (the template of S:305 / R-18, the same
//                 single fp32 product as prnu_pce_template) -> Z
//   ROW_INV_PEAK  Z' [b][H][M] -> C [b][H][W] (unnormalised inverse) and the peak /
//                 energy partials of the CTA's rows: part[b][blockIdx.x]
enum { ROW_FWD_REAL = 0, ROW_FWD_TPL = 1, ROW_INV_PEAK = 2 };
struct RowArgs {
    const float* X;
    const float* K;
    int k_batch;
    const uint8_t* Iq;
    const float2* Zin;
    float2* Zout;
    float* C;
    PeakE* part;
    int H, nparts;
};
constexpr int ROWS = 8;   // rows per CTA

template <int M, int R1, int R2, int R3>
constexpr int row_threads() {
    int t = (4 * M / R2 + 31) / 32 * 32;
    return t < 128 ? 128 : t;
}
template <int M>
constexpr size_t row_smem_bytes() {
    return sizeof(float4) * 4 * (size_t)M + sizeof(float2) * ((M + 1) & ~1);
}

template <int M, int R1, int R2, int R3, int MODE, int NT>
__global__ void __launch_bounds__(NT, (NT <= 384 ? 2 : 1)) k_pce_rows(RowArgs a) {
    static_assert(R1 * R2 * R3 == M, "radix plan");
    static_assert(4 * (M / R2) <= NT, "pass 2: one task per thread");
    constexpr int S = MODE == ROW_INV_PEAK ? 1 : -1;
    constexpr int W = 2 * M;
    extern __shared__ float4 sm4[];
    float4* A = sm4;
    float2* tw = reinterpret_cast<float2*>(sm4 + 4 * M);
    const int tid = threadIdx.x, b = blockIdx.y, H = a.H;
    for (int m = tid; m < M; m += NT) cp_async8(tw + m, &kTw<M>.v[m]);   // waited for before pass 2
    asm volatile("cp.async.commit_group;" ::: "memory");

    // pass 1 (+ the load): task = 4 t + s, rows ra = r0 + 2s, rb = ra + 1; a thread's
    // KT tasks issue all their global loads before any is used
    {
        constexpr int NTASK = M / R1, KT = (4 * NTASK + NT - 1) / NT;
        Cp v[KT][R1];
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            const int tau = tid + q * NT, s = tau & 3, t = tau >> 2;
            const int ra = ROWS * blockIdx.x + 2 * s, rb = ra + 1;
            const bool va = ra < H && tau < 4 * NTASK, vb = rb < H && tau < 4 * NTASK;
            sfor<0, R1>([&](auto j) {
                const int n = t + decltype(j)::value * NTASK;
                float2 za = make_float2(0.f, 0.f), zb = za;
                if constexpr (MODE == ROW_FWD_REAL) {
                    const float* Xb = a.X + (size_t)b * H * W;
                    if (va) za = *reinterpret_cast<const float2*>(Xb + (size_t)ra * W + 2 * n);
                    if (vb) zb = *reinterpret_cast<const float2*>(Xb + (size_t)rb * W + 2 * n);
                } else if constexpr (MODE == ROW_FWD_TPL) {
                    const float* Kb = a.K + (a.k_batch == 1 ? 0 : (size_t)b * H * W);
                    const uint8_t* Ib = a.Iq + (size_t)b * H * W;
                    if (va) {
                        const float2 k = *reinterpret_cast<const float2*>(Kb + (size_t)ra * W + 2 * n);
                        const uchar2 c = *reinterpret_cast<const uchar2*>(Ib + (size_t)ra * W + 2 * n);
                        za = make_float2(k.x * (float)c.x, k.y * (float)c.y);
                    }
                    if (vb) {
                        const float2 k = *reinterpret_cast<const float2*>(Kb + (size_t)rb * W + 2 * n);
                        const uchar2 c = *reinterpret_cast<const uchar2*>(Ib + (size_t)rb * W + 2 * n);
                        zb = make_float2(k.x * (float)c.x, k.y * (float)c.y);
                    }
                } else {
                    const float2* Zb = a.Zin + (size_t)b * H * M;
                    if (va) za = Zb[(size_t)ra * M + n];
                    if (vb) zb = Zb[(size_t)rb * M + n];
                }
                v[q][j] = {make_float2(za.x, zb.x), make_float2(za.y, zb.y)};
            });
        }
#pragma unroll
        for (int q = 0; q < KT; ++q) {
            const int tau = tid + q * NT, s = tau & 3, t = tau >> 2;
            if (tau < 4 * NTASK) {
                Dft<R1, S>::run(v[q]);
                sfor<0, R1>([&](auto r) { st4(A, (t * R1 + decltype(r)::value) * 4 + s, v[q][r]); });
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads(); PRNU_STRESS(50);
    }
    pass4<M, R2, R1, S, NT>(A, tw);
    // pass 3 (+ the store / the peak and energy partials)
    {
        constexpr int NTASK = M / R3, L = R1 * R2;
        // per-thread candidates: one running max per row of the pair (its indices
        // increase with n, so strict > keeps the smallest index), energy in fp32 pairs
        float besta = -1.f, bestb = -1.f;
        int bia = -1, bib = -1;
        float2 ea = make_float2(0.f, 0.f), eb = ea;
        for (int tau = tid; tau < 4 * NTASK; tau += NT) {
            const int s = tau & 3, t = tau >> 2;
            const int ra = ROWS * blockIdx.x + 2 * s, rb = ra + 1;
            const bool va = ra < H, vb = rb < H;
            Cp v[R3];
            sfor<0, R3>([&](auto j) { v[j] = ld4(A, (t + decltype(j)::value * NTASK) * 4 + s); });
            twiddle<M, R3, L, S>(v, t, tw);
            Dft<R3, S>::run(v);
            const int base = (t / L) * L * R3 + (t % L);
            sfor<0, R3>([&](auto r) {
                const int n = base + decltype(r)::value * L;
                const float2 ca = make_float2(v[r].re.x, v[r].im.x), cb = make_float2(v[r].re.y, v[r].im.y);
                if constexpr (MODE == ROW_INV_PEAK) {
                    float* Cb = a.C + (size_t)b * H * W;
                    if (va) {
                        *reinterpret_cast<float2*>(Cb + (size_t)ra * W + 2 * n) = ca;
                        const float m0 = fabsf(ca.x), m1 = fabsf(ca.y);
                        if (m0 > besta) { besta = m0; bia = ra * W + 2 * n; }
                        if (m1 > besta) { besta = m1; bia = ra * W + 2 * n + 1; }
                        ea = fma2(ca, ca, ea);
                    }
                    if (vb) {
                        *reinterpret_cast<float2*>(Cb + (size_t)rb * W + 2 * n) = cb;
                        const float m0 = fabsf(cb.x), m1 = fabsf(cb.y);
                        if (m0 > bestb) { bestb = m0; bib = rb * W + 2 * n; }
                        if (m1 > bestb) { bestb = m1; bib = rb * W + 2 * n + 1; }
                        eb = fma2(cb, cb, eb);
                    }
                } else {
                    float2* Zb = a.Zout + (size_t)b * H * M;
                    if (va) Zb[(size_t)ra * M + n] = ca;
                    if (vb) Zb[(size_t)rb * M + n] = cb;
                }
            });
        }
        float best = besta;
        int bi = bia;
        if (better(bestb, bib, best, bi)) {
            best = bestb;
            bi = bib;
        }
        double e = ((double)ea.x + (double)ea.y) + ((double)eb.x + (double)eb.y);
        if constexpr (MODE == ROW_INV_PEAK) {
            // fixed-shape warp-shuffle reduction, then the NT/32 warp results in warp order
            constexpr int NW = NT / 32;
            __shared__ float sa[NW];
            __shared__ int si[NW];
            __shared__ double se[NW];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float a2 = __shfl_xor_sync(0xffffffffu, best, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(a2, i2, best, bi)) {
                    best = a2;
                    bi = i2;
                }
            }
            e = warp_sum(e);
            if ((tid & 31) == 0) {
                sa[tid >> 5] = best;
                si[tid >> 5] = bi;
                se[tid >> 5] = e;
            }
            __syncthreads(); PRNU_STRESS(51);
            if (tid == 0) {
                float bb = sa[0];
                int ii = si[0];
                double ee = se[0];
                for (int k = 1; k < NW; ++k) {
                    if (better(sa[k], si[k], bb, ii)) {
                        bb = sa[k];
                        ii = si[k];
                    }
                    ee += se[k];
                }
                a.part[(size_t)b * a.nparts + blockIdx.x] = PeakE{bb, ii, ee};
            }
        }
    }
}

template <int M, int R1, int R2, int R3>
static int launch_rows_t(int mode, const RowArgs& a, int batch, cudaStream_t st) {
    constexpr int NT = row_threads<M, R1, R2, R3>();
    static DeviceFlags d0, d1, d2;
    const size_t sm = row_smem_bytes<M>();
    dim3 grid((a.H + ROWS - 1) / ROWS, batch);
    const void* fn = mode == ROW_FWD_REAL ? (const void*)k_pce_rows<M, R1, R2, R3, ROW_FWD_REAL, NT>
                     : mode == ROW_FWD_TPL ? (const void*)k_pce_rows<M, R1, R2, R3, ROW_FWD_TPL, NT>
                                           : (const void*)k_pce_rows<M, R1, R2, R3, ROW_INV_PEAK, NT>;
    if (int rc = set_smem_attr(fn, sm, mode == ROW_FWD_REAL ? d0 : mode == ROW_FWD_TPL ? d1 : d2)) return rc;
    {
        KTimer kt(mode == ROW_INV_PEAK ? "pce_rows_inv" : "pce_rows_fwd", st);
        if (mode == ROW_FWD_REAL)
            k_pce_rows<M, R1, R2, R3, ROW_FWD_REAL, NT><<<grid, NT, sm, st>>>(a);
        else if (mode == ROW_FWD_TPL)
            k_pce_rows<M, R1, R2, R3, ROW_FWD_TPL, NT><<<grid, NT, sm, st>>>(a);
        else
            k_pce_rows<M, R1, R2, R3, ROW_INV_PEAK, NT><<<grid, NT, sm, st>>>(a);
    }
    count_launch();
    return check_launch("k_pce_rows");
}

template <int N, int R1, int R2, int R3>
static int launch_cols(int mode, const float2* Z, const float2* Rs, float2* out, int M, int W, int batch,
                       cudaStream_t st) {
    constexpr int NT = threads<N, R1, R2, R3>();
    static DeviceFlags done0, done1;
    const size_t sm = smem_bytes_f<N>();
    const void* fn =
        mode ? (const void*)k_pce_cols_f<N, R1, R2, R3, 1, NT> : (const void*)k_pce_cols_f<N, R1, R2, R3, 0, NT>;
    if (int rc = set_smem_attr(fn, sm, mode ? done1 : done0)) return rc;
    dim3 grid((M / 2 + 3) / 4 + 1, batch);
    {
        KTimer kt(mode ? "pce_cols_match" : "pce_cols_fwd", st);
        if (mode)
            k_pce_cols_f<N, R1, R2, R3, 1, NT><<<grid, NT, sm, st>>>(Z, Rs, out, M, 2 * M);
        else
            k_pce_cols_f<N, R1, R2, R3, 0, NT><<<grid, NT, sm, st>>>(Z, Rs, out, M, 2 * M);
    }
    count_launch();
    return check_launch("k_pce_cols");
}

}  // namespace fft

// Heights with a compiled radix plan (the PCE plan uses the 2-D cuFFT path otherwise).
#define PRNU_PCE_COL_PLANS(X) \
    X(720, 9, 8, 10)          \
    X(1080, 9, 15, 8)         \
    X(500, 5, 10, 10)         \
    X(480, 5, 16, 6)          \
    X(128, 8, 4, 4)           \
    X(125, 5, 5, 5)           \
    X(96, 3, 8, 4)            \
    X(64, 4, 4, 4)            \
    X(48, 3, 4, 4)            \
    X(45, 3, 3, 5)            \
    X(27, 3, 3, 3)

// Row lengths M = W/2 with a compiled radix plan (first radix odd: stride-R1 stores).
#define PRNU_PCE_ROW_PLANS(X) \
    X(640, 5, 16, 8)          \
    X(960, 15, 8, 8)          \
    X(250, 5, 5, 10)          \
    X(125, 5, 5, 5)           \
    X(96, 3, 4, 8)            \
    X(80, 5, 4, 4)            \
    X(30, 3, 2, 5)            \
    X(27, 3, 3, 3)            \
    X(20, 5, 2, 2)

bool pce_rows_supported(int W) {
    if (W % 2) return false;
#define PRNU_X(n, a, b, c) \
    if (W / 2 == n) return true;
    PRNU_PCE_ROW_PLANS(PRNU_X)
#undef PRNU_X
    return false;
}

int pce_rows_nparts(int H) { return (H + fft::ROWS - 1) / fft::ROWS; }

// mode 0: X -> Z;  1: K (.) Iq -> Z;  2: Z -> C + partials
int launch_pce_rows(int mode, const float* X, const float* K, int k_batch, const uint8_t* Iq, const void* Zin,
                    void* Zout, float* C, void* part, int H, int W, int batch, cudaStream_t st) {
    fft::RowArgs a{X, K, k_batch, Iq, reinterpret_cast<const float2*>(Zin), reinterpret_cast<float2*>(Zout), C,
                   reinterpret_cast<PeakE*>(part), H, pce_rows_nparts(H)};
#define PRNU_X(n, r1, r2, r3) \
    if (W / 2 == n) return fft::launch_rows_t<n, r1, r2, r3>(mode, a, batch, st);
    PRNU_PCE_ROW_PLANS(PRNU_X)
#undef PRNU_X
    return fail(PRNU_INVALID_ARG, "pce rows: no radix plan for this width");
}

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
