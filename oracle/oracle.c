/*
 * oracle.c — plain, slow, fp64 CPU oracle for the SDA-frame PRNU hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1909_04573_b200/) never imports, links or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * Citations: P:<line> = /root/reference/PAPER.md line, S:<line> = SPEC.md line,
 * R-<n> = the reading n listed in DESIGN.md §"Readings" (where the paper is
 * silent and a convention had to be chosen).
 *
 * Every function is a direct transcription of the definition it cites:
 * no blocking, fusion or reordering.  All floating point is IEEE fp64
 * (compiled with -O2 -ffp-contract=off -fno-fast-math).
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"):
 *   sda_average    exhaustive vs IEEE fp32 division (numpy), S:200-202 examples
 *   filters        spectral factorisation of the Daubechies polynomial (numpy
 *                  roots, independent), sum = sqrt2, orthonormality, moments
 *   dwt1d/idwt1d   numpy pad('symmetric') + convolve formulation, perfect
 *                  reconstruction <= 1e-10, constants and cubic polynomials
 *   box_mean       scipy.ndimage.uniform_filter(mode='reflect')
 *   residual       constant -> 0, offset invariance, transpose covariance,
 *                  homogeneity, sigma0 limits, white-noise attenuation,
 *                  impulse, 8x8 brute force with explicit matrices
 *   mle/finalize   closed forms, K recovery, ZM properties
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_LEVELS 8

/* ------------------------------------------------------------------ */
/* a1: SDA grouping and averaging.                                     */
/* P:124 "g non-intersecting equal-sized subgroups ... d = m/g frames" */
/* P:170-175  I_i^SDA = sum_{j=(i-1)d+1}^{id} I_j / d                   */
/* S:188 remainder m mod d dropped; S:189 d > m is an error.           */
/* R-11: the mean is the exact integer sum divided by d, rounded once  */
/* to the nearest fp32 (what S:197 "64-bit accumulation, emitted at    */
/* 32-bit" means for integer frames).                                  */
/* ------------------------------------------------------------------ */
long oracle_sda_groups(long m, long d) {
    if (d < 1 || m < 1 || d > m) return -1;
    return m / d;
}

int oracle_sda_average(const uint8_t* frames, long m, int H, int W, long d, float* out) {
    long ns = oracle_sda_groups(m, d);
    if (ns < 0) return 3;
    long P = (long)H * W;
    int64_t* s = (int64_t*)malloc(sizeof(int64_t) * P);
    for (long i = 0; i < ns; ++i) {
        /* exact integer sum of the group (integer addition: the order of the
           frames does not change the value), frame by frame for locality */
        memset(s, 0, sizeof(int64_t) * P);
        for (long j = i * d; j < (i + 1) * d; ++j)
            for (long p = 0; p < P; ++p) s[p] += frames[j * P + p];
        /* exact rational s/d -> fp32.  s < 2^53 so (double)s is exact;
           the fp64 quotient is then rounded to fp32.  tests/ pin this
           against IEEE fp32 division exhaustively for every depth used. */
        for (long p = 0; p < P; ++p) out[i * P + p] = (float)((double)s[p] / (double)d);
    }
    free(s);
    return 0;
}

/* ------------------------------------------------------------------ */
/* a2-a4: the denoiser F ("a denoising filter F, such as         */
/* [mihcak1999low]"; "The wavelet denoising algorithm [Mihcak]")  */
/* The paper gives no internals; S:117, S:149-150 parameterise it and  */
/* DESIGN.md readings R-1..R-8 fix what remains.                       */
/* ------------------------------------------------------------------ */

/* R-2: 8-tap Daubechies (4 vanishing moments) analysis low-pass, in the
   order used by the convolution below.  Pinned in tests by an independent
   spectral factorisation. */
static const double DEC_LO[8] = {
    -0.010597401785069032, 0.0328830116668852,   0.030841381835560764,
    -0.18703481171909309, -0.027983769416859854, 0.6308807679298589,
     0.7148465705529157,   0.2303778133088965};

/* Quadrature-mirror relations (orthogonal wavelet):
   dec_hi[k] = (-1)^(k+1) dec_lo[7-k]; rec_lo[k] = dec_lo[7-k];
   rec_hi[k] = dec_hi[7-k]. */
void oracle_filters(double* dec_lo, double* dec_hi, double* rec_lo, double* rec_hi) {
    for (int k = 0; k < 8; ++k) {
        double dl = DEC_LO[k];
        double dh = ((k % 2) ? 1.0 : -1.0) * DEC_LO[7 - k];
        if (dec_lo) dec_lo[k] = dl;
        if (dec_hi) dec_hi[k] = dh;
    }
    for (int k = 0; k < 8; ++k) {
        if (rec_lo) rec_lo[k] = DEC_LO[7 - k];
        if (rec_hi) rec_hi[k] = ((7 - k) % 2 ? 1.0 : -1.0) * DEC_LO[k];
    }
}

/* R-4: half-sample symmetric extension ("symmetric (mirror)").
   e_N(i) = r if r < N else 2N-1-r, with r = i mod 2N.                  */
int oracle_ext(long i, long N) {
    long P2 = 2 * N;
    long r = i % P2;
    if (r < 0) r += P2;
    return (int)(r < N ? r : P2 - 1 - r);
}

int oracle_subband_len(int N) { return (N + 7) / 2; }

/* R-5: 1-D analysis, N -> n = floor((N+7)/2):
   a[k] = sum_j dec_lo[j] x[e_N(2k+1-j)],  d[k] = sum_j dec_hi[j] x[e_N(2k+1-j)] */
void oracle_dwt1d(const double* x, long stride, int N, double* a, double* d, long ostride) {
    double lo[8], hi[8];
    oracle_filters(lo, hi, NULL, NULL);
    int n = oracle_subband_len(N);
    for (int k = 0; k < n; ++k) {
        double sa = 0.0, sd = 0.0;
        for (int j = 0; j < 8; ++j) {
            double v = x[(long)oracle_ext(2L * k + 1 - j, N) * stride];
            sa += lo[j] * v;
            sd += hi[j] * v;
        }
        a[(long)k * ostride] = sa;
        d[(long)k * ostride] = sd;
    }
}

/* R-5: 1-D synthesis, n -> N:
   x[t] = sum_k a[k] rec_lo[t+6-2k] + d[k] rec_hi[t+6-2k], only terms whose
   filter index lies in [0,8).  (Offset 6 = filter length - 2.)          */
void oracle_idwt1d(const double* a, const double* d, long istride, int n, int N, double* x, long stride) {
    double rl[8], rh[8];
    oracle_filters(NULL, NULL, rl, rh);
    for (int t = 0; t < N; ++t) {
        double s = 0.0;
        /* only k with 0 <= t+6-2k <= 7 contribute: k in [floor(t/2), floor((t+6)/2)] */
        int k0 = t / 2, k1 = (t + 6) / 2;
        if (k1 > n - 1) k1 = n - 1;
        for (int k = k0; k <= k1; ++k) {
            int f = t + 6 - 2 * k;
            if (f < 0 || f > 7) continue;
            s += a[(long)k * istride] * rl[f] + d[(long)k * istride] * rh[f];
        }
        x[(long)t * stride] = s;
    }
}

/* R-6: one 2-D level.  Rows (along W) first, then columns (along H).
   Output subbands, each nH x nW, row-major:
     aa = lo_y(lo_x)  (approximation)
     da = lo_y(hi_x)  (detail: high-pass along x)
     ad = hi_y(lo_x)  (detail: high-pass along y)
     dd = hi_y(hi_x)  (diagonal detail)                                   */
void oracle_dwt2d(const double* x, int NH, int NW, double* aa, double* da, double* ad, double* dd) {
    int nH = oracle_subband_len(NH), nW = oracle_subband_len(NW);
    double* L = (double*)malloc(sizeof(double) * (size_t)NH * nW);
    double* Hh = (double*)malloc(sizeof(double) * (size_t)NH * nW);
    for (int y = 0; y < NH; ++y)
        oracle_dwt1d(x + (long)y * NW, 1, NW, L + (long)y * nW, Hh + (long)y * nW, 1);
    for (int c = 0; c < nW; ++c) {
        oracle_dwt1d(L + c, nW, NH, aa + c, ad + c, nW);
        oracle_dwt1d(Hh + c, nW, NH, da + c, dd + c, nW);
    }
    free(L);
    free(Hh);
}

/* Inverse of one 2-D level: columns first, then rows (reverse order).
   aa may be NULL (treated as all zeros).                                */
void oracle_idwt2d(const double* aa, const double* da, const double* ad, const double* dd,
                   int NH, int NW, double* x) {
    int nH = oracle_subband_len(NH), nW = oracle_subband_len(NW);
    double* L = (double*)malloc(sizeof(double) * (size_t)NH * nW);
    double* Hh = (double*)malloc(sizeof(double) * (size_t)NH * nW);
    double* zero = NULL;
    if (!aa) {
        zero = (double*)calloc((size_t)nH * nW, sizeof(double));
        aa = zero;
    }
    for (int c = 0; c < nW; ++c) {
        oracle_idwt1d(aa + c, ad + c, nW, nH, NH, L + c, nW);
        oracle_idwt1d(da + c, dd + c, nW, nH, NH, Hh + c, nW);
    }
    for (int y = 0; y < NH; ++y)
        oracle_idwt1d(L + (long)y * nW, Hh + (long)y * nW, 1, nW, NW, x + (long)y * NW, 1);
    free(L);
    free(Hh);
    free(zero);
}

/* R-7: local mean of c^2 over a w x w window centred on (y,x), indices
   mirrored with e_n, always w^2 samples, divided by w^2.       */
void oracle_box_mean_sq(const double* c, int nH, int nW, int w, double* out) {
    int r = w / 2;
    /* mirrored indices e_n(i) for i in [-r, n+r), tabulated once */
    int* ey = (int*)malloc(sizeof(int) * (nH + 2 * r));
    int* ex = (int*)malloc(sizeof(int) * (nW + 2 * r));
    for (int i = -r; i < nH + r; ++i) ey[i + r] = oracle_ext(i, nH);
    for (int i = -r; i < nW + r; ++i) ex[i + r] = oracle_ext(i, nW);
    for (int y = 0; y < nH; ++y)
        for (int x = 0; x < nW; ++x) {
            double s = 0.0;
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx) {
                    double v = c[(long)ey[y + dy + r] * nW + ex[x + dx + r]];
                    s += v * v;
                }
            out[(long)y * nW + x] = s / ((double)w * (double)w);
        }
    free(ey);
    free(ex);
}

/* "each detail coefficient c is attenuated by the local Wiener
   factor est_var/(est_var+sigma0_sq), with est_var the minimum over the
   configured windows of max(0, local second moment - sigma0_sq)".
   Writes the DENOISED coefficient c * v/(v + sigma0^2).                 */
void oracle_shrink(const double* c, int nH, int nW, double sigma0_sq, const int* windows,
                   int n_windows, double* out) {
    long n = (long)nH * nW;
    double* est = (double*)malloc(sizeof(double) * n);
    double* m = (double*)malloc(sizeof(double) * n);
    for (long i = 0; i < n; ++i) est[i] = INFINITY;
    for (int wi = 0; wi < n_windows; ++wi) {
        oracle_box_mean_sq(c, nH, nW, windows[wi], m);
        for (long i = 0; i < n; ++i) {
            double v = m[i] - sigma0_sq;
            if (v < 0.0) v = 0.0;            /* max(0, local second moment - sigma0^2) */
            if (v < est[i]) est[i] = v;      /* minimum over the windows */
        }
    }
    for (long i = 0; i < n; ++i) out[i] = c[i] * (est[i] / (est[i] + sigma0_sq));
    free(est);
    free(m);
}

/* F(I): L-level decomposition, Wiener shrink of every detail subband,
   approximation passes through, inverse transform.
   Returns 2 (PlaneTooSmall) if H or W < 2^levels.                */
int oracle_denoise(const double* I, int H, int W, double sigma0_sq, const int* windows,
                   int n_windows, int levels, double* F) {
    if (levels < 1 || levels > ORACLE_MAX_LEVELS) return 4;
    if (H < (1 << levels) || W < (1 << levels)) return 2;
    int NH[ORACLE_MAX_LEVELS + 1], NW[ORACLE_MAX_LEVELS + 1];
    double *aa[ORACLE_MAX_LEVELS + 1], *da[ORACLE_MAX_LEVELS + 1], *ad[ORACLE_MAX_LEVELS + 1],
        *dd[ORACLE_MAX_LEVELS + 1];
    NH[0] = H;
    NW[0] = W;
    const double* cur = I;
    for (int l = 1; l <= levels; ++l) {
        NH[l] = oracle_subband_len(NH[l - 1]);
        NW[l] = oracle_subband_len(NW[l - 1]);
        size_t sz = sizeof(double) * (size_t)NH[l] * NW[l];
        aa[l] = (double*)malloc(sz);
        da[l] = (double*)malloc(sz);
        ad[l] = (double*)malloc(sz);
        dd[l] = (double*)malloc(sz);
        oracle_dwt2d(cur, NH[l - 1], NW[l - 1], aa[l], da[l], ad[l], dd[l]);
        cur = aa[l];
    }
    for (int l = 1; l <= levels; ++l) {
        size_t n = (size_t)NH[l] * NW[l];
        double* tmp = (double*)malloc(sizeof(double) * n);
        oracle_shrink(da[l], NH[l], NW[l], sigma0_sq, windows, n_windows, tmp);
        memcpy(da[l], tmp, sizeof(double) * n);
        oracle_shrink(ad[l], NH[l], NW[l], sigma0_sq, windows, n_windows, tmp);
        memcpy(ad[l], tmp, sizeof(double) * n);
        oracle_shrink(dd[l], NH[l], NW[l], sigma0_sq, windows, n_windows, tmp);
        memcpy(dd[l], tmp, sizeof(double) * n);
        free(tmp);
    }
    /* inverse, level L -> 1; the approximation aa[L] passes through */
    double* approx = aa[levels];
    for (int l = levels; l >= 1; --l) {
        double* out = (l == 1) ? F : (double*)malloc(sizeof(double) * (size_t)NH[l - 1] * NW[l - 1]);
        oracle_idwt2d(approx, da[l], ad[l], dd[l], NH[l - 1], NW[l - 1], out);
        if (l < levels) free(approx);
        approx = out;
    }
    for (int l = 1; l <= levels; ++l) {
        free(aa[l]);
        free(da[l]);
        free(ad[l]);
        free(dd[l]);
    }
    return 0;
}

/* a4: "W_k = I_k - \hat I^(0)_k, \hat I^(0)_k = F(I_k)";
   P:190-193 W^SDA = I^SDA - F(I^SDA).  The input is the fp32 SDA frame (or
   the u8 frame widened to fp32 at d = 1); the oracle works in fp64 on those
   fp32 values (R-12).  zero_mean != 0 additionally applies the row/column
   zero-mean of S:135 (used for query residuals before PCE, R-9).        */
void oracle_zero_mean(double* x, int H, int W);

int oracle_residual(const float* I, int H, int W, double sigma0_sq, const int* windows,
                    int n_windows, int levels, int zero_mean, double* Wres) {
    long P = (long)H * W;
    double* Id = (double*)malloc(sizeof(double) * P);
    double* F = (double*)malloc(sizeof(double) * P);
    for (long p = 0; p < P; ++p) Id[p] = (double)I[p];
    int st = oracle_denoise(Id, H, W, sigma0_sq, windows, n_windows, levels, F);
    if (st == 0) {
        for (long p = 0; p < P; ++p) Wres[p] = Id[p] - F[p];
        if (zero_mean) oracle_zero_mean(Wres, H, W);
    }
    free(Id);
    free(F);
    return st;
}

/* ------------------------------------------------------------------ */
/* a5: MLE accumulation, Eq. (2) P:151-155 and its SDA form P:200-203: */
/*   K = sum_i W_i I_i / sum_i I_i^2, element-wise, in ascending i     */
/*   (64-bit sums, ascending group order).                  */
/* ------------------------------------------------------------------ */
void oracle_mle_accumulate(const double* Wres, const float* I, long P, double* num, double* den) {
    for (long p = 0; p < P; ++p) {
        double i = (double)I[p];
        num[p] += Wres[p] * i;
        den[p] += i * i;
    }
}

/* "subtract each row's mean from the row, then each column's mean
   from the column; single pass each".                                  */
void oracle_zero_mean(double* x, int H, int W) {
    for (int y = 0; y < H; ++y) {
        double s = 0.0;
        for (int c = 0; c < W; ++c) s += x[(long)y * W + c];
        double mean = s / W;
        for (int c = 0; c < W; ++c) x[(long)y * W + c] -= mean;
    }
    for (int c = 0; c < W; ++c) {
        double s = 0.0;
        for (int y = 0; y < H; ++y) s += x[(long)y * W + c];
        double mean = s / H;
        for (int y = 0; y < H; ++y) x[(long)y * W + c] -= mean;
    }
}

/* a6: "khat = sum_WI / max(sum_I2, eps) element-wise with
   eps = 1e-6; then postprocess_residual applied to khat".              */
void oracle_finalize(const double* num, const double* den, int H, int W, double eps, int zero_mean,
                     double* K) {
    long P = (long)H * W;
    for (long p = 0; p < P; ++p) K[p] = num[p] / (den[p] > eps ? den[p] : eps);
    if (zero_mean) oracle_zero_mean(K, H, W);
}

/* The whole fingerprint path of S:224 (sda(d); d = 1 is conventional):
   plan groups, average, denoise each SDA frame, MLE over the n_s terms in
   ascending order, finalize.  num/den are outputs (zeroed here).        */
int oracle_extract_fingerprint(const uint8_t* frames, long m, int H, int W, long d, double sigma0_sq,
                               const int* windows, int n_windows, int levels, double eps,
                               int zero_mean, double* K, double* num, double* den) {
    long ns = oracle_sda_groups(m, d);
    if (ns < 0) return 3;
    long P = (long)H * W;
    float* S = (float*)malloc(sizeof(float) * P);
    double* Wres = (double*)malloc(sizeof(double) * P);
    memset(num, 0, sizeof(double) * P);
    memset(den, 0, sizeof(double) * P);
    int st = 0;
    for (long i = 0; i < ns && st == 0; ++i) {
        st = oracle_sda_average(frames + i * d * P, d, H, W, d, S);
        if (st) break;
        st = oracle_residual(S, H, W, sigma0_sq, windows, n_windows, levels, 0, Wres);
        if (st) break;
        oracle_mle_accumulate(Wres, S, P, num, den);
    }
    if (st == 0) oracle_finalize(num, den, H, W, eps, zero_mean, K);
    free(S);
    free(Wres);
    return st;
}
