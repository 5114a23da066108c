// wdft.cu — f2: Wiener filtering of a fingerprint in the DFT
// domain ("off by default"; reading R-23 of DESIGN.md).  For each
// zero-mean K [H][W]:
//   F = DFT2(K);  A = |F| / sqrt(HW);  s2 = mean(K^2)  (= mean(A^2), Parseval)
//   m = min_{w in 3,5,7,9} mean_{w x w}(A^2)  (mirror-extended windows, R-7)
//   K' = real(IDFT2( F * s2 / max(m, s2) ))  (the gain's Hermitian part, see k_wdft_apply)
// i.e. the denoiser's local-variance MAP/Wiener noise-domain gain applied to the
// magnitude spectrum with sigma0^2 = s2: flat (noise-like) spectral regions pass,
// peaks (periodic artefacts shared by cameras) are attenuated, phases are kept.
// cuFFT R2C/C2R in fp32 (BASELINE allows cuFFT for PCE; this optional clean-up
// relaxes that rule, as SURVEY §8f anticipates); the box means and the gain are
// the streaming shrink kernel of split.cu on the full-size magnitude plane; the
// energy s2 is a fixed-order fp64 block reduction (deterministic).
#include <cufft.h>

#include "common.cuh"

namespace prnu {

constexpr int WD_BLOCKS = 128;   // a fixed partition (not the SM count) => fixed sum order

struct WdftPlan {
    int H, W, batch;
    cufftHandle r2c, c2r;
    size_t work, ws_bytes;
};

static size_t wd_spec(int H, int W) { return (size_t)H * (W / 2 + 1); }

// partial sums of K^2 per block (fixed grid => fixed order), then s2 = sum / P
__global__ void __launch_bounds__(256) k_wdft_energy(const float* __restrict__ K, long long P, double* part) {
    const float* Kb = K + (size_t)blockIdx.y * P;
    double acc = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P; i += 256LL * gridDim.x) {
        const double v = Kb[i];
        acc = fma(v, v, acc);
    }
    __shared__ double sh[8];
    double t[1] = {acc};
    block_sum(t, sh);
    if (threadIdx.x == 0) part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t[0];
}

__global__ void k_wdft_energy_final(const double* part, int nblk, long long P, float* s2) {
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nblk; ++i) s += part[(size_t)b * nblk + i];
        s2[b] = (float)(s / (double)P);
    }
}

// full magnitude plane A [H][W] from the half spectrum (Hermitian symmetry)
__global__ void __launch_bounds__(256) k_wdft_mag(const cufftComplex* __restrict__ F, int H, int W, float scale,
                                                  float* __restrict__ A) {
    const int b = blockIdx.y;
    const int nf = W / 2 + 1;
    const long long P = (long long)H * W;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P; i += 256LL * gridDim.x) {
        const int u = (int)(i / W), v = (int)(i - (long long)u * W);
        const int uu = v < nf ? u : (H - u) % H, vv = v < nf ? v : W - v;
        const cufftComplex f = F[(size_t)b * H * nf + (size_t)uu * nf + vv];
        A[(size_t)b * P + i] = sqrtf(f.x * f.x + f.y * f.y) * scale;
    }
}

// F *= g / (H W) on the half spectrum, g = the Hermitian part of the gain
// (g(k) + g(-k)) / 2 with g = A_hat / A = s2 / max(m, s2) (0 where A == 0): the
// mirror-extended box means are not symmetric under k -> -k, and real(IDFT2(F g))
// (R-23) equals IDFT2(F (g(k) + g(-k)) / 2), which C2R computes from the half spectrum.
__global__ void __launch_bounds__(256) k_wdft_apply(cufftComplex* __restrict__ F, const float* __restrict__ A,
                                                    const float* __restrict__ Ahat, int H, int W, float inv_n) {
    const int b = blockIdx.y;
    const int nf = W / 2 + 1;
    const long long n = (long long)H * nf;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
        const int u = (int)(i / nf), v = (int)(i - (long long)u * nf);
        const size_t pi = (size_t)b * H * W + (size_t)u * W + v;
        const size_t pj = (size_t)b * H * W + (size_t)((H - u) % H) * W + (W - v) % W;   // -k
        const float a = A[pi];   // |F| is Hermitian-symmetric: A[-k] = A[k]
        const float g = a > 0.f ? 0.5f * (Ahat[pi] + Ahat[pj]) / a : 0.f;
        cufftComplex f = F[(size_t)b * n + i];
        f.x *= g * inv_n;
        f.y *= g * inv_n;
        F[(size_t)b * n + i] = f;
    }
}

int wdft_plan_create(int H, int W, int batch, size_t* ws_bytes, void** out) {
    WdftPlan* p = new WdftPlan{};
    p->H = H;
    p->W = W;
    p->batch = batch;
    int n[2] = {H, W};
    const int nf = W / 2 + 1;
    int inembed_r[2] = {H, W}, onembed_c[2] = {H, nf};
    size_t w1 = 0, w2 = 0;
    cufftResult r;
    if ((r = cufftCreate(&p->r2c)) || (r = cufftCreate(&p->c2r))) {
        delete p;
        return fail(PRNU_CUDA_ERROR, "cufftCreate failed");
    }
    cufftSetAutoAllocation(p->r2c, 0);
    cufftSetAutoAllocation(p->c2r, 0);
    r = cufftMakePlanMany(p->r2c, 2, n, inembed_r, 1, H * W, onembed_c, 1, H * nf, CUFFT_R2C, batch, &w1);
    if (r == CUFFT_SUCCESS)
        r = cufftMakePlanMany(p->c2r, 2, n, onembed_c, 1, H * nf, inembed_r, 1, H * W, CUFFT_C2R, batch, &w2);
    if (r != CUFFT_SUCCESS) {
        cufftDestroy(p->r2c);
        cufftDestroy(p->c2r);
        delete p;
        return fail(PRNU_CUDA_ERROR, "cufftMakePlanMany failed");
    }
    p->work = std::max(w1, w2);
    const size_t P = (size_t)H * W;
    p->ws_bytes = align_up(p->work, 256) + align_up(sizeof(cufftComplex) * wd_spec(H, W) * batch, 256) +
                  2 * align_up(sizeof(float) * P * batch, 256) +
                  align_up(sizeof(double) * WD_BLOCKS * batch, 256) + align_up(sizeof(float) * batch, 256);
    *ws_bytes = p->ws_bytes;
    *out = p;
    return PRNU_OK;
}

int wdft_plan_destroy(void* plan) {
    WdftPlan* p = reinterpret_cast<WdftPlan*>(plan);
    if (!p) return PRNU_OK;
    cufftDestroy(p->r2c);
    cufftDestroy(p->c2r);
    delete p;
    return PRNU_OK;
}

int wdft_plan_dims(void* plan, int* H, int* W, int* batch, size_t* ws_bytes) {
    WdftPlan* p = reinterpret_cast<WdftPlan*>(plan);
    *H = p->H;
    *W = p->W;
    *batch = p->batch;
    *ws_bytes = p->ws_bytes;
    return PRNU_OK;
}

int run_wdft(void* plan, const float* K, float* K_out, void* ws, cudaStream_t st) {
    WdftPlan* p = reinterpret_cast<WdftPlan*>(plan);
    const int H = p->H, W = p->W, B = p->batch;
    const long long P = (long long)H * W;
    char* c = reinterpret_cast<char*>(ws);
    void* work = c;
    c += align_up(p->work, 256);
    cufftComplex* F = reinterpret_cast<cufftComplex*>(c);
    c += align_up(sizeof(cufftComplex) * wd_spec(H, W) * B, 256);
    float* A = reinterpret_cast<float*>(c);
    c += align_up(sizeof(float) * P * B, 256);
    float* Ahat = reinterpret_cast<float*>(c);
    c += align_up(sizeof(float) * P * B, 256);
    double* part = reinterpret_cast<double*>(c);
    c += align_up(sizeof(double) * WD_BLOCKS * B, 256);
    float* s2 = reinterpret_cast<float*>(c);

    int rc;
    {
        KTimer kt("wdft_energy", st);
        k_wdft_energy<<<dim3(WD_BLOCKS, B), 256, 0, st>>>(K, P, part);
        k_wdft_energy_final<<<B, 32, 0, st>>>(part, WD_BLOCKS, P, s2);
    }
    count_launch(2);
    if ((rc = check_launch("k_wdft_energy"))) return rc;
    cufftResult r;
    if ((r = cufftSetStream(p->r2c, st)) || (r = cufftSetStream(p->c2r, st)) || (r = cufftSetWorkArea(p->r2c, work)) ||
        (r = cufftSetWorkArea(p->c2r, work)))
        return fail(PRNU_CUDA_ERROR, "cufft setup failed");
    if ((r = cufftExecR2C(p->r2c, const_cast<float*>(K), F))) return fail(PRNU_CUDA_ERROR, "cufftExecR2C failed");
    const unsigned blocks = (unsigned)std::min<long long>((P + 255) / 256, 8LL * device_sm_count());
    {
        KTimer kt("wdft_mag", st);
        k_wdft_mag<<<dim3(blocks, B), 256, 0, st>>>(F, H, W, (float)(1.0 / sqrt((double)P)), A);
    }
    count_launch();
    if ((rc = check_launch("k_wdft_mag"))) return rc;
    {
        // local-variance Wiener gain on the magnitude plane: A_hat = A s2 / max(m, s2)
        ShrinkParams sp{1.0f, 15};
        const float* src[3] = {A, A, A};
        float* dst[3] = {Ahat, Ahat, Ahat};
        KTimer kt("wdft_shrink", st);
        if ((rc = launch_shrink_strip(src, dst, P, W, H, W, sp, B, st, 1, s2))) return rc;
    }
    count_launch();
    if ((rc = check_launch("k_shrink (wdft)"))) return rc;
    {
        KTimer kt("wdft_apply", st);
        k_wdft_apply<<<dim3(blocks, B), 256, 0, st>>>(F, A, Ahat, H, W, (float)(1.0 / (double)P));
    }
    count_launch();
    if ((rc = check_launch("k_wdft_apply"))) return rc;
    if ((r = cufftExecC2R(p->c2r, F, K_out))) return fail(PRNU_CUDA_ERROR, "cufftExecC2R failed");
    return PRNU_OK;
}

}  // namespace prnu
