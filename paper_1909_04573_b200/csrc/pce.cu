// pce.cu — a8: PCE of residual/template pairs.
//
// C = IFFT2( FFT2(R) . conj(FFT2(T)) ) with the DC bin zeroed (= correlation of
// the mean-removed inputs), cuFFT R2C/C2R in fp32 (BASELINE: cuFFT only here).
// Peak search and energies are deterministic block reductions in fp64.
#include <cufft.h>

#include "common.cuh"
#include "pce.cuh"

namespace prnu {

constexpr int PCE_BLOCKS = 128;   // partial blocks per pair: a fixed partition (not the SM count) => fixed sum order
constexpr double PCE_CAP = 1e12;

// Three paths.  `cols` (H has a radix plan in pcefft.cu, W even): the rows as 1-D
// transforms of the packed real planes + the fused column kernel, the rows either
// by pcefft.cu's row kernel (`rows`: W/2 has a radix plan; the template product
// and the peak/energy partials fused in) or by cuFFT 1-D C2C; otherwise cuFFT
// 2-D R2C/C2R.
struct PcePlan {
    int H, W, batch;
    bool cols, rows;
    cufftHandle r2c, c2r, c2c;
    size_t work;       // bytes of cuFFT work area
    size_t ws_bytes;   // total workspace prnu_pce needs
};

static size_t spectrum_elems(int H, int W) { return (size_t)H * (W / 2 + 1); }
bool pce_cols_supported(int H);
bool pce_rows_supported(int W);
int pce_rows_nparts(int H);
int launch_pce_rows(int mode, const float* X, const float* K, int k_batch, const uint8_t* Iq, const void* Zin,
                    void* Zout, float* C, void* part, int H, int W, int batch, cudaStream_t st);
int launch_pce_cols(int mode, const void* Z, const void* Rs, void* out, int H, int W, int batch, cudaStream_t st);

// ---------------------------------------------------------------- template
__global__ void __launch_bounds__(256) k_pce_template(const float* __restrict__ K, int k_batch,
                                                       const uint8_t* __restrict__ Iq, long long P,
                                                       float* __restrict__ T) {
    const int b = blockIdx.y;
    const float* Kb = K + (size_t)(k_batch == 1 ? 0 : b) * P;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P; i += 256LL * gridDim.x)
        T[(size_t)b * P + i] = Kb[i] * (float)Iq[(size_t)b * P + i];
}
// 4 pixels per thread (P % 4 == 0, 16-byte aligned K / T, 4-byte aligned Iq): one
// 16-byte K load, one 4-byte Iq load and one 16-byte streaming T store per thread
__global__ void __launch_bounds__(256) k_pce_template4(const float4* __restrict__ K, int k_batch,
                                                        const uchar4* __restrict__ Iq, long long P4,
                                                        float4* __restrict__ T) {
    const int b = blockIdx.y;
    const float4* Kb = K + (size_t)(k_batch == 1 ? 0 : b) * P4;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P4; i += 256LL * gridDim.x) {
        const float4 k = Kb[i];
        const uchar4 q = Iq[(size_t)b * P4 + i];
        __stcs(T + (size_t)b * P4 + i, make_float4(k.x * (float)q.x, k.y * (float)q.y, k.z * (float)q.z, k.w * (float)q.w));
    }
}

int launch_pce_template(const float* K, int k_batch, const uint8_t* Iq, int batch, long long P, float* T,
                        cudaStream_t st) {
    const bool vec = P % 4 == 0 && reinterpret_cast<uintptr_t>(K) % 16 == 0 && reinterpret_cast<uintptr_t>(T) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(Iq) % 4 == 0;
    const long long n = vec ? P / 4 : P;
    unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 8LL * device_sm_count());
    {
        KTimer kt("pce_template", st);
        if (vec)
            k_pce_template4<<<dim3(blocks, batch), 256, 0, st>>>(reinterpret_cast<const float4*>(K), k_batch,
                                                                 reinterpret_cast<const uchar4*>(Iq), n,
                                                                 reinterpret_cast<float4*>(T));
        else
            k_pce_template<<<dim3(blocks, batch), 256, 0, st>>>(K, k_batch, Iq, P, T);
    }
    count_launch();
    return check_launch("k_pce_template");
}

// ---------------------------------------------------------------- spectra
// T <- R conj(T), in T's storage: the residual spectrum R survives, so one FFT(R)
// serves every template batch matched against the same residuals (camera ID).
__global__ void __launch_bounds__(256) k_conj_mul(const cufftComplex* __restrict__ R, cufftComplex* __restrict__ T,
                                                   long long n_per, int batch) {
    long long n = n_per * batch;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
        cufftComplex r = R[i], t = T[i];
        cufftComplex o;
        o.x = r.x * t.x + r.y * t.y;       // r * conj(t)
        o.y = r.y * t.x - r.x * t.y;
        if (i % n_per == 0) o.x = o.y = 0.f;   // DC bin: mean removal of both inputs
        T[i] = o;
    }
}

// ---------------------------------------------------------------- reductions
// Warp-shuffle reduction of (|C| peak, index, energy): the xor butterfly picks the
// same winner on both lanes of every exchange (better() is a total order on the
// candidates; NaN never becomes one, k_pce_partial skips it), then
// every thread folds the 8 warp results in warp order.  Fixed shape, deterministic.
__device__ void block_reduce_peak(float& a, int& idx, double& e) {
    __shared__ float sa[8];
    __shared__ int si[8];
    __shared__ double se[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float a2 = __shfl_xor_sync(0xffffffffu, a, o);
        int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
        if (better(a2, i2, a, idx)) {
            a = a2;
            idx = i2;
        }
    }
    e = warp_sum(e);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sa[w] = a;
        si[w] = idx;
        se[w] = e;
    }
    __syncthreads();
    a = sa[0];
    idx = si[0];
    e = se[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        if (better(sa[k], si[k], a, idx)) {
            a = sa[k];
            idx = si[k];
        }
        e += se[k];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_pce_partial(const float* __restrict__ C, long long P, PeakE* __restrict__ part) {
    const int b = blockIdx.y;
    const float* Cb = C + (size_t)b * P;
    float best = -1.f;
    int bi = -1;
    double e = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P; i += 256LL * PCE_BLOCKS) {
        float c = Cb[i];
        float a = fabsf(c);
        if (a > best) {   // strict: keeps the first (smallest) index of this thread's sequence
            best = a;
            bi = (int)i;
        }
        e += (double)c * (double)c;
    }
    block_reduce_peak(best, bi, e);
    if (threadIdx.x == 0) part[(size_t)b * PCE_BLOCKS + blockIdx.x] = PeakE{best, bi, e};
}

__global__ void __launch_bounds__(256) k_pce_final(const float* __restrict__ C, const PeakE* __restrict__ part,
                                                    int nparts, int H, int W, int excl, int aligned, double scale,
                                                    double* __restrict__ pce, int* __restrict__ py,
                                                    int* __restrict__ px, double* __restrict__ peak) {
    const int b = blockIdx.x;
    const long long P = (long long)H * W;
    const float* Cb = C + (size_t)b * P;
    float best = -1.f;
    int bi = -1;
    double e = 0.0;
    for (int k = threadIdx.x; k < nparts; k += 256) {
        PeakE q = part[(size_t)b * nparts + k];
        if (better(q.a, q.idx, best, bi)) {
            best = q.a;
            bi = q.idx;
        }
        e += q.e;
    }
    block_reduce_peak(best, bi, e);
    int p = aligned ? 0 : max(bi, 0);   // bi < 0 only for an all-NaN surface: report position 0
    int y = p / W, x = p - (p / W) * W;
    // circular (2e+1)^2 neighbourhood, distinct positions only (first min(H,2e+1) rows/cols)
    const int nr = min(H, 2 * excl + 1), nc = min(W, 2 * excl + 1);
    double en = 0.0;
    for (int k = threadIdx.x; k < nr * nc; k += 256) {
        int r = k / nc, c = k - r * nc;
        int yy = ((y - excl + r) % H + H) % H;
        int xx = ((x - excl + c) % W + W) % W;
        double v = (double)Cb[(size_t)yy * W + xx];
        en += v * v;
    }
    __shared__ double sh[8];
    double ent[1] = {en};
    block_sum(ent, sh);
    if (threadIdx.x == 0) {
        double v = (double)Cb[p];
        double n_out = (double)(P - (long long)nr * nc);
        double r;
        double bg = n_out > 0 ? (e - ent[0]) / n_out : 0.0;
        if (!(n_out > 0) || !(bg > 0.0)) r = (v >= 0.0) ? PCE_CAP : -PCE_CAP;
        else r = (v >= 0.0 ? 1.0 : -1.0) * v * v / bg;   // scale-invariant ratio
        pce[b] = r;
        py[b] = y;
        px[b] = x;
        peak[b] = v * scale;
    }
}

// ---------------------------------------------------------------- host
static const char* cufft_str(cufftResult r) {
    switch (r) {
        case CUFFT_SUCCESS: return "CUFFT_SUCCESS";
        case CUFFT_INVALID_PLAN: return "CUFFT_INVALID_PLAN";
        case CUFFT_ALLOC_FAILED: return "CUFFT_ALLOC_FAILED";
        case CUFFT_INVALID_VALUE: return "CUFFT_INVALID_VALUE";
        case CUFFT_INTERNAL_ERROR: return "CUFFT_INTERNAL_ERROR";
        case CUFFT_EXEC_FAILED: return "CUFFT_EXEC_FAILED";
        case CUFFT_SETUP_FAILED: return "CUFFT_SETUP_FAILED";
        case CUFFT_INVALID_SIZE: return "CUFFT_INVALID_SIZE";
        default: return "cufft error";
    }
}

int pce_plan_create(int H, int W, int batch, size_t* ws_bytes, void** out) {
    PcePlan* p = new PcePlan{};
    p->H = H;
    p->W = W;
    p->batch = batch;
    p->cols = W % 2 == 0 && pce_cols_supported(H);
    p->rows = p->cols && pce_rows_supported(W);
    size_t w1 = 0, w2 = 0;
    cufftResult r;
    if (p->rows) {
        // no cuFFT plan
    } else if (p->cols) {
        if ((r = cufftCreate(&p->c2c))) {
            delete p;
            return fail(PRNU_CUDA_ERROR, std::string("cufftCreate: ") + cufft_str(r));
        }
        cufftSetAutoAllocation(p->c2c, 0);
        long long m[1] = {W / 2};
        r = cufftMakePlanMany64(p->c2c, 1, m, m, 1, W / 2, m, 1, W / 2, CUFFT_C2C, (long long)H * batch, &w1);
        if (r != CUFFT_SUCCESS) {
            cufftDestroy(p->c2c);
            delete p;
            return fail(PRNU_CUDA_ERROR, std::string("cufftMakePlanMany64: ") + cufft_str(r));
        }
    } else {
        int n[2] = {H, W};
        if ((r = cufftCreate(&p->r2c)) || (r = cufftCreate(&p->c2r))) {
            delete p;
            return fail(PRNU_CUDA_ERROR, std::string("cufftCreate: ") + cufft_str(r));
        }
        cufftSetAutoAllocation(p->r2c, 0);
        cufftSetAutoAllocation(p->c2r, 0);
        int nf = W / 2 + 1;
        int inembed_r[2] = {H, W}, onembed_c[2] = {H, nf};
        r = cufftMakePlanMany(p->r2c, 2, n, inembed_r, 1, H * W, onembed_c, 1, H * nf, CUFFT_R2C, batch, &w1);
        if (r == CUFFT_SUCCESS)
            r = cufftMakePlanMany(p->c2r, 2, n, onembed_c, 1, H * nf, inembed_r, 1, H * W, CUFFT_C2R, batch, &w2);
        if (r != CUFFT_SUCCESS) {
            cufftDestroy(p->r2c);
            cufftDestroy(p->c2r);
            delete p;
            return fail(PRNU_CUDA_ERROR, std::string("cufftMakePlanMany: ") + cufft_str(r));
        }
    }
    p->work = std::max(w1, w2);
    size_t spec = sizeof(cufftComplex) * spectrum_elems(H, W) * batch;
    p->ws_bytes = align_up(p->work, 256) + 2 * align_up(spec, 256) +
                  align_up(sizeof(float) * (size_t)H * W * batch, 256) +
                  align_up(sizeof(PeakE) * (size_t)std::max(PCE_BLOCKS, pce_rows_nparts(H)) * batch, 256);
    *ws_bytes = p->ws_bytes;
    *out = p;
    return PRNU_OK;
}

int pce_plan_destroy(void* plan) {
    PcePlan* p = reinterpret_cast<PcePlan*>(plan);
    if (!p) return PRNU_OK;
    if (p->rows) {
    } else if (p->cols) {
        cufftDestroy(p->c2c);
    } else {
        cufftDestroy(p->r2c);
        cufftDestroy(p->c2r);
    }
    delete p;
    return PRNU_OK;
}

int pce_plan_dims(void* plan, int* H, int* W, int* batch, size_t* ws_bytes) {
    PcePlan* p = reinterpret_cast<PcePlan*>(plan);
    *H = p->H;
    *W = p->W;
    *batch = p->batch;
    *ws_bytes = p->ws_bytes;
    return PRNU_OK;
}

// T == nullptr && K != nullptr: the template K[b or 0] (.) (float)Iq[b] (prnu_pce_template)
// formed inside the row transform (or by prnu_pce_template into Cs on the cuFFT paths).
int run_pce(void* plan, const float* R, const float* T, const float* K, int k_batch, const uint8_t* Iq, int excl,
            int aligned, double* pce, int* py, int* px, double* peak, void* ws, cudaStream_t st) {
    PcePlan* p = reinterpret_cast<PcePlan*>(plan);
    const int H = p->H, W = p->W, batch = p->batch;
    char* c = reinterpret_cast<char*>(ws);
    void* work = c;
    c += align_up(p->work, 256);
    size_t spec = sizeof(cufftComplex) * spectrum_elems(H, W) * batch;
    cufftComplex* Rf = reinterpret_cast<cufftComplex*>(c);
    c += align_up(spec, 256);
    cufftComplex* Tf = reinterpret_cast<cufftComplex*>(c);
    c += align_up(spec, 256);
    float* Cs = reinterpret_cast<float*>(c);
    c += align_up(sizeof(float) * (size_t)H * W * batch, 256);
    PeakE* part = reinterpret_cast<PeakE*>(c);

    cufftResult r;
    const long long P = (long long)H * W;
    const size_t plane_bytes = sizeof(float) * (size_t)P * batch;
    int nparts = PCE_BLOCKS;
    auto mis = [](const void* x, uintptr_t a) { return reinterpret_cast<uintptr_t>(x) % a != 0; };
    if (R && K) return fail(PRNU_INVALID_ARG, "run_pce: template mode needs the cached residual spectrum");
    if (!T && K && (!p->rows || mis(K, 8) || mis(Iq, 2))) {   // template into Cs, then as an explicit T
        if (int rc = launch_pce_template(K, k_batch, Iq, batch, P, Cs, st)) return rc;
        T = Cs;
    }
    if (p->rows) {
        auto fwd_real = [&](const float* X, cufftComplex* dst) -> int {
            if (mis(X, 8)) {
                cudaMemcpyAsync(Cs, X, plane_bytes, cudaMemcpyDeviceToDevice, st);
                X = Cs;
            }
            return launch_pce_rows(0, X, nullptr, 0, nullptr, nullptr, dst, nullptr, nullptr, H, W, batch, st);
        };
        if (R) {
            if (int rc = fwd_real(R, Rf)) return rc;
            if (int rc = launch_pce_cols(0, Rf, nullptr, Rf, H, W, batch, st)) return rc;
        }
        if (!T && !K) return PRNU_OK;
        if (T) {
            if (int rc = fwd_real(T, Tf)) return rc;
        } else if (int rc = launch_pce_rows(1, nullptr, K, k_batch, Iq, nullptr, Tf, nullptr, nullptr, H, W, batch, st)) {
            return rc;
        }
        if (int rc = launch_pce_cols(1, Tf, Rf, Tf, H, W, batch, st)) return rc;
        if (int rc = launch_pce_rows(2, nullptr, nullptr, 0, nullptr, Tf, nullptr, Cs, part, H, W, batch, st)) return rc;
        nparts = pce_rows_nparts(H);
    } else if (p->cols) {
        // rows: the real planes as packed complex rows (8-byte aligned views; a
        // misaligned input is staged through Cs first)
        if ((r = cufftSetStream(p->c2c, st)) || (r = cufftSetWorkArea(p->c2c, work)))
            return fail(PRNU_CUDA_ERROR, std::string("cufft setup: ") + cufft_str(r));
        auto rows = [&](const float* X, cufftComplex* dst) -> int {
            if (reinterpret_cast<uintptr_t>(X) % 8) {
                cudaMemcpyAsync(Cs, X, plane_bytes, cudaMemcpyDeviceToDevice, st);
                X = Cs;
            }
            cufftComplex* src = reinterpret_cast<cufftComplex*>(const_cast<float*>(X));
            if ((r = cufftExecC2C(p->c2c, src, dst, CUFFT_FORWARD)))
                return fail(PRNU_CUDA_ERROR, std::string("cufftExecC2C: ") + cufft_str(r));
            return PRNU_OK;
        };
        if (R) {
            if (int rc = rows(R, Rf)) return rc;
            if (int rc = launch_pce_cols(0, Rf, nullptr, Rf, H, W, batch, st)) return rc;
        }
        if (!T) return PRNU_OK;
        if (int rc = rows(T, Tf)) return rc;
        if (int rc = launch_pce_cols(1, Tf, Rf, Tf, H, W, batch, st)) return rc;
        if ((r = cufftExecC2C(p->c2c, Tf, reinterpret_cast<cufftComplex*>(Cs), CUFFT_INVERSE)))
            return fail(PRNU_CUDA_ERROR, std::string("cufftExecC2C: ") + cufft_str(r));
    } else {
        if ((r = cufftSetStream(p->r2c, st)) || (r = cufftSetStream(p->c2r, st)) ||
            (r = cufftSetWorkArea(p->r2c, work)) || (r = cufftSetWorkArea(p->c2r, work)))
            return fail(PRNU_CUDA_ERROR, std::string("cufft setup: ") + cufft_str(r));
        // R == nullptr: reuse the residual spectrum an earlier call left in this workspace
        if (R && (r = cufftExecR2C(p->r2c, const_cast<float*>(R), Rf)))
            return fail(PRNU_CUDA_ERROR, std::string("cufftExecR2C: ") + cufft_str(r));
        if (!T) return PRNU_OK;   // spectrum only
        if ((r = cufftExecR2C(p->r2c, const_cast<float*>(T), Tf)))
            return fail(PRNU_CUDA_ERROR, std::string("cufftExecR2C: ") + cufft_str(r));
        long long n_per = (long long)spectrum_elems(H, W);
        unsigned blocks = (unsigned)std::min<long long>((n_per * batch + 255) / 256, 8LL * device_sm_count());
        {
            KTimer kt("pce_conj_mul", st);
            k_conj_mul<<<blocks, 256, 0, st>>>(Rf, Tf, n_per, batch);
        }
        count_launch();
        if (int rc = check_launch("k_conj_mul")) return rc;
        if ((r = cufftExecC2R(p->c2r, Tf, Cs)))
            return fail(PRNU_CUDA_ERROR, std::string("cufftExecC2R: ") + cufft_str(r));
    }
    if (!p->rows) {
        {
            KTimer kt("pce_partial", st);
            k_pce_partial<<<dim3(PCE_BLOCKS, batch), 256, 0, st>>>(Cs, P, part);
        }
        count_launch();
    }
    {
        KTimer kt("pce_final", st);
        k_pce_final<<<batch, 256, 0, st>>>(Cs, part, nparts, H, W, excl, aligned, 1.0 / (double)P, pce, py, px, peak);
    }
    count_launch();
    return check_launch("pce reductions");
}

// ---------------------------------------------------------------- f1: block-wise matching
// P:266 ("divided each full resolution fingerprint into 500x500 disjoint
// blocks"); S:275-278 (BlockGrid: disjoint tiles, edge tiles kept),
// S:311-314 (one aligned correlation per tile, no shift search).  Tiles fall in
// at most four size classes (full/last row x full/last column); each class is
// gathered into a contiguous batch and runs the PCE pipeline with the peak
// fixed at (0,0) of the tile's own surface, plus the aligned NCC of the tile.
struct BlockClass {
    int h, w, ty0, tx0, nty, ntx, count;
    void* plan;          // PcePlan for [count][h][w]
    size_t pce_ws;
};

struct BlockPlan {
    int H, W, block, n_ty, n_tx, n_tiles, n_classes;
    BlockClass cls[4];
    size_t gather_bytes;   // largest class: R and T batches
    size_t pce_ws;         // largest class PCE workspace
    size_t ws_bytes;
};

size_t ncc_workspace_bytes(int batch);
int launch_ncc(const float* a, const float* b, int batch, long long P, double* out, void* ws, cudaStream_t st);

__global__ void __launch_bounds__(256) k_gather_tiles(const float* __restrict__ src, int W, int block, int ty0,
                                                       int tx0, int ntx, int h, int w, float* __restrict__ dst) {
    const int i = blockIdx.y;
    const int ty = ty0 + i / ntx, tx = tx0 + i % ntx;
    const float* s0 = src + (size_t)ty * block * W + (size_t)tx * block;
    float* d0 = dst + (size_t)i * h * w;
    for (int e = blockIdx.x * 256 + threadIdx.x; e < h * w; e += 256 * gridDim.x) {
        const int y = e / w, x = e - y * w;
        d0[e] = s0[(size_t)y * W + x];
    }
}

__global__ void k_scatter_tiles(const double* __restrict__ pce_c, const double* __restrict__ ncc_c, int count,
                                int ty0, int tx0, int ntx, int n_tx, double* __restrict__ pce_out,
                                double* __restrict__ ncc_out) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const int id = (ty0 + i / ntx) * n_tx + tx0 + i % ntx;
        pce_out[id] = pce_c[i];
        ncc_out[id] = ncc_c[i];
    }
}

int block_plan_create(int H, int W, int block, int* n_tiles, size_t* ws_bytes, void** out) {
    BlockPlan* bp = new BlockPlan{};
    bp->H = H;
    bp->W = W;
    bp->block = block;
    bp->n_ty = (H + block - 1) / block;
    bp->n_tx = (W + block - 1) / block;
    bp->n_tiles = bp->n_ty * bp->n_tx;
    const int fy = H / block, fx = W / block;          // full tiles per column / row
    const int ry = H - fy * block, rx = W - fx * block; // remainders (0: none)
    const int ys[2][3] = {{block, 0, fy}, {ry, fy, ry ? 1 : 0}};   // (h, ty0, nty)
    const int xs[2][3] = {{block, 0, fx}, {rx, fx, rx ? 1 : 0}};
    int rc = PRNU_OK;
    for (int a = 0; a < 2 && rc == PRNU_OK; ++a)
        for (int c = 0; c < 2 && rc == PRNU_OK; ++c) {
            BlockClass k{};
            k.h = ys[a][0];
            k.ty0 = ys[a][1];
            k.nty = ys[a][2];
            k.w = xs[c][0];
            k.tx0 = xs[c][1];
            k.ntx = xs[c][2];
            k.count = k.nty * k.ntx;
            if (k.count == 0 || k.h == 0 || k.w == 0) continue;
            if (k.count > 65535) {   // the per-class launches put tiles on grid.y
                rc = fail(PRNU_BAD_PARAMETER, "block too small: more than 65535 tiles of one size");
                break;
            }
            rc = pce_plan_create(k.h, k.w, k.count, &k.pce_ws, &k.plan);
            if (rc) break;
            bp->cls[bp->n_classes++] = k;
            bp->gather_bytes = std::max(bp->gather_bytes, 2 * align_up(sizeof(float) * k.count * k.h * k.w, 256));
            bp->pce_ws = std::max(bp->pce_ws, k.pce_ws);
        }
    if (rc) {
        for (int i = 0; i < bp->n_classes; ++i) pce_plan_destroy(bp->cls[i].plan);
        delete bp;
        return rc;
    }
    // per-class outputs: pce, peak (fp64), peak_y, peak_x (int32), ncc (fp64)
    const size_t outs = 3 * align_up(sizeof(double) * bp->n_tiles, 256) + 2 * align_up(sizeof(int) * bp->n_tiles, 256);
    bp->ws_bytes = bp->gather_bytes + bp->pce_ws + align_up(ncc_workspace_bytes(bp->n_tiles), 256) + outs;
    *n_tiles = bp->n_tiles;
    *ws_bytes = bp->ws_bytes;
    *out = bp;
    return PRNU_OK;
}

int block_plan_destroy(void* plan) {
    BlockPlan* bp = reinterpret_cast<BlockPlan*>(plan);
    if (!bp) return PRNU_OK;
    for (int i = 0; i < bp->n_classes; ++i) pce_plan_destroy(bp->cls[i].plan);
    delete bp;
    return PRNU_OK;
}

int block_plan_dims(void* plan, int* H, int* W, int* n_tiles, size_t* ws_bytes) {
    BlockPlan* bp = reinterpret_cast<BlockPlan*>(plan);
    *H = bp->H;
    *W = bp->W;
    *n_tiles = bp->n_tiles;
    *ws_bytes = bp->ws_bytes;
    return PRNU_OK;
}

int run_block_match(void* plan, const float* R, const float* T, int excl, double* pce_out, double* ncc_out, void* ws,
                    cudaStream_t st) {
    BlockPlan* bp = reinterpret_cast<BlockPlan*>(plan);
    char* c = reinterpret_cast<char*>(ws);
    float* Rg = reinterpret_cast<float*>(c);
    float* Tg = reinterpret_cast<float*>(c + bp->gather_bytes / 2);
    c += bp->gather_bytes;
    void* pce_ws = c;
    c += bp->pce_ws;
    void* ncc_ws = c;
    c += align_up(ncc_workspace_bytes(bp->n_tiles), 256);
    double* pc = reinterpret_cast<double*>(c);
    c += align_up(sizeof(double) * bp->n_tiles, 256);
    double* pk = reinterpret_cast<double*>(c);
    c += align_up(sizeof(double) * bp->n_tiles, 256);
    double* nc = reinterpret_cast<double*>(c);
    c += align_up(sizeof(double) * bp->n_tiles, 256);
    int* py = reinterpret_cast<int*>(c);
    c += align_up(sizeof(int) * bp->n_tiles, 256);
    int* px = reinterpret_cast<int*>(c);
    int rc;
    for (int i = 0; i < bp->n_classes; ++i) {
        const BlockClass& k = bp->cls[i];
        const long long P = (long long)k.h * k.w;
        dim3 grid((unsigned)std::min<long long>((P + 255) / 256, 64), k.count);
        {
            KTimer kt("block_gather", st);
            k_gather_tiles<<<grid, 256, 0, st>>>(R, bp->W, bp->block, k.ty0, k.tx0, k.ntx, k.h, k.w, Rg);
            k_gather_tiles<<<grid, 256, 0, st>>>(T, bp->W, bp->block, k.ty0, k.tx0, k.ntx, k.h, k.w, Tg);
        }
        count_launch(2);
        if ((rc = check_launch("k_gather_tiles"))) return rc;
        if ((rc = run_pce(k.plan, Rg, Tg, nullptr, 0, nullptr, excl, 1, pc, py, px, pk, pce_ws, st))) return rc;
        if ((rc = launch_ncc(Rg, Tg, k.count, P, nc, ncc_ws, st))) return rc;
        {
            KTimer kt("block_scatter", st);
            k_scatter_tiles<<<1, 256, 0, st>>>(pc, nc, k.count, k.ty0, k.tx0, k.ntx, bp->n_tx, pce_out, ncc_out);
        }
        count_launch();
        if ((rc = check_launch("k_scatter_tiles"))) return rc;
    }
    return PRNU_OK;
}

}  // namespace prnu
