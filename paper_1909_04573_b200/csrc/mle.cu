// mle.cu — a5 MLE accumulation, a6 finalize + zero-mean, a7 NCC (sm_100a).
//
// Every reduction has a fixed shape (grid size, per-thread stride, tree) that
// depends only on the problem size, so results are bit-reproducible run to run
// and independent of batching.  fp64 throughout the sums.
#include "common.cuh"

namespace prnu {

// ---------------------------------------------------------------- a5
// sum_WI[p] += W_b[p] I_b[p]; sum_I2[p] += I_b[p]^2, b ascending (Eq. 2).
__global__ void __launch_bounds__(256) k_accumulate(const float* __restrict__ Wr, const float* __restrict__ I,
                                                     int batch, long long P, double* __restrict__ num,
                                                     double* __restrict__ den) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P;
         p += (long long)gridDim.x * blockDim.x) {
        double n = num[p], d = den[p];
        for (int b = 0; b < batch; ++b) {
            double w = (double)Wr[(size_t)b * P + p];
            double i = (double)I[(size_t)b * P + p];
            n += w * i;
            d += i * i;
        }
        num[p] = n;
        den[p] = d;
    }
}

int launch_accumulate(const float* W, const float* I, int batch, long long P, double* num, double* den,
                      cudaStream_t st) {
    long long blocks = std::min<long long>((P + 255) / 256, 16LL * device_sm_count());
    {
        KTimer kt("accumulate", st);
        k_accumulate<<<(unsigned)blocks, 256, 0, st>>>(W, I, batch, P, num, den);
    }
    count_launch();
    return check_launch("k_accumulate");
}

// ---------------------------------------------------------------- a6
struct FinalizeSrc {   // K = sum_WI / max(sum_I2, eps); one plane
    const double* num;
    const double* den;
    double eps;
    __device__ __forceinline__ double operator()(int, size_t i) const {
        double d = den[i];
        return num[i] / (d > eps ? d : eps);
    }
};
struct FloatSrc {      // residual planes [b][H][W] to be zero-meaned (in place)
    const float* w;
    long long P;
    __device__ __forceinline__ double operator()(int b, size_t i) const { return (double)w[(size_t)b * P + i]; }
};

// Row / column zero-mean (R-9) of `batch` planes, one launch per step with
// the plane index in the grid.  The source is re-evaluated in every step (the same
// fp64 value each time) instead of being materialised, and every sum keeps a fixed
// order (deterministic, independent of the batch).
// S:135 step 1: each row's mean.
template <class Src>
__global__ void __launch_bounds__(256) k_zm_rows(Src src, int H, int W, double* __restrict__ rowmean) {
    __shared__ double sh[8];
    const int y = blockIdx.x, b = blockIdx.y;
    double s = 0.0;
    for (int x = threadIdx.x; x < W; x += 256) s += src(b, (size_t)y * W + x);
    double t[1] = {s};
    block_sum(t, sh);
    if (threadIdx.x == 0) rowmean[(size_t)b * H + y] = t[0] / W;
}

// S:135 step 2: column means of the row-centred values, in ZM_CHUNKS row chunks
// (so the grid fills the GPU) whose partial sums are then added in chunk order:
// a fixed summation order, independent of launch configuration (deterministic).
constexpr int ZM_CHUNKS = 16;
template <class Src>
__global__ void __launch_bounds__(256) k_zm_cols(Src src, const double* __restrict__ rowmean, int H, int W,
                                                  double* __restrict__ part) {
    __shared__ double sh[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, b = blockIdx.z;
    const int x = blockIdx.x * 32 + tx;
    const int y0 = (int)((long long)H * blockIdx.y / ZM_CHUNKS), y1 = (int)((long long)H * (blockIdx.y + 1) / ZM_CHUNKS);
    const double* rm = rowmean + (size_t)b * H;
    double s = 0.0;
    if (x < W)
        for (int y = y0 + ty; y < y1; y += 8) s += src(b, (size_t)y * W + x) - rm[y];
    sh[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && x < W) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += sh[k][tx];
        part[((size_t)b * ZM_CHUNKS + blockIdx.y) * W + x] = t;
    }
}
__global__ void __launch_bounds__(256) k_zm_cols_final(const double* __restrict__ part, int H, int W,
                                                        double* __restrict__ colmean) {
    const int x = blockIdx.x * 256 + threadIdx.x, b = blockIdx.y;
    if (x >= W) return;
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < ZM_CHUNKS; ++c) t += part[((size_t)b * ZM_CHUNKS + c) * W + x];
    colmean[(size_t)b * W + x] = t / H;
}

template <class Src>
__global__ void __launch_bounds__(256) k_zm_apply(Src src, const double* __restrict__ rowmean,
                                                   const double* __restrict__ colmean, int H, int W,
                                                   float* __restrict__ out) {
    const long long P = (long long)H * W;
    const int b = blockIdx.y;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P;
         i += (long long)gridDim.x * blockDim.x) {
        int y = (int)(i / W), x = (int)(i - (long long)y * W);
        out[(size_t)b * P + i] = (float)((src(b, (size_t)i) - rowmean[(size_t)b * H + y]) - colmean[(size_t)b * W + x]);
    }
}

__global__ void __launch_bounds__(256) k_finalize_plain(FinalizeSrc src, long long P, float* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)src(0, (size_t)i);
}

size_t zm_workspace_bytes(int H, int W, int batch) {
    return align_up(sizeof(double) * (size_t)batch * H, 256) + align_up(sizeof(double) * (size_t)batch * W, 256) +
           align_up(sizeof(double) * (size_t)batch * ZM_CHUNKS * W, 256);
}
size_t zm_workspace_bytes(int H, int W) { return zm_workspace_bytes(H, W, 1); }

template <class Src>
static int run_zero_mean(Src src, int batch, int H, int W, float* out, void* ws, cudaStream_t st) {
    char* p = reinterpret_cast<char*>(ws);
    double* rm = reinterpret_cast<double*>(p);
    p += align_up(sizeof(double) * (size_t)batch * H, 256);
    double* cm = reinterpret_cast<double*>(p);
    p += align_up(sizeof(double) * (size_t)batch * W, 256);
    double* part = reinterpret_cast<double*>(p);
    {
        KTimer kt("zm_rows", st);
        k_zm_rows<Src><<<dim3(H, batch), 256, 0, st>>>(src, H, W, rm);
    }
    {
        KTimer kt("zm_cols", st);
        k_zm_cols<Src><<<dim3((W + 31) / 32, ZM_CHUNKS, batch), 256, 0, st>>>(src, rm, H, W, part);
        k_zm_cols_final<<<dim3((W + 255) / 256, batch), 256, 0, st>>>(part, H, W, cm);
    }
    long long P = (long long)H * W;
    long long blocks = std::max<long long>(1, std::min<long long>((P + 255) / 256, 16LL * device_sm_count() / batch));
    {
        KTimer kt("zm_apply", st);
        k_zm_apply<Src><<<dim3((unsigned)blocks, batch), 256, 0, st>>>(src, rm, cm, H, W, out);
    }
    count_launch(4);
    return check_launch("zero_mean");
}

int launch_finalize(const double* num, const double* den, int H, int W, double eps, int zero_mean, float* K,
                    void* ws, cudaStream_t st) {
    FinalizeSrc src{num, den, eps};
    if (zero_mean) return run_zero_mean(src, 1, H, W, K, ws, st);
    long long P = (long long)H * W;
    long long blocks = std::min<long long>((P + 255) / 256, 16LL * device_sm_count());
    {
        KTimer kt("finalize_plain", st);
        k_finalize_plain<<<(unsigned)blocks, 256, 0, st>>>(src, P, K);
    }
    count_launch();
    return check_launch("k_finalize_plain");
}

// in place over batch planes [b][H][W]; ws: zm_workspace_bytes(H, W, batch)
int launch_zero_mean_f32(float* Wp, int batch, int H, int W, void* ws, cudaStream_t st) {
    if (batch > 65535) return fail(PRNU_INVALID_ARG, "zero mean: batch too large");
    return run_zero_mean(FloatSrc{Wp, (long long)H * W}, batch, H, W, Wp, ws, st);
}

// ---------------------------------------------------------------- a7 NCC
constexpr int NCC_BLOCKS = 256;   // a fixed partition (not the SM count): the same sum order on every device

size_t ncc_workspace_bytes(int batch) {
    return align_up(sizeof(double) * (size_t)batch * NCC_BLOCKS * 2, 256) +
           align_up(sizeof(double) * (size_t)batch * NCC_BLOCKS * 3, 256);
}

__global__ void __launch_bounds__(256) k_ncc_pass1(const float* __restrict__ a, const float* __restrict__ b,
                                                    long long P, double* __restrict__ part) {
    __shared__ double sh[16];
    const int pb = blockIdx.y;
    const float* A = a + (size_t)pb * P;
    const float* B = b + (size_t)pb * P;
    double sa = 0.0, sb = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P; i += 256LL * NCC_BLOCKS) {
        sa += (double)A[i];
        sb += (double)B[i];
    }
    double t[2] = {sa, sb};
    block_sum(t, sh);
    if (threadIdx.x == 0) {
        part[((size_t)pb * NCC_BLOCKS + blockIdx.x) * 2 + 0] = t[0];
        part[((size_t)pb * NCC_BLOCKS + blockIdx.x) * 2 + 1] = t[1];
    }
}

__device__ __forceinline__ void ncc_means(const double* part1, int pb, long long P, double* ma, double* mb,
                                          double* sh) {
    double sa = 0.0, sb = 0.0;
    for (int k = threadIdx.x; k < NCC_BLOCKS; k += 256) {
        sa += part1[((size_t)pb * NCC_BLOCKS + k) * 2 + 0];
        sb += part1[((size_t)pb * NCC_BLOCKS + k) * 2 + 1];
    }
    double t[2] = {sa, sb};
    block_sum(t, sh);
    *ma = t[0] / (double)P;
    *mb = t[1] / (double)P;
}

__global__ void __launch_bounds__(256) k_ncc_pass2(const float* __restrict__ a, const float* __restrict__ b,
                                                    long long P, const double* __restrict__ part1,
                                                    double* __restrict__ part2) {
    __shared__ double sh[24];
    const int pb = blockIdx.y;
    double ma, mb;
    ncc_means(part1, pb, P, &ma, &mb, sh);
    const float* A = a + (size_t)pb * P;
    const float* B = b + (size_t)pb * P;
    double sab = 0.0, saa = 0.0, sbb = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < P; i += 256LL * NCC_BLOCKS) {
        double da = (double)A[i] - ma, db = (double)B[i] - mb;
        sab += da * db;
        saa += da * da;
        sbb += db * db;
    }
    double t[3] = {sab, saa, sbb};
    block_sum(t, sh);
    if (threadIdx.x == 0) {
        double* o = part2 + ((size_t)pb * NCC_BLOCKS + blockIdx.x) * 3;
        o[0] = t[0];
        o[1] = t[1];
        o[2] = t[2];
    }
}

__global__ void __launch_bounds__(256) k_ncc_final(const double* __restrict__ part2, double* __restrict__ out) {
    __shared__ double sh[24];
    const int pb = blockIdx.x;
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < NCC_BLOCKS; k += 256)
        for (int j = 0; j < 3; ++j) s[j] += part2[((size_t)pb * NCC_BLOCKS + k) * 3 + j];
    block_sum(s, sh);
    if (threadIdx.x == 0) out[pb] = s[0] / sqrt(s[1] * s[2]);   // NaN for a constant input
}

int launch_ncc(const float* a, const float* b, int batch, long long P, double* out, void* ws, cudaStream_t st) {
    char* p = reinterpret_cast<char*>(ws);
    double* part1 = reinterpret_cast<double*>(p);
    p += align_up(sizeof(double) * (size_t)batch * NCC_BLOCKS * 2, 256);
    double* part2 = reinterpret_cast<double*>(p);
    dim3 grid(NCC_BLOCKS, batch);
    {
        KTimer kt("ncc_pass1", st);
        k_ncc_pass1<<<grid, 256, 0, st>>>(a, b, P, part1);
    }
    {
        KTimer kt("ncc_pass2", st);
        k_ncc_pass2<<<grid, 256, 0, st>>>(a, b, P, part1, part2);
    }
    {
        KTimer kt("ncc_final", st);
        k_ncc_final<<<batch, 256, 0, st>>>(part2, out);
    }
    count_launch(3);
    return check_launch("ncc");
}

// ---------------------------------------------------------------- result checks
// Flags the data-dependent error kinds (prnu_check_results): bit 0 = some NaN, bit 1 = some
// zero, bit 2 = some non-zero.  An idempotent OR into one word (the result does not
// depend on the order of the atomics).
__global__ void k_check_results(const double* __restrict__ v, long long n, unsigned* __restrict__ flags) {
    unsigned f = 0u;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double x = v[i];
        if (isnan(x)) f |= 1u;
        if (x == 0.0) f |= 2u;
        if (x != 0.0) f |= 4u;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

int check_results(int kind, const double* v, long long n, cudaStream_t st) {
    unsigned* flags = nullptr;
    unsigned h = 0u;
    if (cudaMallocAsync(&flags, sizeof(unsigned), st) != cudaSuccess) return fail(PRNU_CUDA_ERROR, "cudaMallocAsync");
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(unsigned), st);
    if (e == cudaSuccess) {
        const long long blocks = std::min<long long>((n + 255) / 256, 4LL * device_sm_count());
        k_check_results<<<(unsigned)std::max<long long>(blocks, 1), 256, 0, st>>>(v, n, flags);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(flags, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(PRNU_CUDA_ERROR, std::string("check_results: ") + cudaGetErrorString(e));
    if (kind == 0 && (h & 1u)) return fail(PRNU_CONSTANT_INPUT, "NCC of an operand with zero variance (NaN)");
    if (kind == 1 && (h & 2u)) return fail(PRNU_DEGENERATE_SURFACE, "PCE of a surface with all values equal (peak 0)");
    if (kind == 2 && !(h & 4u)) return fail(PRNU_EMPTY_ACCUMULATOR, "sum_I2 is zero everywhere: no frame accumulated");
    return PRNU_OK;
}

}  // namespace prnu
