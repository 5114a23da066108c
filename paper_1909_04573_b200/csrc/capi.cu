// capi.cu — the extern "C" boundary of libprnu.so (declared in include/prnu.h).
// Validation happens here, synchronously, before anything is launched; the
// kernels live in sda.cu / wavelet.cu / mle.cu / pce.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace prnu {

// ---------------------------------------------------------------- state
static thread_local std::string t_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }
int fail(int code, const std::string& msg) {
    t_err = msg;
    return code;
}
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PRNU_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    return PRNU_OK;
}

static int current_device(int* dev) {
    cudaError_t e = cudaGetDevice(dev);
    if (e != cudaSuccess) return fail(PRNU_CUDA_ERROR, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    if (*dev < 0 || *dev >= 64) return fail(PRNU_CUDA_ERROR, "device ordinal beyond 63");
    return PRNU_OK;
}

int set_smem_attr(const void* fn, size_t bytes, DeviceFlags& done) {
    int dev = 0, rc = current_device(&dev);
    if (rc) return rc;
    const uint64_t bit = 1ull << dev;
    if (done.bits.load(std::memory_order_acquire) & bit) return PRNU_OK;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return fail(PRNU_CUDA_ERROR, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    done.bits.fetch_or(bit, std::memory_order_acq_rel);
    return PRNU_OK;
}

int device_sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 1;
    cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

// ---------------------------------------------------------------- profiler
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_ev_pool;

static cudaEvent_t pool_event() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

KTimer::KTimer(const char* name, cudaStream_t s) : slot(-1), st(s) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_on) return;
    ProfRec r{name, pool_event(), pool_event()};
    cudaEventRecord(r.a, s);
    slot = (int)g_prof.size();
    g_prof.push_back(r);
}

KTimer::~KTimer() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (slot < (int)g_prof.size()) cudaEventRecord(g_prof[slot].b, st);
}

bool profiling_active() {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    return g_prof_on;
}

int validate_params(const prnu_denoise_params* p, int H, int W, ShrinkParams* sp) {
    if (!p) return fail(PRNU_INVALID_ARG, "params is NULL");
    if (!(p->sigma0_sq > 0.0f) || !(p->sigma0_sq < 3.0e38f)) return fail(PRNU_BAD_PARAMETER, "sigma0_sq must be > 0");
    if (p->levels < 1 || p->levels > kMaxLevels) return fail(PRNU_BAD_PARAMETER, "levels must be in 1..6");
    if (p->n_windows < 1 || p->n_windows > 4) return fail(PRNU_BAD_PARAMETER, "n_windows must be in 1..4");
    int mask = 0;
    for (int i = 0; i < p->n_windows; ++i) {
        int w = p->windows[i];
        if (w != 3 && w != 5 && w != 7 && w != 9)
            return fail(PRNU_BAD_PARAMETER, "windows must be odd sizes from {3,5,7,9}");
        mask |= 1 << ((w - 3) / 2);
    }
    if (H < (1 << p->levels) || W < (1 << p->levels))
        return fail(PRNU_PLANE_TOO_SMALL, "H and W must be >= 2^levels");
    if (sp) {
        sp->sigma0_sq = p->sigma0_sq;
        sp->wmask = mask;
    }
    return PRNU_OK;
}

// kernels / launchers defined in the other translation units
int launch_sda_average(const uint8_t* frames, long long n_groups, long long P, int d, float* out, cudaStream_t st);
int launch_rgb_to_luma(const uint8_t* rgb, long long n, long long P, int layout, int rounding, void* out,
                       cudaStream_t st);
size_t pyramid_floats_per_frame(const Pyramid& p);
template <typename TIn>
int run_residual(const TIn* in, int nb, int H, int W, const Pyramid& p, const ShrinkParams& sp, float* W_out,
                 float* ws_pyr, cudaStream_t st, int in_pitch = 0);
template <typename TIn>
int run_residual_accumulate(const TIn* in, const TIn* I, int nb, int H, int W, const Pyramid& p,
                            const ShrinkParams& sp, const SdaDiv& div, double* num, double* den, float* ws_pyr,
                            cudaStream_t st, cudaEvent_t acc_wait, cudaEvent_t acc_done, long long frame_stride,
                            int in_pitch = 0);
int launch_sda_sum_u16(const uint8_t* frames, long long n_groups, int H, int W, int d, uint16_t* out, int Wp,
                       cudaStream_t st);
int launch_sda_average_pitched(const uint8_t* frames, long long n_groups, int H, int W, int d, float* out, int Wp,
                               cudaStream_t st);
int launch_pad_rows_u8(const uint8_t* src, long long nb, int H, int W, long long src_stride, uint8_t* dst, int Wp,
                       cudaStream_t st);
int launch_accumulate(const float* W, const float* I, int batch, long long P, double* num, double* den,
                      cudaStream_t st);
size_t zm_workspace_bytes(int H, int W);
size_t zm_workspace_bytes(int H, int W, int batch);
int launch_finalize(const double* num, const double* den, int H, int W, double eps, int zero_mean, float* K,
                    void* ws, cudaStream_t st);
int launch_zero_mean_f32(float* Wp, int batch, int H, int W, void* ws, cudaStream_t st);
size_t ncc_workspace_bytes(int batch);
int launch_ncc(const float* a, const float* b, int batch, long long P, double* out, void* ws, cudaStream_t st);
int launch_pce_template(const float* K, int k_batch, const uint8_t* Iq, int batch, long long P, float* T,
                        cudaStream_t st);
int pce_plan_create(int H, int W, int batch, size_t* ws_bytes, void** out);
int wdft_plan_create(int H, int W, int batch, size_t* ws_bytes, void** out);
int wdft_plan_destroy(void* plan);
int wdft_plan_dims(void* plan, int* H, int* W, int* batch, size_t* ws_bytes);
int run_wdft(void* plan, const float* K, float* K_out, void* ws, cudaStream_t st);
int pce_plan_destroy(void* plan);
int pce_plan_dims(void* plan, int* H, int* W, int* batch, size_t* ws_bytes);
int run_pce(void* plan, const float* R, const float* T, const float* K, int k_batch, const uint8_t* Iq, int excl,
            int aligned, double* pce, int* py, int* px,
            double* peak, void* ws, cudaStream_t st);
int block_plan_create(int H, int W, int block, int* n_tiles, size_t* ws_bytes, void** out);
int block_plan_destroy(void* plan);
int block_plan_dims(void* plan, int* H, int* W, int* n_tiles, size_t* ws_bytes);
int run_block_match(void* plan, const float* R, const float* T, int excl, double* pce_out, double* ncc_out, void* ws,
                    cudaStream_t st);
size_t variant_workspace_bytes(int batch, int H, int W, int levels, int taps, int boundary, int transform);
int run_residual_variant(const float* in, int nb, int H, int W, int levels, int taps, int boundary, int transform,
                         const ShrinkParams& sp, float* W_out, float* ws, cudaStream_t st);
int variant_filter(int taps, double* h);

static int validate_variant(const prnu_denoise_variant* v) {
    if (!v) return fail(PRNU_INVALID_ARG, "variant is NULL");
    if (v->taps != 8 && v->taps != 16) return fail(PRNU_BAD_PARAMETER, "variant taps must be 8 or 16");
    if (v->boundary != 0 && v->boundary != 1) return fail(PRNU_BAD_PARAMETER, "variant boundary must be 0 or 1");
    if (v->transform != 0 && v->transform != 1) return fail(PRNU_BAD_PARAMETER, "variant transform must be 0 or 1");
    if (v->transform == 1 && v->boundary != 1)
        return fail(PRNU_BAD_PARAMETER, "the undecimated transform is circular: boundary must be 1");
    return PRNU_OK;
}
static size_t variant_ws(int batch, int H, int W, const prnu_denoise_params* p, const prnu_denoise_variant* v) {
    return variant_workspace_bytes(batch, H, W, p->levels, v->taps, v->boundary, v->transform) +
           zm_workspace_bytes(H, W, batch);
}

static int pad_pitch_u8(int W);
static size_t residual_pad_bytes(int batch, int H, int W) {   // re-pitched u8 planes (unaligned widths)
    return W % 16 ? align_up((size_t)H * pad_pitch_u8(W) * batch, 256) : 0;
}
static size_t residual_ws(int batch, int H, int W, const Pyramid& pyr) {
    return align_up(sizeof(float) * pyramid_floats_per_frame(pyr) * (size_t)batch, 256) +
           zm_workspace_bytes(H, W, batch) + residual_pad_bytes(batch, H, W);
}

// Waves of SDA frames alternate between kExtractStreams streams (each with its
// own pyramid/SDA workspace) so one wave's small levels overlap the next wave's
// large ones; only the accumulating launches are chained (ascending order).
// Three streams measured best (round 1: 2 -> 3 streams -3.5% per step, 4 no gain).
constexpr int kExtractStreams = 3;
// planes per launch along grid.z (the analysis and synthesis kernels)
constexpr int kMaxBatch = 65535;
static int extract_streams() { return kExtractStreams; }

// Frames that TMA cannot stage (rows not 16-byte multiples, or a misaligned base or
// frame stride) are first copied to rows of align16(W) bytes (one HBM pass) so both
// the analysis and the accumulation keep their TMA paths.  SDA groups (d >= 2) go
// through exact u16 group sums (d <= 257) or fp32 frames (d > 257), both written with
// 16-byte rows by the SDA kernel.
static int pad_pitch_u8(int W) { return (int)align_up((size_t)W, 16); }
static int sum_pitch_u16(int W) { return (int)align_up((size_t)W, 8); }
static int sda_pitch_f32(int W) { return (int)align_up((size_t)W, 4); }
static size_t extract_wave_ws(int H, int W, int batch, int64_t depth, const Pyramid& pyr) {
    size_t s = align_up(sizeof(float) * pyramid_floats_per_frame(pyr) * (size_t)batch, 256);
    if (depth > 257) s += align_up(sizeof(float) * (size_t)H * sda_pitch_f32(W) * batch, 256);
    else if (depth > 1) s += align_up(sizeof(uint16_t) * (size_t)H * sum_pitch_u16(W) * batch, 256);
    else s += align_up((size_t)H * pad_pitch_u8(W) * batch, 256);   // re-pitched u8 frames (when needed)
    return s;
}

static size_t extract_ws(int H, int W, int batch, int64_t depth, const Pyramid& pyr) {
    return extract_streams() * extract_wave_ws(H, W, batch, depth, pyr) + zm_workspace_bytes(H, W);
}

// The workspace contract (include/prnu.h): 256-byte aligned.  The denoiser's pyramid planes
// are carved from it with 128-byte rows and written with 32-byte (256-bit) stores.
static int check_ws_align(const void* ws) {
    if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(PRNU_INVALID_ARG, "workspace must be 256-byte aligned");
    return PRNU_OK;
}

static int check_dims(int H, int W) {
    if (H <= 0 || W <= 0) return fail(PRNU_INVALID_ARG, "H and W must be positive");
    if ((long long)H * W > (1LL << 31) - 1) return fail(PRNU_INVALID_ARG, "H*W must fit in int32");
    return PRNU_OK;
}

// Shared by the device and host extraction entry points: process nb SDA groups
// whose frames start at `frames` (device), with wave workspace `ws`.
// depth > 0: SDA groups of `depth` consecutive frames.  depth < 0: stride
// selection (f4), the frames are every |depth|-th frame, denoised one by one.
static int extract_chunk(const uint8_t* frames, int64_t nb, int H, int W, int64_t depth, const Pyramid& pyr,
                         const ShrinkParams& sp, double* num, double* den, char* ws, cudaStream_t st,
                         cudaEvent_t acc_wait = nullptr, cudaEvent_t acc_done = nullptr) {
    float* pyr_ws = reinterpret_cast<float*>(ws);
    size_t pyr_bytes = align_up(sizeof(float) * pyramid_floats_per_frame(pyr) * (size_t)nb, 256);
    const long long P = (long long)H * W;
    int rc;
    if (depth == 1 || depth < 0) {
        const long long fstride = depth < 0 ? -depth * P : P;
        if (W % 16 || fstride % 16 || (uintptr_t)frames % 16) {   // re-pitched copy (see extract_wave_ws)
            const int Wp = pad_pitch_u8(W);
            uint8_t* padded = reinterpret_cast<uint8_t*>(ws + pyr_bytes);
            if ((rc = launch_pad_rows_u8(frames, nb, H, W, fstride, padded, Wp, st))) return rc;
            return run_residual_accumulate<uint8_t>(padded, padded, (int)nb, H, W, pyr, sp, SdaDiv{}, num, den, pyr_ws,
                                                    st, acc_wait, acc_done, (long long)H * Wp, Wp);
        }
        return run_residual_accumulate<uint8_t>(frames, frames, (int)nb, H, W, pyr, sp, SdaDiv{}, num, den, pyr_ws, st,
                                                acc_wait, acc_done, fstride);
    }
    if (depth == 2 && W % 16 == 0 && P % 16 == 0 && (uintptr_t)frames % 16 == 0 && H >= 32) {
        // SDA pairs: both frames of a group staged by one depth-2 TMA box in the analysis and
        // the accumulation, S = (b0 + b1) / 2 formed there (exact, R-11): no sum pass
        const u8pair* F = reinterpret_cast<const u8pair*>(frames);
        return run_residual_accumulate<u8pair>(F, F, (int)nb, H, W, pyr, sp, SdaDiv{}, num, den, pyr_ws, st, acc_wait,
                                               acc_done, P);
    }
    if (depth <= 257) {   // exact u16 group sums; S = RN(sum / d) inside the kernels (R-11)
        const int Wp = sum_pitch_u16(W);
        uint16_t* S = reinterpret_cast<uint16_t*>(ws + pyr_bytes);
        if ((rc = launch_sda_sum_u16(frames, nb, H, W, (int)depth, S, Wp, st))) return rc;
        SdaDiv div;
        div.d = (float)depth;
        div.r = 1.0f / div.d;   // IEEE fp32 division: RN(1/d)
        return run_residual_accumulate<uint16_t>(S, S, (int)nb, H, W, pyr, sp, div, num, den, pyr_ws, st, acc_wait,
                                                 acc_done, (long long)H * Wp, Wp);
    }
    const int Wp = sda_pitch_f32(W);
    float* S = reinterpret_cast<float*>(ws + pyr_bytes);
    if ((rc = launch_sda_average_pitched(frames, nb, H, W, (int)depth, S, Wp, st))) return rc;
    return run_residual_accumulate<float>(S, S, (int)nb, H, W, pyr, sp, SdaDiv{}, num, den, pyr_ws, st, acc_wait,
                                          acc_done, (long long)H * Wp, Wp);
}

template <typename TIn>
static int residual_impl(const TIn* planes, int batch, int H, int W, const prnu_denoise_params* p, int zero_mean,
                         float* W_out, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if (!planes || !W_out || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > kMaxBatch) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    ShrinkParams sp;
    if ((rc = validate_params(p, H, W, &sp))) return rc;
    Pyramid pyr = make_pyramid(H, W, p->levels);
    if (ws_bytes < residual_ws(batch, H, W, pyr)) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    if ((rc = check_ws_align(ws))) return rc;
    cudaStream_t st = as_stream(stream);
    float* pyr_ws = reinterpret_cast<float*>(ws);
    if (sizeof(TIn) == 1 && W % 16) {   // u8 rows that TMA cannot stage: re-pitch them first
        const int Wp = pad_pitch_u8(W);
        uint8_t* padded = reinterpret_cast<uint8_t*>(ws) + residual_ws(batch, H, W, pyr) -
                          residual_pad_bytes(batch, H, W);
        if ((rc = launch_pad_rows_u8(reinterpret_cast<const uint8_t*>(planes), batch, H, W, (long long)H * W, padded,
                                     Wp, st)))
            return rc;
        if ((rc = run_residual<TIn>(reinterpret_cast<const TIn*>(padded), batch, H, W, pyr, sp, W_out, pyr_ws, st, Wp)))
            return rc;
    } else if ((rc = run_residual<TIn>(planes, batch, H, W, pyr, sp, W_out, pyr_ws, st))) {
        return rc;
    }
    if (zero_mean) {
        char* zm = reinterpret_cast<char*>(ws) +
                   align_up(sizeof(float) * pyramid_floats_per_frame(pyr) * (size_t)batch, 256);
        if ((rc = launch_zero_mean_f32(W_out, batch, H, W, zm, st))) return rc;
    }
    return PRNU_OK;
}

}  // namespace prnu

using namespace prnu;

extern "C" {

int prnu_default_params(prnu_denoise_params* p) {
    if (!p) return fail(PRNU_INVALID_ARG, "params is NULL");
    p->sigma0_sq = 9.0f;
    p->levels = 4;
    p->n_windows = 4;
    p->windows[0] = 3;
    p->windows[1] = 5;
    p->windows[2] = 7;
    p->windows[3] = 9;
    return PRNU_OK;
}

int prnu_sda_groups(int64_t m, int64_t depth, int64_t* n_sda_host) {
    if (m < 1) return fail(PRNU_INVALID_ARG, "m must be >= 1");
    if (depth < 1 || depth > m) return fail(PRNU_DEPTH_EXCEEDS_FRAMES, "depth must be in 1..m");
    if (n_sda_host) *n_sda_host = m / depth;
    return PRNU_OK;
}

int prnu_sda_average(const uint8_t* frames, int64_t m, int H, int W, int64_t depth, float* sda_out,
                     int64_t* n_sda_host, void* stream) {
    int rc;
    if (!frames || !sda_out) return fail(PRNU_INVALID_ARG, "null pointer");
    if ((rc = check_dims(H, W))) return rc;
    int64_t ns;
    if ((rc = prnu_sda_groups(m, depth, &ns))) return rc;
    if (depth > 65793) return fail(PRNU_BAD_PARAMETER, "depth > 65793 (sum would exceed 2^24)");
    if (n_sda_host) *n_sda_host = ns;
    return launch_sda_average(frames, ns, (long long)H * W, (int)depth, sda_out, as_stream(stream));
}

int prnu_rgb_to_luma(const uint8_t* rgb, int64_t n, int H, int W, int layout, int rounding, void* luma_out,
                     void* stream) {
    int rc;
    if (!rgb || !luma_out) return fail(PRNU_INVALID_ARG, "null pointer");
    if (n < 1) return fail(PRNU_INVALID_ARG, "n must be >= 1");
    if ((rc = check_dims(H, W))) return rc;
    if (layout != 0 && layout != 1) return fail(PRNU_BAD_PARAMETER, "layout must be 0 (planar) or 1 (interleaved)");
    if (rounding != 0 && rounding != 1) return fail(PRNU_BAD_PARAMETER, "rounding must be 0 (fp32) or 1 (u8)");
    const long long P = (long long)H * W;
    if (P % 4) return fail(PRNU_BAD_PARAMETER, "H*W must be a multiple of 4");
    if (((uintptr_t)rgb & 3) || ((uintptr_t)luma_out & (rounding ? 3 : 15)))
        return fail(PRNU_INVALID_ARG, "rgb must be 4-byte aligned, luma_out 16-byte (fp32) / 4-byte (u8) aligned");
    return launch_rgb_to_luma(rgb, n, P, layout, rounding, luma_out, as_stream(stream));
}

size_t prnu_residual_workspace_bytes(int batch, int H, int W, const prnu_denoise_params* p) {
    if (batch < 1 || H <= 0 || W <= 0 || validate_params(p, H, W, nullptr)) return 0;
    return residual_ws(batch, H, W, make_pyramid(H, W, p->levels));
}

int prnu_residual(const float* planes, int batch, int H, int W, const prnu_denoise_params* p, int zero_mean,
                  float* W_out, void* ws, size_t ws_bytes, void* stream) {
    return residual_impl<float>(planes, batch, H, W, p, zero_mean, W_out, ws, ws_bytes, stream);
}

int prnu_residual_u8(const uint8_t* planes, int batch, int H, int W, const prnu_denoise_params* p, int zero_mean,
                     float* W_out, void* ws, size_t ws_bytes, void* stream) {
    return residual_impl<uint8_t>(planes, batch, H, W, p, zero_mean, W_out, ws, ws_bytes, stream);
}

int prnu_fingerprint_accumulate(const float* W, const float* I, int batch, int H, int Wd, double* sum_WI,
                                double* sum_I2, void* stream) {
    int rc;
    if (!W || !I || !sum_WI || !sum_I2) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1) return fail(PRNU_INVALID_ARG, "batch must be >= 1");
    if ((rc = check_dims(H, Wd))) return rc;
    return launch_accumulate(W, I, batch, (long long)H * Wd, sum_WI, sum_I2, as_stream(stream));
}

size_t prnu_finalize_workspace_bytes(int H, int W) {
    if (H <= 0 || W <= 0) return 0;
    return zm_workspace_bytes(H, W);
}

int prnu_fingerprint_finalize(const double* sum_WI, const double* sum_I2, int H, int W, double eps, int zero_mean,
                              float* K_out, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if (!sum_WI || !sum_I2 || !K_out) return fail(PRNU_INVALID_ARG, "null pointer");
    if ((rc = check_dims(H, W))) return rc;
    if (!(eps > 0.0)) return fail(PRNU_BAD_PARAMETER, "eps must be > 0");
    if (zero_mean && (!ws || ws_bytes < zm_workspace_bytes(H, W)))
        return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return launch_finalize(sum_WI, sum_I2, H, W, eps, zero_mean, K_out, ws, as_stream(stream));
}

size_t prnu_extract_workspace_bytes(int H, int W, int batch, int64_t depth, const prnu_denoise_params* p) {
    if (batch < 1 || depth < 1 || H <= 0 || W <= 0 || validate_params(p, H, W, nullptr)) return 0;
    return extract_ws(H, W, batch, depth, make_pyramid(H, W, p->levels));
}

// Per-device helper streams and events of the multi-stream extraction, created on
// first use and kept for the life of the process (no per-call create/destroy).
struct ExtractCtx {
    std::mutex mu;
    cudaStream_t helper[kExtractStreams - 1] = {};
    cudaEvent_t ev_start = nullptr, ev_end[kExtractStreams] = {}, acc[kExtractStreams] = {};
};
// One context per (device, stream priority): the helper streams run the waves at the
// priority of the caller's stream, so a caller can rank an extraction against its other work.
static int extract_ctx(ExtractCtx** out, cudaStream_t caller) {
    static std::mutex g_mu;
    constexpr int kPrio = 8;   // priority levels kept apart (CUDA has 6 on sm_100; clamped)
    static ExtractCtx* g_ctx[64][kPrio] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(PRNU_CUDA_ERROR, "cudaGetDevice");
    int prio = 0, lo = 0, hi = 0;
    if (cudaStreamGetPriority(caller, &prio) != cudaSuccess || cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess)
        return fail(PRNU_CUDA_ERROR, "stream priority query");
    const int pi = std::min(std::max(lo - prio, 0), kPrio - 1);   // 0 = the least priority
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_ctx[dev][pi]) {
        ExtractCtx* c = new ExtractCtx();
        cudaError_t e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
        for (int j = 0; j < kExtractStreams && e == cudaSuccess; ++j) {
            if (j > 0) e = cudaStreamCreateWithPriority(&c->helper[j - 1], cudaStreamNonBlocking, lo - pi);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_end[j], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->acc[j], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) {
            delete c;   // (handles created before the failure are leaked: the device is unusable anyway)
            return fail(PRNU_CUDA_ERROR, std::string("extraction streams: ") + cudaGetErrorString(e));
        }
        g_ctx[dev][pi] = c;
    }
    *out = g_ctx[dev][pi];
    return PRNU_OK;
}

// mode 0: SDA depth `depth` (1 = conventional); mode 1: stride selection with
// step `depth` (frames 0, depth, 2 depth, ... < m), each frame denoised.
static int extract_impl(const uint8_t* frames, int64_t m, int H, int W, int64_t depth, int mode,
                        const prnu_denoise_params* p, int batch, double eps, float* K_out, double* sum_WI,
                        double* sum_I2, int64_t* n_sda_host, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if (!frames || !K_out || !sum_WI || !sum_I2 || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > kMaxBatch) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    int64_t ns;
    if ((rc = prnu_sda_groups(m, depth, &ns))) return rc;
    if (mode == 1) ns = (m + depth - 1) / depth;   // frames 0, depth, 2 depth, ... < m
    const int64_t unit = mode == 1 ? 1 : depth;      // frames per unit in the workspace sizing
    const int64_t dsel = mode == 1 ? -depth : depth; // extract_chunk's depth argument
    if (mode == 0 && depth > 65793) return fail(PRNU_BAD_PARAMETER, "depth > 65793");
    if (!(eps > 0.0)) return fail(PRNU_BAD_PARAMETER, "eps must be > 0");
    ShrinkParams sp;
    if ((rc = validate_params(p, H, W, &sp))) return rc;
    Pyramid pyr = make_pyramid(H, W, p->levels);
    if (ws_bytes < extract_ws(H, W, batch, unit, pyr)) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    if ((rc = check_ws_align(ws))) return rc;
    if (n_sda_host) *n_sda_host = ns;
    cudaStream_t st = as_stream(stream);
    const size_t P = (size_t)H * W;
    cudaError_t e1 = cudaMemsetAsync(sum_WI, 0, sizeof(double) * P, st);
    cudaError_t e2 = cudaMemsetAsync(sum_I2, 0, sizeof(double) * P, st);
    if (e1 != cudaSuccess || e2 != cudaSuccess) return fail(PRNU_CUDA_ERROR, "cudaMemsetAsync failed");
    char* wsb = reinterpret_cast<char*>(ws);
    // per-kernel timing (prnu_profile_begin) serialises the waves so that each
    // kernel's event pair measures that kernel alone
    const int nst = extract_streams();
    const bool serial = profiling_active();
    const size_t wave = extract_wave_ws(H, W, batch, unit, pyr);
    char* zm = wsb + nst * wave;
    if (nst == 1 || serial || ns <= batch) {
        for (int64_t g0 = 0; g0 < ns; g0 += batch) {
            int64_t nb = std::min<int64_t>(batch, ns - g0);
            if ((rc = extract_chunk(frames + (size_t)g0 * depth * P, nb, H, W, dsel, pyr, sp, sum_WI, sum_I2, wsb,
                                    st)))
                return rc;
        }
        return launch_finalize(sum_WI, sum_I2, H, W, eps, 1, K_out, zm, st);
    }
    // nst streams: waves rotate over them; each wave's accumulation waits for the
    // previous wave's (events), so the per-pixel order stays ascending.  The helper
    // streams and events are created once per device (ExtractCtx) and reused; the
    // context's mutex serialises the enqueue of concurrent calls on one device.
    ExtractCtx* cx = nullptr;
    if ((rc = extract_ctx(&cx, st))) return rc;
    std::lock_guard<std::mutex> lock(cx->mu);
    cudaStream_t sts[kExtractStreams] = {st};
    for (int j = 1; j < nst; ++j) sts[j] = cx->helper[j - 1];
    cudaError_t e = cudaEventRecord(cx->ev_start, st);   // helper streams start after the caller's prior work
    for (int j = 1; j < nst && e == cudaSuccess; ++j) e = cudaStreamWaitEvent(sts[j], cx->ev_start, 0);
    rc = (e == cudaSuccess) ? PRNU_OK : fail(PRNU_CUDA_ERROR, std::string("stream setup: ") + cudaGetErrorString(e));
    int64_t k = 0;
    for (int64_t g0 = 0; g0 < ns && rc == PRNU_OK; g0 += batch, ++k) {
        int64_t nb = std::min<int64_t>(batch, ns - g0);
        const int j = (int)(k % nst), jp = (int)((k + nst - 1) % nst);
        rc = extract_chunk(frames + (size_t)g0 * depth * P, nb, H, W, dsel, pyr, sp, sum_WI, sum_I2,
                           wsb + j * wave, sts[j], k > 0 ? cx->acc[jp] : nullptr, cx->acc[j]);
    }
    for (int j = 1; j < nst && rc == PRNU_OK; ++j) {   // the caller's stream sees all waves
        e = cudaEventRecord(cx->ev_end[j], sts[j]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, cx->ev_end[j], 0);
        if (e != cudaSuccess) rc = fail(PRNU_CUDA_ERROR, std::string("stream join: ") + cudaGetErrorString(e));
    }
    if (rc == PRNU_OK) rc = launch_finalize(sum_WI, sum_I2, H, W, eps, 1, K_out, zm, st);
    return rc;
}

int prnu_extract_fingerprint(const uint8_t* frames, int64_t m, int H, int W, int64_t depth,
                             const prnu_denoise_params* p, int batch, double eps, float* K_out, double* sum_WI,
                             double* sum_I2, int64_t* n_sda_host, void* ws, size_t ws_bytes, void* stream) {
    return extract_impl(frames, m, H, W, depth, 0, p, batch, eps, K_out, sum_WI, sum_I2, n_sda_host, ws, ws_bytes,
                        stream);
}

int prnu_extract_fingerprint_stride(const uint8_t* frames, int64_t m, int H, int W, int64_t stride,
                                    const prnu_denoise_params* p, int batch, double eps, float* K_out,
                                    double* sum_WI, double* sum_I2, int64_t* n_used_host, void* ws, size_t ws_bytes,
                                    void* stream) {
    return extract_impl(frames, m, H, W, stride, 1, p, batch, eps, K_out, sum_WI, sum_I2, n_used_host, ws, ws_bytes,
                        stream);
}

size_t prnu_extract_host_workspace_bytes(int H, int W, int batch, int64_t depth, const prnu_denoise_params* p) {
    size_t base = prnu_extract_workspace_bytes(H, W, batch, depth, p);
    if (!base) return 0;
    size_t chunk = (size_t)batch * depth * H * W;
    return base + 2 * align_up(chunk, 256) + align_up(sizeof(float) * (size_t)H * W, 256);
}

int prnu_extract_fingerprint_host(const uint8_t* frames_host, int64_t m, int H, int W, int64_t depth,
                                  const prnu_denoise_params* p, int batch, double eps, float* K_out_host,
                                  double* sum_WI, double* sum_I2, int64_t* n_sda_host, void* ws, size_t ws_bytes,
                                  void* stream) {
    int rc;
    if (!frames_host || !K_out_host || !sum_WI || !sum_I2 || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > kMaxBatch) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    int64_t ns;
    if ((rc = prnu_sda_groups(m, depth, &ns))) return rc;
    if (depth > 65793) return fail(PRNU_BAD_PARAMETER, "depth > 65793");
    if (!(eps > 0.0)) return fail(PRNU_BAD_PARAMETER, "eps must be > 0");
    ShrinkParams sp;
    if ((rc = validate_params(p, H, W, &sp))) return rc;
    if (ws_bytes < prnu_extract_host_workspace_bytes(H, W, batch, depth, p))
        return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    if ((rc = check_ws_align(ws))) return rc;
    if (n_sda_host) *n_sda_host = ns;
    Pyramid pyr = make_pyramid(H, W, p->levels);
    const size_t P = (size_t)H * W;
    const size_t base = extract_ws(H, W, batch, depth, pyr);
    const size_t chunk = (size_t)batch * depth * P;
    char* wsb = reinterpret_cast<char*>(ws);
    uint8_t* stage[2] = {reinterpret_cast<uint8_t*>(wsb + base),
                         reinterpret_cast<uint8_t*>(wsb + base + align_up(chunk, 256))};
    float* Kdev = reinterpret_cast<float*>(wsb + base + 2 * align_up(chunk, 256));
    char* zm = wsb + base - zm_workspace_bytes(H, W);
    cudaStream_t st = as_stream(stream);
    cudaStream_t cp = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    cudaError_t e = cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(sum_WI, 0, sizeof(double) * P, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(sum_I2, 0, sizeof(double) * P, st);
    // the copy stream must not overwrite a staging buffer the compute stream still reads
    if (e == cudaSuccess) e = cudaEventRecord(freed[0], st);
    if (e == cudaSuccess) e = cudaEventRecord(freed[1], st);
    rc = (e == cudaSuccess) ? PRNU_OK : fail(PRNU_CUDA_ERROR, std::string("setup: ") + cudaGetErrorString(e));
    int64_t c = 0;
    for (int64_t g0 = 0; g0 < ns && rc == PRNU_OK; g0 += batch, ++c) {
        int64_t nb = std::min<int64_t>(batch, ns - g0);
        int k = (int)(c & 1);
        size_t bytes = (size_t)nb * depth * P;
        e = cudaStreamWaitEvent(cp, freed[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(stage[k], frames_host + (size_t)g0 * depth * P, bytes, cudaMemcpyHostToDevice, cp);
        if (e == cudaSuccess) e = cudaEventRecord(ready[k], cp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ready[k], 0);
        if (e != cudaSuccess) {
            rc = fail(PRNU_CUDA_ERROR, std::string("H2D staging: ") + cudaGetErrorString(e));
            break;
        }
        rc = extract_chunk(stage[k], nb, H, W, depth, pyr, sp, sum_WI, sum_I2, wsb, st);
        if (rc == PRNU_OK && (e = cudaEventRecord(freed[k], st)) != cudaSuccess)
            rc = fail(PRNU_CUDA_ERROR, cudaGetErrorString(e));
    }
    if (rc == PRNU_OK) rc = launch_finalize(sum_WI, sum_I2, H, W, eps, 1, Kdev, zm, st);
    if (rc == PRNU_OK) {
        e = cudaMemcpyAsync(K_out_host, Kdev, sizeof(float) * P, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(PRNU_CUDA_ERROR, std::string("D2H K: ") + cudaGetErrorString(e));
    } else {
        cudaStreamSynchronize(st);
    }
    cudaStreamSynchronize(cp);
    for (int i = 0; i < 2; ++i) {
        if (ready[i]) cudaEventDestroy(ready[i]);
        if (freed[i]) cudaEventDestroy(freed[i]);
    }
    if (cp) cudaStreamDestroy(cp);
    return rc;
}

// ---------------------------------------------------------------- multi-depth, one upload
static constexpr int64_t kMultiChunk = 128;   // frames per H2D chunk (event granularity)

static size_t multi_layout(int64_t m, int H, int W, int batch, const int64_t* depths, int n, const Pyramid& pyr,
                           size_t* off_waves, size_t* off_K, size_t* off_zm) {
    const size_t P = (size_t)H * W;
    size_t o = align_up((size_t)m * P, 256);                      // the whole u8 stack on the device
    *off_waves = o;
    size_t wmax = 0;
    for (int i = 0; i < n; ++i) wmax = std::max(wmax, extract_wave_ws(H, W, batch, depths[i], pyr));
    o += wmax;                                                     // one wave workspace, reused per depth
    *off_K = o;
    o += align_up(sizeof(float) * P * n, 256);
    *off_zm = o;
    o += zm_workspace_bytes(H, W);
    return o;
}

size_t prnu_extract_multi_host_workspace_bytes(int64_t m, int H, int W, int batch, const int64_t* depths_host,
                                               int n_depths, const prnu_denoise_params* p) {
    if (m < 1 || H <= 0 || W <= 0 || batch < 1 || n_depths < 1 || !depths_host || validate_params(p, H, W, nullptr))
        return 0;
    for (int i = 0; i < n_depths; ++i)
        if (depths_host[i] < 1 || depths_host[i] > m) return 0;
    size_t a, b, c;
    return multi_layout(m, H, W, batch, depths_host, n_depths, make_pyramid(H, W, p->levels), &a, &b, &c);
}

int prnu_extract_multi_host(const uint8_t* frames_host, int64_t m, int H, int W, const int64_t* depths_host,
                            int n_depths, const prnu_denoise_params* p, int batch, double eps, float* K_out_host,
                            double* sums, int64_t* n_sda_host, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if (!frames_host || !depths_host || !K_out_host || !sums || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || n_depths < 1) return fail(PRNU_INVALID_ARG, "batch and n_depths must be >= 1");
    if ((rc = check_dims(H, W))) return rc;
    for (int i = 0; i < n_depths; ++i) {
        int64_t ns;
        if ((rc = prnu_sda_groups(m, depths_host[i], &ns))) return rc;
        if (depths_host[i] > 65793) return fail(PRNU_BAD_PARAMETER, "depth > 65793");
        if (n_sda_host) n_sda_host[i] = ns;
    }
    if (!(eps > 0.0)) return fail(PRNU_BAD_PARAMETER, "eps must be > 0");
    ShrinkParams sp;
    if ((rc = validate_params(p, H, W, &sp))) return rc;
    Pyramid pyr = make_pyramid(H, W, p->levels);
    size_t off_w, off_K, off_zm;
    if (ws_bytes < multi_layout(m, H, W, batch, depths_host, n_depths, pyr, &off_w, &off_K, &off_zm))
        return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    if ((rc = check_ws_align(ws))) return rc;
    const size_t P = (size_t)H * W;
    char* wsb = reinterpret_cast<char*>(ws);
    uint8_t* fdev = reinterpret_cast<uint8_t*>(wsb);
    float* Kdev = reinterpret_cast<float*>(wsb + off_K);
    cudaStream_t st = as_stream(stream), cp = nullptr;
    const int64_t n_chunks = (m + kMultiChunk - 1) / kMultiChunk;
    std::vector<cudaEvent_t> ev((size_t)n_chunks, nullptr);
    cudaEvent_t ev_start = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
    for (int64_t c = 0; c < n_chunks && e == cudaSuccess; ++c) e = cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming);
    // the upload starts after the caller's prior work on `stream` (it owns the workspace)
    if (e == cudaSuccess) e = cudaEventRecord(ev_start, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cp, ev_start, 0);
    for (int64_t c = 0; c < n_chunks && e == cudaSuccess; ++c) {
        const int64_t f0 = c * kMultiChunk, nf = std::min<int64_t>(kMultiChunk, m - f0);
        e = cudaMemcpyAsync(fdev + (size_t)f0 * P, frames_host + (size_t)f0 * P, (size_t)nf * P,
                            cudaMemcpyHostToDevice, cp);
        if (e == cudaSuccess) e = cudaEventRecord(ev[c], cp);
    }
    rc = (e == cudaSuccess) ? PRNU_OK : fail(PRNU_CUDA_ERROR, std::string("upload: ") + cudaGetErrorString(e));
    int64_t waited = -1;   // highest chunk the compute stream already waits for
    for (int i = 0; i < n_depths && rc == PRNU_OK; ++i) {
        const int64_t d = depths_host[i], ns = m / d;
        double* num = sums + (size_t)2 * i * P;
        double* den = num + P;
        e = cudaMemsetAsync(num, 0, sizeof(double) * 2 * P, st);
        if (e != cudaSuccess) rc = fail(PRNU_CUDA_ERROR, "cudaMemsetAsync failed");
        for (int64_t g0 = 0; g0 < ns && rc == PRNU_OK; g0 += batch) {
            const int64_t nb = std::min<int64_t>(batch, ns - g0);
            const int64_t need = ((g0 + nb) * d - 1) / kMultiChunk;   // chunk holding the wave's last frame
            for (; waited < need && rc == PRNU_OK; ++waited)
                if (cudaStreamWaitEvent(st, ev[waited + 1], 0) != cudaSuccess)
                    rc = fail(PRNU_CUDA_ERROR, "cudaStreamWaitEvent");
            if (rc == PRNU_OK)
                rc = extract_chunk(fdev + (size_t)g0 * d * P, nb, H, W, d, pyr, sp, num, den, wsb + off_w, st);
        }
        if (rc == PRNU_OK) rc = launch_finalize(num, den, H, W, eps, 1, Kdev + (size_t)i * P, wsb + off_zm, st);
        if (rc == PRNU_OK &&
            (e = cudaMemcpyAsync(K_out_host + (size_t)i * P, Kdev + (size_t)i * P, sizeof(float) * P,
                                 cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            rc = fail(PRNU_CUDA_ERROR, std::string("D2H K: ") + cudaGetErrorString(e));
    }
    // never leave the upload running into memory the caller may reuse
    for (; waited + 1 < n_chunks && rc == PRNU_OK; ++waited) cudaStreamWaitEvent(st, ev[waited + 1], 0);
    cudaError_t es = cudaStreamSynchronize(st);
    if (rc == PRNU_OK && es != cudaSuccess) rc = fail(PRNU_CUDA_ERROR, std::string("sync: ") + cudaGetErrorString(es));
    cudaStreamSynchronize(cp);
    for (cudaEvent_t x : ev)
        if (x) cudaEventDestroy(x);
    if (ev_start) cudaEventDestroy(ev_start);
    if (cp) cudaStreamDestroy(cp);
    return rc;
}

size_t prnu_ncc_workspace_bytes(int batch, int H, int W) {
    if (batch < 1 || H <= 0 || W <= 0) return 0;
    return ncc_workspace_bytes(batch);
}

int prnu_ncc(const float* a, const float* b, int batch, int H, int W, double* ncc_out, void* ws, size_t ws_bytes,
             void* stream) {
    int rc;
    if (!a || !b || !ncc_out || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > 65535) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    if (ws_bytes < ncc_workspace_bytes(batch)) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return launch_ncc(a, b, batch, (long long)H * W, ncc_out, ws, as_stream(stream));
}

int prnu_check_results(int kind, const double* values, int64_t n, void* stream) {
    if (!values) return fail(PRNU_INVALID_ARG, "null pointer");
    if (n < 1) return fail(PRNU_INVALID_ARG, "n must be positive");
    if (kind < 0 || kind > 2) return fail(PRNU_INVALID_ARG, "kind must be 0 (NCC), 1 (PCE) or 2 (sum_I2)");
    return prnu::check_results(kind, values, (long long)n, as_stream(stream));
}

int prnu_pce_template(const float* K, int k_batch, const uint8_t* Iq, int batch, int H, int W, float* T_out,
                      void* stream) {
    int rc;
    if (!K || !Iq || !T_out) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > 65535) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if (k_batch != 1 && k_batch != batch) return fail(PRNU_DIMENSION_MISMATCH, "k_batch must be 1 or batch");
    if ((rc = check_dims(H, W))) return rc;
    return launch_pce_template(K, k_batch, Iq, batch, (long long)H * W, T_out, as_stream(stream));
}

int prnu_pce_plan_create(int H, int W, int batch, size_t* ws_bytes, void** plan) {
    int rc;
    if (!ws_bytes || !plan) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > 65535) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    return pce_plan_create(H, W, batch, ws_bytes, plan);
}

int prnu_pce(void* plan, const float* residual, const float* template_, int batch, int exclusion_half, int aligned,
             double* pce, int* peak_y, int* peak_x, double* peak, void* ws, size_t ws_bytes, void* stream) {
    if (!plan || !residual || !template_ || !pce || !peak_y || !peak_x || !peak || !ws)
        return fail(PRNU_INVALID_ARG, "null pointer");
    int H, W, pb;
    size_t need;
    pce_plan_dims(plan, &H, &W, &pb, &need);
    if (batch != pb) return fail(PRNU_DIMENSION_MISMATCH, "batch differs from the plan's batch");
    if (exclusion_half < 0) return fail(PRNU_BAD_PARAMETER, "exclusion_half must be >= 0");
    if (ws_bytes < need) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return run_pce(plan, residual, template_, nullptr, 0, nullptr, exclusion_half, aligned, pce, peak_y, peak_x, peak, ws,
                   as_stream(stream));
}

int prnu_pce_residual_spectrum(void* plan, const float* residual, void* ws, size_t ws_bytes, void* stream) {
    if (!plan || !residual || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    int H, W, pb;
    size_t need;
    pce_plan_dims(plan, &H, &W, &pb, &need);
    if (ws_bytes < need) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return run_pce(plan, residual, nullptr, nullptr, 0, nullptr, 0, 0, nullptr, nullptr, nullptr, nullptr, ws,
                   as_stream(stream));
}

int prnu_pce_cached(void* plan, const float* template_, int batch, int exclusion_half, int aligned, double* pce,
                    int* peak_y, int* peak_x, double* peak, void* ws, size_t ws_bytes, void* stream) {
    if (!plan || !template_ || !pce || !peak_y || !peak_x || !peak || !ws)
        return fail(PRNU_INVALID_ARG, "null pointer");
    int H, W, pb;
    size_t need;
    pce_plan_dims(plan, &H, &W, &pb, &need);
    if (batch != pb) return fail(PRNU_DIMENSION_MISMATCH, "batch differs from the plan's batch");
    if (exclusion_half < 0) return fail(PRNU_BAD_PARAMETER, "exclusion_half must be >= 0");
    if (ws_bytes < need) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return run_pce(plan, nullptr, template_, nullptr, 0, nullptr, exclusion_half, aligned, pce, peak_y, peak_x, peak,
                   ws, as_stream(stream));
}

int prnu_pce_cached_template(void* plan, const float* K, int k_batch, const uint8_t* Iq, int batch,
                             int exclusion_half, int aligned, double* pce, int* peak_y, int* peak_x, double* peak,
                             void* ws, size_t ws_bytes, void* stream) {
    if (!plan || !K || !Iq || !pce || !peak_y || !peak_x || !peak || !ws)
        return fail(PRNU_INVALID_ARG, "null pointer");
    int H, W, pb;
    size_t need;
    pce_plan_dims(plan, &H, &W, &pb, &need);
    if (batch != pb) return fail(PRNU_DIMENSION_MISMATCH, "batch differs from the plan's batch");
    if (k_batch != 1 && k_batch != batch) return fail(PRNU_DIMENSION_MISMATCH, "k_batch must be 1 or batch");
    if (exclusion_half < 0) return fail(PRNU_BAD_PARAMETER, "exclusion_half must be >= 0");
    if (ws_bytes < need) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return run_pce(plan, nullptr, nullptr, K, k_batch, Iq, exclusion_half, aligned, pce, peak_y, peak_x, peak, ws,
                   as_stream(stream));
}

int prnu_pce_plan_destroy(void* plan) { return pce_plan_destroy(plan); }

int prnu_wdft_plan_create(int H, int W, int batch, size_t* ws_bytes, void** plan) {
    int rc;
    if (!ws_bytes || !plan) return fail(PRNU_INVALID_ARG, "null pointer");
    if ((rc = check_dims(H, W))) return rc;
    if (batch < 1) return fail(PRNU_INVALID_ARG, "batch must be >= 1");
    if (H < 4 || W < 4) return fail(PRNU_PLANE_TOO_SMALL, "WDFT needs H, W >= 4");
    return wdft_plan_create(H, W, batch, ws_bytes, plan);
}

int prnu_wdft(void* plan, const float* K, float* K_out, void* ws, size_t ws_bytes, void* stream) {
    if (!plan || !K || !K_out || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    int H, W, b;
    size_t need;
    wdft_plan_dims(plan, &H, &W, &b, &need);
    if (ws_bytes < need) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return run_wdft(plan, K, K_out, ws, as_stream(stream));
}

int prnu_wdft_plan_destroy(void* plan) { return wdft_plan_destroy(plan); }

int prnu_block_plan_create(int H, int W, int block, int* n_tiles_host, size_t* ws_bytes, void** plan) {
    int rc;
    if (!n_tiles_host || !ws_bytes || !plan) return fail(PRNU_INVALID_ARG, "null pointer");
    if ((rc = check_dims(H, W))) return rc;
    if (block < 2) return fail(PRNU_BAD_PARAMETER, "block must be >= 2");
    return block_plan_create(H, W, block, n_tiles_host, ws_bytes, plan);
}

int prnu_block_match(void* plan, const float* residual, const float* template_, int exclusion_half, double* pce,
                     double* ncc, void* ws, size_t ws_bytes, void* stream) {
    if (!plan || !residual || !template_ || !pce || !ncc || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    int H, W, n;
    size_t need;
    block_plan_dims(plan, &H, &W, &n, &need);
    if (exclusion_half < 0) return fail(PRNU_BAD_PARAMETER, "exclusion_half must be >= 0");
    if (ws_bytes < need) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    return run_block_match(plan, residual, template_, exclusion_half, pce, ncc, ws, as_stream(stream));
}

int prnu_block_plan_destroy(void* plan) { return block_plan_destroy(plan); }

size_t prnu_residual_variant_workspace_bytes(int batch, int H, int W, const prnu_denoise_params* p,
                                             const prnu_denoise_variant* v) {
    if (batch < 1 || H <= 0 || W <= 0 || validate_params(p, H, W, nullptr) || validate_variant(v)) return 0;
    return variant_ws(batch, H, W, p, v);
}

int prnu_residual_variant(const float* planes, int batch, int H, int W, const prnu_denoise_params* p,
                          const prnu_denoise_variant* v, int zero_mean, float* W_out, void* ws, size_t ws_bytes,
                          void* stream) {
    int rc;
    if (!planes || !W_out || !ws) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > kMaxBatch) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    ShrinkParams sp;
    if ((rc = validate_params(p, H, W, &sp))) return rc;
    if ((rc = validate_variant(v))) return rc;
    if (ws_bytes < variant_ws(batch, H, W, p, v)) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    if ((rc = check_ws_align(ws))) return rc;
    cudaStream_t st = as_stream(stream);
    if ((rc = run_residual_variant(planes, batch, H, W, p->levels, v->taps, v->boundary, v->transform, sp, W_out,
                                   reinterpret_cast<float*>(ws), st)))
        return rc;
    if (zero_mean) {
        char* zm = reinterpret_cast<char*>(ws) +
                   variant_workspace_bytes(batch, H, W, p->levels, v->taps, v->boundary, v->transform);
        if ((rc = launch_zero_mean_f32(W_out, batch, H, W, zm, st))) return rc;
    }
    return PRNU_OK;
}

// f3 inside the extraction: SDA average (fp32 S, R-11) -> variant residual -> MLE
// accumulation in ascending group order -> finalize, one wave of `batch` SDA frames at a
// time (the composition prnu_sda_average -> prnu_residual_variant ->
// prnu_fingerprint_accumulate -> prnu_fingerprint_finalize, bit-identical to it).
static size_t extract_variant_ws(int H, int W, int batch, const prnu_denoise_params* p, const prnu_denoise_variant* v) {
    const size_t plane = sizeof(float) * (size_t)batch * H * W;
    return 2 * align_up(plane, 256) + align_up(variant_ws(batch, H, W, p, v), 256) + zm_workspace_bytes(H, W);
}

size_t prnu_extract_variant_workspace_bytes(int H, int W, int batch, const prnu_denoise_params* p,
                                            const prnu_denoise_variant* v) {
    if (batch < 1 || batch > kMaxBatch || H <= 0 || W <= 0 || validate_params(p, H, W, nullptr) ||
        validate_variant(v))
        return 0;
    return extract_variant_ws(H, W, batch, p, v);
}

int prnu_extract_fingerprint_variant(const uint8_t* frames, int64_t m, int H, int W, int64_t depth,
                                     const prnu_denoise_params* p, const prnu_denoise_variant* v, int batch,
                                     double eps, float* K_out, double* sum_WI, double* sum_I2, int64_t* n_sda_host,
                                     void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if (!frames || !K_out || !sum_WI || !sum_I2 || !ws || !p || !v) return fail(PRNU_INVALID_ARG, "null pointer");
    if (batch < 1 || batch > kMaxBatch) return fail(PRNU_INVALID_ARG, "batch must be in 1..65535");
    if ((rc = check_dims(H, W))) return rc;
    int64_t ns;
    if ((rc = prnu_sda_groups(m, depth, &ns))) return rc;
    if (depth > 65793) return fail(PRNU_BAD_PARAMETER, "depth > 65793 (sum would exceed 2^24)");
    if (!(eps > 0.0)) return fail(PRNU_BAD_PARAMETER, "eps must be > 0");
    ShrinkParams sp;
    if ((rc = validate_params(p, H, W, &sp))) return rc;
    if ((rc = validate_variant(v))) return rc;
    if (ws_bytes < extract_variant_ws(H, W, batch, p, v)) return fail(PRNU_WORKSPACE_TOO_SMALL, "workspace too small");
    if ((rc = check_ws_align(ws))) return rc;
    if (n_sda_host) *n_sda_host = ns;
    cudaStream_t st = as_stream(stream);
    const size_t P = (size_t)H * W;
    char* wsb = reinterpret_cast<char*>(ws);
    float* S = reinterpret_cast<float*>(wsb);
    float* Wr = reinterpret_cast<float*>(wsb + align_up(sizeof(float) * (size_t)batch * P, 256));
    float* vws = reinterpret_cast<float*>(wsb + 2 * align_up(sizeof(float) * (size_t)batch * P, 256));
    char* zm = wsb + 2 * align_up(sizeof(float) * (size_t)batch * P, 256) + align_up(variant_ws(batch, H, W, p, v), 256);
    if (cudaMemsetAsync(sum_WI, 0, sizeof(double) * P, st) != cudaSuccess ||
        cudaMemsetAsync(sum_I2, 0, sizeof(double) * P, st) != cudaSuccess)
        return fail(PRNU_CUDA_ERROR, "cudaMemsetAsync");
    for (int64_t g0 = 0; g0 < ns; g0 += batch) {
        const int nb = (int)std::min<int64_t>(batch, ns - g0);
        if ((rc = launch_sda_average(frames + (size_t)g0 * depth * P, nb, (long long)P, (int)depth, S, st))) return rc;
        if ((rc = run_residual_variant(S, nb, H, W, p->levels, v->taps, v->boundary, v->transform, sp, Wr, vws, st)))
            return rc;
        if ((rc = launch_accumulate(Wr, S, nb, (long long)P, sum_WI, sum_I2, st))) return rc;
    }
    return launch_finalize(sum_WI, sum_I2, H, W, eps, 1, K_out, zm, st);
}

int prnu_wavelet_filter(int taps, double* h_out) {
    if (!h_out) return fail(PRNU_INVALID_ARG, "null pointer");
    return variant_filter(taps, h_out);
}

int prnu_profile_begin(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof) {
        g_ev_pool.push_back(r.a);
        g_ev_pool.push_back(r.b);
    }
    g_prof.clear();
    g_prof_on = true;
    return PRNU_OK;
}

int prnu_profile_end(int max_kernels, char* names, double* ms_total, int64_t* launches, int* n_kernels) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = false;
    std::vector<std::string> nm;
    std::vector<double> ms;
    std::vector<int64_t> cnt;
    int rc = PRNU_OK;
    for (auto& r : g_prof) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
        if (e != cudaSuccess) {
            rc = fail(PRNU_CUDA_ERROR, std::string("profile: ") + cudaGetErrorString(e));
            break;
        }
        size_t k = 0;
        while (k < nm.size() && nm[k] != r.name) ++k;
        if (k == nm.size()) {
            nm.push_back(r.name);
            ms.push_back(0.0);
            cnt.push_back(0);
        }
        ms[k] += t;
        cnt[k] += 1;
    }
    int n = (int)std::min<size_t>(nm.size(), (size_t)std::max(max_kernels, 0));
    for (int k = 0; k < n; ++k) {
        if (names) {
            std::strncpy(names + 64 * k, nm[k].c_str(), 63);
            names[64 * k + 63] = 0;
        }
        if (ms_total) ms_total[k] = ms[k];
        if (launches) launches[k] = cnt[k];
    }
    if (n_kernels) *n_kernels = (int)nm.size();
    return rc;
}

const char* prnu_last_error(void) { return t_err.c_str(); }

uint64_t prnu_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* prnu_version(void) {
    return "prnu-b200 0.2.0 (sm_100a)"
#ifdef PRNU_DEBUG
           " +debug"
#endif
#ifdef PRNU_RACE_STRESS
           " +race-stress"
#endif
        ;
}

}  // extern "C"
