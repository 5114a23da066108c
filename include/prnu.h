/*
 * prnu.h — C ABI of libprnu.so, the B200 (sm_100a) hot path of SDA-frame PRNU
 * fingerprint extraction (Taspinar, Mohanty, Memon, arXiv 1909.04573).
 *
 * Citations: P:<n> = PAPER.md line n; S:<n> = SPEC.md line n; R-<n> = a
 * reading of the paper fixed in DESIGN.md §3 where the paper is silent.
 *
 * Conventions (all entry points):
 *  - Every pointer is a DEVICE pointer owned by the caller unless the argument
 *    name ends in `_host`.  The library never allocates or frees caller memory;
 *    scratch space is the caller-owned `ws` of at least the size the matching
 *    `*_workspace_bytes` query returns (256-byte aligned; the denoising entry
 *    points reject a misaligned `ws` with PRNU_INVALID_ARG).
 *  - Planes are row-major and contiguous: `[batch][H][W]`, H rows of W columns,
 *    frames/batch outermost.  "1920x1080" means W = 1920, H = 1080.
 *  - Calls are asynchronous on `stream` (a `cudaStream_t` passed as void*;
 *    NULL = the legacy default stream).  Arguments are validated synchronously
 *    before anything is launched; on a non-zero status nothing was launched
 *    (except PRNU_CUDA_ERROR, which reports a failed launch).
 *  - Results are deterministic: identical inputs give bit-identical outputs,
 *    independent of `batch` (no atomics on any value-carrying path, fixed
 *    reduction orders).
 *  - `prnu_last_error()` returns a thread-local description of the last
 *    failure of the calling thread.
 */
#ifndef PRNU_H
#define PRNU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (SPEC error names in brackets). */
enum {
    PRNU_OK = 0,
    PRNU_INVALID_ARG = 1,          /* null pointer, non-positive size, batch < 1            */
    PRNU_PLANE_TOO_SMALL = 2,      /* H or W < 2^levels                      [S:118]        */
    PRNU_DEPTH_EXCEEDS_FRAMES = 3, /* depth > m or depth < 1                 [S:189]        */
    PRNU_BAD_PARAMETER = 4,        /* sigma0_sq <= 0, levels outside 1..6, window not in
                                      {3,5,7,9}, exclusion_half < 0        [S:110]        */
    PRNU_DIMENSION_MISMATCH = 5,   /*                                        [S:198, S:207] */
    PRNU_EMPTY_ACCUMULATOR = 6,    /* prnu_check_results on sum_I2           [S:216]        */
    PRNU_CONSTANT_INPUT = 7,       /* prnu_check_results on NCC values       [S:288]        */
    PRNU_DEGENERATE_SURFACE = 8,   /* prnu_check_results on PCE peaks        [S:297]        */
    PRNU_WORKSPACE_TOO_SMALL = 9,
    PRNU_CUDA_ERROR = 10           /* a launch / cuFFT call failed; see prnu_last_error() */
};

/* Parameters of the denoiser F (P:150, P:259 cite the Mihcak wavelet filter
 * without internals; S:109-117 and S:149-150 parameterise it; R-1..R-8).
 *   F = 8-tap Daubechies DWT (4 vanishing moments), `levels` levels,
 *       half-sample symmetric extension, subband length floor((N+7)/2);
 *       every detail coefficient c becomes c * v/(v + sigma0_sq) with
 *       v = max(0, min_w mean_{w x w}(c^2) - sigma0_sq) over `windows`
 *       (mirror-extended windows, divided by w^2); the approximation passes
 *       through; inverse DWT.  The residual W = I - F(I).           */
typedef struct {
    float sigma0_sq;   /* base noise variance, [0,255]^2 units; default 9.0      */
    int levels;        /* decomposition depth 1..6; default 4                    */
    int n_windows;     /* number of valid entries in `windows` (1..4); default 4 */
    int windows[4];    /* odd window sizes from {3,5,7,9}; default {3,5,7,9}     */
} prnu_denoise_params;

/* Fill *p with the defaults above. */
int prnu_default_params(prnu_denoise_params* p);

/* ---------------------------------------------------------------------------
 * a1  SDA grouping and averaging — P:124 ("g non-intersecting equal-sized
 * subgroups ... each with d = m/g frames"), P:170-175 (I_i^SDA =
 * sum_{j=(i-1)d+1}^{id} I_j / d).
 *
 * prnu_sda_groups: *n_sda_host = floor(m / depth) (the m mod depth
 *   trailing frames are dropped).  PRNU_DEPTH_EXCEEDS_FRAMES if depth > m or
 *   depth < 1.
 * prnu_sda_average: frames u8 [m][H][W] -> sda_out fp32 [floor(m/depth)][H][W].
 *   Group i averages frames [i*depth, (i+1)*depth).  Each output is the exact
 *   integer sum divided by depth, rounded once to the nearest fp32 (R-11):
 *   bit-exact.  depth == 1 widens u8 to fp32.  n_sda_host (optional, host)
 *   receives the group count.
 * ------------------------------------------------------------------------- */
int prnu_sda_groups(int64_t m, int64_t depth, int64_t* n_sda_host);
int prnu_sda_average(const uint8_t* frames, int64_t m, int H, int W, int64_t depth,
                     float* sda_out, int64_t* n_sda_host, void* stream);

/* ---------------------------------------------------------------------------
 * f4  RGB -> luminance with the BT.601 weights BASELINE
 * config 3 names ("converted to luminance (0.299/0.587/0.114)").
 *
 * prnu_rgb_to_luma: rgb u8, layout 0 = planar [n][3][H][W] (R, G, B planes),
 *   layout 1 = interleaved [n][H][W][3]; luma_out [n][H][W].  With the exact
 *   integer s = 299 R + 587 G + 114 B:
 *     rounding 0: fp32 luma = RN_fp32(s / 1000) (correctly rounded; bit-exact);
 *     rounding 1: u8 luma = s / 1000 rounded half to even (exact rule).
 *   H*W must be a multiple of 4; rgb 4-byte aligned; luma_out 16-byte (fp32)
 *   or 4-byte (u8) aligned.  Errors: INVALID_ARG, BAD_PARAMETER.
 * ------------------------------------------------------------------------- */
int prnu_rgb_to_luma(const uint8_t* rgb, int64_t n, int H, int W, int layout, int rounding, void* luma_out,
                     void* stream);

/* ---------------------------------------------------------------------------
 * a2-a4  Noise residual W = I - F(I) — P:83 (W_k = I_k - F(I_k))
 * (W^SDA = I^SDA - F(I^SDA)).
 *
 * planes fp32 (or u8 for the _u8 variant) [batch][H][W] -> W_out fp32
 * [batch][H][W].  zero_mean != 0 additionally subtracts each row's mean, then
 * each column's mean (used for query residuals before PCE, R-9).  The
 * residual is computed in the noise domain, W = IDWT(0, c - F(c)) (equal to
 * I - F(I) in exact arithmetic, R-10), in fp32; max |error| vs the fp64 oracle
 * <= 1e-3 intensity units (BASELINE tolerance).
 * Errors: PLANE_TOO_SMALL (H or W < 2^levels), BAD_PARAMETER,
 * WORKSPACE_TOO_SMALL.
 * ------------------------------------------------------------------------- */
size_t prnu_residual_workspace_bytes(int batch, int H, int W, const prnu_denoise_params* p);
int prnu_residual(const float* planes, int batch, int H, int W, const prnu_denoise_params* p,
                  int zero_mean, float* W_out, void* ws, size_t ws_bytes, void* stream);
int prnu_residual_u8(const uint8_t* planes, int batch, int H, int W, const prnu_denoise_params* p,
                     int zero_mean, float* W_out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * a5  MLE accumulation — Eq. (2) P:151-155 and its SDA form P:200-203:
 * K = sum_i W_i I_i / sum_i I_i^2.
 * sum_WI[p] += W[b][p] * I[b][p], sum_I2[p] += I[b][p]^2 for b = 0..batch-1 in
 * ascending order, products and sums in fp64 (a product of two
 * fp32 values is exact in fp64).  sum_WI / sum_I2 are fp64 [H][W], in-out;
 * the caller zeroes them before the first contribution.
 * ------------------------------------------------------------------------- */
int prnu_fingerprint_accumulate(const float* W, const float* I, int batch, int H, int Wd,
                                double* sum_WI, double* sum_I2, void* stream);

/* ---------------------------------------------------------------------------
 * a6  Finalize — S:212-220: K = sum_WI / max(sum_I2, eps) element-wise, then
 * (zero_mean != 0) the row/column zero-mean of S:135 computed in fp64
 * (K - rowmean - colmean + totalmean, R-13); K_out fp32 [H][W].
 * An all-zero accumulator yields K = 0 in-band (this call stays asynchronous);
 * prnu_check_results(2, sum_I2, H*W, ...) reports it as EMPTY_ACCUMULATOR.
 * ------------------------------------------------------------------------- */
size_t prnu_finalize_workspace_bytes(int H, int W);
int prnu_fingerprint_finalize(const double* sum_WI, const double* sum_I2, int H, int W, double eps,
                              int zero_mean, float* K_out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * a1-a6 fused  Fingerprint extraction — the three steps of P:58-60 ("frame
 * averaging, denoising, and noise averaging") and S:221-228.
 * frames u8 [m][H][W] (device) -> K_out fp32 [H][W], sum_WI/sum_I2 fp64
 * [H][W] (outputs, zeroed by the call), n_sda_host = floor(m/depth).
 * `batch` SDA frames are denoised per wave (1 <= batch); the result does not
 * depend on it.  depth == 1 is the conventional pipeline and is bit-identical
 * to prnu_residual + prnu_fingerprint_accumulate + prnu_fingerprint_finalize
 * on the widened frames.
 * ------------------------------------------------------------------------- */
size_t prnu_extract_workspace_bytes(int H, int W, int batch, int64_t depth, const prnu_denoise_params* p);
int prnu_extract_fingerprint(const uint8_t* frames, int64_t m, int H, int W, int64_t depth,
                             const prnu_denoise_params* p, int batch, double eps, float* K_out,
                             double* sum_WI, double* sum_I2, int64_t* n_sda_host, void* ws,
                             size_t ws_bytes, void* stream);

/* f4 I-frame emulation ("I-frames only"): stride selection.
 * Frames 0, stride, 2 stride, ... < m are denoised one by one and accumulated
 * exactly as the conventional pipeline; *n_used_host = ceil(m / stride).  The
 * workspace is prnu_extract_workspace_bytes(H, W, batch, 1, p). */
int prnu_extract_fingerprint_stride(const uint8_t* frames, int64_t m, int H, int W, int64_t stride,
                                    const prnu_denoise_params* p, int batch, double eps, float* K_out,
                                    double* sum_WI, double* sum_I2, int64_t* n_used_host, void* ws, size_t ws_bytes,
                                    void* stream);

/* Same, with the frames in (preferably page-locked) HOST memory and K written
 * to HOST memory: frames are streamed host->device in chunks of
 * `batch * depth` frames through a double-buffered staging area inside `ws`,
 * overlapped with the denoising of the previous chunk (copy stream + events
 * created internally).  Synchronous: returns after K_out_host is written.
 * sum_WI/sum_I2 are device buffers as above. */
size_t prnu_extract_host_workspace_bytes(int H, int W, int batch, int64_t depth,
                                         const prnu_denoise_params* p);
int prnu_extract_fingerprint_host(const uint8_t* frames_host, int64_t m, int H, int W, int64_t depth,
                                  const prnu_denoise_params* p, int batch, double eps,
                                  float* K_out_host, double* sum_WI, double* sum_I2,
                                  int64_t* n_sda_host, void* ws, size_t ws_bytes, void* stream);

/* Several SDA depths from ONE upload of a host frame stack (e.g. the paper's
 * depth sweeps).  The whole u8 stack [m][H][W] is copied to the
 * device workspace in chunks of 128 frames on an internal copy stream; each
 * wave of each depth waits only for the chunk holding its last frame, so the
 * upload overlaps the denoising.  Outputs: K_out_host fp32 [n_depths][H][W]
 * (host), sums fp64 [n_depths][2][H][W] (device: sum_WI then sum_I2 per depth),
 * n_sda_host int64 [n_depths] (host).  Each depth's result is bit-identical to
 * prnu_extract_fingerprint on the same frames.  Synchronous. */
size_t prnu_extract_multi_host_workspace_bytes(int64_t m, int H, int W, int batch, const int64_t* depths_host,
                                               int n_depths, const prnu_denoise_params* p);
int prnu_extract_multi_host(const uint8_t* frames_host, int64_t m, int H, int W, const int64_t* depths_host,
                            int n_depths, const prnu_denoise_params* p, int batch, double eps, float* K_out_host,
                            double* sums, int64_t* n_sda_host, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * a7  NCC — P:93, P:259 name it; S:284-287 fixes it (R-16): the Pearson
 * correlation over all pixels at shift (0,0),
 * rho = sum (a-abar)(b-bbar) / sqrt(sum (a-abar)^2 sum (b-bbar)^2),
 * two-pass, fp64 sums, fixed reduction order.  a, b fp32 [batch][H][W];
 * ncc_out fp64 [batch] (device).  A constant input yields NaN in-band (this call
 * stays asynchronous); prnu_check_results(0, ncc_out, batch, ...) reports it as
 * CONSTANT_INPUT.
 * ------------------------------------------------------------------------- */
size_t prnu_ncc_workspace_bytes(int batch, int H, int W);
int prnu_ncc(const float* a, const float* b, int batch, int H, int W, double* ncc_out, void* ws,
             size_t ws_bytes, void* stream);

/* prnu_check_results: the data-dependent error kinds of SPEC, which the
 * asynchronous calls report in-band, as a status.  SYNCHRONOUS: waits for `stream`, then
 * inspects `n` fp64 values (device) the earlier calls wrote:
 *   kind 0  NCC values (prnu_ncc)               -> PRNU_CONSTANT_INPUT if any is NaN
 *           (an operand with zero variance);
 *   kind 1  PCE peak values C[p*] (`peak` of prnu_pce*) -> PRNU_DEGENERATE_SURFACE if any
 *           is 0 (all values of the mean-removed surface equal; a zero background
 *           alone is not degenerate: that PCE is the +-1e12 cap);
 *   kind 2  sum_I2 of a fingerprint (H*W values) -> PRNU_EMPTY_ACCUMULATOR if every value
 *           is 0 (no frame contributed).
 * PRNU_OK otherwise.  Errors: INVALID_ARG (null, n < 1, unknown kind), CUDA_ERROR.         */
int prnu_check_results(int kind, const double* values, int64_t n, void* stream);

/* ---------------------------------------------------------------------------
 * a8  PCE — P:259 ("PCE ... A preset threshold of 60 ... Values higher than
 * this threshold"), formula S:293-301 / S:328-331 (R-17..R-19).
 *
 * prnu_pce_template: T[b] = K[b or 0] (.) (float)Iq[b] (R-18);
 *   K fp32 [k_batch][H][W] with k_batch in {1, batch}, Iq u8 [batch][H][W].
 * prnu_pce: for each pair b, C = circular cross-correlation of the
 *   mean-removed residual[b] and template[b] (C[dy,dx] = sum R0[y,x]
 *   T0[y-dy, x-dx], fp32; mean removal = zeroing the DC bin): for heights and
 *   widths with a compiled radix plan (720, 1080, 500, ... x 1280, 1920, 500,
 *   ...) the library's row and column FFT kernels, else cuFFT 1-D rows + the
 *   column kernel, else cuFFT R2C/C2R), peak p* = argmax |C| (ties: smallest row-major index) or (0,0) if
 *   aligned != 0; PCE = sign(C[p*]) C[p*]^2 / mean of C^2 outside the circular
 *   (2e+1)^2 neighbourhood of p* (e = exclusion_half, default 5), energies in
 *   fp64; zero background energy -> +-1e12.  Outputs (device,
 *   [batch]): pce fp64, peak_y/peak_x int32 (the shift (dy,dx)), peak fp64
 *   (C[p*] in the units of the definition above).  The decision is pce > 60
 *   (strict).
 * prnu_pce_plan_create: the plan (and cuFFT plans where used, no
 *   auto-allocation) for [batch][H][W];
 *   *ws_bytes receives the workspace prnu_pce needs.  *plan is opaque, freed
 *   by prnu_pce_plan_destroy.
 * ------------------------------------------------------------------------- */
int prnu_pce_template(const float* K, int k_batch, const uint8_t* Iq, int batch, int H, int W,
                      float* T_out, void* stream);
int prnu_pce_plan_create(int H, int W, int batch, size_t* ws_bytes, void** plan);
int prnu_pce(void* plan, const float* residual, const float* template_, int batch, int exclusion_half,
             int aligned, double* pce, int* peak_y, int* peak_x, double* peak, void* ws, size_t ws_bytes,
             void* stream);
int prnu_pce_plan_destroy(void* plan);
/* Residual-spectrum reuse (camera identification: the same query residuals against
 * many fingerprints).  prnu_pce_residual_spectrum computes FFT2 of residual
 * [batch][H][W] into the plan workspace `ws`; prnu_pce_cached then runs prnu_pce
 * for template_ against that cached spectrum (same arguments as prnu_pce without
 * `residual`), any number of times, as long as `ws` is not used for another
 * residual in between.  Results are bit-identical to prnu_pce(residual, template_). */
int prnu_pce_residual_spectrum(void* plan, const float* residual, void* ws, size_t ws_bytes, void* stream);
int prnu_pce_cached(void* plan, const float* template_, int batch, int exclusion_half, int aligned, double* pce,
                    int* peak_y, int* peak_x, double* peak, void* ws, size_t ws_bytes, void* stream);
/* prnu_pce_cached_template: prnu_pce_cached for the template K[b or 0] (.) (float)Iq[b]
 * of prnu_pce_template (R-18) without materialising it: the product is
 * formed inside the row transform when the plan has a fused row plan, else by
 * prnu_pce_template into the workspace.  K fp32 [k_batch][H][W] (k_batch in {1,
 * batch}), Iq u8 [batch][H][W] (device).  Results are bit-identical to
 * prnu_pce_cached(prnu_pce_template(K, Iq)).  Errors as prnu_pce_cached, plus
 * PRNU_DIMENSION_MISMATCH for another k_batch. */
int prnu_pce_cached_template(void* plan, const float* K, int k_batch, const uint8_t* Iq, int batch,
                             int exclusion_half, int aligned, double* pce, int* peak_y, int* peak_x, double* peak,
                             void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * f2  Wiener filtering of fingerprints in the DFT domain —
 * S:151 (an off-by-default option the paper does not specify; reading R-23).
 * For each zero-mean K [batch][H][W]:  F = DFT2(K), A = |F|/sqrt(HW),
 * s2 = mean(K^2), m = min over windows {3,5,7,9} of the mirror-extended box mean
 * of A^2 (R-7), K_out = IDFT2(F * s2 / max(m, s2)).  cuFFT R2C/C2R in fp32.
 * prnu_wdft_plan_create: cuFFT plans (no auto-allocation), *ws_bytes = the
 *   workspace prnu_wdft needs; freed by prnu_wdft_plan_destroy.
 * prnu_wdft: K and K_out device [batch][H][W] (K_out may alias K).  Errors:
 *   INVALID_ARG, PLANE_TOO_SMALL (H or W < 4), WORKSPACE_TOO_SMALL, CUDA_ERROR.
 * ------------------------------------------------------------------------- */
int prnu_wdft_plan_create(int H, int W, int batch, size_t* ws_bytes, void** plan);
int prnu_wdft(void* plan, const float* K, float* K_out, void* ws, size_t ws_bytes, void* stream);
int prnu_wdft_plan_destroy(void* plan);

/* ---------------------------------------------------------------------------
 * f1  Block-wise matching — P:266 ("divided each full resolution fingerprint
 * into 500x500 disjoint blocks"), P:321, S:275-278 (BlockGrid).
 * The H x W frame is cut into disjoint block x block tiles in row-major order
 * (edge tiles smaller, kept; n_tiles = ceil(H/block) * ceil(W/block)).  For each
 * tile: the aligned PCE (peak fixed at (0,0) of the tile's own circular
 * correlation surface of the mean-removed residual and template tiles, as
 * prnu_pce with aligned = 1) and the aligned NCC of the tile (as prnu_ncc).
 * residual, template_: fp32 [H][W] (device); pce, ncc: fp64 [n_tiles] (device).
 * prnu_block_plan_create: cuFFT plans for the (at most four) tile sizes;
 *   *n_tiles_host and *ws_bytes (host) receive the tile count and workspace.
 * ------------------------------------------------------------------------- */
int prnu_block_plan_create(int H, int W, int block, int* n_tiles_host, size_t* ws_bytes, void** plan);
int prnu_block_match(void* plan, const float* residual, const float* template_, int exclusion_half, double* pce,
                     double* ncc, void* ws, size_t ws_bytes, void* stream);
int prnu_block_plan_destroy(void* plan);

/* ---------------------------------------------------------------------------
 * f3  Denoiser variants — S:117 ("Daubechies-8 ...
 * undecimated-boundary-safe", garbled) and S:150; readings
 * R-24..R-26 of DESIGN.md.  The method of prnu_residual (decomposition, the
 * local-variance Wiener shrink of every detail subband with the params' sigma0^2
 * and mirror windows, approximation passed through, W = I - F(I)) with:
 *   taps       8 (the default 8-tap Daubechies filter) or 16 (db8, 8 vanishing
 *              moments; Daubechies 1992 Table 6.1);
 *   boundary   0: half-sample symmetric extension, expansive subbands
 *              floor((N + taps - 1)/2) (the default);  1: the plane is padded
 *              (bottom/right, half-sample symmetric) to multiples of 2^levels,
 *              transformed with periodic extension (subbands N/2), and W is
 *              cropped back to H x W;
 *   transform  0: decimated DWT;  1: undecimated (stationary) DWT — level l
 *              filters with taps dilated by 2^(l-1), no decimation, circular
 *              extension (requires boundary = 1), synthesis = adjoint / 2 per axis.
 * {8, 0, 0} is the default denoiser (same result as prnu_residual up to fp32
 * rounding; this generic path is slower).
 * planes, W_out: fp32 device [batch][H][W]; zero_mean as prnu_residual.
 * Errors: INVALID_ARG, PLANE_TOO_SMALL (H or W < 2^levels), BAD_PARAMETER
 * (params, or a variant field out of range), WORKSPACE_TOO_SMALL, CUDA_ERROR.
 * prnu_wavelet_filter: the library's lowpass filter for `taps` (8 or 16) in
 *   minimum-phase order, as the fp32 values the kernels use, widened to double
 *   (host call, no device work).
 * ------------------------------------------------------------------------- */
typedef struct {
    int taps;        /* 8 (default) or 16                        */
    int boundary;    /* 0 symmetric (default) or 1 pad + periodic */
    int transform;   /* 0 decimated (default) or 1 undecimated    */
} prnu_denoise_variant;
size_t prnu_residual_variant_workspace_bytes(int batch, int H, int W, const prnu_denoise_params* p,
                                             const prnu_denoise_variant* v);
int prnu_residual_variant(const float* planes, int batch, int H, int W, const prnu_denoise_params* p,
                          const prnu_denoise_variant* v, int zero_mean, float* W_out, void* ws, size_t ws_bytes,
                          void* stream);
/* prnu_extract_fingerprint_variant: the extraction of P:58-60 (SDA average, denoise,
 * MLE, finalize; as prnu_extract_fingerprint) with denoiser variant v (R-24 ..
 * R-26): waves of `batch` fp32 SDA frames (R-11) through prnu_residual_variant's
 * passes, accumulated in ascending group order, finalized with zero-mean.  Arguments,
 * outputs and errors as prnu_extract_fingerprint (frames u8 [m][H][W] device; K_out fp32
 * [H][W]; sum_WI / sum_I2 fp64 [H][W], zeroed by the call), plus the variant checks of
 * prnu_residual_variant; the workspace is
 * prnu_extract_variant_workspace_bytes(H, W, batch, p, v) (0 for invalid arguments).
 * Bit-identical to prnu_sda_average -> prnu_residual_variant ->
 * prnu_fingerprint_accumulate -> prnu_fingerprint_finalize over the same waves. */
size_t prnu_extract_variant_workspace_bytes(int H, int W, int batch, const prnu_denoise_params* p,
                                            const prnu_denoise_variant* v);
int prnu_extract_fingerprint_variant(const uint8_t* frames, int64_t m, int H, int W, int64_t depth,
                                     const prnu_denoise_params* p, const prnu_denoise_variant* v, int batch,
                                     double eps, float* K_out, double* sum_WI, double* sum_I2, int64_t* n_sda_host,
                                     void* ws, size_t ws_bytes, void* stream);
int prnu_wavelet_filter(int taps, double* h_out);

/* ---------------------------------------------------------------------------
 * Diagnostics.
 * prnu_last_error: thread-local text of the last failure ("" if none).
 * prnu_kernel_launches: process-wide count of kernels this library has
 *   launched (cuFFT's internal kernels excluded), for launch accounting.
 * prnu_version: library version string.
 * ------------------------------------------------------------------------- */
const char* prnu_last_error(void);
uint64_t prnu_kernel_launches(void);
const char* prnu_version(void);

/* Per-kernel timing (diagnostic, process-wide).  Between prnu_profile_begin()
 * and prnu_profile_end() every kernel launch of this library is bracketed by a
 * CUDA event pair recorded on the launching stream.  prnu_profile_end waits
 * for those events, disables timing and reports, per kernel name (at most
 * max_kernels entries; names is max_kernels * 64 bytes, NUL-terminated
 * entries): total milliseconds and launch counts; *n_kernels = number of
 * distinct names seen.  Names are "<kernel>_l<level>" for per-level kernels. */
int prnu_profile_begin(void);
int prnu_profile_end(int max_kernels, char* names, double* ms_total, int64_t* launches, int* n_kernels);

#ifdef __cplusplus
}
#endif
#endif /* PRNU_H */
