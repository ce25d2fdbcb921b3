/* ffca.h -- C ABI of the B200-native FastFCA hot path (libffca.so).
 *
 * Drop-in boundary for the reference's fit / separate entry points
 * (reference proj/include/fastfca/fastfca.hpp:55-66, sigmodel.hpp:58,104).
 * The reference is a C++ library with no FFI of its own; these entry points
 * are what its C++ API (re-exposed in include/fastfca/, implemented in
 * paper_2101_08563_b200/csrc/shim.cpp on top of this ABI) and any ctypes /
 * cgo / JNI binding call.  Plain pointers and sizes only.
 *
 * Host layouts are the reference containers' (Eigen column-major):
 *   x       [batch][bins][frames][dim]   complex (re, im doubles)  Spectrogram::f[i]
 *   W       [batch][bins][dim*dim]       complex, W(r,c) at r + c*dim  FastFcaParams::decorr
 *   L       [batch][bins][dim*sources]   real,    L(m,n) at m + n*dim  FastFcaParams::loading
 *   H       [batch][bins][sources*frames] real,   H(n,j) at n + j*sources  FastFcaParams::act
 *   images  [sources][batch][bins][frames][dim] complex              fastfca_separate output
 *
 * Every function returns a status: FFCA_OK, FFCA_INVALID_ARGUMENT (the
 * reference's std::invalid_argument), FFCA_NUMERICAL (NumericalError,
 * types.hpp:21-24) or FFCA_CUDA_ERROR.  ffca_last_error() returns the message
 * of the calling thread's last failure.  There is no CPU fallback: without a
 * usable sm_100 device every compute entry point fails with FFCA_CUDA_ERROR.
 */
#ifndef FFCA_H_
#define FFCA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFCA_OK 0
#define FFCA_INVALID_ARGUMENT 1
#define FFCA_NUMERICAL 2
#define FFCA_CUDA_ERROR 3

#define FFCA_FLAVOR_EM 0 /* LhFlavor::em (fastfca.hpp:16) */
#define FFCA_FLAVOR_MM 1 /* LhFlavor::mm */

#define FFCA_PREC_FP32 0 /* complex64 / fp32 data path, fp64 reductions and solves */
#define FFCA_PREC_FP64 1 /* fp64 check mode */

#define FFCA_STFT_CENTERED 0    /* StftPadding::centered (stft.hpp:30-37) */
#define FFCA_STFT_FULL_FRAMES 1 /* StftPadding::full_frames */

/* Per-bin status words written by the fit. */
#define FFCA_BIN_OK 0
#define FFCA_BIN_SILENT 1       /* power(i) <= 0: init kept (fastfca.cpp:165-170) */
#define FFCA_BIN_IP_SINGULAR 2  /* ip_update_w failed after its restart (fastfca.cpp:63-65); column in bits 8.. */
#define FFCA_BIN_SINGULAR_W 3   /* log_abs_det2 on a singular W (sigmodel.cpp:124-125) */

typedef struct ffca_ctx ffca_ctx;

typedef struct {
  int batch;   /* independent mixtures (1 for the reference API) */
  int bins;    /* F */
  int dim;     /* M, 1..8 */
  int sources; /* N, 1..16 */
  int frames;  /* T */
  /* Restart-seed numbering (fastfca.cpp:40 seeds bin i with mix_seed(seed+t, i)):
   * when the call covers bins [first_bin, first_bin + bins) of a mixture with
   * mixture_bins bins (frequency sharding), pass them so restarts draw the
   * reference's streams.  0 / 0 for a whole mixture. */
  int first_bin;
  int mixture_bins;
} ffca_dims;

typedef struct {
  int flavor;           /* FFCA_FLAVOR_EM / _MM                    (LhFlavor) */
  int iters;            /* >= 0                                   (fastfca_fit iters) */
  int record_trace;     /* FitOptions::record_trace (sigmodel.hpp:36) */
  uint64_t seed;        /* FitOptions::seed (restart seeds only) */
  int normalize_scales; /* FastFcaOptions::normalize_scales (fastfca.hpp:20) */
  int fix_loadings;     /* FastFcaOptions::fix_loadings (fastfca.hpp:19) */
  int precision;        /* FFCA_PREC_FP32 / FFCA_PREC_FP64 */
} ffca_fit_opts;

/* Library identity / build info. */
int ffca_version(void);
const char* ffca_last_error(void);
int ffca_device_count(void);

/* A context owns one CUDA device's stream and grow-only device buffers.  Not
 * thread-safe: use one per host thread (the reference's fit is a reentrant
 * pure function; the C++ shim creates one context per device). */
int ffca_ctx_create(int device, ffca_ctx** out);
void ffca_ctx_destroy(ffca_ctx* ctx);

/* Page-locked host staging owned by the context (slots 0..7, grow-only, freed
 * with the context).  Host buffers passed to ffca_fit from such memory make
 * its chunked H2D / fit / D2H pipeline asynchronous; any host memory works,
 * pageable buffers just serialise the copies.  NULL on failure. */
void* ffca_pinned_buffer(ffca_ctx* ctx, int slot, size_t bytes);

/* fastfca_fit (fastfca.hpp:55-58, fastfca.cpp:146-191) over `batch`
 * independent mixtures.  W, L, H are the init on entry and the fitted
 * parameters on return (silent bins and iters == 0 keep the init bit-exactly).
 * power: SampleCovSet::power_scale [batch][bins], or NULL to compute it from x
 * (sample_covs, sigmodel.cpp:17-48).  nll: [batch][iters+1] trace (bin-order
 * sums of the per-bin slots, fastfca.cpp:186-189), required when
 * record_trace; nll_slots (nullable): [batch][iters+1][bins]; bin_status
 * (nullable): [batch][bins].  On FFCA_NUMERICAL the contents of W, L, H are
 * unspecified (the pipelined path has copied partial results back by then). */
int ffca_fit(ffca_ctx* ctx, const ffca_dims* dims, const ffca_fit_opts* opts, const double* x,
             const double* power, double* W, double* L, double* H, double* nll,
             double* nll_slots, int32_t* bin_status);

/* ffca_fit on PER-BIN host buffers -- what a caller holding the reference's
 * containers has (one allocation per bin: Spectrogram::f[i],
 * FastFcaParams::decorr[i] / loading[i] / act[i]).  x_bins, W_in, L_in, H_in,
 * W_out, L_out, H_out: arrays of batch*bins pointers, each bin in the layout
 * of ffca_fit (in and out may alias).  The library gathers bin chunks into
 * page-locked staging on `host_threads` host threads (<= 0: hardware
 * concurrency, at most 16) and pipelines gather / H2D / fit / D2H / scatter
 * over the chunks.  Results equal ffca_fit's bit for bit.  On FFCA_NUMERICAL
 * the outputs are unspecified. */
int ffca_fit_bins(ffca_ctx* ctx, const ffca_dims* dims, const ffca_fit_opts* opts,
                  const double* const* x_bins, const double* power, const double* const* W_in,
                  const double* const* L_in, const double* const* H_in, double* const* W_out,
                  double* const* L_out, double* const* H_out, double* nll, double* nll_slots,
                  int32_t* bin_status, int host_threads);

/* ica_mode_fit (fastfca.hpp:76-78, fastfca.cpp:241-264): determined ICA mode.
 * dims->sources must equal dims->dim (else FFCA_INVALID_ARGUMENT with the
 * reference's message).  W: w_init on entry, the fitted W on return; L, H are
 * outputs only (L = identity, H = floored decorrelated powers of w_init, then
 * IP+MM with the loadings fixed).  opts->flavor / fix_loadings /
 * normalize_scales are ignored (the mode fixes them), and so is
 * opts->precision: this mode always runs the fp64 kernels (at its fixed point
 * H tracks |w^H x|^2 and the 1/H weights amplify fp32 cancellation, so an
 * fp32 trajectory cannot follow the reference's).  The rest as ffca_fit. */
int ffca_ica_fit(ffca_ctx* ctx, const ffca_dims* dims, const ffca_fit_opts* opts, const double* x,
                 const double* power, double* W, double* L, double* H, double* nll,
                 double* nll_slots, int32_t* bin_status);

/* ---- block-stationary input (SampleCovSet with block_size B > 1) ----
 * sample_covs(spec, B) / piecewise_prepare (sigmodel.cpp:17-48,
 * fastfca.cpp:266-268): the F x J block covariances mats[i][jb] = (1/width)
 * sum x x^H over B consecutive frames (J = ceil(T/B), the last block ragged).
 * Host layout of `mats`: [batch][bins][blocks][dim*dim] complex (re, im
 * doubles), each block an Eigen col-major dim x dim matrix (X(r,c) at
 * r + c*dim) -- SampleCovSet::mats[i][jb].  The *_covs entry points take
 * such a set (dims->frames = J blocks) and run the same kernels as their
 * snapshot counterparts on packed Hermitian records (weighted_cov
 * fastfca.cpp:29-32, decorrelated_powers sigmodel.cpp:97-105). */

/* sample_covs(spec, block_size): x as in ffca_fit (dims->frames = T); mats
 * (nullable) [batch][bins][J][dim*dim]; power (nullable) [batch][bins] =
 * SampleCovSet::power_scale (sigmodel.cpp:43-44). */
int ffca_block_covs(ffca_ctx* ctx, const ffca_dims* dims, int block_size, const double* x,
                    double* mats, double* power);

/* fastfca_fit / ica_mode_fit on block covariances (dims->frames = J); H is
 * sources x J per bin.  power may be NULL: SampleCovSet::power() then falls
 * back to the block traces (sigmodel.cpp:50-55). */
int ffca_fit_covs(ffca_ctx* ctx, const ffca_dims* dims, const ffca_fit_opts* opts,
                  const double* mats, const double* power, double* W, double* L, double* H,
                  double* nll, double* nll_slots, int32_t* bin_status);
int ffca_ica_fit_covs(ffca_ctx* ctx, const ffca_dims* dims, const ffca_fit_opts* opts,
                      const double* mats, const double* power, double* W, double* L, double* H,
                      double* nll, double* nll_slots, int32_t* bin_status);

/* fastfca_nll_freq per bin and decorrelated_powers (max(0, Re w^H X w),
 * floored when floor_rel >= 0) on block covariances. */
int ffca_nll_bins_covs(ffca_ctx* ctx, const ffca_dims* dims, int precision, const double* mats,
                       const double* W, const double* L, const double* H, double* out);
int ffca_decorrelated_powers_covs(ffca_ctx* ctx, const ffca_dims* dims, int precision,
                                  const double* mats, const double* W, double floor_rel,
                                  double* out);

/* decorrelated_powers (sigmodel.cpp:93-107): out [batch][bins][frames][dim]
 * = |W^H x|^2 per bin (the Eigen col-major dim x frames matrix), floored as
 * floor_positive(u, floor_rel) (sigmodel.cpp:10-15) when floor_rel >= 0. */
int ffca_decorrelated_powers(ffca_ctx* ctx, const ffca_dims* dims, int precision, const double* x,
                             const double* W, double floor_rel, double* out);

/* fastfca_separate (fastfca.hpp:65-66, fastfca.cpp:205-223). */
int ffca_separate(ffca_ctx* ctx, const ffca_dims* dims, int precision, const double* x,
                  const double* W, const double* L, const double* H, double* images);

/* fastfca_nll_freq per bin (sigmodel.cpp:155-162): out [batch][bins]. */
int ffca_nll_bins(ffca_ctx* ctx, const ffca_dims* dims, int precision, const double* x,
                  const double* W, const double* L, const double* H, double* out);

/* SampleCovSet::power_scale (sigmodel.cpp:43-44): out [batch][bins]. */
int ffca_power_scale(ffca_ctx* ctx, const ffca_dims* dims, const double* x, double* out);

/* ---- device-resident entry points (inputs already in HBM; used for the
 * frequency-sharded multi-GPU path and the device-timed benchmark) ----
 * Device layouts keep the reference's per-bin (frame-major) order, so the
 * boundary only converts precision:
 * x_dev  : [P][frames][dim] complex64 (fp32) or complex128 (fp64)
 * H_dev  : [P][frames][sources] fp32 / fp64, in/out
 * W, L   : [P][dim*dim] complex128, [P][dim*sources] fp64, in/out
 * power  : [P] fp64;  nll_slots: [(iters+1)][P] fp64 or NULL;  status: [P]
 * P = batch*bins problems; prob_offset = global index of problem 0 (only the
 * restart seed uses it: bin index i = (prob_offset + p) % bins_per_mixture).
 * stream: a cudaStream_t (NULL = the context's stream).  Asynchronous. */
int ffca_fit_device(ffca_ctx* ctx, int problems, int bins_per_mixture, int prob_offset, int dim,
                    int sources, int frames, const ffca_fit_opts* opts, const void* x_dev,
                    const double* power, double* W, double* L, void* H_dev, double* nll_slots,
                    int32_t* status, void* stream);

/* Block-stationary device path.  rec_dev: [P][blocks][dim*dim] packed
 * Hermitian records in the compute type (fp32 / fp64 by precision):
 * [a*dim+a] = X_aa, [a*dim+c] = Re X_ac, [c*dim+a] = Im X_ac for a < c.
 * ffca_block_covs_device builds them from device x [P][frames][dim]
 * (sample_covs with block_size, blocks = ceil(frames/block_size)) and writes
 * power_scale into power (nullable); ffca_fit_covs_device is
 * ffca_fit_device on them (H_dev [P][blocks][sources]). */
int ffca_block_covs_device(ffca_ctx* ctx, int problems, int dim, int frames, int block_size,
                           int precision, const void* x_dev, void* rec_dev, double* power,
                           void* stream);
int ffca_fit_covs_device(ffca_ctx* ctx, int problems, int bins_per_mixture, int prob_offset,
                         int dim, int sources, int blocks, const ffca_fit_opts* opts,
                         const void* rec_dev, const double* power, double* W, double* L,
                         void* H_dev, double* nll_slots, int32_t* status, void* stream);

/* images_dev: [sources][P][frames][dim] complex64 / complex128. */
int ffca_separate_device(ffca_ctx* ctx, int problems, int dim, int sources, int frames,
                         int precision, const void* x_dev, const double* W, const double* L,
                         const void* H_dev, void* images_dev, void* stream);

/* power_scale from device x (complex64/complex128, [P][frames][dim]): out [P]. */
int ffca_power_scale_device(ffca_ctx* ctx, int problems, int dim, int frames, int precision,
                            const void* x_dev, double* out, void* stream);

/* ---- STFT front end / iSTFT back end (stft.hpp:40-56, stft.cpp:12-128) ----
 * sqrt-Hann window, 50 % overlap (shift == frame_len / 2, frame_len a power
 * of two <= 4096), fp64 FFTs on the GPU.  Layouts are the reference's:
 * samples [length][channels] (MultichannelWave::samples, Eigen col-major
 * channels x length); spec [bins][frames][channels] (Spectrogram::f[b]) with
 * bins = frame_len/2 + 1 -- which is also the fit's x layout [P][T][M], so
 * ffca_stft_device output feeds ffca_fit_device directly. */

/* stft_frame_count (stft.cpp:41-49); -1 (and ffca_last_error) on error. */
long long ffca_stft_frame_count(long long length, int frame_len, int shift, int padding);

/* stft (stft.cpp:51-83): spec [bins][frames][channels] complex128. */
int ffca_stft(ffca_ctx* ctx, int channels, long long length, int frame_len, int shift, int padding,
              const double* samples, double* spec);

/* istft (stft.cpp:85-128): samples [out_len][channels]. */
int ffca_istft(ffca_ctx* ctx, int channels, int bins, int frames, int frame_len, int shift,
               int padding, long long out_len, const double* spec, double* samples);

/* Device-resident variants: samples fp32/fp64 and spec complex64/complex128
 * by `precision` (the FFTs themselves run in fp64); asynchronous on stream. */
int ffca_stft_device(ffca_ctx* ctx, int channels, long long length, int frame_len, int shift,
                     int padding, int precision, const void* samples_dev, void* x_dev,
                     void* stream);
int ffca_istft_device(ffca_ctx* ctx, int channels, int frames, int frame_len, int shift,
                      int padding, long long out_len, int precision, const void* spec_dev,
                      void* samples_dev, void* stream);

/* ---- the reference's public per-step functions, one bin per call ----
 * (fastfca.hpp:30-53; its unit tests call them directly,
 * test_fastfca.cpp:82-228).  fp64 throughout, a few small launches each: the
 * fit kernels fuse these steps, these entry points expose them one by one.
 * x: the bin's snapshots [blocks][dim] complex (is_block_covs == 0) or its
 * block covariances [blocks][dim*dim] col-major (is_block_covs != 0). */

/* weighted_cov (fastfca.cpp:22-34): q [dim*dim] complex col-major =
 * symmetrize((1/blocks) sum_j X_j / sigma2_row[j]). */
int ffca_weighted_cov(ffca_ctx* ctx, int dim, int blocks, int is_block_covs, const double* x,
                      const double* sigma2_row, double* q);

/* ip_update_w (fastfca.cpp:36-72): one IP sweep over the columns of w
 * (in/out, dim*dim complex col-major) with sigma^2 = loading*act +
 * var_eps(power); restart draws follow mix_seed(restart_seed, bin_index).
 * FFCA_NUMERICAL with the reference's message when a column stays singular
 * after its restart (w is then left unchanged). */
int ffca_ip_update_w(ffca_ctx* ctx, int dim, int sources, int blocks, int is_block_covs,
                     const double* x, double power, double* w, const double* loading,
                     const double* act, uint64_t restart_seed, int bin_index);

/* log_abs_det2 (sigmodel.cpp:118-129): *out = ln|det w|^2; FFCA_NUMERICAL
 * ("singular decorrelation matrix") when a pivot is zero or non-finite. */
int ffca_log_abs_det2(ffca_ctx* ctx, int dim, const double* w, double* out);

/* fastfca_mwf (fastfca.cpp:193-203): out [dim*dim] complex col-major =
 * W^-H diag(gains) W^H for source n at one frame; act_col = H(:, j). */
int ffca_mwf(ffca_ctx* ctx, int dim, int sources, const double* w, const double* loading,
             const double* act_col, int n, double* out);

/* reconstruct_scms (fastfca.cpp:270-282): out [bins][sources][dim*dim] complex
 * col-major, R_in = W^-H Lambda_n W^-1. */
int ffca_reconstruct_scms(ffca_ctx* ctx, int bins, int dim, int sources, const double* W,
                          const double* L, double* out);

/* ajd_cost (fastfca.cpp:225-239): *out = sum_j alpha_j D_LD(W^H X_j W |
 * ddiag(.)) over one bin's block covariances mats [blocks][dim*dim]; weights
 * (nullable) [blocks].  FFCA_NUMERICAL when a transformed covariance is not
 * positive definite (hermitian.hpp:93-94). */
int ffca_ajd_cost(ffca_ctx* ctx, int dim, int blocks, const double* mats, const double* w,
                  const double* weights, double* out);

/* source_gain (fastfca.cpp:74-78): gain [dim x frames] col-major =
 * L(:,n) H(n,:) / floor_positive(L H). */
int ffca_source_gain(ffca_ctx* ctx, int dim, int sources, int frames, const double* loading,
                     const double* act, int n, double* gain);

/* em_update_lh / mm_update_lh (fastfca.cpp:80-117): u [dim x frames]
 * col-major decorrelated powers; loading, act in/out. */
int ffca_em_update_lh(ffca_ctx* ctx, int dim, int sources, int frames, const double* u,
                      double* loading, double* act, int update_loading, double eps);
int ffca_mm_update_lh(ffca_ctx* ctx, int dim, int sources, int frames, const double* u,
                      double* loading, double* act, int update_loading, double eps);

/* Number of kernels the last call on this context launched (bench evidence). */
int ffca_last_launch_count(const ffca_ctx* ctx);

/* Diagnostics: the IP restart generator as the device runs it (fastfca.cpp:
 * 13-18, 40-41: std::mt19937_64 seeded with mix_seed(seed, bin_index) feeding
 * std::normal_distribution<double>): n raw 64-bit draws and n normal draws
 * of a freshly seeded generator; *mixed_seed (nullable) = mix_seed. */
int ffca_debug_restart_draws(ffca_ctx* ctx, uint64_t seed, int bin_index, int n,
                             uint64_t* mixed_seed, uint64_t* raw, double* normals);

/* Diagnostics: subsequent ffca_fit_device launches on this context record
 * per-problem phase cycle counters into dev_counters ([P][16] uint64, device
 * memory; NULL disables). */
int ffca_debug_set_timing(ffca_ctx* ctx, unsigned long long* dev_counters);

#ifdef __cplusplus
}
#endif

#endif /* FFCA_H_ */
