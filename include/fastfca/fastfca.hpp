// fastfca.hpp -- the FastFCA fit / separate entry points, B200 backend
// (drop-in for reference proj/include/fastfca/fastfca.hpp:16-84: every
// function the reference header declares).
//
// Same names, argument order, defaults and error behaviour as the reference:
// std::invalid_argument on shape mismatch, NumericalError on a singular IP
// system after its restart or a singular W, `init` copied, `iters == 0` and
// silent bands return the init bit-exactly, record_trace == false returns an
// empty trace.  Every call runs the sm_100a kernels of libffca.so (no CPU
// fallback).  The appended GpuOptions overloads select devices (frequency
// sharding over several GPUs, one host thread per device) and the arithmetic
// (fp32 data path, or the fp64 check mode).
#pragma once

#include <cstdint>
#include <vector>

#include "fastfca/sigmodel.hpp"

namespace fastfca {

enum class LhFlavor { em, mm };  // fastfca.hpp:16

struct FastFcaOptions {  // fastfca.hpp:18-21
  bool fix_loadings = false;
  bool normalize_scales = true;
};

struct FastFcaFitResult {  // fastfca.hpp:23-26
  FastFcaParams params;
  std::vector<double> nll;  // nll[0] at init, then one entry per iteration
};

enum class Precision { fp32, fp64 };

struct GpuOptions {
  std::vector<int> devices = {0};  // bins are split into contiguous ranges, one per device
  Precision precision = Precision::fp32;
  int host_threads = 0;  // container <-> staging copies; 0 = hardware concurrency (at most 16)
};

// The per-step functions (fastfca.hpp:28-53), each a single-bin fp64 launch
// of libffca.so (csrc/steps.cu); the fit kernels fuse the same steps.
// weighted_cov: Q_m = symmetrize((1/J) sum_j Xhat_j / sigma2_mj) at frequency
// i (fastfca.cpp:22-34; sigma2_row is 1 x blocks).
CMat weighted_cov(const SampleCovSet& covs, int i, const RMat& sigma2_row);
// One IP sweep over the columns of W at frequency i (fastfca.cpp:36-72):
// seeded single restart of a singular column, then NumericalError.
void ip_update_w(const SampleCovSet& covs, int i, CMat& w, const RMat& loading, const RMat& act,
                 std::uint64_t restart_seed = 0);
// G_n = (L_{:,n} H_{n,:}) / floor_positive(L H) (fastfca.cpp:74-78).
RMat source_gain(const RMat& loading, const RMat& act, int n);
// IS-NMF updates of (L, H) against the decorrelated powers U: per source with
// the running factors (EM, fastfca.cpp:80-99) or whole-matrix multiplicative
// steps, L first (MM, fastfca.cpp:101-117).
void em_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading = true,
                  double eps = 0.0);
void mm_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading = true,
                  double eps = 0.0);

// The reference signatures run the fp32 data path (GpuOptions{}); pass
// GpuOptions{.precision = Precision::fp64} for the reference's arithmetic
// (IP residual test at 1e-8 instead of 64 FLT_EPSILON).
FastFcaFitResult fastfca_fit(const SampleCovSet& covs, const FastFcaParams& init, LhFlavor flavor,
                             int iters, const FitOptions& fit = {},
                             const FastFcaOptions& opts = {});
FastFcaFitResult fastfca_fit(const SampleCovSet& covs, const FastFcaParams& init, LhFlavor flavor,
                             int iters, const FitOptions& fit, const FastFcaOptions& opts,
                             const GpuOptions& gpu);

// A batch of independent mixtures in one launch; equal to a loop of fastfca_fit.
std::vector<FastFcaFitResult> fastfca_fit_batch(const std::vector<SampleCovSet>& covs,
                                                const std::vector<FastFcaParams>& init,
                                                LhFlavor flavor, int iters,
                                                const FitOptions& fit = {},
                                                const FastFcaOptions& opts = {},
                                                const GpuOptions& gpu = {});

// Determined ICA mode (fastfca.hpp:76-78, fastfca.cpp:241-264): sources ==
// dim, L = identity, H = floored decorrelated powers of w_init (computed on
// the GPU), then IP+MM with the loadings fixed.
FastFcaFitResult ica_mode_fit(const SampleCovSet& covs, int sources, int iters,
                              const std::vector<CMat>& w_init, const FitOptions& fit = {});
// gpu.precision is ignored here: the ICA mode always computes in fp64.
FastFcaFitResult ica_mode_fit(const SampleCovSet& covs, int sources, int iters,
                              const std::vector<CMat>& w_init, const FitOptions& fit,
                              const GpuOptions& gpu);

// Block-stationary statistics; block_size == 1 reproduces sample_covs
// (fastfca.hpp:80-81, fastfca.cpp:266-268).
SampleCovSet piecewise_prepare(const Spectrogram& spec, int block_size);

// Decomposed Wiener filter W^-H diag(gains) W^H at one (i, j, n)
// (fastfca.hpp:60-61, fastfca.cpp:193-203).
CMat fastfca_mwf(const FastFcaParams& params, int i, int j, int n);

// Joint-diagonality cost sum_j alpha_j D_LD(W^H Xhat_j W | ddiag(...))
// (fastfca.hpp:68-71, fastfca.cpp:225-239).  Empty weights mean alpha_j = 1;
// needs the block covariances (`mats`) and throws NumericalError when a
// transformed covariance is not positive definite.
double ajd_cost(const CMat& w, const SampleCovSet& covs, int i, const RVec& weights = RVec());

// R_in = W^-H Lambda_n W^-1 (fastfca.hpp:83-84, fastfca.cpp:270-282).
std::vector<std::vector<CMat>> reconstruct_scms(const FastFcaParams& params);

// Decomposed multichannel Wiener filter (fastfca.cpp:205-223).
std::vector<Spectrogram> fastfca_separate(const Spectrogram& spec, const FastFcaParams& params);
std::vector<Spectrogram> fastfca_separate(const Spectrogram& spec, const FastFcaParams& params,
                                          const GpuOptions& gpu);

}  // namespace fastfca
