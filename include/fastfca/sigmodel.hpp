// sigmodel.hpp -- observation statistics and parameter containers of the
// FastFCA C++ API (reference proj/include/fastfca/sigmodel.hpp:19-111).
//
// block_size == 1 keeps the snapshots the GPU fit reads.  Deviation: for
// block_size == 1 sample_covs does not materialise the per-(i, j) rank-one
// matrices `mats` (F*T M x M heap matrices, ~17 GB at BASELINE config 3); the
// reference's hot path never reads them when snapshots exist
// (fastfca.cpp:25-28, sigmodel.cpp:95-96).  block_size B > 1 fills `mats`
// with the B-frame block covariances (computed on the GPU) and the fit runs
// the block-stationary kernels on them.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "fastfca/stft.hpp"
#include "fastfca/types.hpp"

namespace fastfca {

constexpr double kPowerFloorRel = 1e-12;  // sigmodel.hpp:19
constexpr double kVarEpsRel = 1e-8;       // sigmodel.hpp:26

inline double var_eps(double data_power) {  // sigmodel.hpp:29-31
  return std::max(kVarEpsRel * data_power, 1e-300);
}

struct FitOptions {  // sigmodel.hpp:34-38
  int workers = 1;             // host threads (layout conversion); devices: GpuOptions
  bool record_trace = true;    // benchmark runs disable this
  std::uint64_t seed = 0;      // recovery restarts only
};

struct SampleCovSet {  // sigmodel.hpp:48-56
  int dim = 0, bins = 0, blocks = 0, frames = 0, block_size = 1;
  std::vector<std::vector<CMat>> mats;  // [i][jb], block_size > 1 (see header note)
  std::vector<CMat> snapshots;          // [i], dim x frames (block_size == 1)
  RVec power_scale;                     // [i], mean per-channel data power
  bool has_snapshots() const { return !snapshots.empty(); }
  double power(int i) const {  // sigmodel.cpp:50-55
    if (i < long(power_scale.size())) return power_scale(i);
    double trace_sum = 0.0;
    for (const CMat& m : mats[i])
      for (long k = 0; k < m.rows(); ++k) trace_sum += std::real(m(k, k));
    return trace_sum / (static_cast<double>(blocks) * dim);
  }
};

// sample_covs (sigmodel.cpp:17-48) on the GPU: snapshots + power_scale for
// block_size == 1; the block covariances `mats` + power_scale for B > 1.
SampleCovSet sample_covs(const Spectrogram& spec, int block_size = 1);

struct FastFcaParams {  // sigmodel.hpp:72-78
  int dim = 0, bins = 0, frames = 0, sources = 0;
  std::vector<CMat> decorr;
  std::vector<RMat> loading;
  std::vector<RMat> act;
  // Shape / finiteness / positivity / non-singular-W check with the
  // reference's std::invalid_argument and NumericalError (sigmodel.cpp:74-91);
  // the determinant test runs on the GPU (log_abs_det2).
  void validate() const;
};

// ln|det W|^2 (sigmodel.cpp:118-129) on the GPU; NumericalError when W is
// numerically singular.
double log_abs_det2(const CMat& w);

// Negative log-likelihood (sigmodel.cpp:155-162, 215-222) evaluated on the GPU
// in fp64 (check-mode kernels); per-bin values are summed in bin order.
double fastfca_nll(const SampleCovSet& covs, const FastFcaParams& params);
// |W^H x|^2 of bin i (sigmodel.cpp:93-107), on the GPU (fp64).
RMat decorrelated_powers(const SampleCovSet& covs, int i, const CMat& w);
double fastfca_nll_freq(const SampleCovSet& covs, int i, const CMat& w, const RMat& loading,
                        const RMat& act);

// Expands block-level parameters to frame level (sigmodel.hpp:96-101,
// sigmodel.cpp:164-196): column j of H takes block min(j / B, blocks - 1).
FastFcaParams expand_block_params(const FastFcaParams& params, int block_size, int frames);

}  // namespace fastfca
