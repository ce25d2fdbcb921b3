// oracle.hpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Eigen-free fp64 C++20 restatement of the reference FastFCA hot path
// (arxiv 2101.08563, reference tree /root/reference/proj).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it, and only as the checker or the timed CPU baseline.
//
// Every function cites the reference file:line it restates.  The reference
// itself cannot be compiled here (Eigen3 and doctest are absent; see
// DESIGN.md "Oracle"), so this restatement is pinned by porting the
// reference's own known-answer and property tests (oracle/kat_tests.cpp,
// run by tests/test_oracle_kat.py).  Full-trajectory parity at BASELINE sizes
// is not pinned by any stored reference output ("parity unpinned" for full
// trajectories; pinned by KATs for the kernels).
//
// Layouts follow Eigen's defaults (column major), exactly what the
// reference's containers hold:
//   X  (dim x frames, complex)   element (m, j) at m + j*dim
//   W  (dim x dim, complex)      element (r, c) at r + c*dim
//   L  (dim x sources, real)     element (m, n) at m + n*dim
//   H  (sources x frames, real)  element (n, j) at n + j*sources

#pragma once

#include <complex>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Complex = std::complex<double>;

// Minimal column-major dense matrix (same element order as Eigen::MatrixX*).
template <typename T>
struct Mat {
  int r = 0, c = 0;
  std::vector<T> a;
  Mat() = default;
  Mat(int rows, int cols, T v = T(0)) : r(rows), c(cols), a(size_t(rows) * cols, v) {}
  T& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  const T& operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
  int rows() const { return r; }
  int cols() const { return c; }
  T* data() { return a.data(); }
  const T* data() const { return a.data(); }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = T(1);
    return m;
  }
};
using CMat = Mat<Complex>;
using RMat = Mat<double>;

// types.hpp:21-24
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};

// sigmodel.hpp:19, :26-31
constexpr double kPowerFloorRel = 1e-12;
#ifndef ORACLE_VAR_EPS_REL
#define ORACLE_VAR_EPS_REL 1e-8
#endif
constexpr double kVarEpsRel = ORACLE_VAR_EPS_REL;
inline double var_eps(double p) { return std::max(kVarEpsRel * p, 1e-300); }

enum class LhFlavor { em, mm };  // fastfca.hpp:16

struct FitOptions {  // sigmodel.hpp:34-38
  int workers = 1;
  bool record_trace = true;
  std::uint64_t seed = 0;
};
struct FastFcaOptions {  // fastfca.hpp:18-21
  bool fix_loadings = false;
  bool normalize_scales = true;
};

// SampleCovSet (sigmodel.hpp:48-56).  block_size == 1 keeps the snapshots
// the hot path reads (fastfca.cpp:25-28, sigmodel.cpp:95-96) and builds the
// rank-one `mats` only on request (sample_covs(..., with_mats)); block_size
// B > 1 stores the block covariances mats[i][jb] = (1/width) sum x x^H over
// B consecutive frames (sigmodel.cpp:34-41), the block-stationary input of
// weighted_cov / decorrelated_powers (fastfca.cpp:29-32, sigmodel.cpp:98-105).
struct SampleCovSet {
  int dim = 0, bins = 0, blocks = 0, frames = 0, block_size = 1;
  std::vector<std::vector<CMat>> mats;  // [i][jb], dim x dim
  std::vector<CMat> snapshots;          // [i], dim x frames (block_size == 1)
  std::vector<double> power_scale;      // [i]
  bool has_snapshots() const { return !snapshots.empty(); }
  double power(int i) const;            // sigmodel.cpp:50-55
};

struct FastFcaParams {  // sigmodel.hpp:72-78
  int dim = 0, bins = 0, frames = 0, sources = 0;
  std::vector<CMat> decorr;
  std::vector<RMat> loading;
  std::vector<RMat> act;
};

struct FastFcaFitResult {  // fastfca.hpp:23-26
  FastFcaParams params;
  std::vector<double> nll;
};

// ---- linear algebra helpers (Eigen::PartialPivLU / LLT equivalents) ----
struct PartialPivLU {
  CMat lu;
  std::vector<int> perm;  // row permutation: row k of P*A is row perm[k] of A
  explicit PartialPivLU(const CMat& a);
  std::vector<Complex> solve(const std::vector<Complex>& b) const;
  CMat solve(const CMat& b) const;
  CMat inverse() const;
};

CMat adjoint(const CMat& a);
CMat matmul(const CMat& a, const CMat& b);
RMat matmul(const RMat& a, const RMat& b);
double frob(const CMat& a);

// ---- hot-path restatement ----
void floor_positive(RMat& m, double rel = kPowerFloorRel);         // sigmodel.cpp:10-15
SampleCovSet sample_covs(int dim, int bins, int frames, const Complex* x, int block_size = 1,
                         bool with_mats = false);                   // sigmodel.cpp:17-48
// piecewise_prepare (fastfca.cpp:266-268) == sample_covs(spec, block_size), mats included.
SampleCovSet piecewise_prepare(int dim, int bins, int frames, const Complex* x, int block_size);
// expand_block_params (sigmodel.cpp:164-196): block-level H -> frame level.
FastFcaParams expand_block_params(const FastFcaParams& p, int block_size, int frames);
CMat weighted_cov(const SampleCovSet& covs, int i, const double* sigma2_row,
                  int stride);                                     // fastfca.cpp:22-34
void ip_update_w(const SampleCovSet& covs, int i, CMat& w, const RMat& loading,
                 const RMat& act, std::uint64_t restart_seed = 0);  // fastfca.cpp:36-72
RMat source_gain(const RMat& loading, const RMat& act, int n);     // fastfca.cpp:74-78
void em_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading = true,
                  double eps = 0.0);                               // fastfca.cpp:80-99
void mm_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading = true,
                  double eps = 0.0);                               // fastfca.cpp:101-117
void balance_scales(CMat& w, RMat& loading, RMat& act);            // fastfca.cpp:127-142
RMat decorrelated_powers(const SampleCovSet& covs, int i, const CMat& w);  // sigmodel.cpp:93-107
double log_abs_det2(const CMat& w);                                // sigmodel.cpp:118-129
double fastfca_nll_freq(const SampleCovSet& covs, int i, const CMat& w, const RMat& loading,
                        const RMat& act);                          // sigmodel.cpp:155-162
double fastfca_nll(const SampleCovSet& covs, const FastFcaParams& p);  // sigmodel.cpp:215-222
double fca_nll_freq(const SampleCovSet& covs, int i, const std::vector<CMat>& scm_i,
                    const RMat& power_i);                          // sigmodel.cpp:131-153
std::vector<std::vector<CMat>> reconstruct_scms(const FastFcaParams& p);  // fastfca.cpp:270-282
FastFcaFitResult fastfca_fit(const SampleCovSet& covs, const FastFcaParams& init,
                             LhFlavor flavor, int iters, const FitOptions& fit = {},
                             const FastFcaOptions& opts = {},
                             std::vector<double>* slots_out = nullptr);  // fastfca.cpp:146-191
// slots_out (optional): the per-bin nll_slots matrix, [(iters+1)][bins]
// (fastfca.cpp:155-156), which the driver sums in bin order.
// Determined ICA mode (fastfca.cpp:241-264): L = identity, H = floored
// decorrelated powers of w_init, IP+MM with the loadings fixed.
FastFcaFitResult ica_mode_fit(const SampleCovSet& covs, int sources, int iters,
                              const std::vector<CMat>& w_init, const FitOptions& fit = {},
                              std::vector<double>* slots_out = nullptr);
// hermitian.hpp:74-79, :81-102 and fastfca.cpp:225-239 (ajd_cost): used by
// the reference's block-stationary decomposition tests.
double is_divergence(double w1, double w2);
double logdet_divergence(const CMat& a, const CMat& b);
bool is_positive_definite(const CMat& a);                          // hermitian.hpp (LLT succeeds)
double logdet_hpd(const CMat& a);                                  // ln det of a Hermitian PD matrix
double ajd_cost(const CMat& w, const SampleCovSet& covs, int i,
                const std::vector<double>& weights = {});
CMat fastfca_mwf(const FastFcaParams& p, int i, int j, int n);     // fastfca.cpp:193-203
// Separated images, [n][i] -> dim x frames (fastfca.cpp:205-223).
std::vector<std::vector<CMat>> fastfca_separate(const SampleCovSet& covs,
                                                const FastFcaParams& p);
void parallel_for(int count, int workers, const std::function<void(int)>& fn);  // parallel.cpp:16-45
int default_workers();                                             // parallel.cpp:11-14

}  // namespace oracle
