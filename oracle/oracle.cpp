// oracle.cpp -- TEST INFRASTRUCTURE ONLY.  fp64 restatement of the reference
// FastFCA hot path; see oracle.hpp for the contract and citations.
// Paths below are relative to /root/reference/proj.

#include "oracle.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <exception>
#include <mutex>
#include <random>
#include <thread>

namespace oracle {

namespace {

// fastfca.cpp:13-18
std::uint64_t mix_seed(std::uint64_t seed, int i) {
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (i + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

bool all_finite(const std::vector<Complex>& v) {
  for (const Complex& z : v)
    if (!std::isfinite(z.real()) || !std::isfinite(z.imag())) return false;
  return true;
}

double vnorm(const std::vector<Complex>& v) {
  double s = 0.0;
  for (const Complex& z : v) s += std::norm(z);
  return std::sqrt(s);
}

// L * H (+ eps) as used at fastfca.cpp:45, :86, :104, :111 and sigmodel.cpp:114.
RMat lh_product(const RMat& loading, const RMat& act, double eps) {
  const int m = loading.r, n_src = loading.c, frames = act.c;
  RMat out(m, frames);
  for (int j = 0; j < frames; ++j)
    for (int k = 0; k < m; ++k) {
      double s = 0.0;
      for (int n = 0; n < n_src; ++n) s += loading(k, n) * act(n, j);
      out(k, j) = s + eps;
    }
  return out;
}

}  // namespace

// ---------------------------------------------------------------- algebra --

// Eigen::PartialPivLU: max-modulus pivot per column, unit-lower L, upper U.
PartialPivLU::PartialPivLU(const CMat& a) : lu(a), perm(a.r) {
  const int n = a.r;
  for (int k = 0; k < n; ++k) perm[k] = k;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(lu(k, k));
    for (int r = k + 1; r < n; ++r) {
      const double v = std::abs(lu(r, k));
      if (v > best) best = v, p = r;
    }
    if (p != k) {
      for (int c = 0; c < n; ++c) std::swap(lu(k, c), lu(p, c));
      std::swap(perm[k], perm[p]);
    }
    if (best != 0.0) {
      for (int r = k + 1; r < n; ++r) lu(r, k) /= lu(k, k);
      for (int c = k + 1; c < n; ++c)
        for (int r = k + 1; r < n; ++r) lu(r, c) -= lu(r, k) * lu(k, c);
    }
  }
}

std::vector<Complex> PartialPivLU::solve(const std::vector<Complex>& b) const {
  const int n = lu.r;
  std::vector<Complex> y(n);
  for (int k = 0; k < n; ++k) y[k] = b[perm[k]];
  for (int k = 0; k < n; ++k)
    for (int r = k + 1; r < n; ++r) y[r] -= lu(r, k) * y[k];
  for (int k = n - 1; k >= 0; --k) {
    y[k] /= lu(k, k);
    for (int r = 0; r < k; ++r) y[r] -= lu(r, k) * y[k];
  }
  return y;
}

CMat PartialPivLU::solve(const CMat& b) const {
  CMat out(b.r, b.c);
  std::vector<Complex> col(b.r);
  for (int c = 0; c < b.c; ++c) {
    for (int r = 0; r < b.r; ++r) col[r] = b(r, c);
    const std::vector<Complex> s = solve(col);
    for (int r = 0; r < b.r; ++r) out(r, c) = s[r];
  }
  return out;
}

CMat PartialPivLU::inverse() const { return solve(CMat::identity(lu.r)); }

CMat adjoint(const CMat& a) {
  CMat t(a.c, a.r);
  for (int j = 0; j < a.c; ++j)
    for (int i = 0; i < a.r; ++i) t(j, i) = std::conj(a(i, j));
  return t;
}

CMat matmul(const CMat& a, const CMat& b) {
  CMat out(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int k = 0; k < a.c; ++k) {
      const Complex bkj = b(k, j);
      for (int i = 0; i < a.r; ++i) out(i, j) += a(i, k) * bkj;
    }
  return out;
}

RMat matmul(const RMat& a, const RMat& b) {
  RMat out(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int k = 0; k < a.c; ++k) {
      const double bkj = b(k, j);
      for (int i = 0; i < a.r; ++i) out(i, j) += a(i, k) * bkj;
    }
  return out;
}

double frob(const CMat& a) {
  double s = 0.0;
  for (const Complex& z : a.a) s += std::norm(z);
  return std::sqrt(s);
}

// ------------------------------------------------------------- sigmodel --

// sigmodel.cpp:10-15
void floor_positive(RMat& m, double rel) {
  if (m.a.empty()) return;
  double mean = 0.0;
  for (double v : m.a) mean += v;
  mean /= double(m.a.size());
  const double floor = (mean > 0.0) ? rel * mean : 1e-300;
  for (double& v : m.a) v = std::max(v, floor);
}

// sigmodel.cpp:17-48: snapshots[i] = spec.f[i] for block_size == 1 (:45);
// mats[i][jb] = (1/width) sum_{j in block} x_j x_j^H (:34-41), built for
// block_size > 1 (or on request); power_scale[i] = sum_jb tr(mats[i][jb]) /
// (blocks * M) (:33-44) -- for block_size == 1 the trace of x x^H is |x|^2.
SampleCovSet sample_covs(int dim, int bins, int frames, const Complex* x, int block_size,
                         bool with_mats) {
  if (bins == 0 || frames == 0 || dim == 0)
    throw std::invalid_argument("sample_covs: empty spectrogram");
  if (block_size < 1) throw std::invalid_argument("sample_covs: block size must be >= 1");
  SampleCovSet covs;
  covs.dim = dim;
  covs.bins = bins;
  covs.frames = frames;
  covs.block_size = block_size;
  covs.blocks = (frames + block_size - 1) / block_size;
  const bool mats = block_size > 1 || with_mats;
  if (mats) covs.mats.resize(bins);
  if (block_size == 1) covs.snapshots.resize(bins);
  covs.power_scale.assign(bins, 0.0);
  for (int i = 0; i < bins; ++i) {
    const Complex* xi = x + size_t(i) * frames * dim;
    double trace_sum = 0.0;
    if (mats) {
      covs.mats[i].resize(covs.blocks);
      for (int jb = 0; jb < covs.blocks; ++jb) {
        const int j0 = jb * block_size;
        const int width = std::min(block_size, frames - j0);
        CMat r(dim, dim);
        for (int j = j0; j < j0 + width; ++j)
          for (int c = 0; c < dim; ++c) {
            const Complex xc = std::conj(xi[size_t(j) * dim + c]);
            for (int a = 0; a < dim; ++a) r(a, c) += xi[size_t(j) * dim + a] * xc;
          }
        double tr = 0.0;
        for (auto& z : r.a) z /= double(width);
        for (int a = 0; a < dim; ++a) tr += r(a, a).real();
        trace_sum += tr;
        covs.mats[i][jb] = std::move(r);
      }
    } else {
      for (int j = 0; j < frames; ++j)
        for (int m = 0; m < dim; ++m) trace_sum += std::norm(xi[size_t(j) * dim + m]);
    }
    covs.power_scale[i] = trace_sum / (double(covs.blocks) * dim);
    if (block_size == 1) {
      CMat& s = covs.snapshots[i];
      s = CMat(dim, frames);
      for (int j = 0; j < frames; ++j)
        for (int m = 0; m < dim; ++m) s(m, j) = xi[size_t(j) * dim + m];
    }
  }
  return covs;
}

// sigmodel.cpp:50-55
double SampleCovSet::power(int i) const {
  if (i < int(power_scale.size())) return power_scale[i];
  double trace_sum = 0.0;
  for (const CMat& m : mats[i])
    for (int a = 0; a < m.r; ++a) trace_sum += m(a, a).real();
  return trace_sum / (double(blocks) * dim);
}

// fastfca.cpp:266-268
SampleCovSet piecewise_prepare(int dim, int bins, int frames, const Complex* x, int block_size) {
  return sample_covs(dim, bins, frames, x, block_size, true);
}

// sigmodel.cpp:164-176 (replicate_columns) and :188-196.
FastFcaParams expand_block_params(const FastFcaParams& p, int block_size, int frames) {
  if (block_size == 1 && frames == p.frames) return p;
  FastFcaParams out = p;
  out.frames = frames;
  for (int i = 0; i < p.bins; ++i) {
    const RMat& h = p.act[i];
    RMat e(h.r, frames);
    for (int j = 0; j < frames; ++j) {
      const int jb = std::min(j / block_size, h.c - 1);
      for (int n = 0; n < h.r; ++n) e(n, j) = h(n, jb);
    }
    out.act[i] = std::move(e);
  }
  return out;
}

// sigmodel.cpp:93-107 (snapshot branch :96): U = |W^H X|^2.
RMat decorrelated_powers(const SampleCovSet& covs, int i, const CMat& w) {
  const int m = covs.dim;
  if (!covs.has_snapshots()) {  // :97-105: u(k, j) = max(0, Re w_k^H X_j w_k)
    RMat u(m, covs.blocks);
    for (int j = 0; j < covs.blocks; ++j) {
      const CMat& xm = covs.mats[i][j];
      for (int k = 0; k < m; ++k) {
        Complex acc = 0.0;
        for (int r = 0; r < m; ++r) {
          Complex xw = 0.0;
          for (int c = 0; c < m; ++c) xw += xm(r, c) * w(c, k);
          acc += std::conj(w(r, k)) * xw;
        }
        u(k, j) = std::max(0.0, acc.real());
      }
    }
    return u;
  }
  const CMat& x = covs.snapshots[i];
  RMat u(m, x.c);
  for (int j = 0; j < x.c; ++j)
    for (int k = 0; k < m; ++k) {
      Complex y = 0.0;
      for (int r = 0; r < m; ++r) y += std::conj(w(r, k)) * x(r, j);
      u(k, j) = std::norm(y);
    }
  return u;
}

// sigmodel.cpp:118-129
double log_abs_det2(const CMat& w) {
  PartialPivLU lu(w);
  double acc = 0.0;
  for (int k = 0; k < w.r; ++k) {
    const double a = std::abs(lu.lu(k, k));
    if (!(a > 0.0) || !std::isfinite(a))
      throw NumericalError("singular decorrelation matrix");
    acc += std::log(a);
  }
  return 2.0 * acc;
}

// sigmodel.cpp:155-162 with decorrelated_stats (:109-116).
double fastfca_nll_freq(const SampleCovSet& covs, int i, const CMat& w, const RMat& loading,
                        const RMat& act) {
  const RMat u = decorrelated_powers(covs, i, w);
  const RMat s2 = lh_product(loading, act, var_eps(covs.power(i)));
  const double logdet = log_abs_det2(w);
  double ratio = 0.0, logs = 0.0;
  for (size_t k = 0; k < u.a.size(); ++k) ratio += u.a[k] / s2.a[k];
  for (size_t k = 0; k < s2.a.size(); ++k) logs += std::log(s2.a[k]);
  return -covs.blocks * logdet + ratio + logs;
}

// sigmodel.cpp:215-222
double fastfca_nll(const SampleCovSet& covs, const FastFcaParams& p) {
  if (covs.dim != p.dim || covs.bins != p.bins || covs.blocks != p.frames)
    throw std::invalid_argument("nll: covariance/parameter shape mismatch");
  double acc = 0.0;
  for (int i = 0; i < covs.bins; ++i)
    acc += fastfca_nll_freq(covs, i, p.decorr[i], p.loading[i], p.act[i]);
  return acc;
}

// sigmodel.cpp:131-153 (snapshot branch), Eigen::LLT on the lower triangle.
double fca_nll_freq(const SampleCovSet& covs, int i, const std::vector<CMat>& scm_i,
                    const RMat& power_i) {
  const int m = covs.dim;
  const bool snap = covs.has_snapshots();
  const CMat& xs = snap ? covs.snapshots[i] : covs.mats[i][0];
  double acc = 0.0;
  for (int j = 0; j < covs.blocks; ++j) {
    CMat x(m, m);
    for (size_t n = 0; n < scm_i.size(); ++n)
      for (size_t k = 0; k < x.a.size(); ++k) x.a[k] += power_i(int(n), j) * scm_i[n].a[k];
    CMat l(m, m);
    for (int k = 0; k < m; ++k) {
      double d = x(k, k).real();
      for (int p = 0; p < k; ++p) d -= std::norm(l(k, p));
      if (!(d > 0.0)) throw NumericalError("fca_nll: mixture covariance not PD");
      const double lkk = std::sqrt(d);
      l(k, k) = lkk;
      for (int r = k + 1; r < m; ++r) {
        Complex s = x(r, k);
        for (int p = 0; p < k; ++p) s -= l(r, p) * std::conj(l(k, p));
        l(r, k) = s / lkk;
      }
    }
    for (int k = 0; k < m; ++k) acc += 2.0 * std::log(l(k, k).real());
    if (!snap) {  // :149-150: tr(X^-1 Xhat_j), column by column
      const CMat& xm = covs.mats[i][j];
      for (int c = 0; c < m; ++c) {
        std::vector<Complex> y(m);
        for (int k = 0; k < m; ++k) {
          Complex s = xm(k, c);
          for (int p = 0; p < k; ++p) s -= l(k, p) * y[p];
          y[k] = s / l(k, k);
        }
        for (int k = m - 1; k >= 0; --k) {
          Complex s = y[k];
          for (int p = k + 1; p < m; ++p) s -= std::conj(l(p, k)) * y[p];
          y[k] = s / l(k, k);
        }
        acc += y[c].real();
      }
      continue;
    }
    std::vector<Complex> y(m);
    for (int k = 0; k < m; ++k) {
      Complex s = xs(k, j);
      for (int p = 0; p < k; ++p) s -= l(k, p) * y[p];
      y[k] = s / l(k, k);
    }
    for (int k = m - 1; k >= 0; --k) {
      Complex s = y[k];
      for (int p = k + 1; p < m; ++p) s -= std::conj(l(p, k)) * y[p];
      y[k] = s / l(k, k);
    }
    Complex q = 0.0;
    for (int k = 0; k < m; ++k) q += std::conj(xs(k, j)) * y[k];
    acc += q.real();
  }
  return acc;
}

// -------------------------------------------------------------- fastfca --

// fastfca.cpp:22-34 + symmetrize (hermitian.hpp:31-34).  Snapshot branch
// (:25-28): q = X diag(1/s2) X^H; block branch (:30-31): q = sum_j mats_j / s2_j.
CMat weighted_cov(const SampleCovSet& covs, int i, const double* sigma2_row, int stride) {
  const int m = covs.dim, blocks = covs.blocks;
  CMat q(m, m);
  if (covs.has_snapshots()) {
    const CMat& x = covs.snapshots[i];
    for (int j = 0; j < blocks; ++j) {
      const double inv = 1.0 / sigma2_row[size_t(j) * stride];
      for (int b = 0; b < m; ++b) {
        const Complex xb = std::conj(x(b, j));
        for (int a = 0; a < m; ++a) q(a, b) += (x(a, j) * inv) * xb;
      }
    }
  } else {
    for (int j = 0; j < blocks; ++j) {
      const double s = sigma2_row[size_t(j) * stride];
      const CMat& xm = covs.mats[i][j];
      for (size_t k = 0; k < q.a.size(); ++k) q.a[k] += xm.a[k] / s;
    }
  }
  CMat out(m, m);
  for (int b = 0; b < m; ++b)
    for (int a = 0; a < m; ++a)
      out(a, b) = (q(a, b) / double(blocks) + std::conj(q(b, a)) / double(blocks)) / 2.0;
  return out;
}

// fastfca.cpp:36-72
void ip_update_w(const SampleCovSet& covs, int i, CMat& w, const RMat& loading,
                 const RMat& act, std::uint64_t restart_seed) {
  const int m = covs.dim;
  std::mt19937_64 rng(mix_seed(restart_seed, i));
  std::normal_distribution<double> gauss(0.0, 1.0);
  const RMat sigma2 = lh_product(loading, act, var_eps(covs.power(i)));  // :45
  for (int col = 0; col < m; ++col) {
    const CMat q = weighted_cov(covs, i, &sigma2(col, 0), m);           // :48
    std::vector<Complex> e(m, Complex(0, 0));
    e[col] = Complex(1, 0);
    for (int attempt = 0;; ++attempt) {
      const CMat a = matmul(adjoint(w), q);                              // :52
      PartialPivLU lu(a);
      const std::vector<Complex> wm = lu.solve(e);
      const double scale = frob(a) * vnorm(wm) + 1.0;                    // :55
      std::vector<Complex> res(m);
      for (int r = 0; r < m; ++r) {
        Complex s = 0.0;
        for (int c = 0; c < m; ++c) s += a(r, c) * wm[c];
        res[r] = s - e[r];
      }
      if (all_finite(wm) && vnorm(res) <= 1e-8 * scale) {                // :56
        Complex energy_c = 0.0;
        for (int r = 0; r < m; ++r) {
          Complex qw = 0.0;
          for (int c = 0; c < m; ++c) qw += q(r, c) * wm[c];
          energy_c += std::conj(wm[r]) * qw;
        }
        const double energy = std::real(energy_c);                      // :57
        if (energy > 0.0 && std::isfinite(energy)) {
          const double s = std::sqrt(energy);
          for (int r = 0; r < m; ++r) w(r, col) = wm[r] / s;
          break;
        }
      }
      if (attempt >= 1)
        throw NumericalError("ip_update_w: singular system for column " + std::to_string(col));
      double cn = 0.0;                                                   // :67
      for (int r = 0; r < m; ++r) cn += std::norm(w(r, col));
      const double mag = 1e-8 * (std::sqrt(cn) + 1.0);
      for (int r = 0; r < m; ++r) w(r, col) += mag * Complex(gauss(rng), gauss(rng));
    }
  }
}

// fastfca.cpp:74-78
RMat source_gain(const RMat& loading, const RMat& act, int n) {
  RMat lh = lh_product(loading, act, 0.0);
  floor_positive(lh);
  RMat g(lh.r, lh.c);
  for (int j = 0; j < lh.c; ++j)
    for (int k = 0; k < lh.r; ++k) g(k, j) = (loading(k, n) * act(n, j)) / lh(k, j);
  return g;
}

// fastfca.cpp:80-99
void em_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading, double eps) {
  const int m = u.r, frames = u.c, sources = loading.c;
  RMat phi(m, frames);
  for (int n = 0; n < sources; ++n) {
    const RMat lh = lh_product(loading, act, eps);  // :86, full product per source
    for (int j = 0; j < frames; ++j)
      for (int k = 0; k < m; ++k) {
        const double lnhn = loading(k, n) * act(n, j);
        const double g = lnhn / lh(k, j);
        phi(k, j) = g * g * u(k, j) + (1.0 - g) * lnhn;  // :89-90
      }
    if (update_loading) {
      for (int k = 0; k < m; ++k) {
        double s = 0.0;
        for (int j = 0; j < frames; ++j) s += phi(k, j) * (1.0 / act(n, j));
        loading(k, n) = std::max(s / frames, 1e-300);  // :92-94
      }
    }
    for (int j = 0; j < frames; ++j) {
      double s = 0.0;
      for (int k = 0; k < m; ++k) s += (1.0 / loading(k, n)) * phi(k, j);
      act(n, j) = std::max(s / m, 1e-300);  // :96-97
    }
  }
}

// fastfca.cpp:101-117
void mm_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading, double eps) {
  const int m = u.r, frames = u.c, sources = loading.c;
  if (update_loading) {
    const RMat lh = lh_product(loading, act, eps);
    RMat num(m, sources), den(m, sources);
    for (int j = 0; j < frames; ++j)
      for (int k = 0; k < m; ++k) {
        const double l = lh(k, j);
        const double ul2 = u(k, j) / (l * l);
        const double il = 1.0 / l;
        for (int n = 0; n < sources; ++n) {
          num(k, n) += ul2 * act(n, j);
          den(k, n) += il * act(n, j);
        }
      }
    for (int n = 0; n < sources; ++n)
      for (int k = 0; k < m; ++k) {
        const double d = std::max(den(k, n), 1e-300);
        loading(k, n) = std::max(loading(k, n) * std::sqrt(num(k, n) / d), 1e-300);
      }
  }
  const RMat lh = lh_product(loading, act, eps);
  for (int j = 0; j < frames; ++j) {
    for (int n = 0; n < sources; ++n) {
      double num = 0.0, den = 0.0;
      for (int k = 0; k < m; ++k) {
        const double l = lh(k, j);
        num += loading(k, n) * (u(k, j) / (l * l));
        den += loading(k, n) * (1.0 / l);
      }
      den = std::max(den, 1e-300);
      act(n, j) = std::max(act(n, j) * std::sqrt(num / den), 1e-300);
    }
  }
}

// fastfca.cpp:127-142
void balance_scales(CMat& w, RMat& loading, RMat& act) {
  for (int n = 0; n < act.r; ++n) {
    double mu = 0.0;
    for (int j = 0; j < act.c; ++j) mu += act(n, j);
    mu /= act.c;
    if (mu > 0.0 && std::isfinite(mu)) {
      for (int j = 0; j < act.c; ++j) act(n, j) /= mu;
      for (int k = 0; k < loading.r; ++k) loading(k, n) *= mu;
    }
  }
  for (int k = 0; k < loading.r; ++k) {
    double s = 0.0;
    for (int n = 0; n < loading.c; ++n) s += loading(k, n);
    s /= loading.c;
    if (s > 0.0 && std::isfinite(s)) {
      for (int n = 0; n < loading.c; ++n) loading(k, n) /= s;
      const double r = std::sqrt(s);
      for (int c = 0; c < w.r; ++c) w(c, k) /= r;
    }
  }
}

// fastfca.cpp:146-191
FastFcaFitResult fastfca_fit(const SampleCovSet& covs, const FastFcaParams& init,
                             LhFlavor flavor, int iters, const FitOptions& fit,
                             const FastFcaOptions& opts, std::vector<double>* slots_out) {
  if (init.dim != covs.dim || init.bins != covs.bins || init.frames != covs.blocks)
    throw std::invalid_argument("fastfca_fit: init/covariance shape mismatch");
  FastFcaFitResult result;
  result.params = init;
  std::vector<double> slots;
  if (fit.record_trace) slots.assign(size_t(iters + 1) * covs.bins, 0.0);
  auto slot = [&](int t, int i) -> double& { return slots[size_t(t) * covs.bins + i]; };

  parallel_for(covs.bins, fit.workers, [&](int i) {
    CMat& w = result.params.decorr[i];
    RMat& loading = result.params.loading[i];
    RMat& act = result.params.act[i];
    const double nll0 = fit.record_trace ? fastfca_nll_freq(covs, i, w, loading, act) : 0.0;
    if (fit.record_trace) slot(0, i) = nll0;
    if (!(covs.power(i) > 0.0)) {
      if (fit.record_trace)
        for (int t = 0; t < iters; ++t) slot(t + 1, i) = nll0;
      return;
    }
    const double eps = var_eps(covs.power(i));
    for (int t = 0; t < iters; ++t) {
      ip_update_w(covs, i, w, loading, act, fit.seed + t);
      const RMat u = decorrelated_powers(covs, i, w);
      if (flavor == LhFlavor::em)
        em_update_lh(u, loading, act, !opts.fix_loadings, eps);
      else
        mm_update_lh(u, loading, act, !opts.fix_loadings, eps);
      if (opts.normalize_scales && !opts.fix_loadings) balance_scales(w, loading, act);
      if (fit.record_trace) slot(t + 1, i) = fastfca_nll_freq(covs, i, w, loading, act);
    }
  });

  if (fit.record_trace) {
    result.nll.assign(iters + 1, 0.0);
    for (int t = 0; t <= iters; ++t) {
      double s = 0.0;
      for (int i = 0; i < covs.bins; ++i) s += slot(t, i);
      result.nll[t] = s;
    }
    if (slots_out) *slots_out = slots;
  }
  return result;
}

// fastfca.cpp:241-264
FastFcaFitResult ica_mode_fit(const SampleCovSet& covs, int sources, int iters,
                              const std::vector<CMat>& w_init, const FitOptions& fit,
                              std::vector<double>* slots_out) {
  if (sources != covs.dim)
    throw std::invalid_argument("ica_mode_fit: requires as many sources as channels");
  if (static_cast<int>(w_init.size()) != covs.bins)
    throw std::invalid_argument("ica_mode_fit: one W per frequency required");
  FastFcaParams params;
  params.dim = covs.dim;
  params.bins = covs.bins;
  params.frames = covs.blocks;
  params.sources = sources;
  params.decorr = w_init;
  for (int i = 0; i < covs.bins; ++i) {
    params.loading.push_back(RMat::identity(covs.dim));  // dim == sources
    RMat u = decorrelated_powers(covs, i, w_init[i]);
    floor_positive(u);
    params.act.push_back(u);
  }
  FastFcaOptions opts;
  opts.fix_loadings = true;
  return fastfca_fit(covs, params, LhFlavor::mm, iters, fit, opts, slots_out);
}

// hermitian.hpp:74-79
double is_divergence(double w1, double w2) {
  if (!(w1 > 0.0) || !(w2 > 0.0))
    throw std::domain_error("is_divergence: arguments must be positive");
  const double r = w1 / w2;
  return std::max(0.0, r - std::log(r) - 1.0);
}

namespace {
CMat symmetrize(const CMat& a) {  // hermitian.hpp:31-34
  CMat s(a.r, a.c);
  for (int c = 0; c < a.c; ++c)
    for (int r = 0; r < a.r; ++r) s(r, c) = (a(r, c) + std::conj(a(c, r))) / 2.0;
  return s;
}
// Lower Cholesky factor (Eigen::LLT reads the lower triangle); false when not PD.
bool llt(const CMat& x, CMat& l) {
  const int m = x.r;
  l = CMat(m, m);
  for (int k = 0; k < m; ++k) {
    double d = x(k, k).real();
    for (int p = 0; p < k; ++p) d -= std::norm(l(k, p));
    if (!(d > 0.0)) return false;
    const double lkk = std::sqrt(d);
    l(k, k) = lkk;
    for (int r = k + 1; r < m; ++r) {
      Complex s = x(r, k);
      for (int p = 0; p < k; ++p) s -= l(r, p) * std::conj(l(k, p));
      l(r, k) = s / lkk;
    }
  }
  return true;
}
}  // namespace

// hermitian.hpp:42-47
bool is_positive_definite(const CMat& a) {
  if (a.r != a.c) return false;
  double mx = 0.0, dev = 0.0;
  for (int c = 0; c < a.c; ++c)
    for (int r = 0; r < a.r; ++r) {
      mx = std::max(mx, std::abs(a(r, c)));
      dev = std::max(dev, std::abs(a(r, c) - std::conj(a(c, r))));
    }
  if (!(dev <= 1e-10 * (1.0 + mx))) return false;
  CMat l;
  return llt(symmetrize(a), l);
}

double logdet_hpd(const CMat& a) {
  CMat l;
  if (!llt(symmetrize(a), l)) throw NumericalError("logdet_hpd: not positive definite");
  double s = 0.0;
  for (int k = 0; k < a.r; ++k) s += 2.0 * std::log(l(k, k).real());
  return s;
}

// hermitian.hpp:81-102: tr(A B^-1) - ln det(A B^-1) - M (LLT of both).
double logdet_divergence(const CMat& a, const CMat& b) {
  if (a.r != a.c || b.r != b.c || a.r != b.r)
    throw std::invalid_argument("logdet_divergence: dimension mismatch");
  const int m = a.r;
  CMat la, lb;
  if (!llt(symmetrize(a), la) || !llt(symmetrize(b), lb))
    throw NumericalError("logdet_divergence: argument not positive definite");
  double tr = 0.0;  // tr(B^-1 A) column by column
  for (int c = 0; c < m; ++c) {
    std::vector<Complex> y(m);
    for (int k = 0; k < m; ++k) {
      Complex s = a(k, c);
      for (int p = 0; p < k; ++p) s -= lb(k, p) * y[p];
      y[k] = s / lb(k, k);
    }
    for (int k = m - 1; k >= 0; --k) {
      Complex s = y[k];
      for (int p = k + 1; p < m; ++p) s -= std::conj(lb(p, k)) * y[p];
      y[k] = s / lb(k, k);
    }
    tr += y[c].real();
  }
  double lda = 0.0, ldb = 0.0;
  for (int k = 0; k < m; ++k) {
    lda += 2.0 * std::log(la(k, k).real());
    ldb += 2.0 * std::log(lb(k, k).real());
  }
  return std::max(0.0, tr - (lda - ldb) - double(m));
}

// fastfca.cpp:225-239
double ajd_cost(const CMat& w, const SampleCovSet& covs, int i,
                const std::vector<double>& weights) {
  if (!weights.empty() && int(weights.size()) != covs.blocks)
    throw std::invalid_argument("ajd_cost: weight count mismatch");
  const int m = covs.dim;
  double acc = 0.0;
  for (int j = 0; j < covs.blocks; ++j) {
    const CMat t = matmul(matmul(adjoint(w), covs.mats[i][j]), w);
    CMat d(m, m);
    for (int k = 0; k < m; ++k) d(k, k) = t(k, k);
    const double alpha = weights.empty() ? 1.0 : weights[j];
    acc += alpha * logdet_divergence(t, d);
  }
  return acc;
}

// fastfca.cpp:193-203
CMat fastfca_mwf(const FastFcaParams& p, int i, int j, int n) {
  const int m = p.dim;
  std::vector<double> mix(m, 0.0);
  for (int k = 0; k < m; ++k) {
    for (int s = 0; s < p.sources; ++s) mix[k] += p.loading[i](k, s) * p.act[i](s, j);
    mix[k] = std::max(mix[k], 1e-300);
  }
  const CMat a = adjoint(p.decorr[i]);
  PartialPivLU lu(a);
  CMat ga(m, m);
  for (int c = 0; c < m; ++c)
    for (int k = 0; k < m; ++k)
      ga(k, c) = (p.loading[i](k, n) * p.act[i](n, j) / mix[k]) * a(k, c);
  return lu.solve(ga);
}

// fastfca.cpp:205-223
std::vector<std::vector<CMat>> fastfca_separate(const SampleCovSet& covs,
                                                const FastFcaParams& p) {
  if (covs.dim != p.dim || covs.bins != p.bins || covs.frames != p.frames)
    throw std::invalid_argument("fastfca_separate: shape mismatch");
  std::vector<std::vector<CMat>> images(p.sources, std::vector<CMat>(p.bins));
  for (int i = 0; i < p.bins; ++i) {
    const CMat a = adjoint(p.decorr[i]);
    PartialPivLU lu(a);
    const CMat y = matmul(a, covs.snapshots[i]);
    for (int n = 0; n < p.sources; ++n) {
      const RMat g = source_gain(p.loading[i], p.act[i], n);
      CMat gy(y.r, y.c);
      for (size_t k = 0; k < gy.a.size(); ++k) gy.a[k] = g.a[k] * y.a[k];
      images[n][i] = lu.solve(gy);
    }
  }
  return images;
}

// fastfca.cpp:270-282
std::vector<std::vector<CMat>> reconstruct_scms(const FastFcaParams& p) {
  std::vector<std::vector<CMat>> scms(p.bins);
  for (int i = 0; i < p.bins; ++i) {
    const CMat winv = PartialPivLU(p.decorr[i]).inverse();
    const CMat winv_h = adjoint(winv);
    for (int n = 0; n < p.sources; ++n) {
      CMat d(p.dim, p.dim);
      for (int c = 0; c < p.dim; ++c)
        for (int r = 0; r < p.dim; ++r) d(r, c) = winv_h(r, c) * p.loading[i](c, n);
      scms[i].push_back(matmul(d, winv));
    }
  }
  return scms;
}

// ------------------------------------------------------------- parallel --

// parallel.cpp:11-14
int default_workers() {
  const unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1 : int(n);
}

// parallel.cpp:16-45
void parallel_for(int count, int workers, const std::function<void(int)>& fn) {
  if (count <= 0) return;
  if (workers <= 1 || count == 1) {
    for (int k = 0; k < count; ++k) fn(k);
    return;
  }
  const int crew = std::min(workers, count);
  std::atomic<int> next{0};
  std::exception_ptr first_error;
  std::mutex error_mutex;
  auto run = [&]() {
    for (;;) {
      const int k = next.fetch_add(1, std::memory_order_relaxed);
      if (k >= count) return;
      try {
        fn(k);
      } catch (...) {
        std::lock_guard<std::mutex> lock(error_mutex);
        if (!first_error) first_error = std::current_exception();
        return;
      }
    }
  };
  std::vector<std::thread> threads;
  threads.reserve(crew - 1);
  for (int t = 1; t < crew; ++t) threads.emplace_back(run);
  run();
  for (auto& t : threads) t.join();
  if (first_error) std::rethrow_exception(first_error);
}

}  // namespace oracle
