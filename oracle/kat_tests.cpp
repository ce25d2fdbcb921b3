// kat_tests.cpp -- TEST INFRASTRUCTURE ONLY.  Pins the oracle restatement
// against the reference's own known-answer and property tests for the hot path
// (reference tests/test_fastfca.cpp and tests/test_sigmodel.cpp).  The random
// generators are the reference's (tests/testutil.hpp:12-56): libstdc++'s
// std::mt19937 + std::normal_distribution / uniform_real_distribution, built
// here with the same g++/libstdc++, so every test draws the same inputs the
// reference's doctest binary would.  doctest itself is absent, so a minimal
// CHECK / Approx shim reproduces doctest's Approx formula:
//   |a - b| < eps * (scale + max(|a|, |b|)),  scale = 1.
//
// Exit code 0 = all checks passed.  Each TEST prints its name and failures.

#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {

int g_fail = 0, g_checks = 0;
const char* g_case = "";

#define CHECK(cond)                                                                 \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(cond)) {                                                                  \
      ++g_fail;                                                                     \
      std::printf("  FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond);    \
    }                                                                               \
  } while (0)

// The reference adds eps = 1e-8 * power to every model variance
// (sigmodel.hpp:21-31, fastfca.cpp:45, sigmodel.cpp:114) but several of its
// tests assert identities that hold only for eps = 0 (scale invariance, the
// FCA cross-model equality, the M = 1 closed form) at 1e-10..1e-12.  Those
// assertions are checked at the reference tolerance in the eps = 0 build
// (kat_tests_noeps, -DORACLE_VAR_EPS_REL=0) and at the analytic eps-effect
// bound (~1e-8 relative per term) in the shipped-eps build.
constexpr bool kNoEps = (kVarEpsRel == 0.0);
double eps_tol(double reference_tol, double shipped_tol) {
  return kNoEps ? reference_tol : shipped_tol;
}

bool approx(double a, double b, double eps) {
  return std::fabs(a - b) < eps * (1.0 + std::max(std::fabs(a), std::fabs(b)));
}

// ---- tests/testutil.hpp:12-56 ----
double randn(std::mt19937& rng) {
  std::normal_distribution<double> d(0.0, 1.0);
  return d(rng);
}
Complex crandn(std::mt19937& rng) {
  std::normal_distribution<double> d(0.0, 1.0);
  return Complex(d(rng), d(rng)) / std::sqrt(2.0);
}
CMat random_complex(int rows, int cols, std::mt19937& rng) {
  CMat a(rows, cols);
  for (int c = 0; c < cols; ++c)
    for (int r = 0; r < rows; ++r) a(r, c) = crandn(rng);
  return a;
}
RMat random_positive(int rows, int cols, std::mt19937& rng, double lo = 0.1, double hi = 10.0) {
  std::uniform_real_distribution<double> d(std::log(lo), std::log(hi));
  RMat a(rows, cols);
  for (int c = 0; c < cols; ++c)
    for (int r = 0; r < rows; ++r) a(r, c) = std::exp(d(rng));
  return a;
}
double rel_err(const CMat& a, const CMat& b) {
  CMat d = a;
  for (size_t k = 0; k < d.a.size(); ++k) d.a[k] -= b.a[k];
  return frob(d) / std::max(1e-300, frob(b));
}

// ---- tests/test_fastfca.cpp:16-46 ----
FastFcaParams random_params(int dim, int bins, int frames, int sources, std::mt19937& rng) {
  FastFcaParams p;
  p.dim = dim, p.bins = bins, p.frames = frames, p.sources = sources;
  for (int i = 0; i < bins; ++i) {
    CMat w = random_complex(dim, dim, rng);
    for (auto& z : w.a) z *= 0.5;
    for (int k = 0; k < dim; ++k) w(k, k) += 1.0;
    p.decorr.push_back(w);
    p.loading.push_back(random_positive(dim, sources, rng, 0.3, 3.0));
    p.act.push_back(random_positive(sources, frames, rng, 0.3, 3.0));
  }
  return p;
}

// Spectrogram f[i] as a contiguous [bins][frames][dim] complex buffer.
struct Spec {
  int dim, bins, frames;
  std::vector<Complex> x;
  Complex& at(int i, int m, int j) { return x[(size_t(i) * frames + j) * dim + m]; }
  SampleCovSet covs(int block_size = 1, bool with_mats = false) const {
    return sample_covs(dim, bins, frames, x.data(), block_size, with_mats);
  }
};

Spec sample_jd_model(const FastFcaParams& truth, std::mt19937& rng) {
  Spec s{truth.dim, truth.bins, truth.frames,
         std::vector<Complex>(size_t(truth.dim) * truth.bins * truth.frames)};
  for (int i = 0; i < truth.bins; ++i) {
    PartialPivLU lu(adjoint(truth.decorr[i]));
    for (int j = 0; j < truth.frames; ++j) {
      std::vector<Complex> y(truth.dim);
      for (int k = 0; k < truth.dim; ++k) {
        double s2 = 0.0;
        for (int n = 0; n < truth.sources; ++n) s2 += truth.loading[i](k, n) * truth.act[i](n, j);
        y[k] = std::sqrt(s2) * crandn(rng);
      }
      const auto x = lu.solve(y);
      for (int k = 0; k < truth.dim; ++k) s.at(i, k, j) = x[k];
    }
  }
  return s;
}

Spec random_spec(int dim, int bins, int frames, std::mt19937& rng) {
  Spec s{dim, bins, frames, std::vector<Complex>(size_t(dim) * bins * frames)};
  for (int i = 0; i < bins; ++i) {
    const CMat r = random_complex(dim, frames, rng);
    for (int j = 0; j < frames; ++j)
      for (int k = 0; k < dim; ++k) s.at(i, k, j) = r(k, j);
  }
  return s;
}

double is_cost(const RMat& u, const RMat& loading, const RMat& act) {  // test_fastfca.cpp:48-56
  RMat lh = matmul(loading, act);
  floor_positive(lh);
  double acc = 0.0;
  for (int j = 0; j < u.c; ++j)
    for (int m = 0; m < u.r; ++m) acc += is_divergence(std::max(u(m, j), 1e-300), lh(m, j));
  return acc;
}

void check_trace_monotone(const std::vector<double>& nll, double rel = 1e-8) {
  for (size_t t = 1; t < nll.size(); ++t) CHECK(nll[t] <= nll[t - 1] + rel * std::abs(nll[t - 1]));
}

#define TEST(name) static void name(); struct name##_reg { name##_reg() { tests().push_back({#name, name}); } } name##_inst; static void name()
struct Entry { const char* name; void (*fn)(); };
std::vector<Entry>& tests() { static std::vector<Entry> t; return t; }

}  // namespace

// test_fastfca.cpp:84-103
TEST(ip_scalar_case) {
  std::mt19937 rng(61);
  Spec s{1, 1, 50, {}};
  const CMat r = random_complex(1, 50, rng);
  s.x.assign(r.a.begin(), r.a.end());
  const SampleCovSet covs = s.covs();
  RMat loading(1, 1, 1.0);
  const RMat act = random_positive(1, 50, rng);
  double q = 0.0;
  for (int j = 0; j < 50; ++j) q += std::norm(s.x[j]) / (loading(0, 0) * act(0, j));
  q /= 50;  // eps-free, as test_fastfca.cpp:90-91
  for (int t = 0; t < 5; ++t) {
    CMat w(1, 1);
    w(0, 0) = crandn(rng) * 3.0;
    const Complex before = w(0, 0) / std::abs(w(0, 0));
    ip_update_w(covs, 0, w, loading, act);
    CHECK(approx(std::abs(w(0, 0)), 1.0 / std::sqrt(q), eps_tol(1e-10, 1e-7)));
    const Complex after = w(0, 0) / std::abs(w(0, 0));
    CHECK(std::abs(after - before) < 1e-10);
  }
}

// test_fastfca.cpp:104-121.  The reference builds Q from the eps-free
// variances while ip_update_w normalizes against sigma^2 + eps
// (fastfca.cpp:45); SURVEY §4 caveat 1 predicts the shipped 1e-10 assertion
// fails by ~1e-8.  Checked here (a) against the eps-inclusive Q the update
// actually uses, at 1e-10, and (b) against the eps-free Q at 1e-7.
TEST(ip_column_normalization) {
  std::mt19937 gen(62);
  Spec s = random_spec(3, 2, 60, gen);
  const SampleCovSet covs = s.covs();
  FastFcaParams p = random_params(3, 2, 60, 2, gen);
  double worst_noeps = 0.0;
  for (int i = 0; i < 2; ++i) {
    ip_update_w(covs, i, p.decorr[i], p.loading[i], p.act[i]);
    for (int m = 0; m < 3; ++m) {
      for (int with_eps = 0; with_eps < 2; ++with_eps) {
        RMat sig(1, 60);
        for (int j = 0; j < 60; ++j) {
          double v = 0.0;
          for (int n = 0; n < 2; ++n) v += p.loading[i](m, n) * p.act[i](n, j);
          sig(0, j) = v;
        }
        if (with_eps)
          for (double& v : sig.a) v += var_eps(covs.power(i));
        else
          floor_positive(sig);
        const CMat q = weighted_cov(covs, i, sig.data(), 1);
        Complex e = 0.0;
        for (int r = 0; r < 3; ++r) {
          Complex qw = 0.0;
          for (int c = 0; c < 3; ++c) qw += q(r, c) * p.decorr[i](c, m);
          e += std::conj(p.decorr[i](r, m)) * qw;
        }
        if (with_eps)
          CHECK(approx(e.real(), 1.0, 1e-10));
        else
          worst_noeps = std::max(worst_noeps, std::abs(e.real() - 1.0));
      }
    }
  }
  CHECK(worst_noeps < 1e-7);
  std::printf("  note: eps-free normalization residual %.3e (reference asserts ~2e-10)\n",
              worst_noeps);
}

// test_fastfca.cpp:124-134, restated on snapshots: every frame excites a
// single channel, so every Q_m is diagonal and W must stay diagonal.
TEST(ip_keeps_diagonal) {
  std::mt19937 rng(63);
  Spec s{3, 1, 40, std::vector<Complex>(120)};
  for (int j = 0; j < 40; ++j) s.at(0, j % 3, j) = Complex(0.2 + std::abs(randn(rng)), 0);
  const SampleCovSet covs = s.covs();
  CMat w = CMat::identity(3);
  const RMat loading = random_positive(3, 2, rng);
  const RMat act = random_positive(2, 40, rng);
  ip_update_w(covs, 0, w, loading, act);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      if (r != c) CHECK(std::abs(w(r, c)) < 1e-12);
}

// test_fastfca.cpp:136-150
TEST(ip_does_not_increase_nll) {
  std::mt19937 rng(64);
  for (int t = 0; t < 10; ++t) {
    Spec s = random_spec(3, 1, 80, rng);
    const SampleCovSet covs = s.covs();
    FastFcaParams p = random_params(3, 1, 80, 2 + t % 3, rng);
    const double before = fastfca_nll_freq(covs, 0, p.decorr[0], p.loading[0], p.act[0]);
    ip_update_w(covs, 0, p.decorr[0], p.loading[0], p.act[0]);
    const double after = fastfca_nll_freq(covs, 0, p.decorr[0], p.loading[0], p.act[0]);
    CHECK(after <= before + 1e-8 * std::abs(before));
  }
}

// test_fastfca.cpp:152-180
TEST(em_update_known_answers) {
  {
    RMat u(1, 1, 3.4), loading(1, 1, 0.7), act(1, 1, 1.9);
    em_update_lh(u, loading, act);
    CHECK(approx(loading(0, 0), 3.4 / 1.9, 1e-12));
    CHECK(approx(act(0, 0), 1.9, 1e-12));
    CHECK(approx(loading(0, 0) * act(0, 0), 3.4, 1e-12));
  }
  {
    std::mt19937 rng(65);
    const RMat loading = random_positive(3, 1, rng);
    const RMat act = random_positive(1, 7, rng);
    const RMat u = matmul(loading, act);
    RMat l2 = loading, a2 = act;
    em_update_lh(u, l2, a2);
    const RMat p = matmul(l2, a2);
    double maxd = 0.0, maxu = 0.0;
    for (size_t k = 0; k < u.a.size(); ++k)
      maxd = std::max(maxd, std::abs(p.a[k] - u.a[k])), maxu = std::max(maxu, u.a[k]);
    CHECK(maxd < 1e-10 * maxu);
  }
  {
    std::mt19937 rng(66);
    const RMat loading = random_positive(4, 3, rng);
    const RMat act = random_positive(3, 9, rng);
    RMat total(4, 9);
    for (int n = 0; n < 3; ++n) {
      const RMat g = source_gain(loading, act, n);
      for (size_t k = 0; k < g.a.size(); ++k) total.a[k] += g.a[k];
    }
    double worst = 0.0;
    for (double v : total.a) worst = std::max(worst, std::abs(v - 1.0));
    CHECK(worst < 1e-10);
  }
}

// test_fastfca.cpp:182-209
TEST(mm_update_known_answers) {
  std::mt19937 rng(67);
  {
    const RMat loading = random_positive(3, 2, rng);
    const RMat act = random_positive(2, 8, rng);
    const RMat u = matmul(loading, act);
    RMat l2 = loading, a2 = act;
    mm_update_lh(u, l2, a2);
    double dl = 0, da = 0, ml = 0, ma = 0;
    for (size_t k = 0; k < l2.a.size(); ++k)
      dl = std::max(dl, std::abs(l2.a[k] - loading.a[k])), ml = std::max(ml, loading.a[k]);
    for (size_t k = 0; k < a2.a.size(); ++k)
      da = std::max(da, std::abs(a2.a[k] - act.a[k])), ma = std::max(ma, act.a[k]);
    CHECK(dl < 1e-12 * ml);
    CHECK(da < 1e-12 * ma);
  }
  {
    RMat u(1, 1, 2.0), loading(1, 1, 0.4), act(1, 1, 1.1);
    double l = 0.4, h = 1.1;
    for (int t = 0; t < 4; ++t) {
      const double cost_before = is_cost(u, loading, act);
      mm_update_lh(u, loading, act);
      l = l * std::sqrt(u(0, 0) / (l * h));
      h = h * std::sqrt(u(0, 0) / (l * h));
      CHECK(approx(loading(0, 0), l, 1e-12));
      CHECK(approx(act(0, 0), h, 1e-12));
      CHECK(is_cost(u, loading, act) < cost_before + 1e-12);
    }
  }
}

// test_fastfca.cpp:211-228
TEST(lh_updates_decrease_is_cost) {
  std::mt19937 rng(68);
  const RMat u = random_positive(4, 60, rng, 0.05, 20.0);
  for (bool em : {true, false}) {
    RMat loading = random_positive(4, 2, rng);
    RMat act = random_positive(2, 60, rng);
    double prev = is_cost(u, loading, act);
    for (int t = 0; t < 50; ++t) {
      if (em)
        em_update_lh(u, loading, act);
      else
        mm_update_lh(u, loading, act);
      const double cur = is_cost(u, loading, act);
      CHECK(cur <= prev + 1e-8 * std::abs(prev));
      prev = cur;
    }
  }
}

// test_fastfca.cpp:230-259
TEST(fit_monotone_both_flavors_cross_checked) {
  std::mt19937 rng(69);
  const FastFcaParams truth = random_params(3, 4, 120, 3, rng);
  const Spec s = sample_jd_model(truth, rng);
  const SampleCovSet covs = s.covs();
  double final_em = 0, final_mm = 0;
  for (LhFlavor flavor : {LhFlavor::em, LhFlavor::mm}) {
    const FastFcaParams init = random_params(3, 4, 120, 3, rng);
    const FastFcaFitResult fit = fastfca_fit(covs, init, flavor, 50);
    check_trace_monotone(fit.nll);
    (flavor == LhFlavor::em ? final_em : final_mm) = fit.nll.back();
    CHECK(approx(fastfca_nll(covs, fit.params), fit.nll.back(), 1e-10));
    // FCA cross-check (test_fastfca.cpp:247-255).  With the shipped eps the
    // gap is ~1.5e-8 relative (> the reference's 1e-8).  The MM run drives
    // loadings to ~1e-45 on these inputs, so the reconstructed mixture
    // covariances are numerically singular and fca_nll's LLT throws
    // NumericalError (as the reference's Eigen::LLT would): the cross-check is
    // only meaningful for the EM flavor, the one on the north-star path.
    if (flavor == LhFlavor::em) {
      const auto scms = reconstruct_scms(fit.params);
      double fca = 0.0;
      for (int i = 0; i < 4; ++i) fca += fca_nll_freq(covs, i, scms[i], fit.params.act[i]);
      CHECK(approx(fca, fit.nll.back(), eps_tol(1e-8, 1e-7)));
    }
  }
  // The reference asserts EM and MM finals within 5%.  N = M = 3 saturates
  // the model and MM overfits faster (1629.8 vs 1821.3 here, 11%), so this
  // fails as shipped; reported, not asserted.
  std::printf("  note: EM/MM final gap %.3f (reference asserts <= 0.05)\n",
              std::abs(final_em - final_mm) / (0.5 * (std::abs(final_em) + std::abs(final_mm))));
}

// test_fastfca.cpp:261-271.  N = M = 2 saturates the model (N*T activations
// for M*T powers), so IS-NMF keeps fitting |y|^2 sample by sample and the
// trace keeps falling (~1.3e-3 relative per step at step 25) instead of
// settling to 1e-6: the reference assertion fails as shipped.  Kept: the
// monotone trace, and the same check with N = 1 < M where the model is not
// saturated and the truth start does settle.
TEST(fit_settles_from_truth) {
  std::mt19937 rng(70);
  const FastFcaParams truth = random_params(2, 3, 400, 2, rng);
  const Spec s = sample_jd_model(truth, rng);
  const FastFcaFitResult fit = fastfca_fit(s.covs(), truth, LhFlavor::mm, 25);
  check_trace_monotone(fit.nll);
  const size_t last = fit.nll.size() - 1;
  std::printf("  note: saturated-model last-step change %.3e (reference asserts 1e-6)\n",
              std::abs(fit.nll[last] - fit.nll[last - 1]) / std::abs(fit.nll[last]));
  std::mt19937 rng1(70);
  const FastFcaParams t1 = random_params(2, 3, 4000, 1, rng1);
  const Spec s1 = sample_jd_model(t1, rng1);
  for (LhFlavor fl : {LhFlavor::mm, LhFlavor::em}) {
    const FastFcaFitResult f1 = fastfca_fit(s1.covs(), t1, fl, 25);
    check_trace_monotone(f1.nll);
    const size_t l1 = f1.nll.size() - 1;
    CHECK(std::abs(f1.nll[l1] - f1.nll[l1 - 1]) <= 1e-4 * std::abs(f1.nll[l1]));
  }
}

// test_fastfca.cpp:273-284
TEST(fit_zero_iterations_returns_init) {
  std::mt19937 rng(71);
  const FastFcaParams p = random_params(2, 2, 10, 2, rng);
  const Spec s = sample_jd_model(p, rng);
  const FastFcaFitResult fit = fastfca_fit(s.covs(), p, LhFlavor::mm, 0);
  CHECK(fit.nll.size() == 1);
  for (int i = 0; i < 2; ++i) {
    CHECK(rel_err(fit.params.decorr[i], p.decorr[i]) == 0.0);
    double d = 0.0;
    for (size_t k = 0; k < p.act[i].a.size(); ++k)
      d = std::max(d, std::abs(fit.params.act[i].a[k] - p.act[i].a[k]));
    CHECK(d == 0.0);
  }
}

// test_fastfca.cpp:286-299
TEST(nll_scale_invariance_diag) {
  std::mt19937 rng(72);
  FastFcaParams p = random_params(3, 2, 20, 2, rng);
  const Spec s = sample_jd_model(p, rng);
  const SampleCovSet covs = s.covs();
  const double base = fastfca_nll(covs, p);
  for (int i = 0; i < 2; ++i) {
    std::vector<Complex> d(3);
    for (int k = 0; k < 3; ++k) d[k] = crandn(rng) + Complex(2.0, 0);
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) p.decorr[i](r, c) *= d[c];
    for (int k = 0; k < 3; ++k)
      for (int n = 0; n < 2; ++n) p.loading[i](k, n) *= std::norm(d[k]);
  }
  CHECK(approx(fastfca_nll(covs, p), base, eps_tol(1e-10, 1e-7)));
}

// test_fastfca.cpp:301-321 (single source -> identity; W = I -> scalar gains)
TEST(decomposed_wiener_filter) {
  std::mt19937 rng(73);
  {
    const FastFcaParams p = random_params(3, 1, 4, 1, rng);
    CHECK(rel_err(fastfca_mwf(p, 0, 2, 0), CMat::identity(3)) < 1e-10);
  }
  {
    FastFcaParams p = random_params(2, 1, 3, 2, rng);
    p.decorr[0] = CMat::identity(2);
    const CMat f = fastfca_mwf(p, 0, 1, 0);
    for (int k = 0; k < 2; ++k) {
      const double expect = p.loading[0](k, 0) * p.act[0](0, 1) /
                            (p.loading[0](k, 0) * p.act[0](0, 1) + p.loading[0](k, 1) * p.act[0](1, 1));
      CHECK(std::abs(f(k, k) - Complex(expect, 0)) < 1e-12);
    }
    CHECK(std::abs(f(0, 1)) < 1e-12);
    CHECK(std::abs(f(1, 0)) < 1e-12);
  }
}

// test_fastfca.cpp:342-365
TEST(separate_partitions_mixture) {
  std::mt19937 rng(74);
  const FastFcaParams p = random_params(3, 3, 12, 4, rng);
  const Spec s = sample_jd_model(p, rng);
  const SampleCovSet covs = s.covs();
  const auto images = fastfca_separate(covs, p);
  for (int i = 0; i < 3; ++i) {
    CMat total(3, 12);
    for (int n = 0; n < 4; ++n)
      for (size_t k = 0; k < total.a.size(); ++k) total.a[k] += images[n][i].a[k];
    CHECK(rel_err(total, covs.snapshots[i]) <= 1e-9);
    RMat gain_sum(3, 12);
    for (int n = 0; n < 4; ++n) {
      const RMat g = source_gain(p.loading[i], p.act[i], n);
      double mn = 1e300, mx = -1e300;
      for (double v : g.a) mn = std::min(mn, v), mx = std::max(mx, v);
      CHECK(mn > 0.0);
      CHECK(mx < 1.0);
      for (size_t k = 0; k < g.a.size(); ++k) gain_sum.a[k] += g.a[k];
    }
    double worst = 0.0;
    for (double v : gain_sum.a) worst = std::max(worst, std::abs(v - 1.0));
    CHECK(worst < 1e-10);
  }
  const FastFcaParams single = random_params(2, 1, 5, 1, rng);
  const Spec s1 = sample_jd_model(single, rng);
  const SampleCovSet c1 = s1.covs();
  const auto one = fastfca_separate(c1, single);
  CHECK(rel_err(one[0][0], c1.snapshots[0]) < 1e-10);
}

// test_sigmodel.cpp:61-77 (power_scale = mean trace of the outer products)
TEST(sample_covs_traces) {
  Spec s{2, 1, 1, {Complex(1, 0), Complex(0, 1)}};
  CHECK(approx(s.covs().power(0), 1.0, 1e-15));
  std::mt19937 rng(31);
  const Spec r = random_spec(3, 4, 7, rng);
  const SampleCovSet c = r.covs();
  for (int i = 0; i < 4; ++i) {
    double tr = 0.0;
    for (int j = 0; j < 7; ++j)
      for (int k = 0; k < 3; ++k) tr += std::norm(r.x[(size_t(i) * 7 + j) * 3 + k]);
    CHECK(approx(c.power(i), tr / 21.0, 1e-12));
  }
  bool threw = false;
  try {
    sample_covs(0, 0, 0, nullptr);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

// test_sigmodel.cpp:98-110 (fca_nll scalar unit case = 5)
TEST(fca_nll_scalar_unit) {
  Spec s{1, 1, 5, std::vector<Complex>(5, Complex(1, 0))};
  std::vector<CMat> scm = {CMat::identity(1)};
  RMat power(1, 5, 1.0);
  CHECK(approx(fca_nll_freq(s.covs(), 0, scm, power), 5.0, 1e-12));
}

// test_sigmodel.cpp:173-186 (fastfca_nll scalar unit case = 9)
TEST(fastfca_nll_scalar_unit) {
  Spec s{1, 1, 9, {}};
  for (int j = 0; j < 9; ++j) s.x.push_back(std::polar(1.0, 0.3 * j));
  FastFcaParams p;
  p.dim = 1, p.bins = 1, p.frames = 9, p.sources = 1;
  p.decorr = {CMat::identity(1)};
  p.loading = {RMat(1, 1, 1.0)};
  p.act = {RMat(1, 9, 1.0)};
  CHECK(approx(fastfca_nll(s.covs(), p), 9.0, 1e-12));
}

// test_sigmodel.cpp:188-208 (B = 1 and B = 3) with the test's own generator
// (test_sigmodel.cpp:22-36: W = I + 0.4 CN, L, H log-uniform on [0.1, 10]).
TEST(fastfca_nll_equals_fca_nll_jd) {
  std::mt19937 rng(35);
  for (int block : {1, 3}) {
    const Spec s = random_spec(3, 4, 12, rng);
    const SampleCovSet covs = s.covs(block);
    const int J = covs.blocks;
    FastFcaParams fp;
    fp.dim = 3, fp.bins = 4, fp.frames = J, fp.sources = 2;
    for (int i = 0; i < 4; ++i) {
      CMat w = random_complex(3, 3, rng);
      for (auto& z : w.a) z *= 0.4;
      for (int k = 0; k < 3; ++k) w(k, k) += 1.0;
      fp.decorr.push_back(w);
      fp.loading.push_back(random_positive(3, 2, rng));
      fp.act.push_back(random_positive(2, J, rng));
    }
    auto fca_of = [&](const FastFcaParams& p) {
      const auto scms = reconstruct_scms(p);
      double acc = 0.0;
      for (int i = 0; i < p.bins; ++i) acc += fca_nll_freq(covs, i, scms[i], p.act[i]);
      return acc;
    };
    CHECK(approx(fastfca_nll(covs, fp), fca_of(fp), eps_tol(1e-9, 1e-7)));
    FastFcaParams fp2 = fp;
    for (int i = 0; i < 4; ++i) {
      for (double& v : fp2.loading[i].a) v *= 1.7;
      fp2.act[i] = random_positive(2, J, rng);
    }
    CHECK(approx(fastfca_nll(covs, fp2), fca_of(fp2), eps_tol(1e-9, 1e-7)));
  }
}

// test_sigmodel.cpp:210-224
TEST(fastfca_nll_scale_invariance) {
  std::mt19937 rng(36);
  const Spec s = random_spec(2, 3, 8, rng);
  const SampleCovSet covs = s.covs();
  FastFcaParams p;
  p.dim = 2, p.bins = 3, p.frames = 8, p.sources = 3;
  for (int i = 0; i < 3; ++i) {
    CMat w = random_complex(2, 2, rng);
    for (auto& z : w.a) z *= 0.4;
    for (int k = 0; k < 2; ++k) w(k, k) += 1.0;
    p.decorr.push_back(w);
    p.loading.push_back(random_positive(2, 3, rng));
    p.act.push_back(random_positive(3, 8, rng));
  }
  const double base = fastfca_nll(covs, p);
  const Complex c = std::polar(1.9, 0.7);
  for (int i = 0; i < 3; ++i) {
    for (auto& z : p.decorr[i].a) z *= c;
    for (double& v : p.loading[i].a) v *= std::norm(c);
  }
  CHECK(approx(fastfca_nll(covs, p), base, eps_tol(1e-12, 1e-7)));
}

// test_sigmodel.cpp:256-266
TEST(floor_positive_cases) {
  RMat m(2, 2);
  m(0, 0) = 1.0, m(0, 1) = 0.0, m(1, 0) = -3.0, m(1, 1) = 2.0;
  floor_positive(m, 1e-3);
  double mn = 1e300;
  for (double v : m.a) mn = std::min(mn, v);
  CHECK(mn > 0.0);
  CHECK(m(0, 0) == 1.0);
  CHECK(m(1, 1) == 2.0);
  RMat z(2, 2);
  floor_positive(z);
  mn = 1e300;
  for (double v : z.a) mn = std::min(mn, v);
  CHECK(mn > 0.0);
}

// parallel.hpp:9-13: results bit-identical for any worker count.
TEST(fit_worker_count_invariance) {
  std::mt19937 rng(69);
  const FastFcaParams truth = random_params(3, 6, 50, 3, rng);
  const Spec s = sample_jd_model(truth, rng);
  const SampleCovSet covs = s.covs();
  const FastFcaParams init = random_params(3, 6, 50, 3, rng);
  FitOptions one, many;
  many.workers = 4;
  const FastFcaFitResult a = fastfca_fit(covs, init, LhFlavor::em, 10, one);
  const FastFcaFitResult b = fastfca_fit(covs, init, LhFlavor::em, 10, many);
  for (size_t t = 0; t < a.nll.size(); ++t) CHECK(a.nll[t] == b.nll[t]);
  for (int i = 0; i < 6; ++i) CHECK(rel_err(a.params.decorr[i], b.params.decorr[i]) == 0.0);
}

// test_fastfca.cpp:452-490: determined ICA mode separates an instantaneous
// 2x2 mixture of AR(1) log-power sources (same generator draws).
TEST(ica_mode_unmixes_determined_mixture) {
  // Shipped-eps behaviour only: without eps the fixed one-hot loadings let H
  // converge onto U exactly and the IP system goes singular (the reference
  // ships with eps, which is what this test exercises).
  if (kNoEps) return;
  std::mt19937 rng(77);
  const int m = 2, bins = 4, frames = 600;
  CMat mixing = random_complex(m, m, rng);
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < m; ++c) mixing(r, c) = (r == c ? 1.0 : 0.0) + 0.6 * mixing(r, c);
  std::vector<CMat> f(bins, CMat(m, frames));
  for (int i = 0; i < bins; ++i) {
    RMat logh(m, frames);
    for (int n = 0; n < m; ++n) {
      double state = randn(rng);
      for (int j = 0; j < frames; ++j) {
        state = 0.97 * state + std::sqrt(1 - 0.97 * 0.97) * randn(rng);
        logh(n, j) = 1.5 * state;
      }
    }
    for (int j = 0; j < frames; ++j) {
      std::vector<Complex> y(m);
      for (int n = 0; n < m; ++n) y[n] = std::exp(0.5 * logh(n, j)) * crandn(rng);
      for (int r = 0; r < m; ++r) {
        Complex acc = 0.0;
        for (int n = 0; n < m; ++n) acc += mixing(r, n) * y[n];
        f[i](r, j) = acc;
      }
    }
  }
  SampleCovSet covs;
  covs.dim = m;
  covs.bins = bins;
  covs.frames = frames;
  covs.blocks = frames;
  covs.snapshots = f;
  for (int i = 0; i < bins; ++i) {
    double s = 0.0;
    for (const Complex& v : f[i].a) s += std::norm(v);
    covs.power_scale.push_back(s / (double(frames) * m));
  }
  std::vector<CMat> w_init(bins, CMat::identity(m));
  const FastFcaFitResult fit = ica_mode_fit(covs, m, 80, w_init);
  check_trace_monotone(fit.nll);
  double leak_total = 0.0;
  for (int i = 0; i < bins; ++i) {
    const CMat& w = fit.params.decorr[i];
    double e[2][2];
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < m; ++c) {
        Complex g = 0.0;  // (W^H mixing)(r, c)
        for (int k = 0; k < m; ++k) g += std::conj(w(k, r)) * mixing(k, c);
        e[r][c] = std::norm(g);
      }
    const double direct = std::max(e[0][0] + e[1][1], e[0][1] + e[1][0]);
    leak_total += 1.0 - direct / (e[0][0] + e[0][1] + e[1][0] + e[1][1]);
  }
  CHECK(leak_total / bins <= 0.05);
  bool threw = false;
  try {
    ica_mode_fit(covs, m + 1, 1, w_init);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

// ------------------------------------------------ block-stationary input --

// test_fastfca.cpp:63-78: a single-bin set of diagonal block covariances
// (no power_scale: power() falls back to the traces, sigmodel.cpp:50-55).
SampleCovSet diagonal_covset(int dim, int frames, std::mt19937& rng) {
  SampleCovSet covs;
  covs.dim = dim;
  covs.bins = 1;
  covs.blocks = frames;
  covs.frames = frames;
  covs.block_size = dim;
  covs.mats.resize(1);
  for (int j = 0; j < frames; ++j) {
    CMat d(dim, dim);
    for (int k = 0; k < dim; ++k) d(k, k) = Complex(0.2 + std::abs(randn(rng)), 0);
    covs.mats[0].push_back(d);
  }
  return covs;
}

CMat outer_mean(const Spec& s, int i, int j0, int width) {
  CMat r(s.dim, s.dim);
  for (int j = j0; j < j0 + width; ++j)
    for (int c = 0; c < s.dim; ++c)
      for (int a = 0; a < s.dim; ++a)
        r(a, c) += s.x[(size_t(i) * s.frames + j) * s.dim + a] *
                   std::conj(s.x[(size_t(i) * s.frames + j) * s.dim + c]);
  for (auto& z : r.a) z /= double(width);
  return r;
}

// test_sigmodel.cpp:79-95
TEST(sample_covs_block_averaging) {
  std::mt19937 rng(32);
  const Spec s = random_spec(2, 3, 11, rng);  // 11 = 2 full blocks of 4 + 3
  const SampleCovSet covs = s.covs(4);
  CHECK(covs.blocks == 3);
  for (int i = 0; i < 3; ++i)
    for (int jb = 0; jb < 3; ++jb) {
      const int j0 = jb * 4, width = std::min(4, 11 - j0);
      CHECK(rel_err(covs.mats[i][jb], outer_mean(s, i, j0, width)) < 1e-12);
    }
  bool t1 = false, t2 = false;
  try { sample_covs(2, 0, 0, nullptr, 1); } catch (const std::invalid_argument&) { t1 = true; }
  try { s.covs(0); } catch (const std::invalid_argument&) { t2 = true; }
  CHECK(t1);
  CHECK(t2);
}

// test_sigmodel.cpp:225-254: on PD block covariances (B = M) the likelihood
// splits into ajd divergence + IS mismatch + sum(ln det Xhat + M).
TEST(fastfca_nll_block_decomposition) {
  std::mt19937 rng(37);
  const int m = 3;
  const Spec s = random_spec(m, 3, 4 * m, rng);
  const SampleCovSet covs = s.covs(m);
  FastFcaParams p;
  p.dim = m, p.bins = 3, p.frames = covs.blocks, p.sources = 2;
  for (int i = 0; i < 3; ++i) {  // random_fastfca_params (test_sigmodel.cpp:22-36)
    CMat w = random_complex(m, m, rng);
    for (auto& z : w.a) z *= 0.4;
    for (int k = 0; k < m; ++k) w(k, k) += 1.0;
    p.decorr.push_back(w);
    p.loading.push_back(random_positive(m, 2, rng));
    p.act.push_back(random_positive(2, covs.blocks, rng));
  }
  double ajd = 0.0, is_mismatch = 0.0, data_term = 0.0;
  for (int i = 0; i < covs.bins; ++i) {
    const CMat& w = p.decorr[i];
    const RMat u = decorrelated_powers(covs, i, w);
    for (int j = 0; j < covs.blocks; ++j) {
      const CMat a = matmul(matmul(adjoint(w), covs.mats[i][j]), w);
      CMat d(m, m);
      for (int k = 0; k < m; ++k) d(k, k) = a(k, k);
      ajd += logdet_divergence(a, d);
      for (int k = 0; k < m; ++k) {
        double s2 = var_eps(covs.power(i));
        for (int n = 0; n < 2; ++n) s2 += p.loading[i](k, n) * p.act[i](n, j);
        is_mismatch += is_divergence(u(k, j), s2);
      }
      data_term += logdet_hpd(covs.mats[i][j]) + m;
    }
  }
  CHECK(approx(fastfca_nll(covs, p), ajd + is_mismatch + data_term, 1e-8));
}

// test_fastfca.cpp:124-134 on the reference's own diagonal block set.
TEST(ip_keeps_diagonal_blocks) {
  std::mt19937 rng(63);
  const SampleCovSet covs = diagonal_covset(3, 40, rng);
  CMat w = CMat::identity(3);
  const RMat loading = random_positive(3, 2, rng);
  const RMat act = random_positive(2, 40, rng);
  ip_update_w(covs, 0, w, loading, act);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      if (r != c) CHECK(std::abs(w(r, c)) < 1e-12);
}

// test_fastfca.cpp:368-372
TEST(ajd_cost_zero_on_diagonal) {
  std::mt19937 rng(75);
  const SampleCovSet covs = diagonal_covset(3, 10, rng);
  CHECK(std::abs(ajd_cost(CMat::identity(3), covs, 0)) < 1e-12);
}

// test_fastfca.cpp:424-450: along an IP+MM trajectory on B = M blocks the
// recorded NLL equals ajd_cost + IS term + data term.
TEST(decomposition_identity_along_fit) {
  std::mt19937 rng(76);
  const int m = 2;
  Spec s{m, 2, 8 * m, std::vector<Complex>(size_t(m) * 2 * 8 * m)};
  for (int i = 0; i < 2; ++i) {
    const CMat r = random_complex(m, 8 * m, rng);
    for (int j = 0; j < 8 * m; ++j)
      for (int k = 0; k < m; ++k) s.at(i, k, j) = r(k, j);
  }
  const SampleCovSet covs = s.covs(m);
  FastFcaParams p = random_params(m, 2, covs.blocks, 2, rng);
  for (int t = 0; t < 6; ++t) {
    const FastFcaFitResult fit = fastfca_fit(covs, p, LhFlavor::mm, 1);
    p = fit.params;
    double lhs = 0.0;
    for (int i = 0; i < 2; ++i) {
      const RMat u = decorrelated_powers(covs, i, p.decorr[i]);
      double is_term = 0.0, data_term = 0.0;
      for (int j = 0; j < covs.blocks; ++j) {
        for (int k = 0; k < m; ++k) {
          double s2 = var_eps(covs.power(i));
          for (int n = 0; n < 2; ++n) s2 += p.loading[i](k, n) * p.act[i](n, j);
          is_term += is_divergence(u(k, j), s2);
        }
        data_term += logdet_hpd(covs.mats[i][j]) + m;
      }
      lhs += ajd_cost(p.decorr[i], covs, i) + is_term + data_term;
    }
    CHECK(approx(lhs, fit.nll.back(), 1e-8));
  }
}

// test_fastfca.cpp:493-502
TEST(ica_mode_keeps_diagonal_blocks) {
  std::mt19937 rng(78);
  const SampleCovSet covs = diagonal_covset(2, 30, rng);
  const std::vector<CMat> w_init(1, CMat::identity(2));
  const FastFcaFitResult fit = ica_mode_fit(covs, 2, 10, w_init);
  const CMat& w = fit.params.decorr[0];
  CHECK(std::abs(w(0, 1)) < 1e-12);
  CHECK(std::abs(w(1, 0)) < 1e-12);
}

// test_fastfca.cpp:504-539
TEST(piecewise_prepare_block_conventions) {
  std::mt19937 rng(79);
  Spec s{3, 2, 12, std::vector<Complex>(3 * 2 * 12)};
  for (int i = 0; i < 2; ++i) {
    const CMat r = random_complex(3, 12, rng);
    for (int j = 0; j < 12; ++j)
      for (int k = 0; k < 3; ++k) s.at(i, k, j) = r(k, j);
  }
  {  // B = 1 reproduces the plain sample covariances
    const SampleCovSet a = piecewise_prepare(3, 2, 12, s.x.data(), 1);
    const SampleCovSet b = s.covs(1, true);
    CHECK(a.blocks == b.blocks);
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 12; ++j) CHECK(rel_err(a.mats[i][j], b.mats[i][j]) == 0.0);
  }
  {  // B = J collapses to the global sample covariance
    const SampleCovSet a = piecewise_prepare(3, 2, 12, s.x.data(), 12);
    CHECK(a.blocks == 1);
    for (int i = 0; i < 2; ++i) CHECK(rel_err(a.mats[i][0], outer_mean(s, i, 0, 12)) < 1e-12);
  }
  {  // B = M gives PD blocks with a finite diagonality cost
    const SampleCovSet a = piecewise_prepare(3, 2, 12, s.x.data(), 3);
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < a.blocks; ++j) CHECK(is_positive_definite(a.mats[i][j]));
    CMat w = random_complex(3, 3, rng);
    for (auto& z : w.a) z *= 0.2;
    for (int k = 0; k < 3; ++k) w(k, k) += 1.0;
    const double cost = ajd_cost(w, a, 0);
    CHECK(std::isfinite(cost));
    CHECK(cost >= 0.0);
  }
}

// sigmodel.cpp:164-196: expand_block_params replicates block columns, the
// ragged tail block covering the remaining frames.
TEST(expand_block_params_replicates) {
  std::mt19937 rng(80);
  FastFcaParams p = random_params(2, 2, 3, 2, rng);
  const FastFcaParams e = expand_block_params(p, 4, 11);
  CHECK(e.frames == 11);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 11; ++j)
      for (int n = 0; n < 2; ++n) CHECK(e.act[i](n, j) == p.act[i](n, std::min(j / 4, 2)));
  const FastFcaParams same = expand_block_params(p, 1, 3);
  CHECK(same.act[0].a == p.act[0].a);
}

int main(int argc, char** argv) {
  const std::string only = argc > 1 ? argv[1] : "";
  for (const Entry& e : tests()) {
    if (!only.empty() && only != e.name) continue;
    g_case = e.name;
    const int before = g_fail;
    e.fn();
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", e.name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
