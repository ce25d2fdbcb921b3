// oracle_capi.cpp -- TEST INFRASTRUCTURE ONLY.  C entry points over the fp64
// restatement (oracle.cpp) so pytest (ctypes) and bench.py's cpu_baseline leg
// can drive it.  Buffers use the reference's Eigen layouts (oracle.hpp);
// x is [batch][bins][frames][dim] complex (re, im interleaved), i.e.
// Spectrogram::f[i] column-major (stft.hpp:21-29).
//
// Status codes mirror include/ffca.h: 0 ok, 1 std::invalid_argument,
// 2 NumericalError (types.hpp:21-24), 3 anything else.

#include <chrono>
#include <cstring>
#include <cstdint>

#include "oracle.hpp"

using namespace oracle;

namespace {

int fail(char* err, int errlen, int code, const char* what) {
  if (err && errlen > 0) {
    std::strncpy(err, what, size_t(errlen) - 1);
    err[errlen - 1] = 0;
  }
  return code;
}

template <typename F>
int guard(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const NumericalError& e) {
    return fail(err, errlen, 2, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(err, errlen, 1, e.what());
  } catch (const std::exception& e) {
    return fail(err, errlen, 3, e.what());
  }
}

const Complex* cx(const double* p) { return reinterpret_cast<const Complex*>(p); }
Complex* cx(double* p) { return reinterpret_cast<Complex*>(p); }

FastFcaParams load_params(int bins, int dim, int sources, int frames, const double* W,
                          const double* L, const double* H) {
  FastFcaParams p;
  p.dim = dim, p.bins = bins, p.frames = frames, p.sources = sources;
  for (int i = 0; i < bins; ++i) {
    CMat w(dim, dim);
    std::memcpy(w.data(), W + size_t(i) * dim * dim * 2, sizeof(Complex) * dim * dim);
    RMat l(dim, sources);
    std::memcpy(l.data(), L + size_t(i) * dim * sources, sizeof(double) * dim * sources);
    RMat h(sources, frames);
    std::memcpy(h.data(), H + size_t(i) * sources * frames, sizeof(double) * sources * frames);
    p.decorr.push_back(std::move(w));
    p.loading.push_back(std::move(l));
    p.act.push_back(std::move(h));
  }
  return p;
}

void store_params(const FastFcaParams& p, double* W, double* L, double* H) {
  const int dim = p.dim, sources = p.sources, frames = p.frames;
  for (int i = 0; i < p.bins; ++i) {
    std::memcpy(W + size_t(i) * dim * dim * 2, p.decorr[i].data(), sizeof(Complex) * dim * dim);
    std::memcpy(L + size_t(i) * dim * sources, p.loading[i].data(), sizeof(double) * dim * sources);
    std::memcpy(H + size_t(i) * sources * frames, p.act[i].data(),
                sizeof(double) * sources * frames);
  }
}

// SampleCovSet from caller block covariances [bins][blocks][dim*dim] complex
// (Eigen col-major per block); power (nullable) -> power_scale, else
// power() falls back to the traces (sigmodel.cpp:50-55).
SampleCovSet covs_from_mats(int bins, int dim, int blocks, const double* mats,
                            const double* power) {
  SampleCovSet c;
  c.dim = dim, c.bins = bins, c.blocks = blocks, c.frames = blocks;
  c.block_size = 0;  // unknown for a caller-built set; unused by the path
  c.mats.resize(bins);
  for (int i = 0; i < bins; ++i)
    for (int j = 0; j < blocks; ++j) {
      CMat m(dim, dim);
      std::memcpy(static_cast<void*>(m.data()), mats + (size_t(i) * blocks + j) * dim * dim * 2,
                  sizeof(Complex) * dim * dim);
      c.mats[i].push_back(std::move(m));
    }
  if (power) c.power_scale.assign(power, power + bins);
  return c;
}

}  // namespace

extern "C" {

// sample_covs(spec, block_size) (sigmodel.cpp:17-48): mats out
// [bins][blocks][dim*dim] complex (nullable), power out [bins] (nullable).
int oracle_block_covs(int bins, int dim, int frames, int block_size, const double* x,
                      double* mats, double* power, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet c = sample_covs(dim, bins, frames, cx(x), block_size, true);
    for (int i = 0; i < bins; ++i) {
      if (power) power[i] = c.power_scale[i];
      if (mats)
        for (int j = 0; j < c.blocks; ++j)
          std::memcpy(static_cast<void*>(mats + (size_t(i) * c.blocks + j) * dim * dim * 2),
                      c.mats[i][j].data(), sizeof(Complex) * dim * dim);
    }
  });
}

// fastfca_fit / ica_mode_fit on block covariances (the mats branches of
// weighted_cov and decorrelated_powers); layouts as oracle_fit with frames =
// blocks.  ica != 0: W in = w_init; L, H outputs; flavor etc. ignored.
int oracle_fit_covs(int bins, int dim, int sources, int blocks, const double* mats,
                    const double* power, double* W, double* L, double* H, int flavor, int iters,
                    int record_trace, uint64_t seed, int normalize_scales, int fix_loadings,
                    int workers, int ica, double* nll, double* nll_slots, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = covs_from_mats(bins, dim, blocks, mats, power);
    FitOptions fo;
    fo.workers = workers;
    fo.record_trace = record_trace != 0;
    fo.seed = seed;
    std::vector<double> slots;
    FastFcaFitResult r;
    if (ica) {
      std::vector<CMat> w_init(bins, CMat(dim, dim));
      for (int i = 0; i < bins; ++i)
        std::memcpy(static_cast<void*>(w_init[i].data()), W + size_t(i) * dim * dim * 2,
                    sizeof(Complex) * dim * dim);
      r = ica_mode_fit(covs, sources, iters, w_init, fo, nll_slots ? &slots : nullptr);
    } else {
      const FastFcaParams init = load_params(bins, dim, sources, blocks, W, L, H);
      FastFcaOptions oo;
      oo.normalize_scales = normalize_scales != 0;
      oo.fix_loadings = fix_loadings != 0;
      r = fastfca_fit(covs, init, flavor == 0 ? LhFlavor::em : LhFlavor::mm, iters, fo, oo,
                      nll_slots ? &slots : nullptr);
    }
    store_params(r.params, W, L, H);
    if (record_trace && nll)
      for (int t = 0; t <= iters; ++t) nll[t] = r.nll[t];
    if (record_trace && nll_slots)
      std::memcpy(nll_slots, slots.data(), sizeof(double) * slots.size());
  });
}

int oracle_nll_bins_covs(int bins, int dim, int sources, int blocks, const double* mats,
                         const double* W, const double* L, const double* H, double* out,
                         char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = covs_from_mats(bins, dim, blocks, mats, nullptr);
    const FastFcaParams p = load_params(bins, dim, sources, blocks, W, L, H);
    for (int i = 0; i < bins; ++i)
      out[i] = fastfca_nll_freq(covs, i, p.decorr[i], p.loading[i], p.act[i]);
  });
}

int oracle_decorrelated_powers_covs(int bins, int dim, int blocks, const double* mats,
                                    const double* W, double floor_rel, double* out, char* err,
                                    int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = covs_from_mats(bins, dim, blocks, mats, nullptr);
    for (int i = 0; i < bins; ++i) {
      CMat w(dim, dim);
      std::memcpy(static_cast<void*>(w.data()), W + size_t(i) * dim * dim * 2,
                  sizeof(Complex) * dim * dim);
      RMat u = decorrelated_powers(covs, i, w);
      if (floor_rel >= 0.0) floor_positive(u, floor_rel);
      std::memcpy(out + size_t(i) * dim * blocks, u.data(), sizeof(double) * dim * blocks);
    }
  });
}

int oracle_default_workers() { return default_workers(); }

// sigmodel.cpp:17-48 power_scale for every bin: out[bins].
int oracle_power_scale(int bins, int dim, int frames, const double* x, double* out, char* err,
                       int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet c = sample_covs(dim, bins, frames, cx(x));
    for (int i = 0; i < bins; ++i) out[i] = c.power_scale[i];
  });
}

// fastfca_fit over a batch of independent mixtures (a loop of fastfca_fit,
// fastfca.cpp:146-191).  W/L/H in/out.  nll: [batch][iters+1] (record_trace).
// nll_slots (nullable): [batch][iters+1][bins] per-bin slots.  fit_seconds
// (nullable): wall time of the fastfca_fit calls only (SampleCovSet prebuilt).
int oracle_fit(int batch, int bins, int dim, int sources, int frames, const double* x, double* W,
               double* L, double* H, int flavor, int iters, int record_trace, uint64_t seed,
               int normalize_scales, int fix_loadings, int workers, double* nll,
               double* nll_slots, double* fit_seconds, char* err, int errlen) {
  return guard(err, errlen, [&] {
    double secs = 0.0;
    for (int b = 0; b < batch; ++b) {
      const size_t xo = size_t(b) * bins * frames * dim * 2;
      const size_t wo = size_t(b) * bins * dim * dim * 2;
      const size_t lo = size_t(b) * bins * dim * sources;
      const size_t ho = size_t(b) * bins * sources * frames;
      const SampleCovSet covs = sample_covs(dim, bins, frames, cx(x + xo));
      FastFcaParams init = load_params(bins, dim, sources, frames, W + wo, L + lo, H + ho);
      FitOptions fo;
      fo.workers = workers;
      fo.record_trace = record_trace != 0;
      fo.seed = seed;
      FastFcaOptions oo;
      oo.normalize_scales = normalize_scales != 0;
      oo.fix_loadings = fix_loadings != 0;
      std::vector<double> slots;
      const auto t0 = std::chrono::steady_clock::now();
      const FastFcaFitResult r =
          fastfca_fit(covs, init, flavor == 0 ? LhFlavor::em : LhFlavor::mm, iters, fo, oo,
                      nll_slots ? &slots : nullptr);
      const auto t1 = std::chrono::steady_clock::now();
      secs += std::chrono::duration<double>(t1 - t0).count();
      store_params(r.params, W + wo, L + lo, H + ho);
      if (record_trace && nll)
        for (int t = 0; t <= iters; ++t) nll[size_t(b) * (iters + 1) + t] = r.nll[t];
      if (record_trace && nll_slots)
        std::memcpy(nll_slots + size_t(b) * (iters + 1) * bins, slots.data(),
                    sizeof(double) * slots.size());
    }
    if (fit_seconds) *fit_seconds = secs;
  });
}

// ica_mode_fit (fastfca.cpp:241-264) on one mixture: W in = w_init, out = the
// fitted W; L out [bins][dim*dim]; H out [bins][dim*frames].
int oracle_ica_fit(int bins, int dim, int sources, int frames, const double* x, double* W,
                   double* L, double* H, int iters, int record_trace, uint64_t seed, int workers,
                   double* nll, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = sample_covs(dim, bins, frames, cx(x));
    std::vector<CMat> w_init(bins, CMat(dim, dim));
    for (int i = 0; i < bins; ++i)
      std::memcpy(static_cast<void*>(w_init[i].data()), W + size_t(i) * dim * dim * 2,
                  sizeof(Complex) * dim * dim);
    FitOptions fo;
    fo.workers = workers;
    fo.record_trace = record_trace != 0;
    fo.seed = seed;
    const FastFcaFitResult r = ica_mode_fit(covs, sources, iters, w_init, fo);
    store_params(r.params, W, L, H);
    if (record_trace && nll)
      for (int t = 0; t <= iters; ++t) nll[t] = r.nll[t];
  });
}

// decorrelated_powers + floor_positive per bin (sigmodel.cpp:10-15, 93-107):
// out [bins][dim*frames] (Eigen col-major dim x frames).
int oracle_decorrelated_powers(int bins, int dim, int frames, const double* x, const double* W,
                               double floor_rel, double* out, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = sample_covs(dim, bins, frames, cx(x));
    for (int i = 0; i < bins; ++i) {
      CMat w(dim, dim);
      std::memcpy(static_cast<void*>(w.data()), W + size_t(i) * dim * dim * 2,
                  sizeof(Complex) * dim * dim);
      RMat u = decorrelated_powers(covs, i, w);
      if (floor_rel >= 0.0) floor_positive(u, floor_rel);
      std::memcpy(out + size_t(i) * dim * frames, u.data(), sizeof(double) * dim * frames);
    }
  });
}

// fastfca_nll_freq per bin (sigmodel.cpp:155-162): out[bins].
int oracle_nll_bins(int bins, int dim, int sources, int frames, const double* x, const double* W,
                    const double* L, const double* H, double* out, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = sample_covs(dim, bins, frames, cx(x));
    const FastFcaParams p = load_params(bins, dim, sources, frames, W, L, H);
    for (int i = 0; i < bins; ++i)
      out[i] = fastfca_nll_freq(covs, i, p.decorr[i], p.loading[i], p.act[i]);
  });
}

// fca_nll of the JD reconstruction (second NLL oracle; test_fastfca.cpp:247-255).
int oracle_fca_nll_jd(int bins, int dim, int sources, int frames, const double* x,
                      const double* W, const double* L, const double* H, double* out, char* err,
                      int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = sample_covs(dim, bins, frames, cx(x));
    const FastFcaParams p = load_params(bins, dim, sources, frames, W, L, H);
    const auto scms = reconstruct_scms(p);
    double acc = 0.0;
    for (int i = 0; i < bins; ++i) acc += fca_nll_freq(covs, i, scms[i], p.act[i]);
    *out = acc;
  });
}

// fastfca_separate (fastfca.cpp:205-223): images [sources][bins][frames][dim] complex.
int oracle_separate(int bins, int dim, int sources, int frames, const double* x, const double* W,
                    const double* L, const double* H, double* images, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = sample_covs(dim, bins, frames, cx(x));
    const FastFcaParams p = load_params(bins, dim, sources, frames, W, L, H);
    const auto img = fastfca_separate(covs, p);
    for (int n = 0; n < sources; ++n)
      for (int i = 0; i < bins; ++i)
        std::memcpy(images + (size_t(n) * bins + i) * frames * dim * 2, img[n][i].data(),
                    sizeof(Complex) * frames * dim);
  });
}

// Kernel-level entry points for the ported unit tests.
int oracle_ip_update_w(int dim, int sources, int frames, const double* x, double* W,
                       const double* L, const double* H, uint64_t seed, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const SampleCovSet covs = sample_covs(dim, 1, frames, cx(x));
    FastFcaParams p = load_params(1, dim, sources, frames, W, L, H);
    ip_update_w(covs, 0, p.decorr[0], p.loading[0], p.act[0], seed);
    std::memcpy(W, p.decorr[0].data(), sizeof(Complex) * dim * dim);
  });
}

int oracle_lh_update(int flavor, int dim, int sources, int frames, const double* u, double* L,
                     double* H, int update_loading, double eps, char* err, int errlen) {
  return guard(err, errlen, [&] {
    RMat um(dim, frames), l(dim, sources), h(sources, frames);
    std::memcpy(um.data(), u, sizeof(double) * dim * frames);
    std::memcpy(l.data(), L, sizeof(double) * dim * sources);
    std::memcpy(h.data(), H, sizeof(double) * sources * frames);
    if (flavor == 0)
      em_update_lh(um, l, h, update_loading != 0, eps);
    else
      mm_update_lh(um, l, h, update_loading != 0, eps);
    std::memcpy(L, l.data(), sizeof(double) * dim * sources);
    std::memcpy(H, h.data(), sizeof(double) * sources * frames);
  });
}

int oracle_source_gain(int dim, int sources, int frames, const double* L, const double* H, int n,
                       double* out, char* err, int errlen) {
  return guard(err, errlen, [&] {
    RMat l(dim, sources), h(sources, frames);
    std::memcpy(l.data(), L, sizeof(double) * dim * sources);
    std::memcpy(h.data(), H, sizeof(double) * sources * frames);
    const RMat g = source_gain(l, h, n);
    std::memcpy(out, g.data(), sizeof(double) * dim * frames);
  });
}

}  // extern "C"
