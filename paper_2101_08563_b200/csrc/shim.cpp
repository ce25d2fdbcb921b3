// shim.cpp -- the reference's C++ API (include/fastfca/*.hpp) on top of the
// C ABI (include/ffca.h).  Host work only: validation with the reference's
// exceptions, gathering the per-bin containers into the contiguous buffers
// the ABI takes, and one host thread per device for frequency sharding.
// All arithmetic runs in libffca.so's sm_100a kernels.

#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "fastfca/fastfca.hpp"
#include "ffca.h"

namespace fastfca {

namespace {

void raise(int rc) {
  if (rc == FFCA_OK) return;
  const std::string msg = ffca_last_error();
  if (rc == FFCA_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == FFCA_NUMERICAL) throw NumericalError(msg);
  throw std::runtime_error("ffca: " + msg);
}

// One context per (host thread, device): contexts are not thread-safe.
ffca_ctx* context(int device) {
  struct Holder {
    std::unordered_map<int, ffca_ctx*> m;
    ~Holder() {
      for (auto& kv : m) ffca_ctx_destroy(kv.second);
    }
  };
  thread_local Holder h;
  auto it = h.m.find(device);
  if (it != h.m.end()) return it->second;
  ffca_ctx* c = nullptr;
  raise(ffca_ctx_create(device, &c));
  h.m[device] = c;
  return c;
}

int prec(const GpuOptions& g) {
  return g.precision == Precision::fp64 ? FFCA_PREC_FP64 : FFCA_PREC_FP32;
}

// Host staging of the ABI's flat buffers.  The large ones (x, H) live in
// page-locked memory owned by the device context (ffca_pinned_buffer), so the
// library's chunked H2D / fit / D2H pipeline runs truly asynchronously; small
// ones (power, W, L) are plain vectors.
struct HostBuf {
  double* p = nullptr;
  size_t n = 0;
  std::vector<double> own;
  void resize(size_t count, ffca_ctx* ctx = nullptr, int slot = -1) {
    n = count;
    p = nullptr;
    if (ctx && slot >= 0 && count > 0)
      p = static_cast<double*>(ffca_pinned_buffer(ctx, slot, count * sizeof(double)));
    if (!p) {
      own.resize(count);
      p = own.data();
    }
  }
  double* data() { return p; }
  const double* data() const { return p; }
  bool empty() const { return n == 0; }
};

// Contiguous host copies of bins in the ABI's (reference) layout.
// x: the snapshots [bin][frame][dim], or for a block set (no snapshots) the
// block covariances [bin][block][dim*dim] (ffca.h *_covs entry points).
// power: power_scale, or empty for a block set without one (the library
// then takes SampleCovSet::power()'s trace fallback, sigmodel.cpp:50-55).
struct Packed {
  HostBuf x, power, W, L, H;
  bool snap = true;
  const double* pw() const { return power.empty() ? nullptr : power.data(); }
};

int host_threads(const GpuOptions& g, int work) {
  int n = g.host_threads > 0 ? g.host_threads : int(std::thread::hardware_concurrency());
  n = std::max(1, std::min(n, 16));
  return std::max(1, std::min(n, work));
}

// fn(i) for i in [0, count) on nt host threads (contiguous ranges).
template <typename Fn>
void parallel_bins(int count, int nt, Fn fn) {
  if (nt <= 1 || count < 2 * nt) {
    for (int i = 0; i < count; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([=] {
      const int lo = int((long long)count * t / nt), hi = int((long long)count * (t + 1) / nt);
      for (int i = lo; i < hi; ++i) fn(i);
    });
  for (auto& t : th) t.join();
}

// Size `out` for `total` bins of this shape; ctx != null puts x and H in the
// context's pinned staging.
void size_packed(const SampleCovSet& covs, int sources, int total, Packed& out, ffca_ctx* ctx) {
  const int M = covs.dim, N = sources, T = covs.blocks;
  out.snap = covs.has_snapshots();
  const size_t rec = out.snap ? size_t(M) * 2 : size_t(M) * M * 2;  // doubles per frame / block
  const bool has_pw = long(covs.power_scale.size()) == covs.bins;
  out.x.resize(size_t(total) * T * rec, ctx, 0);
  out.power.resize(has_pw ? total : 0);
  out.W.resize(size_t(total) * M * M * 2);
  out.L.resize(size_t(total) * M * N);
  out.H.resize(size_t(total) * N * T, ctx, 1);
}

// Bins [lo, hi) of (covs, p) into rows [at, at + hi - lo) of `out`.
void pack_into(const SampleCovSet& covs, const FastFcaParams& p, int lo, int hi, Packed& out,
               int at, int nt) {
  const int M = covs.dim, N = p.sources, T = covs.blocks;
  const size_t rec = out.snap ? size_t(M) * 2 : size_t(M) * M * 2;
  const bool has_pw = !out.power.empty();
  parallel_bins(hi - lo, nt, [&, lo, at](int j) {
    const int i = lo + j;
    const size_t k = size_t(at + j);
    if (out.snap) {
      std::memcpy(out.x.data() + k * T * rec, covs.snapshots[i].data(), sizeof(double) * T * rec);
    } else {
      for (int jb = 0; jb < T; ++jb)
        std::memcpy(out.x.data() + (k * T + jb) * rec, covs.mats[i][jb].data(), sizeof(double) * rec);
    }
    if (has_pw) out.power.data()[k] = covs.power_scale(i);
    std::memcpy(out.W.data() + k * M * M * 2, p.decorr[i].data(), sizeof(double) * M * M * 2);
    std::memcpy(out.L.data() + k * M * N, p.loading[i].data(), sizeof(double) * M * N);
    std::memcpy(out.H.data() + k * N * T, p.act[i].data(), sizeof(double) * N * T);
  });
}

void pack_bins(const SampleCovSet& covs, const FastFcaParams& p, int lo, int hi, Packed& out,
               ffca_ctx* ctx = nullptr, int nt = 1) {
  size_packed(covs, p.sources, hi - lo, out, ctx);
  pack_into(covs, p, lo, hi, out, 0, nt);
}

// Rows [at, at + hi - lo) of `in` into bins [lo, hi) of p.
void unpack_bins(const Packed& in, int lo, int hi, FastFcaParams& p, int at = 0, int nt = 1) {
  const int M = p.dim, N = p.sources, T = p.frames;
  parallel_bins(hi - lo, nt, [&, lo, at](int j) {
    const int i = lo + j;
    const size_t k = size_t(at + j);
    std::memcpy(p.decorr[i].data(), in.W.data() + k * M * M * 2, sizeof(double) * M * M * 2);
    std::memcpy(p.loading[i].data(), in.L.data() + k * M * N, sizeof(double) * M * N);
    std::memcpy(p.act[i].data(), in.H.data() + k * N * T, sizeof(double) * N * T);
  });
}

// A set the kernels can read: snapshots (dim x blocks each) with power_scale,
// or block covariances mats[i][jb] (dim x dim) with power_scale or none.
void check_covs(const SampleCovSet& covs, const char* what) {
  const std::string bad = std::string(what) + ": malformed covariance set";
  if (covs.has_snapshots()) {
    if (int(covs.snapshots.size()) != covs.bins || long(covs.power_scale.size()) != covs.bins)
      throw std::invalid_argument(bad);
    for (const CMat& x : covs.snapshots)
      if (x.rows() != covs.dim || x.cols() != covs.blocks) throw std::invalid_argument(bad);
    return;
  }
  if (int(covs.mats.size()) != covs.bins ||
      (covs.power_scale.size() != 0 && long(covs.power_scale.size()) != covs.bins))
    throw std::invalid_argument(bad);
  for (const auto& mi : covs.mats) {
    if (int(mi.size()) != covs.blocks) throw std::invalid_argument(bad);
    for (const CMat& m : mi)
      if (m.rows() != covs.dim || m.cols() != covs.dim) throw std::invalid_argument(bad);
  }
}

void check_fit_shapes(const SampleCovSet& covs, const FastFcaParams& init) {
  // fastfca.cpp:150-152
  if (init.dim != covs.dim || init.bins != covs.bins || init.frames != covs.blocks)
    throw std::invalid_argument("fastfca_fit: init/covariance shape mismatch");
  check_covs(covs, "fastfca_fit");
  if (int(init.decorr.size()) != init.bins || int(init.loading.size()) != init.bins ||
      int(init.act.size()) != init.bins)
    throw std::invalid_argument("fastfca_fit: init/covariance shape mismatch");
  for (int i = 0; i < init.bins; ++i)
    if (init.decorr[i].rows() != init.dim || init.decorr[i].cols() != init.dim ||
        init.loading[i].rows() != init.dim || init.loading[i].cols() != init.sources ||
        init.act[i].rows() != init.sources || init.act[i].cols() != init.frames)
      throw std::invalid_argument("fastfca_fit: init/covariance shape mismatch");
}

ffca_fit_opts fit_opts(LhFlavor flavor, int iters, const FitOptions& fit,
                       const FastFcaOptions& opts, const GpuOptions& gpu) {
  ffca_fit_opts o{};
  o.flavor = flavor == LhFlavor::em ? FFCA_FLAVOR_EM : FFCA_FLAVOR_MM;
  o.iters = iters;
  o.record_trace = fit.record_trace ? 1 : 0;
  o.seed = fit.seed;
  o.normalize_scales = opts.normalize_scales ? 1 : 0;
  o.fix_loadings = opts.fix_loadings ? 1 : 0;
  o.precision = prec(gpu);
  return o;
}

// Run fn(d, lo, hi) for contiguous balanced ranges of `count`, one host
// thread per device; rethrow the first error on the caller (parallel.cpp:30-44).
template <typename Fn>
void over_devices(const std::vector<int>& devs, int count, Fn fn) {
  const int G = std::max(1, std::min<int>(int(devs.size()), count));
  if (G == 1) {
    fn(devs.empty() ? 0 : devs[0], 0, count);
    return;
  }
  std::vector<std::exception_ptr> errs(G);
  std::vector<std::thread> th;
  const int base = count / G, rem = count % G;
  int lo = 0;
  for (int g = 0; g < G; ++g) {
    const int hi = lo + base + (g < rem ? 1 : 0);
    th.emplace_back([&, g, lo, hi] {
      try {
        fn(devs[g], lo, hi);
      } catch (...) {
        errs[g] = std::current_exception();
      }
    });
    lo = hi;
  }
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

// ------------------------------------------------------------------- stft --

RVec sqrt_hann_window(int frame_len) {  // stft.cpp:33-39 (a constant table)
  RVec w(frame_len);
  for (int k = 0; k < frame_len; ++k) w(k) = std::sqrt(0.5 - 0.5 * std::cos(2.0 * M_PI * k / frame_len));
  return w;
}

int stft_frame_count(long length, int frame_len, int shift, StftPadding pad) {
  const long long n = ffca_stft_frame_count(
      length, frame_len, shift, pad == StftPadding::centered ? FFCA_STFT_CENTERED : FFCA_STFT_FULL_FRAMES);
  if (n < 0) throw std::invalid_argument(ffca_last_error());
  return static_cast<int>(n);
}

Spectrogram stft(const MultichannelWave& wave, int frame_len, int shift, StftPadding pad) {
  const int C = wave.channels();
  const long len = wave.length();
  const int padding = pad == StftPadding::centered ? FFCA_STFT_CENTERED : FFCA_STFT_FULL_FRAMES;
  // Validation order and messages follow stft.cpp:52-57.
  if (frame_len <= 0 || (frame_len & (frame_len - 1)) != 0)
    throw std::invalid_argument("stft: frame length must be a power of two");
  if (shift * 2 != frame_len) throw std::invalid_argument("stft: shift must be frame_len/2");
  if (len < frame_len) throw std::invalid_argument("stft: signal shorter than one frame");
  const int bins = frame_len / 2 + 1;
  const int frames = stft_frame_count(len, frame_len, shift, pad);
  std::vector<double> spec(size_t(bins) * frames * C * 2);
  raise(ffca_stft(context(0), C, len, frame_len, shift, padding,
                  reinterpret_cast<const double*>(wave.samples.data()), spec.data()));
  Spectrogram out = Spectrogram::zero(C, bins, frames);
  for (int b = 0; b < bins; ++b)
    std::memcpy(static_cast<void*>(out.f[b].data()), spec.data() + size_t(b) * frames * C * 2,
                sizeof(double) * frames * C * 2);
  return out;
}

MultichannelWave istft(const Spectrogram& spec, int frame_len, int shift, long out_len,
                       double sample_rate, StftPadding pad) {
  const int padding = pad == StftPadding::centered ? FFCA_STFT_CENTERED : FFCA_STFT_FULL_FRAMES;
  const int C = spec.channels;
  std::vector<double> in(size_t(spec.bins) * spec.frames * C * 2);
  for (int b = 0; b < spec.bins && b < int(spec.f.size()); ++b)
    std::memcpy(in.data() + size_t(b) * spec.frames * C * 2, spec.f[b].data(),
                sizeof(double) * spec.frames * C * 2);
  MultichannelWave wave;
  wave.sample_rate = sample_rate;
  wave.samples = RMat::Zero(C, out_len);
  raise(ffca_istft(context(0), C, spec.bins, spec.frames, frame_len, shift, padding, out_len,
                   in.data(), wave.samples.data()));
  return wave;
}

// --------------------------------------------------------------- sigmodel --

SampleCovSet sample_covs(const Spectrogram& spec, int block_size) {
  if (spec.bins == 0 || spec.frames == 0 || spec.channels == 0)
    throw std::invalid_argument("sample_covs: empty spectrogram");
  if (block_size < 1) throw std::invalid_argument("sample_covs: block size must be >= 1");
  const int M = spec.channels, F = spec.bins, T = spec.frames;
  SampleCovSet covs;
  covs.dim = M;
  covs.bins = F;
  covs.frames = T;
  covs.block_size = block_size;
  covs.blocks = (T + block_size - 1) / block_size;
  std::vector<double> x(size_t(F) * T * M * 2);
  for (int i = 0; i < F; ++i)
    std::memcpy(x.data() + size_t(i) * T * M * 2, spec.f[i].data(), sizeof(double) * T * M * 2);
  std::vector<double> pw(F);
  ffca_dims d{1, F, M, 1, T, 0, 0};
  if (block_size == 1) {
    covs.snapshots = spec.f;
    raise(ffca_power_scale(context(0), &d, x.data(), pw.data()));
  } else {
    const int J = covs.blocks;
    std::vector<double> mats(size_t(F) * J * M * M * 2);
    raise(ffca_block_covs(context(0), &d, block_size, x.data(), mats.data(), pw.data()));
    covs.mats.assign(F, std::vector<CMat>(J, CMat::Zero(M, M)));
    for (int i = 0; i < F; ++i)
      for (int j = 0; j < J; ++j)
        std::memcpy(static_cast<void*>(covs.mats[i][j].data()),
                    mats.data() + (size_t(i) * J + j) * M * M * 2, sizeof(double) * M * M * 2);
  }
  covs.power_scale = RVec::Zero(F);
  for (int i = 0; i < F; ++i) covs.power_scale(i) = pw[i];
  return covs;
}

SampleCovSet piecewise_prepare(const Spectrogram& spec, int block_size) {
  return sample_covs(spec, block_size);  // fastfca.cpp:266-268
}

FastFcaParams expand_block_params(const FastFcaParams& params, int block_size, int frames) {
  if (block_size == 1 && frames == params.frames) return params;  // sigmodel.cpp:190
  FastFcaParams out = params;
  out.frames = frames;
  for (int i = 0; i < params.bins; ++i) {
    const RMat& h = params.act[i];
    RMat e = RMat::Zero(h.rows(), frames);
    for (int j = 0; j < frames; ++j) {
      const long jb = std::min<long>(j / block_size, h.cols() - 1);
      for (long n = 0; n < h.rows(); ++n) e(n, j) = h(n, jb);
    }
    out.act[i] = e;
  }
  return out;
}

double fastfca_nll(const SampleCovSet& covs, const FastFcaParams& p) {
  if (covs.dim != p.dim || covs.bins != p.bins || covs.blocks != p.frames)
    throw std::invalid_argument("nll: covariance/parameter shape mismatch");  // sigmodel.cpp:226-229
  check_covs(covs, "nll");
  Packed pk;
  pack_bins(covs, p, 0, covs.bins, pk);
  std::vector<double> out(covs.bins);
  ffca_dims d{1, covs.bins, covs.dim, p.sources, covs.blocks, 0, 0};
  raise((pk.snap ? ffca_nll_bins : ffca_nll_bins_covs)(context(0), &d, FFCA_PREC_FP64,
                                                         pk.x.data(), pk.W.data(), pk.L.data(),
                                                         pk.H.data(), out.data()));
  double acc = 0.0;
  for (double v : out) acc += v;  // bin order
  return acc;
}

double fastfca_nll_freq(const SampleCovSet& covs, int i, const CMat& w, const RMat& loading,
                        const RMat& act) {
  FastFcaParams one;
  one.dim = covs.dim, one.bins = 1, one.frames = covs.blocks, one.sources = int(loading.cols());
  one.decorr = {w};
  one.loading = {loading};
  one.act = {act};
  SampleCovSet c1;
  c1.dim = covs.dim, c1.bins = 1, c1.frames = covs.frames, c1.blocks = covs.blocks;
  c1.block_size = covs.block_size;
  if (covs.has_snapshots())
    c1.snapshots = {covs.snapshots.at(i)};
  else
    c1.mats = {covs.mats.at(i)};
  c1.power_scale = RVec::Zero(1);
  c1.power_scale(0) = covs.power(i);
  return fastfca_nll(c1, one);
}

RMat decorrelated_powers(const SampleCovSet& covs, int i, const CMat& w) {
  if (i < 0 || i >= covs.bins)
    throw std::invalid_argument("decorrelated_powers: bin out of range");
  check_covs(covs, "decorrelated_powers");
  if (w.rows() != covs.dim || w.cols() != covs.dim)
    throw std::invalid_argument("decorrelated_powers: W shape mismatch");
  const int M = covs.dim, T = covs.blocks;
  ffca_dims d{1, 1, M, M, T, 0, 0};
  RMat u(M, T);
  if (covs.has_snapshots()) {
    raise(ffca_decorrelated_powers(context(0), &d, FFCA_PREC_FP64,
                                   reinterpret_cast<const double*>(covs.snapshots[i].data()),
                                   reinterpret_cast<const double*>(w.data()), -1.0, u.data()));
  } else {  // sigmodel.cpp:97-105
    std::vector<double> m(size_t(T) * M * M * 2);
    for (int j = 0; j < T; ++j)
      std::memcpy(m.data() + size_t(j) * M * M * 2, covs.mats[i][j].data(),
                  sizeof(double) * M * M * 2);
    raise(ffca_decorrelated_powers_covs(context(0), &d, FFCA_PREC_FP64, m.data(),
                                        reinterpret_cast<const double*>(w.data()), -1.0,
                                        u.data()));
  }
  return u;
}

// ---------------------------------------------------------------- fastfca --

FastFcaFitResult ica_mode_fit(const SampleCovSet& covs, int sources, int iters,
                              const std::vector<CMat>& w_init, const FitOptions& fit) {
  return ica_mode_fit(covs, sources, iters, w_init, fit, GpuOptions{});
}

FastFcaFitResult ica_mode_fit(const SampleCovSet& covs, int sources, int iters,
                              const std::vector<CMat>& w_init, const FitOptions& fit,
                              const GpuOptions& gpu) {
  // fastfca.cpp:244-249
  if (sources != covs.dim)
    throw std::invalid_argument("ica_mode_fit: requires as many sources as channels");
  if (static_cast<int>(w_init.size()) != covs.bins)
    throw std::invalid_argument("ica_mode_fit: one W per frequency required");
  check_covs(covs, "ica_mode_fit");
  if (iters < 0) throw std::invalid_argument("fastfca_fit: negative iteration count");
  const int F = covs.bins, M = covs.dim, T = covs.blocks;
  for (const CMat& w : w_init)
    if (w.rows() != M || w.cols() != M) throw std::invalid_argument("ica_mode_fit: W shape mismatch");
  FastFcaFitResult result;
  FastFcaParams& p = result.params;
  p.dim = M;
  p.bins = F;
  p.frames = T;
  p.sources = sources;
  p.decorr = w_init;
  p.loading.assign(F, RMat::Zero(M, sources));
  p.act.assign(F, RMat::Zero(sources, T));
  ffca_fit_opts o = fit_opts(LhFlavor::mm, iters, fit, FastFcaOptions{}, gpu);
  std::vector<double> slots(fit.record_trace ? size_t(iters + 1) * F : 0);
  over_devices(gpu.devices, F, [&](int dev, int lo, int hi) {
    Packed pk;
    pack_bins(covs, p, lo, hi, pk);  // x, power, W init (L, H are outputs)
    const int n = hi - lo;
    std::vector<double> sl(fit.record_trace ? size_t(iters + 1) * n : 0);
    ffca_dims d{1, n, M, sources, T, lo, F};
    raise((pk.snap ? ffca_ica_fit : ffca_ica_fit_covs)(
        context(dev), &d, &o, pk.x.data(), pk.pw(), pk.W.data(), pk.L.data(), pk.H.data(),
        nullptr, fit.record_trace ? sl.data() : nullptr, nullptr));
    unpack_bins(pk, lo, hi, p);
    for (int t = 0; fit.record_trace && t <= iters; ++t)
      for (int k = 0; k < n; ++k) slots[size_t(t) * F + lo + k] = sl[size_t(t) * n + k];
  });
  if (fit.record_trace) {  // fastfca.cpp:186-189, bin order
    result.nll.assign(iters + 1, 0.0);
    for (int t = 0; t <= iters; ++t) {
      double s = 0.0;
      for (int i = 0; i < F; ++i) s += slots[size_t(t) * F + i];
      result.nll[t] = s;
    }
  }
  return result;
}

FastFcaFitResult fastfca_fit(const SampleCovSet& covs, const FastFcaParams& init, LhFlavor flavor,
                             int iters, const FitOptions& fit, const FastFcaOptions& opts) {
  return fastfca_fit(covs, init, flavor, iters, fit, opts, GpuOptions{});
}

FastFcaFitResult fastfca_fit(const SampleCovSet& covs, const FastFcaParams& init, LhFlavor flavor,
                             int iters, const FitOptions& fit, const FastFcaOptions& opts,
                             const GpuOptions& gpu) {
  check_fit_shapes(covs, init);
  if (iters < 0) throw std::invalid_argument("fastfca_fit: negative iteration count");
  FastFcaFitResult result;
  const int F = covs.bins;
  {
    // result.params = init (fastfca.cpp:153-154); the activations -- the bulk,
    // 1.6 GB of fresh pages at BASELINE config 3 -- are copied on host threads.
    FastFcaParams& rp = result.params;
    rp.dim = init.dim, rp.bins = init.bins, rp.frames = init.frames, rp.sources = init.sources;
    rp.decorr = init.decorr;
    rp.loading = init.loading;
    rp.act.resize(init.act.size());
    parallel_bins(int(init.act.size()), host_threads(gpu, F), [&](int i) { rp.act[i] = init.act[i]; });
  }
  const ffca_fit_opts o = fit_opts(flavor, iters, fit, opts, gpu);
  std::vector<double> slots(fit.record_trace ? size_t(iters + 1) * F : 0);
  over_devices(gpu.devices, F, [&](int dev, int lo, int hi) {
    const int n = hi - lo;
    const int nt = host_threads(gpu, n);
    std::vector<double> sl(fit.record_trace ? size_t(iters + 1) * n : 0);
    ffca_dims d{1, n, covs.dim, init.sources, covs.blocks, lo, F};
    if (covs.has_snapshots()) {
      // Per-bin pointers straight into the containers: the library gathers bin
      // chunks into pinned staging on host threads and pipelines gather / H2D /
      // fit / D2H / scatter (ffca_fit_bins).  result.params already holds the
      // init, so the outputs alias the inputs.
      FastFcaParams& rp = result.params;
      std::vector<const double*> xb(n), wi(n), li(n), hi_(n);
      std::vector<double*> wo(n), lo_(n), ho(n);
      std::vector<double> pw(n);
      for (int k = 0; k < n; ++k) {
        const int i = lo + k;
        xb[k] = reinterpret_cast<const double*>(covs.snapshots[i].data());
        wo[k] = reinterpret_cast<double*>(rp.decorr[i].data());
        lo_[k] = rp.loading[i].data();
        ho[k] = rp.act[i].data();
        wi[k] = wo[k], li[k] = lo_[k], hi_[k] = ho[k];
        pw[k] = covs.power_scale(i);
      }
      raise(ffca_fit_bins(context(dev), &d, &o, xb.data(), pw.data(), wi.data(), li.data(),
                          hi_.data(), wo.data(), lo_.data(), ho.data(), nullptr,
                          fit.record_trace ? sl.data() : nullptr, nullptr, nt));
    } else {
      Packed pk;
      pack_bins(covs, init, lo, hi, pk, context(dev), nt);
      raise(ffca_fit_covs(context(dev), &d, &o, pk.x.data(), pk.pw(), pk.W.data(), pk.L.data(),
                          pk.H.data(), nullptr, fit.record_trace ? sl.data() : nullptr, nullptr));
      if (iters > 0) unpack_bins(pk, lo, hi, result.params, 0, nt);
    }
    for (int t = 0; fit.record_trace && t <= iters; ++t)
      for (int k = 0; k < n; ++k) slots[size_t(t) * F + lo + k] = sl[size_t(t) * n + k];
  });
  if (fit.record_trace) {  // fastfca.cpp:186-189, bin order
    result.nll.assign(iters + 1, 0.0);
    for (int t = 0; t <= iters; ++t) {
      double s = 0.0;
      for (int i = 0; i < F; ++i) s += slots[size_t(t) * F + i];
      result.nll[t] = s;
    }
  }
  return result;
}

std::vector<FastFcaFitResult> fastfca_fit_batch(const std::vector<SampleCovSet>& covs,
                                                const std::vector<FastFcaParams>& init,
                                                LhFlavor flavor, int iters,
                                                const FitOptions& fit,
                                                const FastFcaOptions& opts,
                                                const GpuOptions& gpu) {
  if (covs.size() != init.size())
    throw std::invalid_argument("fastfca_fit_batch: covariance/init count mismatch");
  const int B = int(covs.size());
  std::vector<FastFcaFitResult> out(B);
  if (B == 0) return out;
  for (int b = 0; b < B; ++b) {
    check_fit_shapes(covs[b], init[b]);
    if (covs[b].dim != covs[0].dim || covs[b].bins != covs[0].bins ||
        covs[b].blocks != covs[0].blocks || init[b].sources != init[0].sources ||
        covs[b].has_snapshots() != covs[0].has_snapshots() ||
        covs[b].power_scale.size() != covs[0].power_scale.size())
      throw std::invalid_argument("fastfca_fit_batch: mixtures must share one shape");
  }
  if (iters < 0) throw std::invalid_argument("fastfca_fit: negative iteration count");
  const ffca_fit_opts o = fit_opts(flavor, iters, fit, opts, gpu);
  const int F = covs[0].bins;
  for (int b = 0; b < B; ++b) out[b].params = init[b];
  over_devices(gpu.devices, B, [&](int dev, int lo, int hi) {  // whole mixtures per device
    const int nb = hi - lo;
    const int nt = host_threads(gpu, F);
    Packed all;
    size_packed(covs[0], init[0].sources, nb * F, all, context(dev));
    for (int b = lo; b < hi; ++b) pack_into(covs[b], init[b], 0, F, all, (b - lo) * F, nt);
    std::vector<double> nll(fit.record_trace ? size_t(nb) * (iters + 1) : 0);
    ffca_dims d{nb, F, covs[0].dim, init[0].sources, covs[0].blocks, 0, 0};
    raise((covs[0].has_snapshots() ? ffca_fit : ffca_fit_covs)(
        context(dev), &d, &o, all.x.data(), all.pw(), all.W.data(), all.L.data(), all.H.data(),
        fit.record_trace ? nll.data() : nullptr, nullptr, nullptr));
    if (iters > 0)
      for (int b = lo; b < hi; ++b) unpack_bins(all, 0, F, out[b].params, (b - lo) * F, nt);
    if (fit.record_trace)
      for (int b = lo; b < hi; ++b)
        out[b].nll.assign(nll.begin() + size_t(b - lo) * (iters + 1),
                          nll.begin() + size_t(b - lo + 1) * (iters + 1));
  });
  return out;
}

std::vector<Spectrogram> fastfca_separate(const Spectrogram& spec, const FastFcaParams& params) {
  return fastfca_separate(spec, params, GpuOptions{});
}

std::vector<Spectrogram> fastfca_separate(const Spectrogram& spec, const FastFcaParams& params,
                                          const GpuOptions& gpu) {
  if (spec.channels != params.dim || spec.bins != params.bins || spec.frames != params.frames)
    throw std::invalid_argument("fastfca_separate: shape mismatch");  // fastfca.cpp:207-209
  const int M = spec.channels, F = spec.bins, T = spec.frames, N = params.sources;
  std::vector<Spectrogram> images(N, Spectrogram::zero(M, F, T));
  over_devices(gpu.devices, F, [&](int dev, int lo, int hi) {
    const int n = hi - lo;
    std::vector<double> x(size_t(n) * T * M * 2), W(size_t(n) * M * M * 2), L(size_t(n) * M * N),
        H(size_t(n) * N * T), img(size_t(N) * n * T * M * 2);
    for (int i = lo; i < hi; ++i) {
      const size_t k = size_t(i - lo);
      std::memcpy(x.data() + k * T * M * 2, spec.f[i].data(), sizeof(double) * T * M * 2);
      std::memcpy(W.data() + k * M * M * 2, params.decorr[i].data(), sizeof(double) * M * M * 2);
      std::memcpy(L.data() + k * M * N, params.loading[i].data(), sizeof(double) * M * N);
      std::memcpy(H.data() + k * N * T, params.act[i].data(), sizeof(double) * N * T);
    }
    ffca_dims d{1, n, M, N, T, lo, F};
    raise(ffca_separate(context(dev), &d, prec(gpu), x.data(), W.data(), L.data(), H.data(),
                        img.data()));
    for (int s = 0; s < N; ++s)
      for (int i = lo; i < hi; ++i)
        std::memcpy(images[s].f[i].data(), img.data() + (size_t(s) * n + (i - lo)) * T * M * 2,
                    sizeof(double) * T * M * 2);
  });
  return images;
}

// ------------------------------------------------------- per-step functions --
// fastfca.hpp:28-53 -- host work is validation and container <-> flat buffer
// copies; the arithmetic is csrc/steps.cu (single-bin fp64 launches).

namespace {

// The bin's statistics as the flat buffer the step ABI takes: snapshots
// [blocks][dim] or block covariances [blocks][dim*dim].
std::vector<double> bin_stats(const SampleCovSet& covs, int i, const char* what) {
  if (i < 0 || i >= covs.bins) throw std::invalid_argument(std::string(what) + ": bin out of range");
  check_covs(covs, what);
  const int M = covs.dim, J = covs.blocks;
  std::vector<double> x;
  if (covs.has_snapshots()) {
    x.resize(size_t(J) * M * 2);
    std::memcpy(x.data(), covs.snapshots[i].data(), sizeof(double) * x.size());
  } else {
    x.resize(size_t(J) * M * M * 2);
    for (int j = 0; j < J; ++j)
      std::memcpy(x.data() + size_t(j) * M * M * 2, covs.mats[i][j].data(), sizeof(double) * M * M * 2);
  }
  return x;
}

}  // namespace

CMat weighted_cov(const SampleCovSet& covs, int i, const RMat& sigma2_row) {
  const std::vector<double> x = bin_stats(covs, i, "weighted_cov");
  if (sigma2_row.size() != covs.blocks)
    throw std::invalid_argument("weighted_cov: variance row length mismatch");
  CMat q(covs.dim, covs.dim);
  raise(ffca_weighted_cov(context(0), covs.dim, covs.blocks, covs.has_snapshots() ? 0 : 1, x.data(),
                          sigma2_row.data(), reinterpret_cast<double*>(q.data())));
  return q;
}

void ip_update_w(const SampleCovSet& covs, int i, CMat& w, const RMat& loading, const RMat& act,
                 std::uint64_t restart_seed) {
  const std::vector<double> x = bin_stats(covs, i, "ip_update_w");
  const int M = covs.dim;
  if (w.rows() != M || w.cols() != M || loading.rows() != M || act.rows() != loading.cols() ||
      act.cols() != covs.blocks)
    throw std::invalid_argument("ip_update_w: shape mismatch");
  raise(ffca_ip_update_w(context(0), M, int(loading.cols()), covs.blocks,
                         covs.has_snapshots() ? 0 : 1, x.data(), covs.power(i),
                         reinterpret_cast<double*>(w.data()), loading.data(), act.data(),
                         restart_seed, i));
}

RMat source_gain(const RMat& loading, const RMat& act, int n) {
  if (act.rows() != loading.cols()) throw std::invalid_argument("source_gain: shape mismatch");
  RMat g(loading.rows(), act.cols());
  raise(ffca_source_gain(context(0), int(loading.rows()), int(loading.cols()), int(act.cols()),
                         loading.data(), act.data(), n, g.data()));
  return g;
}

namespace {
void check_lh(const RMat& u, const RMat& loading, const RMat& act, const char* what) {
  if (loading.rows() != u.rows() || act.rows() != loading.cols() || act.cols() != u.cols())
    throw std::invalid_argument(std::string(what) + ": shape mismatch");
}
}  // namespace

void em_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading, double eps) {
  check_lh(u, loading, act, "em_update_lh");
  raise(ffca_em_update_lh(context(0), int(u.rows()), int(loading.cols()), int(u.cols()), u.data(),
                          loading.data(), act.data(), update_loading ? 1 : 0, eps));
}

void mm_update_lh(const RMat& u, RMat& loading, RMat& act, bool update_loading, double eps) {
  check_lh(u, loading, act, "mm_update_lh");
  raise(ffca_mm_update_lh(context(0), int(u.rows()), int(loading.cols()), int(u.cols()), u.data(),
                          loading.data(), act.data(), update_loading ? 1 : 0, eps));
}

CMat fastfca_mwf(const FastFcaParams& params, int i, int j, int n) {
  if (i < 0 || i >= params.bins || j < 0 || j >= params.frames || n < 0 || n >= params.sources)
    throw std::invalid_argument("fastfca_mwf: index out of range");
  const int M = params.dim, N = params.sources;
  std::vector<double> col(N);
  for (int q = 0; q < N; ++q) col[q] = params.act[i](q, j);
  CMat out(M, M);
  raise(ffca_mwf(context(0), M, N, reinterpret_cast<const double*>(params.decorr[i].data()),
                 params.loading[i].data(), col.data(), n, reinterpret_cast<double*>(out.data())));
  return out;
}

double ajd_cost(const CMat& w, const SampleCovSet& covs, int i, const RVec& weights) {
  if (weights.size() != 0 && weights.size() != covs.blocks)
    throw std::invalid_argument("ajd_cost: weight count mismatch");  // fastfca.cpp:227-228
  if (i < 0 || i >= covs.bins || int(covs.mats.size()) != covs.bins ||
      int(covs.mats[i].size()) != covs.blocks)
    throw std::invalid_argument("ajd_cost: needs the block covariances (SampleCovSet::mats)");
  const int M = covs.dim, J = covs.blocks;
  if (w.rows() != M || w.cols() != M) throw std::invalid_argument("ajd_cost: W shape mismatch");
  std::vector<double> x(size_t(J) * M * M * 2);
  for (int j = 0; j < J; ++j)
    std::memcpy(x.data() + size_t(j) * M * M * 2, covs.mats[i][j].data(), sizeof(double) * M * M * 2);
  double out = 0.0;
  raise(ffca_ajd_cost(context(0), M, J, x.data(), reinterpret_cast<const double*>(w.data()),
                      weights.size() ? weights.data() : nullptr, &out));
  return out;
}

std::vector<std::vector<CMat>> reconstruct_scms(const FastFcaParams& params) {
  const int F = params.bins, M = params.dim, N = params.sources;
  std::vector<std::vector<CMat>> scms(F);
  if (F == 0) return scms;
  std::vector<double> W(size_t(F) * M * M * 2), L(size_t(F) * M * N), out(size_t(F) * N * M * M * 2);
  for (int i = 0; i < F; ++i) {
    std::memcpy(W.data() + size_t(i) * M * M * 2, params.decorr[i].data(), sizeof(double) * M * M * 2);
    std::memcpy(L.data() + size_t(i) * M * N, params.loading[i].data(), sizeof(double) * M * N);
  }
  raise(ffca_reconstruct_scms(context(0), F, M, N, W.data(), L.data(), out.data()));
  for (int i = 0; i < F; ++i)
    for (int n = 0; n < N; ++n) {
      CMat r(M, M);
      std::memcpy(static_cast<void*>(r.data()), out.data() + (size_t(i) * N + n) * M * M * 2,
                  sizeof(double) * M * M * 2);
      scms[i].push_back(r);
    }
  return scms;
}

double log_abs_det2(const CMat& w) {
  if (w.rows() != w.cols() || w.rows() < 1) throw std::invalid_argument("log_abs_det2: not square");
  double out = 0.0;
  raise(ffca_log_abs_det2(context(0), int(w.rows()), reinterpret_cast<const double*>(w.data()), &out));
  return out;
}

void FastFcaParams::validate() const {  // sigmodel.cpp:74-91
  if (int(decorr.size()) != bins || int(loading.size()) != bins || int(act.size()) != bins)
    throw std::invalid_argument("FastFcaParams: bin count mismatch");
  for (int i = 0; i < bins; ++i) {
    if (decorr[i].rows() != dim || decorr[i].cols() != dim)
      throw std::invalid_argument("FastFcaParams: decorrelation shape");
    for (long k = 0; k < decorr[i].size(); ++k)
      if (!std::isfinite(decorr[i].data()[k].real()) || !std::isfinite(decorr[i].data()[k].imag()))
        throw std::invalid_argument("FastFcaParams: non-finite decorrelation");
    log_abs_det2(decorr[i]);  // throws NumericalError when singular
    if (loading[i].rows() != dim || loading[i].cols() != sources || act[i].rows() != sources ||
        act[i].cols() != frames)
      throw std::invalid_argument("FastFcaParams: loading/act shape");
    bool pos = true;
    for (long k = 0; k < loading[i].size(); ++k) pos = pos && loading[i].data()[k] > 0.0;
    for (long k = 0; k < act[i].size(); ++k) pos = pos && act[i].data()[k] > 0.0;
    if (!pos) throw std::invalid_argument("FastFcaParams: nonpositive loading/act");
  }
}

}  // namespace fastfca
