// cpp_e2e.cpp -- bench.py's end-to-end leg through the reference-facing C++
// API: fastfca::fastfca_fit on host containers (SampleCovSet / FastFcaParams
// in, FastFcaFitResult out), timed with the host clock around the call.
// Built as tools/cpp_e2e.so by build.build_all(); bench.py hands it the same
// synthetic mixture it times through the C-ABI.
#include <chrono>
#include <cstring>
#include <string>

#include "fastfca/fastfca.hpp"

extern "C" int ffca_cpp_e2e(int F, int M, int N, int T, int iters, int warmup, int steps,
                            const double* x /*[F][T][M] complex*/, const double* W, const double* L,
                            const double* H, double* ms_out /*[steps]*/, double* nll_last,
                            char* err, int errlen) {
  using namespace fastfca;
  try {
    SampleCovSet covs;
    {
      Spectrogram spec = Spectrogram::zero(M, F, T);
      for (int i = 0; i < F; ++i)
        std::memcpy(static_cast<void*>(spec.f[i].data()), x + size_t(i) * T * M * 2,
                    sizeof(double) * T * M * 2);
      covs = sample_covs(spec, 1);
    }
    FastFcaParams init;
    init.dim = M, init.bins = F, init.frames = T, init.sources = N;
    init.decorr.assign(F, CMat::Zero(M, M));
    init.loading.assign(F, RMat::Zero(M, N));
    init.act.assign(F, RMat::Zero(N, T));
    for (int i = 0; i < F; ++i) {
      std::memcpy(static_cast<void*>(init.decorr[i].data()), W + size_t(i) * M * M * 2, sizeof(double) * M * M * 2);
      std::memcpy(init.loading[i].data(), L + size_t(i) * M * N, sizeof(double) * M * N);
      std::memcpy(init.act[i].data(), H + size_t(i) * N * T, sizeof(double) * N * T);
    }
    for (int s = 0; s < warmup + steps; ++s) {
      const auto t0 = std::chrono::steady_clock::now();
      const FastFcaFitResult r = fastfca_fit(covs, init, LhFlavor::em, iters);
      const auto t1 = std::chrono::steady_clock::now();
      if (s >= warmup) ms_out[s - warmup] = std::chrono::duration<double, std::milli>(t1 - t0).count();
      if (nll_last && !r.nll.empty()) *nll_last = r.nll.back();
    }
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen > 0) {
      std::strncpy(err, e.what(), size_t(errlen - 1));
      err[errlen - 1] = 0;
    }
    return 1;
  }
}
