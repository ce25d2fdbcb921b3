// ffca_api.cu -- the C ABI (include/ffca.h): validation, device buffers,
// boundary precision conversion and kernel dispatch.  No CPU compute path:
// every entry point either runs the sm_100a kernels or returns an error.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "aux_kernels.cuh"
#include "internal.hpp"

namespace {
thread_local std::string g_err;
}  // namespace

int ffca_set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

using namespace ffca;

namespace {

int set_err(int code, const std::string& msg) { return ffca_set_err(code, msg); }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int check_dims(long long problems, int dim, int sources, int frames) {
  if (problems < 1 || frames < 1 || dim < 1 || sources < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca: empty shape (sample_covs: empty spectrogram)");
  if (dim > 8) return set_err(FFCA_INVALID_ARGUMENT, "ffca: dim > 8 is not supported");
  if (sources > 16) return set_err(FFCA_INVALID_ARGUMENT, "ffca: sources > 16 is not supported");
  if (problems > (1LL << 31) - 1) return set_err(FFCA_INVALID_ARGUMENT, "ffca: too many problems");
  return FFCA_OK;
}

int grid_for(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return int(g);
}

template <typename R>
int launch_fit(ffca_ctx* ctx, int M, FitParams& fp, cudaStream_t st) {
  const bool fp64 = sizeof(R) == 8;
  bool handled = false;
  const int rc = launch_fit_big(ctx, fp, st, M, fp64, &handled);
  if (rc != FFCA_OK || handled) return rc;
  switch (M) {
    case 1: return launch_fit_m1(ctx, fp, st, fp64);
    case 2: return launch_fit_m2(ctx, fp, st, fp64);
    case 3: return launch_fit_m3(ctx, fp, st, fp64);
    case 4: return launch_fit_m4(ctx, fp, st, fp64);
    case 5: return launch_fit_m5(ctx, fp, st, fp64);
    case 6: return launch_fit_m6(ctx, fp, st, fp64);
    case 7: return launch_fit_m7(ctx, fp, st, fp64);
    case 8: return launch_fit_m8(ctx, fp, st, fp64);
  }
  return set_err(FFCA_INVALID_ARGUMENT, "ffca: unsupported dim");
}

// Stage host fp64 x and H on the device and convert them to the compute type.
// x keeps its fp64 staging copy in slot kX (power_scale reads it).
template <typename R>
int stage_inputs(ffca_ctx* ctx, size_t P, int M, int N, int T, const double* x, const double* H,
                 void** xs_out, void** hs_out, double** hdbl_out, cudaStream_t st) {
  cudaError_t err;
  const size_t nx = P * T * M * 2, nh = P * T * N;
  if (x) {
    double* dx = static_cast<double*>(ctx->get(kX, nx * 8, &err));
    if (!dx) return set_err(FFCA_CUDA_ERROR, "ffca: x alloc failed");
    FFCA_CUDA(cudaMemcpyAsync(dx, x, nx * 8, cudaMemcpyHostToDevice, st));
    if (sizeof(R) == 8) {
      *xs_out = dx;
    } else {
      void* xs = ctx->get(kXs, nx * sizeof(R), &err);
      if (!xs) return set_err(FFCA_CUDA_ERROR, "ffca: x alloc failed");
      convert_kernel<double, R><<<grid_for(nx, 256), 256, 0, st>>>(dx, static_cast<R*>(xs), nx);
      ctx->launches++;
      FFCA_CUDA(cudaGetLastError());
      *xs_out = xs;
    }
  }
  if (H) {
    double* dh = static_cast<double*>(ctx->get(kH, nh * 8, &err));
    void* hs = ctx->get(kHs, nh * sizeof(R), &err);
    if (!dh || !hs) return set_err(FFCA_CUDA_ERROR, "ffca: H alloc failed");
    FFCA_CUDA(cudaMemcpyAsync(dh, H, nh * 8, cudaMemcpyHostToDevice, st));
    convert_kernel<double, R><<<grid_for(nh, 256), 256, 0, st>>>(dh, static_cast<R*>(hs), nh);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    *hs_out = hs;
    *hdbl_out = dh;
  }
  return FFCA_OK;
}

// ica: ica_mode_fit (fastfca.cpp:241-264) -- H and L are outputs: L is the
// identity, H the floored decorrelated powers of the W init, computed here
// on the device; the fit then runs IP+MM with the loadings fixed.
// Stage caller block covariances (complex128 [P][J][M*M] col-major) as packed
// records in the compute type; power (may be null) receives the trace-based
// SampleCovSet::power() of every problem.
template <typename R>
int stage_covs(ffca_ctx* ctx, size_t P, int M, int J, const double* mats, void** rec_out,
               double* power, cudaStream_t st) {
  cudaError_t err;
  const size_t nm = P * J * M * M;
  double* dm = static_cast<double*>(ctx->get(kX, nm * 16, &err));
  R* rec = static_cast<R*>(ctx->get(kXs, nm * sizeof(R), &err));
  if (!dm || !rec) return set_err(FFCA_CUDA_ERROR, "ffca: covariance alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dm, mats, nm * 16, cudaMemcpyHostToDevice, st));
  pack_covs_kernel<R><<<int(P), 256, 0, st>>>(reinterpret_cast<const double2*>(dm), M, J, rec, power);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  *rec_out = rec;
  return FFCA_OK;
}

// blk: x is SampleCovSet::mats (complex128 [P][J][M*M] col-major, frames = J
// blocks) -- the block-stationary input (fastfca.cpp:29-32, sigmodel.cpp:97-105).
template <typename R>
int fit_host(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
             const double* power, double* W, double* L, double* H, double* nll,
             double* nll_slots, int32_t* bin_status, bool ica = false, bool blk = false) {
  const int P = d->batch * d->bins, M = d->dim, N = d->sources, T = d->frames;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  void* xs = nullptr;
  void* hs = nullptr;
  double* hd = nullptr;
  int rc = stage_inputs<R>(ctx, P, M, N, T, blk ? nullptr : x, ica ? nullptr : H, &xs, &hs, &hd, st);
  if (rc) return rc;
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dL = static_cast<double*>(ctx->get(kL, size_t(P) * M * N * 8, &err));
  double* dpow = static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err));
  if (!dpow) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  if (blk) {
    rc = stage_covs<R>(ctx, P, M, T, x, &xs, power ? nullptr : dpow, st);
    if (rc) return rc;
  }
  const int iters = o->iters;
  const bool record = o->record_trace != 0;
  double* dnll = static_cast<double*>(ctx->get(kNll, size_t(iters + 1) * P * 8, &err));
  int* dstat = static_cast<int*>(ctx->get(kStat, size_t(P) * 4, &err));
  if (!dW || !dL || !dpow || !dnll || !dstat) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dW, W, size_t(P) * M * M * 16, cudaMemcpyHostToDevice, st));
  if (ica) {
    // L = identity (fastfca.cpp:257); a constant, written on the host.
    for (int p = 0; p < P; ++p)
      for (int k = 0; k < M * N; ++k) L[size_t(p) * M * N + k] = (k % M == k / M) ? 1.0 : 0.0;
    const size_t nh = size_t(P) * T * N;
    hd = static_cast<double*>(ctx->get(kH, nh * 8, &err));
    hs = ctx->get(kHs, nh * sizeof(R), &err);
    if (!hd || !hs) return set_err(FFCA_CUDA_ERROR, "ffca: H alloc failed");
    if (blk)
      decorrelated_powers_blk_kernel<R><<<P, 256, 0, st>>>(
          static_cast<const R*>(xs), reinterpret_cast<const double2*>(dW), M, T,
          1e-12 /* kPowerFloorRel */, hd);
    else
      decorrelated_powers_kernel<R><<<P, 256, 0, st>>>(static_cast<const cplx_t<R>*>(xs),
                                                        reinterpret_cast<const double2*>(dW), M, T,
                                                        1e-12 /* kPowerFloorRel */, hd);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    convert_kernel<double, R><<<grid_for(nh, 256), 256, 0, st>>>(hd, static_cast<R*>(hs), nh);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
  }
  FFCA_CUDA(cudaMemcpyAsync(dL, L, size_t(P) * M * N * 8, cudaMemcpyHostToDevice, st));
  if (power) {
    FFCA_CUDA(cudaMemcpyAsync(dpow, power, size_t(P) * 8, cudaMemcpyHostToDevice, st));
  } else if (!blk) {
    power_kernel<double2><<<P, 256, 0, st>>>(static_cast<const double2*>(ctx->bufs[kX].p), dpow,
                                             M, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
  }
  FitParams fp{};
  fp.nprob = P;
  fp.N = N;
  fp.T = T;
  // Restart seeds use the bin's index within its full mixture
  // (fastfca.cpp:40): a sub-range of a mixture passes its first bin and the
  // mixture's bin count.
  fp.F = d->mixture_bins > 0 ? d->mixture_bins : d->bins;
  fp.seed_bin0 = d->first_bin;
  fp.prob_offset = 0;
  fp.x = xs;
  fp.H = hs;
  fp.W = reinterpret_cast<double2*>(dW);
  fp.L = dL;
  fp.power = dpow;
  fp.nll = dnll;
  fp.nll_stride = P;
  fp.status = dstat;
  fp.iters = iters;
  fp.flavor = o->flavor;
  fp.record = record ? 1 : 0;
  fp.normalize = o->normalize_scales;
  fp.fix_loadings = o->fix_loadings;
  fp.seed = o->seed;
  fp.blk = blk ? 1 : 0;
  rc = launch_fit<R>(ctx, M, fp, st);
  if (rc) return rc;
  std::vector<int> stat(P);
  FFCA_CUDA(cudaMemcpyAsync(stat.data(), dstat, size_t(P) * 4, cudaMemcpyDeviceToHost, st));
  std::vector<double> slots;
  if (record) {
    slots.resize(size_t(iters + 1) * P);
    FFCA_CUDA(cudaMemcpyAsync(slots.data(), dnll, slots.size() * 8, cudaMemcpyDeviceToHost, st));
  }
  FFCA_CUDA(cudaStreamSynchronize(st));
  for (int p = 0; p < P; ++p) {
    const int s = stat[p] & 0xff;
    if (s == kStatusIpSingular)
      return set_err(FFCA_NUMERICAL, "ip_update_w: singular system for column " +
                                         std::to_string(stat[p] >> 8));
    if (s == kStatusSingularW) return set_err(FFCA_NUMERICAL, "singular decorrelation matrix");
  }
  if (bin_status) std::memcpy(bin_status, stat.data(), size_t(P) * 4);
  if (ica && iters == 0) {
    FFCA_CUDA(cudaMemcpyAsync(H, hd, size_t(P) * T * N * 8, cudaMemcpyDeviceToHost, st));
    FFCA_CUDA(cudaStreamSynchronize(st));
  }
  if (iters > 0) {
    const size_t nh = size_t(P) * T * N;
    unpack_h_kernel<R><<<grid_for(nh, 256), 256, 0, st>>>(static_cast<const R*>(hs), hd, dstat,
                                                          size_t(T) * N, nh);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    FFCA_CUDA(cudaMemcpyAsync(H, hd, nh * 8, cudaMemcpyDeviceToHost, st));
    FFCA_CUDA(cudaMemcpyAsync(W, dW, size_t(P) * M * M * 16, cudaMemcpyDeviceToHost, st));
    FFCA_CUDA(cudaMemcpyAsync(L, dL, size_t(P) * M * N * 8, cudaMemcpyDeviceToHost, st));
    FFCA_CUDA(cudaStreamSynchronize(st));
  }
  if (record) {
    const int F = d->bins;
    for (int b = 0; b < d->batch; ++b)
      for (int t = 0; t <= iters; ++t) {
        double s = 0.0;  // bin order, fastfca.cpp:188
        for (int i = 0; i < F; ++i) s += slots[size_t(t) * P + size_t(b) * F + i];
        if (nll) nll[size_t(b) * (iters + 1) + t] = s;
        if (nll_slots)
          for (int i = 0; i < F; ++i)
            nll_slots[(size_t(b) * (iters + 1) + t) * F + i] = slots[size_t(t) * P + size_t(b) * F + i];
      }
  }
  return FFCA_OK;
}

// The host-buffer fit pipelined over K bin chunks on K streams: chunk c's
// H2D + conversion overlaps the fit of chunk c-1, and its results go back
// while later chunks still compute.  Each bin's fit is latency-bound (its
// per-iteration dependency chain, not the SM count, sets the time), so the
// chunks' kernels co-reside and the call costs about the transfers plus one
// fit instead of their sum.  Snapshot input, non-ICA, enough bins only.
// On FFCA_NUMERICAL the W/L/H buffers hold the partially updated values.
template <typename R>
int fit_host_chunked(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
                     const double* power, double* W, double* L, double* H, double* nll,
                     double* nll_slots, int32_t* bin_status, int K) {
  const int P = d->batch * d->bins, M = d->dim, N = d->sources, T = d->frames;
  const int iters = o->iters;
  const bool record = o->record_trace != 0;
  cudaError_t err;
  const size_t nx = size_t(P) * T * M * 2, nh = size_t(P) * T * N;
  double* dx = static_cast<double*>(ctx->get(kX, nx * 8, &err));
  R* xs = sizeof(R) == 8 ? reinterpret_cast<R*>(dx) : static_cast<R*>(ctx->get(kXs, nx * sizeof(R), &err));
  double* dh = static_cast<double*>(ctx->get(kH, nh * 8, &err));
  R* hs = static_cast<R*>(ctx->get(kHs, nh * sizeof(R), &err));
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dL = static_cast<double*>(ctx->get(kL, size_t(P) * M * N * 8, &err));
  double* dpow = static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err));
  double* dnll = static_cast<double*>(ctx->get(kNll, size_t(iters + 1) * P * 8, &err));
  int* dstat = static_cast<int*>(ctx->get(kStat, size_t(P) * 4, &err));
  if (!dx || !xs || !dh || !hs || !dW || !dL || !dpow || !dnll || !dstat)
    return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  for (int c = 0; c < K; ++c)
    if (!ctx->cstream[c]) FFCA_CUDA(cudaStreamCreateWithFlags(&ctx->cstream[c], cudaStreamNonBlocking));
  // Breadth-first issue (all uploads, then all kernels, then all downloads):
  // a chunk's download queued before the next chunk's upload would hold the
  // upload behind the first chunk's fit in the copy engine's queue.
  auto range = [&](int c, int& lo, int& n) {
    lo = int((long long)P * c / K);
    n = int((long long)P * (c + 1) / K) - lo;
  };
  for (int c = 0; c < K; ++c) {
    int lo, n;
    range(c, lo, n);
    if (n == 0) continue;
    cudaStream_t s = ctx->cstream[c];
    const size_t xo = size_t(lo) * T * M * 2, xn = size_t(n) * T * M * 2;
    const size_t ho = size_t(lo) * T * N, hn = size_t(n) * T * N;
    FFCA_CUDA(cudaMemcpyAsync(dx + xo, x + xo, xn * 8, cudaMemcpyHostToDevice, s));
    FFCA_CUDA(cudaMemcpyAsync(dh + ho, H + ho, hn * 8, cudaMemcpyHostToDevice, s));
    FFCA_CUDA(cudaMemcpyAsync(dW + size_t(lo) * M * M * 2, W + size_t(lo) * M * M * 2,
                              size_t(n) * M * M * 16, cudaMemcpyHostToDevice, s));
    FFCA_CUDA(cudaMemcpyAsync(dL + size_t(lo) * M * N, L + size_t(lo) * M * N,
                              size_t(n) * M * N * 8, cudaMemcpyHostToDevice, s));
    if (power)
      FFCA_CUDA(cudaMemcpyAsync(dpow + lo, power + lo, size_t(n) * 8, cudaMemcpyHostToDevice, s));
  }
  for (int c = 0; c < K; ++c) {
    int lo, n;
    range(c, lo, n);
    if (n == 0) continue;
    cudaStream_t s = ctx->cstream[c];
    const size_t xo = size_t(lo) * T * M * 2, xn = size_t(n) * T * M * 2;
    const size_t ho = size_t(lo) * T * N, hn = size_t(n) * T * N;
    (void)xn;
    stage_kernel<R><<<n, 256, 0, s>>>(reinterpret_cast<const double2*>(dx + xo),
                                      reinterpret_cast<cplx_t<R>*>(xs + xo), dh + ho, hs + ho,
                                      power ? nullptr : dpow + lo, M, N, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    FitParams fp{};
    fp.nprob = n;
    fp.N = N;
    fp.T = T;
    fp.F = d->mixture_bins > 0 ? d->mixture_bins : d->bins;
    fp.seed_bin0 = d->first_bin + lo;  // restart seed index (first_bin + p) % F
    fp.prob_offset = lo;
    fp.work_total = P;  // streaming scratch: one allocation, disjoint rows per chunk
    fp.work_first = lo;
    fp.x = xs + xo;
    fp.H = hs + ho;
    fp.W = reinterpret_cast<double2*>(dW) + size_t(lo) * M * M;
    fp.L = dL + size_t(lo) * M * N;
    fp.power = dpow + lo;
    fp.nll = dnll;
    fp.nll_stride = P;
    fp.status = dstat + lo;
    fp.iters = iters;
    fp.flavor = o->flavor;
    fp.record = record ? 1 : 0;
    fp.normalize = o->normalize_scales;
    fp.fix_loadings = o->fix_loadings;
    fp.seed = o->seed;
    int rc = launch_fit<R>(ctx, M, fp, s);
    if (rc) return rc;
    if (iters > 0) {
      unpack_h_kernel<R><<<grid_for(hn, 256), 256, 0, s>>>(hs + ho, dh + ho, dstat + lo,
                                                            size_t(T) * N, hn);
      ctx->launches++;
      FFCA_CUDA(cudaGetLastError());
    }
  }
  for (int c = 0; c < K && iters > 0; ++c) {
    int lo, n;
    range(c, lo, n);
    if (n == 0) continue;
    cudaStream_t s = ctx->cstream[c];
    const size_t ho = size_t(lo) * T * N, hn = size_t(n) * T * N;
    FFCA_CUDA(cudaMemcpyAsync(H + ho, dh + ho, hn * 8, cudaMemcpyDeviceToHost, s));
    FFCA_CUDA(cudaMemcpyAsync(W + size_t(lo) * M * M * 2, dW + size_t(lo) * M * M * 2,
                              size_t(n) * M * M * 16, cudaMemcpyDeviceToHost, s));
    FFCA_CUDA(cudaMemcpyAsync(L + size_t(lo) * M * N, dL + size_t(lo) * M * N,
                              size_t(n) * M * N * 8, cudaMemcpyDeviceToHost, s));
  }
  for (int c = 0; c < K; ++c) FFCA_CUDA(cudaStreamSynchronize(ctx->cstream[c]));
  std::vector<int> stat(P);
  FFCA_CUDA(cudaMemcpy(stat.data(), dstat, size_t(P) * 4, cudaMemcpyDeviceToHost));
  std::vector<double> slots;
  if (record) {
    slots.resize(size_t(iters + 1) * P);
    FFCA_CUDA(cudaMemcpy(slots.data(), dnll, slots.size() * 8, cudaMemcpyDeviceToHost));
  }
  for (int p = 0; p < P; ++p) {
    const int st = stat[p] & 0xff;
    if (st == kStatusIpSingular)
      return set_err(FFCA_NUMERICAL, "ip_update_w: singular system for column " +
                                         std::to_string(stat[p] >> 8));
    if (st == kStatusSingularW) return set_err(FFCA_NUMERICAL, "singular decorrelation matrix");
  }
  if (bin_status) std::memcpy(bin_status, stat.data(), size_t(P) * 4);
  if (record) {
    const int F = d->bins;
    for (int b = 0; b < d->batch; ++b)
      for (int t = 0; t <= iters; ++t) {
        double sum = 0.0;  // bin order, fastfca.cpp:188
        for (int i = 0; i < F; ++i) sum += slots[size_t(t) * P + size_t(b) * F + i];
        if (nll) nll[size_t(b) * (iters + 1) + t] = sum;
        if (nll_slots)
          for (int i = 0; i < F; ++i)
            nll_slots[(size_t(b) * (iters + 1) + t) * F + i] = slots[size_t(t) * P + size_t(b) * F + i];
      }
  }
  return FFCA_OK;
}

// fn(i) for i in [0, count) on nt host threads (contiguous ranges).
template <typename Fn>
static void host_parallel(int count, int nt, Fn fn) {
  if (nt <= 1 || count < 2) {
    for (int i = 0; i < count; ++i) fn(i);
    return;
  }
  nt = std::min(nt, count);
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([=] {
      const int lo = int((long long)count * t / nt), hi = int((long long)count * (t + 1) / nt);
      for (int i = lo; i < hi; ++i) fn(i);
    });
  for (auto& t : th) t.join();
}

// The host fit on PER-BIN buffers (ffca_fit_bins): what a caller holding the
// reference's containers has -- one allocation per bin for x, W, L, H.  The
// library gathers bin chunks into page-locked staging on host threads and
// runs the chunks depth-first on their own streams, so the gather of chunk
// c+1 overlaps the transfer and fit of chunk c, and the scatter of chunk c's
// results overlaps the fits of the later chunks.  Snapshot input only.
template <typename R>
int fit_host_gather(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o,
                    const double* const* x_bins, const double* power, const double* const* W_in,
                    const double* const* L_in, const double* const* H_in, double* const* W_out,
                    double* const* L_out, double* const* H_out, double* nll, double* nll_slots,
                    int32_t* bin_status, int host_threads, int K) {
  const int P = d->batch * d->bins, M = d->dim, N = d->sources, T = d->frames;
  const int iters = o->iters;
  const bool record = o->record_trace != 0;
  cudaError_t err;
  const size_t nx = size_t(P) * T * M * 2, nh = size_t(P) * T * N;
  const size_t nw = size_t(P) * M * M * 2, nl = size_t(P) * M * N;
  double* px = static_cast<double*>(ffca_pinned_buffer(ctx, 2, nx * 8));
  double* ph = static_cast<double*>(ffca_pinned_buffer(ctx, 3, nh * 8));
  double* pw = static_cast<double*>(ffca_pinned_buffer(ctx, 4, nw * 8));
  double* pl = static_cast<double*>(ffca_pinned_buffer(ctx, 5, nl * 8));
  int* pstat = static_cast<int*>(ffca_pinned_buffer(ctx, 6, size_t(P) * 4));
  if (!px || !ph || !pw || !pl || !pstat)
    return set_err(FFCA_CUDA_ERROR, "ffca: pinned staging alloc failed");
  double* dx = static_cast<double*>(ctx->get(kX, nx * 8, &err));
  R* xs = sizeof(R) == 8 ? reinterpret_cast<R*>(dx) : static_cast<R*>(ctx->get(kXs, nx * sizeof(R), &err));
  double* dh = static_cast<double*>(ctx->get(kH, nh * 8, &err));
  R* hs = static_cast<R*>(ctx->get(kHs, nh * sizeof(R), &err));
  double* dW = static_cast<double*>(ctx->get(kW, nw * 8, &err));
  double* dL = static_cast<double*>(ctx->get(kL, nl * 8, &err));
  double* dpow = static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err));
  double* dnll = static_cast<double*>(ctx->get(kNll, size_t(iters + 1) * P * 8, &err));
  int* dstat = static_cast<int*>(ctx->get(kStat, size_t(P) * 4, &err));
  if (!dx || !xs || !dh || !hs || !dW || !dL || !dpow || !dnll || !dstat)
    return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  for (int c = 0; c < K; ++c)
    if (!ctx->cstream[c]) FFCA_CUDA(cudaStreamCreateWithFlags(&ctx->cstream[c], cudaStreamNonBlocking));
  auto range = [&](int c, int& lo, int& n) {
    lo = int((long long)P * c / K);
    n = int((long long)P * (c + 1) / K) - lo;
  };
  const size_t bx = size_t(T) * M * 2, bh = size_t(T) * N, bw = size_t(M) * M * 2, bl = size_t(M) * N;
  for (int c = 0; c < K; ++c) {
    int lo, n;
    range(c, lo, n);
    if (n == 0) continue;
    host_parallel(n, host_threads, [&, lo](int j) {
      const size_t p = size_t(lo + j);
      std::memcpy(px + p * bx, x_bins[p], bx * 8);
      std::memcpy(ph + p * bh, H_in[p], bh * 8);
      std::memcpy(pw + p * bw, W_in[p], bw * 8);
      std::memcpy(pl + p * bl, L_in[p], bl * 8);
    });
    cudaStream_t s = ctx->cstream[c];
    const size_t xo = size_t(lo) * bx, ho = size_t(lo) * bh;
    FFCA_CUDA(cudaMemcpyAsync(dx + xo, px + xo, size_t(n) * bx * 8, cudaMemcpyHostToDevice, s));
    FFCA_CUDA(cudaMemcpyAsync(dh + ho, ph + ho, size_t(n) * bh * 8, cudaMemcpyHostToDevice, s));
    FFCA_CUDA(cudaMemcpyAsync(dW + size_t(lo) * bw, pw + size_t(lo) * bw, size_t(n) * bw * 8,
                              cudaMemcpyHostToDevice, s));
    FFCA_CUDA(cudaMemcpyAsync(dL + size_t(lo) * bl, pl + size_t(lo) * bl, size_t(n) * bl * 8,
                              cudaMemcpyHostToDevice, s));
    if (power)
      FFCA_CUDA(cudaMemcpyAsync(dpow + lo, power + lo, size_t(n) * 8, cudaMemcpyHostToDevice, s));
    stage_kernel<R><<<n, 256, 0, s>>>(reinterpret_cast<const double2*>(dx + xo),
                                      reinterpret_cast<cplx_t<R>*>(xs + xo), dh + ho, hs + ho,
                                      power ? nullptr : dpow + lo, M, N, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    FitParams fp{};
    fp.nprob = n;
    fp.N = N;
    fp.T = T;
    fp.F = d->mixture_bins > 0 ? d->mixture_bins : d->bins;
    fp.seed_bin0 = d->first_bin + lo;
    fp.prob_offset = lo;
    fp.work_total = P;
    fp.work_first = lo;
    fp.x = xs + xo;
    fp.H = hs + ho;
    fp.W = reinterpret_cast<double2*>(dW) + size_t(lo) * M * M;
    fp.L = dL + size_t(lo) * bl;
    fp.power = dpow + lo;
    fp.nll = dnll;
    fp.nll_stride = P;
    fp.status = dstat + lo;
    fp.iters = iters;
    fp.flavor = o->flavor;
    fp.record = record ? 1 : 0;
    fp.normalize = o->normalize_scales;
    fp.fix_loadings = o->fix_loadings;
    fp.seed = o->seed;
    int rc = launch_fit<R>(ctx, M, fp, s);
    if (rc) return rc;
    FFCA_CUDA(cudaMemcpyAsync(pstat + lo, dstat + lo, size_t(n) * 4, cudaMemcpyDeviceToHost, s));
    if (iters > 0) {
      const size_t hn = size_t(n) * bh;
      unpack_h_kernel<R><<<grid_for(hn, 256), 256, 0, s>>>(hs + ho, dh + ho, dstat + lo,
                                                            size_t(T) * N, hn);
      ctx->launches++;
      FFCA_CUDA(cudaGetLastError());
      FFCA_CUDA(cudaMemcpyAsync(ph + ho, dh + ho, hn * 8, cudaMemcpyDeviceToHost, s));
      FFCA_CUDA(cudaMemcpyAsync(pw + size_t(lo) * bw, dW + size_t(lo) * bw, size_t(n) * bw * 8,
                                cudaMemcpyDeviceToHost, s));
      FFCA_CUDA(cudaMemcpyAsync(pl + size_t(lo) * bl, dL + size_t(lo) * bl, size_t(n) * bl * 8,
                                cudaMemcpyDeviceToHost, s));
    }
  }
  // Scatter each chunk as it completes (the later chunks still compute).  A
  // numerical failure stops the scatter: the outputs are then unspecified.
  int rc_num = FFCA_OK;
  for (int c = 0; c < K; ++c) {
    int lo, n;
    range(c, lo, n);
    if (n == 0) continue;
    FFCA_CUDA(cudaStreamSynchronize(ctx->cstream[c]));
    for (int p = lo; p < lo + n && rc_num == FFCA_OK; ++p) {
      const int st = pstat[p] & 0xff;
      if (st == kStatusIpSingular)
        rc_num = set_err(FFCA_NUMERICAL, "ip_update_w: singular system for column " +
                                             std::to_string(pstat[p] >> 8));
      else if (st == kStatusSingularW)
        rc_num = set_err(FFCA_NUMERICAL, "singular decorrelation matrix");
    }
    if (rc_num == FFCA_OK && iters > 0)
      host_parallel(n, host_threads, [&, lo](int j) {
        const size_t p = size_t(lo + j);
        std::memcpy(H_out[p], ph + p * bh, bh * 8);
        std::memcpy(W_out[p], pw + p * bw, bw * 8);
        std::memcpy(L_out[p], pl + p * bl, bl * 8);
      });
  }
  if (rc_num != FFCA_OK) return rc_num;
  const int* stat_p = pstat;
  std::vector<double> slots;
  if (record) {
    slots.resize(size_t(iters + 1) * P);
    FFCA_CUDA(cudaMemcpy(slots.data(), dnll, slots.size() * 8, cudaMemcpyDeviceToHost));
  }
  if (bin_status) std::memcpy(bin_status, stat_p, size_t(P) * 4);
  if (record) {
    const int F = d->bins;
    for (int b = 0; b < d->batch; ++b)
      for (int t = 0; t <= iters; ++t) {
        double sum = 0.0;  // bin order, fastfca.cpp:188
        for (int i = 0; i < F; ++i) sum += slots[size_t(t) * P + size_t(b) * F + i];
        if (nll) nll[size_t(b) * (iters + 1) + t] = sum;
        if (nll_slots)
          for (int i = 0; i < F; ++i)
            nll_slots[(size_t(b) * (iters + 1) + t) * F + i] = slots[size_t(t) * P + size_t(b) * F + i];
      }
  }
  return FFCA_OK;
}

// Chunks for the pipelined host fit: one per ~128 bins, at most kMaxChunks;
// 1 (the plain path) below 256 bins.
constexpr int kDefaultMaxChunks = 16;
inline int fit_chunks(int P) {
  if (const char* e = getenv("FFCA_FIT_CHUNKS")) return std::max(1, std::min(kMaxChunks, atoi(e)));
  return P < 256 ? 1 : std::min(kDefaultMaxChunks, P / 128);
}

// ffca_fit / ffca_ica_fit and their block-covariance variants.
int fit_entry(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
              const double* power, double* W, double* L, double* H, double* nll,
              double* nll_slots, int32_t* bin_status, bool ica, bool blk) {
  const char* fn = ica ? "ffca_ica_fit" : "ffca_fit";
  if (!ctx || !d || !o) return set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": null argument");
  if (d->batch < 1 || d->bins < 1)
    return set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": empty shape");
  if (ica && d->sources != d->dim)  // fastfca.cpp:244-246
    return set_err(FFCA_INVALID_ARGUMENT, "ica_mode_fit: requires as many sources as channels");
  int rc = check_dims((long long)d->batch * d->bins, d->dim, d->sources, d->frames);
  if (rc) return rc;
  if (o->iters < 0) return set_err(FFCA_INVALID_ARGUMENT, "fastfca_fit: negative iteration count");
  if (!ica && o->flavor != FFCA_FLAVOR_EM && o->flavor != FFCA_FLAVOR_MM)
    return set_err(FFCA_INVALID_ARGUMENT, "fastfca_fit: unknown flavor");
  if (!x || !W || !L || !H) return set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": null buffer");
  if (o->record_trace && !nll && !nll_slots)
    return set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": record_trace needs an nll buffer");
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  if (!ica) {
    if (o->iters == 0 && !o->record_trace) {
      if (bin_status) std::memset(bin_status, 0, sizeof(int32_t) * d->batch * d->bins);
      return FFCA_OK;
    }
    const int K = blk ? 1 : fit_chunks(d->batch * d->bins);
    if (K > 1)
      return o->precision == FFCA_PREC_FP64
                 ? fit_host_chunked<double>(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status, K)
                 : fit_host_chunked<float>(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status, K);
    if (o->precision == FFCA_PREC_FP64)
      return fit_host<double>(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status, false, blk);
    return fit_host<float>(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status, false, blk);
  }
  ffca_fit_opts m = *o;
  m.flavor = FFCA_FLAVOR_MM;  // fastfca.cpp:262-263
  m.fix_loadings = 1;
  m.normalize_scales = 1;
  // Always the fp64 kernels: at the determined-mode fixed point H tracks
  // U = |w^H x|^2 and the 1/U weights amplify fp32 cancellation in w^H x
  // (measured: the fp32 trajectory leaves the fp64 one by 5e-4 after 20
  // iterations and the IP system then goes singular where the reference
  // converges), so `precision` does not apply to this mode.
  return fit_host<double>(ctx, d, &m, x, power, W, L, H, nll, nll_slots, bin_status, true, blk);
}

}  // namespace

extern "C" {

int ffca_version(void) { return 2; }

const char* ffca_last_error(void) { return g_err.c_str(); }

int ffca_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int ffca_ctx_create(int device, ffca_ctx** out) {
  if (!out) return set_err(FFCA_INVALID_ARGUMENT, "ffca_ctx_create: null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return set_err(FFCA_CUDA_ERROR, std::string("ffca_ctx_create: no CUDA device (") +
                                        cudaGetErrorString(e) + ")");
  if (device < 0 || device >= n) return set_err(FFCA_INVALID_ARGUMENT, "ffca_ctx_create: bad device");
  cudaDeviceProp prop;
  FFCA_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return set_err(FFCA_CUDA_ERROR, "ffca_ctx_create: device is not sm_100 (B200); no fallback");
  DeviceGuard g(device);
  ffca_ctx* c = new ffca_ctx();
  c->device = device;
  cudaError_t se = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (se != cudaSuccess) {
    delete c;
    return set_err(FFCA_CUDA_ERROR, std::string("ffca_ctx_create: ") + cudaGetErrorString(se));
  }
  *out = c;
  return FFCA_OK;
}

void ffca_ctx_destroy(ffca_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->device);
  for (auto& b : ctx->bufs)
    if (b.p) cudaFree(b.p);
  for (auto& b : ctx->pinned)
    if (b.p) cudaFreeHost(b.p);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  for (auto& s : ctx->cstream)
    if (s) cudaStreamDestroy(s);
  delete ctx;
}

void* ffca_pinned_buffer(ffca_ctx* ctx, int slot, size_t bytes) {
  if (!ctx || slot < 0 || slot >= 8) return nullptr;
  DeviceGuard g(ctx->device);
  ffca_ctx::Buf& b = ctx->pinned[slot];
  if (b.p && b.n >= bytes) return b.p;
  if (b.p) cudaFreeHost(b.p);
  b.p = nullptr;
  b.n = 0;
  if (cudaHostAlloc(&b.p, bytes < 4096 ? 4096 : bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return nullptr;
  }
  b.n = bytes;
  return b.p;
}

int ffca_last_launch_count(const ffca_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ffca_fit(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
             const double* power, double* W, double* L, double* H, double* nll,
             double* nll_slots, int32_t* bin_status) {
  return fit_entry(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status, false, false);
}

int ffca_fit_bins(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o,
                  const double* const* x_bins, const double* power, const double* const* W_in,
                  const double* const* L_in, const double* const* H_in, double* const* W_out,
                  double* const* L_out, double* const* H_out, double* nll, double* nll_slots,
                  int32_t* bin_status, int host_threads) {
  if (!ctx || !d || !o || !x_bins || !W_in || !L_in || !H_in || !W_out || !L_out || !H_out)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_bins: null argument");
  if (d->batch < 1 || d->bins < 1) return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_bins: empty shape");
  int rc = check_dims((long long)d->batch * d->bins, d->dim, d->sources, d->frames);
  if (rc) return rc;
  if (o->iters < 0) return set_err(FFCA_INVALID_ARGUMENT, "fastfca_fit: negative iteration count");
  if (o->flavor != FFCA_FLAVOR_EM && o->flavor != FFCA_FLAVOR_MM)
    return set_err(FFCA_INVALID_ARGUMENT, "fastfca_fit: unknown flavor");
  if (o->record_trace && !nll && !nll_slots)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_bins: record_trace needs an nll buffer");
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  const int P = d->batch * d->bins;
  if (o->iters == 0 && !o->record_trace) {
    if (bin_status) std::memset(bin_status, 0, sizeof(int32_t) * P);
    return FFCA_OK;  // the outputs already hold the init (the caller's copy)
  }
  if (host_threads < 1) host_threads = int(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
  const int K = std::max(1, std::min(kMaxChunks, std::max(fit_chunks(P), std::min(P, 4))));
  return o->precision == FFCA_PREC_FP64
             ? fit_host_gather<double>(ctx, d, o, x_bins, power, W_in, L_in, H_in, W_out, L_out,
                                       H_out, nll, nll_slots, bin_status, host_threads, K)
             : fit_host_gather<float>(ctx, d, o, x_bins, power, W_in, L_in, H_in, W_out, L_out,
                                      H_out, nll, nll_slots, bin_status, host_threads, K);
}

int ffca_fit_covs(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* mats,
                  const double* power, double* W, double* L, double* H, double* nll,
                  double* nll_slots, int32_t* bin_status) {
  return fit_entry(ctx, d, o, mats, power, W, L, H, nll, nll_slots, bin_status, false, true);
}

int ffca_ica_fit(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
                 const double* power, double* W, double* L, double* H, double* nll,
                 double* nll_slots, int32_t* bin_status) {
  return fit_entry(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status, true, false);
}

int ffca_ica_fit_covs(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o,
                      const double* mats, const double* power, double* W, double* L, double* H,
                      double* nll, double* nll_slots, int32_t* bin_status) {
  return fit_entry(ctx, d, o, mats, power, W, L, H, nll, nll_slots, bin_status, true, true);
}

int ffca_decorrelated_powers(ffca_ctx* ctx, const ffca_dims* d, int precision, const double* x,
                             const double* W, double floor_rel, double* out) {
  if (!ctx || !d || !x || !W || !out)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_decorrelated_powers: null argument");
  if (d->batch < 1 || d->bins < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_decorrelated_powers: empty shape");
  int rc = check_dims((long long)d->batch * d->bins, d->dim, d->dim, d->frames);
  if (rc) return rc;
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  const int P = d->batch * d->bins, M = d->dim, T = d->frames;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  void* xs = nullptr;
  void* hs = nullptr;
  double* hd = nullptr;
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dout = static_cast<double*>(ctx->get(kH, size_t(P) * T * M * 8, &err));
  if (!dW || !dout) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dW, W, size_t(P) * M * M * 16, cudaMemcpyHostToDevice, st));
  if (precision == FFCA_PREC_FP64) {
    rc = stage_inputs<double>(ctx, P, M, M, T, x, nullptr, &xs, &hs, &hd, st);
    if (rc) return rc;
    decorrelated_powers_kernel<double><<<P, 256, 0, st>>>(
        static_cast<const double2*>(xs), reinterpret_cast<const double2*>(dW), M, T, floor_rel, dout);
  } else {
    rc = stage_inputs<float>(ctx, P, M, M, T, x, nullptr, &xs, &hs, &hd, st);
    if (rc) return rc;
    decorrelated_powers_kernel<float><<<P, 256, 0, st>>>(
        static_cast<const float2*>(xs), reinterpret_cast<const double2*>(dW), M, T, floor_rel, dout);
  }
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  FFCA_CUDA(cudaMemcpyAsync(out, dout, size_t(P) * T * M * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

static int nll_bins_entry(ffca_ctx* ctx, const ffca_dims* d, int precision, const double* x,
                          const double* W, const double* L, const double* H, double* out,
                          bool blk) {
  if (!ctx || !d || !x || !W || !L || !H || !out)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_nll_bins: null argument");
  int rc = check_dims((long long)d->batch * d->bins, d->dim, d->sources, d->frames);
  if (rc) return rc;
  const int P = d->batch * d->bins;
  // A zero-iteration fit records exactly slot 0 = fastfca_nll_freq at the
  // given parameters and leaves W, L, H untouched.
  std::vector<double> w(W, W + size_t(P) * d->dim * d->dim * 2);
  std::vector<double> l(L, L + size_t(P) * d->dim * d->sources);
  std::vector<double> h(H, H + size_t(P) * d->sources * d->frames);
  std::vector<double> slots(P);
  ffca_fit_opts o{FFCA_FLAVOR_EM, 0, 1, 0, 1, 0, precision};
  ffca_dims one = *d;
  one.batch = 1;
  one.bins = P;
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  rc = (precision == FFCA_PREC_FP64)
           ? fit_host<double>(ctx, &one, &o, x, nullptr, w.data(), l.data(), h.data(), nullptr,
                              slots.data(), nullptr, false, blk)
           : fit_host<float>(ctx, &one, &o, x, nullptr, w.data(), l.data(), h.data(), nullptr,
                             slots.data(), nullptr, false, blk);
  if (rc) return rc;
  std::memcpy(out, slots.data(), sizeof(double) * P);
  return FFCA_OK;
}

int ffca_nll_bins(ffca_ctx* ctx, const ffca_dims* d, int precision, const double* x,
                  const double* W, const double* L, const double* H, double* out) {
  return nll_bins_entry(ctx, d, precision, x, W, L, H, out, false);
}

int ffca_nll_bins_covs(ffca_ctx* ctx, const ffca_dims* d, int precision, const double* mats,
                       const double* W, const double* L, const double* H, double* out) {
  return nll_bins_entry(ctx, d, precision, mats, W, L, H, out, true);
}

int ffca_decorrelated_powers_covs(ffca_ctx* ctx, const ffca_dims* d, int precision,
                                  const double* mats, const double* W, double floor_rel,
                                  double* out) {
  if (!ctx || !d || !mats || !W || !out)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_decorrelated_powers: null argument");
  if (d->batch < 1 || d->bins < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_decorrelated_powers: empty shape");
  int rc = check_dims((long long)d->batch * d->bins, d->dim, d->dim, d->frames);
  if (rc) return rc;
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  const int P = d->batch * d->bins, M = d->dim, J = d->frames;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dout = static_cast<double*>(ctx->get(kH, size_t(P) * J * M * 8, &err));
  if (!dW || !dout) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dW, W, size_t(P) * M * M * 16, cudaMemcpyHostToDevice, st));
  void* rec = nullptr;
  if (precision == FFCA_PREC_FP64) {
    rc = stage_covs<double>(ctx, P, M, J, mats, &rec, nullptr, st);
    if (rc) return rc;
    decorrelated_powers_blk_kernel<double><<<P, 256, 0, st>>>(
        static_cast<const double*>(rec), reinterpret_cast<const double2*>(dW), M, J, floor_rel, dout);
  } else {
    rc = stage_covs<float>(ctx, P, M, J, mats, &rec, nullptr, st);
    if (rc) return rc;
    decorrelated_powers_blk_kernel<float><<<P, 256, 0, st>>>(
        static_cast<const float*>(rec), reinterpret_cast<const double2*>(dW), M, J, floor_rel, dout);
  }
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  FFCA_CUDA(cudaMemcpyAsync(out, dout, size_t(P) * J * M * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_block_covs(ffca_ctx* ctx, const ffca_dims* d, int block_size, const double* x,
                    double* mats, double* power) {
  if (!ctx || !d || !x) return set_err(FFCA_INVALID_ARGUMENT, "ffca_block_covs: null argument");
  const long long P = (long long)d->batch * d->bins;
  const int M = d->dim, T = d->frames;
  if (P < 1 || M < 1 || T < 1) return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: empty spectrogram");
  if (block_size < 1) return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: block size must be >= 1");
  if (M > 8) return set_err(FFCA_INVALID_ARGUMENT, "ffca: dim > 8 is not supported");
  const int J = (T + block_size - 1) / block_size;
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  double2* dx = static_cast<double2*>(ctx->get(kX, size_t(P) * T * M * 16, &err));
  double2* dm = mats ? static_cast<double2*>(ctx->get(kImg, size_t(P) * J * M * M * 16, &err)) : nullptr;
  double* dp = power ? static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err)) : nullptr;
  if (!dx || (mats && !dm) || (power && !dp)) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dx, x, size_t(P) * T * M * 16, cudaMemcpyHostToDevice, st));
  block_covs_kernel<double2, double><<<int(P), 256, 0, st>>>(dx, M, T, block_size, J, nullptr, dm, dp);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  if (mats) FFCA_CUDA(cudaMemcpyAsync(mats, dm, size_t(P) * J * M * M * 16, cudaMemcpyDeviceToHost, st));
  if (power) FFCA_CUDA(cudaMemcpyAsync(power, dp, size_t(P) * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_power_scale(ffca_ctx* ctx, const ffca_dims* d, const double* x, double* out) {
  if (!ctx || !d || !x || !out) return set_err(FFCA_INVALID_ARGUMENT, "ffca_power_scale: null argument");
  const long long P = (long long)d->batch * d->bins;
  const int M = d->dim, T = d->frames;
  if (P < 1 || M < 1 || T < 1) return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: empty spectrogram");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaError_t err;
  void* dx = ctx->get(kX, size_t(P) * T * M * 16, &err);
  double* dp = static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err));
  if (!dx || !dp) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dx, x, size_t(P) * T * M * 16, cudaMemcpyHostToDevice, ctx->stream));
  power_kernel<double2><<<int(P), 256, 0, ctx->stream>>>(static_cast<const double2*>(dx), dp, M, T);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  FFCA_CUDA(cudaMemcpyAsync(out, dp, size_t(P) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FFCA_CUDA(cudaStreamSynchronize(ctx->stream));
  return FFCA_OK;
}

int ffca_separate(ffca_ctx* ctx, const ffca_dims* d, int precision, const double* x,
                  const double* W, const double* L, const double* H, double* images) {
  if (!ctx || !d || !x || !W || !L || !H || !images)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_separate: null argument");
  int rc = check_dims((long long)d->batch * d->bins, d->dim, d->sources, d->frames);
  if (rc) return rc;
  const int P = d->batch * d->bins, M = d->dim, N = d->sources, T = d->frames;
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  void* xs = nullptr;
  void* hs = nullptr;
  double* hd = nullptr;
  rc = (precision == FFCA_PREC_FP64) ? stage_inputs<double>(ctx, P, M, N, T, x, H, &xs, &hs, &hd, st)
                                     : stage_inputs<float>(ctx, P, M, N, T, x, H, &xs, &hs, &hd, st);
  if (rc) return rc;
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dL = static_cast<double*>(ctx->get(kL, size_t(P) * M * N * 8, &err));
  const size_t nimg = size_t(N) * P * T * M;
  double2* dimg = static_cast<double2*>(ctx->get(kImg, nimg * 16, &err));
  if (!dW || !dL || !dimg) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dW, W, size_t(P) * M * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dL, L, size_t(P) * M * N * 8, cudaMemcpyHostToDevice, st));
  rc = launch_separate(ctx, M, precision == FFCA_PREC_FP64, true, xs, dW, dL, hs, P, N, T, dimg, st);
  if (rc) return rc;
  FFCA_CUDA(cudaMemcpyAsync(images, dimg, nimg * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

static int fit_device_entry(ffca_ctx* ctx, int problems, int bins_per_mixture, int prob_offset,
                            int dim, int sources, int frames, const ffca_fit_opts* o,
                            const void* x_dev, const double* power, double* W, double* L,
                            void* H_dev, double* nll_slots, int32_t* status, void* stream,
                            bool blk) {
  if (!ctx || !o || !x_dev || !power || !W || !L || !H_dev || !status)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_device: null argument");
  int rc = check_dims(problems, dim, sources, frames);
  if (rc) return rc;
  if (bins_per_mixture < 1 || o->iters < 0 || prob_offset < 0)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_device: bad arguments");
  if (o->record_trace && !nll_slots)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_device: record_trace needs nll_slots");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  FitParams fp{};
  fp.nprob = problems;
  fp.N = sources;
  fp.T = frames;
  fp.F = bins_per_mixture;
  fp.prob_offset = prob_offset;
  fp.seed_bin0 = prob_offset % bins_per_mixture;
  fp.x = x_dev;
  fp.H = H_dev;
  fp.W = reinterpret_cast<double2*>(W);
  fp.L = L;
  fp.power = power;
  fp.nll = nll_slots ? nll_slots - size_t(prob_offset) : nullptr;  // kernel indexes by global p
  fp.nll_stride = problems;
  fp.status = status;
  fp.iters = o->iters;
  fp.flavor = o->flavor;
  fp.record = o->record_trace ? 1 : 0;
  fp.normalize = o->normalize_scales;
  fp.fix_loadings = o->fix_loadings;
  fp.seed = o->seed;
  fp.timing = ctx->timing;
  fp.blk = blk ? 1 : 0;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return o->precision == FFCA_PREC_FP64 ? launch_fit<double>(ctx, dim, fp, st)
                                        : launch_fit<float>(ctx, dim, fp, st);
}

int ffca_fit_device(ffca_ctx* ctx, int problems, int bins_per_mixture, int prob_offset, int dim,
                    int sources, int frames, const ffca_fit_opts* o, const void* x_dev,
                    const double* power, double* W, double* L, void* H_dev, double* nll_slots,
                    int32_t* status, void* stream) {
  return fit_device_entry(ctx, problems, bins_per_mixture, prob_offset, dim, sources, frames, o,
                          x_dev, power, W, L, H_dev, nll_slots, status, stream, false);
}

int ffca_fit_covs_device(ffca_ctx* ctx, int problems, int bins_per_mixture, int prob_offset,
                         int dim, int sources, int blocks, const ffca_fit_opts* o,
                         const void* rec_dev, const double* power, double* W, double* L,
                         void* H_dev, double* nll_slots, int32_t* status, void* stream) {
  return fit_device_entry(ctx, problems, bins_per_mixture, prob_offset, dim, sources, blocks, o,
                          rec_dev, power, W, L, H_dev, nll_slots, status, stream, true);
}

int ffca_block_covs_device(ffca_ctx* ctx, int problems, int dim, int frames, int block_size,
                           int precision, const void* x_dev, void* rec_dev, double* power,
                           void* stream) {
  if (!ctx || !x_dev || !rec_dev) return set_err(FFCA_INVALID_ARGUMENT, "ffca_block_covs_device: null");
  if (problems < 1 || dim < 1 || frames < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: empty spectrogram");
  if (block_size < 1) return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: block size must be >= 1");
  if (dim > 8) return set_err(FFCA_INVALID_ARGUMENT, "ffca: dim > 8 is not supported");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const int J = (frames + block_size - 1) / block_size;
  if (precision == FFCA_PREC_FP64)
    block_covs_kernel<double2, double><<<problems, 256, 0, st>>>(
        static_cast<const double2*>(x_dev), dim, frames, block_size, J,
        static_cast<double*>(rec_dev), nullptr, power);
  else
    block_covs_kernel<float2, float><<<problems, 256, 0, st>>>(
        static_cast<const float2*>(x_dev), dim, frames, block_size, J,
        static_cast<float*>(rec_dev), nullptr, power);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

int ffca_separate_device(ffca_ctx* ctx, int problems, int dim, int sources, int frames,
                         int precision, const void* x_dev, const double* W, const double* L,
                         const void* H_dev, void* images_dev, void* stream) {
  if (!ctx || !x_dev || !W || !L || !H_dev || !images_dev)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_separate_device: null argument");
  int rc = check_dims(problems, dim, sources, frames);
  if (rc) return rc;
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return launch_separate(ctx, dim, precision == FFCA_PREC_FP64, false, x_dev, W, L, H_dev, problems,
                         sources, frames, images_dev, st);
}

int ffca_power_scale_device(ffca_ctx* ctx, int problems, int dim, int frames, int precision,
                            const void* x_dev, double* out, void* stream) {
  if (!ctx || !x_dev || !out) return set_err(FFCA_INVALID_ARGUMENT, "ffca_power_scale_device: null");
  if (problems < 1 || dim < 1 || frames < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: empty spectrogram");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (precision == FFCA_PREC_FP64)
    power_kernel<double2><<<problems, 256, 0, st>>>(static_cast<const double2*>(x_dev), out, dim,
                                                     frames);
  else
    power_kernel<float2><<<problems, 256, 0, st>>>(static_cast<const float2*>(x_dev), out, dim,
                                                    frames);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

}  // extern "C"

extern "C" int ffca_debug_set_timing(ffca_ctx* ctx, unsigned long long* dev_counters) {
  if (!ctx) return set_err(FFCA_INVALID_ARGUMENT, "ffca_debug_set_timing: null ctx");
  ctx->timing = dev_counters;
  return FFCA_OK;
}
