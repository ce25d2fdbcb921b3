// ffca_capi.cu -- the C ABI (include/ffca.h): validation, device buffers,
// boundary layout conversion and kernel dispatch.  No CPU compute path: every
// entry point either runs the sm_100a kernels or returns an error.

#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"
#include "aux_kernels.cuh"

namespace {
thread_local std::string g_err;
}  // namespace

int ffca_set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

using ffca::kX;
using ffca::kXs;
using ffca::kH;
using ffca::kHs;
using ffca::kW;
using ffca::kL;
using ffca::kPow;
using ffca::kNll;
using ffca::kStat;
using ffca::kImg;

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

int check_dims(int problems, int dim, int sources, int frames) {
  if (problems < 1 || frames < 1 || dim < 1 || sources < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca: empty shape (sample_covs: empty spectrogram)");
  if (dim > 8) return set_err(FFCA_INVALID_ARGUMENT, "ffca: dim > 8 is not supported");
  if (sources > 16) return set_err(FFCA_INVALID_ARGUMENT, "ffca: sources > 16 is not supported");
  return FFCA_OK;
}

int grid_for(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return int(g);
}

template <typename R>
int launch_fit(ffca_ctx* ctx, int M, ffca::FitParams& fp, cudaStream_t st) {
  const bool fp64 = sizeof(R) == 8;
  switch (M) {
    case 1: return ffca::launch_fit_m1(ctx, fp, st, fp64);
    case 2: return ffca::launch_fit_m2(ctx, fp, st, fp64);
    case 3: return ffca::launch_fit_m3(ctx, fp, st, fp64);
    case 4: return ffca::launch_fit_m4(ctx, fp, st, fp64);
    case 5: return ffca::launch_fit_m5(ctx, fp, st, fp64);
    case 6: return ffca::launch_fit_m6(ctx, fp, st, fp64);
    case 7: return ffca::launch_fit_m7(ctx, fp, st, fp64);
    case 8: return ffca::launch_fit_m8(ctx, fp, st, fp64);
  }
  return set_err(FFCA_INVALID_ARGUMENT, "ffca: unsupported dim");
}

template <int M, typename R>
int launch_sep_m(ffca_ctx* ctx, const void* xs, const double* W, const double* L, const void* Hs,
                 int P, int N, int T, double* out_aos, void* out_soa, cudaStream_t st) {
  using C = ffca::cplx_t<R>;
  ffca::separate_kernel<M, R><<<P, 256, 0, st>>>(
      reinterpret_cast<const C*>(xs), reinterpret_cast<const double2*>(W), L,
      reinterpret_cast<const R*>(Hs), P, N, T, reinterpret_cast<double2*>(out_aos),
      reinterpret_cast<C*>(out_soa));
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

template <typename R>
int launch_sep(ffca_ctx* ctx, int M, const void* xs, const double* W, const double* L,
               const void* Hs, int P, int N, int T, double* out_aos, void* out_soa,
               cudaStream_t st) {
  switch (M) {
    case 1: return launch_sep_m<1, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 2: return launch_sep_m<2, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 3: return launch_sep_m<3, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 4: return launch_sep_m<4, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 5: return launch_sep_m<5, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 6: return launch_sep_m<6, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 7: return launch_sep_m<7, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
    case 8: return launch_sep_m<8, R>(ctx, xs, W, L, Hs, P, N, T, out_aos, out_soa, st);
  }
  return set_err(FFCA_INVALID_ARGUMENT, "ffca: unsupported dim");
}

template <typename R>
int pack_inputs(ffca_ctx* ctx, int P, int M, int N, int T, const double* x, const double* H,
                void** xs_out, void** hs_out, double** hdbl_out, cudaStream_t st) {
  using C = ffca::cplx_t<R>;
  cudaError_t err;
  const size_t nx = size_t(P) * T * M, nh = size_t(P) * T * N;
  if (x) {
    void* dx = ctx->get(kX, nx * 16, &err);
    void* xs = ctx->get(kXs, nx * sizeof(C), &err);
    if (!dx || !xs) return set_err(FFCA_CUDA_ERROR, "ffca: x alloc failed");
    FFCA_CUDA(cudaMemcpyAsync(dx, x, nx * 16, cudaMemcpyHostToDevice, st));
    ffca::pack_x_kernel<R><<<grid_for(size_t(P) * T, 256), 256, 0, st>>>(
        reinterpret_cast<const double2*>(dx), reinterpret_cast<C*>(xs), P, M, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    *xs_out = xs;
  }
  if (H) {
    double* dh = static_cast<double*>(ctx->get(kH, nh * 8, &err));
    void* hs = ctx->get(kHs, nh * sizeof(R), &err);
    if (!dh || !hs) return set_err(FFCA_CUDA_ERROR, "ffca: H alloc failed");
    FFCA_CUDA(cudaMemcpyAsync(dh, H, nh * 8, cudaMemcpyHostToDevice, st));
    ffca::pack_h_kernel<R><<<grid_for(size_t(P) * T, 256), 256, 0, st>>>(
        dh, reinterpret_cast<R*>(hs), P, N, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    *hs_out = hs;
    *hdbl_out = dh;
  }
  return FFCA_OK;
}

template <typename R>
int fit_host(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
             const double* power, double* W, double* L, double* H, double* nll,
             double* nll_slots, int32_t* bin_status) {
  const int P = d->batch * d->bins, M = d->dim, N = d->sources, T = d->frames;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  void* xs = nullptr;
  void* hs = nullptr;
  double* hd = nullptr;
  int rc = pack_inputs<R>(ctx, P, M, N, T, x, H, &xs, &hs, &hd, st);
  if (rc) return rc;
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dL = static_cast<double*>(ctx->get(kL, size_t(P) * M * N * 8, &err));
  double* dpow = static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err));
  const int iters = o->iters;
  const bool record = o->record_trace != 0;
  double* dnll = static_cast<double*>(ctx->get(kNll, size_t(iters + 1) * P * 8, &err));
  int* dstat = static_cast<int*>(ctx->get(kStat, size_t(P) * 4, &err));
  if (!dW || !dL || !dpow || !dnll || !dstat) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dW, W, size_t(P) * M * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dL, L, size_t(P) * M * N * 8, cudaMemcpyHostToDevice, st));
  if (power) {
    FFCA_CUDA(cudaMemcpyAsync(dpow, power, size_t(P) * 8, cudaMemcpyHostToDevice, st));
  } else {
    ffca::power_aos_kernel<<<P, 256, 0, st>>>(
        reinterpret_cast<const double2*>(ctx->bufs[kX].p), dpow, M, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
  }
  ffca::FitParams fp{};
  fp.nprob = P;
  fp.N = N;
  fp.T = T;
  fp.F = d->bins;
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
    if (s == ffca::kStatusIpSingular)
      return set_err(FFCA_NUMERICAL, "ip_update_w: singular system for column " +
                                         std::to_string(stat[p] >> 8));
    if (s == ffca::kStatusSingularW) return set_err(FFCA_NUMERICAL, "singular decorrelation matrix");
  }
  if (bin_status) std::memcpy(bin_status, stat.data(), size_t(P) * 4);
  if (iters > 0) {
    ffca::unpack_h_kernel<R><<<grid_for(size_t(P) * T, 256), 256, 0, st>>>(
        reinterpret_cast<const R*>(hs), hd, dstat, P, N, T);
    ctx->launches++;
    FFCA_CUDA(cudaGetLastError());
    FFCA_CUDA(cudaMemcpyAsync(H, hd, size_t(P) * T * N * 8, cudaMemcpyDeviceToHost, st));
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

}  // namespace

extern "C" {

int ffca_version(void) { return 1; }

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
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int ffca_last_launch_count(const ffca_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ffca_fit(ffca_ctx* ctx, const ffca_dims* d, const ffca_fit_opts* o, const double* x,
             const double* power, double* W, double* L, double* H, double* nll,
             double* nll_slots, int32_t* bin_status) {
  if (!ctx || !d || !o) return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit: null argument");
  int rc = check_dims(d->batch * d->bins, d->dim, d->sources, d->frames);
  if (rc) return rc;
  if (d->batch < 1 || d->bins < 1) return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit: empty shape");
  if (o->iters < 0) return set_err(FFCA_INVALID_ARGUMENT, "fastfca_fit: negative iteration count");
  if (o->flavor != FFCA_FLAVOR_EM && o->flavor != FFCA_FLAVOR_MM)
    return set_err(FFCA_INVALID_ARGUMENT, "fastfca_fit: unknown flavor");
  if (!x || !W || !L || !H) return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit: null buffer");
  if (o->record_trace && !nll && !nll_slots)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit: record_trace needs an nll buffer");
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  if (o->iters == 0 && !o->record_trace) {
    if (bin_status) std::memset(bin_status, 0, sizeof(int32_t) * d->batch * d->bins);
    return FFCA_OK;
  }
  if (o->precision == FFCA_PREC_FP64)
    return fit_host<double>(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status);
  return fit_host<float>(ctx, d, o, x, power, W, L, H, nll, nll_slots, bin_status);
}

int ffca_nll_bins(ffca_ctx* ctx, const ffca_dims* d, int precision, const double* x,
                  const double* W, const double* L, const double* H, double* out) {
  if (!ctx || !d || !x || !W || !L || !H || !out)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_nll_bins: null argument");
  int rc = check_dims(d->batch * d->bins, d->dim, d->sources, d->frames);
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
  ctx->launches = 0;
  DeviceGuard g(ctx->device);
  rc = (precision == FFCA_PREC_FP64)
           ? fit_host<double>(ctx, &one, &o, x, nullptr, w.data(), l.data(), h.data(), nullptr,
                              slots.data(), nullptr)
           : fit_host<float>(ctx, &one, &o, x, nullptr, w.data(), l.data(), h.data(), nullptr,
                             slots.data(), nullptr);
  if (rc) return rc;
  std::memcpy(out, slots.data(), sizeof(double) * P);
  return FFCA_OK;
}

int ffca_power_scale(ffca_ctx* ctx, const ffca_dims* d, const double* x, double* out) {
  if (!ctx || !d || !x || !out) return set_err(FFCA_INVALID_ARGUMENT, "ffca_power_scale: null argument");
  const int P = d->batch * d->bins, M = d->dim, T = d->frames;
  if (P < 1 || M < 1 || T < 1) return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: empty spectrogram");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaError_t err;
  void* dx = ctx->get(kX, size_t(P) * T * M * 16, &err);
  double* dp = static_cast<double*>(ctx->get(kPow, size_t(P) * 8, &err));
  if (!dx || !dp) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dx, x, size_t(P) * T * M * 16, cudaMemcpyHostToDevice, ctx->stream));
  ffca::power_aos_kernel<<<P, 256, 0, ctx->stream>>>(reinterpret_cast<const double2*>(dx), dp, M, T);
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
  int rc = check_dims(d->batch * d->bins, d->dim, d->sources, d->frames);
  if (rc) return rc;
  const int P = d->batch * d->bins, M = d->dim, N = d->sources, T = d->frames;
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  void* xs = nullptr;
  void* hs = nullptr;
  double* hd = nullptr;
  rc = (precision == FFCA_PREC_FP64) ? pack_inputs<double>(ctx, P, M, N, T, x, H, &xs, &hs, &hd, st)
                                     : pack_inputs<float>(ctx, P, M, N, T, x, H, &xs, &hs, &hd, st);
  if (rc) return rc;
  double* dW = static_cast<double*>(ctx->get(kW, size_t(P) * M * M * 16, &err));
  double* dL = static_cast<double*>(ctx->get(kL, size_t(P) * M * N * 8, &err));
  const size_t nimg = size_t(N) * P * T * M;
  double* dimg = static_cast<double*>(ctx->get(kImg, nimg * 16, &err));
  if (!dW || !dL || !dimg) return set_err(FFCA_CUDA_ERROR, "ffca: alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dW, W, size_t(P) * M * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dL, L, size_t(P) * M * N * 8, cudaMemcpyHostToDevice, st));
  rc = (precision == FFCA_PREC_FP64)
           ? launch_sep<double>(ctx, M, xs, dW, dL, hs, P, N, T, dimg, nullptr, st)
           : launch_sep<float>(ctx, M, xs, dW, dL, hs, P, N, T, dimg, nullptr, st);
  if (rc) return rc;
  FFCA_CUDA(cudaMemcpyAsync(images, dimg, nimg * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_fit_device(ffca_ctx* ctx, int problems, int bins_per_mixture, int prob_offset, int dim,
                    int sources, int frames, const ffca_fit_opts* o, const void* x_soa,
                    const double* power, double* W, double* L, void* H_soa, double* nll_slots,
                    int32_t* status, void* stream) {
  if (!ctx || !o || !x_soa || !power || !W || !L || !H_soa || !status)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_device: null argument");
  int rc = check_dims(problems, dim, sources, frames);
  if (rc) return rc;
  if (bins_per_mixture < 1 || o->iters < 0)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_device: bad arguments");
  if (o->record_trace && !nll_slots)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_fit_device: record_trace needs nll_slots");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  ffca::FitParams fp{};
  fp.nprob = problems;
  fp.N = sources;
  fp.T = frames;
  fp.F = bins_per_mixture;
  fp.prob_offset = prob_offset;
  fp.x = x_soa;
  fp.H = H_soa;
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
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return o->precision == FFCA_PREC_FP64 ? launch_fit<double>(ctx, dim, fp, st)
                                        : launch_fit<float>(ctx, dim, fp, st);
}

int ffca_separate_device(ffca_ctx* ctx, int problems, int dim, int sources, int frames,
                         int precision, const void* x_soa, const double* W, const double* L,
                         const void* H_soa, void* images_soa, void* stream) {
  if (!ctx || !x_soa || !W || !L || !H_soa || !images_soa)
    return set_err(FFCA_INVALID_ARGUMENT, "ffca_separate_device: null argument");
  int rc = check_dims(problems, dim, sources, frames);
  if (rc) return rc;
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return precision == FFCA_PREC_FP64
             ? launch_sep<double>(ctx, dim, x_soa, W, L, H_soa, problems, sources, frames, nullptr,
                                  images_soa, st)
             : launch_sep<float>(ctx, dim, x_soa, W, L, H_soa, problems, sources, frames, nullptr,
                                 images_soa, st);
}

int ffca_power_scale_device(ffca_ctx* ctx, int problems, int dim, int frames, int precision,
                            const void* x_soa, double* out, void* stream) {
  if (!ctx || !x_soa || !out) return set_err(FFCA_INVALID_ARGUMENT, "ffca_power_scale_device: null");
  if (problems < 1 || dim < 1 || frames < 1)
    return set_err(FFCA_INVALID_ARGUMENT, "sample_covs: empty spectrogram");
  DeviceGuard g(ctx->device);
  ctx->launches = 0;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (precision == FFCA_PREC_FP64)
    ffca::power_soa_kernel<double><<<problems, 256, 0, st>>>(
        reinterpret_cast<const double2*>(x_soa), out, dim, frames);
  else
    ffca::power_soa_kernel<float><<<problems, 256, 0, st>>>(
        reinterpret_cast<const float2*>(x_soa), out, dim, frames);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

}  // extern "C"
