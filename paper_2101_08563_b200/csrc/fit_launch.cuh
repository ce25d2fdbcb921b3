// fit_launch.cuh -- per-dim fit launcher; instantiated once per M in
// fit_m<M>.cu so the kernel variants compile in parallel.
//
// fp32 variants for M <= 4 are specialized on the source count N in
// {2,3,4,6,12} (no source-loop guards); every other shape uses NT in {4,8,16}
// with runtime guards.  The fp64 check mode uses NT in {4,16}.
#pragma once

#include "internal.hpp"

namespace ffca {

template <int M, int NT, bool EXACT, typename R>
int launch_fit_t(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  const int threads = fit_threads(M, fp.T, Launch<M>::threads);
  const int nwarps = threads / 32;
  int nc = 16 / M;
  if (nc < 1) nc = 1;
  fp.nc = nc;
  int dev_max = 0;
  cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const FitSmem<M, NT, R> res_lay(nwarps, fp.N, fp.T, nc, true);
  const int budget = dev_max > 0 ? dev_max - 2048 : 200 * 1024;
  fp.resident = (res_lay.total <= budget) ? 1 : 0;
  const FitSmem<M, NT, R> lay(nwarps, fp.N, fp.T, nc, fp.resident != 0);
  cudaError_t err;
  if (!fp.resident) {
    fp.work = ctx->get(kU, size_t(fp.nprob) * 2 * M * fp.T * sizeof(R), &err);
    if (!fp.work)
      return ffca_set_err(FFCA_CUDA_ERROR, std::string("ffca: scratch alloc: ") + cudaGetErrorString(err));
  }
  auto kern = fit_kernel<M, NT, EXACT, R>;
  FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total));
  kern<<<fp.nprob, threads, lay.total, st>>>(fp);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

template <int M>
int launch_fit_f32(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  if constexpr (M <= 4) {
    // Exact source-count specializations for the common shapes.
    switch (fp.N) {
      case 2: return launch_fit_t<M, 2, true, float>(ctx, fp, st);
      case 3: return launch_fit_t<M, 3, true, float>(ctx, fp, st);
      case 4: return launch_fit_t<M, 4, true, float>(ctx, fp, st);
      case 6: return launch_fit_t<M, 6, true, float>(ctx, fp, st);
      case 12: return launch_fit_t<M, 12, true, float>(ctx, fp, st);
      default: break;
    }
  }
  if (fp.N <= 4) return launch_fit_t<M, 4, false, float>(ctx, fp, st);
  if (fp.N <= 8) return launch_fit_t<M, 8, false, float>(ctx, fp, st);
  return launch_fit_t<M, 16, false, float>(ctx, fp, st);
}

template <int M>
int launch_fit_f64(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  if (fp.N <= 4) return launch_fit_t<M, 4, false, double>(ctx, fp, st);
  return launch_fit_t<M, 16, false, double>(ctx, fp, st);
}

}  // namespace ffca

#define FFCA_DEFINE_FIT_LAUNCHER(M)                                               \
  namespace ffca {                                                                \
  int launch_fit_m##M(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, bool fp64) { \
    return fp64 ? launch_fit_f64<M>(ctx, fp, st) : launch_fit_f32<M>(ctx, fp, st); \
  }                                                                               \
  }
