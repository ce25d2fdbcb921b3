// fit_launch.cuh -- per-dim fit launcher template; instantiated once per M in
// fit_m<M>.cu so the 32 kernel variants compile in parallel.
#pragma once

#include "internal.hpp"

namespace ffca {

template <int M, int NMAX, typename R>
int launch_fit_t(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  const int threads = fit_threads(M, fp.T);
  const int nwarps = threads / 32;
  int nc = 16 / M;
  if (nc < 1) nc = 1;
  fp.nc = nc;
  int dev_max = 0;
  cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const FitSmem<M, NMAX, R> res_lay(nwarps, fp.N, fp.T, nc, true);
  const int budget = dev_max > 0 ? dev_max - 2048 : 200 * 1024;
  fp.resident = (res_lay.total <= budget) ? 1 : 0;
  const FitSmem<M, NMAX, R> lay(nwarps, fp.N, fp.T, nc, fp.resident != 0);
  cudaError_t err;
  if (!fp.resident) {
    fp.U = ctx->get(kU, size_t(fp.nprob) * M * fp.T * sizeof(R), &err);
    if (!fp.U)
      return ffca_set_err(FFCA_CUDA_ERROR, std::string("ffca: scratch alloc: ") + cudaGetErrorString(err));
  }
  auto kern = fit_kernel<M, NMAX, R>;
  FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total));
  kern<<<fp.nprob, threads, lay.total, st>>>(fp);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

template <int M, typename R>
int launch_fit_nmax(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  if (fp.N <= 4) return launch_fit_t<M, 4, R>(ctx, fp, st);
  return launch_fit_t<M, 16, R>(ctx, fp, st);
}

}  // namespace ffca

#define FFCA_DEFINE_FIT_LAUNCHER(M)                                                   \
  namespace ffca {                                                                    \
  int launch_fit_m##M(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, bool fp64) {     \
    return fp64 ? launch_fit_nmax<M, double>(ctx, fp, st)                             \
                : launch_fit_nmax<M, float>(ctx, fp, st);                             \
  }                                                                                   \
  }
