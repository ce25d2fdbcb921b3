// fit_launch.cuh -- per-dim fit launcher; instantiated once per M in
// fit_m<M>.cu so the kernel variants compile in parallel.
//
// fp32 variants for M <= 4 are specialized on the source count N in
// {2,3,4,6,12} (no source-loop guards); every other shape uses NT in {4,8,16}
// with runtime guards.  The fp64 check mode uses NT in {4,16}.
//
// Placement: a bin whose records (16M + 4N bytes per frame) fit one CTA's
// shared memory runs on one CTA; otherwise its frames are split over a
// thread-block cluster of C = 2..16 CTAs (guarded variants, DSMEM
// reductions); beyond 16 CTAs the bin streams from global memory.
#pragma once

#include <cstdlib>

#include "internal.hpp"

namespace ffca {

template <int M, int NT, bool EXACT, typename R, bool CL, bool RES, bool BLK = false>
int launch_fit_cfg(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, int C, int dev_max) {
  int threads = fit_threads(M, fp.tloc, Launch<M>::threads, Split<M>::MSPLIT);
  if (const char* e = getenv("FFCA_FIT_THREADS")) {  // tuning experiments only
    const int v = atoi(e);
    const int per = (M <= 4) ? 32 : 32 * M;
    if (v >= per && v <= Launch<M>::threads && v % per == 0) threads = v;
  }
  const int nwarps = threads / 32;
  const FitSmem<M, NT, R, BLK> lay(nwarps, fp.N, fp.tloc, fp.nc, RES);
  fp.lay = lay;  // the kernel reads its carve-up from the parameters
  if (lay.total > dev_max)
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca: fit kernel shared memory exceeds the device limit");
  auto kern = fit_kernel<M, NT, EXACT, R, CL, RES, BLK>;
  FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total));
  if constexpr (CL) {
    if (C > 8) FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(fp.nprob) * unsigned(C));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = lay.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FFCA_CUDA(cudaLaunchKernelEx(&cfg, kern, fp));
  } else {
    kern<<<fp.nprob, threads, lay.total, st>>>(fp);
  }
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

// Cluster size for a bin: the smallest C in {1, 2, 4, 8, 16} whose per-CTA
// frame range fits the shared-memory budget; 0 when even 16 does not.
template <int M, int NT, typename R, bool BLK = false>
int pick_cluster(const FitParams& fp, int budget) {
  for (int C = 1; C <= 16; C *= 2) {
    const int tloc = (fp.T + C - 1) / C;
    const int nwarps = fit_threads(M, tloc, Launch<M>::threads, Split<M>::MSPLIT) / 32;
    if (FitSmem<M, NT, R, BLK>(nwarps, fp.N, tloc, fp.nc, true).total <= budget) return C;
  }
  return 0;
}

// BLK (block-covariance records): one CTA per bin when the bin fits, else
// streaming (no cluster variants).
template <int M, int NT, bool EXACT, typename R, bool BLK = false>
int launch_fit_t(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  fp.nc = MmChunk<M, NT>::value;
  int dev_max = 0;
  cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  if (dev_max <= 0) dev_max = 227 * 1024;
  const int budget = dev_max - 2048;
  int C = pick_cluster<M, NT, R, BLK>(fp, budget);
  if (const char* e = getenv("FFCA_FORCE_CLUSTER")) {  // tuning experiments only
    const int f = atoi(e);
    if (!EXACT && f > C && f <= 16) C = f;
  }
  cudaError_t err;
  if (C == 1) {
    fp.resident = 1;
    fp.tloc = fp.T;
    return launch_fit_cfg<M, NT, EXACT, R, false, true, BLK>(ctx, fp, st, 1, dev_max);
  }
  if (C > 1) {
    if constexpr (!BLK) {
      fp.resident = 1;
      fp.tloc = (fp.T + C - 1) / C;
      return launch_fit_cfg<M, NT, EXACT, R, true, true>(ctx, fp, st, C, dev_max);
    }
  }
  // Streaming: the bin's records stay in global memory (L2/HBM).  Only the
  // guarded variants get here (needs_cluster routes large bins to them, the
  // exact M = 8, N = 12 variant included when a 16-CTA cluster holds them).
  if constexpr (!EXACT) {
    fp.resident = 0;
    fp.tloc = fp.T;
    // One scratch region for every problem of the CALL, this launch's rows
    // at work_first: the chunks of the pipelined host fit run concurrently on
    // their own streams and must neither share rows nor regrow (free) the
    // buffer under each other.
    const size_t per = size_t(2) * M * fp.T * sizeof(R);
    const size_t nall = size_t(fp.work_total > 0 ? fp.work_total : fp.nprob);
    char* base = static_cast<char*>(ctx->get(kU, nall * per, &err));
    if (!base)
      return ffca_set_err(FFCA_CUDA_ERROR, std::string("ffca: scratch alloc: ") + cudaGetErrorString(err));
    fp.work = base + size_t(fp.work_total > 0 ? fp.work_first : 0) * per;
    return launch_fit_cfg<M, NT, EXACT, R, false, false, BLK>(ctx, fp, st, 1, dev_max);
  } else {
    (void)err;
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca: internal: exact-N variant selected for a large bin");
  }
}

// Large bins go to the guarded (cluster-capable) variants.
template <int M, typename R>
bool needs_cluster(const FitParams& fp) {
  int dev_max = 227 * 1024;
  return pick_cluster<M, 16, R>(fp, dev_max - 2048) != 1;
}

template <int M>
int launch_fit_f32(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  if (fp.blk) {
    if (fp.N <= 4) return launch_fit_t<M, 4, false, float, true>(ctx, fp, st);
    return launch_fit_t<M, 16, false, float, true>(ctx, fp, st);
  }
  if constexpr (M <= 4) {
    if (!needs_cluster<M, float>(fp) && !getenv("FFCA_FORCE_CLUSTER")) {
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
  }
  if constexpr (M == 8) {
    // BASELINE config 3 (M = 8, N = 12): exact source count (vector H loads,
    // no source guards), single CTA or cluster.
    if (fp.N == 12 && pick_cluster<M, 12, float>(fp, 227 * 1024 - 2048) > 0)
      return launch_fit_t<M, 12, true, float>(ctx, fp, st);
  }
  if (fp.N <= 4) return launch_fit_t<M, 4, false, float>(ctx, fp, st);
  if (fp.N <= 8) return launch_fit_t<M, 8, false, float>(ctx, fp, st);
  return launch_fit_t<M, 16, false, float>(ctx, fp, st);
}

template <int M>
int launch_fit_f64(ffca_ctx* ctx, FitParams& fp, cudaStream_t st) {
  if (fp.blk) {
    if (fp.N <= 4) return launch_fit_t<M, 4, false, double, true>(ctx, fp, st);
    return launch_fit_t<M, 16, false, double, true>(ctx, fp, st);
  }
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
