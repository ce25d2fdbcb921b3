// fit_big.cu -- instantiations and launcher of the large-bin fit kernel
// (fit_big.cuh): M = 8, N = 12 (BASELINE config 3) in fp32 and the fp64
// check mode, and M = 4, N = 6 (BASELINE config 2) in fp32.
#include <cstdlib>

#include "fit_big.cuh"
#include "internal.hpp"

namespace ffca {

namespace {

template <int M, int N, typename R, int SLOTS, int NTHR, int MS, int MINB = 1, bool AUXG = false,
          bool EXACTVAR = false>
int launch_big_t(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, bool* handled) {
  using Cfg = BigCfg<M, N, R, SLOTS, NTHR, MS, AUXG>;
  *handled = false;
  int dev_max = 0;
  cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  if (dev_max <= 0) dev_max = 227 * 1024;
  const int C = (fp.T + Cfg::TCAP - 1) / Cfg::TCAP;
  if (C < 1 || C > 16) return FFCA_OK;  // not handled: the streaming kernel takes it
  const BigLayout lay = Cfg::layout(C, fp.T);
  if (lay.total > dev_max) return FFCA_OK;
  *handled = true;
  if (fp.nprob == 0) return FFCA_OK;
  if (AUXG) {
    // Cold-path scratch (restart generator, saved W, reference-order IP
    // matrices) in global memory: AUX_BYTES per CTA of the CALL (concurrent chunks of the
    // pipelined host fit take disjoint rows).
    cudaError_t err;
    const size_t per = size_t(C) * Cfg::AUX_BYTES;
    const size_t nall = size_t(fp.work_total > 0 ? fp.work_total : fp.nprob);
    char* base = static_cast<char*>(ctx->get(kAux, nall * per, &err));
    if (!base)
      return ffca_set_err(FFCA_CUDA_ERROR, std::string("ffca: aux scratch alloc: ") + cudaGetErrorString(err));
    fp.aux = base + size_t(fp.work_total > 0 ? fp.work_first : 0) * per;
  }
  if (big_incr<M, R, SLOTS>() && !EXACTVAR) {
    // U scratch [problem][T][M] (fit_big.cuh INCR): one allocation for the
    // whole call, this launch's rows at work_first (concurrent chunks of the
    // pipelined host fit must not share rows or regrow the buffer).
    cudaError_t err;
    const size_t per = size_t(fp.T) * M * sizeof(R);
    const size_t nall = size_t(fp.work_total > 0 ? fp.work_total : fp.nprob);
    char* base = static_cast<char*>(ctx->get(kU, nall * per, &err));
    if (!base)
      return ffca_set_err(FFCA_CUDA_ERROR, std::string("ffca: U scratch alloc: ") + cudaGetErrorString(err));
    fp.work = base + size_t(fp.work_total > 0 ? fp.work_first : 0) * per;
  }
  if (C == 1) {
    auto kern = big_fit_kernel<M, N, R, SLOTS, NTHR, MS, false, MINB, AUXG, EXACTVAR>;
    FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total));
    kern<<<fp.nprob, NTHR, lay.total, st>>>(fp, lay);
  } else {
    auto kern = big_fit_kernel<M, N, R, SLOTS, NTHR, MS, true, MINB, AUXG, EXACTVAR>;
    FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lay.total));
    if (C > 8) FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(fp.nprob) * unsigned(C));
    cfg.blockDim = dim3(NTHR);
    cfg.dynamicSmemBytes = lay.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FFCA_CUDA(cudaLaunchKernelEx(&cfg, kern, fp, lay));
  }
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

}  // namespace

// The large-bin kernel takes IP+EM fits of snapshot records with the
// shapes instantiated here; *handled = false leaves the fit to fit_kernel.
int launch_fit_big(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, int M, bool fp64, bool* handled) {
  *handled = false;
  if (getenv("FFCA_NO_BIG")) return FFCA_OK;  // A/B experiments against fit_kernel
  if (fp.blk || fp.flavor != 0 || fp.fix_loadings) return FFCA_OK;
  if (M == 8 && fp.N == 12) {
    if (fp64) return launch_big_t<8, 12, double, 4, 448, 2>(ctx, fp, st, handled);
    // fp32: 256 threads x 8 slots = 2048 frames per CTA and TWO CTAs per SM
    // (111 KB of shared memory and 256 tensor-memory columns each): a c3 bin
    // is a 4-CTA cluster, and every SM hosts slices of two bins, so one bin's
    // reductions, cluster barriers and IP overlap the other's frame passes.
    // FFCA_BIG_WIDE=1: the 512-thread, one-CTA-per-SM shape (2-CTA clusters).
    // FFCA_EXACT_VARIANCES=1: the mixture variances are summed afresh in
    // every EM sweep instead of being updated incrementally (~5 % slower).
    if (getenv("FFCA_EXACT_VARIANCES"))
      return launch_big_t<8, 12, float, 8, 256, 1, 2, true, true>(ctx, fp, st, handled);
    if (getenv("FFCA_BIG_WIDE")) return launch_big_t<8, 12, float, 8, 512, 1>(ctx, fp, st, handled);
    return launch_big_t<8, 12, float, 8, 256, 1, 2, true>(ctx, fp, st, handled);
  }
  // BASELINE config 2 (M = 4, N = 6, T = 2000): 256 threads x 8 frame slots
  // hold a 2048-frame bin in one CTA; three CTAs (three bins) share an SM
  // (66 KB of H planes and 128 tensor-memory columns each), so one bin's
  // reductions and IP overlap the others' frame passes.  Short bins stay with
  // fit_kernel (one resident CTA in shared memory is cheaper there).
  if (M == 4 && fp.N == 6 && !fp64 && fp.T > 512)
    return launch_big_t<4, 6, float, 8, 256, 1, 3>(ctx, fp, st, handled);
  // BASELINE config 4 (M = 3, N = 4, T = 626): 96 threads x 7 frame slots hold
  // a 672-frame bin; 11 KB of H planes and 64 tensor-memory columns per bin,
  // eight bins per SM, so the per-bin serial sections (N + 1 reductions, the
  // IP, the balance) of one bin overlap the frame passes of seven others.
  if (M == 3 && fp.N == 4 && !fp64 && fp.T > 192 && fp.T <= 672 && !getenv("FFCA_NO_BIG3"))
    return launch_big_t<3, 4, float, 7, 96, 1, 8>(ctx, fp, st, handled);
  return FFCA_OK;
}

}  // namespace ffca
