// internal.hpp -- host-side internals shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/ffca.h"
#include "fit_kernel.cuh"

// Set the calling thread's ffca_last_error() message; returns `code`.
int ffca_set_err(int code, const std::string& msg);

#define FFCA_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return ffca_set_err(FFCA_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kMaxChunks = 16;

struct ffca_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t cstream[16] = {};  // host-fit chunk pipeline (kMaxChunks)
  int launches = 0;
  unsigned long long* timing = nullptr;  // diagnostics: per-problem phase counters
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
  };
  Buf bufs[16];
  Buf pinned[8];  // page-locked host staging (ffca_pinned_buffer)
  // Grow-only device scratch, slot k.
  void* get(int k, size_t bytes, cudaError_t* err) {
    Buf& b = bufs[k];
    *err = cudaSuccess;
    if (b.n >= bytes && b.p) return b.p;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
    *err = cudaMalloc(&b.p, bytes < 256 ? 256 : bytes);
    if (*err != cudaSuccess) return nullptr;
    b.n = bytes;
    return b.p;
  }
};

namespace ffca {

enum Slot { kX = 0, kXs, kH, kHs, kW, kL, kPow, kNll, kStat, kU, kImg, kWave, kSpec, kFrames, kSepRec, kAux, kNumSlots };

// Threads per fit CTA: about 4 frames per thread, capped at the kernel's
// launch bound; a multiple of 32*M when the weighted-covariance pass is split
// by channel (M > 4).
inline int fit_threads(int M, int T, int maxt, int msplit = 0) {
  const int per = (msplit > 1) ? 32 * msplit : ((M <= 4) ? 32 : 32 * M);
  const int want = (T + 3) / 4;
  int th = ((want + per - 1) / per) * per;
  const int cap = (maxt / per) * per;
  if (th > cap) th = cap;
  if (th < per) th = per;
  if (M <= 4 && th < 64) th = 64;
  return th;
}

// Per-dim launchers (fit_m<M>.cu): fp64 selects the check-mode instantiation.
#define FFCA_DECLARE_FIT_LAUNCHER(M) \
  int launch_fit_m##M(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, bool fp64);
FFCA_DECLARE_FIT_LAUNCHER(1)
FFCA_DECLARE_FIT_LAUNCHER(2)
FFCA_DECLARE_FIT_LAUNCHER(3)
FFCA_DECLARE_FIT_LAUNCHER(4)
FFCA_DECLARE_FIT_LAUNCHER(5)
FFCA_DECLARE_FIT_LAUNCHER(6)
FFCA_DECLARE_FIT_LAUNCHER(7)
FFCA_DECLARE_FIT_LAUNCHER(8)

// fastfca_separate (separate.cu).  xs / Hs: device x [P][T][M], H [P][T][N] in
// the compute type; out: images [N][P][T][M] in the compute type, or fp64
// images from the fp32 compute path when out_double (host-path staging).
int launch_separate(ffca_ctx* ctx, int M, bool fp64, bool out_double, const void* xs,
                    const double* W, const double* L, const void* Hs, int P, int N, int T,
                    void* out, cudaStream_t st);

// Large-bin kernel (fit_big.cu): sets *handled when it took the fit.
int launch_fit_big(ffca_ctx* ctx, FitParams& fp, cudaStream_t st, int M, bool fp64, bool* handled);

}  // namespace ffca
