// stft.cu -- C ABI of the STFT front end / iSTFT back end (include/ffca.h),
// reference stft.hpp:40-56 / stft.cpp:12-128.  Validation with the
// reference's messages, device buffers, kernel dispatch; no CPU path.

#include <cuda_runtime.h>

#include <string>

#include "internal.hpp"
#include "stft_kernels.cuh"

using namespace ffca;

namespace {

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int log2_exact(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// stft.cpp:14-19
int validate(int frame_len, int shift) {
  if (frame_len <= 0 || (frame_len & (frame_len - 1)) != 0)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: frame length must be a power of two");
  if (shift * 2 != frame_len)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: shift must be frame_len/2");
  if (frame_len > 4096)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: frame length above 4096 is not supported");
  return FFCA_OK;
}

// stft.cpp:41-49; -1 with the error set when the signal is too short.
long long frame_count(long long length, int frame_len, int shift, int padding) {
  if (padding == FFCA_STFT_CENTERED) return (length + shift - 1) / shift + 1;
  if (length < frame_len) {
    ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: signal shorter than one frame");
    return -1;
  }
  return (length - frame_len) / shift + 1;
}

int fft_threads(int n) { return n / 2 < 256 ? (n / 2 < 32 ? 32 : n / 2) : 256; }

template <typename K>
int smem_attr(K kern, int bytes) {
  if (bytes > 48 * 1024)
    FFCA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return FFCA_OK;
}

template <typename In, typename OutC>
int launch_stft(ffca_ctx* ctx, const In* wave, long long len, int C, int n, int shift,
                long long offset, int frames, OutC* spec, cudaStream_t st) {
  const int bytes = 2 * n * int(sizeof(double2));
  auto kern = stft_kernel<In, OutC>;
  int rc = smem_attr(kern, bytes);
  if (rc) return rc;
  kern<<<dim3(frames, C), fft_threads(n), bytes, st>>>(wave, len, C, n, log2_exact(n), shift,
                                                        offset, frames, spec);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

template <typename InC, typename Out>
int launch_istft(ffca_ctx* ctx, const InC* spec, int C, int n, int shift, int frames,
                 long long offset, long long out_len, Out* wave, cudaStream_t st) {
  cudaError_t err;
  double* fr = static_cast<double*>(ctx->get(kFrames, size_t(C) * frames * n * 8, &err));
  if (!fr) return ffca_set_err(FFCA_CUDA_ERROR, "ffca: istft scratch alloc failed");
  const int bytes = 2 * n * int(sizeof(double2));
  auto kern = istft_frame_kernel<InC>;
  int rc = smem_attr(kern, bytes);
  if (rc) return rc;
  kern<<<dim3(frames, C), fft_threads(n), bytes, st>>>(spec, C, n, log2_exact(n), frames, fr);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  const long long total = out_len * C;
  istft_ola_kernel<Out><<<unsigned((total + 255) / 256), 256, 0, st>>>(fr, C, n, shift, frames,
                                                                       offset, out_len, wave);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

}  // namespace

extern "C" {

long long ffca_stft_frame_count(long long length, int frame_len, int shift, int padding) {
  if (padding != FFCA_STFT_CENTERED && padding != FFCA_STFT_FULL_FRAMES) {
    ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: unknown padding");
    return -1;
  }
  return frame_count(length, frame_len, shift, padding);
}

int ffca_stft(ffca_ctx* ctx, int channels, long long length, int frame_len, int shift, int padding,
              const double* samples, double* spec) {
  if (!ctx || !samples || !spec || channels < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_stft: null argument or no channels");
  int rc = validate(frame_len, shift);
  if (rc) return rc;
  if (length < frame_len)  // stft.cpp:54-55
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: signal shorter than one frame");
  const long long frames = ffca_stft_frame_count(length, frame_len, shift, padding);
  if (frames < 0) return FFCA_INVALID_ARGUMENT;
  ctx->launches = 0;
  Guard g(ctx->device);
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  const int bins = frame_len / 2 + 1;
  const size_t nin = size_t(length) * channels, nout = size_t(bins) * frames * channels;
  double* dw = static_cast<double*>(ctx->get(kWave, nin * 8, &err));
  double2* ds = static_cast<double2*>(ctx->get(kSpec, nout * 16, &err));
  if (!dw || !ds) return ffca_set_err(FFCA_CUDA_ERROR, "ffca: stft alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dw, samples, nin * 8, cudaMemcpyHostToDevice, st));
  const long long offset = padding == FFCA_STFT_CENTERED ? shift : 0;
  rc = launch_stft<double, double2>(ctx, dw, length, channels, frame_len, shift, offset,
                                    int(frames), ds, st);
  if (rc) return rc;
  FFCA_CUDA(cudaMemcpyAsync(spec, ds, nout * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_istft(ffca_ctx* ctx, int channels, int bins, int frames, int frame_len, int shift,
               int padding, long long out_len, const double* spec, double* samples) {
  if (!ctx || !spec || !samples || channels < 1 || frames < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_istft: null argument or empty shape");
  int rc = validate(frame_len, shift);
  if (rc) return rc;
  if (bins != frame_len / 2 + 1)  // stft.cpp:89-90
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "istft: bin count does not match frame_len");
  const long long want = ffca_stft_frame_count(out_len, frame_len, shift, padding);
  if (want != frames)  // stft.cpp:91-93
    return ffca_set_err(FFCA_INVALID_ARGUMENT,
                        "istft: frame count inconsistent with out_len and padding");
  ctx->launches = 0;
  Guard g(ctx->device);
  cudaStream_t st = ctx->stream;
  cudaError_t err;
  const size_t nin = size_t(bins) * frames * channels, nout = size_t(out_len) * channels;
  double2* ds = static_cast<double2*>(ctx->get(kSpec, nin * 16, &err));
  double* dw = static_cast<double*>(ctx->get(kWave, nout * 8 > 0 ? nout * 8 : 8, &err));
  if (!ds || !dw) return ffca_set_err(FFCA_CUDA_ERROR, "ffca: istft alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(ds, spec, nin * 16, cudaMemcpyHostToDevice, st));
  const long long offset = padding == FFCA_STFT_CENTERED ? shift : 0;
  rc = launch_istft<double2, double>(ctx, ds, channels, frame_len, shift, frames, offset, out_len,
                                     dw, st);
  if (rc) return rc;
  if (nout) FFCA_CUDA(cudaMemcpyAsync(samples, dw, nout * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_stft_device(ffca_ctx* ctx, int channels, long long length, int frame_len, int shift,
                     int padding, int precision, const void* samples_dev, void* x_dev,
                     void* stream) {
  if (!ctx || !samples_dev || !x_dev || channels < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_stft_device: null argument or no channels");
  int rc = validate(frame_len, shift);
  if (rc) return rc;
  if (length < frame_len)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "stft: signal shorter than one frame");
  const long long frames = ffca_stft_frame_count(length, frame_len, shift, padding);
  if (frames < 0) return FFCA_INVALID_ARGUMENT;
  Guard g(ctx->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const long long offset = padding == FFCA_STFT_CENTERED ? shift : 0;
  if (precision == FFCA_PREC_FP64)
    return launch_stft<double, double2>(ctx, static_cast<const double*>(samples_dev), length,
                                        channels, frame_len, shift, offset, int(frames),
                                        static_cast<double2*>(x_dev), st);
  return launch_stft<float, float2>(ctx, static_cast<const float*>(samples_dev), length, channels,
                                    frame_len, shift, offset, int(frames),
                                    static_cast<float2*>(x_dev), st);
}

int ffca_istft_device(ffca_ctx* ctx, int channels, int frames, int frame_len, int shift,
                      int padding, long long out_len, int precision, const void* spec_dev,
                      void* samples_dev, void* stream) {
  if (!ctx || !spec_dev || !samples_dev || channels < 1 || frames < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_istft_device: null argument or empty shape");
  int rc = validate(frame_len, shift);
  if (rc) return rc;
  if (ffca_stft_frame_count(out_len, frame_len, shift, padding) != frames)
    return ffca_set_err(FFCA_INVALID_ARGUMENT,
                        "istft: frame count inconsistent with out_len and padding");
  Guard g(ctx->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const long long offset = padding == FFCA_STFT_CENTERED ? shift : 0;
  if (precision == FFCA_PREC_FP64)
    return launch_istft<double2, double>(ctx, static_cast<const double2*>(spec_dev), channels,
                                         frame_len, shift, frames, offset, out_len,
                                         static_cast<double*>(samples_dev), st);
  return launch_istft<float2, float>(ctx, static_cast<const float2*>(spec_dev), channels, frame_len,
                                     shift, frames, offset, out_len,
                                     static_cast<float*>(samples_dev), st);
}

}  // extern "C"
