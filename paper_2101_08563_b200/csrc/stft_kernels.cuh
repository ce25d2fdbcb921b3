// stft_kernels.cuh -- STFT analysis / synthesis on the GPU (SURVEY §8(f) next
// #3): the front and back ends on either side of the fit, producing and
// consuming the fit kernel's device layout directly.
//
// Reference: stft.cpp:33-39 (periodic sqrt-Hann window), :41-49 (frame
// counts), :51-83 (stft), :85-128 (istft).  Every FFT here is a hand-written
// radix-2 Stockham transform in fp64 in shared memory (one CTA per frame and
// channel); the data converts to the caller's precision only at the edges.
//
// Layouts (the reference's containers, Eigen column-major):
//   samples [length][channels]          MultichannelWave::samples (ch, t)
//   spec    [bins][frames][channels]    Spectrogram::f[b] (ch, j) -- also the
//                                       fit kernel's x_dev layout [P][T][M]
#pragma once

#include "common.cuh"

namespace ffca {

// sqrt_hann_window (stft.cpp:33-39), periodic: squared windows at 50 %
// overlap sum to one.
__device__ __forceinline__ double sqrt_hann(int k, int n) {
  return sqrt(0.5 - 0.5 * cos(2.0 * 3.14159265358979323846 * k / n));
}

// In-place-ish radix-2 Stockham FFT of n = 2^logn points held in a (result
// returned: a or b).  sign = -1 forward, +1 inverse (unscaled).  Called by the
// whole CTA.
__device__ double2* stockham_fft(double2* a, double2* b, int n, int logn, double sign) {
  const int tid = threadIdx.x, nth = blockDim.x;
  int len = n, stride = 1;
  for (int s = 0; s < logn; ++s) {
    const int m = len >> 1;
    for (int t = tid; t < (n >> 1); t += nth) {
      const int p = t / stride, q = t - p * stride;
      double sn, cs;
      sincospi(sign * 2.0 * p / len, &sn, &cs);  // exp(sign * 2 pi i p / len)
      const double2 u = a[q + stride * p];
      const double2 v = a[q + stride * (p + m)];
      const double2 d = make_double2(u.x - v.x, u.y - v.y);
      b[q + stride * (2 * p)] = make_double2(u.x + v.x, u.y + v.y);
      b[q + stride * (2 * p + 1)] = make_double2(d.x * cs - d.y * sn, d.x * sn + d.y * cs);
    }
    __syncthreads();
    double2* t2 = a;
    a = b;
    b = t2;
    len = m;
    stride <<= 1;
  }
  return a;
}

template <typename T> __device__ __forceinline__ double as_double(T v) { return double(v); }

template <typename C> __device__ __forceinline__ C to_cplx(double2 v);
template <> __device__ __forceinline__ float2 to_cplx<float2>(double2 v) {
  return make_float2(float(v.x), float(v.y));
}
template <> __device__ __forceinline__ double2 to_cplx<double2>(double2 v) { return v; }

// stft (stft.cpp:51-83): one CTA per (frame j, channel ch).  Frame j covers
// samples [j*shift - offset, +n), zero outside the signal, times the window;
// bins 0..n/2 of its DFT go to spec[b][j][ch].
template <typename In, typename OutC>
__global__ void stft_kernel(const In* __restrict__ samples, long long len, int channels, int n,
                            int logn, int shift, long long offset, int frames,
                            OutC* __restrict__ spec) {
  extern __shared__ double2 fsm[];
  const int j = blockIdx.x, ch = blockIdx.y;
  double2* a = fsm;
  double2* b = fsm + n;
  const long long start = (long long)j * shift - offset;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const long long t = start + k;
    const double v = (t >= 0 && t < len) ? as_double(samples[t * channels + ch]) * sqrt_hann(k, n) : 0.0;
    a[k] = make_double2(v, 0.0);
  }
  __syncthreads();
  const double2* r = stockham_fft(a, b, n, logn, -1.0);
  const int bins = n / 2 + 1;
  for (int k = threadIdx.x; k < bins; k += blockDim.x)
    spec[(size_t(k) * frames + j) * channels + ch] = to_cplx<OutC>(r[k]);
}

template <typename C> __device__ __forceinline__ double2 cplx_to_d(C v) {
  return make_double2(double(v.x), double(v.y));
}

// istft, per frame (stft.cpp:110-118): the one-sided spectrum of (ch, j) is
// extended Hermitian (the imaginary parts of DC and Nyquist drop out, as in a
// real inverse FFT), inverse transformed, scaled 1/n and windowed into
// frames_out[ch][j][k].
template <typename InC>
__global__ void istft_frame_kernel(const InC* __restrict__ spec, int channels, int n, int logn,
                                   int frames, double* __restrict__ frames_out) {
  extern __shared__ double2 fsm[];
  const int j = blockIdx.x, ch = blockIdx.y;
  double2* a = fsm;
  double2* b = fsm + n;
  const int half = n / 2;
  for (int k = threadIdx.x; k <= half; k += blockDim.x) {
    double2 v = cplx_to_d(spec[(size_t(k) * frames + j) * channels + ch]);
    if (k == 0 || k == half) v.y = 0.0;
    a[k] = v;
    if (k > 0 && k < half) a[n - k] = make_double2(v.x, -v.y);
  }
  __syncthreads();
  const double2* r = stockham_fft(a, b, n, logn, 1.0);
  const double inv_n = 1.0 / double(n);
  double* fo = frames_out + (size_t(ch) * frames + j) * n;
  for (int k = threadIdx.x; k < n; k += blockDim.x) fo[k] = sqrt_hann(k, n) * (r[k].x * inv_n);
}

// istft overlap-add (stft.cpp:99-127): sample t of channel ch sits at buffer
// position p = t + offset; its frames are added in ascending j (the
// reference's accumulation order) and divided by max(sum w^2, 1e-12).
template <typename Out>
__global__ void istft_ola_kernel(const double* __restrict__ frames_in, int channels, int n,
                                 int shift, int frames, long long offset, long long out_len,
                                 Out* __restrict__ samples) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= out_len * channels) return;
  const long long t = i / channels;
  const int ch = int(i - t * channels);
  const long long p = t + offset;
  const long long buf_len = (long long)(frames - 1) * shift + n;
  double v = 0.0;
  if (p < buf_len) {
    long long jlo = (p - n) / shift + 1;
    if (p - n < 0) jlo = 0;
    if (jlo < 0) jlo = 0;
    long long jhi = p / shift;
    if (jhi > frames - 1) jhi = frames - 1;
    double acc = 0.0, ws = 0.0;
    for (long long j = jlo; j <= jhi; ++j) {
      const int k = int(p - j * shift);
      if (k < 0 || k >= n) continue;
      const double w = sqrt_hann(k, n);
      ws += w * w;
      acc += frames_in[(size_t(ch) * frames + j) * n + k];
    }
    v = acc / fmax(ws, 1e-12);
  }
  samples[t * channels + ch] = Out(v);
}

}  // namespace ffca
