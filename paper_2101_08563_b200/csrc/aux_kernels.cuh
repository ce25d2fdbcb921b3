// aux_kernels.cuh -- layout conversion at the boundary, per-bin power and the
// decomposed multichannel Wiener filter output kernel.
#pragma once

#include "common.cuh"

namespace ffca {

// ------------------------------------------------------------------ layout --
// Reference Spectrogram::f[i] is dim x frames column-major complex<double>,
// i.e. [p][t][m] (re, im).  The kernels read SoA [p][m][t] in the compute type
// so that consecutive threads (frames) touch consecutive addresses.
template <typename R>
__global__ void pack_x_kernel(const double2* __restrict__ in, cplx_t<R>* __restrict__ out, int P,
                              int M, int T) {
  const size_t n = size_t(P) * T;
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
       k += size_t(gridDim.x) * blockDim.x) {
    const size_t p = k / T, t = k - p * T;
    const double2* src = in + k * M;
    cplx_t<R>* dst = out + p * M * T + t;
    for (int m = 0; m < M; ++m) {
      const double2 v = src[m];
      dst[size_t(m) * T] = mkc<R>(R(v.x), R(v.y));
    }
  }
}

// H(n, j) at n + j*N per problem  ->  [p][n][t]
template <typename R>
__global__ void pack_h_kernel(const double* __restrict__ in, R* __restrict__ out, int P, int N,
                              int T) {
  const size_t n = size_t(P) * T;
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
       k += size_t(gridDim.x) * blockDim.x) {
    const size_t p = k / T, t = k - p * T;
    const double* src = in + k * N;
    R* dst = out + p * N * T + t;
    for (int s = 0; s < N; ++s) dst[size_t(s) * T] = R(src[s]);
  }
}

// Inverse of pack_h; problems whose status is not OK keep the staged init.
template <typename R>
__global__ void unpack_h_kernel(const R* __restrict__ in, double* __restrict__ out,
                                const int* __restrict__ status, int P, int N, int T) {
  const size_t n = size_t(P) * T;
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
       k += size_t(gridDim.x) * blockDim.x) {
    const size_t p = k / T, t = k - p * T;
    if (status[p] != 0) continue;
    const R* src = in + p * N * T + t;
    double* dst = out + k * N;
    for (int s = 0; s < N; ++s) dst[s] = double(src[size_t(s) * T]);
  }
}

// SampleCovSet::power_scale (sigmodel.cpp:43-44) from the AoS double input:
// sum_j tr(x_j x_j^H) / (T * M), one CTA per problem, fixed-order reduction.
__global__ void power_aos_kernel(const double2* __restrict__ x, double* __restrict__ out, int M,
                                 int T) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  const double2* xp = x + size_t(p) * T * M;
  double s = 0.0;
  for (int k = threadIdx.x; k < T * M; k += blockDim.x) s += cabs2(xp[k]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    out[p] = tot / (double(T) * M);
  }
}

template <typename R>
__global__ void power_soa_kernel(const cplx_t<R>* __restrict__ x, double* __restrict__ out, int M,
                                 int T) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  const cplx_t<R>* xp = x + size_t(p) * T * M;
  double s = 0.0;
  for (int k = threadIdx.x; k < T * M; k += blockDim.x) s += double(cabs2(xp[k]));
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    out[p] = tot / (double(T) * M);
  }
}

// ------------------------------------------------------------ separation --
// fastfca_separate (fastfca.cpp:205-223): y = W^H x; per source
// g_n = L_n H_n / floor_positive(L H) (source_gain :74-78, sigmodel.cpp:10-15,
// no eps); c_n = (W^H)^{-1} (g_n .* y).  One CTA per problem.
//   out_aos: images[n][p][t][m] complex<double> (reference layout), or
//   out_soa: images[n][p][m][t] in the compute type (device path).
template <int M, typename R>
__global__ void __launch_bounds__(256) separate_kernel(const cplx_t<R>* __restrict__ x,
                                                       const double2* __restrict__ W,
                                                       const double* __restrict__ L,
                                                       const R* __restrict__ H, int P, int N,
                                                       int T, double2* __restrict__ out_aos,
                                                       cplx_t<R>* __restrict__ out_soa) {
  using C = cplx_t<R>;
  __shared__ C wr[M * M];
  __shared__ C ainv[M * M];
  __shared__ R lr[M * 16];
  __shared__ double red[32];
  __shared__ R floor_s;
  const int p = blockIdx.x, tid = threadIdx.x;
  const C* xp = x + size_t(p) * M * T;
  const R* hp = H + size_t(p) * N * T;
  for (int k = tid; k < M * N; k += blockDim.x) lr[k] = R(L[size_t(p) * M * N + k]);
  for (int k = tid; k < M * M; k += blockDim.x) {
    const double2 w = W[size_t(p) * M * M + k];
    wr[k] = mkc<R>(R(w.x), R(w.y));
  }
  if (tid == 0) {
    // (W^H)^{-1} in fp64 via Gauss-Jordan with partial pivoting.
    double2 a[M * M], inv[M * M];
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < M; ++c) {
        const double2 w = W[size_t(p) * M * M + c + r * M];  // W(c, r)
        a[r + c * M] = make_double2(w.x, -w.y);               // (W^H)(r, c)
        inv[r + c * M] = make_double2(r == c ? 1.0 : 0.0, 0.0);
      }
    for (int k = 0; k < M; ++k) {
      int piv = k;
      double best = cabs(a[k + k * M]);
      for (int r = k + 1; r < M; ++r) {
        const double v = cabs(a[r + k * M]);
        if (v > best) best = v, piv = r;
      }
      if (piv != k)
        for (int c = 0; c < M; ++c) {
          double2 t = a[k + c * M]; a[k + c * M] = a[piv + c * M]; a[piv + c * M] = t;
          t = inv[k + c * M]; inv[k + c * M] = inv[piv + c * M]; inv[piv + c * M] = t;
        }
      const double2 d = a[k + k * M];
      for (int c = 0; c < M; ++c) {
        a[k + c * M] = cdiv(a[k + c * M], d);
        inv[k + c * M] = cdiv(inv[k + c * M], d);
      }
      for (int r = 0; r < M; ++r) {
        if (r == k) continue;
        const double2 f = a[r + k * M];
        for (int c = 0; c < M; ++c) {
          a[r + c * M] = csub(a[r + c * M], cmul(f, a[k + c * M]));
          inv[r + c * M] = csub(inv[r + c * M], cmul(f, inv[k + c * M]));
        }
      }
    }
    for (int k = 0; k < M * M; ++k) ainv[k] = mkc<R>(R(inv[k].x), R(inv[k].y));
  }
  __syncthreads();
  // floor_positive: rel 1e-12 of the mean of L H over the bin.
  double s = 0.0;
  for (int t = tid; t < T; t += blockDim.x)
    for (int m = 0; m < M; ++m) {
      R lh = R(0);
      for (int n = 0; n < N; ++n) lh += lr[m + n * M] * hp[size_t(n) * T + t];
      s += double(lh);
    }
  s = warp_sum(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    const double mean = tot / (double(M) * T);
    const double fl = mean > 0.0 ? 1e-12 * mean : 1e-300;
    floor_s = narrow_pos<R>(fl);
  }
  __syncthreads();
  const R fl = floor_s;
  for (int t = tid; t < T; t += blockDim.x) {
    C xv[M], y[M];
    R lh[M];
    for (int m = 0; m < M; ++m) xv[m] = xp[size_t(m) * T + t];
    for (int m = 0; m < M; ++m) {
      C acc = mkc<R>(R(0), R(0));
      for (int c = 0; c < M; ++c) acc = cadd(acc, cmulc(wr[c + m * M], xv[c]));
      y[m] = acc;
      R v = R(0);
      for (int n = 0; n < N; ++n) v += lr[m + n * M] * hp[size_t(n) * T + t];
      lh[m] = v > fl ? v : fl;
    }
    for (int n = 0; n < N; ++n) {
      const R hn = hp[size_t(n) * T + t];
      C z[M];
      for (int m = 0; m < M; ++m) {
        const R g = (lr[m + n * M] * hn) / lh[m];
        z[m] = mkc<R>(g * y[m].x, g * y[m].y);
      }
      for (int r = 0; r < M; ++r) {
        C c = mkc<R>(R(0), R(0));
        for (int k = 0; k < M; ++k) c = cadd(c, cmul(ainv[r + k * M], z[k]));
        if (out_aos)
          out_aos[((size_t(n) * P + p) * T + t) * M + r] = make_double2(double(c.x), double(c.y));
        else
          out_soa[((size_t(n) * P + p) * M + r) * T + t] = c;
      }
    }
  }
}

}  // namespace ffca
