// aux_kernels.cuh -- boundary precision conversion, per-bin power and the
// decomposed multichannel Wiener filter output kernel.
//
// Device layouts are the reference containers' per-bin order (frame-major):
// x [p][t][m] complex, H [p][t][n] real, images [n][p][t][m] complex.  The
// boundary only converts precision (fp64 host buffers -> fp32 compute path).
#pragma once

#include "common.cuh"

namespace ffca {

// ------------------------------------------------------------ conversion --
template <typename Src, typename Dst>
__global__ void convert_kernel(const Src* __restrict__ in, Dst* __restrict__ out, size_t n) {
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
       k += size_t(gridDim.x) * blockDim.x)
    out[k] = Dst(in[k]);
}

// Compute type -> fp64 for the fitted H; problems whose status is not OK keep
// the staged fp64 init (silent bands return the init bit-exactly).
template <typename R>
__global__ void unpack_h_kernel(const R* __restrict__ in, double* __restrict__ out,
                                const int* __restrict__ status, size_t per_problem, size_t n) {
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
       k += size_t(gridDim.x) * blockDim.x) {
    if (status[k / per_problem] != 0) continue;
    out[k] = double(in[k]);
  }
}

// SampleCovSet::power_scale (sigmodel.cpp:43-44): sum_j tr(x_j x_j^H) / (T M),
// one CTA per problem, fixed-order reduction.
template <typename C>
__global__ void power_kernel(const C* __restrict__ x, double* __restrict__ out, int M, int T) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  const C* xp = x + size_t(p) * T * M;
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

// decorrelated_powers (sigmodel.cpp:93-107, snapshot branch :96) followed by
// floor_positive (sigmodel.cpp:10-15) when floor_rel >= 0: U(m, t) =
// |w_m^H x_t|^2, then U = max(U, rel * mean(U)) (1e-300 if the mean is not
// positive).  One CTA per problem; out is [p][t][m] fp64 (the Eigen
// col-major M x T matrix of each bin).  ica_mode_fit's H init.
template <typename R>
__global__ void __launch_bounds__(256) decorrelated_powers_kernel(
    const cplx_t<R>* __restrict__ x, const double2* __restrict__ W, int M, int T, double floor_rel,
    double* __restrict__ out) {
  using C = cplx_t<R>;
  __shared__ C w[64];
  __shared__ double red[32];
  __shared__ double fl;
  const int p = blockIdx.x;
  for (int k = threadIdx.x; k < M * M; k += blockDim.x) {
    const double2 v = W[size_t(p) * M * M + k];
    w[k] = mkc<R>(R(v.x), R(v.y));
  }
  __syncthreads();
  const C* xp = x + size_t(p) * T * M;
  double* op = out + size_t(p) * T * M;
  double s = 0.0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    C xv[8];
    for (int c = 0; c < M; ++c) xv[c] = xp[size_t(t) * M + c];
    for (int m = 0; m < M; ++m) {
      C y = cmulc(w[m * M], xv[0]);  // conj(W(0, m)) x_0 + ...
      for (int c = 1; c < M; ++c) y = cadd(y, cmulc(w[c + m * M], xv[c]));
      const double u = double(cabs2(y));
      op[size_t(t) * M + m] = u;
      s += u;
    }
  }
  if (floor_rel < 0.0) return;
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int k = 0; k < int(blockDim.x >> 5); ++k) tot += red[k];
    const double mean = tot / (double(T) * M);
    fl = mean > 0.0 ? floor_rel * mean : 1e-300;
  }
  __syncthreads();
  const double f = fl;
  for (int k = threadIdx.x; k < T * M; k += blockDim.x) op[k] = fmax(op[k], f);
}

// ------------------------------------------------------------ separation --
// fastfca_separate (fastfca.cpp:205-223): y = W^H x; per source
// g_n = L_n H_n / floor_positive(L H) (source_gain :74-78, sigmodel.cpp:10-15,
// no eps); c_n = (W^H)^{-1} (g_n .* y).  One CTA per problem; the output is
// the reference layout images[n][p][t][m] in fp64 (host path) or in the
// compute type (device path).
template <int M, typename R, typename OutC>
__global__ void __launch_bounds__(256) separate_kernel(const cplx_t<R>* __restrict__ x,
                                                       const double2* __restrict__ W,
                                                       const double* __restrict__ L,
                                                       const R* __restrict__ H, int P, int N,
                                                       int T, OutC* __restrict__ out) {
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
    // (W^H)^{-1} in fp64 by Gauss-Jordan with partial pivoting.
    double2 a[M * M], inv[M * M];
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < M; ++c) {
        const double2 w = W[size_t(p) * M * M + c + r * M];  // W(c, r)
        a[r + c * M] = make_double2(w.x, -w.y);               // (W^H)(r, c)
        inv[r + c * M] = make_double2(r == c ? 1.0 : 0.0, 0.0);
      }
    for (int k = 0; k < M; ++k) {
      int piv = k;
      double best = cabs2(a[k + k * M]);
      for (int r = k + 1; r < M; ++r) {
        const double v = cabs2(a[r + k * M]);
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
  for (int t = tid; t < T; t += blockDim.x) {
    R ssum = R(0);
    for (int m = 0; m < M; ++m) {
      R lh = R(0);
      for (int n = 0; n < N; ++n) lh += lr[m + n * M] * hp[size_t(t) * N + n];
      ssum += lh;
    }
    s += double(ssum);
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
    R hv[16];
    for (int n = 0; n < N; ++n) hv[n] = hp[size_t(t) * N + n];
#pragma unroll
    for (int m = 0; m < M; ++m) xv[m] = xp[size_t(t) * M + m];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      C acc = mkc<R>(R(0), R(0));
#pragma unroll
      for (int c = 0; c < M; ++c) acc = cadd(acc, cmulc(wr[c + m * M], xv[c]));
      y[m] = acc;
      R v = R(0);
      for (int n = 0; n < N; ++n) v += lr[m + n * M] * hv[n];
      lh[m] = v > fl ? v : fl;
    }
    for (int n = 0; n < N; ++n) {
      C z[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const R g = (lr[m + n * M] * hv[n]) / lh[m];
        z[m] = mkc<R>(g * y[m].x, g * y[m].y);
      }
      OutC* o = out + ((size_t(n) * P + p) * T + t) * M;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        C c = mkc<R>(R(0), R(0));
#pragma unroll
        for (int k = 0; k < M; ++k) c = cadd(c, cmul(ainv[r + k * M], z[k]));
        OutC v;
        v.x = c.x;
        v.y = c.y;
        o[r] = v;
      }
    }
  }
}

}  // namespace ffca
