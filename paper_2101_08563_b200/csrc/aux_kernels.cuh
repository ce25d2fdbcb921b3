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

// The host fit's per-chunk staging in one launch: x (fp64 -> compute type,
// skipped when R is double), H (fp64 -> compute type) and, when power is
// non-null, power_scale exactly as power_kernel computes it (same loop and
// reduction order, so the same bits).  One CTA of 256 threads per problem.
template <typename R>
__global__ void __launch_bounds__(256) stage_kernel(const double2* __restrict__ x,
                                                    cplx_t<R>* __restrict__ xs,
                                                    const double* __restrict__ h,
                                                    R* __restrict__ hs, double* __restrict__ power,
                                                    int M, int N, int T) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  const double2* xp = x + size_t(p) * T * M;
  cplx_t<R>* xo = xs + size_t(p) * T * M;
  double s = 0.0;
  for (int k = threadIdx.x; k < T * M; k += blockDim.x) {
    const double2 v = xp[k];
    if (sizeof(R) != 8) xo[k] = mkc<R>(R(v.x), R(v.y));
    s += cabs2(v);
  }
  const double* hp = h + size_t(p) * T * N;
  R* ho = hs + size_t(p) * T * N;
  for (int k = threadIdx.x; k < T * N; k += blockDim.x) ho[k] = R(hp[k]);
  if (!power) return;
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    power[p] = tot / (double(T) * M);
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

// ------------------------------------------------- block-stationary input --
// Packed Hermitian record of an M x M covariance (the fit kernel's BLK record):
// [a*M+a] = X_aa, [a*M+c] = Re X_ac, [c*M+a] = Im X_ac for a < c.  A user's
// matrix that is not exactly Hermitian is symmetrised, (X + X^H)/2, which is
// what weighted_cov's symmetrize (fastfca.cpp:33) and the real part in
// decorrelated_powers (sigmodel.cpp:103) see of it.

// sample_covs with block_size B (sigmodel.cpp:17-48): block jb of problem p
// averages x x^H over frames [jb*B, jb*B + width), width = min(B, T - jb*B)
// (:37-40), in fp64.  Writes the packed records (rec, compute type R; may be
// null), the full complex128 col-major matrices (mats [p][jb][M*M], may be
// null) and power_scale = sum_jb tr / (J M) (:43-44; may be null).  One CTA
// per problem, one thread per block, fixed-order power reduction.
template <typename Cin, typename R>
__global__ void __launch_bounds__(256) block_covs_kernel(const Cin* __restrict__ x, int M, int T,
                                                         int B, int J, R* __restrict__ rec,
                                                         double2* __restrict__ mats,
                                                         double* __restrict__ power) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  const Cin* xp = x + size_t(p) * T * M;
  double trs = 0.0;
  for (int jb = threadIdx.x; jb < J; jb += blockDim.x) {
    const int j0 = jb * B, width = min(B, T - j0);
    double2 acc[36];  // upper triangle incl. diagonal, M <= 8
    int k = 0;
    for (int a = 0; a < M; ++a)
      for (int c = a; c < M; ++c) acc[k++] = make_double2(0.0, 0.0);
    for (int j = j0; j < j0 + width; ++j) {
      double2 xv[8];
      for (int m = 0; m < M; ++m) {
        const Cin v = xp[size_t(j) * M + m];
        xv[m] = make_double2(double(v.x), double(v.y));
      }
      k = 0;
      for (int a = 0; a < M; ++a)
        for (int c = a; c < M; ++c, ++k) {  // x_a conj(x_c)
          acc[k].x += xv[a].x * xv[c].x + xv[a].y * xv[c].y;
          acc[k].y += xv[a].y * xv[c].x - xv[a].x * xv[c].y;
        }
    }
    const double iw = 1.0 / double(width);
    k = 0;
    R* rp = rec ? rec + (size_t(p) * J + jb) * M * M : nullptr;
    double2* mp = mats ? mats + (size_t(p) * J + jb) * M * M : nullptr;
    for (int a = 0; a < M; ++a)
      for (int c = a; c < M; ++c, ++k) {
        const double re = acc[k].x * iw, im = (a == c) ? 0.0 : acc[k].y * iw;
        if (a == c) trs += re;
        if (rp) {
          rp[a * M + c] = R(re);
          if (c != a) rp[c * M + a] = R(im);
        }
        if (mp) {
          mp[a + c * M] = make_double2(re, im);
          mp[c + a * M] = make_double2(re, -im);
        }
      }
  }
  if (!power) return;
  trs = warp_sum(trs);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = trs;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    power[p] = tot / (double(J) * M);
  }
}

// Caller-supplied block covariances (SampleCovSet::mats, complex128 col-major
// [p][j][M*M]) -> packed records; power (may be null) = SampleCovSet::power()
// without power_scale: sum_j tr / (J M) (sigmodel.cpp:50-55).
template <typename R>
__global__ void __launch_bounds__(256) pack_covs_kernel(const double2* __restrict__ mats, int M,
                                                        int J, R* __restrict__ rec,
                                                        double* __restrict__ power) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  double trs = 0.0;
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    const double2* mp = mats + (size_t(p) * J + j) * M * M;
    R* rp = rec + (size_t(p) * J + j) * M * M;
    for (int a = 0; a < M; ++a) {
      const double d = mp[a + a * M].x;
      trs += d;
      rp[a * M + a] = R(d);
      for (int c = a + 1; c < M; ++c) {
        const double2 u = mp[a + c * M], l = mp[c + a * M];
        rp[a * M + c] = R(0.5 * (u.x + l.x));
        rp[c * M + a] = R(0.5 * (u.y - l.y));
      }
    }
  }
  if (!power) return;
  trs = warp_sum(trs);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = trs;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    power[p] = tot / (double(J) * M);
  }
}

// decorrelated_powers, block branch (sigmodel.cpp:97-105): U(m, j) =
// max(0, Re w_m^H X_j w_m) from packed records, then floor_positive when
// floor_rel >= 0 (ica_mode_fit's H init on block input).  out [p][j][m] fp64.
template <typename R>
__global__ void __launch_bounds__(256) decorrelated_powers_blk_kernel(
    const R* __restrict__ rec, const double2* __restrict__ W, int M, int J, double floor_rel,
    double* __restrict__ out) {
  __shared__ double2 w[64];
  __shared__ double red[32];
  __shared__ double fl;
  const int p = blockIdx.x;
  for (int k = threadIdx.x; k < M * M; k += blockDim.x) w[k] = W[size_t(p) * M * M + k];
  __syncthreads();
  double* op = out + size_t(p) * J * M;
  double s = 0.0;
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    const R* rp = rec + (size_t(p) * J + j) * M * M;
    for (int m = 0; m < M; ++m) {
      double acc = 0.0;
      for (int a = 0; a < M; ++a) {
        const double2 wa = w[a + m * M];
        acc += cabs2(wa) * double(rp[a * M + a]);
        for (int c = a + 1; c < M; ++c) {
          const double2 wc = w[c + m * M];
          acc += 2.0 * ((wa.x * wc.x + wa.y * wc.y) * double(rp[a * M + c]) -
                        (wa.x * wc.y - wa.y * wc.x) * double(rp[c * M + a]));
        }
      }
      const double u = fmax(acc, 0.0);
      op[size_t(j) * M + m] = u;
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
    const double mean = tot / (double(J) * M);
    fl = mean > 0.0 ? floor_rel * mean : 1e-300;
  }
  __syncthreads();
  const double f = fl;
  for (int k = threadIdx.x; k < J * M; k += blockDim.x) op[k] = fmax(op[k], f);
}

}  // namespace ffca
