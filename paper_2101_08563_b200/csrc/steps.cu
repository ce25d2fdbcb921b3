// steps.cu -- the reference's public per-step functions as single-bin GPU
// launches: weighted_cov (fastfca.cpp:22-34), ip_update_w (:36-72),
// source_gain (:74-78), em_update_lh (:80-99), mm_update_lh (:101-117).
//
// The fit kernels fuse these steps per bin for every iteration; these entry
// points expose each step on its own, as the reference's header does
// (fastfca.hpp:30-53) and its unit tests call them (test_fastfca.cpp:82-228).
// One bin per call, fp64 throughout (the reference's arithmetic), one or a
// few small launches: they are test/diagnostic surface, not the hot path.
// Every reduction runs in a fixed order (thread-strided partials, then a
// fixed tree), so results are reproducible run to run.
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"
#include "serial_math.cuh"

namespace ffca {

namespace {

constexpr int kStepThreads = 256;

// Fixed-order block sum of one double per thread (all threads get the total).
__device__ double block_sum(double v, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // red is reused between calls
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int k = 0; k < kStepThreads / 32; ++k) s += red[k];
  return s;
}

// sigma^2(m, j) = sum_n L(m, n) H(n, j) + eps (fastfca.cpp:45).
__global__ void step_sigma2_kernel(const double* __restrict__ L, const double* __restrict__ H,
                                   int M, int N, int T, double eps, double* __restrict__ sig) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < M * T; k += gridDim.x * blockDim.x) {
    const int m = k % M, j = k / M;
    double s = 0.0;
    for (int n = 0; n < N; ++n) s += L[m + n * M] * H[n + size_t(j) * N];
    sig[m + size_t(j) * M] = s + eps;
  }
}

// Raw weighted sums raw[col][a + c*M] = sum_j X_j(a, c) / sigma^2(row col, j):
// X_j = x_j x_j^H (snapshots [J][M]) or the block covariance (mats
// [J][M*M] col-major).  Grid (M*M entries, ncol).  sig: [J][sig_ld], the row
// of column `col` at offset col*sig_col (sig_ld = 1 for a bare 1 x J row).
__global__ void __launch_bounds__(kStepThreads)
    step_wcov_kernel(const double2* __restrict__ x, int blk, int M, int J,
                     const double* __restrict__ sig, int sig_ld, int sig_col,
                     double2* __restrict__ raw) {
  __shared__ double red[kStepThreads / 32];
  const int e = blockIdx.x, a = e % M, c = e / M, col = blockIdx.y;
  double sr = 0.0, si = 0.0;
  for (int j = threadIdx.x; j < J; j += kStepThreads) {
    const double inv = 1.0 / sig[size_t(j) * sig_ld + col * sig_col];
    double2 v;
    if (blk) {
      v = x[size_t(j) * M * M + e];
    } else {
      const double2 xa = x[size_t(j) * M + a], xc = x[size_t(j) * M + c];
      v = make_double2(xa.x * xc.x + xa.y * xc.y, xa.y * xc.x - xa.x * xc.y);  // x_a conj(x_c)
    }
    sr += v.x * inv;
    si += v.y * inv;
  }
  sr = block_sum(sr, red);
  si = block_sum(si, red);
  if (threadIdx.x == 0) raw[size_t(col) * M * M + e] = make_double2(sr, si);
}

// symmetrize(q / blocks) (fastfca.cpp:33, hermitian.hpp:31-34): either the
// col-major Hermitian matrix (qout) or the IP's packed raw layout (qpack:
// [a*M+a] diagonal, [a*M+c] Re and [c*M+a] Im of entry (a, c), a < c;
// un-normalised sums, the IP applies 1/blocks).
__global__ void step_wcov_finish_kernel(const double2* __restrict__ raw, int M, int ncol,
                                        double inv_blocks, double2* __restrict__ qout,
                                        double* __restrict__ qpack) {
  for (int k = threadIdx.x; k < ncol * M * M; k += blockDim.x) {
    const int col = k / (M * M), e = k % (M * M), a = e % M, c = e / M;
    const double2 u = raw[size_t(col) * M * M + a + c * M], v = raw[size_t(col) * M * M + c + a * M];
    const double re = 0.5 * (u.x + v.x), im = 0.5 * (u.y - v.y);  // (q + q^H)/2
    if (qout) qout[k] = make_double2(re * inv_blocks, im * inv_blocks);
    if (qpack) {
      double* p = qpack + size_t(col) * M * M;
      if (a == c) p[a * M + a] = re;
      else if (a < c) p[a * M + c] = re, p[c * M + a] = im;
    }
  }
}

// The reference's column sweep with its residual test and seeded restart
// (serial_math.cuh ip_update_gen in fp64), one thread.
template <int M>
__global__ void step_ip_kernel(double2* w, const double* qpack, double inv_blocks,
                               unsigned long long seed, int bin, RestartRng* rng, int* status) {
  if (threadIdx.x != 0) return;
  int bad = -1;
  const bool ok = ip_update_f64<M>(w, qpack, inv_blocks, seed, bin, rng, bad);
  *status = ok ? kStatusOk : (kStatusIpSingular | (bad << 8));
}

// Diagnostics: the restart generator's streams (common.cuh Mt19937_64 /
// PolarNormal seeded with mix_seed(seed, bin), fastfca.cpp:40-41) -- n raw
// 64-bit draws, and n normal draws from a freshly seeded copy.
__global__ void debug_rng_kernel(unsigned long long seed, int bin, int n, RestartRng* rr,
                                 unsigned long long* raw, double* normals) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  rr->mt.seed(mix_seed(seed, bin));
  for (int k = 0; k < n; ++k) raw[k] = rr->mt.next();
  rr->mt.seed(mix_seed(seed, bin));
  rr->gauss.saved = 0.0;
  rr->gauss.has_saved = false;
  for (int k = 0; k < n; ++k) normals[k] = rr->gauss(rr->mt);
}

// log_abs_det2 (sigmodel.cpp:118-129): LU with partial pivoting, one thread.
template <int M>
__global__ void step_logdet_kernel(const double2* w, double* out, int* status) {
  if (threadIdx.x != 0) return;
  double v = 0.0;
  const bool ok = log_abs_det2<M, double>(w, v);
  *out = v;
  *status = ok ? kStatusOk : kStatusSingularW;
}

// source_gain (fastfca.cpp:74-78): G = L_n H_n / floor_positive(L H).
__global__ void __launch_bounds__(kStepThreads)
    step_gain_kernel(const double* __restrict__ L, const double* __restrict__ H, int M, int N,
                     int T, int n, double floor_rel, double* __restrict__ G) {
  __shared__ double red[kStepThreads / 32];
  double acc = 0.0;
  for (int k = threadIdx.x; k < M * T; k += kStepThreads) {
    const int m = k % M, j = k / M;
    double s = 0.0;
    for (int q = 0; q < N; ++q) s += L[m + q * M] * H[q + size_t(j) * N];
    G[k] = s;  // L H, floored below
    acc += s;
  }
  const double mean = block_sum(acc, red) / (double(M) * double(T));
  const double floor = mean > 0.0 ? floor_rel * mean : 1e-300;  // sigmodel.cpp:10-15
  for (int k = threadIdx.x; k < M * T; k += kStepThreads) {
    const int m = k % M, j = k / M;
    G[k] = (L[m + n * M] * H[n + size_t(j) * N]) / fmax(G[k], floor);
  }
}

// em_update_lh (fastfca.cpp:80-99): per source, sequentially, with the
// running factors.  One CTA; phi is staged in global scratch [T][M].
__global__ void __launch_bounds__(kStepThreads)
    step_em_kernel(const double* __restrict__ U, double* L, double* H, int M, int N, int T,
                   int update_loading, double eps, double* phi) {
  __shared__ double red[kStepThreads / 32];
  extern __shared__ double ls[];  // L (M*N), running
  for (int k = threadIdx.x; k < M * N; k += kStepThreads) ls[k] = L[k];
  __syncthreads();
  for (int n = 0; n < N; ++n) {
    for (int k = threadIdx.x; k < M * T; k += kStepThreads) {
      const int m = k % M, j = k / M;
      double lh = 0.0;
      for (int q = 0; q < N; ++q) lh += ls[m + q * M] * H[q + size_t(j) * N];
      lh += eps;
      const double lnhn = ls[m + n * M] * H[n + size_t(j) * N];
      const double g = lnhn / lh;
      phi[k] = g * g * U[k] + (1.0 - g) * lnhn;
    }
    __syncthreads();
    if (update_loading) {
      for (int m = 0; m < M; ++m) {
        double acc = 0.0;
        for (int j = threadIdx.x; j < T; j += kStepThreads)
          acc += phi[m + size_t(j) * M] / H[n + size_t(j) * N];
        const double tot = block_sum(acc, red);
        if (threadIdx.x == 0) ls[m + n * M] = fmax(tot / double(T), 1e-300);
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < T; j += kStepThreads) {
      double s = 0.0;
      for (int m = 0; m < M; ++m) s += phi[m + size_t(j) * M] / ls[m + n * M];
      H[n + size_t(j) * N] = fmax(s / double(M), 1e-300);
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < M * N; k += kStepThreads) L[k] = ls[k];
}

// mm_update_lh (fastfca.cpp:101-117): whole-matrix multiplicative steps, L
// first.  One CTA.
__global__ void __launch_bounds__(kStepThreads)
    step_mm_kernel(const double* __restrict__ U, double* L, double* H, int M, int N, int T,
                   int update_loading, double eps) {
  __shared__ double red[kStepThreads / 32];
  extern __shared__ double ls[];  // L (M*N), then num/den scratch (2*M*N)
  double* num = ls + M * N;
  double* den = num + M * N;
  for (int k = threadIdx.x; k < M * N; k += kStepThreads) ls[k] = L[k];
  __syncthreads();
  if (update_loading) {
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double an = 0.0, ad = 0.0;
        for (int j = threadIdx.x; j < T; j += kStepThreads) {
          double lh = 0.0;
          for (int q = 0; q < N; ++q) lh += ls[m + q * M] * H[q + size_t(j) * N];
          lh += eps;
          const double h = H[n + size_t(j) * N];
          an += U[m + size_t(j) * M] / (lh * lh) * h;
          ad += h / lh;
        }
        an = block_sum(an, red);
        ad = block_sum(ad, red);
        if (threadIdx.x == 0) num[m + n * M] = an, den[m + n * M] = fmax(ad, 1e-300);
      }
    __syncthreads();
    for (int k = threadIdx.x; k < M * N; k += kStepThreads)
      ls[k] = fmax(ls[k] * sqrt(num[k] / den[k]), 1e-300);
    __syncthreads();
  }
  for (int j = threadIdx.x; j < T; j += kStepThreads) {
    double hn[64];  // new column (N <= 64 checked on the host)
    for (int n = 0; n < N; ++n) {
      double an = 0.0, ad = 0.0;
      for (int m = 0; m < M; ++m) {
        double lh = 0.0;
        for (int q = 0; q < N; ++q) lh += ls[m + q * M] * H[q + size_t(j) * N];
        lh += eps;
        an += ls[m + n * M] * (U[m + size_t(j) * M] / (lh * lh));
        ad += ls[m + n * M] / lh;
      }
      ad = fmax(ad, 1e-300);
      hn[n] = fmax(H[n + size_t(j) * N] * sqrt(an / ad), 1e-300);
    }
    for (int n = 0; n < N; ++n) H[n + size_t(j) * N] = hn[n];
  }
  for (int k = threadIdx.x; k < M * N; k += kStepThreads) L[k] = ls[k];
}

// ---- small dense helpers for the diagnostics below (one thread, fp64) ----
constexpr int kMaxDim = 8;

// Solve A X = B in place (B <- X) by Gauss-Jordan with partial pivoting
// (largest modulus, lowest row on ties -- Eigen::PartialPivLU's choice).
// A, B: M x M column-major.  Returns false on a zero / non-finite pivot.
__device__ bool gj_solve(double2* A, double2* B, int M) {
  for (int k = 0; k < M; ++k) {
    int piv = k;
    double best = cabs2(A[k + k * M]);
    for (int r = k + 1; r < M; ++r) {
      const double v = cabs2(A[r + k * M]);
      if (v > best) best = v, piv = r;
    }
    if (!(best > 0.0) || !isfinite(best)) return false;
    if (piv != k)
      for (int c = 0; c < M; ++c) {
        double2 t = A[k + c * M]; A[k + c * M] = A[piv + c * M]; A[piv + c * M] = t;
        t = B[k + c * M]; B[k + c * M] = B[piv + c * M]; B[piv + c * M] = t;
      }
    const double2 d = A[k + k * M];
    for (int c = 0; c < M; ++c) {
      A[k + c * M] = cdiv(A[k + c * M], d);
      B[k + c * M] = cdiv(B[k + c * M], d);
    }
    for (int r = 0; r < M; ++r) {
      if (r == k) continue;
      const double2 f = A[r + k * M];
      for (int c = 0; c < M; ++c) {
        A[r + c * M] = csub(A[r + c * M], cmul(f, A[k + c * M]));
        B[r + c * M] = csub(B[r + c * M], cmul(f, B[k + c * M]));
      }
    }
  }
  return true;
}

// fastfca_mwf (fastfca.cpp:193-203): W^-H diag(gains) W^H at one (i, j, n).
__global__ void step_mwf_kernel(const double2* W, const double* L, const double* hcol, int M, int N,
                                int n, double2* out, int* status) {
  if (threadIdx.x != 0) return;
  double2 a[kMaxDim * kMaxDim], b[kMaxDim * kMaxDim];
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) {
      const double2 w = W[c + r * M];
      a[r + c * M] = make_double2(w.x, -w.y);  // a = W^H
    }
  for (int k = 0; k < M; ++k) {
    double mix = 0.0;
    for (int q = 0; q < N; ++q) mix += L[k + q * M] * hcol[q];
    mix = fmax(mix, 1e-300);
    const double g = L[k + n * M] * hcol[n] / mix;
    for (int c = 0; c < M; ++c) b[k + c * M] = make_double2(g * a[k + c * M].x, g * a[k + c * M].y);
  }
  const bool ok = gj_solve(a, b, M);
  for (int k = 0; k < M * M; ++k) out[k] = b[k];
  *status = ok ? kStatusOk : kStatusSingularW;
}

// reconstruct_scms (fastfca.cpp:270-282): R_in = W^-H Lambda_n W^-1, one
// thread per bin.
__global__ void step_scms_kernel(const double2* W, const double* L, int P, int M, int N,
                                 double2* out, int* status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double2 a[kMaxDim * kMaxDim], winv[kMaxDim * kMaxDim];
  for (int k = 0; k < M * M; ++k) {
    a[k] = W[size_t(p) * M * M + k];
    winv[k] = make_double2((k % M) == (k / M) ? 1.0 : 0.0, 0.0);
  }
  const bool ok = gj_solve(a, winv, M);
  if (!ok) atomicMax(status, kStatusSingularW);
  for (int n = 0; n < N; ++n)
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < M; ++c) {
        double2 acc = make_double2(0.0, 0.0);  // sum_k conj(winv(k, r)) lam_k winv(k, c)
        for (int k = 0; k < M; ++k) {
          const double lam = L[size_t(p) * M * N + k + n * M];
          const double2 u = winv[k + r * M], v = winv[k + c * M];
          acc.x += lam * (u.x * v.x + u.y * v.y);
          acc.y += lam * (u.x * v.y - u.y * v.x);
        }
        out[(size_t(p) * N + n) * M * M + r + c * M] = acc;
      }
}

// ajd_cost terms (fastfca.cpp:225-239, hermitian.hpp:85-102): per block j,
// t = W^H X_j W and D_LD(t | ddiag(t)) = max(0, sum_k log Re t_kk - logdet
// sym(t)) (tr(ddiag(t)^-1 t) = M exactly); Cholesky decides positive
// definiteness.  One thread per block; the weighted sum runs in block order on
// the host side of the ABI call.
__global__ void step_ajd_kernel(const double2* X, const double2* W, int M, int J, double* terms,
                                int* status) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  double2 xw[kMaxDim * kMaxDim], t[kMaxDim * kMaxDim];
  const double2* Xj = X + size_t(j) * M * M;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) {
      double2 acc = make_double2(0.0, 0.0);
      for (int k = 0; k < M; ++k) acc = cadd(acc, cmul(Xj[r + k * M], W[k + c * M]));
      xw[r + c * M] = acc;
    }
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) {
      double2 acc = make_double2(0.0, 0.0);
      for (int k = 0; k < M; ++k) acc = cadd(acc, cmulc(W[k + r * M], xw[k + c * M]));
      t[r + c * M] = acc;
    }
  // symmetrize, then Cholesky (lower), logdet = 2 sum log l_kk
  double2 s[kMaxDim * kMaxDim];
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c)
      s[r + c * M] = make_double2(0.5 * (t[r + c * M].x + t[c + r * M].x),
                                  0.5 * (t[r + c * M].y - t[c + r * M].y));
  bool pd = true;
  double logdet_a = 0.0, logdet_b = 0.0;
  for (int k = 0; k < M && pd; ++k) {
    double d = s[k + k * M].x;
    for (int q = 0; q < k; ++q) d -= cabs2(s[k + q * M]);
    if (!(d > 0.0) || !isfinite(d)) { pd = false; break; }
    const double l = sqrt(d);
    s[k + k * M] = make_double2(l, 0.0);
    logdet_a += 2.0 * log(l);
    for (int r = k + 1; r < M; ++r) {
      double2 v = s[r + k * M];
      for (int q = 0; q < k; ++q) v = csub(v, cmul(s[r + q * M], make_double2(s[k + q * M].x, -s[k + q * M].y)));
      s[r + k * M] = make_double2(v.x / l, v.y / l);
    }
    const double dk = t[k + k * M].x;
    if (!(dk > 0.0) || !isfinite(dk)) { pd = false; break; }
    logdet_b += log(dk);
  }
  if (!pd) {
    atomicMax(status, 1);
    terms[j] = 0.0;
    return;
  }
  terms[j] = fmax(0.0, logdet_b - logdet_a);
}

struct DevBuf {  // call-scoped device memory (these entry points are not hot)
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes < 256 ? 256 : bytes); }
  template <typename T>
  T* as() { return static_cast<T*>(p); }
};

struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

int check_step_dims(const char* fn, int M, int N, int T) {
  if (M < 1 || N < 1 || T < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": empty shape");
  if (M > 64 || N > 64)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": dim/sources above 64");
  return FFCA_OK;
}

// Launch the raw-sum + finish kernels for ncol weight rows.
int run_wcov(ffca_ctx* ctx, cudaStream_t st, const double2* dx, int blk, int M, int J,
             const double* dsig, int sig_ld, int sig_col, int ncol, double2* draw,
             double2* dq, double* dpack) {
  step_wcov_kernel<<<dim3(M * M, ncol), kStepThreads, 0, st>>>(dx, blk, M, J, dsig, sig_ld,
                                                               sig_col, draw);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  step_wcov_finish_kernel<<<1, 256, 0, st>>>(draw, M, ncol, 1.0 / double(J), dq, dpack);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

template <int M>
void launch_ip(cudaStream_t st, double2* w, const double* qpack, double invb,
               unsigned long long seed, int bin, RestartRng* rng, int* status) {
  step_ip_kernel<M><<<1, 32, 0, st>>>(w, qpack, invb, seed, bin, rng, status);
}

}  // namespace

}  // namespace ffca

using namespace ffca;

extern "C" {

int ffca_weighted_cov(ffca_ctx* ctx, int dim, int blocks, int is_block_covs, const double* x,
                      const double* sigma2_row, double* q) {
  if (!ctx || !x || !sigma2_row || !q)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_weighted_cov: null argument");
  if (int rc = check_step_dims("ffca_weighted_cov", dim, 1, blocks)) return rc;
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const int M = dim, J = blocks;
  const size_t nx = size_t(J) * (is_block_covs ? M * M : M);
  DevBuf dx, ds, draw, dq;
  if (dx.alloc(nx * 16) || ds.alloc(size_t(J) * 8) || draw.alloc(size_t(M) * M * 16) ||
      dq.alloc(size_t(M) * M * 16))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_weighted_cov: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dx.p, x, nx * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(ds.p, sigma2_row, size_t(J) * 8, cudaMemcpyHostToDevice, st));
  if (int rc = run_wcov(ctx, st, dx.as<double2>(), is_block_covs, M, J, ds.as<double>(), 1, 0, 1,
                        draw.as<double2>(), dq.as<double2>(), nullptr))
    return rc;
  FFCA_CUDA(cudaMemcpyAsync(q, dq.p, size_t(M) * M * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_ip_update_w(ffca_ctx* ctx, int dim, int sources, int blocks, int is_block_covs,
                     const double* x, double power, double* w, const double* loading,
                     const double* act, uint64_t restart_seed, int bin_index) {
  if (!ctx || !x || !w || !loading || !act)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_ip_update_w: null argument");
  if (int rc = check_step_dims("ffca_ip_update_w", dim, sources, blocks)) return rc;
  if (dim > 8) return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_ip_update_w: dim above 8");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const int M = dim, N = sources, J = blocks;
  const size_t nx = size_t(J) * (is_block_covs ? M * M : M);
  DevBuf dx, dl, dh, dsig, draw, dpack, dw, drng, dstat;
  if (dx.alloc(nx * 16) || dl.alloc(size_t(M) * N * 8) || dh.alloc(size_t(N) * J * 8) ||
      dsig.alloc(size_t(M) * J * 8) || draw.alloc(size_t(M) * M * M * 16) ||
      dpack.alloc(size_t(M) * M * M * 8) || dw.alloc(size_t(M) * M * 16) ||
      drng.alloc(sizeof(RestartRng)) || dstat.alloc(4))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_ip_update_w: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dx.p, x, nx * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dl.p, loading, size_t(M) * N * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dh.p, act, size_t(N) * J * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dw.p, w, size_t(M) * M * 16, cudaMemcpyHostToDevice, st));
  const double eps = power * 1e-8 > 1e-300 ? power * 1e-8 : 1e-300;  // var_eps, sigmodel.hpp:29-31
  step_sigma2_kernel<<<64, 256, 0, st>>>(dl.as<double>(), dh.as<double>(), M, N, J, eps,
                                         dsig.as<double>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  // Q_col for every column: sigma^2 is fixed before the sweep (fastfca.cpp:45).
  if (int rc = run_wcov(ctx, st, dx.as<double2>(), is_block_covs, M, J, dsig.as<double>(), M, 1, M,
                        draw.as<double2>(), nullptr, dpack.as<double>()))
    return rc;
  const double invb = 1.0 / double(J);
  auto* W = dw.as<double2>();
  auto* Q = dpack.as<double>();
  auto* R = drng.as<RestartRng>();
  int* S = dstat.as<int>();
  switch (M) {
    case 1: launch_ip<1>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    case 2: launch_ip<2>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    case 3: launch_ip<3>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    case 4: launch_ip<4>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    case 5: launch_ip<5>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    case 6: launch_ip<6>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    case 7: launch_ip<7>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
    default: launch_ip<8>(st, W, Q, invb, restart_seed, bin_index, R, S); break;
  }
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  int status = 0;
  FFCA_CUDA(cudaMemcpyAsync(&status, S, 4, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  if ((status & 0xff) == kStatusIpSingular)
    return ffca_set_err(FFCA_NUMERICAL, "ip_update_w: singular system for column " +
                                            std::to_string(status >> 8));
  FFCA_CUDA(cudaMemcpyAsync(w, dw.p, size_t(M) * M * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_debug_restart_draws(ffca_ctx* ctx, uint64_t seed, int bin_index, int n,
                             uint64_t* mixed_seed, uint64_t* raw, double* normals) {
  if (!ctx || !raw || !normals || n < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_debug_restart_draws: bad argument");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  DevBuf drng, draw, dn;
  if (drng.alloc(sizeof(RestartRng)) || draw.alloc(size_t(n) * 8) || dn.alloc(size_t(n) * 8))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_debug_restart_draws: device alloc failed");
  debug_rng_kernel<<<1, 32, 0, st>>>(seed, bin_index, n, drng.as<RestartRng>(),
                                     draw.as<unsigned long long>(), dn.as<double>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  FFCA_CUDA(cudaMemcpyAsync(raw, draw.p, size_t(n) * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaMemcpyAsync(normals, dn.p, size_t(n) * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  if (mixed_seed) *mixed_seed = mix_seed(seed, bin_index);
  return FFCA_OK;
}

int ffca_log_abs_det2(ffca_ctx* ctx, int dim, const double* w, double* out) {
  if (!ctx || !w || !out)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_log_abs_det2: null argument");
  if (dim < 1 || dim > 8)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_log_abs_det2: dim outside 1..8");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  DevBuf dw, dout, dstat;
  if (dw.alloc(size_t(dim) * dim * 16) || dout.alloc(8) || dstat.alloc(4))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_log_abs_det2: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dw.p, w, size_t(dim) * dim * 16, cudaMemcpyHostToDevice, st));
  auto* W = dw.as<double2>();
  double* O = dout.as<double>();
  int* S = dstat.as<int>();
  switch (dim) {
    case 1: step_logdet_kernel<1><<<1, 32, 0, st>>>(W, O, S); break;
    case 2: step_logdet_kernel<2><<<1, 32, 0, st>>>(W, O, S); break;
    case 3: step_logdet_kernel<3><<<1, 32, 0, st>>>(W, O, S); break;
    case 4: step_logdet_kernel<4><<<1, 32, 0, st>>>(W, O, S); break;
    case 5: step_logdet_kernel<5><<<1, 32, 0, st>>>(W, O, S); break;
    case 6: step_logdet_kernel<6><<<1, 32, 0, st>>>(W, O, S); break;
    case 7: step_logdet_kernel<7><<<1, 32, 0, st>>>(W, O, S); break;
    default: step_logdet_kernel<8><<<1, 32, 0, st>>>(W, O, S); break;
  }
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  int status = 0;
  FFCA_CUDA(cudaMemcpyAsync(&status, S, 4, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaMemcpyAsync(out, O, 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  if (status == kStatusSingularW) return ffca_set_err(FFCA_NUMERICAL, "singular decorrelation matrix");
  return FFCA_OK;
}

int ffca_mwf(ffca_ctx* ctx, int dim, int sources, const double* w, const double* loading,
             const double* act_col, int n, double* out) {
  if (!ctx || !w || !loading || !act_col || !out)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_mwf: null argument");
  if (dim < 1 || dim > kMaxDim || sources < 1 || n < 0 || n >= sources)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_mwf: bad shape or source index");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const int M = dim, N = sources;
  DevBuf dw, dl, dh, dout, dstat;
  if (dw.alloc(size_t(M) * M * 16) || dl.alloc(size_t(M) * N * 8) || dh.alloc(size_t(N) * 8) ||
      dout.alloc(size_t(M) * M * 16) || dstat.alloc(4))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_mwf: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dw.p, w, size_t(M) * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dl.p, loading, size_t(M) * N * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dh.p, act_col, size_t(N) * 8, cudaMemcpyHostToDevice, st));
  step_mwf_kernel<<<1, 32, 0, st>>>(dw.as<double2>(), dl.as<double>(), dh.as<double>(), M, N, n,
                                    dout.as<double2>(), dstat.as<int>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  int status = 0;
  FFCA_CUDA(cudaMemcpyAsync(&status, dstat.p, 4, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaMemcpyAsync(out, dout.p, size_t(M) * M * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  if (status != kStatusOk) return ffca_set_err(FFCA_NUMERICAL, "fastfca_mwf: singular decorrelation matrix");
  return FFCA_OK;
}

int ffca_reconstruct_scms(ffca_ctx* ctx, int bins, int dim, int sources, const double* W,
                          const double* L, double* out) {
  if (!ctx || !W || !L || !out)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_reconstruct_scms: null argument");
  if (bins < 1 || dim < 1 || dim > kMaxDim || sources < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_reconstruct_scms: bad shape");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t M = dim, N = sources, P = bins;
  DevBuf dw, dl, dout, dstat;
  if (dw.alloc(P * M * M * 16) || dl.alloc(P * M * N * 8) || dout.alloc(P * N * M * M * 16) ||
      dstat.alloc(4))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_reconstruct_scms: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dw.p, W, P * M * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dl.p, L, P * M * N * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemsetAsync(dstat.p, 0, 4, st));
  step_scms_kernel<<<(bins + 63) / 64, 64, 0, st>>>(dw.as<double2>(), dl.as<double>(), bins, dim,
                                                     sources, dout.as<double2>(), dstat.as<int>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  int status = 0;
  FFCA_CUDA(cudaMemcpyAsync(&status, dstat.p, 4, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaMemcpyAsync(out, dout.p, P * N * M * M * 16, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  if (status != kStatusOk)
    return ffca_set_err(FFCA_NUMERICAL, "reconstruct_scms: singular decorrelation matrix");
  return FFCA_OK;
}

int ffca_ajd_cost(ffca_ctx* ctx, int dim, int blocks, const double* mats, const double* w,
                  const double* weights, double* out) {
  if (!ctx || !mats || !w || !out)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_ajd_cost: null argument");
  if (dim < 1 || dim > kMaxDim || blocks < 1)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_ajd_cost: bad shape");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t M = dim, J = blocks;
  DevBuf dx, dw, dt, dstat;
  if (dx.alloc(J * M * M * 16) || dw.alloc(M * M * 16) || dt.alloc(J * 8) || dstat.alloc(4))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_ajd_cost: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dx.p, mats, J * M * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dw.p, w, M * M * 16, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemsetAsync(dstat.p, 0, 4, st));
  step_ajd_kernel<<<(blocks + 63) / 64, 64, 0, st>>>(dx.as<double2>(), dw.as<double2>(), dim, blocks,
                                                      dt.as<double>(), dstat.as<int>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  std::vector<double> terms(J);
  int status = 0;
  FFCA_CUDA(cudaMemcpyAsync(&status, dstat.p, 4, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaMemcpyAsync(terms.data(), dt.p, J * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  if (status != 0)
    return ffca_set_err(FFCA_NUMERICAL, "logdet_divergence: argument not positive definite");
  double acc = 0.0;  // block order, as the reference's loop (fastfca.cpp:231-237)
  for (size_t j = 0; j < J; ++j) acc += (weights ? weights[j] : 1.0) * terms[j];
  *out = acc;
  return FFCA_OK;
}

int ffca_source_gain(ffca_ctx* ctx, int dim, int sources, int frames, const double* loading,
                     const double* act, int n, double* gain) {
  if (!ctx || !loading || !act || !gain)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_source_gain: null argument");
  if (int rc = check_step_dims("ffca_source_gain", dim, sources, frames)) return rc;
  if (n < 0 || n >= sources)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca_source_gain: source index out of range");
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const int M = dim, N = sources, T = frames;
  DevBuf dl, dh, dg;
  if (dl.alloc(size_t(M) * N * 8) || dh.alloc(size_t(N) * T * 8) || dg.alloc(size_t(M) * T * 8))
    return ffca_set_err(FFCA_CUDA_ERROR, "ffca_source_gain: device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(dl.p, loading, size_t(M) * N * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dh.p, act, size_t(N) * T * 8, cudaMemcpyHostToDevice, st));
  step_gain_kernel<<<1, kStepThreads, 0, st>>>(dl.as<double>(), dh.as<double>(), M, N, T, n,
                                               1e-12 /* kPowerFloorRel */, dg.as<double>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  FFCA_CUDA(cudaMemcpyAsync(gain, dg.p, size_t(M) * T * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

static int lh_update(ffca_ctx* ctx, const char* fn, bool mm, int dim, int sources, int frames,
                     const double* u, double* loading, double* act, int update_loading,
                     double eps) {
  if (!ctx || !u || !loading || !act)
    return ffca_set_err(FFCA_INVALID_ARGUMENT, std::string(fn) + ": null argument");
  if (int rc = check_step_dims(fn, dim, sources, frames)) return rc;
  ctx->launches = 0;
  DeviceScope g(ctx->device);
  cudaStream_t st = ctx->stream;
  const int M = dim, N = sources, T = frames;
  DevBuf du, dl, dh, dphi;
  if (du.alloc(size_t(M) * T * 8) || dl.alloc(size_t(M) * N * 8) || dh.alloc(size_t(N) * T * 8) ||
      dphi.alloc(size_t(M) * T * 8))
    return ffca_set_err(FFCA_CUDA_ERROR, std::string(fn) + ": device alloc failed");
  FFCA_CUDA(cudaMemcpyAsync(du.p, u, size_t(M) * T * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dl.p, loading, size_t(M) * N * 8, cudaMemcpyHostToDevice, st));
  FFCA_CUDA(cudaMemcpyAsync(dh.p, act, size_t(N) * T * 8, cudaMemcpyHostToDevice, st));
  if (mm)
    step_mm_kernel<<<1, kStepThreads, size_t(3) * M * N * 8, st>>>(
        du.as<double>(), dl.as<double>(), dh.as<double>(), M, N, T, update_loading, eps);
  else
    step_em_kernel<<<1, kStepThreads, size_t(M) * N * 8, st>>>(
        du.as<double>(), dl.as<double>(), dh.as<double>(), M, N, T, update_loading, eps,
        dphi.as<double>());
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  FFCA_CUDA(cudaMemcpyAsync(loading, dl.p, size_t(M) * N * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaMemcpyAsync(act, dh.p, size_t(N) * T * 8, cudaMemcpyDeviceToHost, st));
  FFCA_CUDA(cudaStreamSynchronize(st));
  return FFCA_OK;
}

int ffca_em_update_lh(ffca_ctx* ctx, int dim, int sources, int frames, const double* u,
                      double* loading, double* act, int update_loading, double eps) {
  return lh_update(ctx, "ffca_em_update_lh", false, dim, sources, frames, u, loading, act,
                   update_loading, eps);
}

int ffca_mm_update_lh(ffca_ctx* ctx, int dim, int sources, int frames, const double* u,
                      double* loading, double* act, int update_loading, double eps) {
  return lh_update(ctx, "ffca_mm_update_lh", true, dim, sources, frames, u, loading, act,
                   update_loading, eps);
}

}  // extern "C"
