// fit_kernel.cuh -- the persistent FastFCA IP+EM (and IP+MM) fit kernel.
//
// One CTA owns one frequency problem (bin i of mixture b) for ALL iterations
// of fastfca_fit (reference src/fastfca.cpp:158-184): the CTA grid replaces
// parallel_for over bins (src/parallel.cpp:16-45).  When the per-bin working
// set (x: M*T complex, H: N*T, U: M*T) fits in shared memory the CTA keeps it
// on chip for the whole fit, so HBM sees x and H once; otherwise the same code
// streams them from global memory (L2/HBM) and keeps U in a global scratch.
//
// Per iteration (fastfca.cpp:172-183), with T the frame count:
//   pass A   one sweep over T: balance-pending scales, sigma^2 = L H + eps,
//            the per-bin NLL of the previous iterate (sigmodel.cpp:155-162)
//            and all M weighted covariances Q_m (fastfca.cpp:22-34), reduced
//            once for the whole CTA.
//   IP       one thread, fp64 in registers: M sequential column solves with the
//            residual check and the libstdc++-faithful seeded restart
//            (fastfca.cpp:36-72).
//   EM       N+1 sweeps: sweep n finishes source n-1's H row with the freshly
//            reduced L column and accumulates source n's L reduction
//            (em_update_lh, fastfca.cpp:80-99); sweep 0 also forms U = |W^H x|^2
//            (sigmodel.cpp:93-107).
//   MM       two sweeps (mm_update_lh, fastfca.cpp:101-117).
//   balance  one thread on the reduced row means (fastfca.cpp:127-142); the H
//            row scale is applied lazily by the next sweep that touches H.
// Every reduction is: warp shuffles -> per-warp partials in shared memory ->
// barrier -> warp 0 sums the partials in a fixed order (fp64) -> lane 0 does
// the serial update -> barrier.  The order is fixed for a launch shape, so
// per-bin results do not depend on how bins are sharded over GPUs.
#pragma once

#include "common.cuh"

namespace ffca {

struct FitParams {
  int nprob;        // problems in this launch (= gridDim.x)
  int N, T;         // sources, frames
  int F;            // bins per mixture (restart seed index i = global % F)
  int prob_offset;  // global problem index of blockIdx.x == 0
  const void* x;    // R2 [nprob][M][T]   SoA, t fastest
  void* H;          // R  [nprob][N][T]   in/out
  void* U;          // R  [nprob][M][T]   scratch (streaming mode only)
  double2* W;       // [nprob][M*M] col-major (r + c*M), in/out
  double* L;        // [nprob][M*N] col-major (m + n*M), in/out
  const double* power;  // [nprob] SampleCovSet::power_scale
  double* nll;      // slot(t, p) at nll[t * nll_stride + prob_offset + p]; may be null
  int nll_stride;
  int* status;      // [nprob]: 0 ok, 1 silent band, 2 IP singular, 3 singular W
  int iters, flavor, record, normalize, fix_loadings, resident;
  int nc;           // MM: sources per L-reduction chunk
  unsigned long long seed;
};

enum : int { kStatusOk = 0, kStatusSilent = 1, kStatusIpSingular = 2, kStatusSingularW = 3 };

template <int M>
struct Split {
  // M <= 4: every thread accumulates all M weighted covariances (M^3 values).
  // M  > 4: the CTA splits into M groups of warps, group g owns Q_g (M^2).
  static constexpr int MSPLIT = (M <= 4) ? 1 : M;
  static constexpr int MG = M / MSPLIT;
  static constexpr int KA = MG * M * M + 1;  // pass-A values per thread
};

// Occupancy target: CTAs per SM the register budget must allow (256 threads).
template <int M>
struct Occ {
  static constexpr int value = (M <= 3) ? 4 : (M == 4 ? 2 : 1);
};

// Shared-memory carve-up, identical on host and device.
template <int M, int NT, typename R>
struct FitSmem {
  int off_wd, off_wr, off_ld, off_lr, off_lold, off_linv, off_hs, off_us, off_hsum, off_num,
      off_den, off_red, off_res, off_scal, off_big, kred, kres, total;
  __host__ __device__ static int al(int v) { return (v + 15) & ~15; }
  __host__ __device__ FitSmem(int nwarps, int N, int T, int nc, bool resident) {
    using S = Split<M>;
    kred = S::KA;
    if (M + 1 > kred) kred = M + 1;
    if (2 * M * nc > kred) kred = 2 * M * nc;
    if (NT > kred) kred = NT;
    kres = M * M * M + 1;
    if (kres < kred) kres = kred;
    int o = 0;
    off_wd = o; o = al(o + M * M * 16);
    off_wr = o; o = al(o + M * M * 2 * (int)sizeof(R));
    off_ld = o; o = al(o + M * NT * 8);
    off_lr = o; o = al(o + M * NT * (int)sizeof(R));
    off_lold = o; o = al(o + M * (int)sizeof(R));
    off_linv = o; o = al(o + M * (int)sizeof(R));
    off_hs = o; o = al(o + NT * (int)sizeof(R));
    off_us = o; o = al(o + M * (int)sizeof(R));
    off_hsum = o; o = al(o + NT * 8);
    off_num = o; o = al(o + M * NT * 8);
    off_den = o; o = al(o + M * NT * 8);
    off_red = o;  // also the restart RNG state during the (serial) IP stage
    {
      const int need = nwarps * kred * 8;
      o = al(o + (need > (int)sizeof(Mt19937_64) ? need : (int)sizeof(Mt19937_64)));
    }
    off_res = o; o = al(o + kres * 8);
    off_scal = o; o = al(o + 64);
    off_big = o;
    if (resident) o = al(o + T * (M * 2 * (int)sizeof(R) + N * (int)sizeof(R) + M * (int)sizeof(R)));
    total = o;
  }
};

struct Scalars {
  double eps, logdet, nll0;
  int stop, status;
};

// ------------------------------------------------------------- fp64 algebra --
// Everything below runs in one thread on register arrays (M is a compile-time
// constant, every loop unrolls).  Pivot order follows Eigen::PartialPivLU
// (largest modulus; compared as squared modulus, the same order).
template <int M>
__device__ __forceinline__ void lu_factor(double2 (&a)[M * M], int (&perm)[M]) {
#pragma unroll
  for (int k = 0; k < M; ++k) perm[k] = k;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    int p = k;
    double best = cabs2(a[k + k * M]);
#pragma unroll
    for (int r = k + 1; r < M; ++r) {
      const double v = cabs2(a[r + k * M]);
      if (v > best) best = v, p = r;
    }
    // Swap rows k and p with static indices (p is runtime).
#pragma unroll
    for (int r = k + 1; r < M; ++r) {
      if (r == p) {
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double2 t = a[k + c * M];
          a[k + c * M] = a[r + c * M];
          a[r + c * M] = t;
        }
        const int t = perm[k];
        perm[k] = perm[r];
        perm[r] = t;
      }
    }
    if (best != 0.0) {
      const double2 piv = a[k + k * M];
#pragma unroll
      for (int r = k + 1; r < M; ++r) a[r + k * M] = cdiv(a[r + k * M], piv);
#pragma unroll
      for (int c = k + 1; c < M; ++c)
#pragma unroll
        for (int r = k + 1; r < M; ++r)
          a[r + c * M] = csub(a[r + c * M], cmul(a[r + k * M], a[k + c * M]));
    }
  }
}

// Solve (P^T L U) y = e_col.
template <int M>
__device__ __forceinline__ void lu_solve_unit(const double2 (&lu)[M * M], const int (&perm)[M],
                                              int col, double2 (&y)[M]) {
#pragma unroll
  for (int k = 0; k < M; ++k) y[k] = make_double2(perm[k] == col ? 1.0 : 0.0, 0.0);
#pragma unroll
  for (int k = 0; k < M; ++k)
#pragma unroll
    for (int r = k + 1; r < M; ++r) y[r] = csub(y[r], cmul(lu[r + k * M], y[k]));
#pragma unroll
  for (int k = M - 1; k >= 0; --k) {
    y[k] = cdiv(y[k], lu[k + k * M]);
#pragma unroll
    for (int r = 0; r < k; ++r) y[r] = csub(y[r], cmul(lu[r + k * M], y[k]));
  }
}

// log|det W|^2 (sigmodel.cpp:118-129).  Returns false when W is numerically
// singular (a zero or non-finite U diagonal).
template <int M>
__device__ __forceinline__ bool log_abs_det2(const double2* w, double& out) {
  double2 a[M * M];
  int perm[M];
#pragma unroll
  for (int k = 0; k < M * M; ++k) a[k] = w[k];
  lu_factor<M>(a, perm);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double v = cabs2(a[k + k * M]);
    if (!(v > 0.0) || !isfinite(v)) return false;
    acc += log(v);
  }
  out = acc;  // sum of log|u_kk|^2 = 2 * sum log|u_kk|
  return true;
}

// Cold path of ip_update_w: one seeded perturbation of column `col`
// (fastfca.cpp:66-69).  The generator is seeded lazily on the first restart
// of the sweep and its state lives in shared scratch.
static __device__ __noinline__ void ip_perturb(double2* wcol, int m, Mt19937_64* rng, bool* seeded,
                                        PolarNormal* gauss, unsigned long long seed, int bin) {
  if (!*seeded) {
    rng->seed(mix_seed(seed, bin));
    *seeded = true;
  }
  double cn = 0.0;
  for (int r = 0; r < m; ++r) cn += cabs2(wcol[r]);
  const double mag = 1e-8 * (sqrt(cn) + 1.0);
  for (int r = 0; r < m; ++r) {
    const double im = (*gauss)(*rng);  // g++ evaluates Complex(g(), g()) right to left
    const double re = (*gauss)(*rng);
    wcol[r].x += mag * re;
    wcol[r].y += mag * im;
  }
}

// ip_update_w (fastfca.cpp:36-72) on the reduced weighted covariances.
// qraw[m*M*M + ...] holds sum_t x x^H / sigma2_m packed as: (a,a) real,
// (a,b) a<b real part at a*M+b and imaginary part at b*M+a.
template <int M>
__device__ __forceinline__ bool ip_update(double2* w, const double* qraw, int T,
                                          unsigned long long seed, int bin, Mt19937_64* rng,
                                          int& bad_col) {
  bool seeded = false;
  PolarNormal gauss{0.0, false};
  const double invT = 1.0 / double(T);
#pragma unroll 1
  for (int col = 0; col < M; ++col) {
    double2 q[M * M];
    const double* p = qraw + col * M * M;
#pragma unroll
    for (int a = 0; a < M; ++a) {
      q[a + a * M] = make_double2(p[a * M + a] * invT, 0.0);
#pragma unroll
      for (int b = a + 1; b < M; ++b) {
        const double re = p[a * M + b] * invT, im = p[b * M + a] * invT;
        q[a + b * M] = make_double2(re, im);   // Q(a,b) = sum x_a conj(x_b)
        q[b + a * M] = make_double2(re, -im);  // Hermitian (symmetrize, hermitian.hpp:31-34)
      }
    }
    for (int attempt = 0;; ++attempt) {
      double2 wr[M * M];
#pragma unroll
      for (int k = 0; k < M * M; ++k) wr[k] = w[k];
      double2 a[M * M], lu[M * M], wm[M];
      int perm[M];
      double anorm = 0.0;
#pragma unroll
      for (int r = 0; r < M; ++r)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double2 s = make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < M; ++k) s = cadd(s, cmulc(wr[k + r * M], q[k + c * M]));
          a[r + c * M] = s;  // (W^H Q)(r,c)
          lu[r + c * M] = s;
          anorm += cabs2(s);
        }
      lu_factor<M>(lu, perm);
      lu_solve_unit<M>(lu, perm, col, wm);
      double wn = 0.0, rn = 0.0;
      bool fin = true;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        wn += cabs2(wm[k]);
        fin = fin && isfinite(wm[k].x) && isfinite(wm[k].y);
      }
#pragma unroll
      for (int r = 0; r < M; ++r) {
        double2 s = make_double2(r == col ? -1.0 : 0.0, 0.0);
#pragma unroll
        for (int c = 0; c < M; ++c) s = cadd(s, cmul(a[r + c * M], wm[c]));
        rn += cabs2(s);
      }
      const double scale = sqrt(anorm) * sqrt(wn) + 1.0;
      if (fin && sqrt(rn) <= 1e-8 * scale) {
        double en = 0.0;
#pragma unroll
        for (int r = 0; r < M; ++r) {
          double2 qw = make_double2(0.0, 0.0);
#pragma unroll
          for (int c = 0; c < M; ++c) qw = cadd(qw, cmul(q[r + c * M], wm[c]));
          en += cmulc(wm[r], qw).x;
        }
        if (en > 0.0 && isfinite(en)) {
          const double s = 1.0 / sqrt(en);
#pragma unroll
          for (int r = 0; r < M; ++r) w[r + col * M] = make_double2(wm[r].x * s, wm[r].y * s);
          break;
        }
      }
      if (attempt >= 1) {
        bad_col = col;
        return false;
      }
      ip_perturb(w + col * M, M, rng, &seeded, &gauss, seed, bin);
    }
  }
  return true;
}

// ------------------------------------------------------------------ kernel --
template <int M, int NT, bool EXACT, typename R>
__global__ void __launch_bounds__(256, Occ<M>::value) fit_kernel(FitParams p) {
  using C = cplx_t<R>;
  using S = Split<M>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int nthreads = blockDim.x, tid = threadIdx.x, nwarps = nthreads >> 5;
  const int lane = tid & 31, warp = tid >> 5;
  const int N = EXACT ? NT : p.N;
  const int T = p.T;
  const int b = blockIdx.x;
  const FitSmem<M, NT, R> lay(nwarps, N, T, p.nc, p.resident != 0);
  double2* Wd = reinterpret_cast<double2*>(smem + lay.off_wd);
  C* Wr = reinterpret_cast<C*>(smem + lay.off_wr);
  double* Ld = reinterpret_cast<double*>(smem + lay.off_ld);
  R* Lr = reinterpret_cast<R*>(smem + lay.off_lr);
  R* Lold = reinterpret_cast<R*>(smem + lay.off_lold);
  R* Linv = reinterpret_cast<R*>(smem + lay.off_linv);
  R* hs = reinterpret_cast<R*>(smem + lay.off_hs);
  R* us = reinterpret_cast<R*>(smem + lay.off_us);
  double* hsumv = reinterpret_cast<double*>(smem + lay.off_hsum);
  double* numd = reinterpret_cast<double*>(smem + lay.off_num);
  double* dend = reinterpret_cast<double*>(smem + lay.off_den);
  double* red = reinterpret_cast<double*>(smem + lay.off_red);
  double* res = reinterpret_cast<double*>(smem + lay.off_res);
  Scalars* sc = reinterpret_cast<Scalars*>(smem + lay.off_scal);

  // Source-loop guard: folds away when N is the compile-time NT.
#define FFCA_NK(k) (EXACT || (k) < N)

  const C* xg = reinterpret_cast<const C*>(p.x) + size_t(b) * M * T;
  R* Hg = reinterpret_cast<R*>(p.H) + size_t(b) * N * T;
  const C* xs;
  R* Hs;
  R* Us;
  if (p.resident) {
    C* xsm = reinterpret_cast<C*>(smem + lay.off_big);
    Hs = reinterpret_cast<R*>(xsm + M * T);
    Us = Hs + N * T;
    for (int k = tid; k < M * T; k += nthreads) xsm[k] = xg[k];
    for (int k = tid; k < N * T; k += nthreads) Hs[k] = Hg[k];
    xs = xsm;
  } else {
    xs = xg;
    Hs = Hg;
    Us = reinterpret_cast<R*>(p.U) + size_t(b) * M * T;
  }
  for (int k = tid; k < M * M; k += nthreads) {
    const double2 w = p.W[size_t(b) * M * M + k];
    Wd[k] = w;
    Wr[k] = mkc<R>(R(w.x), R(w.y));
  }
  for (int k = tid; k < M * N; k += nthreads) {
    const double l = p.L[size_t(b) * M * N + k];
    Ld[k] = l;
    Lr[k] = R(l);
  }
  for (int k = tid; k < NT; k += nthreads) hs[k] = R(1);
  for (int k = tid; k < M; k += nthreads) us[k] = R(1);
  const double power = p.power[b];
  if (tid == 0) {
    sc->eps = fmax(1e-8 * power, 1e-300);  // var_eps, sigmodel.hpp:29-31
    sc->stop = 0;
    sc->status = kStatusOk;
  }
  __syncthreads();
  const R eps = R(sc->eps);
  const bool update_loading = !p.fix_loadings;
  const int bin_index = (p.prob_offset + b) % p.F;

  // Warp-0 fixed-order sum of per-warp partials red[w*K + o] -> res[o].
  auto gather = [&](int K, int kact) {
    if (warp == 0) {
      for (int o = lane; o < kact; o += 32) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) s += red[w * K + o];
        res[o] = s;
      }
      __syncwarp();
    }
  };

  // ---------------------------------------------------------------- pass A --
  // first: U from x and the current W; else U = stored U * us (balance).
  // Leaves the reduced Q_m (packed) in res[0, M^3) and the NLL in res[M^3],
  // visible to warp 0 (the caller's serial section runs on thread 0).
  auto pass_a = [&](bool first, bool want_q, bool want_nll) {
    constexpr int MSPLIT = S::MSPLIT, MG = S::MG, KA = S::KA;
    const int gs = nthreads / MSPLIT;
    const int g = tid / gs, lt = tid - g * gs;
    const int m0 = g * MG;
    R q[MG * M * M];
#pragma unroll
    for (int k = 0; k < MG * M * M; ++k) q[k] = R(0);
    double nll = 0.0;
    for (int t = lt; t < T; t += gs) {
      C xv[M];
#pragma unroll
      for (int m = 0; m < M; ++m) xv[m] = xs[m * T + t];
      R h[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) h[k] = FFCA_NK(k) ? Hs[k * T + t] * hs[k] : R(0);
      R P[M * M];
      if (want_q) {
#pragma unroll
        for (int a = 0; a < M; ++a) {
          P[a * M + a] = cabs2(xv[a]);
#pragma unroll
          for (int c = a + 1; c < M; ++c) {
            const C z = cmulc(xv[c], xv[a]);  // x_a * conj(x_c)
            P[a * M + c] = z.x;
            P[c * M + a] = z.y;
          }
        }
      }
      R nll_t = R(0);
#pragma unroll
      for (int mi = 0; mi < MG; ++mi) {
        const int m = m0 + mi;
        R s2 = eps;
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (FFCA_NK(k)) s2 += Lr[m + k * M] * h[k];
        const R r = rcp_fast(s2);
        if (want_nll) {
          R u;
          if (first) {
            C y = mkc<R>(R(0), R(0));
#pragma unroll
            for (int c = 0; c < M; ++c) y = cadd(y, cmulc(Wr[c + m * M], xv[c]));
            u = cabs2(y);
          } else {
            u = Us[m * T + t] * us[m];
          }
          nll_t += u * r + flog(s2);
        }
        if (want_q) {
#pragma unroll
          for (int k = 0; k < M * M; ++k) q[mi * M * M + k] += r * P[k];
        }
      }
      nll += double(nll_t);
    }
    if (want_q) {
#pragma unroll
      for (int k = 0; k < MG * M * M; ++k) {
        const R s = warp_sum(q[k]);
        if (lane == 0) red[warp * KA + k] = double(s);
      }
    }
    {
      const double s = warp_sum(nll);
      if (lane == 0) red[warp * KA + KA - 1] = s;
    }
    __syncthreads();
    if (warp == 0) {
      const int wpg = nwarps / MSPLIT;  // warps per channel group
      const int nout = want_q ? M * M * M : 0;
      for (int o = lane; o <= nout; o += 32) {
        double s = 0.0;
        if (o == nout) {
          for (int w = 0; w < nwarps; ++w) s += red[w * KA + KA - 1];
          res[M * M * M] = s;
        } else {
          const int m = o / (M * M), k = o - m * M * M;
          const int grp = m / MG, mi = m - grp * MG;
          for (int w = grp * wpg; w < (grp + 1) * wpg; ++w) s += red[w * KA + mi * M * M + k];
          res[o] = s;
        }
      }
      __syncwarp();
    }
  };

  // ------------------------------------------------- EM sweep n (0..N) --
  // Finishes source n-1 (H row with the new L column) and accumulates the L
  // reduction of source n (fastfca.cpp:85-97).
  auto em_sweep = [&](int n, bool apply_hs) {
    R acc[M + 1];
#pragma unroll
    for (int k = 0; k <= M; ++k) acc[k] = R(0);
    const int j = n - 1;
    for (int t = tid; t < T; t += nthreads) {
      R h[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (FFCA_NK(k)) {
          R v = Hs[k * T + t];
          if (apply_hs) {
            v *= hs[k];
            Hs[k * T + t] = v;
          }
          h[k] = v;
        } else {
          h[k] = R(0);
        }
      }
      R u[M];
      if (n == 0) {
        C xv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) xv[m] = xs[m * T + t];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          C y = mkc<R>(R(0), R(0));
#pragma unroll
          for (int c = 0; c < M; ++c) y = cadd(y, cmulc(Wr[c + m * M], xv[c]));
          u[m] = cabs2(y);
          Us[m * T + t] = u[m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < M; ++m) u[m] = Us[m * T + t];
      }
      if (j >= 0) {
        R hj = R(0);
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (k == j) hj = h[k];
        R hsum_m = R(0);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          R lh = eps;
#pragma unroll
          for (int k = 0; k < NT; ++k)
            if (FFCA_NK(k)) lh += ((k == j) ? Lold[m] : Lr[m + k * M]) * h[k];
          const R lnhn = Lold[m] * hj;
          const R gg = lnhn * rcp_fast(lh);
          const R phi = gg * gg * u[m] + (R(1) - gg) * lnhn;
          hsum_m += Linv[m] * phi;
        }
        R hn = hsum_m * R(1.0 / M);
        hn = hn > tiny<R>() ? hn : tiny<R>();
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (k == j) h[k] = hn;
        Hs[j * T + t] = hn;
        acc[M] += hn;
      }
      if (n < N) {
        R hn = R(0);
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (k == n) hn = h[k];
        const R ihn = rcp_fast(hn);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          R lh = eps;
#pragma unroll
          for (int k = 0; k < NT; ++k)
            if (FFCA_NK(k)) lh += Lr[m + k * M] * h[k];
          const R lnhn = Lr[m + n * M] * hn;
          const R gg = lnhn * rcp_fast(lh);
          const R phi = gg * gg * u[m] + (R(1) - gg) * lnhn;
          acc[m] += phi * ihn;
        }
      }
    }
#pragma unroll
    for (int k = 0; k <= M; ++k) {
      const R s = warp_sum(acc[k]);
      if (lane == 0) red[warp * (M + 1) + k] = double(s);
    }
    __syncthreads();
    gather(M + 1, M + 1);
  };

  // ------------------------------------------------------ MM sweeps --
  // L update: num/den reductions over t for sources [n0, n0+nc).
  auto mm_l_sweep = [&](int n0, int ncnt, bool compute_u, bool apply_hs) {
    constexpr int NCMAX = (16 / M) > 0 ? (16 / M) : 1;
    constexpr int K = 2 * M * NCMAX;
    R acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = R(0);
    for (int t = tid; t < T; t += nthreads) {
      R h[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (FFCA_NK(k)) {
          R v = Hs[k * T + t];
          if (apply_hs) {
            v *= hs[k];
            Hs[k * T + t] = v;
          }
          h[k] = v;
        } else {
          h[k] = R(0);
        }
      }
      R u[M];
      if (compute_u) {
        C xv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) xv[m] = xs[m * T + t];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          C y = mkc<R>(R(0), R(0));
#pragma unroll
          for (int c = 0; c < M; ++c) y = cadd(y, cmulc(Wr[c + m * M], xv[c]));
          u[m] = cabs2(y);
          Us[m * T + t] = u[m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < M; ++m) u[m] = Us[m * T + t];
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R lh = eps;
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (FFCA_NK(k)) lh += Lr[m + k * M] * h[k];
        const R il = rcp_fast(lh);
        const R ul2 = u[m] * il * il;
#pragma unroll
        for (int c = 0; c < NCMAX; ++c) {
          if (c < ncnt) {
            R hn = R(0);
#pragma unroll
            for (int k = 0; k < NT; ++k)
              if (k == n0 + c) hn = h[k];
            acc[(c * M + m) * 2 + 0] += ul2 * hn;
            acc[(c * M + m) * 2 + 1] += il * hn;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k < 2 * M * ncnt) {
        const R s = warp_sum(acc[k]);
        if (lane == 0) red[warp * K + k] = double(s);
      }
    }
    __syncthreads();
    gather(K, 2 * M * ncnt);
  };

  auto mm_h_sweep = [&](bool compute_u, bool apply_hs) {
    R acc[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) acc[k] = R(0);
    for (int t = tid; t < T; t += nthreads) {
      R h[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (FFCA_NK(k)) {
          R v = Hs[k * T + t];
          if (apply_hs) v *= hs[k];
          h[k] = v;
        } else {
          h[k] = R(0);
        }
      }
      R u[M];
      if (compute_u) {
        C xv[M];
#pragma unroll
        for (int m = 0; m < M; ++m) xv[m] = xs[m * T + t];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          C y = mkc<R>(R(0), R(0));
#pragma unroll
          for (int c = 0; c < M; ++c) y = cadd(y, cmulc(Wr[c + m * M], xv[c]));
          u[m] = cabs2(y);
          Us[m * T + t] = u[m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < M; ++m) u[m] = Us[m * T + t];
      }
      R il[M], ul2[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R lh = eps;
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (FFCA_NK(k)) lh += Lr[m + k * M] * h[k];
        il[m] = rcp_fast(lh);
        ul2[m] = u[m] * il[m] * il[m];
      }
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (FFCA_NK(k)) {
          R num = R(0), den = R(0);
#pragma unroll
          for (int m = 0; m < M; ++m) {
            num += Lr[m + k * M] * ul2[m];
            den += Lr[m + k * M] * il[m];
          }
          den = den > tiny<R>() ? den : tiny<R>();
          R hv = h[k] * fsqrt(num / den);
          hv = hv > tiny<R>() ? hv : tiny<R>();
          Hs[k * T + t] = hv;
          acc[k] += hv;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if (FFCA_NK(k)) {
        const R s = warp_sum(acc[k]);
        if (lane == 0) red[warp * NT + k] = double(s);
      }
    }
    __syncthreads();
    gather(NT, N);
  };

  // -------------------------------------------------------------- driver --
  const bool record = p.record != 0;
  const bool silent = !(power > 0.0);
  pass_a(true, p.iters > 0 && !silent, record);
  if (tid == 0) {
    if (record) {
      double ld = 0.0;
      if (!log_abs_det2<M>(Wd, ld)) {
        sc->status = kStatusSingularW;
        sc->stop = 1;
      }
      sc->nll0 = -double(T) * ld + res[M * M * M];
      p.nll[size_t(0) * p.nll_stride + p.prob_offset + b] = sc->nll0;
    }
    if (silent && !sc->stop) {
      // Entirely silent band: parameters stay at the init (fastfca.cpp:165-170).
      sc->status = kStatusSilent;
      sc->stop = 1;
      if (record)
        for (int t = 0; t < p.iters; ++t)
          p.nll[size_t(t + 1) * p.nll_stride + p.prob_offset + b] = sc->nll0;
    }
    if (!sc->stop && p.iters > 0) {
      // IP sweep of iteration 0 (fastfca.cpp:36-72), fused into this serial section.
      int bad = -1;
      if (!ip_update<M>(Wd, res, T, p.seed, bin_index, reinterpret_cast<Mt19937_64*>(red), bad)) {
        sc->status = kStatusIpSingular | (bad << 8);
        sc->stop = 1;
      }
#pragma unroll
      for (int k = 0; k < M * M; ++k) Wr[k] = mkc<R>(R(Wd[k].x), R(Wd[k].y));
    }
  }
  __syncthreads();
  if (!sc->stop) {
    for (int it = 0; it < p.iters; ++it) {
      // ---- L/H updates (the IP sweep of this iteration already ran)
      if (p.flavor == 0) {
        for (int n = 0; n <= N; ++n) {
          em_sweep(n, n == 0);
          if (tid == 0) {
            if (n == 0)
              for (int k = 0; k < NT; ++k) hs[k] = R(1);
            if (n >= 1) hsumv[n - 1] = res[M];
            if (n < N) {
#pragma unroll
              for (int m = 0; m < M; ++m) {
                Lold[m] = Lr[m + n * M];
                if (update_loading) {
                  const double l = fmax(res[m] / double(T), 1e-300);  // :92-94
                  Ld[m + n * M] = l;
                  Lr[m + n * M] = narrow_pos<R>(l);
                }
                Linv[m] = rcp_fast(Lr[m + n * M]);
              }
            }
          }
          __syncthreads();
        }
      } else {
        bool first = true;
        if (update_loading) {
          for (int n0 = 0; n0 < N; n0 += p.nc) {
            const int cnt = min(p.nc, N - n0);
            mm_l_sweep(n0, cnt, first, first);
            if (tid == 0) {
              if (first)
                for (int k = 0; k < NT; ++k) hs[k] = R(1);
              for (int c = 0; c < cnt; ++c)
                for (int m = 0; m < M; ++m) {
                  numd[m + (n0 + c) * M] = res[(c * M + m) * 2 + 0];
                  dend[m + (n0 + c) * M] = res[(c * M + m) * 2 + 1];
                }
              if (n0 + cnt >= N) {
                for (int k = 0; k < M * N; ++k) {
                  const double den = fmax(dend[k], 1e-300);
                  const double l = fmax(Ld[k] * sqrt(numd[k] / den), 1e-300);  // :107-109
                  Ld[k] = l;
                  Lr[k] = narrow_pos<R>(l);
                }
              }
            }
            __syncthreads();
            first = false;
          }
        }
        mm_h_sweep(first, first);
        if (tid == 0) {
          if (first)
            for (int k = 0; k < NT; ++k) hs[k] = R(1);
          for (int k = 0; k < N; ++k) hsumv[k] = res[k];
        }
        __syncthreads();
      }
      // ---- one serial section: balance_scales (fastfca.cpp:127-142),
      //      log|det W|^2 for the trace, and the R copies of W and L.
      if (tid == 0) {
        if (p.normalize && update_loading) {
          for (int n = 0; n < N; ++n) {
            const double mu = hsumv[n] / double(T);
            if (mu > 0.0 && isfinite(mu)) {
              hs[n] = R(1.0 / mu);
#pragma unroll
              for (int m = 0; m < M; ++m) Ld[m + n * M] *= mu;
            }
          }
#pragma unroll
          for (int m = 0; m < M; ++m) {
            double s = 0.0;
            for (int n = 0; n < N; ++n) s += Ld[m + n * M];
            s /= double(N);
            if (s > 0.0 && isfinite(s)) {
              for (int n = 0; n < N; ++n) Ld[m + n * M] /= s;
              const double r = 1.0 / sqrt(s);
#pragma unroll
              for (int c = 0; c < M; ++c) {
                Wd[c + m * M].x *= r;
                Wd[c + m * M].y *= r;
              }
              us[m] = R(1.0 / s);
            }
          }
        }
        if (record) {
          double ld = 0.0;
          if (!log_abs_det2<M>(Wd, ld)) {
            sc->status = kStatusSingularW;
            sc->stop = 1;
          }
          sc->logdet = ld;
        }
        for (int k = 0; k < M * N; ++k) Lr[k] = narrow_pos<R>(Ld[k]);
#pragma unroll
        for (int k = 0; k < M * M; ++k) Wr[k] = mkc<R>(R(Wd[k].x), R(Wd[k].y));
      }
      __syncthreads();
      if (sc->stop) break;
      const bool more = it + 1 < p.iters;
      if (more || record) {
        pass_a(false, more, record);
        if (tid == 0) {
          if (record)
            p.nll[size_t(it + 1) * p.nll_stride + p.prob_offset + b] =
                -double(T) * sc->logdet + res[M * M * M];
          if (more) {
            // Next iteration's IP sweep, fused into the pass-A serial section.
#pragma unroll
            for (int m = 0; m < M; ++m) us[m] = R(1);
            int bad = -1;
            if (!ip_update<M>(Wd, res, T, p.seed + (unsigned long long)(it + 1), bin_index,
                              reinterpret_cast<Mt19937_64*>(red), bad)) {
              sc->status = kStatusIpSingular | (bad << 8);
              sc->stop = 1;
            }
#pragma unroll
            for (int k = 0; k < M * M; ++k) Wr[k] = mkc<R>(R(Wd[k].x), R(Wd[k].y));
          }
        }
        __syncthreads();
        if (sc->stop) break;
      }
    }
  }
#undef FFCA_NK
  __syncthreads();
  // ------------------------------------------------------------- epilogue --
  for (int k = tid; k < M * M; k += nthreads) p.W[size_t(b) * M * M + k] = Wd[k];
  for (int k = tid; k < M * N; k += nthreads) p.L[size_t(b) * M * N + k] = Ld[k];
  if (p.resident) {
    for (int k = tid; k < N * T; k += nthreads) Hg[k] = Hs[k] * hs[k / T];
  } else {
    bool pending = false;
    for (int k = 0; k < N; ++k) pending = pending || hs[k] != R(1);
    if (pending)
      for (int k = tid; k < N * T; k += nthreads) Hg[k] = Hg[k] * hs[k / T];
  }
  if (tid == 0) p.status[b] = sc->status;
}

}  // namespace ffca
