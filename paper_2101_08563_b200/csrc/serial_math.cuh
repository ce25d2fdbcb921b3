// serial_math.cuh -- the per-bin serial algebra of the fit (one thread, M x M
// complex, registers only), templated on its arithmetic type SR.
//
// SR = double in the fp64 check mode: faithful to the reference's fp64
// Eigen::PartialPivLU arithmetic up to rounding.  SR = float in the fp32
// path: the weighted covariances it consumes are fp32-accurate sums anyway,
// and fp32 SFU reciprocals / square roots shorten the dependent chain that
// every thread of the CTA waits on, by ~4x versus fp64 division.  The only
// semantic knob is the IP residual test of fastfca.cpp:55-56: the reference's
// 1e-8 relative threshold is below fp32 rounding of a backward-stable 2x2 /
// LU solve (~1e-7 ||a|| ||w||), so the fp32 path tests at 64 * FLT_EPSILON
// (7.6e-6) -- still a singularity guard, restarts stay the rare event the
// reference intends.
#pragma once

#include "common.cuh"

namespace ffca {

template <typename SR>
struct SMath;

template <>
struct SMath<float> {
  static constexpr float kResidTol2 = 7.62939453125e-06f * 7.62939453125e-06f;  // (64 eps)^2
  __device__ static __forceinline__ float rcp(float x) { return rcp_fast(x); }
  __device__ static __forceinline__ float rsq(float x) { return rsqrtf(x); }
  __device__ static __forceinline__ float sq(float x) { return sqrtf(x); }
  __device__ static __forceinline__ double log_d(float x) {
    return double(flog2_ftz(x)) * 0.69314718055994531;
  }
  // log of a positive normal double to fp32 relative accuracy over the full
  // double range: exponent + SFU log2 of the mantissa in [1, 2).
  __device__ static __forceinline__ double log_wide(double x) {
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int e = (hi >> 20) & 0x7ff;
    if (e == 0 || e == 0x7ff) return log(x);
    const float m = float(__hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo));
    return (double(e - 1023) + double(flog2_ftz(m))) * 0.69314718055994531;
  }
};

template <>
struct SMath<double> {
  static constexpr double kResidTol2 = 1e-16;  // (1e-8)^2, fastfca.cpp:56
  // 1/x to within an ulp without the division slow path: an SFU fp32 seed on
  // the mantissa refined by two fp64 Newton steps (zero/denormal/huge fall
  // back to the IEEE division).
  __device__ static __forceinline__ double rcp(double x) {
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int e = (hi >> 20) & 0x7ff;
    if (e == 0 || e >= 2046) return 1.0 / x;
    const double m = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, lo);  // |m| in [1, 2)
    double r = double(rcp_fast(float(m)));
    r = fma(r, fma(-m, r, 1.0), r);
    r = fma(r, fma(-m, r, 1.0), r);
    return r * __hiloint2double((2046 - e) << 20, 0);  // * 2^(1023 - e)
  }
  __device__ static __forceinline__ double rsq(double x) { return rsqrt(x); }
  __device__ static __forceinline__ double sq(double x) { return sqrt(x); }
  __device__ static __forceinline__ double log_d(double x) { return log(x); }
  __device__ static __forceinline__ double log_wide(double x) { return log(x); }
};

__device__ __forceinline__ double fast_rcp(double x) { return SMath<double>::rcp(x); }

// In-place LU with partial pivoting.  Pivot order follows Eigen::PartialPivLU
// (largest modulus; compared as squared modulus, the same order).
template <int M, typename SR>
__device__ __forceinline__ void lu_factor(cplx_t<SR> (&a)[M * M], int (&perm)[M]) {
  using SC = cplx_t<SR>;
#pragma unroll
  for (int k = 0; k < M; ++k) perm[k] = k;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    int p = k;
    SR best = cabs2(a[k + k * M]);
#pragma unroll
    for (int r = k + 1; r < M; ++r) {
      const SR v = cabs2(a[r + k * M]);
      if (v > best) best = v, p = r;
    }
#pragma unroll
    for (int r = k + 1; r < M; ++r) {
      if (r == p) {
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const SC t = a[k + c * M];
          a[k + c * M] = a[r + c * M];
          a[r + c * M] = t;
        }
        const int t = perm[k];
        perm[k] = perm[r];
        perm[r] = t;
      }
    }
    if (best != SR(0)) {
      const SC piv = a[k + k * M];
      const SR s = SMath<SR>::rcp(best);
      const SC ipiv = mkc<SR>(piv.x * s, -piv.y * s);  // 1 / piv
#pragma unroll
      for (int r = k + 1; r < M; ++r) a[r + k * M] = cmul(a[r + k * M], ipiv);
#pragma unroll
      for (int c = k + 1; c < M; ++c)
#pragma unroll
        for (int r = k + 1; r < M; ++r)
          a[r + c * M] = csub(a[r + c * M], cmul(a[r + k * M], a[k + c * M]));
    }
  }
}

// Solve (P^T L U) y = e_col.
template <int M, typename SR>
__device__ __forceinline__ void lu_solve_unit(const cplx_t<SR> (&lu)[M * M], const int (&perm)[M],
                                              int col, cplx_t<SR> (&y)[M]) {
#pragma unroll
  for (int k = 0; k < M; ++k) y[k] = mkc<SR>(perm[k] == col ? SR(1) : SR(0), SR(0));
#pragma unroll
  for (int k = 0; k < M; ++k)
#pragma unroll
    for (int r = k + 1; r < M; ++r) y[r] = csub(y[r], cmul(lu[r + k * M], y[k]));
#pragma unroll
  for (int k = M - 1; k >= 0; --k) {
    const cplx_t<SR> d = lu[k + k * M];
    const SR s = SMath<SR>::rcp(cabs2(d));
    y[k] = cmul(y[k], mkc<SR>(d.x * s, -d.y * s));
#pragma unroll
    for (int r = 0; r < k; ++r) y[r] = csub(y[r], cmul(lu[r + k * M], y[k]));
  }
}

// log|det W|^2 (sigmodel.cpp:118-129) of the fp64 master W, computed in SR.
// Returns false when W is numerically singular (a zero or non-finite pivot).
template <int M, typename SR>
__device__ __forceinline__ bool log_abs_det2(const double2* w, double& out) {
  using SC = cplx_t<SR>;
  if constexpr (M == 1) {
    const SR v = SR(w[0].x) * SR(w[0].x) + SR(w[0].y) * SR(w[0].y);
    if (!(v > SR(0)) || !isfinite(v)) return false;
    out = SMath<SR>::log_d(v);
    return true;
  } else if constexpr (M == 2) {
    // |u00 u11|^2 of the pivoted LU equals |det W|^2; a vanishing pivot is
    // the singular case the reference rejects.
    const SC w00 = mkc<SR>(SR(w[0].x), SR(w[0].y)), w10 = mkc<SR>(SR(w[1].x), SR(w[1].y));
    const SC w01 = mkc<SR>(SR(w[2].x), SR(w[2].y)), w11 = mkc<SR>(SR(w[3].x), SR(w[3].y));
    const SR a0 = cabs2(w00), a1 = cabs2(w10);
    const SR d = cabs2(csub(cmul(w00, w11), cmul(w01, w10)));
    if (!((a0 > SR(0) || a1 > SR(0)) && d > SR(0)) || !isfinite(d)) return false;
    out = SMath<SR>::log_d(d);
    return true;
  } else {
    SC a[M * M];
    int perm[M];
#pragma unroll
    for (int k = 0; k < M * M; ++k) a[k] = mkc<SR>(SR(w[k].x), SR(w[k].y));
    lu_factor<M, SR>(a, perm);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const SR v = cabs2(a[k + k * M]);
      if (!(v > SR(0)) || !isfinite(v)) return false;
      acc += SMath<SR>::log_d(v);  // sum of log|u_kk|^2 = 2 * sum log|u_kk|
    }
    out = acc;
    return true;
  }
}

// Cold path of ip_update_w: one seeded perturbation of a column
// (fastfca.cpp:66-69).  The generator is seeded lazily on the first restart
// of the sweep and its state lives in shared scratch.
static __device__ __noinline__ void ip_perturb(double2* wcol, int m, RestartRng* rr, bool first,
                                               unsigned long long seed, int bin) {
  if (first) {  // a fresh generator + distribution per sweep (fastfca.cpp:40-41)
    rr->mt.seed(mix_seed(seed, bin));
    rr->gauss.saved = 0.0;
    rr->gauss.has_saved = false;
  }
  double cn = 0.0;
  for (int r = 0; r < m; ++r) cn += cabs2(wcol[r]);
  const double mag = 1e-8 * (sqrt(cn) + 1.0);
  for (int r = 0; r < m; ++r) {
    const double im = rr->gauss(rr->mt);  // g++ evaluates Complex(g(), g()) right to left
    const double re = rr->gauss(rr->mt);
    wcol[r].x += mag * re;
    wcol[r].y += mag * im;
  }
}

// Optional side jobs of an IP sweep, folded in to keep them off the serial
// path: wscale -- balance column scales still to be applied to W first;
// wout -- compute-type copy of the new W; ldet/ldok -- log|det W_new|^2
// (M = 2 only; sigmodel.cpp:118-129).
template <typename SR>
struct IpExtras {
  const SR* wscale = nullptr;
  cplx_t<SR>* wout = nullptr;
  double* ldet = nullptr;
  int* ldok = nullptr;
};

// One column of the M = 2 sweep: candidate w (normalised) and whether it
// passes the reference's acceptance tests.
template <typename SR>
__device__ __forceinline__ bool ip_col_m2(const cplx_t<SR> (&wr)[4], int col, SR q00, SR q11,
                                          cplx_t<SR> q01, cplx_t<SR> (&out)[2]) {
  using SC = cplx_t<SR>;
  // A(r, c) = sum_k conj(W(k, r)) Q(k, c), Q(1, 0) = conj(q01).
  SC a[4];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const SC u0 = wr[2 * r], u1 = wr[2 * r + 1];  // column r of W
    // conj(u0) q00 + conj(u1) conj(q01)
    a[r] = mkc<SR>(u0.x * q00 + (u1.x * q01.x - u1.y * q01.y),
                   -u0.y * q00 - (u1.x * q01.y + u1.y * q01.x));
    // conj(u0) q01 + conj(u1) q11
    a[r + 2] = mkc<SR>((u0.x * q01.x + u0.y * q01.y) + u1.x * q11,
                       (u0.x * q01.y - u0.y * q01.x) - u1.y * q11);
  }
  const SC det = csub(cmul(a[0], a[3]), cmul(a[2], a[1]));
  const SR s = SMath<SR>::rcp(cabs2(det));
  const SC idet = mkc<SR>(det.x * s, -det.y * s);
  SC wm[2];
  if (col == 0) {
    wm[0] = cmul(a[3], idet);
    wm[1] = cmul(mkc<SR>(-a[1].x, -a[1].y), idet);
  } else {
    wm[0] = cmul(mkc<SR>(-a[2].x, -a[2].y), idet);
    wm[1] = cmul(a[0], idet);
  }
  const SR anorm = (cabs2(a[0]) + cabs2(a[1])) + (cabs2(a[2]) + cabs2(a[3]));
  const SR wn = cabs2(wm[0]) + cabs2(wm[1]);
  const bool fin = isfinite(wm[0].x) && isfinite(wm[0].y) && isfinite(wm[1].x) && isfinite(wm[1].y);
  SC r0 = cadd(cmul(a[0], wm[0]), cmul(a[2], wm[1]));
  SC r1 = cadd(cmul(a[1], wm[0]), cmul(a[3], wm[1]));
  if (col == 0) r0.x -= SR(1); else r1.x -= SR(1);
  const SR rn = cabs2(r0) + cabs2(r1);
  const SR scale = SR(sqrt_approx(float(anorm * wn))) + SR(1);
  // w^H Q w = q00 |w0|^2 + q11 |w1|^2 + 2 Re(conj(w0) q01 w1)
  const SC qw1 = cmul(q01, wm[1]);
  const SR en = (q00 * cabs2(wm[0]) + q11 * cabs2(wm[1])) +
                SR(2) * (wm[0].x * qw1.x + wm[0].y * qw1.y);
  const SR sc = SMath<SR>::rsq(en);
  out[0] = mkc<SR>(wm[0].x * sc, wm[0].y * sc);
  out[1] = mkc<SR>(wm[1].x * sc, wm[1].y * sc);
  return fin && rn <= SMath<SR>::kResidTol2 * scale * scale && en > SR(0) && isfinite(en);
}

// The reference's M = 2 sweep in fp64, column by column with the seeded
// restart (fastfca.cpp:36-72): the cold fallback of ip_update_m2.
static __device__ __noinline__ bool ip_m2_careful(double2* w, const double* qraw, double invT,
                                                  unsigned long long seed, int bin,
                                                  RestartRng* rr, int& bad_col) {
  double2 wr[4];
  for (int k = 0; k < 4; ++k) wr[k] = w[k];
  bool restarted = false;
  for (int col = 0; col < 2; ++col) {
    const double* p = qraw + 4 * col;
    const double q00 = p[0] * invT, q11 = p[3] * invT;
    const double2 q01 = make_double2(p[1] * invT, p[2] * invT);
    for (int attempt = 0;; ++attempt) {
      double2 o[2];
      if (ip_col_m2<double>(wr, col, q00, q11, q01, o)) {
        wr[2 * col] = o[0];
        wr[2 * col + 1] = o[1];
        w[2 * col] = o[0];
        w[2 * col + 1] = o[1];
        break;
      }
      if (attempt >= 1) {
        bad_col = col;
        return false;
      }
      ip_perturb(w + 2 * col, 2, rr, !restarted, seed, bin);
      restarted = true;
      wr[2 * col] = w[2 * col];
      wr[2 * col + 1] = w[2 * col + 1];
    }
  }
  return true;
}

// M = 2 IP sweep in closed form on the Hermitian structure of Q (real
// diagonal, Q(1,0) = conj Q(0,1)): A = W^H Q_k, w = A^{-1} e_k from the 2x2
// adjugate, the residual test, w /= sqrt(w^H Q_k w) -- the same steps as the
// general path below with the zero imaginary parts and the symmetric half
// folded away.  Both columns are first solved speculatively (no branch on
// the acceptance tests between them, so the tests overlap the next column);
// only if a test fails is the sweep redone column by column with the
// reference's seeded restart.
template <typename SR>
__device__ __forceinline__ bool ip_update_m2(double2* w, const double* qraw, double invT,
                                             unsigned long long seed, int bin, RestartRng* rr,
                                             int& bad_col, IpExtras<SR> ex) {
  using SC = cplx_t<SR>;
  SR qd0[2], qd1[2];
  SC qo[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const double* p = qraw + 4 * c;
    qd0[c] = SR(p[0] * invT);
    qd1[c] = SR(p[3] * invT);
    qo[c] = mkc<SR>(SR(p[1] * invT), SR(p[2] * invT));  // Q(0,1)
  }
  SC wr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) wr[k] = mkc<SR>(SR(w[k].x), SR(w[k].y));
  auto finish = [&](const SC (&f)[4]) {
    if (ex.wout)
#pragma unroll
      for (int k = 0; k < 4; ++k) ex.wout[k] = f[k];
    if (ex.ldet) {
      const SR a0 = cabs2(f[0]), a1 = cabs2(f[1]);
      const SR d = cabs2(csub(cmul(f[0], f[3]), cmul(f[2], f[1])));
      const bool ok = (a0 > SR(0) || a1 > SR(0)) && d > SR(0) && isfinite(d);
      *ex.ldok = ok ? 1 : 0;
      *ex.ldet = ok ? SMath<SR>::log_d(d) : 0.0;
    }
  };
  {
    SC f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[k] = wr[k];
      if (ex.wscale) f[k].x *= ex.wscale[k >> 1], f[k].y *= ex.wscale[k >> 1];
    }
    SC o[2];
    const bool ok0 = ip_col_m2<SR>(f, 0, qd0[0], qd1[0], qo[0], o);
    f[0] = o[0], f[1] = o[1];
    const bool ok1 = ip_col_m2<SR>(f, 1, qd0[1], qd1[1], qo[1], o);
    f[2] = o[0], f[3] = o[1];
    if (ok0 && ok1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = make_double2(double(f[k].x), double(f[k].y));
      finish(f);
      return true;
    }
  }
  // Careful path, in fp64 whatever SR is: the reference's arithmetic and
  // 1e-8 residual test, column by column with the seeded restart, from the
  // (scaled) master.  In the fp32 path this catches ill-conditioned systems
  // (e.g. ICA mode, where H converges onto U) that fp32 cannot resolve to
  // the fp32 tolerance but the reference's fp64 solve accepts.
  if (ex.wscale) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double c = double(ex.wscale[k >> 1]);
      w[k].x *= c;
      w[k].y *= c;
    }
  }
  if (!ip_m2_careful(w, qraw, invT, seed, bin, rr, bad_col)) return false;
#pragma unroll
  for (int k = 0; k < 4; ++k) wr[k] = mkc<SR>(SR(w[k].x), SR(w[k].y));
  finish(wr);
  return true;
}

// ip_update_w (fastfca.cpp:36-72) on the reduced weighted covariances.
// qraw[m*M*M + ...] holds sum_t x x^H / sigma2_m packed as: (a,a) real,
// (a,b) a<b real part at a*M+b and imaginary part at b*M+a.  w is the fp64
// master W (updated in place).
// SPEC: speculative pass -- registers only, no restart; returns false on the
// first failed acceptance test without touching w (the caller then reruns
// the sweep the reference's way).
template <int M, typename SR, bool SPEC>
__device__ __forceinline__ bool ip_update_gen(double2* w, const double* qraw, double invT,
                                              unsigned long long seed, int bin, RestartRng* rr,
                                              int& bad_col, IpExtras<SR> ex) {
  using SC = cplx_t<SR>;
  bool restarted = false;
  if (!SPEC && ex.wscale)
    for (int k = 0; k < M * M; ++k) {
      const double c = double(ex.wscale[k / M]);
      w[k].x *= c;
      w[k].y *= c;
    }
  SC wr[M * M];
#pragma unroll
  for (int k = 0; k < M * M; ++k) {
    wr[k] = mkc<SR>(SR(w[k].x), SR(w[k].y));
    if (SPEC && ex.wscale) wr[k].x *= ex.wscale[k / M], wr[k].y *= ex.wscale[k / M];
  }
  // Unrolled for M <= 3: every register-array index is a compile-time
  // constant (a rolled column loop indexes wr[] dynamically and demotes it to
  // local memory); M = 4 keeps the rolled loop (the unrolled body spills).
#pragma unroll(M <= 3 ? M : 1)
  for (int col = 0; col < M; ++col) {
    SC q[M * M];
    const double* p = qraw + col * M * M;
#pragma unroll
    for (int a = 0; a < M; ++a) {
      q[a + a * M] = mkc<SR>(SR(p[a * M + a] * invT), SR(0));
#pragma unroll
      for (int b = a + 1; b < M; ++b) {
        const SR re = SR(p[a * M + b] * invT), im = SR(p[b * M + a] * invT);
        q[a + b * M] = mkc<SR>(re, im);   // Q(a,b) = sum x_a conj(x_b)
        q[b + a * M] = mkc<SR>(re, -im);  // Hermitian (symmetrize, hermitian.hpp:31-34)
      }
    }
    for (int attempt = 0;; ++attempt) {
      SC a[M * M], wm[M];
      SR anorm = SR(0);
#pragma unroll
      for (int r = 0; r < M; ++r)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          SC s = cmulc(wr[r * M], q[c * M]);
#pragma unroll
          for (int k = 1; k < M; ++k) s = cadd(s, cmulc(wr[k + r * M], q[k + c * M]));
          a[r + c * M] = s;  // (W^H Q)(r,c)
          anorm += cabs2(s);
        }
      if constexpr (M == 1) {
        const SR s = SMath<SR>::rcp(cabs2(a[0]));
        wm[0] = mkc<SR>(a[0].x * s, -a[0].y * s);
      } else if constexpr (M == 2) {
        // Closed-form inverse column; the same solution as the pivoted LU.
        const SC det = csub(cmul(a[0], a[3]), cmul(a[2], a[1]));
        const SR s = SMath<SR>::rcp(cabs2(det));
        const SC idet = mkc<SR>(det.x * s, -det.y * s);
        if (col == 0) {
          wm[0] = cmul(a[3], idet);
          wm[1] = cmul(mkc<SR>(-a[1].x, -a[1].y), idet);
        } else {
          wm[0] = cmul(mkc<SR>(-a[2].x, -a[2].y), idet);
          wm[1] = cmul(a[0], idet);
        }
      } else {
        SC lu[M * M];
        int perm[M];
#pragma unroll
        for (int k = 0; k < M * M; ++k) lu[k] = a[k];
        lu_factor<M, SR>(lu, perm);
        lu_solve_unit<M, SR>(lu, perm, col, wm);
      }
      SR wn = SR(0), rn = SR(0);
      bool fin = true;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        wn += cabs2(wm[k]);
        fin = fin && isfinite(wm[k].x) && isfinite(wm[k].y);
      }
#pragma unroll
      for (int r = 0; r < M; ++r) {
        SC s = mkc<SR>(r == col ? SR(-1) : SR(0), SR(0));
#pragma unroll
        for (int c = 0; c < M; ++c) s = cadd(s, cmul(a[r + c * M], wm[c]));
        rn += cabs2(s);
      }
      // Residual test ||a w - e|| <= tol (||a|| ||w|| + 1) (fastfca.cpp:55-56),
      // squared; the scale is a tolerance, so an fp32 square root suffices.
      const SR scale = SR(sqrt_approx(float(anorm * wn))) + SR(1);
      if (fin && rn <= SMath<SR>::kResidTol2 * scale * scale) {
        SR en = SR(0);
#pragma unroll
        for (int r = 0; r < M; ++r) {
          SC qw = cmul(q[r], wm[0]);
#pragma unroll
          for (int c = 1; c < M; ++c) qw = cadd(qw, cmul(q[r + c * M], wm[c]));
          en += cmulc(wm[r], qw).x;
        }
        if (en > SR(0) && isfinite(en)) {
          const SR s = SMath<SR>::rsq(en);
#pragma unroll
          for (int r = 0; r < M; ++r) {
            wr[r + col * M] = mkc<SR>(wm[r].x * s, wm[r].y * s);
            if (!SPEC)
              w[r + col * M] = make_double2(double(wr[r + col * M].x), double(wr[r + col * M].y));
          }
          break;
        }
      }
      if (SPEC) return false;
      if (attempt >= 1) {
        bad_col = col;
        return false;
      }
      ip_perturb(w + col * M, M, rr, !restarted, seed, bin);
      restarted = true;
#pragma unroll
      for (int k = 0; k < M * M; ++k) wr[k] = mkc<SR>(SR(w[k].x), SR(w[k].y));
    }
  }
  if (SPEC)
#pragma unroll
    for (int k = 0; k < M * M; ++k) w[k] = make_double2(double(wr[k].x), double(wr[k].y));
  if (ex.wout)
#pragma unroll
    for (int k = 0; k < M * M; ++k) ex.wout[k] = wr[k];
  return true;
}

// The reference's sweep in fp64 (cold fallback of the fp32 path).
template <int M>
__device__ __noinline__ bool ip_update_f64(double2* w, const double* qraw, double invT,
                                           unsigned long long seed, int bin, RestartRng* rr,
                                           int& bad_col) {
  return ip_update_gen<M, double, false>(w, qraw, invT, seed, bin, rr, bad_col,
                                         IpExtras<double>());
}

// ip_update_w (fastfca.cpp:36-72).  fp32 path: a speculative fp32 sweep; if
// any column fails its acceptance test, the sweep is redone from the master W
// in fp64 with the reference's 1e-8 residual test and seeded restart.
template <int M, typename SR>
__device__ __forceinline__ bool ip_update(double2* w, const double* qraw, double invT,
                                          unsigned long long seed, int bin, RestartRng* rr,
                                          int& bad_col, IpExtras<SR> ex = IpExtras<SR>()) {
  if constexpr (M == 2) {
    return ip_update_m2<SR>(w, qraw, invT, seed, bin, rr, bad_col, ex);
  } else if constexpr (sizeof(SR) == 4) {
    if (ip_update_gen<M, SR, true>(w, qraw, invT, seed, bin, rr, bad_col, ex)) return true;
    if (ex.wscale)
      for (int k = 0; k < M * M; ++k) {
        const double c = double(ex.wscale[k / M]);
        w[k].x *= c;
        w[k].y *= c;
      }
    if (!ip_update_f64<M>(w, qraw, invT, seed, bin, rr, bad_col)) return false;
    if (ex.wout)
      for (int k = 0; k < M * M; ++k) ex.wout[k] = mkc<SR>(SR(w[k].x), SR(w[k].y));
    return true;
  } else {
    return ip_update_gen<M, SR, false>(w, qraw, invT, seed, bin, rr, bad_col, ex);
  }
}

// ------------------------------------------------ warp-cooperative (M > 4) --
// For M > 4 the single-thread register algebra above spills and serialises
// ~M^3 complex operations; one warp shares the work instead: matrices live in
// shared scratch, lanes own matrix entries, Gauss-Jordan elimination with the
// same partial pivoting (largest modulus, lowest row on ties) replaces the
// LU + substitution, and reductions are warp shuffles.

// Warp argmax of v over lanes [k, M) (ties -> lowest lane); result broadcast.
template <typename SR>
__device__ __forceinline__ int warp_pivot(SR v, int k, int M, int lane) {
  SR best = (lane >= k && lane < M) ? v : SR(-1);
  int idx = lane;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const SR ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) best = ob, idx = oi;
  }
  return idx;
}

template <typename SR>
__device__ __forceinline__ SR warp_allsum(SR v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// In-place Gauss-Jordan on the augmented M x (M+1) matrix A (column-major,
// column M is the right-hand side).  Returns false on a zero pivot; the
// pivots' log|.|^2 sum (log-det of the original matrix) goes to *logdet2.
template <int M, typename SR>
__device__ bool warp_gauss_jordan(cplx_t<SR>* A, int lane, double* logdet2) {
  using SC = cplx_t<SR>;
  constexpr int MA = M + 1;
  double ld = 0.0;
  bool ok = true;
  for (int k = 0; k < M; ++k) {
    const SR v = lane < M ? cabs2(A[lane + k * M]) : SR(-1);
    const int p = warp_pivot(v, k, M, lane);
    if (p != k)
      for (int c = lane; c < MA; c += 32) {
        const SC t = A[k + c * M];
        A[k + c * M] = A[p + c * M];
        A[p + c * M] = t;
      }
    __syncwarp();
    const SC piv = A[k + k * M];
    const SR pm = cabs2(piv);
    if (!(pm > SR(0)) || !isfinite(pm)) ok = false;
    ld += SMath<SR>::log_d(pm);
    const SR s = SMath<SR>::rcp(pm);
    const SC ipiv = mkc<SR>(piv.x * s, -piv.y * s);
    // Scale the pivot row by 1/A(k,k) (columns > k); column k keeps the
    // elimination factors A(r,k) of the other rows.
    for (int c = k + 1 + lane; c < MA; c += 32) A[k + c * M] = cmul(A[k + c * M], ipiv);
    __syncwarp();
    // Eliminate column k from every other row: A(r,c) -= A(r,k) A(k,c)/A(k,k), c > k.
    for (int e = lane; e < M * (MA - k - 1); e += 32) {
      const int r = e % M, c = k + 1 + e / M;
      if (r != k) A[r + c * M] = csub(A[r + c * M], cmul(A[r + k * M], A[k + c * M]));
    }
    __syncwarp();
  }
  *logdet2 = ld;
  return ok;
}

template <int M, typename SR>
__device__ bool warp_log_abs_det2(const double2* w, cplx_t<SR>* scratch, int lane, double& out) {
  for (int e = lane; e < M * (M + 1); e += 32)
    scratch[e] = e < M * M ? mkc<SR>(SR(w[e].x), SR(w[e].y)) : mkc<SR>(SR(0), SR(0));
  __syncwarp();
  double ld = 0.0;
  const bool ok = warp_gauss_jordan<M, SR>(scratch, lane, &ld);
  out = ld;
  return ok;
}

// ip_update_w (fastfca.cpp:36-72) by one warp.  scratch: 3*M*M + 2*M complex.
template <int M, typename SR>
__device__ bool ip_update_warp(double2* w, const double* qraw, double invT,
                               unsigned long long seed, int bin, RestartRng* rng,
                               cplx_t<SR>* scratch, int lane, int& bad_col) {
  using SC = cplx_t<SR>;
  SC* Q = scratch;              // M x M
  SC* A = Q + M * M;            // M x (M+1) augmented, eliminated in place
  SC* A0 = A + M * (M + 1);     // M x M, W^H Q kept for the residual
  SC* Wc = A0 + M * M;          // M x M compute-type copy of W
  bool restarted = false;
  for (int e = lane; e < M * M; e += 32) Wc[e] = mkc<SR>(SR(w[e].x), SR(w[e].y));
  for (int col = 0; col < M; ++col) {
    const double* p = qraw + col * M * M;
    for (int e = lane; e < M * M; e += 32) {
      const int a = e % M, b = e / M;
      if (a == b) Q[e] = mkc<SR>(SR(p[a * M + a] * invT), SR(0));
      else if (a < b) Q[e] = mkc<SR>(SR(p[a * M + b] * invT), SR(p[b * M + a] * invT));
      else Q[e] = mkc<SR>(SR(p[b * M + a] * invT), SR(-p[a * M + b] * invT));
    }
    __syncwarp();
    for (int attempt = 0;; ++attempt) {
      SR an = SR(0);
      for (int e = lane; e < M * M; e += 32) {
        const int r = e % M, c = e / M;
        SC s = cmulc(Wc[r * M], Q[c * M]);
        for (int k = 1; k < M; ++k) s = cadd(s, cmulc(Wc[k + r * M], Q[k + c * M]));
        A[e] = s;  // (W^H Q)(r,c), column-major like the augmented matrix
        A0[e] = s;
        an += cabs2(s);
      }
      if (lane < M) A[lane + M * M] = mkc<SR>(lane == col ? SR(1) : SR(0), SR(0));
      const SR anorm = warp_allsum(an);
      __syncwarp();
      double ldummy;
      warp_gauss_jordan<M, SR>(A, lane, &ldummy);
      // w = the eliminated right-hand side (lane r holds w_r).
      const SC wmr = lane < M ? A[lane + M * M] : mkc<SR>(SR(0), SR(0));
      const bool fin = __all_sync(0xffffffffu, isfinite(wmr.x) && isfinite(wmr.y));
      const SR wn = warp_allsum(cabs2(wmr));
      SC rr = mkc<SR>(lane == col ? SR(-1) : SR(0), SR(0));
      SC qw = mkc<SR>(SR(0), SR(0));
      for (int c = 0; c < M; ++c) {
        const SC wc = mkc<SR>(__shfl_sync(0xffffffffu, wmr.x, c), __shfl_sync(0xffffffffu, wmr.y, c));
        if (lane < M) {
          rr = cadd(rr, cmul(A0[lane + c * M], wc));
          qw = cadd(qw, cmul(Q[lane + c * M], wc));
        }
      }
      const SR rn = warp_allsum(lane < M ? cabs2(rr) : SR(0));
      const SR en = warp_allsum(lane < M ? cmulc(wmr, qw).x : SR(0));
      const SR scale = SR(sqrt_approx(float(anorm * wn))) + SR(1);
      if (fin && rn <= SMath<SR>::kResidTol2 * scale * scale && en > SR(0) && isfinite(en)) {
        const SR s = SMath<SR>::rsq(en);
        if (lane < M) {
          const SC nw = mkc<SR>(wmr.x * s, wmr.y * s);
          Wc[lane + col * M] = nw;
          w[lane + col * M] = make_double2(double(nw.x), double(nw.y));
        }
        __syncwarp();
        break;
      }
      if (attempt >= 1) {
        bad_col = col;
        return false;
      }
      if (lane == 0) ip_perturb(w + col * M, M, rng, !restarted, seed, bin);
      restarted = true;
      __syncwarp();
      for (int e = lane; e < M * M; e += 32) Wc[e] = mkc<SR>(SR(w[e].x), SR(w[e].y));
      __syncwarp();
    }
  }
  return true;
}

// ip_update_w (fastfca.cpp:36-72) by one warp with the system in registers:
// lane r (< M) holds row r of A = W^H Q_col (and of the right-hand side e_col)
// and column r of W.  Gauss-Jordan with partial pivoting runs on virtual row
// positions: the pivot is the largest |A(., k)|^2 among the rows not yet used
// (ties -> lowest current position, exactly the order the physical row swaps
// of ip_update_warp / Eigen::PartialPivLU produce), its row is broadcast by
// shuffles and every other row eliminates against it -- no shared-memory
// round trips or warp syncs inside the elimination.  Q_col is read from
// `scratch` (M x M).  Same arithmetic, acceptance tests and seeded restart as
// ip_update_warp.
template <int M, typename SR>
__device__ bool ip_update_warp_reg(double2* w, const double* qraw, double invT,
                                   unsigned long long seed, int bin, RestartRng* rng,
                                   cplx_t<SR>* scratch, int lane, int& bad_col) {
  using SC = cplx_t<SR>;
  SC* Q = scratch;  // M x M, column-major
  const bool act = lane < M;
  const int r = act ? lane : 0;
  bool restarted = false;
  SC wcol[M];  // column r of W, compute type
#pragma unroll
  for (int k = 0; k < M; ++k) wcol[k] = mkc<SR>(SR(w[k + r * M].x), SR(w[k + r * M].y));
  for (int col = 0; col < M; ++col) {
    const double* p = qraw + col * M * M;
    for (int e = lane; e < M * M; e += 32) {
      const int a = e % M, b = e / M;
      if (a == b) Q[e] = mkc<SR>(SR(p[a * M + a] * invT), SR(0));
      else if (a < b) Q[e] = mkc<SR>(SR(p[a * M + b] * invT), SR(p[b * M + a] * invT));
      else Q[e] = mkc<SR>(SR(p[b * M + a] * invT), SR(-p[a * M + b] * invT));
    }
    __syncwarp();
    for (int attempt = 0;; ++attempt) {
      // Row r of A = W^H Q (column r of W against every column of Q).
      SC row[M + 1], a0[M];
      SR an = SR(0);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        SC s = cmulc(wcol[0], Q[c * M]);
#pragma unroll
        for (int k = 1; k < M; ++k) s = cadd(s, cmulc(wcol[k], Q[k + c * M]));
        row[c] = s;
        a0[c] = s;
        an += act ? cabs2(s) : SR(0);
      }
      row[M] = mkc<SR>(r == col ? SR(1) : SR(0), SR(0));
      const SR anorm = warp_allsum(an);
      // Gauss-Jordan on virtual positions.
      bool used = !act;
      int pos = lane;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        SR best = used ? SR(-1) : cabs2(row[k]);
        int bpos = used ? 1 << 20 : pos, blane = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const SR ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
          const int ol = __shfl_xor_sync(0xffffffffu, blane, o);
          if (ob > best || (ob == best && op < bpos)) best = ob, bpos = op, blane = ol;
        }
        const int pl = blane;  // pivot lane
        SC prow[M + 1];
#pragma unroll
        for (int c = k; c <= M; ++c)
          prow[c] = mkc<SR>(__shfl_sync(0xffffffffu, row[c].x, pl),
                            __shfl_sync(0xffffffffu, row[c].y, pl));
        const SR pm = cabs2(prow[k]);
        const SR sc = SMath<SR>::rcp(pm);
        const SC ipiv = mkc<SR>(prow[k].x * sc, -prow[k].y * sc);
        // Scaled pivot row (columns > k): A(k,c) / A(k,k).
#pragma unroll
        for (int c = k + 1; c <= M; ++c) prow[c] = cmul(prow[c], ipiv);
        if (lane == pl) {
#pragma unroll
          for (int c = k + 1; c <= M; ++c) row[c] = prow[c];
        } else if (act) {
          const SC f = row[k];
#pragma unroll
          for (int c = k + 1; c <= M; ++c) row[c] = csub(row[c], cmul(f, prow[c]));
        }
        // Position bookkeeping of the emulated swap of rows k and bpos.
        const int ppos = bpos;
        if (pos == k) pos = ppos;
        if (lane == pl) pos = k, used = true;
      }
      // The row now at position i holds w_i in its right-hand side; lane r
      // collects w_r.
      SC wm = mkc<SR>(SR(0), SR(0));
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const unsigned bal = __ballot_sync(0xffffffffu, act && pos == i);
        const int src = __ffs(bal) - 1;
        const SR vx = __shfl_sync(0xffffffffu, row[M].x, src < 0 ? 0 : src);
        const SR vy = __shfl_sync(0xffffffffu, row[M].y, src < 0 ? 0 : src);
        if (lane == i) wm = mkc<SR>(vx, vy);
      }
      const bool fin = __all_sync(0xffffffffu, !act || (isfinite(wm.x) && isfinite(wm.y)));
      const SR wn = warp_allsum(act ? cabs2(wm) : SR(0));
      SC rr = mkc<SR>(r == col ? SR(-1) : SR(0), SR(0));
      SC qw = mkc<SR>(SR(0), SR(0));
      SC wall[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        wall[c] = mkc<SR>(__shfl_sync(0xffffffffu, wm.x, c), __shfl_sync(0xffffffffu, wm.y, c));
        rr = cadd(rr, cmul(a0[c], wall[c]));
        qw = cadd(qw, cmul(Q[r + c * M], wall[c]));
      }
      const SR rn = warp_allsum(act ? cabs2(rr) : SR(0));
      const SR en = warp_allsum(act ? cmulc(wm, qw).x : SR(0));
      const SR scale = SR(sqrt_approx(float(anorm * wn))) + SR(1);
      if (fin && rn <= SMath<SR>::kResidTol2 * scale * scale && en > SR(0) && isfinite(en)) {
        const SR s = SMath<SR>::rsq(en);
        if (act) {
          const SC nw = mkc<SR>(wm.x * s, wm.y * s);
          w[lane + col * M] = make_double2(double(nw.x), double(nw.y));
        }
        if (lane == col) {
#pragma unroll
          for (int k = 0; k < M; ++k) wcol[k] = mkc<SR>(wall[k].x * s, wall[k].y * s);
        }
        __syncwarp();
        break;
      }
      if (attempt >= 1) {
        bad_col = col;
        return false;
      }
      if (lane == 0) ip_perturb(w + col * M, M, rng, !restarted, seed, bin);
      restarted = true;
      __syncwarp();
      if (lane == col) {
#pragma unroll
        for (int k = 0; k < M; ++k) wcol[k] = mkc<SR>(SR(w[k + col * M].x), SR(w[k + col * M].y));
      }
      __syncwarp();
    }
  }
  return true;
}

}  // namespace ffca
