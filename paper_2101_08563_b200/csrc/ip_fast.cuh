// ip_fast.cuh -- the IP sweep of ip_update_w (reference src/fastfca.cpp:36-72)
// as a short dependent chain, for the large-bin kernel.
//
// The reference solves, column by column, (W^H Q_m) w = e_m with an LU
// factorisation of W^H Q_m (W holding the columns already updated this
// sweep), then normalises w by sqrt(w^H Q_m w).  Equivalently, with
// V = W^{-H} and v_m its column m,
//     w   = Q_m^{-1} v_m,   s^2 = w^H Q_m w = w^H v_m,   w_m <- w / s,
// and the rank-one change of column m of W moves V by Sherman-Morrison:
//     V <- V - v_m (w_m^H V - e_m^T) / s
// (w_m^H v_m = s and w_old^H V = e_m^T, so the denominator 1 + delta^H v_m
// is s).  The M inverses Q_m^{-1} do not depend on W, so they are computed in
// parallel before the sweep (8-lane warp segments, Gauss-Jordan on the
// Hermitian positive definite Q_m), together with V = (W^H)^{-1} (partial
// pivoting, whose pivots also give log|det W|^2).  The sequential part per
// column is then a mat-vec, a dot product and a rank-one update on M lanes.
// The column change multiplies det W by s, so log|det W_new|^2 =
// log|det W_old|^2 + sum_m log s_m^2 (sigmodel.cpp:118-129) comes for free.
//
// Acceptance: every s_m^2 finite and > 0 (the reference's energy test) and
// every inverse finite.  Otherwise the caller reruns the sweep through the
// reference's column solves with the residual test and the seeded restart
// (ip_update_warp_reg) from the saved W.
#pragma once

#include "common.cuh"
#include "serial_math.cuh"

namespace ffca {

template <int M, typename SR>
struct IpFastScratch {
  cplx_t<SR> qinv[M][M * M];  // row-major Q_m^{-1}
  cplx_t<SR> V[M * M];        // row-major (W^H)^{-1}
  double logdet_old;
  int ok;
};

// Width-M segment shuffle helpers.
template <typename SR>
__device__ __forceinline__ cplx_t<SR> shfl_c(cplx_t<SR> v, int src, int width) {
  return mkc<SR>(__shfl_sync(0xffffffffu, v.x, src, width), __shfl_sync(0xffffffffu, v.y, src, width));
}

// Preparation, called by EVERY warp of the CTA (roles by warp index):
//   warps [0, M/SEG): Q_m^{-1}, SEG = 32/M matrices per warp (lane segment per m);
//   warp  M/SEG     : applies the pending balance column scales to W, saves W,
//                     V = (W^H)^{-1} and log|det W|^2.
// The caller synchronises the CTA afterwards.
// Lane segments are ML = pow2ceil(M) wide; for M not a power of two the
// systems are padded with identity rows / columns (block-diagonal, so the
// M x M blocks of the inverses are the inverses of the blocks).
template <int M, typename SR, typename B>
__device__ void ip_fast_prep(int warp, int lane, double2* Wd, const B* wsc, const double* qraw,
                             double invT, IpFastScratch<M, SR>* sc, double2* wsave) {
  using SC = cplx_t<SR>;
  constexpr int ML = Pow2Ceil<M>::value;
  static_assert(32 % ML == 0, "segments");
  constexpr int SEG = 32 / ML;                 // matrices per warp
  constexpr int QW = (M + SEG - 1) / SEG;      // warps inverting Q
  const int r = lane % ML;                     // row of this lane (rows >= M: padding)
  if (warp < QW) {
    const int m = warp * SEG + lane / ML;
    const bool act = m < M;
    const double* q = qraw + (act ? m : 0) * M * M;
    SC row[2 * ML];
#pragma unroll
    for (int c = 0; c < ML; ++c) {
      SR re, im;
      if (r >= M || c >= M) {
        re = (c == r) ? SR(1) : SR(0), im = SR(0);
      } else if (c == r) {
        re = SR(q[r * M + r] * invT), im = SR(0);
      } else if (r < c) {
        re = SR(q[r * M + c] * invT), im = SR(q[c * M + r] * invT);
      } else {
        re = SR(q[c * M + r] * invT), im = SR(-q[r * M + c] * invT);
      }
      row[c] = mkc<SR>(re, im);
      row[ML + c] = mkc<SR>(c == r ? SR(1) : SR(0), SR(0));
    }
    // Gauss-Jordan without pivoting (Q_m Hermitian positive definite).
#pragma unroll
    for (int k = 0; k < M; ++k) {
      SC pk[2 * ML];
#pragma unroll
      for (int c = k; c < 2 * ML; ++c) pk[c] = shfl_c<SR>(row[c], k, ML);
      const SR pm = cabs2(pk[k]);
      const SR s = SMath<SR>::rcp(pm);
      const SC ipiv = mkc<SR>(pk[k].x * s, -pk[k].y * s);
#pragma unroll
      for (int c = k + 1; c < 2 * ML; ++c) pk[c] = cmul(pk[c], ipiv);
      if (r == k) {
#pragma unroll
        for (int c = k + 1; c < 2 * ML; ++c) row[c] = pk[c];
      } else {
        const SC f = row[k];
#pragma unroll
        for (int c = k + 1; c < 2 * ML; ++c) row[c] = csub(row[c], cmul(f, pk[c]));
      }
    }
    if (act && r < M) {
#pragma unroll
      for (int c = 0; c < M; ++c) sc->qinv[m][r * M + c] = row[ML + c];
    }
  } else if (warp == QW) {
    // Pending balance scales on the fp64 master (fastfca.cpp:139-141), saved
    // for the fallback sweep.
    for (int k = lane; k < M * M; k += 32) {
      const double c = double(wsc[k / M]);
      double2 w = Wd[k];
      w.x *= c;
      w.y *= c;
      Wd[k] = w;
      wsave[k] = w;  // W at the start of the sweep: the fallback's input
    }
    __syncwarp();
    // V = (W^H)^{-1}: Gauss-Jordan with partial pivoting on lanes [0, M)
    // (row r of W^H = conj of column r of W), rows chosen in place.
    const bool act = lane < M;
    SC row[2 * ML];
#pragma unroll
    for (int c = 0; c < ML; ++c) {
      if (r < M && c < M) {
        const double2 w = Wd[c + r * M];
        row[c] = mkc<SR>(SR(w.x), SR(-w.y));
      } else {
        row[c] = mkc<SR>(c == r ? SR(1) : SR(0), SR(0));
      }
      row[ML + c] = mkc<SR>(c == r ? SR(1) : SR(0), SR(0));
    }
    // Padding rows never compete for a pivot (their columns < M are zero and
    // the steps stop at M); lanes >= ML run duplicate copies in their segments.
    bool used = r >= M;
    int step = -1;  // the step at which this row was the pivot
    double ld = 0.0;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      SR best = used ? SR(-1) : cabs2(row[k]);
      int bl = lane;
#pragma unroll
      for (int o = ML / 2; o > 0; o >>= 1) {
        const SR ob = __shfl_xor_sync(0xffffffffu, best, o, ML);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o, ML);
        if (ob > best || (ob == best && ol < bl)) best = ob, bl = ol;
      }
      const int pl = bl % ML;
      SC pk[2 * ML];
#pragma unroll
      for (int c = k; c < 2 * ML; ++c) pk[c] = shfl_c<SR>(row[c], pl, ML);
      const SR pm = cabs2(pk[k]);
      if (!(pm > SR(0)) || !isfinite(pm)) ok = false;
      ld += SMath<SR>::log_d(pm);
      const SR s = SMath<SR>::rcp(pm);
      const SC ipiv = mkc<SR>(pk[k].x * s, -pk[k].y * s);
#pragma unroll
      for (int c = k + 1; c < 2 * ML; ++c) pk[c] = cmul(pk[c], ipiv);
      if (r == pl) {
#pragma unroll
        for (int c = k + 1; c < 2 * ML; ++c) row[c] = pk[c];
        used = true;
        step = k;
      } else {
        const SC f = row[k];
#pragma unroll
        for (int c = k + 1; c < 2 * ML; ++c) row[c] = csub(row[c], cmul(f, pk[c]));
      }
    }
    // Row chosen at step k carries row k of the inverse in its right half.
    if (act && step >= 0) {
#pragma unroll
      for (int c = 0; c < M; ++c) sc->V[step * M + c] = row[ML + c];
    }
    if (lane == 0) {
      sc->logdet_old = ld;
      sc->ok = ok ? 1 : 0;
    }
  }
}

// The sequential sweep (one warp; lanes [0, M) active).  Writes the new
// columns into Wd and returns false on a failed acceptance test (Wd then
// holds partial results: the caller restores the saved W).
template <int M, typename SR>
__device__ bool ip_fast_sweep(int lane, double2* Wd, IpFastScratch<M, SR>* sc, double& logdet_new) {
  using SC = cplx_t<SR>;
  constexpr int ML = Pow2Ceil<M>::value;
  const int j = lane % ML < M ? lane % ML : 0;  // padding lanes shadow row / column 0
  const bool live = lane % ML < M;
  SC vcol[M];  // column j of V
#pragma unroll
  for (int i = 0; i < M; ++i) vcol[i] = sc->V[i * M + j];
  bool ok = sc->ok != 0;
  double lsum = 0.0;
#pragma unroll 1
  for (int m = 0; m < M; ++m) {
    SC vm[M];
#pragma unroll
    for (int i = 0; i < M; ++i) vm[i] = shfl_c<SR>(vcol[i], m, ML);
    // lane i: w_i = sum_c Q_m^{-1}(i, c) v_m(c)
    const SC* qi = sc->qinv[m] + j * M;
    SC w = mkc<SR>(SR(0), SR(0));
#pragma unroll
    for (int c = 0; c < M; ++c) w = cadd(w, cmul(qi[c], vm[c]));
    // Re(conj(w_j) v_m(j)) for this lane's row j, summed over the rows
    SC vj = vm[0];
#pragma unroll
    for (int i = 1; i < M; ++i)
      if (i == j) vj = vm[i];
    SR e = live ? w.x * vj.x + w.y * vj.y : SR(0);
#pragma unroll
    for (int o = ML / 2; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o, ML);
    const bool good = isfinite(e) && e > SR(0) && isfinite(w.x) && isfinite(w.y);
    ok = ok && __all_sync(0xffffffffu, good);
    const SR is = SMath<SR>::rsq(e);
    const SC wn = mkc<SR>(w.x * is, w.y * is);
    if (lane < M) Wd[j + m * M] = make_double2(double(wn.x), double(wn.y));
    lsum += SMath<SR>::log_d(e);
    // r_j = w_new^H v_j ; V(:, j) -= v_m (r_j - [j == m]) / s
    SC wp[M];
#pragma unroll
    for (int i = 0; i < M; ++i) wp[i] = shfl_c<SR>(wn, i, ML);
    SC rj = mkc<SR>(SR(0), SR(0));
#pragma unroll
    for (int i = 0; i < M; ++i) rj = cadd(rj, cmulc(wp[i], vcol[i]));
    if (j == m) rj.x -= SR(1);
    const SC f = mkc<SR>(rj.x * is, rj.y * is);
#pragma unroll
    for (int i = 0; i < M; ++i) vcol[i] = csub(vcol[i], cmul(vm[i], f));
  }
  __syncwarp();
  logdet_new = sc->logdet_old + lsum;
  return ok;
}

}  // namespace ffca
