// fit_big.cuh -- the large-bin FastFCA IP+EM fit kernel (BASELINE config 3:
// M = 8 channels, N = 12 sources, T = 8000 frames per bin).
//
// Same per-bin algorithm as fit_kernel.cuh (one CTA group owns one frequency
// problem for every iteration of fastfca_fit, reference src/fastfca.cpp:
// 158-184), re-laid-out for bins whose records do not fit one SM:
//
//  * Per-frame state is split between shared memory and registers so a bin
//    needs as few SMs as possible (the per-iteration serial chain -- 13
//    reductions and the IP sweep -- is paid once per SM group, so fewer SMs
//    per bin means more bins in flight and less idle time):
//      H   [NHP planes][t] 16-byte vectors   shared   (persistent, in/out)
//      U   [NUP planes][t] 16-byte vectors   shared   (|W^H x|^2, then 1/sigma^2)
//      Phi [SLOTS][M]                        registers (posterior of the
//                                            current source, sweep to sweep)
//      x   [t][M] complex                    global (L2-resident: ~0.5 MB per
//                                            bin, read twice per iteration)
//    For c3 in fp32 that is 215 KB of shared memory per CTA and a 3-CTA
//    cluster per bin (448 threads x 6 frame slots = 2688 frames per CTA).
//  * Two thread-to-frame mappings.  The EM sweeps and the variance pass use
//    one thread per frame (SLOTS frames per thread, fixed across sweeps so the
//    posterior stays in registers).  The two passes that read x use M lanes
//    per frame: the decorrelation pass (lane j owns channel j: y_j = w_j^H x
//    with w_j in registers) and the weighted-covariance pass, where lane a
//    forms the products x_a conj(x_{a+d mod M}), d = 0..M/2 -- every entry of
//    the Hermitian outer product exactly once (the d = M/2 products of lanes
//    a >= M/2 are the only duplicates) -- and accumulates them against all M
//    weights 1/sigma^2_m (a [M x T] . [T x M^2] product with no recomputed
//    outer products).
//
// Per iteration (fastfca.cpp:172-183):
//   IP       warp 0: ip_update_warp_reg (serial_math.cuh), the reference's
//            column sweep with the seeded restart (fastfca.cpp:36-72), on the
//            cluster-reduced weighted covariances.
//   U        decorrelated powers U = |W^H x|^2 (sigmodel.cpp:93-107).
//   EM       N sweeps (em_update_lh, fastfca.cpp:80-99): sweep n finishes H
//            row n-1 from the registered posterior and the freshly reduced L
//            column, forms the posterior of source n and reduces its L column.
//   balance  every warp, lane-parallel (fastfca.cpp:127-142); H row scales
//            are folded into the effective loadings (lazy), W column scales
//            into the next IP.
//   A1       finishes H row N-1, sigma^2 = L H + eps, the NLL terms of the
//            iterate (sigmodel.cpp:155-162) and 1/sigma^2 (stored over U).
//   A2       the M weighted covariances Q_m (fastfca.cpp:22-34).
// Reductions: warp shuffles -> per-warp partials -> CTA totals in a fixed
// order -> cluster totals in rank order (DSMEM), so every CTA of a bin holds
// bit-identical per-bin scalars and runs the identical serial algebra.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "fit_kernel.cuh"
#include "serial_math.cuh"

namespace ffca {

// Shared-memory carve-up of a big-bin CTA (byte offsets), computed on the host.
struct BigLayout {
  int off_h, off_u, ps;  // planes: ps 16-byte vectors per plane
  int off_le, off_ld, off_hsc, off_hinv, off_linv, off_us, off_wsc, off_hsum, off_psum;
  int off_wd, off_wr, off_q, off_ipscr, off_ldscr, off_red, off_cx, off_scal;
  int off_gscr, off_ex, off_rng;  // inside the U region (dead while used)
  int total;
  int csize, tcap;
};

template <typename R> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

template <int M, int N, typename R, int SLOTS, int NTHR, int MS>
struct BigCfg {
  static constexpr int VE = Vec16<R>::n;           // reals per 16-byte vector
  static constexpr int NHP = (N + VE - 1) / VE;    // H planes
  static constexpr int NUP = M / VE;               // U planes
  static constexpr int NW = NTHR / 32;
  static constexpr int TCAP = NTHR * SLOTS;        // frames per CTA
  static constexpr int D = M / 2;                  // cyclic product distances
  static constexpr int NP = 1 + 2 * D;             // reals per covariance lane
  static constexpr int MW = M / MS;                // weights per covariance lane
  static constexpr int KA = NP * MW;               // accumulators per covariance lane
  static constexpr int GS = M * MS;                // covariance lanes per frame
  static constexpr int KRED = 2 * M + 1;           // EM sweep partials
  static constexpr int KQ = M * M * M + M + 1;     // covariance + NLL totals
  static_assert(M % VE == 0, "channel planes");
  static_assert(32 % GS == 0 && 32 % M == 0, "lanes per frame must divide a warp");
  static_assert(NTHR % 32 == 0, "whole warps");

  static int al(int v) { return (v + 15) & ~15; }
  static BigLayout layout(int csize) {
    BigLayout L{};
    L.csize = csize;
    L.tcap = TCAP;
    // plane stride = TCAP + 4 vectors: consecutive planes start 16 banks apart,
    // so the decorrelation pass's scalar stores (4 frames x 2 planes per warp)
    // are conflict-free.
    L.ps = TCAP + ((TCAP % 8 == 0) ? 4 : (12 - TCAP % 8) % 8);
    int o = 0;
    L.off_h = o; o = al(o + NHP * L.ps * 16);
    L.off_u = o; o = al(o + NUP * L.ps * 16);
    const int rs = int(sizeof(R));
    L.off_le = o; o = al(o + N * M * rs);
    L.off_ld = o; o = al(o + 2 * M * N * rs);
    L.off_hsc = o; o = al(o + 2 * N * rs);
    L.off_hinv = o; o = al(o + 2 * N * rs);
    L.off_linv = o; o = al(o + M * rs);
    L.off_us = o; o = al(o + M * rs);
    L.off_wsc = o; o = al(o + M * rs);
    L.off_hsum = o; o = al(o + N * rs);
    L.off_psum = o; o = al(o + M * rs);
    L.off_wd = o; o = al(o + M * M * 16);
    L.off_wr = o; o = al(o + M * M * 2 * rs);
    L.off_q = o; o = al(o + M * M * M * 8);
    L.off_ipscr = o; o = al(o + M * M * 2 * rs);
    L.off_ldscr = o; o = al(o + M * (M + 1) * 2 * rs);
    L.off_red = o; o = al(o + 2 * NW * KRED * rs);
    L.off_cx = o; o = al(o + 2 * csize * KRED * 8);
    L.off_scal = o; o = al(o + 128);
    L.total = o;
    // Inside the U region: covariance scratch, the CTA totals (read by the
    // other CTAs of the cluster) and the IP restart generator.
    L.off_gscr = L.off_u;
    L.off_ex = al(L.off_gscr + NW * GS * KA * int(sizeof(R)));
    L.off_rng = al(L.off_ex + (KQ + M + 1) * 8);
    return L;
  }
  static bool fits_u(const BigLayout& L) {
    return L.off_rng + int(sizeof(RestartRng)) <= L.off_u + NUP * L.ps * 16;
  }
};

struct BigScalars {
  double eps, nll0, logdet0, logs;
  int stop, status, ldok;
};

// Fixed-order pairwise sum of the per-warp partials red[w*K + k], w < NW
// (any NW; tree_sum_warps assumes a power of two).
template <int NW, typename T>
__device__ __forceinline__ T tree_sum_any(const T* red, int K, int k) {
  T v[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) v[w] = red[w * K + k];
#pragma unroll
  for (int h = 1; h < NW; h <<= 1)
#pragma unroll
    for (int w = 0; w + h < NW; w += 2 * h) v[w] += v[w + h];
  return v[0];
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int M, int N, typename R, int SLOTS, int NTHR, int MS, bool CL>
__global__ void __launch_bounds__(NTHR, 1) big_fit_kernel(FitParams p, BigLayout lay) {
  using Cfg = BigCfg<M, N, R, SLOTS, NTHR, MS>;
  using C = cplx_t<R>;
  using V = typename Vec16<R>::type;
  constexpr int VE = Cfg::VE, NHP = Cfg::NHP, NUP = Cfg::NUP, NW = Cfg::NW;
  constexpr int D = Cfg::D, NP = Cfg::NP, MW = Cfg::MW, KA = Cfg::KA, GS = Cfg::GS;
  constexpr int KRED = Cfg::KRED;
  using B = R;
  using BM = SMath<B>;
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int crank = 0, csize = 1;
  if constexpr (CL) {
    const cg::cluster_group cl = cg::this_cluster();
    crank = int(cl.block_rank());
    csize = int(cl.num_blocks());
  }
  const int b = CL ? blockIdx.x / csize : blockIdx.x;
  const int T = p.T;
  const int t0g = int((long long)T * crank / csize);
  const int Tl = int((long long)T * (crank + 1) / csize) - t0g;
  const bool lead = crank == 0;
  const int ps = lay.ps;
  // Phase timing (diagnostics build, -DFFCA_PHASE_TIMING): thread 0 of each
  // CTA accumulates clock64 deltas; CTA rank 0 reports them per bin.
  // 0 U pass, 1 EM frames, 2 EM reduce/update, 3 balance, 4 A1, 5 A2 frames,
  // 6 A2 reduce, 7 IP, 8 iteration sync, 9 init.
#ifdef FFCA_PHASE_TIMING
  unsigned long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tlast = clock64();
#define FFCA_BTIC(k)                               \
  do {                                             \
    if (tid == 0) {                                \
      const unsigned long long now_ = clock64();   \
      tacc[k] += now_ - tlast;                     \
      tlast = now_;                                \
    }                                              \
  } while (0)
#else
#define FFCA_BTIC(k) \
  do {               \
  } while (0)
#endif

  V* Hp = reinterpret_cast<V*>(smem + lay.off_h);
  V* Up = reinterpret_cast<V*>(smem + lay.off_u);
  R* Hs = reinterpret_cast<R*>(Hp);
  R* Us = reinterpret_cast<R*>(Up);
  R* Le = reinterpret_cast<R*>(smem + lay.off_le);  // [N][M]: column n at Le + n M
  B* const Ld0 = reinterpret_cast<B*>(smem + lay.off_ld);
  B* const hsc0 = reinterpret_cast<B*>(smem + lay.off_hsc);
  B* const hinv0 = reinterpret_cast<B*>(smem + lay.off_hinv);
  R* Linv = reinterpret_cast<R*>(smem + lay.off_linv);
  B* us = reinterpret_cast<B*>(smem + lay.off_us);
  B* wsc = reinterpret_cast<B*>(smem + lay.off_wsc);
  B* hsumv = reinterpret_cast<B*>(smem + lay.off_hsum);
  B* psum = reinterpret_cast<B*>(smem + lay.off_psum);
  double2* Wd = reinterpret_cast<double2*>(smem + lay.off_wd);
  C* Wr = reinterpret_cast<C*>(smem + lay.off_wr);
  double* qraw = reinterpret_cast<double*>(smem + lay.off_q);
  C* ipscr = reinterpret_cast<C*>(smem + lay.off_ipscr);
  C* ldscr = reinterpret_cast<C*>(smem + lay.off_ldscr);
  R* red = reinterpret_cast<R*>(smem + lay.off_red);
  double* cx = reinterpret_cast<double*>(smem + lay.off_cx);
  BigScalars* sc = reinterpret_cast<BigScalars*>(smem + lay.off_scal);
  R* gscr = reinterpret_cast<R*>(smem + lay.off_gscr);
  double* ex = reinterpret_cast<double*>(smem + lay.off_ex);
  RestartRng* rng = reinterpret_cast<RestartRng*>(smem + lay.off_rng);
  B* Ld = Ld0;
  B* hsc = hsc0;
  B* hinv = hinv0;
  int par = 0;

  const C* xg = reinterpret_cast<const C*>(p.x) + (size_t(b) * T + t0g) * M;
  R* Hg = reinterpret_cast<R*>(p.H) + (size_t(b) * T + t0g) * N;

  // ---- load the bin: H into planes (pad entries 0), W, L, scalars.
  for (int k = tid; k < NHP * VE * Tl; k += NTHR) {
    const int t = k / (NHP * VE), e = k - t * (NHP * VE);
    Hs[((e / VE) * ps + t) * VE + (e % VE)] = e < N ? Hg[size_t(t) * N + e] : R(0);
  }
  for (int k = tid; k < M * M; k += NTHR) {
    const double2 w = p.W[size_t(b) * M * M + k];
    Wd[k] = w;
    Wr[k] = mkc<R>(R(w.x), R(w.y));
  }
  for (int k = tid; k < M * N; k += NTHR) {
    const double l = p.L[size_t(b) * M * N + k];
    Ld[k] = narrow_pos<B>(l);
    Le[k] = narrow_pos<R>(l);  // col-major m + n M == [n][m]
  }
  for (int k = tid; k < N; k += NTHR) hsc[k] = B(1), hinv[k] = B(1);
  for (int k = tid; k < M; k += NTHR) us[k] = B(1), wsc[k] = B(1);
  const double power = p.power[b];
  if (tid == 0) {
    sc->eps = fmax(1e-8 * power, 1e-300);  // var_eps, sigmodel.hpp:29-31
    sc->stop = 0;
    sc->status = kStatusOk;
    sc->ldok = 1;
    sc->logs = 0.0;
  }
  __syncthreads();
  const R eps = R(sc->eps);
  const double invT = 1.0 / double(T);
  const int bin_index = (p.seed_bin0 + b) % p.F;  // mix_seed index (fastfca.cpp:40)
  const bool record = p.record != 0;
  const bool silent = !(power > 0.0);
  const bool bal = p.normalize != 0;

  // ---- cluster helpers
  auto cl_sync = [&]() {
    if constexpr (CL) {
      cluster_arrive();
      cluster_wait();
    }
  };

  // ---- frame records, thread-per-frame mapping
  auto load_h = [&](int t, R (&h)[NHP * VE]) {
#pragma unroll
    for (int q = 0; q < NHP; ++q) {
      const V v = Hp[q * ps + t];
      if constexpr (VE == 4) {
        h[q * 4] = v.x, h[q * 4 + 1] = v.y, h[q * 4 + 2] = v.z, h[q * 4 + 3] = v.w;
      } else {
        h[q * 2] = v.x, h[q * 2 + 1] = v.y;
      }
    }
  };
  auto load_u = [&](int t, R (&u)[M]) {
#pragma unroll
    for (int q = 0; q < NUP; ++q) {
      const V v = Up[q * ps + t];
      if constexpr (VE == 4) {
        u[q * 4] = v.x, u[q * 4 + 1] = v.y, u[q * 4 + 2] = v.z, u[q * 4 + 3] = v.w;
      } else {
        u[q * 2] = v.x, u[q * 2 + 1] = v.y;
      }
    }
  };
  auto store_u = [&](int t, const R (&u)[M]) {
#pragma unroll
    for (int q = 0; q < NUP; ++q) {
      V v;
      if constexpr (VE == 4) {
        v.x = u[q * 4], v.y = u[q * 4 + 1], v.z = u[q * 4 + 2], v.w = u[q * 4 + 3];
      } else {
        v.x = u[q * 2], v.y = u[q * 2 + 1];
      }
      Up[q * ps + t] = v;
    }
  };
  auto hidx = [&](int n, int t) { return ((n / VE) * ps + t) * VE + (n % VE); };
  // Loading column k of the effective loadings as vectors.  Volatile shared
  // loads: re-read per frame from the broadcast bank instead of being hoisted
  // into 12 x M registers the frame loops cannot afford.
  auto load_le = [&](int k, R (&l)[M]) {
    const unsigned a = unsigned(__cvta_generic_to_shared(Le + k * M));
#pragma unroll
    for (int q = 0; q < M / VE; ++q) {
      if constexpr (VE == 4) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(l[q * 4]), "=f"(l[q * 4 + 1]), "=f"(l[q * 4 + 2]), "=f"(l[q * 4 + 3])
                     : "r"(a + 16 * q));
      } else {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(l[q * 2]), "=d"(l[q * 2 + 1])
                     : "r"(a + 16 * q));
      }
    }
  };
  // Mixture variances sigma^2(m) = eps + sum_k Le(m,k) h_k.
  auto mix_var = [&](const R (&h)[NHP * VE], R (&lh)[M]) {
#pragma unroll
    for (int m = 0; m < M; ++m) lh[m] = eps;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      R l[M];
      load_le(k, l);
#pragma unroll
      for (int m = 0; m < M; ++m) lh[m] += l[m] * h[k];
    }
  };

  // Posterior of the current source, per frame slot (registers).
  R phi[SLOTS][M];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int m = 0; m < M; ++m) phi[s][m] = R(0);

  // ---------------------------------------------------- decorrelation pass --
  // U(j, t) = |w_j^H x_t|^2: M lanes per frame, lane j owns column j of W.
  auto u_pass = [&]() {
    const int j = lane % M;
    const int g = (warp * 32 + lane) / M;
    constexpr int NG = NTHR / M;
    C wc[M];
#pragma unroll
    for (int c = 0; c < M; ++c) wc[c] = Wr[c + j * M];
    R* ucol = Us + (j / VE) * ps * VE + (j % VE);
#pragma unroll 2
    for (int t = g; t < Tl; t += NG) {
      const V* xv = reinterpret_cast<const V*>(xg + size_t(t) * M);
      C xc[M];
#pragma unroll
      for (int q = 0; q < M * 2 / VE; ++q) {
        const V v = __ldg(xv + q);
        if constexpr (VE == 4) {
          xc[2 * q] = mkc<R>(v.x, v.y);
          xc[2 * q + 1] = mkc<R>(v.z, v.w);
        } else {
          xc[q] = mkc<R>(v.x, v.y);
        }
      }
      R yr = wc[0].x * xc[0].x + wc[0].y * xc[0].y;
      R yi = wc[0].x * xc[0].y - wc[0].y * xc[0].x;
#pragma unroll
      for (int c = 1; c < M; ++c) {
        yr += wc[c].x * xc[c].x + wc[c].y * xc[c].y;
        yi += wc[c].x * xc[c].y - wc[c].y * xc[c].x;
      }
      ucol[t * VE] = yr * yr + yi * yi;
    }
  };

  // ---------------------------------------------------- EM sweep n --------
  // Ends with the per-warp partials in red[par] and ONE barrier.
  auto em_sweep = [&](int n, bool phis, R* rd) {
    R linv[M];
#pragma unroll
    for (int m = 0; m < M; ++m) linv[m] = (n > 0) ? Linv[m] : R(0);
    R lc[M];  // L_n (effective), constant over the sweep
    load_le(n, lc);
    R acc[KRED];
#pragma unroll
    for (int k = 0; k < KRED; ++k) acc[k] = R(0);
    // Branch-free over the frame slots: a slot past the CTA's frame range
    // computes on frame 0 with its posterior forced to 0 and its stores and
    // sums masked (no divergent joins for the register allocator to merge).
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int t0 = tid + s * NTHR;
      const bool ok = t0 < Tl;
      const int t = ok ? t0 : 0;
      if (n > 0) {  // H row n-1 (fastfca.cpp:95-97), stored before the row is read
        R sum = phi[s][0] * linv[0];
#pragma unroll
        for (int m = 1; m < M; ++m) sum += phi[s][m] * linv[m];
        R hn1 = sum * R(1.0 / M);
        hn1 = hn1 > tiny<R>() ? hn1 : tiny<R>();
        if (ok) Hs[hidx(n - 1, t)] = hn1;
        acc[M] += ok ? hn1 : R(0);
      }
      R h[NHP * VE], u[M], lh[M];
      load_h(t, h);
      load_u(t, u);
      mix_var(h, lh);
      const R hn = Hs[hidx(n, t)];
      const R ihn = rcp_fast(hn);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const R lnhn = lc[m] * hn;
        const R gg = lnhn * rcp_fast(lh[m]);
        R ph = gg * (gg * u[m] - lnhn) + lnhn;  // G^2 U + (1 - G) L_n H_n
        ph = ok ? ph : R(0);
        phi[s][m] = ph;
        acc[m] += ph * ihn;
        if (phis) acc[M + 1 + m] += ph;
      }
    }
    if (phis) {
      warp_reduce_store<KRED>(acc, rd + warp * KRED, lane);
    } else {
      R a1[M + 1];
#pragma unroll
      for (int k = 0; k <= M; ++k) a1[k] = acc[k];
      warp_reduce_store<M + 1>(a1, rd + warp * KRED, lane);
    }
    __syncthreads();
  };

  // CTA totals of K partials (lane k), then cluster totals in rank order.
  // Every warp calls this; returns lane k's total (0 for k >= K).
  auto reduce_tot = [&](const R* rd, int K, int cbuf) -> R {
    R tot = (lane < K) ? tree_sum_any<NW>(rd, KRED, lane) : R(0);
    if constexpr (CL) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      double* slot = cx + cbuf * (csize * KRED) + crank * KRED;
      if (warp == 0 && lane < K)
        for (int r = 0; r < csize; ++r) cl.map_shared_rank(slot, r)[lane] = double(tot);
      cl_sync();
      double s = 0.0;
      if (lane < K)
        for (int r = 0; r < csize; ++r) s += cx[cbuf * (csize * KRED) + r * KRED + lane];
      tot = R(s);
    }
    return tot;
  };

  // ------------------------------------------------------ A1: variances --
  // finish: store H row N-1 first.  Accumulates sum_t U r per channel and
  // sum log2 sigma^2 into nacc; writes r = 1/sigma^2 over U.
  auto a1_pass = [&](bool finish, R (&nacc)[M + 1]) {
    R linv[M];
#pragma unroll
    for (int m = 0; m < M; ++m) linv[m] = finish ? Linv[m] : R(0);
#pragma unroll
    for (int k = 0; k <= M; ++k) nacc[k] = R(0);
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int t0 = tid + s * NTHR;
      const bool ok = t0 < Tl;
      const int t = ok ? t0 : 0;
      if (finish) {
        R sum = phi[s][0] * linv[0];
#pragma unroll
        for (int m = 1; m < M; ++m) sum += phi[s][m] * linv[m];
        R hn1 = sum * R(1.0 / M);
        hn1 = hn1 > tiny<R>() ? hn1 : tiny<R>();
        if (ok) Hs[hidx(N - 1, t)] = hn1;
      }
      R h[NHP * VE], u[M], lh[M];
      load_h(t, h);
      load_u(t, u);
      mix_var(h, lh);
      R r[M];
      R lsum = R(0);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        r[m] = rcp_fast(lh[m]);
        nacc[m] += ok ? u[m] * r[m] : R(0);
        lsum += flog2_ftz(lh[m]);
      }
      nacc[M] += ok ? lsum : R(0);
      if (ok) store_u(t, r);
    }
  };

  // ------------------------------------------ A2: weighted covariances --
  // Lane a of a frame's GS lanes forms x_a conj(x_{a+d}), d = 0..M/2, and
  // accumulates them against weights [mh*MW, (mh+1)*MW).  Then reduces the
  // products (and the NLL partials) to CTA totals in ex[], cluster totals in
  // qraw[] (packed Hermitian, the layout ip_update_warp_reg reads) and res.
  auto a2_pass = [&](bool want_q, const R (&nacc)[M + 1], double (&nll_tot)[M + 1]) {
    const int a = lane % M, mh = (lane / M) % MS;
    const int g = (warp * 32 + lane) / GS;
    constexpr int NG = NTHR / GS;
    R acc[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) acc[k] = R(0);
    int coff[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) coff[d] = (a + d) % M;
    if (want_q) {
#pragma unroll 2
      for (int t = g; t < Tl; t += NG) {
        const C* xf = xg + size_t(t) * M;
        C xr[D + 1];
#pragma unroll
        for (int d = 0; d <= D; ++d) xr[d] = xf[coff[d]];
        R rr[MW];
        {
          const V* rv = Up + t;
#pragma unroll
          for (int q = 0; q < MW / VE; ++q) {
            const V v = rv[(mh * MW / VE + q) * ps];
            if constexpr (VE == 4) {
              rr[q * 4] = v.x, rr[q * 4 + 1] = v.y, rr[q * 4 + 2] = v.z, rr[q * 4 + 3] = v.w;
            } else {
              rr[q * 2] = v.x, rr[q * 2 + 1] = v.y;
            }
          }
        }
        R P[NP];
        P[0] = xr[0].x * xr[0].x + xr[0].y * xr[0].y;
#pragma unroll
        for (int d = 1; d <= D; ++d) {
          // x_a conj(x_c): Re = ar cr + ai ci, Im = ai cr - ar ci
          P[2 * d - 1] = xr[0].x * xr[d].x + xr[0].y * xr[d].y;
          P[2 * d] = xr[0].y * xr[d].x - xr[0].x * xr[d].y;
        }
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
          for (int mm = 0; mm < MW; ++mm) acc[j * MW + mm] += P[j] * rr[mm];
      }
    }
    FFCA_BTIC(5);
    // Lanes of equal role (lane mod GS) hold partials of the same products:
    // reduce-scatter over the groups of the warp.
    constexpr int GPW = 32 / GS;  // groups per warp (power of two)
    int base = 0;
    int cnt = KA;
#pragma unroll
    for (int o = 16; o >= GS; o >>= 1) {
      const bool up = (lane & o) != 0;
      const int h2 = cnt / 2;  // KA is even for M >= 2
#pragma unroll
      for (int i = 0; i < KA / 2; ++i) {
        if (i < h2) {
          const R send = up ? acc[i] : acc[i + h2];
          const R keep = up ? acc[i + h2] : acc[i];
          acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (up) base += h2;
      cnt = h2;
    }
    (void)GPW;
    // NLL partials of A1 (thread-per-frame accumulators).
    R* rd = red;  // EM partial buffers are idle here
    warp_reduce_store<M + 1>(nacc, rd + warp * KRED, lane);
    __syncthreads();  // every warp is done reading 1/sigma^2 from U
    if (want_q) {
      // gscr[warp][role][KA] (role = lane % GS)
      R* dst = gscr + (warp * GS + (lane % GS)) * KA + base;
      for (int i = 0; i < cnt; ++i) dst[i] = acc[i];
    }
    __syncthreads();
    // CTA totals in the packed layout: ex[m*M*M + (a*M + c)] (a < c: Re at
    // a*M+c, Im at c*M+a; diagonal at a*M+a), then the NLL terms.
    constexpr int KQ = M * M * M;
    if (want_q) {
      for (int o = tid; o < GS * KA; o += NTHR) {
        const int role = o / KA, k = o - role * KA;
        const int ra = role % M, rmh = role / M;
        const int j = k / MW, mm = k - j * MW;
        const int m = rmh * MW + mm;
        double s = 0.0;
        {
          double v[NW];
#pragma unroll
          for (int w = 0; w < NW; ++w) v[w] = double(gscr[(w * GS + role) * KA + k]);
          // fixed-order pairwise tree
#pragma unroll
          for (int hh = 1; hh < NW; hh <<= 1)
#pragma unroll
            for (int w = 0; w + hh < NW; w += 2 * hh) v[w] += v[w + hh];
          s = v[0];
        }
        int idx = -1;
        double val = s;
        if (j == 0) {
          idx = ra * M + ra;
        } else {
          const int d = (j + 1) / 2;
          const bool im = (j % 2) == 0;
          const int c = (ra + d) % M;
          if (d * 2 == M && ra >= M / 2) {
            idx = -1;  // duplicate of (c, ra)
          } else if (ra < c) {
            idx = im ? c * M + ra : ra * M + c;
          } else {
            // x_ra conj(x_c) = conj(x_c conj(x_ra)), c < ra
            idx = im ? ra * M + c : c * M + ra;
            if (im) val = -val;
          }
        }
        if (idx >= 0) ex[m * M * M + idx] = val;
      }
    }
    if (warp == 0 && lane <= M) ex[KQ + lane] = double(tree_sum_any<NW>(rd, KRED, lane));
    __syncthreads();
    // Cluster totals, rank order (every CTA the same bits).
    const int nq = want_q ? KQ : 0;
    if constexpr (CL) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      cl_sync();
      for (int o = tid; o < nq + M + 1; o += NTHR) {
        const int oo = o < nq ? o : KQ + (o - nq);
        double s = 0.0;
        for (int r = 0; r < csize; ++r) s += cl.map_shared_rank(ex, r)[oo];
        if (o < nq) qraw[o] = s;
        else ex[KQ + M + 1 + (o - nq)] = s;  // cluster NLL totals after the CTA ones
      }
      cluster_arrive();  // this CTA is done reading the others' ex[]
    } else {
      for (int o = tid; o < nq; o += NTHR) qraw[o] = ex[o];
      for (int o = tid; o <= M; o += NTHR) ex[KQ + M + 1 + o] = ex[KQ + o];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k <= M; ++k) nll_tot[k] = ex[KQ + M + 1 + k];
  };

  // NLL of the current iterate.
  auto nll_value = [&](const double (&nt)[M + 1], double logdet) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < M; ++m) s += double(us[m]) * nt[m];
    return -double(T) * logdet + s + 0.69314718055994531 * nt[M];
  };

  // ------------------------------------------------ balance (all warps) --
  // fastfca.cpp:127-142, lane-parallel, into the other parity buffers.
  auto balance_all = [&](bool on) {
    const int nx = par ^ 1;
    B* hscn = hsc0 + nx * N;
    B* hinvn = hinv0 + nx * N;
    B* Ldn = Ld0 + nx * (M * N);
    for (int n = lane; n < N; n += 32) {
      B mu;
      if (n == N - 1) {
        B c = B(0);
#pragma unroll
        for (int m = 0; m < M; ++m) c += psum[m] * BM::rcp(Ld[m + n * M]);
        mu = c * B(invT / double(M));
      } else {
        mu = hsumv[n] * B(invT);
      }
      const bool v = on && mu > B(0) && isfinite(mu);
      hscn[n] = v ? BM::rcp(mu) : B(1);
      hinvn[n] = v ? mu : B(1);
    }
    __syncwarp();
    double ls = 0.0;
    if (lane < M) {
      const int m = lane;
      B s = B(0);
      for (int n = 0; n < N; ++n) s += Ld[m + n * M] * hinvn[n];
      s *= B(1.0 / double(N));
      const bool v = on && s > B(0) && isfinite(s);
      us[m] = v ? BM::rcp(s) : B(1);
      wsc[m] = v ? BM::rsq(s) : B(1);
      if (v) ls = BM::log_d(s);
    }
    __syncwarp();
    for (int k = lane; k < M * N; k += 32) {
      const int m = k % M, n = k / M;
      const B l0 = Ld[k];
      B l = l0 * hinvn[n] * us[m];
      l = (l0 > B(0) && !(l > B(0))) ? tiny<B>() : l;
      Ldn[k] = l;
      const B le = l * hscn[n];
      Le[k] = R((l > B(0) && !(le > B(0))) ? tiny<B>() : le);
    }
    __syncwarp();
#pragma unroll
    for (int o = Pow2Ceil<M>::value / 2; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    if (lane == 0) sc->logs = ls;
    par = nx;
    Ld = Ldn;
    hsc = hscn;
    hinv = hinvn;
    __syncwarp();
  };

  // IP sweep (warp 0): pending balance W column scales first.
  auto run_ip = [&](unsigned long long seed) {
    for (int k = lane; k < M * M; k += 32) {
      const double c = double(wsc[k / M]);
      Wd[k].x *= c;
      Wd[k].y *= c;
    }
    __syncwarp();
    int bad = -1;
    const bool ok = ip_update_warp_reg<M, R>(Wd, qraw, invT, seed, bin_index, rng, ipscr, lane, bad);
    if (lane == 0 && !ok) {
      sc->status = kStatusIpSingular | (bad << 8);
      sc->stop = 1;
    }
    __syncwarp();
    for (int k = lane; k < M * M; k += 32) Wr[k] = mkc<R>(R(Wd[k].x), R(Wd[k].y));
  };
  auto logdet_warp = [&](double& ld) -> bool { return warp_log_abs_det2<M, R>(Wd, ldscr, lane, ld); };

  // -------------------------------------------------------------- driver --
  R nacc[M + 1];
  double ntot[M + 1];
  // Initial decorrelated powers, variances, NLL of the init and the first Q.
  u_pass();
  __syncthreads();
  a1_pass(false, nacc);
  __syncthreads();
  a2_pass(p.iters > 0 && !silent, nacc, ntot);
  if (warp == 0) {
    if (record) {
      double ld = 0.0;
      const bool ok = logdet_warp(ld);
      if (lane == 0) {
        if (!ok) {
          sc->status = kStatusSingularW;
          sc->stop = 1;
        }
        sc->nll0 = nll_value(ntot, ld);
        if (lead) p.nll[p.prob_offset + b] = sc->nll0;
      }
    }
    if (lane == 0 && silent && !sc->stop) {
      sc->status = kStatusSilent;  // parameters stay at the init (fastfca.cpp:165-170)
      sc->stop = 1;
      if (record && lead)
        for (int t = 0; t < p.iters; ++t) p.nll[size_t(t + 1) * p.nll_stride + p.prob_offset + b] = sc->nll0;
    }
    __syncwarp();
    if (!sc->stop && p.iters > 0) run_ip(p.seed);
  }
  if constexpr (CL) cluster_wait();  // pairs the arrive of a2_pass
  __syncthreads();
  FFCA_BTIC(9);
  bool touched = false;
  if (!sc->stop) {
    for (int it = 0; it < p.iters; ++it) {
      // log|det W|^2 of the IP output (warp 1, off the other warps' path).
      if (record && warp == (NW > 1 ? 1 : 0)) {
        double ld = 0.0;
        const bool ok = logdet_warp(ld);
        if (lane == 0) {
          sc->ldok = ok ? 1 : 0;
          sc->logdet0 = ld;
        }
        __syncwarp();
      }
      FFCA_BTIC(7);
      u_pass();
      __syncthreads();
      FFCA_BTIC(0);
      // EM sweeps (fastfca.cpp:80-99).  Sweep 0 is peeled so the posterior
      // registers are provably written before they are read (no live range
      // across the other passes).
      auto em_step = [&](int n) {
        const bool phis = bal && n == N - 1;
        R* rd = red + (n & 1) * NW * KRED;
        em_sweep(n, phis, rd);
        FFCA_BTIC(1);
        const int K = phis ? KRED : M + 1;
        const R tot = reduce_tot(rd, K, n & 1);
        const R hs = __shfl_sync(0xffffffffu, tot, M);
        const R pss = __shfl_down_sync(0xffffffffu, tot, M + 1);
        if (lane < M) {
          const int m = lane;
          const B l = fmax(B(tot) * B(invT) * hinv[n], tiny<B>());  // fastfca.cpp:92-94
          const R lr = R(l);
          Ld[m + n * M] = l;
          if (!phis) Le[m + n * M] = lr;
          Linv[m] = rcp_fast(lr);
          if (phis) psum[m] = B(pss);
        }
        if (lane == 0 && n >= 1) hsumv[n - 1] = B(hs);
        __syncwarp();
        FFCA_BTIC(2);
      };
      em_step(0);
      for (int n = 1; n < N; ++n) em_step(n);
      balance_all(bal);
      FFCA_BTIC(3);
      touched = true;
      const bool more = it + 1 < p.iters;
      a1_pass(true, nacc);
      __syncthreads();
      FFCA_BTIC(4);
      a2_pass(more, nacc, ntot);
      FFCA_BTIC(6);
      if (warp == 0) {
        if (lane == 0 && record) {
          if (!sc->ldok) {  // log_abs_det2 throws on a singular W (sigmodel.cpp:124-125)
            sc->status = kStatusSingularW;
            sc->stop = 1;
          }
          const double v = nll_value(ntot, sc->logdet0 - sc->logs);
          if (lead) p.nll[size_t(it + 1) * p.nll_stride + p.prob_offset + b] = v;
        }
        __syncwarp();
        if (more && !sc->stop) {
          run_ip(p.seed + (unsigned long long)(it + 1));
        } else {
          for (int k = lane; k < M * M; k += 32) {  // the last balance's W scales
            const double c = double(wsc[k / M]);
            Wd[k].x *= c;
            Wd[k].y *= c;
          }
        }
      }
      FFCA_BTIC(7);
      if constexpr (CL) cluster_wait();
      __syncthreads();
      FFCA_BTIC(8);
      if (sc->stop) break;
    }
  }
  __syncthreads();
  // ------------------------------------------------------------- epilogue --
  if (lead) {
    for (int k = tid; k < M * M; k += NTHR) p.W[size_t(b) * M * M + k] = Wd[k];
    if (touched)
      for (int k = tid; k < M * N; k += NTHR) p.L[size_t(b) * M * N + k] = double(Ld[k]);
  }
  for (int k = tid; k < N * Tl; k += NTHR) {
    const int t = k / N, n = k - t * N;
    Hg[k] = R(double(Hs[hidx(n, t)]) * double(hsc[n]));
  }
  if (tid == 0 && lead) p.status[b] = sc->status;
#ifdef FFCA_PHASE_TIMING
  if (p.timing && tid == 0 && lead)
    for (int k = 0; k < 10; ++k) p.timing[size_t(b) * 16 + k] = tacc[k];
#endif
#undef FFCA_BTIC
  if constexpr (CL) cl_sync();  // no CTA exits while others may read its shared memory
}

}  // namespace ffca
