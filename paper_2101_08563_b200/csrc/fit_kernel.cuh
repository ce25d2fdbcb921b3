// fit_kernel.cuh -- the persistent FastFCA IP+EM (and IP+MM) fit kernel.
//
// One CTA owns one frequency problem (bin i of mixture b) for ALL iterations
// of fastfca_fit (reference src/fastfca.cpp:158-184): the CTA grid replaces
// parallel_for over bins (src/parallel.cpp:16-45).  When the per-bin working
// set fits in shared memory the CTA keeps it on chip for the whole fit, so HBM
// sees x and H once; otherwise the same code streams it from global memory
// (L2/HBM) with the per-frame scratch in a global buffer.
//
// Data layout (frame-major records, the reference's own per-bin order):
//   x   [t][m]  complex   (Spectrogram::f[i] column-major, stft.hpp:21-29)
//       or, block-stationary input (BLK, block_size > 1, sigmodel.cpp:34-41):
//   X   [j][M*M] real     packed Hermitian block covariance of block j:
//                         [a*M+a] = X_aa, [a*M+c] = Re X_ac, [c*M+a] = Im X_ac
//                         (a < c) -- exactly the outer-product layout pass A
//                         forms from a snapshot, so Q accumulates it directly
//                         (fastfca.cpp:29-32) and U = max(0, w^H X w)
//                         (sigmodel.cpp:98-105).
//   H   [t][n]  real      (FastFcaParams::act[i] column-major, sigmodel.hpp:76)
//   wk  [t][2M] real      U(m) = |w_m^H x_t|^2, then Phi(m) of the current source
// so one thread reads a frame's record with a few vector loads.
//
// Per iteration (fastfca.cpp:172-183):
//   pass A   sigma^2 = L H + eps; the per-bin NLL of the previous iterate
//            (sigmodel.cpp:155-162) and all M weighted covariances Q_m
//            (fastfca.cpp:22-34), one CTA reduction.
//   IP       one thread, fp64 in registers: M sequential column solves with the
//            residual check and the libstdc++-faithful seeded restart
//            (fastfca.cpp:36-72).
//   EM       N+1 sweeps: sweep n stores U (n = 0), finishes source n-1's H row
//            from the stored Phi and the freshly reduced L column, then forms
//            Phi for source n and reduces its L column (em_update_lh,
//            fastfca.cpp:80-99).  Each sweep ends in ONE barrier: every warp
//            then sums the per-warp partials itself and applies the identical
//            L-column update (no serial section between sweeps).
//   MM       two sweeps (mm_update_lh, fastfca.cpp:101-117).
//   balance  one thread on the reduced row means (fastfca.cpp:127-142).  The H
//            row scale 1/mu_n is kept as a per-source factor hsc[n] (H_true =
//            H_stored * hsc) and folded into the effective loadings
//            Le = L * hsc used by every product, so no sweep rescales H; the
//            next H update stores true values.  The W column scale is folded
//            the same way into the stored U (us[m]).
// Reductions: multi-value warp butterflies -> per-warp partials in shared
// memory -> barrier -> fixed-order cross-warp sums.  The order is fixed for a
// launch shape, so per-bin results do not depend on how bins are sharded.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "serial_math.cuh"

namespace ffca {

// Shared-memory carve-up of one fit CTA (byte offsets).  Computed on the
// host (FitSmem below) and passed in the kernel parameters, so the kernel
// reads every offset from the constant bank instead of re-deriving the
// layout (the compiler rematerialised that chain inside the frame loops of
// register-capped variants: 15 % of the instructions of the M = 3 kernel).
struct FitLayout {
  int off_wd, off_wlg, off_wsc, off_wr, off_ld, off_le, off_linv, off_hsc, off_hinv, off_hscr,
      off_us, off_hsum,
      off_num, off_den, off_reda, off_redb, off_res, off_rng, off_cx, off_wsm, off_scal, off_big,
      off_x, off_h, off_w,  // resident records: x, H, work
      kred, kres,
      total;
};

struct FitParams {
  int nprob;        // problems in this launch (= gridDim.x)
  int N, T;         // sources, frames
  int F;            // bins per mixture (restart seed index i = (seed_bin0 + b) % F)
  int prob_offset;  // global problem index of blockIdx.x == 0 (NLL slot column)
  int seed_bin0;    // bin index of blockIdx.x == 0 within its mixture's numbering
  const void* x;    // R2 [nprob][T][M]
  void* H;          // R  [nprob][T][N]   in/out
  void* work;       // R  [nprob][T][2M]  scratch (streaming mode only)
  double2* W;       // [nprob][M*M] col-major (r + c*M), in/out
  double* L;        // [nprob][M*N] col-major (m + n*M), in/out
  const double* power;  // [nprob] SampleCovSet::power_scale
  double* nll;      // slot(t, p) at nll[t * nll_stride + prob_offset + p]; may be null
  int nll_stride;
  int* status;      // [nprob]: 0 ok, 1 silent band, 2 IP singular, 3 singular W
  int iters, flavor, record, normalize, fix_loadings, resident;
  int nc;           // MM: sources per L-reduction chunk
  int tloc;         // frames held per CTA (= T, or ceil(T/C) for a C-CTA cluster)
  int blk;          // x holds packed block covariances [nprob][T][M*M] (T = blocks)
  void* aux;        // large-bin kernel: cold-path global scratch, AUX_BYTES per CTA
  int work_total, work_first;  // host: scratch rows of the whole call and this launch's first
                               // row (pipelined chunks share one allocation); 0, 0 = nprob rows
  unsigned long long* timing;  // optional per-problem phase cycle counters [nprob][16]
  unsigned long long seed;
  FitLayout lay;
};

enum : int { kStatusOk = 0, kStatusSilent = 1, kStatusIpSingular = 2, kStatusSingularW = 3 };

// M > 4 IP: registers (ip_update_warp_reg) or shared-memory Gauss-Jordan.
#ifndef FFCA_IP_WARP_REG
#define FFCA_IP_WARP_REG 1
#endif
// Smallest M whose IP runs warp-cooperatively (below: one lane in registers).
#ifndef FFCA_IP_WARP_MIN
#define FFCA_IP_WARP_MIN 3
#endif
#ifndef FFCA_SPLIT_MIN
#define FFCA_SPLIT_MIN 5
#endif
template <int M>
struct Split {
  // M <  FFCA_SPLIT_MIN: every thread accumulates all M weighted covariances
  // (M^3 values).  Else the CTA splits into M groups of warps, group g owns
  // Q_g (M^2).
  static constexpr int MSPLIT = (M < FFCA_SPLIT_MIN) ? 1 : M;
  static constexpr int MG = M / MSPLIT;
  static constexpr int KQ = MG * M * M;          // Q values per thread
  static constexpr int KA = KQ + MG + 1;         // + sum U r per channel + sum log2 s2
};

// Launch shape: threads per CTA (upper bound) and the CTAs per SM the
// register budget must allow.  Small M: 128 threads x 4 CTAs (up to 128
// registers), so the 513 bins of a 1024-point STFT fit on 148 SMs in one
// wave; 4 warps per bin keep the per-warp share of the reductions and of the
// all-warp updates small (c1: 128 threads beat 192 by ~6%).
// M = 4 runs one CTA per SM (its pass A needs the full register file: the
// bound of 2 CTAs forced 128 registers and spilled; c2 1.84 -> 1.42 ms).
#ifndef FFCA_MINB_M3
#define FFCA_MINB_M3 4
#endif
#ifndef FFCA_MINB_M4
#define FFCA_MINB_M4 1
#endif
#ifndef FFCA_THREADS_BIG
#define FFCA_THREADS_BIG 256
#endif
#ifndef FFCA_THREADS_SMALL
#define FFCA_THREADS_SMALL 128
#endif
#ifndef FFCA_THREADS_M4
#define FFCA_THREADS_M4 FFCA_THREADS_BIG
#endif
template <int M>
struct Launch {
  static constexpr int threads =
      (M <= 3) ? FFCA_THREADS_SMALL : (M == 4 ? FFCA_THREADS_M4 : FFCA_THREADS_BIG);
  static constexpr int minb = (M <= 2) ? 4 : (M == 3 ? FFCA_MINB_M3 : (M == 4 ? FFCA_MINB_M4 : 1));
};

// Fixed-order pairwise sum of K per-warp partials red[w*K + k], w < nwarps
// <= NW (issued as independent loads; slots beyond nwarps masked to zero):
// depth log2(NW) instead of a serial chain.
template <int NW, typename T>
__device__ __forceinline__ T tree_sum_warps(const T* red, int K, int k, int nwarps) {
  T v[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) v[w] = (w < nwarps) ? red[w * K + k] : T(0);
#pragma unroll
  for (int h = NW / 2; h > 0; h >>= 1)
#pragma unroll
    for (int w = 0; w < h; ++w) v[w] += v[w + h];
  return v[0];
}

#ifndef FFCA_FRAMES_IN_FLIGHT
#define FFCA_FRAMES_IN_FLIGHT 1
#endif

// MM: sources per L-reduction chunk (2 M values each, <= 32 per warp pass).
template <int M, int NT>
struct MmChunk {
  static constexpr int nc0 = (16 / M) > 0 ? (16 / M) : 1;
  static constexpr int value = nc0 < NT ? nc0 : NT;
};

// Shared-memory carve-up, identical on host and device.
template <int M, int NT, typename R, bool BLK = false>
struct FitSmem : FitLayout {
  static constexpr int XR = BLK ? M * M : 2 * M;  // reals per x record
  __host__ __device__ static int al(int v) { return (v + 15) & ~15; }
  __host__ __device__ FitSmem(int nwarps, int N, int T, int nc, bool resident) {
    using S = Split<M>;
    kred = 2 * M + 1;  // EM sweep partials (+ Phi sums in the last sweep)
    if (2 * M * MmChunk<M, NT>::value > kred) kred = 2 * M * MmChunk<M, NT>::value;
    if (NT > kred) kred = NT;
    kres = M * M * M + M + 1;
    if (kres < kred) kres = kred;
    int o = 0;
    off_wd = o; o = al(o + M * M * 16);
    off_wlg = o; o = al(o + M * M * 16);  // W after the IP sweep (log-det input)
    off_wsc = o; o = al(o + M * 8);       // balance: W column scales
    off_wr = o; o = al(o + M * M * 2 * (int)sizeof(R));
    off_ld = o; o = al(o + 2 * M * NT * 8);  // parity double-buffered (balance)
    off_le = o; o = al(o + M * NT * (int)sizeof(R));
    off_linv = o; o = al(o + M * (int)sizeof(R));
    off_hsc = o; o = al(o + 2 * NT * 8);
    off_hinv = o; o = al(o + 2 * NT * 8);
    off_hscr = o; o = al(o + NT * (int)sizeof(R));
    off_us = o; o = al(o + M * 8);
    off_hsum = o; o = al(o + NT * 8);
    off_num = o; o = al(o + M * NT * 8);
    off_den = o; o = al(o + M * NT * 8);
    off_reda = o; o = al(o + nwarps * S::KA * 8);       // pass-A partials
    // Sweep partials, double-buffered.  The IP restart generator (cold, live
    // only inside one IP sweep, when no sweep partials are pending) shares
    // the region; the phase-timing diagnostics keep their counters there, so
    // that build gives the generator its own space.
    off_redb = o;
    {
      int rb = 2 * nwarps * kred * 8;
#ifndef FFCA_PHASE_TIMING
      if (rb < (int)sizeof(RestartRng)) rb = (int)sizeof(RestartRng);
      off_rng = o;
#endif
      o = al(o + rb);
    }
#ifdef FFCA_PHASE_TIMING
    off_rng = o; o = al(o + (int)sizeof(RestartRng));
#endif
    off_res = o; o = al(o + kres * 8);
    off_cx = o; o = al(o + 2 * kres * 8);               // cluster exchange, double-buffered
    off_wsm = o;  // warp-cooperative algebra scratch (M > 4): warp 0 then warp 1
    o = al(o + ((M > 4 || M >= FFCA_IP_WARP_MIN) ? (4 * M * M + M + M * (M + 1)) * 2 * (int)sizeof(R)
                                                  : 0));
    off_scal = o; o = al(o + 64);
    off_big = o;
    // x, H and work records, each region 16-byte aligned.
    off_x = o;
    off_h = al(off_x + T * XR * (int)sizeof(R));
    off_w = al(off_h + T * N * (int)sizeof(R));
    if (resident) o = al(off_w + T * 2 * M * (int)sizeof(R));
    total = o;
  }
};

// The kernel's view of its layout: M <= 2 derives it in registers (measured
// faster for c1: 0.655 vs 0.677 ms), larger M reads the host-computed copy in
// the kernel parameters (c4: 46.9 -> 40.5 ms per 10 iterations).
template <bool LOCAL, int M, int NT, typename R, bool BLK, typename P>
__device__ __forceinline__ decltype(auto) fit_layout(const P& p, int nwarps, int N, bool res) {
  if constexpr (LOCAL)
    return FitSmem<M, NT, R, BLK>(nwarps, N, p.tloc, p.nc, res);
  else
    return (p.lay);
}

struct Scalars {
  double eps, nll0, logdet0, logs;
  int stop, status, ldok;
};

// --------------------------------------------------------- vector records --
template <int K, typename R>
__device__ __forceinline__ void ld_rec(const R* p, R (&v)[K]) {
  if constexpr (sizeof(R) == 4 && K % 4 == 0) {
#pragma unroll
    for (int k = 0; k < K; k += 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + k);
      v[k] = q.x, v[k + 1] = q.y, v[k + 2] = q.z, v[k + 3] = q.w;
    }
  } else if constexpr (K % 2 == 0) {
    using V2 = typename Cplx<R>::type;
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      const V2 q = *reinterpret_cast<const V2*>(p + k);
      v[k] = q.x, v[k + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = p[k];
  }
}

template <int K, typename R>
__device__ __forceinline__ void st_rec(R* p, const R (&v)[K]) {
  if constexpr (sizeof(R) == 4 && K % 4 == 0) {
#pragma unroll
    for (int k = 0; k < K; k += 4)
      *reinterpret_cast<float4*>(p + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
  } else if constexpr (K % 2 == 0) {
    using V2 = typename Cplx<R>::type;
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      V2 q;
      q.x = v[k], q.y = v[k + 1];
      *reinterpret_cast<V2*>(p + k) = q;
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = v[k];
  }
}

// Small uniform per-bin parameters: copied into registers at the top of a
// pass when they fit, else read from shared memory in the loop.
template <int K, bool REG, typename R>
struct Uniform {
  R v[REG ? K : 1];
  const R* s;
  __device__ __forceinline__ void load(const R* src) {
    s = src;
    if constexpr (REG) {
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = src[k];
    }
  }
  __device__ __forceinline__ R operator[](int k) const {
    if constexpr (REG) return v[k];
    else return s[k];
  }
};

// ------------------------------------------------------------------ kernel --
// CL: the bin's frames are split over a thread-block cluster (one CTA per
// frame range, cluster rank order); reductions add a DSMEM exchange and every
// CTA repeats the (identical) serial algebra, so no broadcast is needed.
// RES: the bin's records live in shared memory (compile-time, so the record
// accesses are LDS/STS rather than generic loads); !RES streams them from
// global memory (bins beyond a 16-CTA cluster).
// BLK: the records are packed block covariances (block-stationary input).
template <int M, int NT, bool EXACT, typename R, bool CL, bool RES, bool BLK = false>
__global__ void __launch_bounds__(Launch<M>::threads, Launch<M>::minb) fit_kernel(FitParams p) {
  using C = cplx_t<R>;
  using S = Split<M>;
  using Lay = FitSmem<M, NT, R, BLK>;
  constexpr int XR = Lay::XR;  // reals per x record
  constexpr int WR = 2 * M;  // reals per work record: U[M], Phi[M]
  constexpr bool HOIST = (M * NT <= 32);
  constexpr int FU = FFCA_FRAMES_IN_FLIGHT;  // frames per loop trip (ILP vs registers)
#ifdef FFCA_FRAMES_IN_FLIGHT_EM
  constexpr int FUE = FFCA_FRAMES_IN_FLIGHT_EM;  // EM sweeps (tuning experiments)
#else
  constexpr int FUE = FU;
#endif
  using WU = Uniform<2 * M * M, (2 * M * M <= 32), R>;  // W in the compute type
  extern __shared__ __align__(16) unsigned char smem[];
  const int nthreads = blockDim.x, tid = threadIdx.x, nwarps = nthreads >> 5;
  const int lane = tid & 31, warp = tid >> 5;
  const int N = EXACT ? NT : p.N;
  const int T = p.T;  // the bin's frame count (all global formulas use T)
  int crank = 0, csize = 1;
  if constexpr (CL) {
    namespace cg = cooperative_groups;
    const cg::cluster_group cl = cg::this_cluster();
    crank = int(cl.block_rank());
    csize = int(cl.num_blocks());
  }
  const int b = CL ? blockIdx.x / csize : blockIdx.x;
  const int t0g = int((long long)T * crank / csize);  // this CTA's frames [t0g, t0g + Tl)
  const int Tl = int((long long)T * (crank + 1) / csize) - t0g;
  const bool lead = crank == 0;  // writes the per-bin outputs
  const auto& lay = fit_layout<(M <= 2), M, NT, R, BLK>(p, nwarps, N, RES);
  double2* Wd = reinterpret_cast<double2*>(smem + lay.off_wd);
  double2* Wlg = reinterpret_cast<double2*>(smem + lay.off_wlg);
  // Per-bin scalar algebra (L master, balance scales, sweep updates) runs in
  // the compute type B = R: fp32 in the fp32 path (short SFU chains; every
  // value it feeds is consumed in fp32 by the frame loops anyway), fp64 in
  // the check mode.  Slots are 8 bytes either way.
  using B = R;
  using BM = SMath<B>;
  const B tinyB = tiny<B>();
  B* wsc = reinterpret_cast<B*>(smem + lay.off_wsc);
  C* Wr = reinterpret_cast<C*>(smem + lay.off_wr);
  // Ld, hsc and hinv are double-buffered by iteration parity: every warp
  // computes the balance itself and writes the other buffer, so no warp can
  // overwrite a value another warp still reads (see balance_all below).
  B* const Ld0 = reinterpret_cast<B*>(smem + lay.off_ld);
  B* const hsc0 = reinterpret_cast<B*>(smem + lay.off_hsc);
  B* const hinv0 = reinterpret_cast<B*>(smem + lay.off_hinv);
  B* Ld = Ld0;      // current L (master)
  B* hsc = hsc0;    // current lazy H row scales
  B* hinv = hinv0;  // 1 / hsc
  int par = 0;
  R* Le = reinterpret_cast<R*>(smem + lay.off_le);      // L * hsc, compute type
  R* Linv = reinterpret_cast<R*>(smem + lay.off_linv);  // 1 / L(:, n) of the new column
  R* hscr = reinterpret_cast<R*>(smem + lay.off_hscr);  // hsc in the compute type (MM)
  B* us = reinterpret_cast<B*>(smem + lay.off_us);
  B* hsumv = reinterpret_cast<B*>(smem + lay.off_hsum);
  B* numd = reinterpret_cast<B*>(smem + lay.off_num);
  B* psum = numd;  // EM: sum_t Phi(m) of the last sweep (numd is MM-only)
  B* dend = reinterpret_cast<B*>(smem + lay.off_den);
  double* reda = reinterpret_cast<double*>(smem + lay.off_reda);
  double* redb = reinterpret_cast<double*>(smem + lay.off_redb);
  double* res = reinterpret_cast<double*>(smem + lay.off_res);
  RestartRng* rng = reinterpret_cast<RestartRng*>(smem + lay.off_rng);
  Scalars* sc = reinterpret_cast<Scalars*>(smem + lay.off_scal);
  double* cx = reinterpret_cast<double*>(smem + lay.off_cx);
  const int kred = lay.kred, kres = lay.kres;
  int cxbuf = 0;
  // Cluster sum of v[0..K) (per-CTA totals in this CTA's shared memory):
  // publish, cluster barrier, add every rank's copy in rank order.  Called by
  // all threads; `who` selects the threads that need the result in out[].
  auto cluster_sum = [&](const double* v, int K, double* out, bool who) {
    if constexpr (CL) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      double* slot = cx + cxbuf * kres;
      if (warp == 0)  // v was produced by warp 0
        for (int k = lane; k < K; k += 32) slot[k] = v[k];
      cl.sync();
      if (who)
        for (int k = lane; k < K; k += 32) {
          double s = 0.0;
          for (int r = 0; r < csize; ++r) s += cl.map_shared_rank(slot, r)[k];
          out[k] = s;
        }
      cxbuf ^= 1;
      __syncwarp();
    }
  };

  // Source-loop guard: folds away when N is the compile-time NT.
#define FFCA_NK(k) (EXACT || (k) < N)

  const R* xg = reinterpret_cast<const R*>(p.x) + (size_t(b) * T + t0g) * XR;
  R* Hg = reinterpret_cast<R*>(p.H) + (size_t(b) * T + t0g) * N;
  const R* xs;
  R* Hs;
  R* wk;
  if constexpr (RES) {
    const int ox = lay.off_x, oh = lay.off_h, ow = lay.off_w;
    R* xsm = reinterpret_cast<R*>(smem + ox);
    Hs = reinterpret_cast<R*>(smem + oh);
    wk = reinterpret_cast<R*>(smem + ow);
    if constexpr (XR % 2 == 0) {
      const C* src = reinterpret_cast<const C*>(xg);
      C* dst = reinterpret_cast<C*>(xsm);
      for (int k = tid; k < (XR / 2) * Tl; k += nthreads) dst[k] = src[k];
    } else {  // odd M under BLK: records are not 8-byte aligned
      for (int k = tid; k < XR * Tl; k += nthreads) xsm[k] = xg[k];
    }
    for (int k = tid; k < N * Tl; k += nthreads) Hs[k] = Hg[k];
    xs = xsm;
  } else {
    xs = xg;
    Hs = Hg;
    wk = reinterpret_cast<R*>(p.work) + (size_t(b) * T + t0g) * WR;
  }
  for (int k = tid; k < M * M; k += nthreads) {
    const double2 w = p.W[size_t(b) * M * M + k];
    Wd[k] = w;
    Wr[k] = mkc<R>(R(w.x), R(w.y));
  }
  for (int k = tid; k < M * N; k += nthreads) {
    const double l = p.L[size_t(b) * M * N + k];
    Ld[k] = narrow_pos<B>(l);
    Le[k] = narrow_pos<R>(l);
  }
  for (int k = tid; k < NT; k += nthreads) hsc[k] = B(1), hinv[k] = B(1);
  for (int k = tid; k < M; k += nthreads) us[k] = B(1);
  bool touched = false;  // L was updated (else the caller's fp64 L is returned untouched)
  const double power = p.power[b];
  if (tid == 0) {
    sc->eps = fmax(1e-8 * power, 1e-300);  // var_eps, sigmodel.hpp:29-31
    sc->stop = 0;
    sc->status = kStatusOk;
  }
  __syncthreads();
  const R eps = R(sc->eps);
  const double invT = 1.0 / double(T);
  const bool update_loading = !p.fix_loadings;
  const int bin_index = (p.seed_bin0 + b) % p.F;  // mix_seed index (fastfca.cpp:40)
  // Phase timing: diagnostics builds only (-DFFCA_PHASE_TIMING, see build.py);
  // the counters would otherwise cost live registers across the whole kernel.
#ifdef FFCA_PHASE_TIMING
  // Counters live in shared memory (reuse of the restart-RNG scratch: cold),
  // so the probe adds no live registers to the instrumented kernel.
  unsigned long long* tacc = reinterpret_cast<unsigned long long*>(rng);
  if (tid == 0)
    for (int k = 0; k < 11; ++k) tacc[k] = 0;
  if (tid == 0) tacc[10] = clock64();
#define tlast tacc[10]
#define FFCA_TIC(k)                              \
  do {                                           \
    if (p.timing && tid == 0) {                  \
      const unsigned long long now_ = clock64(); \
      tacc[k] += now_ - tlast;                   \
      tlast = now_;                              \
    }                                            \
  } while (0)
#else
#define FFCA_TIC(k) \
  do {              \
  } while (0)
#endif

  auto load_h = [&](int t, R (&h)[NT]) {
    if constexpr (EXACT) {
      ld_rec<NT>(Hs + t * NT, h);
    } else {
#pragma unroll
      for (int k = 0; k < NT; ++k) h[k] = (k < N) ? Hs[t * N + k] : R(0);
    }
  };

  // y = W^H x and U = |y|^2 of one frame; BLK: U = max(0, w_m^H X w_m) of
  // one block from the packed Hermitian record (sigmodel.cpp:98-105).
  auto decorrelate = [&](const WU& w, const R (&xv)[XR], R (&u)[M]) {
    if constexpr (BLK) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R acc = R(0);
#pragma unroll
        for (int a = 0; a < M; ++a) {
          const R ar = w[2 * (a + m * M)], ai = w[2 * (a + m * M) + 1];
          acc += (ar * ar + ai * ai) * xv[a * M + a];
#pragma unroll
          for (int c = a + 1; c < M; ++c) {
            const R cr = w[2 * (c + m * M)], ci = w[2 * (c + m * M) + 1];
            // 2 Re(conj(w_a) X_ac w_c), conj(w_a) w_c = (ar cr + ai ci) + i (ar ci - ai cr)
            acc += R(2) * ((ar * cr + ai * ci) * xv[a * M + c] - (ar * ci - ai * cr) * xv[c * M + a]);
          }
        }
        u[m] = acc > R(0) ? acc : R(0);
      }
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R yr = w[2 * m * M] * xv[0] + w[2 * m * M + 1] * xv[1];
        R yi = w[2 * m * M] * xv[1] - w[2 * m * M + 1] * xv[0];
#pragma unroll
        for (int c = 1; c < M; ++c) {
          const R wx = w[2 * (c + m * M)], wy = w[2 * (c + m * M) + 1];
          yr += wx * xv[2 * c] + wy * xv[2 * c + 1];
          yi += wx * xv[2 * c + 1] - wy * xv[2 * c];
        }
        u[m] = yr * yr + yi * yi;
      }
    }
  };

  // Fixed-order sum of the per-warp partials red[w*K + k] (issued as
  // independent loads, then added in warp order).
  constexpr int NWMAX = Launch<M>::threads / 32;
  auto sum_warps = [&](const double* red, int K, int k) {
    return tree_sum_warps<NWMAX>(red, K, k, nwarps);
  };

  // ---------------------------------------------------------------- pass A --
  // first: U from x and the current W; else U = stored U (times us[m] after
  // the reduction).  Leaves Q_m packed in res[0, M^3), sum_t U r per channel
  // in res[M^3 + m] and sum log2 sigma^2 in res[M^3 + M] (warp 0 visible).
  // finish (EM): first completes H row N-1 of the iteration from the stored
  // Phi and Linv (em_update_lh's last H update, fastfca.cpp:95-97), so the
  // last EM sweep and the next pass A share one trip over the frames.
  auto pass_a = [&](bool first, bool want_q, bool want_nll, bool finish) {
    constexpr int MSPLIT = S::MSPLIT, MG = S::MG, KQ = S::KQ, KA = S::KA;
    const int gs = nthreads / MSPLIT;
    // g must fold to 0 for MSPLIT == 1: a runtime channel offset would index
    // the register-resident loadings dynamically (local memory).
    const int g = MSPLIT == 1 ? 0 : tid / gs, lt = tid - g * gs;
    const int m0 = g * MG;
    const int jf = N - 1;
    Uniform<M * NT, HOIST, R> le;
    le.load(Le);
    WU wr;
    if (first) wr.load(reinterpret_cast<const R*>(Wr));
    R linv[M];
#pragma unroll
    for (int m = 0; m < M; ++m) linv[m] = finish ? Linv[m] : R(0);
    const bool need_w = (want_nll && !first) || finish;
    R acc[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) acc[k] = R(0);
    // FU frames per trip: all loads first, then independent arithmetic chains.
    for (int tb = lt; tb < Tl; tb += FU * gs) {
      R xv[FU][XR], h[FU][NT], u[FU][M];
      bool ok[FU];
#pragma unroll
      for (int f = 0; f < FU; ++f) {
        const int t = tb + f * gs;
        ok[f] = t < Tl;
        const int tt = ok[f] ? t : tb;  // always a valid record
        ld_rec<XR>(xs + tt * XR, xv[f]);
        load_h(tt, h[f]);
        if (need_w) {
          R w[WR];
          ld_rec<WR>(wk + tt * WR, w);
#pragma unroll
          for (int m = 0; m < M; ++m) u[f][m] = w[m];
          if (finish) {
            R s = linv[0] * w[M];
#pragma unroll
            for (int m = 1; m < M; ++m) s += linv[m] * w[M + m];
            R hn = s * R(1.0 / M);
            hn = hn > tiny<R>() ? hn : tiny<R>();  // fastfca.cpp:96-97
#pragma unroll
            for (int k = 0; k < NT; ++k)
              if (k == jf) h[f][k] = hn;
            if (ok[f] && g == 0) Hs[tt * N + jf] = hn;
          }
        }
      }
#pragma unroll
      for (int f = 0; f < FU; ++f) {
        if (!ok[f]) continue;
        R P[M * M];
        if constexpr (BLK) {
          if (want_q) {
#pragma unroll
            for (int k = 0; k < M * M; ++k) P[k] = xv[f][k];
          }
        } else if (want_q) {
#pragma unroll
          for (int a = 0; a < M; ++a) {
            P[a * M + a] = xv[f][2 * a] * xv[f][2 * a] + xv[f][2 * a + 1] * xv[f][2 * a + 1];
#pragma unroll
            for (int c = a + 1; c < M; ++c) {
              // x_a conj(x_c)
              P[a * M + c] = xv[f][2 * a] * xv[f][2 * c] + xv[f][2 * a + 1] * xv[f][2 * c + 1];
              P[c * M + a] = xv[f][2 * a + 1] * xv[f][2 * c] - xv[f][2 * a] * xv[f][2 * c + 1];
            }
          }
        }
        if (want_nll && first) decorrelate(wr, xv[f], u[f]);
#pragma unroll
        for (int mi = 0; mi < MG; ++mi) {
          const int m = m0 + mi;
          R s2 = eps;
#pragma unroll
          for (int k = 0; k < NT; ++k)
            if (FFCA_NK(k)) s2 += le[m + k * M] * h[f][k];
          const R r = rcp_fast(s2);
          if (want_nll) {
            R um = u[f][0];
#pragma unroll
            for (int mm = 0; mm < M; ++mm)
              if (mm == m) um = u[f][mm];
            acc[KQ + mi] += um * r;
            acc[KQ + MG] += flog2_ftz(s2);
          }
          if (want_q) {
#pragma unroll
            for (int k = 0; k < M * M; ++k) acc[mi * M * M + k] += r * P[k];
          }
        }
      }
    }
    FFCA_TIC(0);
    if constexpr (KA <= 32) {
      warp_reduce_store<KA>(acc, reda + warp * KA, lane);
    } else {
#pragma unroll
      for (int k = 0; k < KA; ++k) {
        const R s = warp_sum(acc[k]);
        if (lane == 0) reda[warp * KA + k] = double(s);
      }
    }
    __syncthreads();
    if (warp == 0) {
      const int wpg = nwarps / MSPLIT;  // warps per channel group
      const int nq = want_q ? M * M * M : 0;
      const int nout = nq + (want_nll ? M + 1 : 0);
      for (int o = lane; o < nout; o += 32) {
        if constexpr (MSPLIT == 1) {
          const int k = o < nq ? o : (o < nq + M ? KQ + (o - nq) : KQ + MG);
          res[o < nq ? o : M * M * M + (o - nq)] = sum_warps(reda, KA, k);
        } else {
          double s = 0.0;
          if (o < nq) {
            const int m = o / (M * M), k = o - m * M * M;
            const int grp = m / MG, mi = m - grp * MG;
            for (int w = grp * wpg; w < (grp + 1) * wpg; ++w) s += reda[w * KA + mi * M * M + k];
            res[o] = s;
          } else if (o < nq + M) {
            const int m = o - nq;
            const int grp = m / MG, mi = m - grp * MG;
            for (int w = grp * wpg; w < (grp + 1) * wpg; ++w) s += reda[w * KA + KQ + mi];
            res[M * M * M + m] = s;
          } else {
            for (int w = 0; w < nwarps; ++w) s += reda[w * KA + KQ + MG];
            res[M * M * M + M] = s;
          }
        }
      }
      __syncwarp();
    }
    cluster_sum(res, M * M * M + M + 1, res, warp == 0);
  };

  // NLL of the current iterate from pass-A sums (thread 0).
  auto nll_from_res = [&](double logdet) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < M; ++m) s += double(us[m]) * res[M * M * M + m];
    return -double(T) * logdet + s + 0.69314718055994531 * res[M * M * M + M];
  };

  // ------------------------------------------------- EM sweep n (0..N) --
  // n == 0: U = |W^H x|^2 (stored); n >= 1: finish source n-1 (H row from the
  // stored Phi and the new L column); n < N: Phi of source n (stored) and its
  // L reduction sum_t Phi / H_true (fastfca.cpp:85-97).  Ends with the per-warp
  // partials in red and one barrier.  phis (the last sweep, balance on): also
  // reduce sum_t Phi(m) -- the mean of H row N-1 then follows from the new L
  // column without a sweep of its own (see balance_all).
  auto em_sweep = [&](int n, double* red, bool phis) {
    Uniform<M * NT, HOIST, R> le;
    le.load(Le);
    WU wr;
    if (n == 0) wr.load(reinterpret_cast<const R*>(Wr));
    R linv[M];
#pragma unroll
    for (int m = 0; m < M; ++m) linv[m] = Linv[m];
    R acc[2 * M + 1];
#pragma unroll
    for (int k = 0; k <= 2 * M; ++k) acc[k] = R(0);
    const int j = n - 1;
    // FUE frames per trip: loads, independent arithmetic chains, then stores.
    for (int tb = tid; tb < Tl; tb += FUE * nthreads) {
      R h[FUE][NT], w[FUE][WR];
      bool ok[FUE];
#pragma unroll
      for (int f = 0; f < FUE; ++f) {
        const int t = tb + f * nthreads;
        ok[f] = t < Tl;
        const int tt = ok[f] ? t : tb;  // always a valid record
        load_h(tt, h[f]);
        if (n == 0) {
          R xv[XR], u[M];
          ld_rec<XR>(xs + tt * XR, xv);
          decorrelate(wr, xv, u);
#pragma unroll
          for (int m = 0; m < M; ++m) w[f][m] = u[m];
        } else {
          ld_rec<WR>(wk + tt * WR, w[f]);
        }
      }
#pragma unroll
      for (int f = 0; f < FUE; ++f) {
        if (!ok[f]) continue;
        if (j >= 0) {
          R s = linv[0] * w[f][M];
#pragma unroll
          for (int m = 1; m < M; ++m) s += linv[m] * w[f][M + m];
          R hn = s * R(1.0 / M);
          hn = hn > tiny<R>() ? hn : tiny<R>();  // fastfca.cpp:96-97
#pragma unroll
          for (int k = 0; k < NT; ++k)
            if (k == j) h[f][k] = hn;
          acc[M] += hn;
        }
        if (n < N) {
          R hn = R(0);
#pragma unroll
          for (int k = 0; k < NT; ++k)
            if (k == n) hn = h[f][k];
          const R ihn = rcp_fast(hn);
          // Mixture variances L H + eps of all channels.  With the loadings
          // in shared memory (M * NT > 32) and M % 4 == 0 they are read one
          // column per vector load (the scalar form issued M * N loads).
          R lhs[M];
          if constexpr (!HOIST && M % 4 == 0 && sizeof(R) == 4) {
#pragma unroll
            for (int m = 0; m < M; ++m) lhs[m] = eps;
#pragma unroll
            for (int k = 0; k < NT; ++k) {
              if (FFCA_NK(k)) {
#pragma unroll
                for (int q = 0; q < M; q += 4) {
                  const float4 c = *reinterpret_cast<const float4*>(Le + k * M + q);
                  lhs[q] += c.x * h[f][k];
                  lhs[q + 1] += c.y * h[f][k];
                  lhs[q + 2] += c.z * h[f][k];
                  lhs[q + 3] += c.w * h[f][k];
                }
              }
            }
          } else {
#pragma unroll
            for (int m = 0; m < M; ++m) {
              R v = eps;
#pragma unroll
              for (int k = 0; k < NT; ++k)
                if (FFCA_NK(k)) v += le[m + k * M] * h[f][k];
              lhs[m] = v;
            }
          }
#pragma unroll
          for (int m = 0; m < M; ++m) {
            const R lh = lhs[m];
            const R lnhn = le[m + n * M] * hn;
            const R gg = lnhn * rcp_fast(lh);
            const R phi = gg * (gg * w[f][m] - lnhn) + lnhn;  // G^2 U + (1 - G) L_n H_n
            w[f][M + m] = phi;
            acc[m] += phi * ihn;
            if (phis) acc[M + 1 + m] += phi;
          }
        }
      }
#pragma unroll
      for (int f = 0; f < FUE; ++f) {
        if (!ok[f]) continue;
        const int t = tb + f * nthreads;
        if (j >= 0) {
          R hj = R(0);
#pragma unroll
          for (int k = 0; k < NT; ++k)
            if (k == j) hj = h[f][k];
          Hs[t * N + j] = hj;
        }
        if (n < N) st_rec<WR>(wk + t * WR, w[f]);
      }
    }
    FFCA_TIC(4);
    // Per-warp partials in the compute type (the cross-warp sum of NWMAX
    // fp32 partials adds nothing to the per-thread fp32 accumulation error).
    R* redr = reinterpret_cast<R*>(red);
    if (phis) {
      warp_reduce_store<2 * M + 1>(acc, redr + warp * (2 * M + 1), lane);
    } else {
      R a1[M + 1];
#pragma unroll
      for (int k = 0; k <= M; ++k) a1[k] = acc[k];
      warp_reduce_store<M + 1>(a1, redr + warp * (M + 1), lane);
    }
    __syncthreads();
  };

  // ------------------------------------------------------ MM sweeps --
  // L update: num/den reductions over t for sources [n0, n0+nc).
  auto mm_l_sweep = [&](int n0, int ncnt, bool compute_u, double* red) {
    constexpr int NCMAX = MmChunk<M, NT>::value;
    constexpr int K = 2 * M * NCMAX;
    Uniform<M * NT, HOIST, R> le;
    le.load(Le);
    WU wr;
    if (compute_u) wr.load(reinterpret_cast<const R*>(Wr));
    R acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = R(0);
    for (int t = tid; t < Tl; t += nthreads) {
      R h[NT];
      load_h(t, h);
      R w[WR];
      if (compute_u) {
        R xv[XR], u[M];
        ld_rec<XR>(xs + t * XR, xv);
        decorrelate(wr, xv, u);
#pragma unroll
        for (int m = 0; m < M; ++m) w[m] = u[m], w[M + m] = R(0);
        st_rec<WR>(wk + t * WR, w);
      } else {
        ld_rec<WR>(wk + t * WR, w);
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R lh = eps;
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (FFCA_NK(k)) lh += le[m + k * M] * h[k];
        const R il = rcp_fast(lh);
        const R ul2 = w[m] * il * il;
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
    warp_reduce_store<K>(acc, red + warp * K, lane);
    __syncthreads();
    if (warp == 0) {
      for (int o = lane; o < 2 * M * ncnt; o += 32) res[o] = sum_warps(red, K, o);
      __syncwarp();
    }
    cluster_sum(res, 2 * M * ncnt, res, warp == 0);
  };

  // H update with the new L (all sources from one lh, fastfca.cpp:111-116).
  // Stores true H values; the caller resets hsc[] to 1.
  auto mm_h_sweep = [&](bool compute_u, double* red) {
    Uniform<M * NT, HOIST, R> le;
    le.load(Le);
    WU wr;
    if (compute_u) wr.load(reinterpret_cast<const R*>(Wr));
    R acc[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) acc[k] = R(0);
    for (int t = tid; t < Tl; t += nthreads) {
      R h[NT];
      load_h(t, h);
      R u[M];
      if (compute_u) {
        R xv[XR];
        ld_rec<XR>(xs + t * XR, xv);
        decorrelate(wr, xv, u);
        R w[WR];
#pragma unroll
        for (int m = 0; m < M; ++m) w[m] = u[m], w[M + m] = R(0);
        st_rec<WR>(wk + t * WR, w);
      } else {
        R w[WR];
        ld_rec<WR>(wk + t * WR, w);
#pragma unroll
        for (int m = 0; m < M; ++m) u[m] = w[m];
      }
      R il[M], ul2[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        R lh = eps;
#pragma unroll
        for (int k = 0; k < NT; ++k)
          if (FFCA_NK(k)) lh += le[m + k * M] * h[k];
        il[m] = rcp_fast(lh);
        ul2[m] = u[m] * il[m] * il[m];
      }
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (FFCA_NK(k)) {
          // Le = L_new * hsc and H_true = H * hsc: the hsc factors cancel in
          // the ratio, the product H_true * sqrt(num/den) keeps one.
          R num = R(0), den = R(0);
#pragma unroll
          for (int m = 0; m < M; ++m) {
            num += le[m + k * M] * ul2[m];
            den += le[m + k * M] * il[m];
          }
          den = den > tiny<R>() ? den : tiny<R>();
          R hv = h[k] * hscr[k] * fsqrt(num / den);
          hv = hv > tiny<R>() ? hv : tiny<R>();
          Hs[t * N + k] = hv;
          acc[k] += hv;
        }
      }
    }
    warp_reduce_store<NT>(acc, red + warp * NT, lane);
    __syncthreads();
    if (warp == 0) {
      for (int o = lane; o < N; o += 32) res[o] = sum_warps(red, NT, o);
      __syncwarp();
    }
    cluster_sum(res, N, res, warp == 0);
  };

  // Le = L * hsc in the compute type (thread 0).
  auto refresh_le = [&]() {
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int m = 0; m < M; ++m) Le[m + n * M] = R(fmax(Ld[m + n * M] * hsc[n], tinyB));
  };

  // Serial algebra entry points, called by a whole warp: M <= 4 runs on lane 0
  // in registers; M > 4 uses the warp-cooperative versions on shared scratch.
  C* wsm0 = reinterpret_cast<C*>(smem + lay.off_wsm);  // warp 0 (IP, first log-det)
  C* wsm1 = wsm0 + 4 * M * M + M;                       // warp 1 (balance log-det)
  auto logdet_warp = [&](const double2* w, C* scratch, double& ld) -> bool {
    if constexpr (M > 4) {
      return warp_log_abs_det2<M, R>(w, scratch, lane, ld);
    } else {
      bool ok = true;
      if (lane == 0) ok = log_abs_det2<M, R>(w, ld);
      ok = __shfl_sync(0xffffffffu, ok, 0);
      ld = __shfl_sync(0xffffffffu, ld, 0);
      return ok;
    }
  };
  auto logdet_w0 = [&](const double2* w, double& ld) { return logdet_warp(w, wsm0, ld); };
  auto logdet_w1 = [&](const double2* w, double& ld) { return logdet_warp(w, wsm1, ld); };
  // scaled: apply the pending balance W column scales (wsc) first.
  auto run_ip = [&](unsigned long long seed, bool with_logdet, bool scaled) {
    int bad = -1;
    bool ok = true;
    constexpr bool WIP = (M > 4) || (M >= FFCA_IP_WARP_MIN);  // warp-cooperative IP
    if constexpr (WIP) {
      if (scaled) {
        for (int k = lane; k < M * M; k += 32) {
          const double c = double(wsc[k / M]);
          Wd[k].x *= c;
          Wd[k].y *= c;
        }
        __syncwarp();
      }
      if constexpr (FFCA_IP_WARP_REG || M <= 4)
        ok = ip_update_warp_reg<M, R>(Wd, res, invT, seed, bin_index, rng, wsm0, lane, bad);
      else
        ok = ip_update_warp<M, R>(Wd, res, invT, seed, bin_index, rng, wsm0, lane, bad);
    } else {
      if (lane == 0) {
        IpExtras<R> ex;
        ex.wscale = scaled ? wsc : nullptr;
        ex.wout = Wr;
        if (M == 2 && with_logdet) {  // log|det W|^2 for the next trace entry
          ex.ldet = &sc->logdet0;
          ex.ldok = &sc->ldok;
        }
        ok = ip_update<M, R>(Wd, res, invT, seed, bin_index, rng, bad, ex);
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
    }
    if (lane == 0 && !ok) {
      sc->status = kStatusIpSingular | (bad << 8);
      sc->stop = 1;
    }
    __syncwarp();
    if constexpr (WIP)
      for (int k = lane; k < M * M; k += 32) Wr[k] = mkc<R>(R(Wd[k].x), R(Wd[k].y));
    if constexpr (M > 2)
      for (int k = lane; k < M * M; k += 32) Wlg[k] = Wd[k];  // log-det input (ldwarp)
    if constexpr (M == 1) {
      if (with_logdet) {
        double ld = 0.0;
        const bool lok = logdet_w0(Wd, ld);
        if (lane == 0) {
          sc->ldok = lok ? 1 : 0;
          sc->logdet0 = ld;
        }
      }
    }
  };


  // ---- balance_scales (fastfca.cpp:127-142), computed by EVERY warp
  //      (lane-parallel: mu_n per source lane, s_m per channel lane) from
  //      values no warp modifies after the last sweep's barrier; results go to
  //      the other parity buffer (Ld, hsc, hinv) or are written with the same
  //      bits by every warp (Le, us, wsc, logs).  No serial section, no
  //      barrier.  The W column scales wsc are applied to the fp64 master by
  //      warp 0 in the next serial section (nothing reads W before it).
  //      phi_mean: the mean of H row N-1 follows from the last EM sweep's
  //      sums, (1/(M T)) sum_m (sum_t Phi(m)) / L(m, N-1) -- the row itself is
  //      stored by the next pass A (fastfca.cpp:95-97).
  auto balance_all = [&](bool on, bool phi_mean) {
    const int nx = par ^ 1;
    B* hscn = hsc0 + nx * NT;
    B* hinvn = hinv0 + nx * NT;
    B* Ldn = Ld0 + nx * (M * NT);
    if constexpr (M * NT <= 32) {
      // Small models: lane k owns L(m, n), k = m + n M, and derives every
      // row mean and channel scale it needs itself, in registers -- the same
      // operations in the same order as the general path below (so the same
      // bits), without its shared-memory round trips and warp syncs.
      const int k = lane < M * N ? lane : 0;
      const int m = k % M, n = k / M;
      B hv[NT];  // hinv of every source
      unsigned vmask = 0u;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        B mu = B(1);
        if (FFCA_NK(j)) {
          if (phi_mean && j == N - 1) {
            B c = B(0);
#pragma unroll
            for (int mm = 0; mm < M; ++mm) c += psum[mm] * BM::rcp(Ld[mm + j * M]);
            mu = c * B(invT / double(M));
          } else {
            mu = hsumv[j] * B(invT);
          }
        }
        const bool v = on && mu > B(0) && isfinite(mu);
        hv[j] = v ? mu : B(1);
        vmask |= v ? (1u << j) : 0u;
      }
      B hn = hv[0];
#pragma unroll
      for (int j = 1; j < NT; ++j)
        if (j == n) hn = hv[j];
      const B hs = ((vmask >> n) & 1u) ? BM::rcp(hn) : B(1);
      B s = B(0);
#pragma unroll
      for (int j = 0; j < NT; ++j)
        if (FFCA_NK(j)) s += Ld[m + j * M] * hv[j];
      s *= B(1.0 / double(N));
      const bool vs = on && s > B(0) && isfinite(s);
      const B usm = vs ? BM::rcp(s) : B(1);
      double ls = (vs && n == 0 && lane < M * N) ? double(BM::log_d(s)) : 0.0;
      const B l0 = Ld[k];
      B l = l0 * hn * usm;
      l = (l0 > B(0) && !(l > B(0))) ? tinyB : l;
      const B le = l * hs;
      if (lane < M * N) {
        Ldn[k] = l;
        Le[k] = R((l > B(0) && !(le > B(0))) ? tinyB : le);
        if (m == 0) hscn[n] = hs, hinvn[n] = hn;
        if (n == 0) us[m] = usm, wsc[m] = vs ? BM::rsq(s) : B(1);
      }
      // sum_m log s_m over lanes 0..M-1 (n == 0), fixed order.
#pragma unroll
      for (int o = Pow2Ceil<M>::value / 2; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
      if (lane == 0) sc->logs = ls;
      par = nx;
      Ld = Ldn;
      hsc = hscn;
      hinv = hinvn;
      __syncwarp();
      return;
    }
    for (int n = lane; n < N; n += 32) {
      B mu;
      if (phi_mean && n == N - 1) {
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
      us[m] = v ? BM::rcp(s) : B(1);  // U and L-row scale 1/s
      wsc[m] = v ? BM::rsq(s) : B(1);  // W column scale
      if (v) ls = BM::log_d(s);
    }
    __syncwarp();
    for (int k = lane; k < M * N; k += 32) {
      const int m = k % M, n = k / M;
      // L(m,n) mu_n / s_m; exact zeros stay zero (ica_mode_fit's one-hot
      // loadings), a positive value that underflows the compute type
      // becomes its smallest normal.
      const B l0 = Ld[k];
      B l = l0 * hinvn[n] * us[m];
      l = (l0 > B(0) && !(l > B(0))) ? tinyB : l;
      Ldn[k] = l;
      const B le = l * hscn[n];
      Le[k] = R((l > B(0) && !(le > B(0))) ? tinyB : le);
    }
    __syncwarp();  // converged before the shuffles
    // sum_m log s_m over the lowest Pow2Ceil(M) lanes (fixed order).
#pragma unroll
    for (int o = Pow2Ceil<M>::value / 2; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    const double lsum = ls;
    if (lane == 0) sc->logs = lsum;
    par = nx;
    Ld = Ldn;
    hsc = hscn;
    hinv = hinvn;
    __syncwarp();
  };

  // -------------------------------------------------------------- driver --
  const bool record = p.record != 0;
  const bool silent = !(power > 0.0);
  const bool bal = p.normalize && update_loading;
  const int ldwarp = nwarps - 1;  // M > 2: log-det of the IP output, off the serial path
  FFCA_TIC(9);
  pass_a(true, p.iters > 0 && !silent, record, false);
  FFCA_TIC(1);
  if (warp == 0) {
    if (record) {
      double ld = 0.0;
      const bool ok = logdet_w0(Wd, ld);
      if (lane == 0) {
        if (!ok) {
          sc->status = kStatusSingularW;
          sc->stop = 1;
        }
        sc->nll0 = nll_from_res(ld);
        if (lead) p.nll[size_t(0) * p.nll_stride + p.prob_offset + b] = sc->nll0;
      }
    }
    if (lane == 0 && silent && !sc->stop) {
      // Entirely silent band: parameters stay at the init (fastfca.cpp:165-170).
      sc->status = kStatusSilent;
      sc->stop = 1;
      if (record && lead)
        for (int t = 0; t < p.iters; ++t)
          p.nll[size_t(t + 1) * p.nll_stride + p.prob_offset + b] = sc->nll0;
    }
    __syncwarp();
    // IP sweep of iteration 0 (fastfca.cpp:36-72), fused into this serial section.
    if (!sc->stop && p.iters > 0) run_ip(p.seed, record, false);
  }
  __syncthreads();
  if (!sc->stop) {
    for (int it = 0; it < p.iters; ++it) {
      if constexpr (M > 2) {
        if (record && warp == ldwarp) {
          double ld = 0.0;
          const bool ok = logdet_w1(Wlg, ld);
          if (lane == 0) {
            sc->ldok = ok ? 1 : 0;
            sc->logdet0 = ld;
          }
          __syncwarp();
        }
      }
      // ---- L/H updates (the IP sweep of this iteration already ran)
      if (p.flavor == 0) {
        for (int n = 0; n < N; ++n) {
          const bool phis = bal && n == N - 1;
          const int K = phis ? 2 * M + 1 : M + 1;
          double* red = redb + (n & 1) * nwarps * kred;
          em_sweep(n, red, phis);
          FFCA_TIC(5);
          // Every warp sums the partials (lane k holds value k) and applies
          // the identical update; each shared value below is written with the
          // same bits by every warp and is not read in its old state after
          // the barrier.
          R tot = (lane < K) ? tree_sum_warps<NWMAX>(reinterpret_cast<const R*>(red), K, lane,
                                                     nwarps)
                             : R(0);
          if constexpr (CL) {
            // CTA totals -> cluster totals (rank order); every warp reads them.
            if (warp == 0 && lane < K) res[lane] = double(tot);
            __syncwarp();
            cluster_sum(res, K, res, true);
            tot = (lane < K) ? R(res[lane]) : R(0);
            __syncwarp();
          }
          // Shuffles while the warp is converged: the H row n-1 sum and (last
          // sweep) sum_t Phi(m) on lane m.
          const R hs = __shfl_sync(0xffffffffu, tot, M);
          const R ps = __shfl_down_sync(0xffffffffu, tot, M + 1);
          FFCA_TIC(8);
          if (lane < M) {
            // L(:, n) = max(sum_t Phi / H_true / T, tiny) with H_true = H * hsc
            // (fastfca.cpp:92-94).  The next sweep (or pass A) stores the true
            // H row n, so Le(:, n) becomes the new L column (no hsc).
            const int m = lane;
            const B l = update_loading ? fmax(B(tot) * B(invT) * hinv[n], tinyB) : Ld[m + n * M];
            const R lr = R(l);
            Ld[m + n * M] = l;
            if (!phis) Le[m + n * M] = lr;  // with phis the balance rewrites all of Le
            Linv[m] = rcp_fast(lr);
            if (phis) psum[m] = B(ps);
          }
          if (lane == 0 && n >= 1) hsumv[n - 1] = B(hs);
          __syncwarp();
          FFCA_TIC(6);
        }
      } else {
        bool first = true;
        int pb = 0;
        if (update_loading) {
          for (int n0 = 0; n0 < N; n0 += p.nc) {
            const int cnt = min(p.nc, N - n0);
            mm_l_sweep(n0, cnt, first, redb + (pb++ & 1) * nwarps * kred);
            if (tid == 0) {
              for (int c = 0; c < cnt; ++c)
#pragma unroll
                for (int m = 0; m < M; ++m) {
                  numd[m + (n0 + c) * M] = B(res[(c * M + m) * 2 + 0]);
                  dend[m + (n0 + c) * M] = B(res[(c * M + m) * 2 + 1]);
                }
              if (n0 + cnt >= N) {
                // num, den were accumulated with H_stored; H_true = H * hsc scales
                // both by hsc[n], which cancels in num/den.
                for (int k = 0; k < M * N; ++k) {
                  const B den = fmax(dend[k], tinyB);
                  Ld[k] = fmax(Ld[k] * BM::sq(numd[k] * BM::rcp(den)), tinyB);  // :107-109
                }
                refresh_le();
                for (int k = 0; k < N; ++k) hscr[k] = R(hsc[k]);
              }
            }
            __syncthreads();
            first = false;
          }
        } else {
          if (tid == 0) {
            for (int k = 0; k < N; ++k) hscr[k] = R(hsc[k]);
          }
          __syncthreads();
        }
        mm_h_sweep(first, redb + (pb & 1) * nwarps * kred);
        if (tid == 0) {
          for (int k = 0; k < N; ++k) hsumv[k] = B(res[k]);
        }
        __syncthreads();
        FFCA_TIC(5);
      }
      balance_all(bal, p.flavor == 0);
      touched = touched || update_loading;
      FFCA_TIC(7);
      const bool more = it + 1 < p.iters;
      // EM: pass A also stores H row N-1, so it runs after the last iteration too.
      if (more || record || p.flavor == 0) pass_a(false, more, record, p.flavor == 0);
      FFCA_TIC(1);
      if (warp == 0) {
        // Balance W column scales on the fp64 master (fastfca.cpp:139-141):
        // folded into the IP sweep when one follows.
        const bool ip_next = more && !(record && !sc->ldok);
        if (!ip_next) {
          for (int k = lane; k < M * M; k += 32) {
            double2 w = Wd[k];
            const double c = double(wsc[k / M]);
            w.x *= c;
            w.y *= c;
            Wd[k] = w;
          }
          __syncwarp();
        }
        if (lane == 0 && record) {
          if (!sc->ldok) {  // log_abs_det2 throws on a singular W (sigmodel.cpp:124-125)
            sc->status = kStatusSingularW;
            sc->stop = 1;
          }
          if (lead)
            p.nll[size_t(it + 1) * p.nll_stride + p.prob_offset + b] =
                nll_from_res(sc->logdet0 - sc->logs);
        }
        __syncwarp();
        // Next iteration's IP sweep, fused into the pass-A serial section.
        if (ip_next) run_ip(p.seed + (unsigned long long)(it + 1), record, true);
      }
      FFCA_TIC(2);
      __syncthreads();
      FFCA_TIC(3);
      if (sc->stop) break;
    }
  }
#undef FFCA_NK
#undef FFCA_TIC
  __syncthreads();
  // ------------------------------------------------------------- epilogue --
  if (lead) {
    for (int k = tid; k < M * M; k += nthreads) p.W[size_t(b) * M * M + k] = Wd[k];
    if (touched)
      for (int k = tid; k < M * N; k += nthreads) p.L[size_t(b) * M * N + k] = double(Ld[k]);
  }
  bool pending = false;
  for (int k = 0; k < N; ++k) pending = pending || hsc[k] != B(1);
  if (RES || pending)
    for (int k = tid; k < N * Tl; k += nthreads) Hg[k] = R(double(Hs[k]) * double(hsc[k % N]));
#ifdef FFCA_PHASE_TIMING
  if (p.timing && tid == 0)
    for (int k = 0; k < 10; ++k) p.timing[size_t(b) * 16 + k] = tacc[k];
#undef tlast
#endif
  if (tid == 0 && lead) p.status[b] = sc->status;
}

}  // namespace ffca
