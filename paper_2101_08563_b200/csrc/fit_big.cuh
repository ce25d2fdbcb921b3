// fit_big.cuh -- the large-bin FastFCA IP+EM fit kernel (BASELINE config 3:
// M = 8 channels, N = 12 sources, T = 8000 frames per bin).
//
// Same per-bin algorithm as fit_kernel.cuh (one CTA group owns one frequency
// problem for every iteration of fastfca_fit, reference src/fastfca.cpp:
// 158-184), laid out for bins whose per-frame state does not fit one SM's
// shared memory.  The per-iteration serial chain (N + 1 reductions and the IP
// sweep) is paid once per SM group, so the design goal is the fewest SMs per
// bin: every per-frame array lives on chip, split over the SM's three stores:
//
//      H    [NHP planes][t] 16-byte vectors  shared memory (persistent, in/out)
//      U    [slot] M values                  tensor memory (|W^H x|^2, then 1/sigma^2)
//      Phi  [slot] M values                  tensor memory (posterior of the
//                                            current source, sweep to sweep)
//      x    [t][M] complex                   global (L2-resident: ~0.5 MB per
//                                            bin, read twice per iteration)
//
// Tensor memory (256 KB per SM, unused by this non-GEMM path otherwise) is the
// lever: thread (warp w, lane l) owns TMEM lane 32 (w % 4) + l and a 128-column
// strip per warp group, and moves a frame's U and Phi with one 32x32b
// tcgen05.ld / tcgen05.st.  For c3 in fp32 a CTA holds 4096 frames (512
// threads x 8 slots): a bin needs a 2-CTA cluster and all 148 SMs are used
// (74 bins in flight).
//
// Two thread-to-frame mappings, both warp-local (a warp only ever touches the
// frames its lanes own, so no barrier separates the passes):
//  * one thread per frame (slots s: frame 32 w + lane + s NTHR) for the EM
//    sweeps and the variance pass;
//  * M lanes per frame for the two passes that read x -- the decorrelation
//    pass (lane j owns channel j: y_j = w_j^H x with w_j in registers; the
//    owner lane gathers U with shuffles) and the weighted-covariance pass,
//    where lane a forms x_a conj(x_{a+d mod M}), d = 0..M/2 -- every entry of
//    the Hermitian outer product once (the d = M/2 products of lanes a >= M/2
//    are the only duplicates) -- and accumulates them against the M weights
//    1/sigma^2_m shuffled from the owner lane (a [M x T] . [T x M^2] product
//    with no recomputed outer products).
//
// Per iteration (fastfca.cpp:172-183):
//   IP       ip_fast.cuh (Q^{-1} and W^{-H} in parallel, Sherman-Morrison
//            column chain; the reference's column solves with the seeded
//            restart as the fallback, fastfca.cpp:36-72).
//   U        decorrelated powers U = |W^H x|^2 (sigmodel.cpp:93-107).
//   EM       N sweeps (em_update_lh, fastfca.cpp:80-99): sweep n finishes H
//            row n-1 from the stored posterior and the freshly reduced L
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

#include <type_traits>

#include "common.cuh"
#include "fit_kernel.cuh"
#include "ip_fast.cuh"
#include "serial_math.cuh"

#ifndef FFCA_BIG_INCR
#define FFCA_BIG_INCR 1  // incremental mixture variances in the fp32 EM sweeps
#endif
#ifndef FFCA_BIG_PREFETCH
#define FFCA_BIG_PREFETCH 0  // prefetch the next EM trip's U into registers (measured: no gain)
#endif
#ifndef FFCA_BIG_PACK_ODD
#define FFCA_BIG_PACK_ODD 0  // packed EM sweep for odd M (padded channel): measured slower at M = 3
#endif
#ifndef FFCA_BIG_A2_SCALAR
#define FFCA_BIG_A2_SCALAR 0  // scalar FFMA instead of FFMA2 in the covariance pass (experiment)
#endif
#ifndef FFCA_BIG_A2_UNROLL
#define FFCA_BIG_A2_UNROLL 8  // frame batches of the covariance pass unrolled together (8 = all)
#endif
#ifndef FFCA_BIG_FS
#define FFCA_BIG_FS 2  // frame slots per trip of the incremental EM sweep (4: spills at M = 8)
#endif

namespace ffca {

constexpr int kA2Unroll = FFCA_BIG_A2_UNROLL;

// Shared-memory carve-up of a big-bin CTA (byte offsets), computed on the host.
struct BigLayout {
  int off_h, ps;  // H planes: ps 16-byte vectors per plane
  int off_le, off_ld, off_hsc, off_hinv, off_linv, off_lprev, off_us, off_wsc, off_hsum, off_psum;
  int off_wd, off_wr, off_ipscr, off_ldscr, off_red, off_cx, off_scal;
  int off_scr;                                    // reused scratch region:
  int off_gscr, off_ex, off_q, off_ipf, off_rng;  //   covariance tree, then the rest
  int total;
  int csize, tcap;
};

template <typename R> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

// Incremental mixture variances in the fp32 EM sweeps (see big_fit_kernel).
template <int M, typename R, int SLOTS>
constexpr bool big_incr() {
  return FFCA_BIG_INCR != 0 && sizeof(R) == 4 && SLOTS % FFCA_BIG_FS == 0 && M == 8;
}

constexpr int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

template <int M, int N, typename R, int SLOTS, int NTHR, int MS, bool AUXG = false>
struct BigCfg {
  static constexpr int VE = Vec16<R>::n;           // reals per 16-byte vector
  static constexpr int NHP = (N + VE - 1) / VE;    // H planes
  static constexpr int NW = NTHR / 32;
  static constexpr int TCAP = NTHR * SLOTS;        // frames per CTA
  static constexpr int D = M / 2;                  // cyclic product distances
  static constexpr int NP = 1 + 2 * D;             // reals per covariance lane
  static constexpr int ML = pow2_at_least(M);      // lanes per frame in the M-lane passes
  static constexpr int LES = ((M + VE - 1) / VE) * VE;  // stride of an effective-loading column
  static constexpr int MW = M / MS;                // weights per covariance lane
  static constexpr int KA = NP * MW;               // accumulators per covariance lane
  static constexpr int GS = ML * MS;               // covariance lanes per frame (lanes >= M idle)
  static constexpr int KAP = ((KA + 32 / GS - 1) / (32 / GS)) * (32 / GS);  // padded so that the
                                                   // in-warp reduce-scatter halves evenly
  static constexpr int KRED = 2 * M + 1;           // EM sweep partials
  static constexpr int KQ = M * M * M;             // covariance totals
  static constexpr int WPR = pow2_at_least(M) * int(sizeof(R)) / 4;  // TMEM columns per record
  static constexpr int SCOL = 2 * WPR;             // columns per slot (U, Phi)
  static constexpr int WGROUPS = (NW + 3) / 4;     // warps sharing a TMEM lane quarter
  static constexpr int PW = pow2_at_least(NW);
  static constexpr int HW = PW / 2 > 0 ? PW / 2 : 1;  // warps publishing in the first tree step
  static constexpr int CNT = KAP / (32 / GS);  // covariance partials per lane after the
                                               // in-warp reduce-scatter
  static constexpr int TMCOLS = [] {           // tensor-memory columns (a power of two >= 32)
    int c = 32;
    while (c < SLOTS * SCOL * WGROUPS) c <<= 1;
    return c;
  }();
  static_assert(32 % GS == 0 && M % MS == 0, "lanes per frame must divide a warp");
  static_assert(NTHR % 32 == 0, "whole warps");
  static_assert(SLOTS * SCOL * WGROUPS <= 512, "tensor memory columns");
  static_assert(WPR == 4 || WPR == 8 || WPR == 16, "record width");

  static int al(int v) { return (v + 15) & ~15; }
  // Cold-path scratch of a CTA in global memory (FitParams::aux): the restart
  // generator, the saved W and the two small matrices of the reference-order
  // IP / log-det -- kept out of shared memory so that two CTAs share an SM.
  static constexpr int AUX_RNG = 0;
  static constexpr int AUX_WSAVE = (int(sizeof(RestartRng)) + 15) & ~15;
  static constexpr int AUX_IPSCR = AUX_WSAVE + M * M * 16;
  static constexpr int AUX_LDSCR = AUX_IPSCR + ((M * M * 2 * int(sizeof(R)) + 15) & ~15);
  static constexpr int AUX_BYTES = (AUX_LDSCR + M * (M + 1) * 2 * int(sizeof(R)) + 255) & ~255;

  static BigLayout layout(int csize, int T) {
    BigLayout L{};
    L.csize = csize;
    L.tcap = TCAP;
    const int tloc = (T + csize - 1) / csize;     // frames of the largest CTA
    L.ps = ((tloc + 3) & ~3) + 4;  // planes start 16 banks apart
    int o = 0;
    L.off_h = o; o = al(o + NHP * L.ps * 16);
    const int rs = int(sizeof(R));
    L.off_le = o; o = al(o + N * LES * rs);
    L.off_ld = o; o = al(o + 2 * M * N * rs);
    L.off_hsc = o; o = al(o + 2 * N * rs);
    L.off_hinv = o; o = al(o + 2 * N * rs);
    L.off_linv = o; o = al(o + M * rs);
    L.off_lprev = o; o = al(o + M * rs);
    L.off_us = o; o = al(o + M * rs);
    L.off_wsc = o; o = al(o + M * rs);
    L.off_hsum = o; o = al(o + N * rs);
    L.off_psum = o; o = al(o + M * rs);
    L.off_wd = o; o = al(o + M * M * 16);
    L.off_wr = o; o = al(o + M * M * 2 * rs);
    L.off_ipscr = o; if (!AUXG) o = al(o + M * M * 2 * rs);  // AUXG: global (aux)
    L.off_ldscr = o; if (!AUXG) o = al(o + M * (M + 1) * 2 * rs);
    L.off_red = o; o = al(o + 2 * NW * KRED * rs);
    L.off_cx = o; o = al(o + 2 * csize * KRED * 8);
    L.off_scal = o; o = al(o + 128);
    // Scratch, reused: the covariance tree (HW warps' partials), then the
    // CTA totals ex[] (read by the other CTAs of the cluster), the cluster
    // totals qraw[], the fast-IP scratch and the restart generator.
    L.off_scr = o;
    const int gscr = HW * 32 * CNT * rs;
    L.off_gscr = o;
    L.off_ex = o;
    int e = al(o + (KQ + 2 * (M + 1)) * 8);
    L.off_q = e; e = al(e + KQ * 8);
    L.off_ipf = e; e = al(e + int(sizeof(IpFastScratch<M, R>)));
    L.off_rng = e; if (!AUXG) e = al(e + AUX_IPSCR);  // restart generator + saved W
    o = al(o + gscr) > e ? al(o + gscr) : e;
    L.total = o;
    return L;
  }
};

struct BigScalars {
  double eps, nll0, logdet0, logs;
  int stop, status, ldok;
  unsigned tmem;
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
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ---------------------------------------------------------------- TMEM --
// 32x32b register transfers: thread l of the warp reads / writes TMEM lane
// (quarter base + l), columns [col, col + n).  Raw 32-bit words; a double is
// two columns (low word first).
__device__ __forceinline__ void tm_ld4(unsigned a, unsigned (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(a));
}
__device__ __forceinline__ void tm_st4(unsigned a, const unsigned (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
template <int NWORDS>
__device__ __forceinline__ void tm_ld(unsigned a, unsigned (&v)[NWORDS]);
template <int NWORDS>
__device__ __forceinline__ void tm_st(unsigned a, const unsigned (&v)[NWORDS]);
__device__ __forceinline__ void tm_ld8(unsigned a, unsigned (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(a));
}
__device__ __forceinline__ void tm_ld16(unsigned a, unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(a));
}
__device__ __forceinline__ void tm_st8(unsigned a, const unsigned (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tm_st16(unsigned a, const unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(a),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

template <> __device__ __forceinline__ void tm_ld<4>(unsigned a, unsigned (&v)[4]) { tm_ld4(a, v); }
template <> __device__ __forceinline__ void tm_ld<8>(unsigned a, unsigned (&v)[8]) { tm_ld8(a, v); }
template <> __device__ __forceinline__ void tm_ld<16>(unsigned a, unsigned (&v)[16]) { tm_ld16(a, v); }
template <> __device__ __forceinline__ void tm_st<4>(unsigned a, const unsigned (&v)[4]) { tm_st4(a, v); }
template <> __device__ __forceinline__ void tm_st<8>(unsigned a, const unsigned (&v)[8]) { tm_st8(a, v); }
template <> __device__ __forceinline__ void tm_st<16>(unsigned a, const unsigned (&v)[16]) { tm_st16(a, v); }

// Words <-> values of the compute type.
template <int M, typename R>
__device__ __forceinline__ void words_to(const unsigned* w, R (&v)[M]) {
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if constexpr (sizeof(R) == 4) v[m] = __uint_as_float(w[m]);
    else v[m] = __hiloint2double(int(w[2 * m + 1]), int(w[2 * m]));
  }
}
// One record of M values in the compute type.
template <int M, typename R>
__device__ __forceinline__ void tm_load_rec(unsigned a, R (&v)[M]) {
  constexpr int NWD = pow2_at_least(M) * int(sizeof(R)) / 4;
  unsigned w[NWD];
  tm_ld<NWD>(a, w);
  tm_wait_ld();
  words_to<M, R>(w, v);
}
// Two adjacent records (U then Phi) in one transfer when they fit 16 words.
template <int M, typename R>
__device__ __forceinline__ void tm_load_rec2(unsigned a, R (&u)[M], R (&ph)[M]) {
  constexpr int NWD = pow2_at_least(M) * int(sizeof(R)) / 4;
  if constexpr (2 * NWD <= 16) {
    unsigned w[2 * NWD];
    tm_ld<2 * NWD>(a, w);
    tm_wait_ld();
    words_to<M, R>(w, u);
    words_to<M, R>(w + NWD, ph);
  } else {
    tm_load_rec<M, R>(a, u);
    tm_load_rec<M, R>(a + NWD, ph);
  }
}
template <int M, typename R>
__device__ __forceinline__ void tm_store_rec(unsigned a, const R (&v)[M]) {
  constexpr int NWD = pow2_at_least(M) * int(sizeof(R)) / 4;
  unsigned w[NWD];
#pragma unroll
  for (int k = M * int(sizeof(R)) / 4; k < NWD; ++k) w[k] = 0u;  // record padding (odd M)
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if constexpr (sizeof(R) == 4) {
      w[m] = __float_as_uint(v[m]);
    } else {
      w[2 * m] = unsigned(__double2loint(v[m]));
      w[2 * m + 1] = unsigned(__double2hiint(v[m]));
    }
  }
  tm_st<NWD>(a, w);
}

// Two adjacent records in one transfer (fp32, 2 M <= 16 words).
template <int M>
__device__ __forceinline__ void tm_store_rec2(unsigned a, const float (&v0)[M], const float (&v1)[M]) {
  static_assert(2 * M <= 16 && (M == 4 || M == 8), "two fp32 records per store");
  unsigned w[2 * M];
#pragma unroll
  for (int m = 0; m < M; ++m) w[m] = __float_as_uint(v0[m]), w[M + m] = __float_as_uint(v1[m]);
  tm_st<2 * M>(a, w);
}

// Packed fp32 pairs (FFMA2 / FMUL2 on sm_100): the frame loops are issue
// bound, and one packed instruction does two lanes' worth of FMA work
// (measured: 95 FMA/clk/SM at 1.5 issue slots vs 111 at 3.5 for FFMA).
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fma2s(float2 a, float s, float2 c) { return __ffma2_rn(a, f2(s, s), c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fmul2s(float2 a, float s) { return __fmul2_rn(a, f2(s, s)); }
__device__ __forceinline__ float2 fneg2(float2 a) { return f2(-a.x, -a.y); }

template <int M, int N, typename R, int SLOTS, int NTHR, int MS, bool CL, int MINB = 1, bool AUXG = false,
          bool EXACTVAR = false>
__global__ void __launch_bounds__(NTHR, MINB) big_fit_kernel(FitParams p, BigLayout lay) {
  using Cfg = BigCfg<M, N, R, SLOTS, NTHR, MS, AUXG>;
  using C = cplx_t<R>;
  using V = typename Vec16<R>::type;
  constexpr int VE = Cfg::VE, NHP = Cfg::NHP, NW = Cfg::NW, PW = Cfg::PW, HW = Cfg::HW;
  constexpr int D = Cfg::D, NP = Cfg::NP, MW = Cfg::MW, KA = Cfg::KA, GS = Cfg::GS;
  constexpr int KRED = Cfg::KRED, KQ = Cfg::KQ, WPR = Cfg::WPR, SCOL = Cfg::SCOL, CNT = Cfg::CNT;
  constexpr int KAP = Cfg::KAP, TMCOLS = Cfg::TMCOLS, ML = Cfg::ML, LES = Cfg::LES;
  // fp32 path: the mixture variances sigma^2 = eps + L H live in tensor memory
  // (where U used to be) and follow each EM sweep's row update incrementally
  // (sigma^2 += L_new h_new - L_old h_old, 4M flops instead of the 2MN of a
  // fresh sum); the variance pass A1 rebuilds them exactly every iteration.
  // U, read-only during the sweeps, moves to an L2-resident global scratch.
  // Measured: c3 (M = 8, N = 12) 97.0 -> 94.5 ms; at M = 4, N = 6 the fresh
  // sum is only 12 packed FMAs per frame and the extra L2 reads cost more
  // than they save (c2 4.54 -> 4.60 ms), so it stays on the exact path.
  // EXACTVAR (FFCA_EXACT_VARIANCES=1 at run time) keeps the fresh sum.
  constexpr bool INCR = big_incr<M, R, SLOTS>() && !EXACTVAR;
  using B = R;
  using BM = SMath<B>;
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  // Provably warp-uniform (a shuffle from lane 0), so branches on the warp
  // index stay convergent and shuffles inside them need no collective
  // fallback code.
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
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
  // Frame slots in use: short bins skip the empty ones (an even count, the
  // fp32 EM sweep takes two slots per trip).
  constexpr int SLQ = (big_incr<M, R, SLOTS>() && !EXACTVAR) ? FFCA_BIG_FS : 2;
  const int nsl = min(SLOTS, (((Tl + NTHR - 1) / NTHR) + SLQ - 1) / SLQ * SLQ);
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
  R* Hs = reinterpret_cast<R*>(Hp);
  R* Le = reinterpret_cast<R*>(smem + lay.off_le);  // [N][LES]: column n at Le + n LES
  B* const Ld0 = reinterpret_cast<B*>(smem + lay.off_ld);
  B* const hsc0 = reinterpret_cast<B*>(smem + lay.off_hsc);
  B* const hinv0 = reinterpret_cast<B*>(smem + lay.off_hinv);
  R* Linv = reinterpret_cast<R*>(smem + lay.off_linv);
  R* Lprev = reinterpret_cast<R*>(smem + lay.off_lprev);  // effective column n before its update
  B* us = reinterpret_cast<B*>(smem + lay.off_us);
  B* wsc = reinterpret_cast<B*>(smem + lay.off_wsc);
  B* hsumv = reinterpret_cast<B*>(smem + lay.off_hsum);
  B* psum = reinterpret_cast<B*>(smem + lay.off_psum);
  double2* Wd = reinterpret_cast<double2*>(smem + lay.off_wd);
  C* Wr = reinterpret_cast<C*>(smem + lay.off_wr);
  // Cold-path scratch: shared memory, or (AUXG) this CTA's slice of FitParams::aux.
  unsigned char* aux = AUXG ? reinterpret_cast<unsigned char*>(p.aux) + size_t(blockIdx.x) * Cfg::AUX_BYTES
                            : smem + lay.off_rng;
  C* ipscr = AUXG ? reinterpret_cast<C*>(aux + Cfg::AUX_IPSCR) : reinterpret_cast<C*>(smem + lay.off_ipscr);
  C* ldscr = AUXG ? reinterpret_cast<C*>(aux + Cfg::AUX_LDSCR) : reinterpret_cast<C*>(smem + lay.off_ldscr);
  R* red = reinterpret_cast<R*>(smem + lay.off_red);
  double* cx = reinterpret_cast<double*>(smem + lay.off_cx);
  BigScalars* sc = reinterpret_cast<BigScalars*>(smem + lay.off_scal);
  R* gscr = reinterpret_cast<R*>(smem + lay.off_gscr);
  double* ex = reinterpret_cast<double*>(smem + lay.off_ex);
  double* qraw = reinterpret_cast<double*>(smem + lay.off_q);
  IpFastScratch<M, R>* ipf = reinterpret_cast<IpFastScratch<M, R>*>(smem + lay.off_ipf);
  RestartRng* rng = reinterpret_cast<RestartRng*>(aux + Cfg::AUX_RNG);
  double2* wsave = reinterpret_cast<double2*>(aux + Cfg::AUX_WSAVE);
  B* Ld = Ld0;
  B* hsc = hsc0;
  B* hinv = hinv0;
  int par = 0;

  const C* xg = reinterpret_cast<const C*>(p.x) + (size_t(b) * T + t0g) * M;
  R* Hg = reinterpret_cast<R*>(p.H) + (size_t(b) * T + t0g) * N;
  R* Ug = reinterpret_cast<R*>(p.work) + (size_t(b) * T + t0g) * M;  // INCR only

  // ---- tensor memory: TMCOLS columns (all 512 for the one-CTA-per-SM shapes).
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
        unsigned(__cvta_generic_to_shared(&sc->tmem))), "n"(TMCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
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
  if constexpr (LES != M) {  // zero the column padding (odd M)
    for (int k = tid; k < N * LES; k += NTHR) Le[k] = R(0);
    __syncthreads();
  }
  for (int k = tid; k < M * N; k += NTHR) {
    const double l = p.L[size_t(b) * M * N + k];
    Ld[k] = narrow_pos<B>(l);
    Le[(k % M) + (k / M) * LES] = narrow_pos<R>(l);  // [n][m], column stride LES
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
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // This thread's TMEM strip: lane quarter (warp % 4), columns of its warp group.
  const unsigned tmrow =
      sc->tmem + (unsigned(32 * (warp & 3)) << 16) + unsigned((warp >> 2) * SLOTS * SCOL);
  auto tm_u = [&](int s) { return tmrow + unsigned(s * SCOL); };          // U (then 1/sigma^2)
  auto tm_phi = [&](int s) { return tmrow + unsigned(s * SCOL + WPR); };  // posterior
  const R eps = R(sc->eps);
  const double invT = 1.0 / double(T);
  const int bin_index = (p.seed_bin0 + b) % p.F;  // mix_seed index (fastfca.cpp:40)
  const bool record = p.record != 0;
  const bool silent = !(power > 0.0);
  const bool bal = p.normalize != 0;

  // ---- frame records
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
  auto hidx = [&](int n, int t) { return ((n / VE) * ps + t) * VE + (n % VE); };
  // Column k of the effective loadings as vectors.  Volatile shared loads:
  // re-read per frame from the broadcast bank instead of being hoisted into
  // 12 x M registers the frame loops cannot afford.
  auto load_le = [&](int k, R (&l)[M]) {
    const unsigned a = unsigned(__cvta_generic_to_shared(Le + k * LES));
    R v[LES];
#pragma unroll
    for (int q = 0; q < LES / VE; ++q) {
      if constexpr (VE == 4) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[q * 4]), "=f"(v[q * 4 + 1]), "=f"(v[q * 4 + 2]), "=f"(v[q * 4 + 3])
                     : "r"(a + 16 * q));
      } else {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(v[q * 2]), "=d"(v[q * 2 + 1])
                     : "r"(a + 16 * q));
      }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) l[m] = v[m];
  };
  // The first MC = M rounded up to even entries of column k (entries >= M are
  // the zero padding written at start-up).
  auto load_le_pad = [&](int k, R (&l)[(M + 1) & ~1]) {
    const unsigned a = unsigned(__cvta_generic_to_shared(Le + k * LES));
    R v[LES];
#pragma unroll
    for (int q = 0; q < LES / VE; ++q) {
      if constexpr (VE == 4) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[q * 4]), "=f"(v[q * 4 + 1]), "=f"(v[q * 4 + 2]), "=f"(v[q * 4 + 3])
                     : "r"(a + 16 * q));
      } else {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(v[q * 2]), "=d"(v[q * 2 + 1])
                     : "r"(a + 16 * q));
      }
    }
#pragma unroll
    for (int m = 0; m < ((M + 1) & ~1); ++m) l[m] = v[m];
  };
  // Mixture variances sigma^2(m) = eps + sum_k Le(m,k) h_k.
  auto mix_var = [&](const R (&h)[NHP * VE], R (&lh)[M]) {
    if constexpr (sizeof(R) == 4 && M % 2 == 0) {
      float2 a[M / 2];
#pragma unroll
      for (int q = 0; q < M / 2; ++q) a[q] = f2(eps, eps);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        R l[M];
        load_le(k, l);
#pragma unroll
        for (int q = 0; q < M / 2; ++q) a[q] = fma2s(f2(l[2 * q], l[2 * q + 1]), h[k], a[q]);
      }
#pragma unroll
      for (int q = 0; q < M / 2; ++q) lh[2 * q] = a[q].x, lh[2 * q + 1] = a[q].y;
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) lh[m] = eps;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        R l[M];
        load_le(k, l);
#pragma unroll
        for (int m = 0; m < M; ++m) lh[m] += l[m] * h[k];
      }
    }
  };
  auto frame_of = [&](int s, int owner) { return warp * 32 + owner + s * NTHR; };

  // ---------------------------------------------------- decorrelation pass --
  // U(j, t) = |w_j^H x_t|^2: M lanes per frame, lane j owns column j of W;
  // the frame's owner lane gathers its M values and stores them to TMEM.
  auto u_pass = [&]() {
    if constexpr (sizeof(R) == 4 && M % 2 != 0) {
      // fp32, odd M: one thread per frame, 8-byte loads, scalar complex algebra.
#pragma unroll 1
      for (int s = 0; s < nsl; ++s) {
        const int t0 = frame_of(s, lane);
        const int t = t0 < Tl ? t0 : 0;
        C xc[M];
#pragma unroll
        for (int c = 0; c < M; ++c) xc[c] = __ldg(xg + size_t(t) * M + c);
        R uo[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          R yr = R(0), yi = R(0);
#pragma unroll
          for (int c = 0; c < M; ++c) {
            const C w = Wr[c + m * M];  // y_m = sum_c conj(W(c, m)) x_c
            yr += w.x * xc[c].x + w.y * xc[c].y;
            yi += w.x * xc[c].y - w.y * xc[c].x;
          }
          uo[m] = yr * yr + yi * yi;
        }
        tm_store_rec<M, R>(tm_u(s), uo);
      }
      tm_wait_st();
    } else if constexpr (sizeof(R) == 4) {
      // fp32: one thread per frame (the owner loads its record, coalesced),
      // W columns from broadcast shared loads, packed FFMA2:
      // y_m = sum_c conj(W(c,m)) x_c = sum_c Re W(c,m) x_c + i sum_c Im W(c,m) (Im x_c, -Re x_c),
      // U(m) written straight to the frame's TMEM column.
#pragma unroll 1
      for (int s = 0; s < nsl; ++s) {
        const int t0 = frame_of(s, lane);
        const int t = t0 < Tl ? t0 : 0;
        float2 xc[M];
        const float4* xv = reinterpret_cast<const float4*>(xg + size_t(t) * M);
#pragma unroll
        for (int q = 0; q < M / 2; ++q) {
          const float4 v = __ldg(xv + q);
          xc[2 * q] = f2(v.x, v.y);
          xc[2 * q + 1] = f2(v.z, v.w);
        }
        const unsigned ta = tm_u(s);
        auto u_of = [&](int m) -> float {
          float wc[2 * M];  // column m of W: (re, im) pairs
          const unsigned a = unsigned(__cvta_generic_to_shared(Wr + m * M));
#pragma unroll
          for (int q = 0; q < M / 2; ++q)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(wc[4 * q]), "=f"(wc[4 * q + 1]), "=f"(wc[4 * q + 2]), "=f"(wc[4 * q + 3])
                         : "r"(a + 16 * q));
          float2 y1 = f2(0.f, 0.f), y2 = f2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < M; ++c) {
            y1 = fma2s(xc[c], wc[2 * c], y1);
            y2 = fma2s(xc[c], wc[2 * c + 1], y2);
          }
          const float yr = y1.x + y2.y, yi = y1.y - y2.x;
          return yr * yr + yi * yi;
        };
        if constexpr (INCR) {
          // U to the global scratch, four channels per 16-byte store.
          float4* uw = reinterpret_cast<float4*>(Ug + size_t(t) * M);
#pragma unroll 1
          for (int q = 0; q < M / 4; ++q) {
            const float4 v = make_float4(u_of(4 * q), u_of(4 * q + 1), u_of(4 * q + 2), u_of(4 * q + 3));
            if (t0 < Tl) uw[q] = v;
          }
        } else {
#pragma unroll 2
          for (int m = 0; m < M; ++m) {
            const float u = u_of(m);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(ta + unsigned(m)),
                         "r"(__float_as_uint(u))
                         : "memory");
          }
        }
      }
      tm_wait_st();
    } else {
    constexpr int FPB = 32 / M;  // frames per batch
    const int j = lane % M, g = lane / M;
    C wc[M];
#pragma unroll
    for (int c = 0; c < M; ++c) wc[c] = Wr[c + j * M];
#pragma unroll 1
    for (int s = 0; s < nsl; ++s) {
      R uo[M];
#pragma unroll
      for (int m = 0; m < M; ++m) uo[m] = R(0);
#pragma unroll
      for (int bb = 0; bb < 32 / FPB; ++bb) {
        const int t0 = frame_of(s, bb * FPB + g);
        const int t = t0 < Tl ? t0 : 0;
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
        // y = sum_c conj(w_c) x_c = sum wr x + i sum wi (xi, -xr)
        R yr, yi;
        if constexpr (sizeof(R) == 4) {
          float2 y1 = f2(0.f, 0.f), y2 = f2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < M; ++c) {
            y1 = fma2s(xc[c], wc[c].x, y1);
            y2 = fma2s(xc[c], wc[c].y, y2);
          }
          yr = y1.x + y2.y;
          yi = y1.y - y2.x;
        } else {
          yr = wc[0].x * xc[0].x + wc[0].y * xc[0].y;
          yi = wc[0].x * xc[0].y - wc[0].y * xc[0].x;
#pragma unroll
          for (int c = 1; c < M; ++c) {
            yr += wc[c].x * xc[c].x + wc[c].y * xc[c].y;
            yi += wc[c].x * xc[c].y - wc[c].y * xc[c].x;
          }
        }
        const R uval = yr * yr + yi * yi;
        // owner lane bb*FPB + g' takes channel m from lane g'*M + m
        const bool mine = (lane / FPB) == bb;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const R v = __shfl_sync(0xffffffffu, uval, (lane % FPB) * M + m);
          uo[m] = mine ? v : uo[m];
        }
      }
      tm_store_rec<M, R>(tm_u(s), uo);
    }
    tm_wait_st();
    }
  };

  // ---------------------------------------------------- EM sweep n --------
  // Ends with the per-warp partials in rd and ONE barrier.
  auto em_sweep = [&](int n, bool phis, R* rd) {
    R linv[M];
#pragma unroll
    for (int m = 0; m < M; ++m) linv[m] = (n > 0) ? Linv[m] : R(0);
    R lc[M];  // L_n (effective), constant over the sweep
    load_le(n, lc);
    R acc[KRED];
#pragma unroll
    for (int k = 0; k < KRED; ++k) acc[k] = R(0);
    if constexpr (INCR) {
      // fp32, incremental variances: sigma^2 (tensor memory) takes the row
      // n-1 update as sigma^2 += L_new h_new - L_old h_old before it is used;
      // U comes from the global scratch.  Two frame slots per trip.
      constexpr int MP = M / 2;
      float2 lc2[MP], li2[MP], ln2[MP], lo2[MP];
      {
        R lnw[M];
        load_le(n > 0 ? n - 1 : 0, lnw);  // column n-1 after its update
#pragma unroll
        for (int q = 0; q < MP; ++q) {
          lc2[q] = f2(lc[2 * q], lc[2 * q + 1]);
          li2[q] = f2(linv[2 * q], linv[2 * q + 1]);
          ln2[q] = f2(lnw[2 * q], lnw[2 * q + 1]);
          lo2[q] = n > 0 ? f2(Lprev[2 * q], Lprev[2 * q + 1]) : f2(0.f, 0.f);
        }
      }
      float2 a2[MP], p2[MP];
#pragma unroll
      for (int q = 0; q < MP; ++q) a2[q] = f2(0.f, 0.f), p2[q] = f2(0.f, 0.f);
      float hacc = 0.f;
      // FS frame slots per trip: independent dependency chains (tensor-memory
      // and L2 loads, reciprocals, stores) in flight per warp.
      constexpr int FS = FFCA_BIG_FS;
      static_assert(SLOTS % FS == 0, "frame slots per trip");
#if FFCA_BIG_PREFETCH
      float4 un[FS][M / 4];  // the next trip's U, fetched (L2) while this trip computes
      auto fetch_u = [&](int s) {
#pragma unroll
        for (int f = 0; f < FS; ++f) {
          const int t0 = frame_of(s + f, lane);
          const float4* uw = reinterpret_cast<const float4*>(Ug + size_t(t0 < Tl ? t0 : 0) * M);
#pragma unroll
          for (int q = 0; q < M / 4; ++q) un[f][q] = __ldcg(uw + q);
        }
      };
      fetch_u(0);
#endif
#pragma unroll 1
      for (int s = 0; s < nsl; s += FS) {
        int t[FS];
        bool ok[FS];
        float2 u[FS][MP], lh[FS][MP];
#pragma unroll
        for (int f = 0; f < FS; ++f) {
          const int t0 = frame_of(s + f, lane);
          ok[f] = t0 < Tl;
          t[f] = ok[f] ? t0 : 0;
#if FFCA_BIG_PREFETCH
#pragma unroll
          for (int q = 0; q < M / 4; ++q)
            u[f][2 * q] = f2(un[f][q].x, un[f][q].y), u[f][2 * q + 1] = f2(un[f][q].z, un[f][q].w);
#else
          const float4* uw = reinterpret_cast<const float4*>(Ug + size_t(t[f]) * M);
#pragma unroll
          for (int q = 0; q < M / 4; ++q) {
            const float4 v = __ldcg(uw + q);
            u[f][2 * q] = f2(v.x, v.y), u[f][2 * q + 1] = f2(v.z, v.w);
          }
#endif
        }
#if FFCA_BIG_PREFETCH
        if (s + FS < nsl) fetch_u(s + FS);
#endif
#pragma unroll
        for (int f = 0; f < FS; ++f) {
          float sg[M], pp[M];
          tm_load_rec2<M, R>(tm_u(s + f), sg, pp);
#pragma unroll
          for (int q = 0; q < MP; ++q) lh[f][q] = f2(sg[2 * q], sg[2 * q + 1]);
          if (n > 0) {  // H row n-1 (fastfca.cpp:95-97), then its change in sigma^2
            float2 s2 = fmul2(f2(pp[0], pp[1]), li2[0]);
#pragma unroll
            for (int q = 1; q < MP; ++q) s2 = fma2(f2(pp[2 * q], pp[2 * q + 1]), li2[q], s2);
            float hn1 = (s2.x + s2.y) * (1.f / M);
            hn1 = hn1 > tiny<R>() ? hn1 : tiny<R>();
            const float hold = Hs[hidx(n - 1, t[f])];
            if (ok[f]) Hs[hidx(n - 1, t[f])] = hn1;
            hacc += ok[f] ? hn1 : 0.f;
#pragma unroll
            for (int q = 0; q < MP; ++q)
              lh[f][q] = fma2s(ln2[q], hn1, fma2s(lo2[q], -hold, lh[f][q]));
          }
        }
#pragma unroll
        for (int f = 0; f < FS; ++f) {
          const float hn = Hs[hidx(n, t[f])];
          const float ihn = ok[f] ? rcp_fast(hn) : 0.f;
          const float okf = ok[f] ? 1.f : 0.f;
          float v[M], sg[M];
#pragma unroll
          for (int q = 0; q < MP; ++q) {
            const float2 ln = fmul2s(lc2[q], hn);                      // L_n H_n
            const float2 rl = f2(rcp_fast(lh[f][q].x), rcp_fast(lh[f][q].y));
            const float2 gg = fmul2(ln, rl);                           // G
            const float2 w = fma2(gg, u[f][q], fneg2(ln));             // G U - L_n H_n
            const float2 vv = fma2(gg, w, ln);                         // G^2 U + (1 - G) L_n H_n
            v[2 * q] = vv.x, v[2 * q + 1] = vv.y;
            sg[2 * q] = lh[f][q].x, sg[2 * q + 1] = lh[f][q].y;
            a2[q] = fma2s(vv, ihn, a2[q]);
            if (phis) p2[q] = fma2s(vv, okf, p2[q]);
          }
          tm_store_rec2<M>(tm_u(s + f), sg, v);
        }
      }
#pragma unroll
      for (int q = 0; q < MP; ++q) {
        acc[2 * q] = a2[q].x, acc[2 * q + 1] = a2[q].y;
        acc[M + 1 + 2 * q] = p2[q].x, acc[M + 2 + 2 * q] = p2[q].y;
      }
      acc[M] = hacc;
    } else if constexpr (sizeof(R) == 4 && (M % 2 == 0 || FFCA_BIG_PACK_ODD != 0)) {
      // fp32: two frame slots per trip share the loading-column loads, and
      // the per-channel algebra runs on packed pairs (FFMA2 / FMUL2); an odd
      // slot count ends with a one-slot trip.  Odd M is padded to MC = M + 1
      // channels whose loadings, posteriors and powers are zero (their
      // variance is eps, so every padded quantity is an exact 0).  A slot
      // past the CTA's frames computes on frame 0; its H store is skipped and
      // its contributions are zeroed through the weights (okf, ihn = 0).
      constexpr int MC = (M + 1) & ~1, MP = MC / 2;
      float2 lc2[MP], li2[MP];
      {
        float lcp[MC];
        load_le_pad(n, lcp);
#pragma unroll
        for (int q = 0; q < MP; ++q) {
          lc2[q] = f2(lcp[2 * q], lcp[2 * q + 1]);
          li2[q] = f2(linv[2 * q], (2 * q + 1 < M) ? linv[(2 * q + 1 < M) ? 2 * q + 1 : 0] : 0.f);
        }
      }
      float2 a2[MP], p2[MP];
#pragma unroll
      for (int q = 0; q < MP; ++q) a2[q] = f2(0.f, 0.f), p2[q] = f2(0.f, 0.f);
      float hacc = 0.f;
      auto trip = [&](auto fsc, int s) {
        constexpr int FS = decltype(fsc)::value;
        int t[FS];
        bool ok[FS];
        float2 u[FS][MP], ph[FS][MP], lh[FS][MP];
        float h[FS][NHP * VE];
#pragma unroll
        for (int f = 0; f < FS; ++f) {
          const int t0 = frame_of(s + f, lane);
          ok[f] = t0 < Tl;
          t[f] = ok[f] ? t0 : 0;
          float uu[M], pp[M];
          tm_load_rec2<M, R>(tm_u(s + f), uu, pp);
#pragma unroll
          for (int q = 0; q < MP; ++q) {
            u[f][q] = f2(uu[2 * q], (2 * q + 1 < M) ? uu[(2 * q + 1 < M) ? 2 * q + 1 : 0] : 0.f);
            ph[f][q] = f2(pp[2 * q], (2 * q + 1 < M) ? pp[(2 * q + 1 < M) ? 2 * q + 1 : 0] : 0.f);
          }
          if (n > 0) {  // H row n-1 (fastfca.cpp:95-97), stored before the row is read
            float2 s2 = fmul2(ph[f][0], li2[0]);
#pragma unroll
            for (int q = 1; q < MP; ++q) s2 = fma2(ph[f][q], li2[q], s2);
            float hn1 = (s2.x + s2.y) * (1.f / M);
            hn1 = hn1 > tiny<R>() ? hn1 : tiny<R>();
            if (ok[f]) Hs[hidx(n - 1, t[f])] = hn1;
            hacc += ok[f] ? hn1 : 0.f;
          }
          load_h(t[f], h[f]);
#pragma unroll
          for (int q = 0; q < MP; ++q) lh[f][q] = f2(eps, eps);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          float l[MC];
          load_le_pad(k, l);
#pragma unroll
          for (int q = 0; q < MP; ++q) {
            const float2 lq = f2(l[2 * q], l[2 * q + 1]);
#pragma unroll
            for (int f = 0; f < FS; ++f) lh[f][q] = fma2s(lq, h[f][k], lh[f][q]);
          }
        }
#pragma unroll
        for (int f = 0; f < FS; ++f) {
          const float hn = Hs[hidx(n, t[f])];
          const float ihn = ok[f] ? rcp_fast(hn) : 0.f;
          const float okf = ok[f] ? 1.f : 0.f;
          R v[M];
#pragma unroll
          for (int q = 0; q < MP; ++q) {
            const float2 ln = fmul2s(lc2[q], hn);                      // L_n H_n
            const float2 rl = f2(rcp_fast(lh[f][q].x), rcp_fast(lh[f][q].y));
            const float2 gg = fmul2(ln, rl);                           // G
            const float2 w = fma2(gg, u[f][q], fneg2(ln));             // G U - L_n H_n
            const float2 vv = fma2(gg, w, ln);                         // G^2 U + (1 - G) L_n H_n
            v[2 * q] = vv.x;
            if (2 * q + 1 < M) v[(2 * q + 1 < M) ? 2 * q + 1 : 0] = vv.y;
            a2[q] = fma2s(vv, ihn, a2[q]);
            if (phis) p2[q] = fma2s(vv, okf, p2[q]);
          }
          tm_store_rec<M, R>(tm_phi(s + f), v);
        }
      };
      {
        int s = 0;
#pragma unroll 1
        for (; s + 2 <= nsl; s += 2) trip(std::integral_constant<int, 2>{}, s);
        if (s < nsl) trip(std::integral_constant<int, 1>{}, s);
      }
#pragma unroll
      for (int q = 0; q < MP; ++q) {
        acc[2 * q] = a2[q].x;
        acc[M + 1 + 2 * q] = p2[q].x;
        if (2 * q + 1 < M) {
          acc[(2 * q + 1 < M) ? 2 * q + 1 : 0] = a2[q].y;
          acc[(2 * q + 1 < M) ? M + 2 + 2 * q : 0] = p2[q].y;
        }
      }
      acc[M] = hacc;
    } else {
#pragma unroll 1
    for (int s = 0; s < nsl; ++s) {
      const int t0 = frame_of(s, lane);
      const bool ok = t0 < Tl;
      const int t = ok ? t0 : 0;
      R u[M], php[M];
      tm_load_rec2<M, R>(tm_u(s), u, php);
      if (n > 0) {  // H row n-1 (fastfca.cpp:95-97), stored before the row is read
        R sum = php[0] * linv[0];
#pragma unroll
        for (int m = 1; m < M; ++m) sum += php[m] * linv[m];
        R hn1 = sum * R(1.0 / M);
        hn1 = hn1 > tiny<R>() ? hn1 : tiny<R>();
        if (ok) Hs[hidx(n - 1, t)] = hn1;
        acc[M] += ok ? hn1 : R(0);
      }
      R h[NHP * VE], lh[M];
      load_h(t, h);
      mix_var(h, lh);
      const R hn = Hs[hidx(n, t)];
      const R ihn = rcp_fast(hn);
      R ph[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const R lnhn = lc[m] * hn;
        const R gg = lnhn * rcp_fast(lh[m]);
        R v = gg * (gg * u[m] - lnhn) + lnhn;  // G^2 U + (1 - G) L_n H_n
        v = ok ? v : R(0);
        ph[m] = v;
        acc[m] += v * ihn;
        if (phis) acc[M + 1 + m] += v;
      }
      tm_store_rec<M, R>(tm_phi(s), ph);
    }
    }
    tm_wait_st();
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
  // Every warp calls this; returns lane k's total (0 for k >= K).  Only warp
  // 0 writes remote slots, so only it needs release semantics.
  auto reduce_tot = [&](const R* rd, int K, int cbuf) -> R {
    R tot = (lane < K) ? tree_sum_any<NW>(rd, KRED, lane) : R(0);
    if constexpr (CL) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      double* slot = cx + cbuf * (csize * KRED) + crank * KRED;
      if (warp == 0) {
        if (lane < K)
          for (int r = 0; r < csize; ++r) cl.map_shared_rank(slot, r)[lane] = double(tot);
        cluster_arrive();
      } else {
        cluster_arrive_relaxed();
      }
      cluster_wait();
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
#pragma unroll 1
    for (int s = 0; s < nsl; ++s) {
      const int t0 = frame_of(s, lane);
      const bool ok = t0 < Tl;
      const int t = ok ? t0 : 0;
      R u[M], php[M];
      tm_load_rec2<M, R>(tm_u(s), u, php);
      if constexpr (INCR) {  // the U slot holds sigma^2: U comes from the global scratch
        const float4* uw = reinterpret_cast<const float4*>(Ug + size_t(t) * M);
#pragma unroll
        for (int q = 0; q < M / 4; ++q) {
          const float4 v = __ldcg(uw + q);
          u[4 * q] = v.x, u[4 * q + 1] = v.y, u[4 * q + 2] = v.z, u[4 * q + 3] = v.w;
        }
      }
      if (finish) {
        R sum = php[0] * linv[0];
#pragma unroll
        for (int m = 1; m < M; ++m) sum += php[m] * linv[m];
        R hn1 = sum * R(1.0 / M);
        hn1 = hn1 > tiny<R>() ? hn1 : tiny<R>();
        if (ok) Hs[hidx(N - 1, t)] = hn1;
      }
      R h[NHP * VE], lh[M];
      load_h(t, h);
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
      if constexpr (INCR) {
        // exact sigma^2 for the next iteration's sweeps, 1/sigma^2 (the
        // covariance weights) over the spent posterior
        tm_store_rec2<M>(tm_u(s), lh, r);
      } else {
        tm_store_rec<M, R>(tm_u(s), r);
      }
    }
    tm_wait_st();
  };

  // ------------------------------------------ A2: weighted covariances --
  // Lane a of a frame's GS lanes forms x_a conj(x_{a+d}), d = 0..M/2, and
  // accumulates them against weights [mh*MW, (mh+1)*MW) shuffled from the
  // frame's owner lane.  Then reduces the products (and the NLL partials) to
  // CTA totals in ex[], cluster totals in qraw[] (packed Hermitian, the
  // layout the IP reads) and nll_tot.
  auto a2_pass = [&](bool want_q, const R (&nacc)[M + 1], double (&nll_tot)[M + 1]) {
    constexpr int FPB = 32 / GS;  // frames per batch
    const int a = lane % ML, mh = (lane / ML) % MS, g = lane / GS;
    const bool live = a < M;  // odd M: the padding lane of each frame group idles
    R acc[KAP];  // [jj * MW + mm], zero padding up to KAP
#pragma unroll
    for (int k = 0; k < KAP; ++k) acc[k] = R(0);
    int coff[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) coff[d] = live ? (a + d) % M : 0;
    if (want_q) {
#pragma unroll 1
      for (int s = 0; s < nsl; ++s) {
        R ro[M];  // this lane's own frame weights 1/sigma^2
        tm_load_rec<M, R>(INCR ? tm_phi(s) : tm_u(s), ro);
#pragma unroll(kA2Unroll)
        for (int bb = 0; bb < 32 / FPB; ++bb) {
          const int owner = bb * FPB + g;
          const int t0 = frame_of(s, owner);
          const bool ok = t0 < Tl;
          const C* xf = xg + size_t(ok ? t0 : 0) * M;
          C xr[D + 1];
#pragma unroll
          for (int d = 0; d <= D; ++d) xr[d] = xf[coff[d]];
          R P[NP];
          P[0] = xr[0].x * xr[0].x + xr[0].y * xr[0].y;
#pragma unroll
          for (int d = 1; d <= D; ++d) {
            // x_a conj(x_c): Re = ar cr + ai ci, Im = ai cr - ar ci
            P[2 * d - 1] = xr[0].x * xr[d].x + xr[0].y * xr[d].y;
            P[2 * d] = xr[0].y * xr[d].x - xr[0].x * xr[d].y;
          }
          R rw[MW];
#pragma unroll
          for (int mm = 0; mm < MW; ++mm) {
            R rm;
            if constexpr (MS == 1) {
              rm = __shfl_sync(0xffffffffu, ro[mm], owner);
            } else {
              const R r0 = __shfl_sync(0xffffffffu, ro[mm], owner);
              const R r1 = __shfl_sync(0xffffffffu, ro[MW + mm], owner);
              rm = mh == 0 ? r0 : r1;
            }
            rw[mm] = (ok && live) ? rm : R(0);
          }
          if constexpr (sizeof(R) == 4 && MW % 2 == 0 && FFCA_BIG_A2_SCALAR == 0) {
            // acc pairs (jj, mm), (jj, mm + 1): weights packed, product broadcast
#pragma unroll
            for (int jj = 0; jj < NP; ++jj)
#pragma unroll
              for (int q = 0; q < MW / 2; ++q) {
                float2 a2 = f2(acc[jj * MW + 2 * q], acc[jj * MW + 2 * q + 1]);
                a2 = fma2s(f2(rw[2 * q], rw[2 * q + 1]), P[jj], a2);
                acc[jj * MW + 2 * q] = a2.x;
                acc[jj * MW + 2 * q + 1] = a2.y;
              }
          } else {
#pragma unroll
            for (int mm = 0; mm < MW; ++mm)
#pragma unroll
              for (int jj = 0; jj < NP; ++jj) acc[jj * MW + mm] += P[jj] * rw[mm];
          }
        }
      }
    }
    FFCA_BTIC(5);
    // Lanes of equal role (lane mod GS) hold partials of the same products:
    // reduce-scatter over the frame groups of the warp.
    int base = 0;
    int cnt = KAP;
#pragma unroll
    for (int o = 16; o >= GS; o >>= 1) {
      const bool up = (lane & o) != 0;
      const int h2 = cnt / 2;  // KAP halves evenly down to CNT
#pragma unroll
      for (int i = 0; i < KAP / 2; ++i) {
        if (i < h2) {
          const R send = up ? acc[i] : acc[i + h2];
          const R keep = up ? acc[i + h2] : acc[i];
          acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (up) base += h2;
      cnt = h2;
    }
    // NLL partials of A1 (thread-per-frame accumulators).
    R* rd = red;  // EM partial buffers are idle here
    warp_reduce_store<M + 1>(nacc, rd + warp * KRED, lane);
    // Cross-warp tree through the scratch (fixed order): at step h, warps
    // [h, 2h) publish, warps [0, h) add.  Warp 0 ends with the CTA totals.
#pragma unroll 1
    for (int h = HW; h >= 1; h >>= 1) {
      if (want_q && warp >= h && warp < 2 * h && warp < NW) {
        R* dst = gscr + ((warp - h) * 32 + lane) * CNT;
#pragma unroll
        for (int i = 0; i < CNT; ++i) dst[i] = acc[i];
      }
      __syncthreads();
      if (want_q && warp < h && warp + h < NW) {
        const R* src = gscr + (warp * 32 + lane) * CNT;
#pragma unroll
        for (int i = 0; i < CNT; ++i) acc[i] += src[i];
      }
      __syncthreads();
    }
    (void)PW;
    // CTA totals (warp 0) in the packed layout: ex[m*M*M + (a*M + c)]
    // (a < c: Re at a*M+c, Im at c*M+a; diagonal at a*M+a), then the NLL.
    if (warp == 0) {
      if (want_q) {
        const int ra = lane % ML, rmh = (lane / ML) % MS;
#pragma unroll
        for (int i = 0; i < CNT; ++i) {
          const int k = base + i;
          const int j = k / MW, mm = k - j * MW;
          const int m = rmh * MW + mm;
          int idx = -1;
          double val = double(acc[i]);
          if (k >= KA || ra >= M) {
            idx = -1;  // padding
          } else if (j == 0) {
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
      if (lane <= M) ex[KQ + lane] = double(tree_sum_any<NW>(rd, KRED, lane));
    }
    __syncthreads();
    // Cluster totals, rank order (every CTA the same bits).
    const int nq = want_q ? KQ : 0;
    if constexpr (CL) {
      namespace cg = cooperative_groups;
      cg::cluster_group cl = cg::this_cluster();
      cluster_arrive();
      cluster_wait();
      for (int o = tid; o < nq + M + 1; o += NTHR) {
        const int oo = o < nq ? o : KQ + (o - nq);
        double s = 0.0;
        for (int r = 0; r < csize; ++r) s += cl.map_shared_rank(ex, r)[oo];
        if (o < nq) qraw[o] = s;
        else ex[KQ + M + 1 + (o - nq)] = s;  // cluster NLL totals after the CTA ones
      }
      cluster_arrive_relaxed();  // done reading the others' ex[] (its wait comes later)
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
      Le[m + n * LES] = R((l > B(0) && !(le > B(0))) ? tiny<B>() : le);
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

  // IP sweep, called by EVERY thread: Q^{-1} and (W^H)^{-1} in parallel
  // (ip_fast.cuh), then the sequential column updates on warp 0; on a failed
  // acceptance test warp 0 reruns the sweep the reference's way
  // (ip_update_warp_reg: LU-equivalent solves, residual test, seeded
  // restart) from the saved W.  Leaves log|det W|^2 of the result in
  // sc->logdet0 / sc->ldok for the next trace entry.
  auto run_ip = [&](unsigned long long seed) {
    ip_fast_prep<M, R, B>(warp, lane, Wd, wsc, qraw, invT, ipf, wsave);
    __syncthreads();
    if (warp == 0) {
      double ldn = 0.0;
      const bool fast_ok = ip_fast_sweep<M, R>(lane, Wd, ipf, ldn);
      if (fast_ok) {
        if (lane == 0) {
          sc->logdet0 = ldn;
          sc->ldok = 1;
        }
      } else {
        for (int k = lane; k < M * M; k += 32) Wd[k] = wsave[k];
        __syncwarp();
        int bad = -1;
        const bool ok = ip_update_warp_reg<M, R>(Wd, qraw, invT, seed, bin_index, rng, ipscr, lane, bad);
        if (lane == 0 && !ok) {
          sc->status = kStatusIpSingular | (bad << 8);
          sc->stop = 1;
        }
        __syncwarp();
        double ld = 0.0;
        const bool lok = warp_log_abs_det2<M, R>(Wd, ldscr, lane, ld);
        if (lane == 0) {
          sc->logdet0 = ld;
          sc->ldok = lok ? 1 : 0;
        }
      }
      __syncwarp();
      for (int k = lane; k < M * M; k += 32) Wr[k] = mkc<R>(R(Wd[k].x), R(Wd[k].y));
    }
  };

  // -------------------------------------------------------------- driver --
  R nacc[M + 1];
  double ntot[M + 1];
  // Initial decorrelated powers, variances, NLL of the init and the first Q.
  u_pass();
  a1_pass(false, nacc);
  a2_pass(p.iters > 0 && !silent, nacc, ntot);
  if (warp == 0) {
    if (record) {
      double ld = 0.0;
      const bool ok = warp_log_abs_det2<M, R>(Wd, ldscr, lane, ld);
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
  }
  __syncthreads();
  if (!sc->stop && p.iters > 0) run_ip(p.seed);
  if constexpr (CL) cluster_wait();  // pairs the arrive of a2_pass
  __syncthreads();
  FFCA_BTIC(9);
  bool touched = false;
  if (!sc->stop) {
    for (int it = 0; it < p.iters; ++it) {
      FFCA_BTIC(7);
      u_pass();
      FFCA_BTIC(0);
      // EM sweeps (fastfca.cpp:80-99).  The last sweep also sums Phi (balance).
      auto em_step = [&](int n) {
        const bool phis = bal && n == N - 1;
        R* rd = red + (n & 1) * NW * KRED;
        const R lold = lane < M ? Le[lane + n * LES] : R(0);  // effective column n before its update
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
          if (!phis) Le[m + n * LES] = lr;
          if constexpr (INCR) Lprev[m] = lold;
          Linv[m] = rcp_fast(lr);
          if (phis) psum[m] = B(pss);
        }
        if (lane == 0 && n >= 1) hsumv[n - 1] = B(hs);
        __syncwarp();
        FFCA_BTIC(2);
      };
#pragma unroll 1
      for (int n = 0; n < N; ++n) em_step(n);
      balance_all(bal);
      FFCA_BTIC(3);
      touched = true;
      const bool more = it + 1 < p.iters;
      a1_pass(true, nacc);
      FFCA_BTIC(4);
      a2_pass(more, nacc, ntot);
      FFCA_BTIC(6);
      if (warp == 0 && lane == 0 && record) {
        if (!sc->ldok) {  // log_abs_det2 throws on a singular W (sigmodel.cpp:124-125)
          sc->status = kStatusSingularW;
          sc->stop = 1;
        }
        const double v = nll_value(ntot, sc->logdet0 - sc->logs);
        if (lead) p.nll[size_t(it + 1) * p.nll_stride + p.prob_offset + b] = v;
      }
      __syncthreads();
      if (more && !sc->stop) {
        run_ip(p.seed + (unsigned long long)(it + 1));
      } else if (warp == 0) {
        for (int k = lane; k < M * M; k += 32) {  // the last balance's W scales
          const double c = double(wsc[k / M]);
          Wd[k].x *= c;
          Wd[k].y *= c;
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
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(sc->tmem), "n"(TMCOLS));
  if constexpr (CL) {  // no CTA exits while others may read its shared memory
    cluster_arrive();
    cluster_wait();
  }
}

}  // namespace ffca
