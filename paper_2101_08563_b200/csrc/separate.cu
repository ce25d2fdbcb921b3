// separate.cu -- fastfca_separate (reference src/fastfca.cpp:205-223): the
// decomposed multichannel Wiener filter.  Per frame
//     y = W^H x,   g_n = L_n H_n / floor_positive(L H)   (source_gain :74-78,
//     sigmodel.cpp:10-15, no eps),   c_n = (W^H)^{-1} (g_n .* y),
// written as images[n][p][t][m] (the reference's N Spectrograms).
//
// Write-bound: 8M + 4N bytes read and 8NM bytes written per frame in the fp32
// path (c3: 880 B, 12.6 GB of images).  Two launches:
//   sep_prep_kernel   one CTA per bin: the bin's constants -- W, (W^H)^{-1}
//                     (fp64 Gauss-Jordan with partial pivoting, one warp), L,
//                     and the floor 1e-12 mean(L H), whose mean needs only
//                     the N row sums of H (mean(LH) = sum_n colsum L_n rowsum
//                     H_n / (M T)) -- into a small per-bin record.
//   sep_apply_kernel  CTAs over (bin, frame chunk), one thread per frame, no
//                     reduction: the grid fills the machine for any T.
// The per-source product is reassociated for the fp32 path: with
// B(r,k) = Ainv(r,k) y_k formed once per frame, c_n(r) = sum_k B(r,k) g_n(k)
// is one packed complex-times-real FMA (FFMA2) per term instead of a complex
// multiply-add -- half the FP32 work of the per-source M x M product, which
// at M = 8, N = 12 would otherwise cost as much time as the HBM traffic.
#include "aux_kernels.cuh"
#include "internal.hpp"

namespace ffca {

namespace {

// Per-bin record, in the compute type R (reals), every section starting on a
// 16-byte boundary: W [2 M^2] col-major, Ainv = (W^H)^{-1} [2 M^2] col-major,
// L [M N] col-major, L again with every entry doubled [2 M N] (ready-made
// packed-FMA operands), floor.
__host__ __device__ constexpr int pad4(int n) { return (n + 3) & ~3; }
__host__ __device__ constexpr int sep_off_ainv(int M) { return pad4(2 * M * M); }
__host__ __device__ constexpr int sep_off_l(int M) { return 2 * pad4(2 * M * M); }
__host__ __device__ constexpr int sep_off_ld(int M, int N) { return sep_off_l(M) + pad4(M * N); }
__host__ __device__ constexpr int sep_off_floor(int M, int N) { return sep_off_ld(M, N) + pad4(2 * M * N); }
__host__ __device__ constexpr int sep_rec_size(int M, int N) { return sep_off_floor(M, N) + 4; }

constexpr int kPrepThreads = 128;

template <int M, typename R>
__global__ void __launch_bounds__(kPrepThreads)
    sep_prep_kernel(const double2* __restrict__ W, const double* __restrict__ L,
                    const R* __restrict__ H, int N, int T, R* __restrict__ rec) {
  __shared__ double2 aug[M * 2 * M];  // [A | I], column-major, A = W^H
  __shared__ double red[kPrepThreads];
  __shared__ double rowsum[16];
  const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  R* out = rec + size_t(p) * sep_rec_size(M, N);
  const double2* Wp = W + size_t(p) * M * M;
  const double* Lp = L + size_t(p) * M * N;
  // ---- row sums of H: thread (n, j) walks frames j, j + G, ... of row n.
  {
    const R* hp = H + size_t(p) * N * T;
    const int G = kPrepThreads / N;  // frames per step
    double acc = 0.0;
    if (tid < G * N) {
      const int n = tid % N;
      for (int t = tid / N; t < T; t += G) acc += double(hp[size_t(t) * N + n]);
    }
    red[tid] = acc;
    __syncthreads();
    if (tid < N) {
      double s = 0.0;
      for (int j = 0; j < G; ++j) s += red[j * N + tid];  // fixed order
      rowsum[tid] = s;
    }
  }
  // ---- (W^H)^{-1}: warp 0, lane c owns column c of [A | I].
  if (warp == 0) {
    for (int e = lane; e < M * M; e += 32) {
      const int r = e % M, c = e / M;
      const double2 w = Wp[c + r * M];            // W(c, r)
      aug[r + c * M] = make_double2(w.x, -w.y);   // (W^H)(r, c)
      aug[r + (M + c) * M] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
    __syncwarp();
    for (int k = 0; k < M; ++k) {
      // pivot: largest modulus in column k, rows k.., lowest row on ties
      int piv = k;
      double best = cabs2(aug[k + k * M]);
      for (int r = k + 1; r < M; ++r) {
        const double v = cabs2(aug[r + k * M]);
        if (v > best) best = v, piv = r;
      }
      double2 f[M];  // column k before this step (row-swapped)
#pragma unroll
      for (int r = 0; r < M; ++r) f[r] = aug[(r == k ? piv : (r == piv ? k : r)) + k * M];
      __syncwarp();
      if (lane < 2 * M) {
        double2* col = aug + lane * M;
        if (piv != k) {
          const double2 t = col[k];
          col[k] = col[piv];
          col[piv] = t;
        }
        const double2 pk = cdiv(col[k], f[k]);
        col[k] = pk;
#pragma unroll
        for (int r = 0; r < M; ++r)
          if (r != k) col[r] = csub(col[r], cmul(f[r], pk));
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < M * M; e += kPrepThreads) {
    const double2 w = Wp[e];
    out[2 * e] = R(w.x), out[2 * e + 1] = R(w.y);
    const double2 a = aug[e + M * M];
    out[sep_off_ainv(M) + 2 * e] = R(a.x), out[sep_off_ainv(M) + 2 * e + 1] = R(a.y);
  }
  for (int e = tid; e < M * N; e += kPrepThreads) {
    const R l = R(Lp[e]);
    out[sep_off_l(M) + e] = l;
    out[sep_off_ld(M, N) + 2 * e] = l, out[sep_off_ld(M, N) + 2 * e + 1] = l;
  }
  if (tid == 0) {
    double tot = 0.0;
    for (int n = 0; n < N; ++n) {
      double cs = 0.0;
      for (int m = 0; m < M; ++m) cs += double(R(Lp[m + n * M]));
      tot += cs * rowsum[n];
    }
    const double mean = tot / (double(M) * double(T));
    const double fl = mean > 0.0 ? 1e-12 * mean : 1e-300;  // sigmodel.cpp:10-15
    out[sep_off_floor(M, N)] = narrow_pos<R>(fl);
  }
}

// ------------------------------------------------------------ helpers --
__device__ __forceinline__ float2 mac_s(float2 a, float s, float2 c) {  // c + a s
  return __ffma2_rn(a, make_float2(s, s), c);
}
__device__ __forceinline__ float2 mul_s(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }

// COUNT reals from a record-aligned address with the widest loads the record
// size allows (records are COUNT * sizeof(R) bytes apart from an aligned base).
template <int COUNT, typename R>
__device__ __forceinline__ void load_rec(const R* __restrict__ p, R (&v)[COUNT]) {
  constexpr int BYTES = COUNT * int(sizeof(R));
  if constexpr (BYTES % 16 == 0) {
    constexpr int PER = 16 / int(sizeof(R));
    using V = typename std::conditional<sizeof(R) == 4, float4, double2>::type;
#pragma unroll
    for (int q = 0; q < BYTES / 16; ++q) {
      const V t = __ldg(reinterpret_cast<const V*>(p) + q);
      if constexpr (PER == 4) {
        v[4 * q] = t.x, v[4 * q + 1] = t.y, v[4 * q + 2] = t.z, v[4 * q + 3] = t.w;
      } else {
        v[2 * q] = t.x, v[2 * q + 1] = t.y;
      }
    }
  } else if constexpr (BYTES % 8 == 0 && sizeof(R) == 4) {
#pragma unroll
    for (int q = 0; q < BYTES / 8; ++q) {
      const float2 t = __ldg(reinterpret_cast<const float2*>(p) + q);
      v[2 * q] = t.x, v[2 * q + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < COUNT; ++q) v[q] = __ldg(p + q);
  }
}

// COUNT reals from shared memory at an ALIGN-byte aligned address.
// Volatile loads: the per-bin constants are re-read from the broadcast bank
// where they are used instead of being hoisted out of the frame loop into
// hundreds of registers (and spilled).
template <int COUNT, int ALIGN, typename R>
__device__ __forceinline__ void load_sh(const R* p, R (&v)[COUNT]) {
  constexpr int BYTES = COUNT * int(sizeof(R));
  if constexpr (sizeof(R) == 4) {
    const unsigned a = unsigned(__cvta_generic_to_shared(p));
    if constexpr (BYTES % 16 == 0 && ALIGN % 16 == 0) {
#pragma unroll
      for (int q = 0; q < BYTES / 16; ++q)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v[4 * q]), "=f"(v[4 * q + 1]), "=f"(v[4 * q + 2]), "=f"(v[4 * q + 3])
                     : "r"(a + 16 * q));
    } else if constexpr (BYTES % 8 == 0 && ALIGN % 8 == 0) {
#pragma unroll
      for (int q = 0; q < BYTES / 8; ++q)
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                     : "=f"(v[2 * q]), "=f"(v[2 * q + 1])
                     : "r"(a + 8 * q));
    } else {
#pragma unroll
      for (int q = 0; q < COUNT; ++q)
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[q]) : "r"(a + 4 * q));
    }
  } else {
#pragma unroll
    for (int q = 0; q < COUNT; ++q) v[q] = p[q];
  }
}

// CNT consecutive complex outputs (streaming stores: the images are written
// once and never re-read by this kernel).  V16: the address is 16-byte aligned.
template <int CNT, bool V16, typename OutC, typename C>
__device__ __forceinline__ void store_out(OutC* __restrict__ o, const C (&c)[CNT]) {
  if constexpr (sizeof(OutC) == 8 && CNT % 2 == 0 && V16) {
#pragma unroll
    for (int q = 0; q < CNT / 2; ++q)
      __stcs(reinterpret_cast<float4*>(o) + q,
             make_float4(float(c[2 * q].x), float(c[2 * q].y), float(c[2 * q + 1].x),
                         float(c[2 * q + 1].y)));
  } else if constexpr (sizeof(OutC) == 8) {
#pragma unroll
    for (int q = 0; q < CNT; ++q)
      __stcs(reinterpret_cast<float2*>(o) + q, make_float2(float(c[q].x), float(c[q].y)));
  } else {
#pragma unroll
    for (int q = 0; q < CNT; ++q)
      __stcs(reinterpret_cast<double2*>(o) + q, make_double2(double(c[q].x), double(c[q].y)));
  }
}

constexpr int kApplyThreads = 256;

// NC: compile-time source count (0: runtime N <= 16, H read source by source).
template <int M, int NC, typename R, typename OutC>
__global__ void __launch_bounds__(kApplyThreads, 2)
    sep_apply_kernel(const cplx_t<R>* __restrict__ x, const R* __restrict__ H,
                     const R* __restrict__ rec, int P, int Nrt, int T, int chunk, int nchunk,
                     OutC* __restrict__ out) {
  using C = cplx_t<R>;
  constexpr int NV = NC ? NC : 1;
  constexpr int RS_MAX = sep_rec_size(M, 16);
  const int N = NC ? NC : Nrt;
  __shared__ __align__(16) R srec[RS_MAX];
  const int p = blockIdx.x / nchunk, ck = blockIdx.x - p * nchunk, tid = threadIdx.x;
  {
    const int rs = sep_rec_size(M, N);
    const R* g = rec + size_t(p) * rs;
    for (int k = tid; k < rs; k += kApplyThreads) srec[k] = g[k];
  }
  __syncthreads();
  const R* wr = srec;                        // W(c, m): (re, im) at 2 (c + m M)
  const R* ainv = srec + sep_off_ainv(M);    // Ainv(r, k): (re, im) at 2 (r + k M)
  const R* lr = srec + sep_off_l(M);         // L(m, n) at m + n M
  const R* ld = srec + sep_off_ld(M, N);     // (L(m, n), L(m, n)) at 2 (m + n M)
  const R fl = srec[sep_off_floor(M, N)];
  // Alignment (bytes) of the vector reads below: a column of W / doubled L,
  // a row block of Ainv, a column of L.
  constexpr int AL_C = (8 * M) % 16 == 0 ? 16 : 8;
  constexpr int AL_L = (4 * M) % 16 == 0 ? 16 : ((4 * M) % 8 == 0 ? 8 : 4);
  const int t1 = min(T, (ck + 1) * chunk);
  for (int t = ck * chunk + tid; t < t1; t += kApplyThreads) {
    const size_t ft = size_t(p) * T + t;
    const R* hrow = H + ft * N;
    R xv[2 * M], hv[NV];
    load_rec<2 * M, R>(reinterpret_cast<const R*>(x + ft * M), xv);
    if constexpr (NC != 0) load_rec<NV, R>(hrow, hv);
    auto hval = [&](int n) -> R {
      if constexpr (NC != 0) return hv[n];
      else return __ldg(hrow + n);
    };
    // y = W^H x
    C y[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      R wc[2 * M];
      load_sh<2 * M, AL_C, R>(wr + 2 * m * M, wc);
      C y1 = mkc<R>(R(0), R(0)), y2 = y1;
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const C xc = mkc<R>(xv[2 * c], xv[2 * c + 1]);
        if constexpr (sizeof(R) == 4) {
          y1 = mac_s(xc, wc[2 * c], y1);
          y2 = mac_s(xc, wc[2 * c + 1], y2);
        } else {
          y1.x += xc.x * wc[2 * c], y1.y += xc.y * wc[2 * c];
          y2.x += xc.x * wc[2 * c + 1], y2.y += xc.y * wc[2 * c + 1];
        }
      }
      y[m] = mkc<R>(y1.x + y2.y, y1.y - y2.x);
    }
    // max(L H, floor) (fp32: its reciprocal)
    R rl[M];
#pragma unroll
    for (int m = 0; m < M; ++m) rl[m] = R(0);
#pragma unroll(NC != 0 ? NC : 1)
    for (int n = 0; n < N; ++n) {
      R lc[M];
      load_sh<M, AL_L, R>(lr + n * M, lc);
      const R hn = hval(n);
#pragma unroll
      for (int m = 0; m < M; ++m) rl[m] += lc[m] * hn;
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const R v = rl[m] > fl ? rl[m] : fl;
      if constexpr (sizeof(R) == 4) rl[m] = rcp_fast(v);
      else rl[m] = v;
    }
    if constexpr (sizeof(R) == 4) {
      // fp32: with y'_k = y_k / max(LH, floor)_k and B(r, k) = Ainv(r, k) y'_k
      // (RP rows at a time), c_n(r) = H_n sum_k B(r, k) L(k, n): one packed
      // FMA per (row, channel, source) against the per-bin constants L (read
      // as doubled pairs, so the scalar needs no packing move).
      constexpr int RP = M <= 4 ? M : (M + 1) / 2;
      constexpr bool V16 = (M % 2 == 0) && (RP % 2 == 0);
#pragma unroll
      for (int k = 0; k < M; ++k) y[k] = mul_s(y[k], rl[k]);
#pragma unroll
      for (int r0 = 0; r0 < M; r0 += RP) {
        float2 B[RP][M];
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const float2 ys = make_float2(-y[k].y, y[k].x);
          if (r0 + RP <= M) {
            float a[2 * RP];
            load_sh<2 * RP, ((8 * M) % 16 == 0 && (8 * RP) % 16 == 0) ? 16 : 8, R>(ainv + 2 * (r0 + k * M), a);
#pragma unroll
            for (int rr = 0; rr < RP; ++rr)
              B[rr][k] = mac_s(ys, a[2 * rr + 1], mul_s(y[k], a[2 * rr]));
          } else {
#pragma unroll
            for (int rr = 0; rr < RP; ++rr) {
              const int r = r0 + rr < M ? r0 + rr : M - 1;
              B[rr][k] = mac_s(ys, ainv[2 * (r + k * M) + 1], mul_s(y[k], ainv[2 * (r + k * M)]));
            }
          }
        }
#pragma unroll 1
        for (int n = 0; n < N; ++n) {
          float l2[2 * M];
          load_sh<2 * M, AL_C, R>(ld + 2 * n * M, l2);
          float2 c[RP];
#pragma unroll
          for (int rr = 0; rr < RP; ++rr) c[rr] = __fmul2_rn(B[rr][0], make_float2(l2[0], l2[1]));
#pragma unroll
          for (int k = 1; k < M; ++k)
#pragma unroll
            for (int rr = 0; rr < RP; ++rr)
              c[rr] = __ffma2_rn(B[rr][k], make_float2(l2[2 * k], l2[2 * k + 1]), c[rr]);
          const float hn = __ldg(hrow + n);  // L1 hit: the row was read above
#pragma unroll
          for (int rr = 0; rr < RP; ++rr) c[rr] = mul_s(c[rr], hn);
          OutC* o = out + ((size_t(n) * P + p) * T + t) * M + r0;
          if (r0 + RP <= M) {
            store_out<RP, V16>(o, c);
          } else {  // odd M: the last pass is one row short
#pragma unroll
            for (int rr = 0; rr < RP; ++rr)
              if (r0 + rr < M) {
                OutC v;
                v.x = c[rr].x, v.y = c[rr].y;
                o[rr] = v;
              }
          }
        }
      }
    } else {
      // fp64 check mode: the reference's order, exact divisions.
      for (int n = 0; n < N; ++n) {
        const R hn = hval(n);
        C z[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const R g = (lr[m + n * M] * hn) / rl[m];
          z[m] = mkc<R>(g * y[m].x, g * y[m].y);
        }
        C c[M];
#pragma unroll
        for (int r = 0; r < M; ++r) {
          C acc = mkc<R>(R(0), R(0));
#pragma unroll
          for (int k = 0; k < M; ++k)
            acc = cadd(acc, cmul(mkc<R>(ainv[2 * (r + k * M)], ainv[2 * (r + k * M) + 1]), z[k]));
          c[r] = acc;
        }
        store_out<M, true>(out + ((size_t(n) * P + p) * T + t) * M, c);
      }
    }
  }
}

template <int M, int NC, typename R, typename OutC>
int launch_apply(ffca_ctx* ctx, const void* xs, const void* Hs, const R* rec, int P, int N, int T,
                 OutC* out, cudaStream_t st) {
  // Frames per CTA: two per thread, fewer CTAs than 2^31.
  int chunk = 2 * kApplyThreads;
  while ((long long)P * ((T + chunk - 1) / chunk) > 0x7fffffffLL) chunk *= 2;
  const int nchunk = (T + chunk - 1) / chunk;
  sep_apply_kernel<M, NC, R, OutC><<<unsigned(P) * unsigned(nchunk), kApplyThreads, 0, st>>>(
      reinterpret_cast<const cplx_t<R>*>(xs), reinterpret_cast<const R*>(Hs), rec, P, N, T, chunk,
      nchunk, out);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  return FFCA_OK;
}

template <int M, typename R, typename OutC>
int launch_sep_m(ffca_ctx* ctx, const void* xs, const double* W, const double* L, const void* Hs,
                 int P, int N, int T, OutC* out, cudaStream_t st) {
  if (N > 16) return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca: more than 16 sources");
  cudaError_t err;
  R* rec = static_cast<R*>(ctx->get(kSepRec, size_t(P) * sep_rec_size(M, N) * sizeof(R), &err));
  if (!rec) return ffca_set_err(FFCA_CUDA_ERROR, "ffca: separation scratch alloc failed");
  sep_prep_kernel<M, R><<<P, kPrepThreads, 0, st>>>(reinterpret_cast<const double2*>(W), L,
                                                    reinterpret_cast<const R*>(Hs), N, T, rec);
  ctx->launches++;
  FFCA_CUDA(cudaGetLastError());
  // Exact source counts for the BASELINE shapes of the fp32 device path
  // (vector H loads, unrolled source loops); the guarded variant otherwise.
  if constexpr (sizeof(R) == 4 && sizeof(OutC) == 8) {
    if (M == 2 && N == 2) return launch_apply<M, (M == 2 ? 2 : 0), R, OutC>(ctx, xs, Hs, rec, P, N, T, out, st);
    if (M == 2 && N == 3) return launch_apply<M, (M == 2 ? 3 : 0), R, OutC>(ctx, xs, Hs, rec, P, N, T, out, st);
    if (M == 3 && N == 4) return launch_apply<M, (M == 3 ? 4 : 0), R, OutC>(ctx, xs, Hs, rec, P, N, T, out, st);
    if (M == 4 && N == 6) return launch_apply<M, (M == 4 ? 6 : 0), R, OutC>(ctx, xs, Hs, rec, P, N, T, out, st);
    if (M == 8 && N == 12) return launch_apply<M, (M == 8 ? 12 : 0), R, OutC>(ctx, xs, Hs, rec, P, N, T, out, st);
  }
  return launch_apply<M, 0, R, OutC>(ctx, xs, Hs, rec, P, N, T, out, st);
}

template <typename R, typename OutC>
int launch_sep(ffca_ctx* ctx, int M, const void* xs, const double* W, const double* L,
               const void* Hs, int P, int N, int T, OutC* out, cudaStream_t st) {
  switch (M) {
    case 1: return launch_sep_m<1, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 2: return launch_sep_m<2, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 3: return launch_sep_m<3, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 4: return launch_sep_m<4, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 5: return launch_sep_m<5, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 6: return launch_sep_m<6, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 7: return launch_sep_m<7, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
    case 8: return launch_sep_m<8, R>(ctx, xs, W, L, Hs, P, N, T, out, st);
  }
  return ffca_set_err(FFCA_INVALID_ARGUMENT, "ffca: unsupported dim");
}

}  // namespace

// out_kind: 0 = images in the compute type (device path), 1 = fp64 images
// from the fp32 compute path (host path staging).
int launch_separate(ffca_ctx* ctx, int M, bool fp64, bool out_double, const void* xs,
                    const double* W, const double* L, const void* Hs, int P, int N, int T,
                    void* out, cudaStream_t st) {
  if (fp64) return launch_sep<double>(ctx, M, xs, W, L, Hs, P, N, T, static_cast<double2*>(out), st);
  if (out_double)
    return launch_sep<float>(ctx, M, xs, W, L, Hs, P, N, T, static_cast<double2*>(out), st);
  return launch_sep<float>(ctx, M, xs, W, L, Hs, P, N, T, static_cast<float2*>(out), st);
}

}  // namespace ffca
