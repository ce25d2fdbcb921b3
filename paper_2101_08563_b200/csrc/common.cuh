// common.cuh -- shared device helpers for the FastFCA sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ffca {

// ------------------------------------------------------------ real/complex --
template <typename R> struct Cplx;
template <> struct Cplx<float> { using type = float2; };
template <> struct Cplx<double> { using type = double2; };
template <typename R> using cplx_t = typename Cplx<R>::type;

template <typename R> __device__ __forceinline__ cplx_t<R> mkc(R re, R im) {
  cplx_t<R> z; z.x = re; z.y = im; return z;
}
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { a.x += b.x; a.y += b.y; return a; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { a.x -= b.x; a.y -= b.y; return a; }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
  C z; z.x = a.x * b.x - a.y * b.y; z.y = a.x * b.y + a.y * b.x; return z;
}
// conj(a) * b
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
  C z; z.x = a.x * b.x + a.y * b.y; z.y = a.x * b.y - a.y * b.x; return z;
}
template <typename C> __device__ __forceinline__ C cconj(C a) { a.y = -a.y; return a; }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ float cabs2(float2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith-free scaled division; adequate for the tiny LU pivots (never 0 here).
  const double s = 1.0 / (b.x * b.x + b.y * b.y);
  double2 z; z.x = (a.x * b.x + a.y * b.y) * s; z.y = (a.y * b.x - a.x * b.y) * s; return z;
}
__device__ __forceinline__ double cabs(double2 a) { return hypot(a.x, a.y); }

// Precision-dispatched transcendental helpers.  The fp32 path uses the SFU
// approximations (the NLL is accumulated in fp64, tolerance 1e-5 relative);
// the fp64 check mode uses correctly rounded division and libdevice log.
__device__ __forceinline__ float rcp(float a) { return __frcp_rn(a); }
__device__ __forceinline__ double rcp(double a) { return 1.0 / a; }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fdiv(double a, double b) { return a / b; }
__device__ __forceinline__ float flog(float a) { return __logf(a); }
__device__ __forceinline__ double flog(double a) { return log(a); }
__device__ __forceinline__ float fsqrt(float a) { return sqrtf(a); }
__device__ __forceinline__ double fsqrt(double a) { return sqrt(a); }

// Smallest positive normal of the compute type.  The reference clamps with
// 1e-300 (fastfca.cpp:94,97,107,109,114,116), which underflows to 0 in fp32;
// FLT_MIN plays its role there (SURVEY §7 "fp32 pitfalls").
template <typename R> __device__ __forceinline__ R tiny();
template <> __device__ __forceinline__ float tiny<float>() { return 1.17549435e-38f; }
template <> __device__ __forceinline__ double tiny<double>() { return 1e-300; }

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

// ------------------------------------------------------------- reductions --
template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --------------------------------------------- libstdc++-compatible restart --
// The reference perturbs a failed IP column with
//   std::mt19937_64 rng(mix_seed(seed + t, i)); std::normal_distribution<double>
//   w(r, col) += mag * Complex(gauss(rng), gauss(rng))   (fastfca.cpp:40-41,67-69)
// libstdc++'s normal_distribution is the Marsaglia polar method with one cached
// value, generate_canonical<double,53> over mt19937_64 is one draw / 2^64, and
// g++ evaluates the two constructor arguments right to left (imag drawn first).
// Reproduced here so restart trajectories follow the reference's draws.
struct Mt19937_64 {
  uint64_t mt[312];
  int idx;
  __device__ void seed(uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < 312; ++i)
      mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    idx = 312;
  }
  __device__ uint64_t next() {
    if (idx >= 312) {
      const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
      const uint64_t MA = 0xB5026F5AA96619E9ULL;
      for (int i = 0; i < 312; ++i) {
        const uint64_t x = (mt[i] & UM) | (mt[(i + 1) % 312] & LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= MA;
        mt[i] = mt[(i + 156) % 312] ^ xa;
      }
      idx = 0;
    }
    uint64_t x = mt[idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
  }
};

struct PolarNormal {
  double saved;
  bool has_saved;
  __device__ double canonical(Mt19937_64& g) {
    double r = double(g.next()) / 18446744073709551616.0;
    if (r >= 1.0) r = 0.99999999999999989;  // nextafter(1, 0)
    return r;
  }
  __device__ double operator()(Mt19937_64& g) {
    if (has_saved) {
      has_saved = false;
      return saved;
    }
    double x, y, r2;
    do {
      x = 2.0 * canonical(g) - 1.0;
      y = 2.0 * canonical(g) - 1.0;
      // separately rounded products and sum, as the reference's baseline
      // x86-64 build evaluates libstdc++'s x * x + y * y (no FMA contraction)
      r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2.0 * log(r2) / r2);
    saved = x * mult;
    has_saved = true;
    return y * mult;
  }
};

// Restart state of one IP sweep, kept in shared scratch so the hot path of
// the column solves holds no address-taken locals (those live in local
// memory and cost a round trip per call).
struct RestartRng {
  Mt19937_64 mt;
  PolarNormal gauss;
};

// fastfca.cpp:13-18
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, int i) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * uint64_t(int64_t(i) + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace ffca

namespace ffca {
// Narrow a non-negative fp64 parameter to the compute type without letting an
// underflow turn a positive value into 0 (exact zeros, e.g. the one-hot ICA
// loadings of fastfca.cpp:256, stay zero).
template <typename R> __device__ __forceinline__ R narrow_pos(double v) {
  const R r = R(v);
  return (v > 0.0 && !(r > R(0))) ? tiny<R>() : r;
}
}  // namespace ffca

namespace ffca {
// Reciprocal on the SFU (MUFU.RCP, ~1 ulp) for the fp32 data path; exact
// division in the fp64 check mode.
__device__ __forceinline__ float rcp_fast(float a) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double rcp_fast(double a) { return 1.0 / a; }
// SFU square root (for tolerance scales only).
__device__ __forceinline__ float sqrt_approx(float a) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
}  // namespace ffca

namespace ffca {
__device__ __forceinline__ float flog2(float a) { return __log2f(a); }
__device__ __forceinline__ double flog2(double a) { return log2(a); }
}  // namespace ffca

namespace ffca {
// log2 on the SFU with denormal flushing (fp32 path); libdevice log2 in fp64.
__device__ __forceinline__ float flog2_ftz(float a) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double flog2_ftz(double a) { return log2(a); }

template <int K>
struct Pow2Ceil {
  static constexpr int value = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : K <= 16 ? 16 : 32;
};

// Reduce K per-lane values over the warp and store the K totals to dst[0..K)
// (converted to D).  Recursive halving: at each step the lanes split the remaining
// values in two and exchange the half they give away, so the warp issues
// Kp - 1 + (5 - log2 Kp) shuffles instead of 5K (Kp = K rounded up to a power
// of two, <= 32).  The summation tree is fixed, so results are deterministic.
template <int K, typename T, typename D>
__device__ __forceinline__ void warp_reduce_store(const T (&in)[K], D* dst, int lane) {
  static_assert(K <= 32, "warp_reduce_store: at most 32 values");
  constexpr int KP = Pow2Ceil<K>::value;
  T v[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) v[i] = i < K ? in[i] : T(0);
  int idx = 0;
  int o = 16;
#pragma unroll
  for (int c = KP; c > 1; c >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < c / 2; ++i) {
      const T send = up ? v[i] : v[i + c / 2];
      const T keep = up ? v[i + c / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    if (up) idx += c / 2;
    o >>= 1;
  }
  T s = v[0];
  for (int oo = o; oo > 0; oo >>= 1) s += __shfl_xor_sync(0xffffffffu, s, oo);
  // Lanes whose low (plain-reduction) bits are zero hold distinct totals.
  const int lowmask = o == 0 ? 0 : (o << 1) - 1;
  if ((lane & lowmask) == 0 && idx < K) dst[idx] = D(s);
}
}  // namespace ffca
