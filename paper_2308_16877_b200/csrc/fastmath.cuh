// fastmath.cuh — FP64 exp / log / erfc / reciprocal for the Blackscholes
// accurate path (black_scholes_call, bench/blackscholes.hpp:21-36).
//
// Why not libdevice: its exp/log/erfc build every polynomial constant with
// two UMOVs per use; in bs_stream_kernel those were 25.6 % of all issued
// instructions and the kernel was issue-bound at 26 % of HBM bandwidth
// (profiles/r01i_bs_exact_sass_hist.txt). Here the coefficients live in
// __constant__ arrays (LDCU.128: two doubles per instruction), the
// reciprocals are MUFU.RCP64H + one cubic Newton step, and erfc is one
// branch-free polynomial in a rational transform of |x| (no interval split).
//
// Accuracy (tests/test_fastmath.py on the host build; tests/
// test_gpu_fastmath.py on the device against libdevice): exp <= 1 ulp,
// log <= 1 ulp, erfc <= 4 ulp relative for |x| <= 26 — the same bounds
// libdevice documents. Inputs outside the finite positive range follow IEEE
// (NaN propagates, exp(-inf) = 0, log(0) = -inf, erfc(-inf) = 2).
//
// Compiles as CUDA (device functions, __constant__ tables) and as plain C++
// (host test harness, tests/fastmath_host.cpp): same arithmetic either way,
// except that the host reciprocal seed is the IEEE quotient truncated to
// 20 mantissa bits.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#include "fastmath_coeffs.h"

#ifdef __CUDACC__
#define HPAC_FM_FN __device__ __forceinline__
#define HPAC_FM_TABLE static __constant__
#else
#define HPAC_FM_FN static inline
#define HPAC_FM_TABLE static const
#endif

namespace hpac {
namespace fm {

HPAC_FM_TABLE double kExpQ[HPAC_FM_EXP_N] = {HPAC_FM_EXP_COEFFS};
HPAC_FM_TABLE double kLogR[HPAC_FM_LOG_N] = {HPAC_FM_LOG_COEFFS};
HPAC_FM_TABLE double kErfcP[HPAC_FM_ERFC_N] = {HPAC_FM_ERFC_COEFFS};

HPAC_FM_FN int32_t hi_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2hiint(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return (int32_t)(u >> 32);
#endif
}
HPAC_FM_FN int32_t lo_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2loint(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return (int32_t)(uint32_t)u;
#endif
}
HPAC_FM_FN double from_words(int32_t hi, int32_t lo) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(hi, lo);
#else
  uint64_t u = ((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo;
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

// 1/d for d with a normal, non-extreme exponent (|d| in [2^-1000, 2^1000]):
// hardware seed (relative error < 2^-22) and one cubic Newton step.
HPAC_FM_FN double rcp_core(double d) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
#else
  double r = from_words(hi_word(1.0 / d), 0);  // a 20-bit seed, like the device's
#endif
  const double e = fma(-d, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// a/b to within 1 ulp for |b| in [2^-1000, 2^1000] (the seed's range)
HPAC_FM_FN double div_core(double a, double b) {
  const double r = rcp_core(b);
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}

// a/b to within 1 ulp; IEEE division when b is outside the seed's range
HPAC_FM_FN double div(double a, double b) {
  const uint32_t eb = ((uint32_t)hi_word(b) >> 20) & 0x7ff;
  if (eb < 0x3ff - 1000 || eb > 0x3ff + 1000) return a / b;
  return div_core(a, b);
}

// e^y for y in [-756.25, 710] (no NaN): 2^n is applied as two normal
// factors (n in [-1091, 1025]), so results underflow/overflow correctly
HPAC_FM_FN double exp_core(double y) {
  const double magic = 0x1.8p52;
  const double t = fma(y, HPAC_FM_LOG2E, magic);
  const double n = t - magic;
  const int32_t ni = lo_word(t);
  double r = fma(n, -HPAC_FM_LN2_HI, y);
  r = fma(n, -HPAC_FM_LN2_LO, r);
  double q = kExpQ[HPAC_FM_EXP_N - 1];
#pragma unroll
  for (int k = HPAC_FM_EXP_N - 2; k >= 0; --k) q = fma(q, r, kExpQ[k]);
  const double p = fma(r, fma(r, q, 1.0), 1.0);
  const int32_t n1 = ni >> 1, n2 = ni - n1;
  return p * from_words((n1 + 1023) << 20, 0) * from_words((n2 + 1023) << 20, 0);
}

// e^y
HPAC_FM_FN double exp(double y) {
  if (y != y) return y;
  return exp_core(y < -746.0 ? -746.0 : (y > 710.0 ? 710.0 : y));
}

// natural log of a positive normal finite x, with an exponent adjustment
// (fdlibm decomposition, our own fit of R)
HPAC_FM_FN double log_reduced(double x, int32_t hx, int32_t kadj) {
  hx += 0x3ff00000 - 0x3fe6a09e;
  const int32_t k = (hx >> 20) - 0x3ff + kadj;
  hx = (hx & 0x000fffff) + 0x3fe6a09e;
  const double f = from_words(hx, lo_word(x)) - 1.0;
  const double hfsq = 0.5 * f * f;
  const double d = 2.0 + f;
  const double rd = rcp_core(d);
  double s = f * rd;
  s = fma(fma(-d, s, f), rd, s);
  const double z = s * s;
  double R = kLogR[HPAC_FM_LOG_N - 1];
#pragma unroll
  for (int i = HPAC_FM_LOG_N - 2; i >= 0; --i) R = fma(R, z, kLogR[i]);
  R *= z;
  const double dk = (double)k;
  return dk * HPAC_FM_LN2_HI_K - ((hfsq - (s * (hfsq + R) + dk * HPAC_FM_LN2_LO_K)) - f);
}

// natural log of a positive normal finite x
HPAC_FM_FN double log_core(double x) { return log_reduced(x, hi_word(x), 0); }

// natural log
HPAC_FM_FN double log(double x) {
  int32_t hx = hi_word(x);
  int32_t kadj = 0;
  // one integer test routes zero, negatives, subnormals, inf and NaN aside
  if (hx < 0x00100000 || hx >= 0x7ff00000) {
    if (x == 0.0) return -INFINITY;
    if (!(x > 0.0) || x == INFINITY) return x == INFINITY ? x : NAN;
    x *= 0x1p54;  // subnormal
    kadj = -54;
    hx = hi_word(x);
  }
  return log_reduced(x, hx, kadj);
}

// erfcx(a) = e^(a^2) erfc(a) for a in [0, AMAX]
HPAC_FM_FN double erfcx_core(double a) {
  const double v = a + HPAC_FM_ERFC_K;  // t = (a-K)/(a+K)
  const double w = fma(2.0, a, 1.0);   // 1 + 2a
  const double r = rcp_core(v * w);    // v*w in [4, 1650]: seed range ok
  const double rw = r * w;             // 1/(a+K)
  const double u = fma(HPAC_FM_ERFC_P, a, HPAC_FM_ERFC_Q) * rw;
  const double s = (HPAC_FM_ERFC_P1 * a) * rw;  // u + 1, no cancellation
  double q = kErfcP[HPAC_FM_ERFC_N - 1];
#pragma unroll
  for (int i = HPAC_FM_ERFC_N - 2; i >= 0; --i) q = fma(q, u, kErfcP[i]);
  const double p = fma(s, q, 1.0);     // P(u) = erfcx(a) (1+2a)
  return p * (r * v);
}

// e^(-a^2) for a in [0, AMAX], with a^2 = hi + lo split
// (exp(-hi-lo) = exp(-hi)(1-lo))
HPAC_FM_FN double exp_neg_sq(double a) {
  const double hi = a * a;
  const double lo = fma(a, a, -hi);
  const double e = exp_core(-hi);  // a <= 27.5: -hi >= -756.25
  return fma(-lo, e, e);
}

// complementary error function
HPAC_FM_FN double erfc(double x) {
  if (x != x) return x;
  const double a = fmin(fabs(x), HPAC_FM_ERFC_AMAX);
  const double y = exp_neg_sq(a) * erfcx_core(a);
  return x < 0.0 ? 2.0 - y : y;
}

}  // namespace fm
}  // namespace hpac
