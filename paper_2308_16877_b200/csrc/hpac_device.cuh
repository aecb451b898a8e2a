// hpac_device.cuh — device-side building blocks shared by the region engines.
//
// Decision-critical floating point (TAF RSD, iACT distances, the synthetic
// fixture) uses explicit round-to-nearest intrinsics so nvcc cannot contract
// into FMA; results are then bit-identical to the reference's x86-64 build
// (taf.hpp:29-40, iact.hpp:43-53, bench/synthetic.hpp:36-53).
#pragma once

#include <cstdint>

#include "hpac_offload.h"

namespace hpac {

constexpr int kTafFilling = 0;
constexpr int kTafChecking = 1;
constexpr int kTafPredicting = 2;

// ---------------------------------------------------------------------------
// SplitMix64 (the public mixer; same constants as bench/synthetic.hpp:26-31)
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// synthetic_value / synthetic_eval, bench/synthetic.hpp:36-53 (exact rounding)
__device__ __forceinline__ double synthetic_value(int profile, int64_t i, uint64_t seed) {
  if (profile == HPAC_SYNTH_CONSTANT) return 7.5;
  if (profile == HPAC_SYNTH_SLOW_DRIFT)
    return __dmul_rn(50.0, __dadd_rn(1.0, __dmul_rn(1e-5, (double)i)));
  uint64_t h = splitmix64(seed ^ (uint64_t)i);
  return __dadd_rn(1.0, __dmul_rn((double)(h >> 11), 0x1.0p-53));
}
__device__ __forceinline__ double synthetic_eval(double x) {
  return __dadd_rn(__dmul_rn(3.0, x), 1.0);
}

// RANDOM perforation key (extension; restated in oracle/hpac_oracle.c).
__device__ __forceinline__ bool random_skip(uint64_t seed, int64_t tid, int64_t counter,
                                           int percent) {
  uint64_t k = splitmix64(((uint64_t)tid << 32) ^ (uint64_t)counter);
  uint64_t h = splitmix64(seed ^ k);
  return (int)(h % 100u) < percent;
}

// should_skip, perfo.hpp:52-72 (+RANDOM). `trip` only for INI/FINI.
__device__ __forceinline__ bool perfo_should_skip(int kind, int modulus, int percent,
                                                  uint64_t seed, int64_t key, int64_t trip,
                                                  int64_t tid) {
  switch (kind) {
    case HPAC_PERFO_SMALL:
    case HPAC_PERFO_HERDED_SMALL: return key % modulus == modulus - 1;
    case HPAC_PERFO_LARGE:
    case HPAC_PERFO_HERDED_LARGE: return key % modulus != 0;
    case HPAC_PERFO_INI: return key < ((int64_t)percent * trip) / 100;
    case HPAC_PERFO_FINI: return key >= trip - ((int64_t)percent * trip) / 100;
    case HPAC_PERFO_RANDOM: return random_skip(seed, tid, key, percent);
  }
  return false;
}

// The same with 32-bit step keys (streaming engines: steps < 2^31); the
// 64-bit modulo of the general form is a ~60-instruction subroutine.
__device__ __forceinline__ bool perfo_should_skip32(int kind, int modulus, int percent,
                                                    uint64_t seed, int key, int trip,
                                                    int64_t tid) {
  switch (kind) {
    case HPAC_PERFO_SMALL:
    case HPAC_PERFO_HERDED_SMALL: return (unsigned)key % (unsigned)modulus == (unsigned)(modulus - 1);
    case HPAC_PERFO_LARGE:
    case HPAC_PERFO_HERDED_LARGE: return (unsigned)key % (unsigned)modulus != 0u;
    case HPAC_PERFO_INI: return key < (int)(((int64_t)percent * trip) / 100);
    case HPAC_PERFO_FINI: return key >= trip - (int)(((int64_t)percent * trip) / 100);
    case HPAC_PERFO_RANDOM: return random_skip(seed, tid, key, percent);
  }
  return false;
}

// Number of valid grid-stride steps of `owner` (engine.hpp:178-185).
__device__ __forceinline__ int64_t trip_count(int64_t owner, int64_t stride, int64_t n,
                                              int64_t steps) {
  if (owner >= n) return 0;
  int64_t t = (n - 1 - owner) / stride + 1;
  return t < steps ? t : steps;
}

// rsd, taf.hpp:29-40: two-pass population sigma / |mu|, window order,
// no contraction, IEEE sqrt/div.
template <int H>
__device__ __forceinline__ bool taf_window_passes_exact(const double (&w)[H], double thr) {
  double mean = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) mean = __dadd_rn(mean, w[i]);
  mean = __ddiv_rn(mean, (double)H);
  double ssd = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double d = __dsub_rn(w[i], mean);
    ssd = __dadd_rn(ssd, __dmul_rn(d, d));
  }
  double sigma = __dsqrt_rn(__ddiv_rn(ssd, (double)H));
  double r;
  if (mean == 0.0)
    r = sigma == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
  else
    r = __ddiv_rn(sigma, fabs(mean));
  return r <= thr;
}

// reciprocal to ~2^-50 relative: MUFU seed + two Newton steps (no IEEE path)
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Same decision as taf_window_passes_exact, computed first without IEEE
// division / square root: r^2 ~= ssd / (H mean^2) from an approximate mean.
// The approximation is within ~1e-14 relative plus ~1e-30 absolute (the
// mean's last-ulp error feeding ssd) of the exact r^2, so whenever it lies
// outside thr^2 (1 +- 1e-9) +- 1e-27 the exact test must agree; NaN/inf
// windows, mean ~ 0 and near-threshold windows take the exact path.
template <int H>
__device__ __forceinline__ bool taf_window_passes(const double (&w)[H], double thr) {
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) sum = __dadd_rn(sum, w[i]);
  const double mean_a = sum * (1.0 / H);
  double ssd_a = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double d = w[i] - mean_a;
    ssd_a = fma(d, d, ssd_a);
  }
  const double den = (double)H * mean_a * mean_a;
  const double r2 = ssd_a * rcp_fast(den);
  const double t2 = thr * thr;
  if (den > 1e-290 && den < 1e290) {
    if (r2 < t2 * (1.0 - 1e-9) - 1e-27) return true;
    if (r2 > t2 * (1.0 + 1e-9) + 1e-27) return false;
  }
  return taf_window_passes_exact<H>(w, thr);
}

// Same RSD over a strided window in shared memory: w[j*stride] for j in
// [0, len) in ring order starting at `head` (taf.hpp:82-88).
__device__ __forceinline__ bool taf_ring_passes_exact(const double* ring, int stride, int h,
                                                      int head, int len, double thr) {
  double mean = 0.0;
  for (int j = 0; j < len; ++j) {
    int slot = head + j;
    if (slot >= h) slot -= h;
    mean = __dadd_rn(mean, ring[slot * stride]);
  }
  mean = __ddiv_rn(mean, (double)len);
  double ssd = 0.0;
  for (int j = 0; j < len; ++j) {
    int slot = head + j;
    if (slot >= h) slot -= h;
    double d = __dsub_rn(ring[slot * stride], mean);
    ssd = __dadd_rn(ssd, __dmul_rn(d, d));
  }
  double sigma = __dsqrt_rn(__ddiv_rn(ssd, (double)len));
  double r;
  if (mean == 0.0)
    r = sigma == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
  else
    r = __ddiv_rn(sigma, fabs(mean));
  return r <= thr;
}

// division-free estimate first, exact RSD near the threshold (see
// taf_window_passes for the margin argument)
__device__ __forceinline__ bool taf_ring_passes(const double* ring, int stride, int h, int head,
                                                int len, double thr) {
  double sum = 0.0;
  for (int j = 0; j < len; ++j) {
    int slot = head + j;
    if (slot >= h) slot -= h;
    sum = __dadd_rn(sum, ring[slot * stride]);
  }
  const double mean_a = sum * rcp_fast((double)len);
  double ssd_a = 0.0;
  for (int j = 0; j < len; ++j) {
    int slot = head + j;
    if (slot >= h) slot -= h;
    const double d = ring[slot * stride] - mean_a;
    ssd_a = fma(d, d, ssd_a);
  }
  const double den = (double)len * mean_a * mean_a;
  const double r2 = ssd_a * rcp_fast(den);
  const double t2 = thr * thr;
  if (den > 1e-290 && den < 1e290) {
    if (r2 < t2 * (1.0 - 1e-9) - 1e-27) return true;
    if (r2 > t2 * (1.0 + 1e-9) + 1e-27) return false;
  }
  return taf_ring_passes_exact(ring, stride, h, head, len, thr);
}

// Ring window of compile-time length H, full (count == H, which is the only
// state a TAF check sees): division-free estimate over the slots in any
// order, the exact ring-order RSD only near the threshold. t_lo / t_hi are
// thr^2 (1 -+ 1e-9) -+ 1e-27 (see taf_window_passes).
template <int H>
__device__ __forceinline__ bool taf_ring_passes_fixed(const double* ring, int stride, int head,
                                                      double thr, double t_lo, double t_hi) {
  double w[H];
#pragma unroll
  for (int i = 0; i < H; ++i) w[i] = ring[i * stride];
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) sum += w[i];
  const double mean_a = sum * (1.0 / H);
  double ssd_a = 0.0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double d = w[i] - mean_a;
    ssd_a = fma(d, d, ssd_a);
  }
  const double den = (double)H * mean_a * mean_a;
  if (den > 1e-290 && den < 1e290) {
    if (ssd_a < den * t_lo) return true;
    if (ssd_a > den * t_hi) return false;
  }
  return taf_ring_passes_exact(ring, stride, H, head, H, thr);
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }

// FP64 tensor-core MMA, D = A(8x4, row) * B(4x8, col) + D, one warp. Lane L
// holds A[L/4][L%4], B[L%4][L/4] and D[L/4][2(L%4)], D[L/4][2(L%4)+1].
// (tcgen05 has no FP64 kind; the sm_80+ DMMA path is the FP64 tensor op.)
__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Writer key for the iACT max-min selection (iact.hpp:166-180): larger
// distance wins, ties to the lower lane. Non-candidates carry d = -1.
__device__ __forceinline__ bool writer_better(double da, int la, double db, int lb) {
  return da > db || (da == db && la < lb);
}

}  // namespace hpac
