// apps.cuh — application kernels (the reference's Regions, bench/*.hpp) as
// device functions. Each app supplies load (the iACT key, and the inputs
// of the accurate path), eval (the accurate region) and store.
#pragma once

#include <cstdint>

#include "engine.h"
#include "fastmath.cuh"
#include "hpac_device.cuh"

namespace hpac {

// black_scholes_call, bench/blackscholes.hpp:21-36, for any arguments.
// Returns false where the reference throws ConfigError (invalid
// parameters). The transcendental functions are csrc/fastmath.cuh's (<= 1 ulp
// exp/log, <= 4 ulp erfc, the libdevice bounds, at about half libdevice's
// instruction count).
#ifndef HPAC_BS_GENERAL_ATTR
#define HPAC_BS_GENERAL_ATTR __forceinline__  // __noinline__: 90.5 vs 78.1 us exact (call ABI spills)
#endif
static __device__ HPAC_BS_GENERAL_ATTR bool bs_call_general(double spot, double strike, double rate,
                                                    double vol, double mat, double& price) {
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol >= 0) || !isfinite(rate))
    return false;
  double disc_strike = strike * fm::exp(-rate * mat);
  double sst = vol * sqrt(mat);
  if (sst == 0.0) {
    double v = spot - disc_strike;
    price = v < 0.0 ? 0.0 : v;
    return true;
  }
  double d1 = fm::div(fm::log(fm::div(spot, strike)) + (rate + 0.5 * vol * vol) * mat, sst);
  double d2 = d1 - sst;
  // norm_cdf(x) = erfc(-x/sqrt2)/2 (blackscholes.hpp:21); the division by
  // sqrt2 is a multiplication by 1/sqrt2 here (<= 1 ulp in the argument).
  // erfc(-d/sqrt2) = y or 2 - y with y = e^(-d^2/2) erfcx(|d|/sqrt2), and
  // S e^(-d1^2/2) = K e^(-rT) e^(-d2^2/2) (d1 sst - sst^2/2 = log(S/K) + rT),
  // so the second Gaussian factor is a product instead of a second exp:
  // D N(d2) = D - S e1 erfcx(a2)/2 (d2 > 0) or S e1 erfcx(a2)/2. N(d1) is
  // bit-equal to the two-erfc form; D N(d2) agrees to a few ulp.
  // Infinite spot/strike/vol/maturity (S e1 = inf * 0) and a discounted
  // strike that overflowed or underflowed (the identity needs 0 < D < inf)
  // keep the two-erfc form.
  if (!((spot * strike) * (vol * mat) < INFINITY) || !(disc_strike > 0.0 && disc_strike < INFINITY)) {
    price = 0.5 * fm::erfc(d1 * -0.70710678118654752440) * spot -
            disc_strike * (0.5 * fm::erfc(d2 * -0.70710678118654752440));
    return true;
  }
  const double a1 = fmin(fabs(d1) * 0.70710678118654752440, HPAC_FM_ERFC_AMAX);
  const double a2 = fmin(fabs(d2) * 0.70710678118654752440, HPAC_FM_ERFC_AMAX);
  const double e1 = fm::exp_neg_sq(a1);
  const double y1 = e1 * fm::erfcx_core(a1);                   // erfc(|d1|/sqrt2)
  const double t2 = 0.5 * (spot * (e1 * fm::erfcx_core(a2)));  // D erfc(|d2|/sqrt2) / 2
  const double n1 = d1 > 0.0 ? 1.0 - 0.5 * y1 : 0.5 * y1;
  price = spot * n1 - (d2 > 0.0 ? disc_strike - t2 : t2);
  return true;
}

// The same function, with the argument checks of every step hoisted into one
// integer range test: spot, strike in [2^-500, 2^500), vol in [2^-500, 2^8),
// maturity in [2^-500, 2^5), |rate| < 2^3. Inside that box every check of
// bs_call_general passes (valid arguments, finite S e1, sst > 0, exp
// argument within [-256, 256] so 0 < D < inf, divisors and the log argument
// normal and in the reciprocal seed's range), so the straight-line code below
// returns the same bits; anything else takes bs_call_general.
__device__ __forceinline__ bool bs_call(double spot, double strike, double rate, double vol,
                                        double mat, double& price) {
  const uint64_t lo = 0x20B0000000000000ull;  // 2^-500
  const uint64_t bs = (uint64_t)__double_as_longlong(spot), bk = (uint64_t)__double_as_longlong(strike),
                 bv = (uint64_t)__double_as_longlong(vol), bt = (uint64_t)__double_as_longlong(mat),
                 br = (uint64_t)__double_as_longlong(rate) & 0x7fffffffffffffffull;
  const bool fast = bs - lo < 0x5F30000000000000ull - lo && bk - lo < 0x5F30000000000000ull - lo &&
                    bv - lo < 0x4070000000000000ull - lo && bt - lo < 0x4040000000000000ull - lo &&
                    br < 0x4020000000000000ull;
  if (!fast) return bs_call_general(spot, strike, rate, vol, mat, price);
  const double disc_strike = strike * fm::exp_core(-rate * mat);
  const double sst = vol * sqrt(mat);
  const double d1 = fm::div_core(fm::log_core(fm::div_core(spot, strike)) + (rate + 0.5 * vol * vol) * mat, sst);
  const double d2 = d1 - sst;
  const double a1 = fmin(fabs(d1) * 0.70710678118654752440, HPAC_FM_ERFC_AMAX);
  const double a2 = fmin(fabs(d2) * 0.70710678118654752440, HPAC_FM_ERFC_AMAX);
  const double e1 = fm::exp_neg_sq(a1);
  const double y1 = e1 * fm::erfcx_core(a1);
  const double t2 = 0.5 * (spot * (e1 * fm::erfcx_core(a2)));
  const double n1 = d1 > 0.0 ? 1.0 - 0.5 * y1 : 0.5 * y1;
  price = spot * n1 - (d2 > 0.0 ? disc_strike - t2 : t2);
  return true;
}

// The same formula on libdevice's exp/log/erfc and IEEE division (the
// round-1 kernel); kept for the device accuracy test (hpac_fm_eval).
__device__ __forceinline__ double bs_call_libdevice(double spot, double strike, double rate,
                                                    double vol, double mat) {
  double disc_strike = strike * ::exp(-rate * mat);
  double sst = vol * sqrt(mat);
  if (sst == 0.0) {
    double v = spot - disc_strike;
    return v < 0.0 ? 0.0 : v;
  }
  double d1 = (::log(spot / strike) + (rate + 0.5 * vol * vol) * mat) / sst;
  double d2 = d1 - sst;
  return spot * (0.5 * ::erfc(d1 * -0.70710678118654752440)) -
         disc_strike * (0.5 * ::erfc(d2 * -0.70710678118654752440));
}

// Hooks every app inherits: encounters per item (Region::encounters,
// engine.hpp:29; 1 by default) and a per-round staging step executed by
// every thread of the team outside the approximated region.
struct AppBase {
  // techniques the runtime accepts for the app (others are not instantiated)
  static constexpr bool HAS_TAF = true, HAS_IACT = true;
  // occupancy hint for the 256-thread engine instantiation (launch bounds)
  static constexpr int MIN_BLOCKS_256 = 1;
  static constexpr int min_blocks_256(int) { return -1; }  // -1: MIN_BLOCKS_256
  __device__ static int encounters(const EngineParams& p, int64_t idx) {
    return p.region.encounters ? p.region.encounters[idx] : 1;
  }
  __device__ static void round_begin(const EngineParams&, int64_t, int, double*, bool, bool) {}
  // warp-cooperative evaluation (EngineParams::warp_eval): called by all 32
  // lanes of a hardware warp, converged; `want` = this lane evaluates
  static constexpr bool WARP_EVAL = false;
  __device__ static double warp_eval(const EngineParams&, int64_t, bool, const double*, int) {
    return 0.0;
  }
};

// Generic pure region over a work index (HPAC_APP_TABLE): load_input reads
// `in`, evaluate returns the precomputed accurate output `table_out`.
struct AppTable : AppBase {
  static constexpr int IN_MAX = 8;
  static constexpr int OUT_MAX = 4;
  __device__ static void load(const EngineParams& p, int64_t idx, double (&in)[IN_MAX]) {
    const double* src = p.region.in + idx * p.in_dims;
#pragma unroll
    for (int d = 0; d < IN_MAX; ++d)
      if (d < p.in_dims) in[d] = src[d];
  }
  __device__ static void init(const EngineParams&, double*) {}
  __device__ static bool eval(const EngineParams& p, int64_t idx, const double (&)[IN_MAX],
                              double (&out)[OUT_MAX], const double*, int, int) {
    const double* src = p.region.table_out + idx * p.out_dims;
#pragma unroll
    for (int d = 0; d < OUT_MAX; ++d)
      if (d < p.out_dims) out[d] = src[d];
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX], int) {
    double* dst = p.region.out;
    if (!dst) return;
    dst += idx * p.out_dims;
#pragma unroll
    for (int d = 0; d < OUT_MAX; ++d)
      if (d < p.out_dims) {
        if (p.accumulate)
          dst[d] = __dadd_rn(dst[d], out[d]);
        else
          dst[d] = out[d];
      }
  }
};

// bench/synthetic.hpp:56-71
struct AppSynthetic : AppBase {
  static constexpr int IN_MAX = 1;
  static constexpr int OUT_MAX = 1;
  __device__ static void load(const EngineParams& p, int64_t idx, double (&in)[IN_MAX]) {
    in[0] = synthetic_value(p.region.synthetic_profile, idx, p.region.seed);
  }
  __device__ static void init(const EngineParams&, double*) {}
  __device__ static bool eval(const EngineParams& p, int64_t idx, const double (&)[IN_MAX],
                              double (&out)[OUT_MAX], const double*, int, int) {
    out[0] = synthetic_eval(synthetic_value(p.region.synthetic_profile, idx, p.region.seed));
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX], int) {
    if (p.region.out) p.region.out[idx] = out[0];
  }
};

// bench/blackscholes.hpp:72-92 (AoS option = 5 doubles)
struct AppBlackScholes : AppBase {
  static constexpr int IN_MAX = 5;
  static constexpr int OUT_MAX = 1;
  __device__ static void load(const EngineParams& p, int64_t idx, double (&in)[IN_MAX]) {
    const double* o = p.region.in + idx * 5;
#pragma unroll
    for (int d = 0; d < 5; ++d) in[d] = __ldg(o + d);
  }
  __device__ static void init(const EngineParams&, double*) {}
  __device__ static bool eval(const EngineParams&, int64_t, const double (&in)[IN_MAX],
                              double (&out)[OUT_MAX], const double*, int, int) {
    return bs_call(in[0], in[1], in[2], in[3], in[4], out[0]);
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX], int) {
    if (p.region.out) __stcs(p.region.out + idx, out[0]);
  }
};


// K-Means distance region (bench/kmeans.hpp:82-102). The region's outputs
// are the k distances; the host argmin (kmeans.hpp:111-121) is fused here,
// so the engine payload is the label (stored as a double) and the k
// distances are written only when the caller asks for them (region.out).
// Centroids (and their squared norms) are staged once per CTA in shared
// memory (broadcast reads).
//
// Labels are bit-identical to the reference's (sqrt of the no-FMA,
// dimension-order sum, strict <, lowest index) but are found with a filter:
// d2(c) ~= |x|^2 + |c|^2 - 2 x.c costs one DFMA per (c, d) instead of three
// FP64 ops; with a rigorous error bound E(c) (a multiple of the unit
// roundoff times |x|^2 + |c|^2, covering both this estimate and the
// reference's own rounding) the estimated minimiser is the reference's
// argmin whenever every other centroid's estimate exceeds it by more than
// E(best) + E(other) (+16 ulp so the sqrt values cannot collide). Any
// closer pair (near-ties, duplicate centroids, non-finite data) re-runs the
// reference computation over all centroids.
struct AppKmeans : AppBase {
#ifndef HPAC_KM_MINB
#define HPAC_KM_MINB 2
#endif
  // the point (32 doubles) lives in registers: cap at 128 so >= 16 warps fit
  static constexpr int MIN_BLOCKS_256 = HPAC_KM_MINB;
  static constexpr bool HAS_TAF = false;  // rejected by the runtime (64-dim window)
  static constexpr int IN_MAX = 32;
  static constexpr int OUT_MAX = 1;
  __device__ static void init(const EngineParams& p, double* scratch) {
    if (p.warp_eval) return;  // warp_eval reads the per-launch km_aux block (L1-resident)
    const int k = p.region.kmeans_k, dims = p.region.kmeans_dims;
    const int kd = k * dims;
    for (int i = threadIdx.x; i < kd; i += blockDim.x) scratch[i] = p.region.centroids[i];
    __syncthreads();
    double* cc = scratch + kd;  // [k] squared norms, then [1] their maximum
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
      double s = 0.0;
      for (int d = 0; d < dims; ++d) s = fma(scratch[c * dims + d], scratch[c * dims + d], s);
      cc[c] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int c = 0; c < k; ++c) m = fmax(m, cc[c]);  // NaN norms: caught by chk
      cc[k] = m;
    }
    __syncthreads();
  }
  __device__ static void load(const EngineParams& p, int64_t idx, double (&in)[IN_MAX]) {
    const int dims = p.region.kmeans_dims;
    const double* src = p.region.in + idx * dims;
    if ((dims & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
#pragma unroll
      for (int d = 0; d < IN_MAX; d += 2)
        if (d < dims) {
          double2 t = __ldg(reinterpret_cast<const double2*>(src + d));
          in[d] = t.x;
          in[d + 1] = t.y;
        }
    } else {
#pragma unroll
      for (int d = 0; d < IN_MAX; ++d)
        if (d < dims) in[d] = __ldg(src + d);
    }
  }
  // reference distances: sqrt of the dimension-order sum without contraction
  __device__ static int exact_argmin(const double (&in)[IN_MAX], const double* cent, int dims,
                                     int k, bool fast, double* dist) {
    int best = 0;
    double best_ssq = 0.0, best_d = 0.0;
    for (int c = 0; c < k; ++c) {
      const double* cc = cent + c * dims;
      double ssq = 0.0;
      if (fast) {
#pragma unroll
        for (int d = 0; d < IN_MAX; ++d)
          if (d < dims) {
            double df = in[d] - cc[d];
            ssq = fma(df, df, ssq);
          }
      } else {
#pragma unroll
        for (int d = 0; d < IN_MAX; ++d)
          if (d < dims) {
            double df = __dsub_rn(in[d], cc[d]);
            ssq = __dadd_rn(ssq, __dmul_rn(df, df));
          }
      }
      if (dist) {
        double dd = __dsqrt_rn(ssq);
        dist[c] = dd;
        if (c == 0 || dd < best_d) {
          best = c;
          best_d = dd;
        }
      } else if (c == 0) {
        best_ssq = ssq;
        best_d = __dsqrt_rn(ssq);
      } else if (ssq < best_ssq) {
        // sqrt is monotone: only an improving squared distance can win
        double dd = __dsqrt_rn(ssq);
        if (dd < best_d) {
          best = c;
          best_d = dd;
          best_ssq = ssq;
        }
      }
    }
    return best;
  }
  // rare fallback, out of line so the fast path keeps its registers: the
  // point is re-read from global memory
  __device__ static __noinline__ int exact_argmin_reload(const EngineParams& p, int64_t idx,
                                                         const double* cent) {
    double x[IN_MAX];
    load(p, idx, x);
    return exact_argmin(x, cent, p.region.kmeans_dims, p.region.kmeans_k, false, nullptr);
  }
  __device__ static bool eval(const EngineParams& p, int64_t idx, const double (&in)[IN_MAX],
                              double (&out)[OUT_MAX], const double* cent, int, int) {
    const int dims = p.region.kmeans_dims, k = p.region.kmeans_k;
    const bool fast = (p.region.flags & HPAC_REGION_KMEANS_FAST_MATH) != 0;
    double* dist = p.region.out ? p.region.out + idx * k : nullptr;
    if (dist || fast || dims != IN_MAX || (k & 3) || k < 2) {
      out[0] = (double)exact_argmin(in, cent, dims, k, fast, dist);
      return true;
    }
    const double* cc = cent + k * dims;
    double xx0 = 0.0, xx1 = 0.0;
#pragma unroll
    for (int d = 0; d < IN_MAX; d += 2) {
      xx0 = fma(in[d], in[d], xx0);
      xx1 = fma(in[d + 1], in[d + 1], xx1);
    }
    const double xx = xx0 + xx1;
    // E = G (|x|^2 + max_c |c|^2) bounds |estimate - reference ssq| for every
    // centroid: 4x the (4d+8)u first-order bound
    const double G = 4.0 * (4.0 * IN_MAX + 8.0) * 0x1.0p-53;
    const double E = G * (xx + cc[k]);
    int best = 0;
    double m1 = dinf(), m2 = dinf(), chk = 0.0;
    // four centroids per pass (eight independent DFMA chains per thread);
    // the next dimension pair's centroid values are loaded one step ahead so
    // the shared-memory latency overlaps the FMAs
    for (int c = 0; c < k; c += 4) {
      const double2* c0 = reinterpret_cast<const double2*>(cent + c * IN_MAX);
      double acc[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
      double2 u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) u[j] = c0[j * (IN_MAX / 2)];
#pragma unroll
      for (int d = 0; d < IN_MAX; d += 2) {
        double2 v[4];
        if (d + 2 < IN_MAX) {
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = c0[j * (IN_MAX / 2) + d / 2 + 1];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[j][0] = fma(in[d], u[j].x, acc[j][0]);
          acc[j][1] = fma(in[d + 1], u[j].y, acc[j][1]);
        }
        if (d + 2 < IN_MAX) {
#pragma unroll
          for (int j = 0; j < 4; ++j) u[j] = v[j];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double a = fma(-2.0, acc[j][0] + acc[j][1], xx + cc[c + j]);
        chk += a;  // NaN / inf anywhere -> reference path
        if (a < m1) {
          m2 = m1;
          m1 = a;
          best = c + j;
        } else if (a < m2) {
          m2 = a;
        }
      }
    }
    // every other centroid provably farther, by more than the bound on both
    // estimates plus 16 ulp (so the reference's sqrt values cannot collide)
    if (!(isfinite(chk) && m2 - m1 > 2.0 * E + 16.0 * 0x1.0p-53 * fabs(m2)))
      best = exact_argmin_reload(p, idx, cent);
    out[0] = (double)best;
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX], int) {
    if (p.region.labels) p.region.labels[idx] = (int32_t)out[0];
  }
};

// (smallest, runner-up, argmin) update with one candidate, as predicated
// selects (strict <: ties keep the earlier candidate; NaN never enters)
__device__ __forceinline__ void top2_update(double e, int c, double& m1, double& m2, int& best) {
  asm("{\n\t.reg .pred p0, p1;\n\t.reg .f64 t;\n\t"
      "setp.lt.f64 p0, %3, %0;\n\t"
      "setp.lt.f64 p1, %3, %1;\n\t"
      "selp.f64 t, %3, %1, p1;\n\t"
      "selp.f64 %1, %0, t, p0;\n\t"
      "selp.f64 %0, %3, %0, p0;\n\t"
      "selp.s32 %2, %4, %2, p0;\n\t}"
      : "+d"(m1), "+d"(m2), "+r"(best)
      : "d"(e), "r"(c));
}

// K-Means region with the warp-cooperative DMMA filter (EngineParams::warp_eval
// set by the runtime for its shape); load/eval/store as AppKmeans.
struct AppKmeansDmma : AppKmeans {
#ifndef HPAC_KMD_MINB
#define HPAC_KMD_MINB 4
#endif
  static constexpr int MIN_BLOCKS_256 = HPAC_KMD_MINB;
  // Warp-cooperative filtered argmin on the FP64 tensor op (dims == 32,
  // k % 8 == 0, no distance output; host-gated). The 32 items of a hardware
  // warp are consecutive (per-thread mapping), so the warp computes the
  // 32 x k block of x.c products as 4 x (k/8) m8n8k4 tiles over 8 k-steps.
  // The reduction index is permuted (k-step s, slot t <-> dimension 8(s/2) + 2t + s%2)
  // so every lane's operands are 16-byte pairs: points come straight from
  // HBM as 2 KB coalesced rows per m-tile, centroids from a fragment-ordered
  // copy (each 16-byte load contiguous across the warp, each element read
  // once per warp instead of once per lane; a per-launch block prepared by
  // kmeans_dmma_aux_kernel, L1-resident, so CTAs stage nothing). Each operand
  // feeds 4 FMAs from registers, which lifts the shared-memory operand bound
  // of eval() above.
  // The estimate is certified exactly as in eval(): the bound E covers any
  // summation order of the 32 products, so the label is the reference's.
  static constexpr bool WARP_EVAL = true;
  // build-time tuning knobs (tools/build_variant.sh; A/B results in DESIGN
  // §4.2): m-tiles per pass, n-tiles per step, L1 prefetch of the next rows,
  // and HPAC_KMD_MINB above (CTAs of 256 threads per SM -> register cap)
#ifndef HPAC_KM_MT
#define HPAC_KM_MT 1
#endif
#ifndef HPAC_KM_NT
#define HPAC_KM_NT 2
#endif
#ifndef HPAC_KM_PF
#define HPAC_KM_PF 1
#endif
  // NT n-tiles starting at centroid j against MT m-tiles: x.c by DMMA, then
  // the (smallest, runner-up, argmin) update with this lane's 2 NT candidates
  // (bj = this lane's fragment pointer for n-tile j/8, cj = &norm[j + 2t]:
  // the loads below use constant offsets from them)
  template <int NT, int MT>
  __device__ __forceinline__ static void dmma_tiles(const double2* bj, const double* cj, int j, int t,
                                                    const double (&a)[MT][8], const double (&xx)[MT],
                                                    double (&m1)[MT], double (&m2)[MT], int (&best)[MT]) {
    double b[NT][8];
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 v = __ldg(bj + (u * 4 + q) * 32);
        b[u][2 * q] = v.x;
        b[u][2 * q + 1] = v.y;
      }
    double acc[NT][MT][2];
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
      for (int i = 0; i < MT; ++i) acc[u][i][0] = acc[u][i][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int i = 0; i < MT; ++i) dmma_m8n8k4(acc[u][i][0], acc[u][i][1], a[i][s], b[u][s]);
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      const int c0 = j + 8 * u + 2 * t;
      const double n0 = __ldg(cj + 8 * u), n1 = __ldg(cj + 8 * u + 1);
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        // non-finite data never passes: E in warp_eval is then inf/NaN
        top2_update(fma(-2.0, acc[u][i][0], xx[i] + n0), c0, m1[i], m2[i], best[i]);
        top2_update(fma(-2.0, acc[u][i][1], xx[i] + n1), c0 + 1, m1[i], m2[i], best[i]);
      }
    }
  }

  __device__ static double warp_eval(const EngineParams& p, int64_t idx, bool want,
                                     const double*, int lane) {
    const int k = p.region.kmeans_k;
    const int g = lane >> 2, t = lane & 3;
    const int64_t base = idx - lane;  // item of lane 0
    const unsigned wm = __ballot_sync(0xffffffffu, want);
    const double* cc = p.km_aux + k * IN_MAX;  // norms [k], max norm
    const double2* bf = reinterpret_cast<const double2*>(p.km_aux) + lane;
    const double G = 4.0 * (4.0 * IN_MAX + 8.0) * 0x1.0p-53;
    constexpr int MT = HPAC_KM_MT;  // m-tiles (8 points each) per pass
    int mine = 0;
#pragma unroll 1
    for (int m0 = 0; m0 < 4; m0 += MT) {
#if HPAC_KM_PF
      // L1 prefetch of the rows the next pass loads (after the last pass:
      // the first rows of this thread's next step), one 128-byte line per
      // lane, so their HBM latency overlaps this pass's DMMAs
      if (lane < 16 * MT) {
        const int64_t row = (m0 + MT < 4 ? base + 8 * (m0 + MT) : base + p.stride) + (lane >> 1);
        if (row < p.n)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p.region.in + row * IN_MAX + (lane & 1) * 16));
      }
#endif
      if (!((wm >> (8 * m0)) & ((1ull << (8 * MT)) - 1))) continue;  // no point of this pass
      double a[MT][8], xx[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int src = 8 * (m0 + i) + g;
        if ((wm >> src) & 1u) {
          // k-step s of slot t <-> dimension 8(s/2) + 2t + s%2: 64 contiguous
          // bytes per (row, chunk) across the group's four lanes
          const double2* x =
              reinterpret_cast<const double2*>(p.region.in + (base + src) * IN_MAX) + t;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 v = __ldg(x + 4 * q);
            a[i][2 * q] = v.x;
            a[i][2 * q + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int s = 0; s < 8; ++s) a[i][s] = 0.0;
        }
        double ss = 0.0;
#pragma unroll
        for (int s = 0; s < 8; ++s) ss = fma(a[i][s], a[i][s], ss);
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        xx[i] = ss + __shfl_xor_sync(0xffffffffu, ss, 2);
      }
      double m1[MT], m2[MT];
      int best[MT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        m1[i] = m2[i] = dinf();
        best[i] = 0;
      }
      // NT n-tiles (8 centroids each) per step: NT independent accumulation
      // chains per m-tile; a k % (8 NT) tail runs one n-tile at a time
      int j = 0;
      const double2* bj = bf;
      const double* cj = cc + 2 * t;
      for (; j + 8 * HPAC_KM_NT <= k; j += 8 * HPAC_KM_NT, bj += 128 * HPAC_KM_NT, cj += 8 * HPAC_KM_NT)
        dmma_tiles<HPAC_KM_NT, MT>(bj, cj, j, t, a, xx, m1, m2, best);
      for (; j < k; j += 8, bj += 128, cj += 8) dmma_tiles<1, MT>(bj, cj, j, t, a, xx, m1, m2, best);
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        // merge the four lanes of the group (each saw 2 of every 8 centroids)
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
          const double o1 = __shfl_xor_sync(0xffffffffu, m1[i], off);
          const double o2 = __shfl_xor_sync(0xffffffffu, m2[i], off);
          const int ob = __shfl_xor_sync(0xffffffffu, best[i], off);
          if (o1 < m1[i] || (o1 == m1[i] && ob < best[i])) {
            m2[i] = fmin(m1[i], o2);
            m1[i] = o1;
            best[i] = ob;
          } else {
            m2[i] = fmin(m2[i], o1);
          }
        }
        // cc[k] = max norm, NaN when any centroid is non-finite: E then
        // fails the test and the point takes the reference path; so does a
        // non-finite point (|x|^2 = inf/NaN) and any overflowing estimate
        const double E = G * (xx[i] + __ldg(cc + k));
        const int code = (m2[i] - m1[i] > 2.0 * E + 16.0 * 0x1.0p-53 * fabs(m2[i])) ? best[i] : -1;
        // point L's result sits in lanes 4(L%8) .. +3 of m-tile L/8
        const int v = __shfl_sync(0xffffffffu, code, 4 * (lane & 7));
        if ((lane >> 3) == m0 + i) mine = v;
      }
    }
    if (want && mine < 0) mine = exact_argmin_reload(p, idx, p.region.centroids);
    return (double)mine;
  }
};

// ---------------------------------------------------------------------------
// LavaMD (Rodinia lavaMD, restated per SURVEY.md Appendix C; not in the
// reference, parity against oracle/hpac_oracle.c). Boxes on a boxes1d^3 grid,
// `particles` per box (= threads_per_team: lane = home particle). Item =
// home box (per-team mapping); encounter r = neighbour box r (self first,
// then the 26-neighbourhood in z,y,x order inside the grid). The
// approximated region is one neighbour box's force contribution to the
// lane's particle: out = (v, x, y, z) accumulated into fv. Neighbour
// particles are staged in shared memory by the whole team OUTSIDE the
// region (round_begin), so thread/warp decisions never skip a barrier.
// exp() is a fixed sequence of correctly rounded operations and fused
// multiply-adds (fma() is exactly rounded on both sides), shared with the
// oracle, so the contributions (and TAF decisions on them) are bit-identical
// to the CPU restatement.
// e^x = 2^k * 2^(j/64) * e^r, n = rint(64 x/ln2) = 64k + j, r = x - n ln2/64
// (two-constant reduction, |r| <= ln2/128) and e^r by its degree-5 Taylor
// polynomial (truncation <= 3.5e-17 relative); 2^(j/64) from a 64-entry
// table (correctly rounded, staged in shared memory by AppLavaMD::init). A
// fixed sequence of correctly rounded operations and fused multiply-adds, so
// the oracle's restatement (oracle/hpac_oracle.c lava_exp) is bit-identical.
// 10 FP64 operations instead of the 14 of a degree-11 polynomial on
// |r| <= ln2/2, and <= 1.5 ulp instead of 1.2e-15.
static __constant__ double kLavaExpT[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};
#define HPAC_LAVA_L64 0x1.71547652b82fep+6  /* 64/ln2 */
#define HPAC_LAVA_LN2_64_HI 0x1.62e42fefa39efp-7
#define HPAC_LAVA_LN2_64_LO 0x1.abc9e3b39803fp-62
#define HPAC_LAVA_SHIFT 0x1.8p52
// the 64-bit constants of lava_exp as a constant-bank array: the DFMAs take
// them as c[bank][offset] operands. As literals, ptxas rebuilt each one per
// pair with two UMOV/IMAD.MOV (12 of ~53 warp instructions per pair).
static __constant__ double kLavaC[6] = {HPAC_LAVA_L64, HPAC_LAVA_LN2_64_HI, HPAC_LAVA_LN2_64_LO,
                                        0x1.1111111111111p-7, 0x1.5555555555555p-5,
                                        0x1.5555555555555p-3};

__device__ __forceinline__ double lava_exp(double x, const double* tab) {
  const double ts = fma(x, kLavaC[0], HPAC_LAVA_SHIFT);  // 1.5*2^52 + n: n in the low word
  const double kd = __dsub_rn(ts, HPAC_LAVA_SHIFT);
  double r = fma(-kd, kLavaC[1], x);
  r = fma(-kd, kLavaC[2], r);
  double s = kLavaC[3];  // 1/120
  s = fma(s, r, kLavaC[4]);
  s = fma(s, r, kLavaC[5]);
  s = fma(s, r, 0x1.0000000000000p-1);
  s = fma(s, r, 1.0);
  s = fma(s, r, 1.0);
  const int n = __double2loint(ts);  // == (int)kd, without an F2I
  const double t = __dmul_rn(tab[n & 63], s);
  const int k = n >> 6;  // floor(n / 64)
  // exact power-of-two scaling == ldexp while the result stays normal: add
  // k to the exponent field (t in [0.99, 2.01]) on the integer pipe
  if (k > -1021 && k < 1022) return __longlong_as_double(__double_as_longlong(t) + ((long long)k << 52));
  return ldexp(t, k);
}

__host__ __device__ __forceinline__ int lava_neighbours(int64_t box, int b1, int64_t* nb) {
  const int bx = (int)(box % b1), by = (int)((box / b1) % b1), bz = (int)(box / ((int64_t)b1 * b1));
  int c = 0;
  if (nb) nb[c] = box;
  ++c;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        const int x = bx + dx, y = by + dy, z = bz + dz;
        if (x < 0 || y < 0 || z < 0 || x >= b1 || y >= b1 || z >= b1) continue;
        if (nb) nb[c] = ((int64_t)z * b1 + y) * b1 + x;
        ++c;
      }
  return c;
}

// the r-th neighbour box of `box` in lava_neighbours order (no local array)
__host__ __device__ __forceinline__ int64_t lava_neighbour_at(int64_t box, int b1, int r) {
  if (r == 0) return box;
  const int bx = (int)(box % b1), by = (int)((box / b1) % b1), bz = (int)(box / ((int64_t)b1 * b1));
  int c = 1;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (!dx && !dy && !dz) continue;
        const int x = bx + dx, y = by + dy, z = bz + dz;
        if (x < 0 || y < 0 || z < 0 || x >= b1 || y >= b1 || z >= b1) continue;
        if (c == r) return ((int64_t)z * b1 + y) * b1 + x;
        ++c;
      }
  return -1;
}

// The pair loop over a staged neighbour box, kept out of line so its register
// allocation (and the code ptxas generates for it) does not depend on the
// engine state live around it (TAF windows, votes): the exact and the
// approximate kernels run the identical loop.
static __device__ __noinline__ double4 lava_box_contribution(const double* rv_home, const double* s, int P,
                                                      double na2, const double* etab) {
  const double4 me = *reinterpret_cast<const double4*>(rv_home);
  // exponent argument -a2 (vA + vB - dot) with -a2 folded into the home
  // particle (once) and into the staged vB (staging): 5 ops instead of 6
  // -nax = na2 x etc.: the exponent argument is an + (-a2 vB - a2 rA.rB) as
  // three FMAs onto the staged -a2 vB and one add (5 ops before: DMUL, two
  // FMAs, add, subtract)
  const double an = __dmul_rn(na2, me.x), nax = -__dmul_rn(na2, me.y), nay = -__dmul_rn(na2, me.z),
               naz = -__dmul_rn(na2, me.w);
  double fv = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
#ifndef HPAC_LAVA_UNROLL
#define HPAC_LAVA_UNROLL 1  // measured: 1 (32.7 ms) < 4 (35.5) < 2 (36.5) at 32^3
#endif
  constexpr int kUnroll = HPAC_LAVA_UNROLL;
#pragma unroll kUnroll
  for (int j = 0; j < P; ++j) {
    const double2 b01 = *reinterpret_cast<const double2*>(s + j * 4);
    const double2 b23 = *reinterpret_cast<const double2*>(s + j * 4 + 2);
    const double q2 = s[P * 4 + j];  // 2*qv, staged (exact doubling)
    const double sb = fma(naz, b23.y, fma(nay, b23.x, fma(nax, b01.y, b01.x)));  // b01.x = -a2 vB
    const double vij = lava_exp(__dadd_rn(an, sb), etab);
    // t = 2 q vij exactly as before (power-of-two scaling is exact); the
    // potential is accumulated doubled and halved once at the end: the
    // same bits as summing q*vij
    const double t = __dmul_rn(q2, vij);
    fv = __dadd_rn(fv, t);
    // sum_j t (rA - rB) = rA sum_j t - sum_j t rB: one FMA per component
    // and pair instead of a subtraction and an FMA
    sx = fma(t, b01.y, sx);
    sy = fma(t, b23.x, sy);
    sz = fma(t, b23.y, sz);
  }
  return make_double4(0.5 * fv, fma(me.y, fv, -sx), fma(me.z, fv, -sy), fma(me.w, fv, -sz));
}

struct AppLavaMD : AppBase {
  // FP64-latency-bound pair loop: keep >= 24 warps per SM (<= 85 registers)
#ifndef HPAC_LAVA_MINB
#define HPAC_LAVA_MINB 3
#endif
  static constexpr int MIN_BLOCKS_256 = HPAC_LAVA_MINB;
  // the TAF kernel (4 outputs x h window, votes) runs best at 64 registers
  // (32 warps/SM): 96.3 vs 102.5 ms at 48^3; exact prefers 80 (93.3 vs 95.8)
#ifndef HPAC_LAVA_TAF_MINB
#define HPAC_LAVA_TAF_MINB 4
#endif
  static constexpr int min_blocks_256(int tech) {
    return tech == HPAC_TECH_TAF ? HPAC_LAVA_TAF_MINB : HPAC_LAVA_MINB;
  }
  static constexpr bool HAS_IACT = false;  // no region inputs (iACT needs in(...))
  static constexpr int IN_MAX = 1;
  static constexpr int OUT_MAX = 4;
  // the exp table (lava_exp) after the staged particles: [P*5, P*5 + 64)
  __device__ static void init(const EngineParams& p, double* scratch) {
    double* tab = scratch + (size_t)p.region.lavamd_particles * 5;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) tab[i] = kLavaExpT[i];
  }
  __device__ static int encounters(const EngineParams& p, int64_t idx) {
    return lava_neighbours(idx, p.region.lavamd_boxes1d, nullptr);
  }
  // stage neighbour box `round` of home box idx: rv (4) + qv (1) per particle
  // `need`: this thread evaluates in this round. The first barrier also
  // retires the previous round's readers of s; nothing is staged when no
  // thread of the team evaluates (team-uniform result of the barrier).
  __device__ static void round_begin(const EngineParams& p, int64_t idx, int round, double* s,
                                     bool valid, bool need) {
    if (!__syncthreads_or(need)) return;
    if (valid) {
      const int64_t b = lava_neighbour_at(idx, p.region.lavamd_boxes1d, round);
      if (b >= 0) {
        const int P = p.region.lavamd_particles;
        const double2* src = reinterpret_cast<const double2*>(p.region.in + b * P * 4);
        double2* dst = reinterpret_cast<double2*>(s);
        const double na2 = -__dmul_rn(__dmul_rn(2.0, p.region.lavamd_alpha), p.region.lavamd_alpha);
        for (int i = threadIdx.x; i < P * 2; i += blockDim.x) {
          double2 v = __ldg(src + i);
          if ((i & 1) == 0) v.x = __dmul_rn(na2, v.x);  // (v, x) half: stage -a2 v
          dst[i] = v;
        }
        for (int i = threadIdx.x; i < P; i += blockDim.x)
          s[P * 4 + i] = 2.0 * __ldg(p.region.table_out + b * P + i);
      }
    }
    __syncthreads();
  }
  __device__ static void load(const EngineParams&, int64_t, double (&)[IN_MAX]) {}
  // one neighbour box's contribution to the lane's particle (Rodinia
  // lavaMD kernel body, FMA form restated identically in the oracle)
  __device__ static bool eval(const EngineParams& p, int64_t idx, const double (&)[IN_MAX],
                              double (&out)[OUT_MAX], const double* s, int local, int) {
    const int P = p.region.lavamd_particles;
    const double na2 = -__dmul_rn(__dmul_rn(2.0, p.region.lavamd_alpha), p.region.lavamd_alpha);
    const double4 f = lava_box_contribution(p.region.in + (idx * P + local) * 4, s, P, na2, s + P * 5);
    out[0] = f.x;
    out[1] = f.y;
    out[2] = f.z;
    out[3] = f.w;
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX],
                               int local) {
    double* f = p.region.out + (idx * p.region.lavamd_particles + local) * 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) f[c] = __dadd_rn(f[c], out[c]);
  }
};

}  // namespace hpac
