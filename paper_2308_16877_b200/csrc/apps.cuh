// apps.cuh — application kernels (the reference's Regions, bench/*.hpp) as
// device functions. Each app supplies load (the iACT key, and the inputs
// of the accurate path), eval (the accurate region) and store.
#pragma once

#include <cstdint>

#include "engine.h"
#include "hpac_device.cuh"

namespace hpac {

// black_scholes_call, bench/blackscholes.hpp:21-36. Returns false where the
// reference throws ConfigError (invalid parameters).
__device__ __forceinline__ bool bs_call(double spot, double strike, double rate, double vol,
                                        double mat, double& price) {
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol >= 0) || !isfinite(rate))
    return false;
  double disc_strike = strike * exp(-rate * mat);
  double sst = vol * sqrt(mat);
  if (sst == 0.0) {
    double v = spot - disc_strike;
    price = v < 0.0 ? 0.0 : v;
    return true;
  }
  double d1 = (log(spot / strike) + (rate + 0.5 * vol * vol) * mat) / sst;
  double d2 = d1 - sst;
  double n1 = 0.5 * erfc(-d1 / 1.4142135623730951);
  double n2 = 0.5 * erfc(-d2 / 1.4142135623730951);
  price = spot * n1 - disc_strike * n2;
  return true;
}

// Generic pure region over a work index (HPAC_APP_TABLE): load_input reads
// `in`, evaluate returns the precomputed accurate output `table_out`.
struct AppTable {
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
                              double (&out)[OUT_MAX], const double*) {
    const double* src = p.region.table_out + idx * p.out_dims;
#pragma unroll
    for (int d = 0; d < OUT_MAX; ++d)
      if (d < p.out_dims) out[d] = src[d];
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX]) {
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
struct AppSynthetic {
  static constexpr int IN_MAX = 1;
  static constexpr int OUT_MAX = 1;
  __device__ static void load(const EngineParams& p, int64_t idx, double (&in)[IN_MAX]) {
    in[0] = synthetic_value(p.region.synthetic_profile, idx, p.region.seed);
  }
  __device__ static void init(const EngineParams&, double*) {}
  __device__ static bool eval(const EngineParams& p, int64_t idx, const double (&)[IN_MAX],
                              double (&out)[OUT_MAX], const double*) {
    out[0] = synthetic_eval(synthetic_value(p.region.synthetic_profile, idx, p.region.seed));
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX]) {
    if (p.region.out) p.region.out[idx] = out[0];
  }
};

// bench/blackscholes.hpp:72-92 (AoS option = 5 doubles)
struct AppBlackScholes {
  static constexpr int IN_MAX = 5;
  static constexpr int OUT_MAX = 1;
  __device__ static void load(const EngineParams& p, int64_t idx, double (&in)[IN_MAX]) {
    const double* o = p.region.in + idx * 5;
#pragma unroll
    for (int d = 0; d < 5; ++d) in[d] = __ldg(o + d);
  }
  __device__ static void init(const EngineParams&, double*) {}
  __device__ static bool eval(const EngineParams&, int64_t, const double (&in)[IN_MAX],
                              double (&out)[OUT_MAX], const double*) {
    return bs_call(in[0], in[1], in[2], in[3], in[4], out[0]);
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX]) {
    if (p.region.out) __stcs(p.region.out + idx, out[0]);
  }
};

// K-Means distance region (bench/kmeans.hpp:82-102). The region's outputs
// are the k distances; the host argmin (kmeans.hpp:111-121) is fused here,
// so the engine payload is the label (stored as a double) and the k
// distances are written only when the caller asks for them (region.out).
// Centroids are staged once per CTA in shared memory (broadcast reads).
// Default arithmetic is the reference's order without contraction, so
// distances and labels are bit-identical to the CPU; the argmin takes a
// sqrt only when a squared distance improves (sqrt is monotone, so the
// strict-< / lowest-index result is unchanged).
struct AppKmeans {
  static constexpr int IN_MAX = 32;
  static constexpr int OUT_MAX = 1;
  __device__ static void init(const EngineParams& p, double* scratch) {
    const int kd = p.region.kmeans_k * p.region.kmeans_dims;
    for (int i = threadIdx.x; i < kd; i += blockDim.x) scratch[i] = p.region.centroids[i];
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
  __device__ static bool eval(const EngineParams& p, int64_t idx, const double (&in)[IN_MAX],
                              double (&out)[OUT_MAX], const double* cent) {
    const int dims = p.region.kmeans_dims, k = p.region.kmeans_k;
    const bool fast = (p.region.flags & HPAC_REGION_KMEANS_FAST_MATH) != 0;
    double* dist = p.region.out ? p.region.out + idx * k : nullptr;
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
          best_ssq = ssq;
        }
      } else if (c == 0) {
        best_ssq = ssq;
        best_d = __dsqrt_rn(ssq);
      } else if (ssq < best_ssq) {
        double dd = __dsqrt_rn(ssq);
        if (dd < best_d) {
          best = c;
          best_d = dd;
          best_ssq = ssq;
        }
      }
    }
    out[0] = (double)best;
    return true;
  }
  __device__ static void store(const EngineParams& p, int64_t idx, const double (&out)[OUT_MAX]) {
    if (p.region.labels) p.region.labels[idx] = (int32_t)out[0];
  }
};

}  // namespace hpac
