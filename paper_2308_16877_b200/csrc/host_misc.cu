// host_misc.cu — quality metrics on the device (metrics.hpp:17-45) and the
// seeded input generators (bench/blackscholes.hpp:42-68,
// bench/binomial.hpp:54-69, bench/kmeans.hpp:25-47). The generators use the
// same libstdc++ engines and distributions (std::mt19937_64,
// std::uniform_real_distribution, std::normal_distribution) in the same
// draw order, so a given seed yields the reference's inputs bit for bit.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "apps.cuh"
#include "hpac_device.cuh"
#include "hpac_offload.h"

#define HPAC_API extern "C" __attribute__((visibility("default")))

namespace hpac {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs
constexpr int kRedThreads = 256;

// MAPE partials: |a-b|/|a|; a == 0 && b != 0 flags infinity (metrics.hpp:17-33)
__global__ void mape_partial(const double* a, const double* b, int64_t n, double* part,
                             unsigned long long* inf) {
  __shared__ double sh[kRedThreads];
  double s = 0.0;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = a[i], y = b[i];
    if (x == 0.0) {
      if (y != 0.0) bad = true;
      continue;
    }
    s += fabs(x - y) / fabs(x);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(inf, 1ull);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// fixed-order final sum (deterministic run to run)
__global__ void sum_partials(const double* part, int m, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += part[i];
    out[0] = s;
  }
}

__global__ void mcr_kernel(const int32_t* a, const int32_t* b, int64_t n,
                           unsigned long long* cnt) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += a[i] != b[i];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

cudaError_t mape_launch(const double* a, const double* b, int64_t n, double* d_sum,
                        unsigned long long* d_inf, cudaStream_t st) {
  double* part;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * kRedBlocks, st);
  if (e != cudaSuccess) return e;
  mape_partial<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, n, part, d_inf);
  sum_partials<<<1, 32, 0, st>>>(part, kRedBlocks, d_sum);
  cudaFreeAsync(part, st);
  return cudaGetLastError();
}

cudaError_t mcr_launch(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* d_cnt,
                       cudaStream_t st) {
  mcr_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, n, d_cnt);
  return cudaGetLastError();
}

// Independent DFMA chains: 8 per thread, no memory traffic in the loop.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double* sink, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1.2345) sink[0] = s;
}

// Independent FP64 tensor-op (DMMA m8n8k4) chains: 8 per warp.
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* sink, int iters, double a, double b) {
  double d[8][2];
#pragma unroll
  for (int u = 0; u < 8; ++u) d[u][0] = d[u][1] = threadIdx.x + u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma_m8n8k4(d[u][0], d[u][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += d[u][0] + d[u][1];
  if (s == 1.2345) sink[0] = s;
}

}  // namespace hpac

namespace {
template <class K>
int probe_peak(K kernel, int blocks_per_sm, int iters, double flops_per_thread_iter, double* tflops) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HPAC_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink;
  if (cudaMalloc(&sink, 8) != cudaSuccess) return HPAC_ERR_CUDA;
  const int blocks = sms * blocks_per_sm, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kernel<<<blocks, threads>>>(sink, 64, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kernel<<<blocks, threads>>>(sink, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return HPAC_ERR_CUDA;
  *tflops = flops_per_thread_iter * iters * (double)blocks * threads / (best * 1e-3) / 1e12;
  return HPAC_OK;
}
}  // namespace

// FP64 tensor-op peak (the K-Means DMMA filter's roofline): 8 chains of
// m8n8k4 (512 flops per warp-instruction = 16 per thread) per warp.
HPAC_API int hpac_probe_dmma_peak(double* tflops) {
  return probe_peak(hpac::dmma_probe_kernel, 4, 1024, 8.0 * 16.0, tflops);
}

HPAC_API int hpac_probe_fp64_peak(double* tflops) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HPAC_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink;
  if (cudaMalloc(&sink, 8) != cudaSuccess) return HPAC_ERR_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  hpac::fp64_probe_kernel<<<blocks, threads>>>(sink, 64, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    hpac::fp64_probe_kernel<<<blocks, threads>>>(sink, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return HPAC_ERR_CUDA;
  double flops = 2.0 * 8.0 * 8.0 * iters * (double)blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return HPAC_OK;
}

// ---- generators -----------------------------------------------------------

// Desk portfolio: `base_block` distinct options tiled with multiplicative
// jitter on spot and vol (bench/blackscholes.hpp:42-68). out = n x 5.
HPAC_API int hpac_make_bs_portfolio(int64_t n, uint64_t seed, int32_t base_block, double jitter,
                                    double* out) {
  if (n < 0 || base_block < 1 || !out) return HPAC_ERR_CONFIG;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> spot(40.0, 160.0);
  std::uniform_real_distribution<double> moneyness(0.8, 1.2);
  std::uniform_real_distribution<double> vol(0.1, 0.5);
  std::uniform_real_distribution<double> maturity(0.25, 2.0);
  std::vector<double> base((size_t)base_block * 5);
  for (int b = 0; b < base_block; ++b) {
    double* o = &base[(size_t)b * 5];
    o[0] = spot(rng);
    o[1] = o[0] * moneyness(rng);
    o[2] = 0.03;
    o[3] = vol(rng);
    o[4] = maturity(rng);
  }
  std::normal_distribution<double> wiggle(1.0, jitter);
  for (int64_t i = 0; i < n; ++i) {
    const double* b = &base[(size_t)(i % base_block) * 5];
    double* o = out + (size_t)i * 5;
    for (int d = 0; d < 5; ++d) o[d] = b[d];
    if (i >= base_block) {
      o[0] *= std::abs(wiggle(rng));
      o[3] *= std::abs(wiggle(rng));
    }
  }
  return HPAC_OK;
}

// American-put portfolio with a moneyness ramp (bench/binomial.hpp:54-69).
HPAC_API int hpac_make_binomial_portfolio(int64_t n, uint64_t seed, double jitter, double* out) {
  if (n < 0 || !out) return HPAC_ERR_CONFIG;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> wiggle(1.0, jitter);
  const long long denom = n - 1 > 1 ? n - 1 : 1;
  for (int64_t i = 0; i < n; ++i) {
    double* o = out + (size_t)i * 5;
    double m = 0.8 + 0.4 * static_cast<double>(i) / denom;
    o[0] = 100.0 * std::abs(wiggle(rng));
    o[1] = o[0] * m * std::abs(wiggle(rng));
    o[2] = 0.05;
    o[3] = 0.25 * std::abs(wiggle(rng));
    o[4] = 1.0;
  }
  return HPAC_OK;
}

// LavaMD particles (Rodinia lavaMD: (rand() % 10 + 1) / 10 per value).
HPAC_API int hpac_make_lavamd(int32_t boxes1d, int32_t particles, uint64_t seed, double* rv,
                              double* qv) {
  if (boxes1d < 1 || particles < 1 || !rv || !qv) return HPAC_ERR_CONFIG;
  const int64_t n = (int64_t)boxes1d * boxes1d * boxes1d * particles;
  for (int64_t i = 0; i < n; ++i) {
    for (int c = 0; c < 5; ++c) {
      uint64_t h = hpac::splitmix64(seed ^ (uint64_t)(5 * i + c));
      double v = (double)(h % 10 + 1) / 10.0;
      if (c < 4)
        rv[i * 4 + c] = v;
      else
        qv[i] = v;
    }
  }
  return HPAC_OK;
}

// Gaussian blobs around k centres on a circle (bench/kmeans.hpp:25-47).
HPAC_API int hpac_make_blobs(int64_t n, int32_t dims, int32_t k, uint64_t seed,
                             double separation, double* out) {
  if (n < 0 || dims < 1 || k < 1 || !out) return HPAC_ERR_CONFIG;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> noise(0.0, 1.0);
  std::vector<double> centers((size_t)k * dims, 0.0);
  for (int c = 0; c < k; ++c) {
    double angle = 2.0 * M_PI * c / k;
    centers[(size_t)c * dims] = separation * std::cos(angle);
    if (dims > 1) centers[(size_t)c * dims + 1] = separation * std::sin(angle);
  }
  for (int64_t i = 0; i < n; ++i) {
    int c = (int)(i % k);
    for (int d = 0; d < dims; ++d)
      out[(size_t)i * dims + d] = centers[(size_t)c * dims + d] + noise(rng);
  }
  return HPAC_OK;
}

// ---- diagnostics: fastmath vs libdevice (tests/test_gpu_fastmath.py) ----
namespace hpac {
__global__ void fm_eval_kernel(int kind, const double* __restrict__ x, double* __restrict__ y,
                               int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    switch (kind) {
      case HPAC_FM_EXP: v = fm::exp(x[i]); break;
      case HPAC_FM_LOG: v = fm::log(x[i]); break;
      case HPAC_FM_ERFC: v = fm::erfc(x[i]); break;
      case HPAC_FM_BS: {
        const double* o = x + i * 5;
        if (!bs_call(o[0], o[1], o[2], o[3], o[4], v)) v = NAN;
        break;
      }
      case HPAC_FM_LIBDEVICE_EXP: v = ::exp(x[i]); break;
      case HPAC_FM_LIBDEVICE_LOG: v = ::log(x[i]); break;
      case HPAC_FM_LIBDEVICE_ERFC: v = ::erfc(x[i]); break;
      case HPAC_FM_LIBDEVICE_BS: {
        const double* o = x + i * 5;
        v = bs_call_libdevice(o[0], o[1], o[2], o[3], o[4]);
        break;
      }
    }
    y[i] = v;
  }
}
}  // namespace hpac

HPAC_API int hpac_fm_eval(int32_t kind, const double* x, double* y, int64_t n, void* stream) {
  if (kind < HPAC_FM_EXP || kind > HPAC_FM_LIBDEVICE_BS || n < 0 || (n > 0 && (!x || !y)))
    return HPAC_ERR_CONFIG;
  if (n == 0) return HPAC_OK;
  const int64_t blocks = (n + 255) / 256;
  hpac::fm_eval_kernel<<<(int)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0,
                         (cudaStream_t)stream>>>(kind, x, y, n);
  return cudaGetLastError() == cudaSuccess ? HPAC_OK : HPAC_ERR_CUDA;
}
