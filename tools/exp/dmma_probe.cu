// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu && ./dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(acc[i][0], acc[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(av, acc[i], bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 26);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int blocks = sms * 4, threads = warps * 32 / 4;
    if (threads < 32) threads = 32;
    float ms = timeit([&] { k_dmma<8><<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999); });
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * threads / 32;
    float ms2 = timeit([&] { k_dfma<8><<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999); });
    double flops2 = 2.0 * 8 * (double)iters * blocks * threads;
    printf("warps/SM %2d: DMMA %.2f TFLOP/s (%.3f ms)  DFMA %.2f TFLOP/s (%.3f ms)\n", warps,
           flops / ms / 1e9, ms, flops2 / ms2 / 1e9, ms2);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
