// Probe: FP32 FMA issue rate, 3-register form vs immediate form, and FP64.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float a0, float b0, int iters) {
  float acc[16];
  float b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc[i] = a0 + i; b[i] = b0 * (i + 1); }
  float x = threadIdx.x * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) acc[i] = fmaf(x, b[i], acc[i]);          // 3 registers
      else acc[i] = fmaf(x, 1.0001f + 0.001f * i, acc[i]);    // immediate
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void kd(double* out, double a0, double b0, int iters) {
  double acc[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i] = a0 + i; b[i] = b0 * (i + 1); }
  double x = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(x, b[i], acc[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int blocks = sms * (2048 / threads);
      auto launch = [&]() {
        if (mode == 0) k<0><<<blocks, threads>>>(o, 1.f, 0.5f, iters);
        else if (mode == 1) k<1><<<blocks, threads>>>(o, 1.f, 0.5f, iters);
        else kd<<<blocks, threads>>>((double*)o, 1.0, 0.5, iters / 2);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = (double)blocks * threads * (mode == 2 ? iters / 2 * 8.0 : iters * 16.0);
      printf("threads %4d mode %s: %.3f ms  %.2f T FMA/s  = %.1f FMA/clk/SM at 1.965 GHz\n", threads,
             mode == 0 ? "ffma-3reg" : mode == 1 ? "ffma-imm " : "dfma     ", ms, fmas / ms / 1e9,
             fmas / ms / 1e-3 / sms / 1.965e9);
    }
  }
  return 0;
}
