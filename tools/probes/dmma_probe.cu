// Probe: can FP64 tensor-core MMAs (mma.sync f64) run beside vector DFMA?
// c128 layered passes are bound by the FP64 FMA pipe (profiles/r02_*): if
// DMMA issues to a separate unit, phases could split their work between the
// two.  Measures DFMA alone, DMMA m8n8k4 alone, and both interleaved in one
// warp's instruction stream.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// MODE 0: DFMA only (16 chains); 1: DMMA only (8 accumulators);
// 2: both (16 DFMA chains + 8 DMMA per iteration)
template <int MODE>
__global__ void k(double* out, double a0, double b0, int iters) {
  double acc[16], b[16], d[8][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc[i] = a0 + i; b[i] = b0 * (i + 1); }
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = a0 - i;
  const double x = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fma(x, b[i], acc[i]);
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(d[i], x, b[i]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, 64 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int threads : {256, 512}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int blocks = sms * (1024 / threads);
      auto launch = [&]() {
        if (mode == 0) k<0><<<blocks, threads>>>(o, 1.0, 0.5, iters);
        else if (mode == 1) k<1><<<blocks, threads>>>(o, 1.0, 0.5, iters);
        else k<2><<<blocks, threads>>>(o, 1.0, 0.5, iters);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)blocks * threads / 32;
      // DFMA: 32 FMA per warp instruction; DMMA m8n8k4: 8*8*4 = 256 FMA per warp instruction
      const double f_dfma = mode != 1 ? warps * iters * 16 * 32 : 0;
      const double f_dmma = mode != 0 ? warps * iters * 8 * 256 : 0;
      printf("threads %4d mode %s: %.3f ms  DFMA %.2f TFLOP/s  DMMA %.2f TFLOP/s  total %.2f TFLOP/s\n", threads,
             mode == 0 ? "dfma " : mode == 1 ? "dmma " : "mixed", ms, 2 * f_dfma / ms / 1e9, 2 * f_dmma / ms / 1e9,
             2 * (f_dfma + f_dmma) / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
