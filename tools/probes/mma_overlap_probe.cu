// Probe: can independent FP32 work issue while mma.sync HMMAs occupy the
// tensor pipe?  8 warps/SM; per iteration 4 HMMA (4 chains) + F FFMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int F>
__global__ void k(float* out, int iters) {
  uint32_t a0 = 0x3c003c00u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = b0 + 1;
  float d[4][4];
  float x[16];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 0.001f + i;
  const float c = 1.0001f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
#pragma unroll
      for (int f = 0; f < F / 4; ++f) x[f % 16] = fmaf(x[f % 16], c, x[(f + 7) % 16]);
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][3];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int F>
void run(int sms, float* o) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  k<F><<<sms, 256>>>(o, iters);
  cudaEventRecord(e0);
  k<F><<<sms, 256>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * 1.965e9;
  printf("FFMA per 4 HMMA %3d: %.1f cycles per iteration (per SM, 8 warps)\n", F, cyc / iters);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 64 << 20);
  run<0>(sms, o); run<8>(sms, o); run<16>(sms, o); run<32>(sms, o); run<64>(sms, o); run<128>(sms, o);
  return 0;
}
