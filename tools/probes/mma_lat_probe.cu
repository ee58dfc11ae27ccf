// Probe: mma.sync m16n8k16 f16 latency / per-warp throughput vs independent
// accumulator chains and warps per SM (sm_100a).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void k(float* out, int iters) {
  uint32_t a0 = 0x3c003c00u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = b0 + 1;
  float d[CH][4];
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += d[j][0] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
void run(int warps, int sms, float* o) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  k<CH><<<sms, 32 * warps>>>(o, iters);
  cudaEventRecord(e0);
  k<CH><<<sms, 32 * warps>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * 1.965e9;
  printf("chains %d warps/SM %2d: %.1f cycles per mma per warp, %.3f mma/clk/SM\n", CH, warps,
         cyc / (double(iters) * CH), double(iters) * CH * warps / cyc);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 64 << 20);
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, sms, o); run<2>(w, sms, o); run<4>(w, sms, o); run<8>(w, sms, o);
  }
  return 0;
}
