// Probe: legacy warp-level mma.sync throughput on sm_100a (registers only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void k(float* out, int iters) {
  uint32_t a[4], b[2];
  float d[8][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u + threadIdx.x * 3 + i;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (KIND == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += d[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int kind = 0; kind < 2; ++kind)
    for (int threads : {128, 256, 512}) {
      const int blocks = sms * (1024 / threads);
      auto launch = [&]() {
        if (kind == 0) k<0><<<blocks, threads>>>(o, iters);
        else k<1><<<blocks, threads>>>(o, iters);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double macs = (double)blocks * (threads / 32) * iters * 8 * (kind == 0 ? 16 * 8 * 16 : 16 * 8 * 8);
      printf("%s warps/SM %2d: %.3f ms  %.1f TFLOP/s  (%.1f mma/clk/SM)\n", kind == 0 ? "f16 m16n8k16 " : "tf32 m16n8k8 ",
             blocks * threads / 32 / sms, ms, 2 * macs / ms / 1e9,
             (double)blocks * (threads / 32) * iters * 8 / (ms * 1e-3) / sms / 1.965e9);
    }
  return 0;
}
