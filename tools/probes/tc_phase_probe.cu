// Probe: one register phase as a tcgen05 TF32 GEMM.
//   D[m][n] = sum_k A[m][k] * B[n][k]   (M=128 rows, K=N=64 real: 32 complex amps)
// A (the tile rows) is written by the 128 threads into TMEM with tcgen05.st,
// B (the real block form of a 32x32 complex unitary) sits in shared memory in
// the K-major SWIZZLE_NONE core-matrix layout.  3xTF32: A_hi B_hi + A_lo B_hi +
// A_hi B_lo.  Checks correctness against FP64 and times repeated phases.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// B[n][k] -> byte offset in the K-major no-swizzle canonical layout:
// core matrix = 8 rows x 16 B; k-chunks (4 tf32) adjacent (LBO = 128 B);
// 8-row groups SBO = (K/4) * 128 B apart.
__host__ __device__ inline uint32_t bofs(int n, int k, int K) {
  return (n / 8) * (K / 4) * 128 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) k_probe(const float* __restrict__ A, const float* __restrict__ Bhi,
                                                  const float* __restrict__ Blo, float* __restrict__ D, int reps,
                                                  int terms) {
  constexpr int M = 128, N = 64, K = 64;
  __shared__ __align__(128) uint8_t sB[2][N * K * 4];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // B hi/lo into the canonical layout
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<float*>(sB[0] + bofs(n, k, K)) = Bhi[i];
    *reinterpret_cast<float*>(sB[1] + bofs(n, k, K)) = Blo[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // B written by generic proxy, read by the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  // TMEM columns: [0,64) A_hi, [64,128) A_lo, [128,192) D
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  float a[K];
  for (int k = 0; k < K; ++k) a[k] = A[tid * K + k];
  uint32_t phase = 0;
  for (int r = 0; r < reps; ++r) {
    uint32_t hi[32], lo[32];
    for (int half = 0; half < 2; ++half) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = a[half * 32 + j];
        hi[j] = to_tf32(x);
        lo[j] = to_tf32(x - __uint_as_float(hi[j]));
      }
      const uint32_t ah = tbase + lane_off + half * 32, al = tbase + lane_off + 64 + half * 32;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ah),
          "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]), "r"(hi[8]),
          "r"(hi[9]), "r"(hi[10]), "r"(hi[11]), "r"(hi[12]), "r"(hi[13]), "r"(hi[14]), "r"(hi[15]), "r"(hi[16]),
          "r"(hi[17]), "r"(hi[18]), "r"(hi[19]), "r"(hi[20]), "r"(hi[21]), "r"(hi[22]), "r"(hi[23]), "r"(hi[24]),
          "r"(hi[25]), "r"(hi[26]), "r"(hi[27]), "r"(hi[28]), "r"(hi[29]), "r"(hi[30]), "r"(hi[31]));
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(al),
          "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]), "r"(lo[8]),
          "r"(lo[9]), "r"(lo[10]), "r"(lo[11]), "r"(lo[12]), "r"(lo[13]), "r"(lo[14]), "r"(lo[15]), "r"(lo[16]),
          "r"(lo[17]), "r"(lo[18]), "r"(lo[19]), "r"(lo[20]), "r"(lo[21]), "r"(lo[22]), "r"(lo[23]), "r"(lo[24]),
          "r"(lo[25]), "r"(lo[26]), "r"(lo[27]), "r"(lo[28]), "r"(lo[29]), "r"(lo[30]), "r"(lo[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      constexpr uint32_t idesc = idesc_tf32<M, N>();
      const uint32_t d_t = tbase + 128;
      const uint32_t bh = smem_u32(sB[0]), bl = smem_u32(sB[1]);
      int issued = 0;
      for (int term = 0; term < terms; ++term) {
        const uint32_t a_col = (term == 1) ? 64 : 0;        // A_lo for term 1
        const uint32_t bsrc = (term == 2) ? bl : bh;         // B_lo for term 2
        for (int s = 0; s < K / 8; ++s) {
          const uint64_t bdesc = make_desc(bsrc + s * 256, 128, (K / 4) * 128);
          const uint32_t a_t = tbase + a_col + s * 8;
          const uint32_t acc = issued > 0 ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_t),
              "r"(a_t), "l"(bdesc), "r"(idesc), "r"(acc));
          ++issued;
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)));
    }
    // wait for the MMAs
    {
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(&mbar)), "r"(phase));
      phase ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[32];
    for (int half = 0; half < 2; ++half) {
      const uint32_t dt = tbase + lane_off + 128 + half * 32;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
          "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
            "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]),
            "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]),
            "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
          : "r"(dt));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 32; ++j) a[half * 32 + j] = __uint_as_float(d[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  for (int k = 0; k < K; ++k) D[tid * K + k] = a[k];
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
  constexpr int M = 128, K = 64, N = 64, C = 32;
  srand(7);
  auto rnd = [] { return (double)rand() / RAND_MAX * 2 - 1; };
  // random complex unitary via Gram-Schmidt
  std::vector<double> ur(C * C), ui(C * C);
  for (int i = 0; i < C * C; ++i) { ur[i] = rnd(); ui[i] = rnd(); }
  for (int r = 0; r < C; ++r) {
    for (int q = 0; q < r; ++q) {
      double pr = 0, pi = 0;  // <q|r>
      for (int k = 0; k < C; ++k) {
        pr += ur[q * C + k] * ur[r * C + k] + ui[q * C + k] * ui[r * C + k];
        pi += ur[q * C + k] * ui[r * C + k] - ui[q * C + k] * ur[r * C + k];
      }
      for (int k = 0; k < C; ++k) {
        ur[r * C + k] -= pr * ur[q * C + k] - pi * ui[q * C + k];
        ui[r * C + k] -= pr * ui[q * C + k] + pi * ur[q * C + k];
      }
    }
    double nn = 0;
    for (int k = 0; k < C; ++k) nn += ur[r * C + k] * ur[r * C + k] + ui[r * C + k] * ui[r * C + k];
    nn = sqrt(nn);
    for (int k = 0; k < C; ++k) { ur[r * C + k] /= nn; ui[r * C + k] /= nn; }
  }
  std::vector<double> B(N * K);
  for (int n = 0; n < C; ++n)
    for (int k = 0; k < C; ++k) {
      B[n * K + k] = ur[n * C + k];
      B[n * K + k + C] = -ui[n * C + k];
      B[(n + C) * K + k] = ui[n * C + k];
      B[(n + C) * K + k + C] = ur[n * C + k];
    }
  auto tf32r = [](double x) { float f = (float)x; uint32_t u; memcpy(&u, &f, 4); u = (u + 0x1000) & ~0x1FFFu; float g; memcpy(&g, &u, 4); return g; };
  std::vector<float> bh(N * K), bl(N * K), a(M * K);
  for (int i = 0; i < N * K; ++i) { bh[i] = tf32r(B[i]); bl[i] = tf32r((float)B[i] - bh[i]); }
  for (int i = 0; i < M * K; ++i) a[i] = (float)(rnd() * 0.01);
  float *dA, *dBh, *dBl, *dD;
  cudaMalloc(&dA, M * K * 4); cudaMalloc(&dBh, N * K * 4); cudaMalloc(&dBl, N * K * 4); cudaMalloc(&dD, M * K * 4);
  cudaMemcpy(dA, a.data(), M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dBh, bh.data(), N * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dBl, bl.data(), N * K * 4, cudaMemcpyHostToDevice);
  for (int terms : {1, 3}) {
    for (int reps : {1, 8}) {
      k_probe<<<1, 128>>>(dA, dBh, dBl, dD, reps, terms);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> d(M * K);
      cudaMemcpy(d.data(), dD, M * K * 4, cudaMemcpyDeviceToHost);
      // reference: apply B reps times in double
      std::vector<double> x(a.begin(), a.end()), y(M * K);
      for (int r = 0; r < reps; ++r) {
        for (int m = 0; m < M; ++m)
          for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += x[m * K + k] * B[n * K + k];
            y[m * K + n] = s;
          }
        x = y;
      }
      double maxerr = 0, maxv = 0;
      for (int i = 0; i < M * K; ++i) { maxerr = fmax(maxerr, fabs(d[i] - x[i])); maxv = fmax(maxv, fabs(x[i])); }
      printf("terms %d reps %d: %s  max|err| %.3e  rel %.3e\n", terms, reps, cudaGetErrorString(e), maxerr, maxerr / maxv);
    }
  }
  // throughput: many CTAs, many reps
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ctas : {1, 2}) {
    const int reps = 2000;
    k_probe<<<sms * ctas, 128>>>(dA, dBh, dBl, dD, 10, 3);
    cudaEventRecord(e0);
    k_probe<<<sms * ctas, 128>>>(dA, dBh, dBl, dD, reps, 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double macs = 3.0 * M * N * K * reps * sms * ctas;
    printf("ctas/SM %d: %.3f ms  %.1f TFLOP/s (3xTF32 counted), per phase per CTA %.0f ns (%s)\n", ctas, ms,
           2 * macs / ms / 1e9, ms * 1e6 / reps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
