// k_tc_pass -- register phases on the 5th-generation tensor cores (c64).
//
// Same pass structure as k_reg_pass (TMA tensor-map tile loads, register
// phases, swizzled shared-memory transposes, direct stores), with 128 compute
// threads each holding one *row* of 32 amplitudes: tile = 12 qubits = 5
// register bits x 7 thread bits.  A phase whose dense gates the planner fused
// into one 32x32 complex matrix U runs as a GEMM  out[row] = U . in[row]  for
// the 128 rows of the tile:
//   * rows go to TMEM (tcgen05.st, SASS STTM) as TF32 hi/lo splits of the real
//     and imaginary parts (A operand: lane = row, column = register index);
//   * U sits in shared memory as TF32 hi/lo in the K-major no-swizzle
//     core-matrix layout (B operand, one smem descriptor per K step);
//   * one elected thread issues 48 tcgen05.mma.kind::tf32 (M=128, N=32, K=8):
//     Re = A_re.Ur - A_im.Ui (b_negate), Im = A_re.Ui + A_im.Ur, each with the
//     3-term split  A_hi.B_hi + A_lo.B_hi + A_hi.B_lo  (FP32-level accuracy);
//   * tcgen05.commit -> mbarrier; the rows come back with tcgen05.ld (LDTM).
// A GEMM phase replaces 16 FMA per amplitude per fused 2-qubit gate by a fixed
// ~8 tensor MACs x 3 terms per amplitude, several times cheaper once a phase
// holds 3+ gates (tools/probes/tc_phase_probe.cu).
#pragma once
#include "svb_regpass.cuh"

namespace svb {

constexpr int kTcCompute = 128;
constexpr int kTcThreads = kTcCompute + 32;
constexpr int kTcCols = 256;  // TMEM columns per CTA: A re/im hi/lo (128) + D re/im (64)

__device__ __forceinline__ void tc_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kTcCompute) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&d)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
        "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]),
        "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]),
        "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
      : "r"(taddr)
      : "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_NONE, sm100 version bits
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// instruction descriptor: D f32, A/B tf32, K-major, N = 32, M = 128
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kTcIdescNegB = kTcIdesc | (1u << 14);

__device__ __forceinline__ void tc_mma(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

inline size_t tc_pass_smem_bytes(const PassHeader& h) {
  return 256 + align_up(size_t(h.coeff_count) * sizeof(float2), 1024) + size_t(h.tc_count) * kTcMatBytes +
         size_t(h.stages) * (sizeof(float2) << 12);
}

__global__ void __launch_bounds__(kTcThreads, 2) k_tc_pass(float2* __restrict__ amps,
                                                           const __grid_constant__ PassArgs<float2> args) {
  using C = float2;
  constexpr int RB = 5, NR = 32, T = 12, NT = kTcCompute;
  extern __shared__ __align__(1024) unsigned char smem[];
  const PassHeader& h = args.h;
  const int S = h.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  uint64_t* mma_bar = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 1);
  C* pool = reinterpret_cast<C*>(smem + 256);
  float* tcm = reinterpret_cast<float*>(smem + 256 + align_up(size_t(h.coeff_count) * sizeof(C), 1024));
  C* tiles = reinterpret_cast<C*>(reinterpret_cast<unsigned char*>(tcm) + size_t(h.tc_count) * kTcMatBytes);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT);
    }
    mbar_init(mma_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "n"(kTcCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int e = tid; e < h.coeff_count; e += kTcThreads) pool[e] = args.coeff[e];
  {
    const float4* src = reinterpret_cast<const float4*>(h.tc_mats);
    float4* dst = reinterpret_cast<float4*>(tcm);
    for (int i = tid; i < h.tc_count * (kTcMatBytes / 16); i += kTcThreads) dst[i] = src[i];
  }
  fence_proxy_async_smem();  // B operands written by the generic proxy, read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  const long long n_tiles = h.n_tiles;
  const long long mine = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (tid >= NT) {
    // ------------------------------------------------ producer: TMA loads
    const int lane = tid - NT;
    if (h.tma_rank > 0) {
      if (lane != 0) return;
      const int ne = h.n_enum;
      const int sub = T - ne;
      int s = 0;
      uint32_t ph = 0;
      for (long long it = 0; it < mine; ++it) {
        if (it >= S) mbar_wait_bounded(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], uint32_t(sizeof(C)) << T);
        const long long tb = tile_base((long long)blockIdx.x + it * gridDim.x, h);
        C* buf = tiles + (size_t(s) << T);
        for (int e = 0; e < (1 << ne); ++e) {
          long long origin = tb;
          for (int j = 0; j < ne; ++j)
            if ((e >> j) & 1) origin += 1LL << h.high[h.m - ne + j];
          const long long w = origin << h.word_shift;
          int c[5];
#pragma unroll
          for (int d = 0; d < 5; ++d)
            c[d] = (d < h.tma_rank && h.tma_box[d] == 0) ? int((w >> h.tma_start[d]) & ((1LL << h.tma_bits[d]) - 1)) : 0;
          tma_load(buf + (size_t(e) << sub), &args.tmap, c, h.tma_rank, &full[s]);
        }
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
      return;
    }
    const int n_chunks = 1 << h.m;
    const uint32_t chunk_bytes = uint32_t(sizeof(C)) << h.L;
    const uint64_t pol = policy_evict_first();
    for (long long it = 0; it < mine; ++it) {
      const int s = int(it % S);
      if (it >= S) mbar_wait_bounded(&empty[s], uint32_t(((it - S) / S) & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[s], chunk_bytes * uint32_t(n_chunks));
      __syncwarp();
      const long long base = tile_base((long long)blockIdx.x + it * gridDim.x, h);
      C* buf = tiles + (size_t(s) << T);
      for (int c = lane; c < n_chunks; c += 32)
        bulk_load(buf + (size_t(c) << h.L), amps + base + chunk_offset(c, h), chunk_bytes, &full[s], pol);
    }
    return;
  }

  // ---------------------------------------------------------- compute warps
  const int np = h.n_phases;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  const uint32_t a_t = tbase + lane_off;           // A re_hi [0,32) im_hi [32,64) re_lo [64,96) im_lo [96,128)
  const uint32_t d_t = tbase + lane_off + 128;     // D re [128,160) im [160,192)
  uint32_t mma_parity = 0;
  GlobalAddr<RB> lin_g;  // linear layout x = rho * 128 + tid
  lin_g.gthr = global_of(tid, h);
#pragma unroll
  for (int i = 0; i < RB; ++i) lin_g.goff[i] = 1LL << gpos(7 + i, h);
  GlobalAddr<RB> last_g;
  {
    const PhaseDesc& lp = args.phases[np - 1];
    const PhaseAddr<C, RB> la(lp, tid);
    last_g.gthr = global_of(la.base, h);
#pragma unroll
    for (int i = 0; i < RB; ++i) last_g.goff[i] = 1LL << gpos(lp.map[i], h);
  }

  int s = 0;
  uint32_t parity = 0;
  for (long long it = 0; it < mine; ++it, (++s == S ? (s = 0, parity ^= 1) : 0)) {
    const long long tile = (long long)blockIdx.x + it * gridDim.x;
    C* buf = tiles + (size_t(s) << T);
    const long long origin = tile_base(tile, h);
    mbar_wait_bounded(&full[s], parity);
    C v[NR];
    for (int p = 0; p < np; ++p) {
      const PhaseDesc& ph = args.phases[p];
      const PhaseAddr<C, RB> a(ph, tid);
      const bool last = p == np - 1;
      const bool tout = last && (ph.flags & PH_TRANSPOSE_OUT);
      if (p == 0) {
        if (ph.flags & PH_TRANSPOSE_IN) {
#pragma unroll
          for (int r = 0; r < NR; ++r) v[r] = buf[r * NT + tid];
          tc_bar();
#pragma unroll
          for (int r = 0; r < NR; ++r) buf[Swz<C>::f(r * NT + tid)] = v[r];
          tc_bar();
#pragma unroll
          for (int r = 0; r < NR; ++r) v[r] = buf[a.swz(r)];
        } else {
#pragma unroll
          for (int r = 0; r < NR; ++r) v[r] = buf[a.lin(r)];
          if (np > 1 || tout) tc_bar();
        }
      } else {
        tc_bar();
#pragma unroll
        for (int r = 0; r < NR; ++r) v[r] = buf[a.swz(r)];
      }
      if (last && !tout) mbar_arrive(&empty[s]);
      for (int o = ph.op_begin; o < ph.op_mid; ++o) reg_apply<C, RB>(v, args.ops[o], pool, args.ops[o].kind == OP_DIAG ? diag_base(args.ops[o], tid, origin) : 0);
      if (ph.tc >= 0) {
        // ---- fused phase matrix on the tensor cores
        {
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            hi[j] = f2tf32(v[j].x);
            lo[j] = f2tf32(v[j].x - __uint_as_float(hi[j]));
          }
          tmem_st32(a_t + 0, hi);
          tmem_st32(a_t + 64, lo);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            hi[j] = f2tf32(v[j].y);
            lo[j] = f2tf32(v[j].y - __uint_as_float(hi[j]));
          }
          tmem_st32(a_t + 32, hi);
          tmem_st32(a_t + 96, lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        tc_bar();
        if (tid == 0) {
          tc_fence_after();
          const uint32_t B = smem_addr(tcm) + uint32_t(ph.tc) * kTcMatBytes;  // Ur_hi Ui_hi Ur_lo Ui_lo
          const uint32_t dre = tbase + 128, dim = tbase + 160;
#pragma unroll
          for (int term = 0; term < 3; ++term) {
            const uint32_t aoff = term == 1 ? 64u : 0u;
            const uint32_t bur = B + (term == 2 ? 8192u : 0u), bui = bur + 4096u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t dur = umma_desc(bur + 256u * k, 128, 1024), dui = umma_desc(bui + 256u * k, 128, 1024);
              const uint32_t are = tbase + aoff + 8u * k, aim = tbase + aoff + 32u + 8u * k;
              const uint32_t first = (term == 0 && k == 0) ? 0u : 1u;
              tc_mma(dre, are, dur, kTcIdesc, first);
              tc_mma(dre, aim, dui, kTcIdescNegB, 1u);
              tc_mma(dim, are, dui, kTcIdesc, first);
              tc_mma(dim, aim, dur, kTcIdesc, 1u);
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_addr(mma_bar))
                       : "memory");
        }
        mbar_wait_bounded(mma_bar, mma_parity);
        mma_parity ^= 1;
        tc_fence_after();
        {
          uint32_t d[32];
          tmem_ld32(d_t + 0, d);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j].x = __uint_as_float(d[j]);
          tmem_ld32(d_t + 32, d);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j].y = __uint_as_float(d[j]);
        }
        tc_fence_before();
      }
      for (int o = ph.op_mid; o < ph.op_end; ++o) reg_apply<C, RB>(v, args.ops[o], pool, args.ops[o].kind == OP_DIAG ? diag_base(args.ops[o], tid, origin) : 0);
      if (!last) {
#pragma unroll
        for (int r = 0; r < NR; ++r) buf[a.swz(r)] = v[r];
      } else if (!tout) {
        C* __restrict__ dst = amps + tile_base(tile, h) + last_g.gthr;
#pragma unroll
        for (int r = 0; r < NR; ++r) dst[last_g.at(r) - last_g.gthr] = v[r];
      } else {
#pragma unroll
        for (int r = 0; r < NR; ++r) buf[a.swz(r)] = v[r];
        tc_bar();
        C* __restrict__ dst = amps + tile_base(tile, h);
#pragma unroll
        for (int r = 0; r < NR; ++r) dst[lin_g.at(r)] = buf[Swz<C>::f(r * NT + tid)];
        mbar_arrive(&empty[s]);
      }
    }
  }
  tc_fence_before();
  tc_bar();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTcCols) : "memory");
  }
}

}  // namespace svb
