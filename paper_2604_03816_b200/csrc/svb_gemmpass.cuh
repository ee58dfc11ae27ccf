// k_gemm_pass -- c64 tile pass whose every dense op runs on the tcgen05 tensor
// cores with BOTH operands in shared memory (the production path for c64
// passes that carry two or more dense gates).
//
// A pass is  load -> ops_0 -> GEMM_1 -> ops_1 -> ... -> GEMM_P -> ops_P -> store
// over 12-qubit tiles (4096 amplitudes, 32 KB).  GEMM_p multiplies the tile,
// viewed as 128 rows x 32 complex columns (the phase's five register qubits
// are the columns), by the fused 32x32 phase matrix U_p in its real 64x64
// block form; ops_p are element-wise diagonal tables (planner: diagonal gates
// that commute past the GEMM).  Unlike the k_reg_pass tensor-core phases,
// nothing is transposed through registers and shared memory twice:
//
//   * the tile lands (TMA) in the stream's 32 KB buffer; each thread reads 32
//     amplitudes, scales them by a power of two chosen from the tile 2-norm
//     (all ops of the pass are unitary, so |amp| * S < 2^15 for the whole
//     pass and the values stay scaled until the store), splits them into fp16
//     hi + lo and writes them back IN PLACE as the A operand of GEMM_1:
//     A_hi | A_lo, 128 rows x 128 B each, K-major SWIZZLE_128B -- the layout
//     the tensor core reads directly through a shared-memory descriptor;
//   * one elected thread issues the 12 tcgen05.mma.kind::f16 (M 128, N 64,
//     K 16: Ah Bh + Al Bh + Ah Bl) into the stream's 64 TMEM columns and
//     commits to an mbarrier;
//   * each thread reads its D row back (tcgen05.ld: 32 complex = the row),
//     applies ops_p in registers and -- the transpose to the next phase's
//     column qubits -- writes hi/lo straight into A of GEMM_{p+1}
//     (one XOR per amplitude: the swizzled word address is GF(2)-linear in
//     the tile index);
//   * after the last GEMM the buffer is free, so the stream's next tile load
//     is issued at once and overlaps the store of this one; the store undoes
//     the scale and restores the tile 2-norm (fp32 tensor-core accumulation
//     truncates: ~1e-6 norm per GEMM).
//
// Four tile streams (warp groups of 128 threads, one buffer each) per CTA,
// one CTA per SM: one stream's conversions overlap another's GEMM.  The
// planner (build_gemm_pass) orders each phase's register and row qubits so
// the writes land conflict-free in the shared-memory banks and the final
// stores are coalesced.
#pragma once
#include "svb_regpass.cuh"

namespace svb {

constexpr int kGemmT = 12;            // tile qubits
constexpr int kGemmTileBytes = 32768;  // 4096 x float2
constexpr int kGemmAWords = 4096;      // A_hi words (f16x2); A_lo follows

// lowest set bit of a loop index 1..31: the Gray code of i differs from that
// of i - 1 in this bit.  Plain selects, so that after unrolling the index of
// every register-array access folds to a constant (a dynamic index would put
// the array in local memory)
__host__ __device__ __forceinline__ constexpr int ctz_c(int x) {
  return (x & 1) ? 0 : (x & 2) ? 1 : (x & 4) ? 2 : (x & 8) ? 3 : 4;
}

// Tile-invariant addressing, computed once per CTA (gemm_tables): the
// thread parts and register bases of every layout change of the pass.
struct GemmTables {
  uint32_t wb[kMaxMmaPerPass][128];   // [p][thread] A word of register 0, layout p -> A of GEMM p + 1
  uint32_t wr[kMaxMmaPerPass][8];     // [p][register bit] A word offsets (uniform)
  uint32_t ld[128];                   // [thread] tile index of register 0 in the load layout
  uint32_t ldr[8];                    // load layout: tile index offsets of the register bits
  long long st[128];                  // [thread] shard offset of register 0 in the last layout
  long long str[8];                   // last layout: shard offsets of the register bits
};

struct GemmSmem {
  size_t pool, dthr, dout, red, orig, iss, tabs, mats, tiles, total;
};
// `base` = shared-window address of the dynamic shared memory (the tile
// buffers are placed 16 KB-aligned in that window so that an A word's byte
// address is (buffer | offset): XOR-composable, no add per store)
__host__ __device__ inline GemmSmem gemm_smem_layout(const PassHeader& h, int ng, uint32_t base) {
  GemmSmem l;
  l.pool = 128;  // barriers + TMEM slot
  l.dthr = l.pool + align_up(size_t(h.coeff_count) * sizeof(float2), 128);
  const int nb = h.gemm_bufs > ng ? h.gemm_bufs : ng;  // tile buffers (ring)
  l.dout = l.dthr + align_up(size_t(h.n_ops) * 128, 128);
  l.red = l.dout + align_up(size_t(nb) * 2 * kMaxOps * sizeof(int), 128);
  l.orig = align_up(l.red + size_t(ng) * 16 * sizeof(float), 128);
  l.iss = align_up(l.orig + size_t(nb) * 2 * sizeof(long long), 128);
  l.tabs = align_up(l.iss + size_t(nb) * sizeof(int), 128);
  l.mats = align_up(l.tabs + sizeof(GemmTables), 1024);
  l.tiles = align_up(base + l.mats + size_t(h.tc_count) * kMmaMatBytes, 16384) - base;
  l.total = l.tiles + size_t(nb) * kGemmTileBytes;
  return l;
}

// K-major SWIZZLE_128B shared-memory descriptor (8-row x 128-B atoms, SBO 1 KB)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor: D f32, A/B f16, both K-major, M = 128, N = 64 / 128
constexpr uint32_t kIdescN64 = (1u << 4) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescN128 = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void t5_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t acc,
                                          uint32_t idesc = kIdescN64) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(acc), "r"(idesc)
      : "memory");
}

// The 12 MMAs of one GEMM (Ah Bh, Al Bh, Ah Bl; 4 K-steps each) in one asm
// block from two base descriptors: every other descriptor is a small
// constant added to the base's start-address field (A: +2 per 32-B K-step,
// +1024 for A_lo 16 KB on; B: +16 per 256-B K-step, +512 for Bl 8 KB on; the
// 14-bit field cannot carry: shared addresses < 256 KB).  Generated code
// otherwise rebuilt and re-broadcast both 64-bit descriptors per MMA (~18
// instructions each, serialised in the issuing thread on the tile's chain).
__device__ __forceinline__ void gemm_issue12(uint32_t d, uint64_t ad, uint64_t bd) {
  asm volatile(
      "{\n .reg .pred pf, pt;\n .reg .b64 a0, a1, a2, a3, l0, l1, l2, l3, b0, b1, b2, b3, c0, c1, c2, c3;\n"
      " setp.ne.b32 pf, %0, %0;\n setp.eq.b32 pt, %0, %0;\n"
      " mov.b64 a0, %1;\n add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      " add.s64 l0, %1, 1024;\n add.s64 l1, %1, 1026;\n add.s64 l2, %1, 1028;\n add.s64 l3, %1, 1030;\n"
      " mov.b64 b0, %2;\n add.s64 b1, %2, 16;\n add.s64 b2, %2, 32;\n add.s64 b3, %2, 48;\n"
      " add.s64 c0, %2, 512;\n add.s64 c1, %2, 528;\n add.s64 c2, %2, 544;\n add.s64 c3, %2, 560;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %3, pf;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], l0, b0, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], l1, b1, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], l2, b2, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], l3, b3, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a0, c0, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a1, c1, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a2, c2, %3, pt;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], a3, c3, %3, pt;\n}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(kIdescN64)
      : "memory");
}

// GEMM-completion wait: plain try_wait polling (no suspend hint: the GEMM takes
// a few hundred cycles, a suspended warp may wake later than that), bounded
// by %globaltimer like mbar_wait_bounded
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity, bool spin) {
  if (!spin) {
    mbar_wait_bounded(bar, parity);
    return;
  }
  const uint32_t a = smem_addr(bar);
  if (mbar_try_wait(a, parity)) return;
  const unsigned long long t0 = global_ns();
  while (!mbar_try_wait(a, parity))
    if (global_ns() - t0 > 4000000000ULL) __trap();
}

// fp16 hi/lo split of a (scaled) complex amplitude, stored as the f16x2 words
// of A_hi and A_lo (re in the low half: K index 2j, im: 2j + 1)
__device__ __forceinline__ void gemm_split_store(uint32_t addr, float xr, float xi) {
  const uint32_t hh = pack_half2(xr, xi);
  const float2 hf = unpack_half2(hh);
  const uint32_t ll = pack_half2(xr - hf.x, xi - hf.y);
  asm volatile("st.shared.b32 [%0], %1;\n st.shared.b32 [%0+16384], %2;" ::"r"(addr), "r"(hh), "r"(ll) : "memory");
}

// tcgen05.ld 16x256b, 8 repetitions: 16 TMEM lanes x 64 columns per warp;
// thread t gets rows t/4 and t/4 + 8, columns 8c + 2 (t % 4) + {0, 1}
__device__ __forceinline__ void t5_ld16x256_x8(uint32_t taddr, uint32_t (&d)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
        "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]),
        "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]),
        "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
      : "r"(taddr)
      : "memory");
}

// One half (register index bit 4 = `half`) of this thread's 32 amplitudes of
// the D tile, in the phase's thread layout:
//  * 32x32b (thread = row m; register index = column j): columns 32 half ..;
//  * 16x256b (PH_LD16): register index = j2 j3 j4 | row bit 3 | row bit 4 =
//    half; lanes = j0 j1 | row bits 0..2 -- two column bits on the lanes,
//    which lets the planner put low tile qubits there (coalesced stores,
//    conflict-free A writes).
template <bool LD16>
__device__ __forceinline__ void gemm_ld_issue(uint32_t dcol, int half, uint32_t (&d)[32]) {
  if constexpr (!LD16)
    t5_ld32(dcol + 32u * half, d);
  else
    t5_ld16x256_x8(dcol + (uint32_t(16 * half) << 16), d);
}

// tcgen05.wait::ld with the loaded registers tied to it, so no consumer can be
// scheduled before the wait
__device__ __forceinline__ void t5_wait_ld_tied(uint32_t (&d)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]), "+r"(d[4]), "+r"(d[5]), "+r"(d[6]), "+r"(d[7]),
                 "+r"(d[8]), "+r"(d[9]), "+r"(d[10]), "+r"(d[11]), "+r"(d[12]), "+r"(d[13]), "+r"(d[14]),
                 "+r"(d[15]), "+r"(d[16]), "+r"(d[17]), "+r"(d[18]), "+r"(d[19]), "+r"(d[20]), "+r"(d[21]),
                 "+r"(d[22]), "+r"(d[23]), "+r"(d[24]), "+r"(d[25]), "+r"(d[26]), "+r"(d[27]), "+r"(d[28]),
                 "+r"(d[29]), "+r"(d[30]), "+r"(d[31])
               :
               : "memory");
}

// Registers of one half in the phase's thread layout:
//  * 32x32b (thread = row m; register index = column j): columns 32 half ..;
//  * 16x256b (PH_LD16): register index = j2 j3 j4 | row bit 3 | row bit 4 =
//    half; lanes = j0 j1 | row bits 0..2 -- two column bits on the lanes,
//    which lets the planner put low tile qubits there (coalesced stores,
//    conflict-free A writes).
template <bool LD16>
__device__ __forceinline__ void gemm_unpack(const uint32_t (&d)[32], float2 (&u)[16]) {
  if constexpr (!LD16) {
#pragma unroll
    for (int q = 0; q < 16; ++q) u[q] = make_float2(__uint_as_float(d[2 * q]), __uint_as_float(d[2 * q + 1]));
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        u[c | hh << 3] = make_float2(__uint_as_float(d[4 * c + 2 * hh]), __uint_as_float(d[4 * c + 2 * hh + 1]));
  }
}

// One half when D is split over two accumulators (N128: columns 0..63 hold
// Ah Bh + Al Bh, columns 64..127 hold Ah Bl): both loads in flight, summed.
template <bool LD16>
__device__ __forceinline__ void gemm_read_half_sum(uint32_t dcol, int half, float2 (&u)[16]) {
  uint32_t d1[32], d2[32];
  gemm_ld_issue<LD16>(dcol, half, d1);
  gemm_ld_issue<LD16>(dcol + 64u, half, d2);
  t5_wait_ld_tied(d1);
  t5_wait_ld_tied(d2);
  float2 v[16];
  gemm_unpack<LD16>(d1, u);
  gemm_unpack<LD16>(d2, v);
#pragma unroll
  for (int q = 0; q < 16; ++q) u[q] = make_float2(u[q].x + v[q].x, u[q].y + v[q].y);
}

// Both halves of this thread's D row: two loads in flight, one wait.
template <bool LD16>
__device__ __forceinline__ void gemm_read_row(uint32_t dcol, float2 (&u0)[16], float2 (&u1)[16]) {
  uint32_t d0[32], d1[32];
  gemm_ld_issue<LD16>(dcol, 0, d0);
  gemm_ld_issue<LD16>(dcol, 1, d1);
  t5_wait_ld_tied(d0);
  t5_wait_ld_tied(d1);
  gemm_unpack<LD16>(d0, u0);
  gemm_unpack<LD16>(d1, u1);
}

// Diagonal op on one half: one table factor per amplitude (table index =
// thread part | register part rmap[rho] | outside-tile part); no hoisted
// factors, so register pressure stays at the 16 amplitudes.
__device__ __forceinline__ void gemm_diag_half(float2 (&u)[16], const OpDesc& op, const float2* __restrict__ table,
                                               int dbase, int half) {
  const unsigned char* rmap = reinterpret_cast<const unsigned char*>(op.tgt);
#pragma unroll
  for (int q = 0; q < 16; ++q) u[q] = cmul(u[q], table[dbase | rmap[q | half << 4]]);
}

// Convert one half into the A operand of the next GEMM: the shared address of
// register rho = wbase ^ XOR of wr[bit] (byte offsets) over rho's bits,
// visited in Gray-code order -- one LOP3 per amplitude.
__device__ __forceinline__ void gemm_write_half(const float2 (&u)[16], uint32_t wbase, const uint32_t* __restrict__ wr,
                                                int half) {
  uint32_t basis[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) basis[i] = wr[i];
  uint32_t w = wbase ^ (half ? wr[4] : 0u);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i) w ^= basis[ctz_c(i)];
    const int r = i ^ (i >> 1);
    gemm_split_store(w, u[r].x, u[r].y);
  }
}

// One tile's GEMM-phase epilogue with a compile-time read-out shape: D ->
// registers -> diagonal ops -> hi/lo A words of the next GEMM.
// The halves a thread owns: both (4 warps per tile stream) or the one its
// warp index selects (8 warps: register bit 4 becomes a warp bit).
template <int NH, bool LD16, bool N128 = false, bool SEQ = false>
__device__ __forceinline__ void gemm_read_owned(uint32_t dcol, int h0, float2 (&u)[NH][16]) {
  if constexpr (SEQ && !N128) {
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      uint32_t d[32];
      gemm_ld_issue<LD16>(dcol, h0 + k, d);
      t5_wait_ld_tied(d);
      gemm_unpack<LD16>(d, u[k]);
    }
  } else if constexpr (N128) {
#pragma unroll
    for (int k = 0; k < NH; ++k) gemm_read_half_sum<LD16>(dcol, h0 + k, u[k]);
  } else if constexpr (NH == 2) {
    gemm_read_row<LD16>(dcol, u[0], u[1]);
  } else {
    uint32_t d[32];
    gemm_ld_issue<LD16>(dcol, h0, d);
    t5_wait_ld_tied(d);
    gemm_unpack<LD16>(d, u[0]);
  }
}

template <int NH, bool LD16, bool N128, bool SEQ = false>
__device__ __forceinline__ void gemm_phase_body(uint32_t dcol, const PassArgs<float2>& args,
                                                const PhaseDesc& ph, const float2* pool, const unsigned char* dthr,
                                                const int* dslot, int gt7, int h0, uint32_t wbase,
                                                const uint32_t* wr) {
  if constexpr (SEQ) {
    // one half in registers at a time (the 5-stream kernel's register budget)
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      const int half = h0 + k;
      float2 u[1][16];
      gemm_read_owned<1, LD16, N128, true>(dcol, half, u);
      for (int o = ph.op_begin; o < ph.op_end; ++o)
        gemm_diag_half(u[0], args.ops[o], pool + args.ops[o].coeff_off,
                       int(dthr[o * 128 + gt7]) | (args.h.has_outside ? dslot[o] : 0), half);
      gemm_write_half(u[0], wbase, wr, half);
    }
  } else {
    float2 u[NH][16];
    gemm_read_owned<NH, LD16, N128>(dcol, h0, u);
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      const int half = h0 + k;
      for (int o = ph.op_begin; o < ph.op_end; ++o)
        gemm_diag_half(u[k], args.ops[o], pool + args.ops[o].coeff_off,
                       int(dthr[o * 128 + gt7]) | (args.h.has_outside ? dslot[o] : 0), half);
      gemm_write_half(u[k], wbase, wr, half);
    }
  }
}

// sum of |amp|^2 with 8 independent FMA chains (one chain would serialise
// 64 dependent FMAs)
template <int N>
__device__ __forceinline__ float norm2_chains(const float2 (&u)[N]) {
  float acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = 0.f;
#pragma unroll
  for (int q = 0; q < N; ++q) acc[q & 7] = fmaf(u[q].x, u[q].x, fmaf(u[q].y, u[q].y, acc[q & 7]));
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

template <int NH, bool LD16, bool N128>
__device__ __forceinline__ float gemm_norm_body(uint32_t dcol, int h0) {
  float2 u[NH][16];
  gemm_read_owned<NH, LD16, N128>(dcol, h0, u);
  float w = 0.f;
#pragma unroll
  for (int k = 0; k < NH; ++k) w += norm2_chains(u[k]);
  return w;
}

// Final store of one tile (last layout): diagonal ops, undo the scale /
// restore the norm (factor f), 16-byte stores when register bit 0 is tile
// bit 0 (`pairs`), else 8-byte.
// OFF: int when every offset of the tile fits 31 bits (n_local <= 31: one
// IADD per store instead of a 64-bit add), else long long.
template <int NH, bool LD16, bool N128, class OFF, bool SEQ = false>
__device__ __forceinline__ float gemm_store_body(float2* __restrict__ dst, uint32_t dcol, const PassArgs<float2>& args,
                                                const PhaseDesc& ph, const float2* pool, const unsigned char* dthr,
                                                const int* dslot, int gt7, int h0, const long long* __restrict__ sr,
                                                float f, bool pairs) {
  float2 uu[SEQ ? 1 : NH][16];
  if constexpr (!SEQ) gemm_read_owned<NH, LD16, N128>(dcol, h0, uu);
  float wsum = 0.f;
#pragma unroll
  for (int k = 0; k < NH; ++k) {
    const int half = h0 + k;
    if constexpr (SEQ) gemm_read_owned<1, LD16, N128, true>(dcol, half, uu);
    float2 (&u)[16] = uu[SEQ ? 0 : k];
    for (int o = ph.op_begin; o < ph.op_end; ++o)
      gemm_diag_half(u, args.ops[o], pool + args.ops[o].coeff_off,
                     int(dthr[o * 128 + gt7]) | (args.h.has_outside ? dslot[o] : 0), half);
    OFF goff[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) goff[i] = OFF(sr[i]);
    OFF o = half ? OFF(sr[4]) : OFF(0);
    if (pairs) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i) {
          const int b = ctz_c(i) + 1;
          o += (((i ^ (i >> 1)) << 1) >> b) & 1 ? goff[b] : -goff[b];
        }
        const int r = (i ^ (i >> 1)) << 1;
        *reinterpret_cast<float4*>(dst + o) = make_float4(u[r].x * f, u[r].y * f, u[r | 1].x * f, u[r | 1].y * f);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i) {
          const int b = ctz_c(i);
          o += ((i ^ (i >> 1)) >> b) & 1 ? goff[b] : -goff[b];
        }
        const int r = i ^ (i >> 1);
        dst[o] = make_float2(u[r].x * f, u[r].y * f);
      }
    }
    wsum += norm2_chains(u);
  }
  return wsum * f * f;  // norm^2 of what was stored (diagonal ops included)
}

// Address tables of the pass (threads 0..127 compute them once per CTA).
__device__ __forceinline__ void gemm_tables(GemmTables& t, const PassArgs<float2>& args, int gt) {
  const PassHeader& h = args.h;
  const int P = h.n_phases - 1;
  for (int p = 0; p < P; ++p) {
    const PhaseDesc& cur = args.phases[p];
    const unsigned short* wt = reinterpret_cast<const unsigned short*>(args.phases[p + 1].R);
    uint32_t w = 0;
    for (int b = 0; b < 7; ++b)
      if ((gt >> b) & 1) w ^= wt[cur.map[5 + b]];
    t.wb[p][gt] = 4 * w;  // byte offsets within A_hi
    if (gt < 5) t.wr[p][gt] = 4u * wt[cur.map[gt]];
  }
  const PhaseDesc& p0 = args.phases[0];
  uint32_t x = 0;
  for (int b = 0; b < 7; ++b) x |= uint32_t((gt >> b) & 1) << p0.map[5 + b];
  t.ld[gt] = x;
  if (gt < 5) t.ldr[gt] = 1u << p0.map[gt];
  const PhaseDesc& pl = args.phases[P];
  long long g = 0;
  for (int b = 0; b < 7; ++b)
    if ((gt >> b) & 1) g += 1LL << gpos(pl.map[5 + b], h);
  t.st[gt] = g;
  if (gt < 5) t.str[gt] = 1LL << gpos(pl.map[gt], h);
}

// NG tile streams of WPG warps: WPG 4 -> a thread holds 32 amplitudes (both
// register halves); WPG 8 -> 16 (register bit 4 is warp bit 2 of the stream),
// twice the warps per scheduler to hide the GEMM / TMEM / barrier latency.
// N128: the hi products run as one N = 128 GEMM, Ah [Bh | Bl], plus Al Bh
// (8 instead of 12 MMAs, 56 instead of 72 KB of operand reads per tile and
// GEMM); 128 TMEM columns per stream, summed at read-out.
template <int NG, int WPG = 4, bool N128 = true>
__global__ void __launch_bounds__(NG * WPG * 32, 1)
    k_gemm_pass(float2* __restrict__ amps, const __grid_constant__ PassArgs<float2> args) {
  constexpr int NTG = WPG * 32;
  constexpr int NH = WPG == 8 ? 1 : 2;  // register halves per thread
  constexpr bool SEQ = NG >= 5;         // 640 threads: one register half in flight
  constexpr int T = kGemmT;
  constexpr uint32_t kColsPerGroup = N128 ? 128 : 64;
  constexpr uint32_t kTmemCols = NG * kColsPerGroup > 256 ? 512 : NG * kColsPerGroup > 128 ? 256 : 128;
  static_assert(NG * kColsPerGroup <= 512, "TMEM columns");
  extern __shared__ __align__(1024) unsigned char smem[];
  const PassHeader& h = args.h;
  const GemmSmem lay = gemm_smem_layout(h, NG, smem_addr(smem));
  const int NB = h.gemm_bufs > NG ? h.gemm_bufs : NG;  // tile buffers: tile t -> buffer t % NB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [buffer] tile landed
  uint64_t* mbar = full + 8;                            // [group] GEMM committed (<= 6)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + NG);
  float2* pool = reinterpret_cast<float2*>(smem + lay.pool);
  unsigned char* dthr = smem + lay.dthr;                 // [op][thread] diagonal index, thread part
  int* dout = reinterpret_cast<int*>(smem + lay.dout);  // [buffer][2][op] outside-tile part
  float* red = reinterpret_cast<float*>(smem + lay.red);  // [group][in 8 | out 8] norm partials
  long long* orig = reinterpret_cast<long long*>(smem + lay.orig);  // [buffer][2] tile origins
  // [buffer] the tile whose load was last issued into it: a stream waits for
  // its tile's load to be issued before it waits on the buffer's mbarrier
  // parity (with a spare buffer a stream can run one use ahead of a buffer)
  volatile int* iss = reinterpret_cast<volatile int*>(smem + lay.iss);
  const uint32_t mats = smem_addr(smem + lay.mats);
  unsigned char* tiles = smem + lay.tiles;
  const int tid = threadIdx.x;
  const int group = tid / NTG, gt = tid % NTG, wig = gt >> 5, lane = tid & 31;
  const int gt7 = gt & 127;                 // the thread's 7 row bits (lane + warp quarter)
  const int h0 = NH == 2 ? 0 : gt >> 7;     // first register half owned
  const int P = h.n_phases - 1;  // GEMM phases

  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      iss[b] = -1;
    }
    for (int g = 0; g < NG; ++g) mbar_init(&mbar[g], 1);
    fence_mbar_init();
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tslot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int e = tid; e < h.coeff_count; e += NG * NTG) pool[e] = pool_elem(args, e);
  {
    const uint4* src = reinterpret_cast<const uint4*>(h.tc_mats);
    uint4* dst = reinterpret_cast<uint4*>(smem + lay.mats);
    for (int e = tid; e < h.tc_count * (kMmaMatBytes / 16); e += NG * NTG) dst[e] = src[e];
  }
  for (int e = tid; e < h.n_ops * 128; e += NG * NTG) {
    const OpDesc& op = args.ops[e / 128];
    dthr[e] = op.kind == OP_DIAG ? (unsigned char)diag_thread_part(op, e % 128) : 0;
  }
  GemmTables& tab = *reinterpret_cast<GemmTables*>(smem + lay.tabs);
  if (tid < 128) gemm_tables(tab, args, tid);
  fence_proxy_async_smem();  // B operands written by the generic proxy, read by the tensor core
  t5_fence_before();
  __syncthreads();
  t5_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t dcol = tbase + uint32_t(group) * kColsPerGroup + (uint32_t((wig & 3) * 32) << 16);  // this warp's D lanes

  const int n_tiles = int(h.n_tiles);
  const int mine = int(blockIdx.x) < n_tiles ? (n_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  if (smem_addr(tiles) & 16383u) __trap();  // host and device disagree on the shared window
  // every shard offset of a tile fits 31 bits (int store offsets)
  const bool small = (h.m == 0 ? h.L : h.high_sorted[h.m - 1] + 1) <= 31;

  // Tile t (this CTA's t-th tile, processed by stream t % NG) lands in buffer
  // t % NB.  With a spare buffer (NB = NG + 1) the load of tile t is issued
  // when tile t - NB leaves its buffer (after its last GEMM), one tile slot
  // ahead of the stream that needs it: the HBM latency hides behind other
  // work.  Issued by warp 0 of the freeing stream (lane 0 issues the TMA, all
  // lanes publish the tile origin and the outside-tile diagonal index parts).
  auto load = [&](int t) {
    const int tile = int(blockIdx.x) + t * int(gridDim.x);
    const int b = t % NB, xs = (t / NB) & 1;
    float2* lbuf = reinterpret_cast<float2*>(tiles + size_t(b) * kGemmTileBytes);
    const long long tb = tile_base(tile, h);
    if (lane == 0) orig[b * 2 + xs] = tb;  // published with the tile (mbarrier release)
    if (h.has_outside) {
      int* slot = dout + (b * 2 + xs) * kMaxOps;
      for (int i = lane; i < h.n_ops; i += 32)
        slot[i] = args.ops[i].kind == OP_DIAG ? diag_outside_part(args.ops[i], tb) : 0;
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_expect_tx(&full[b], uint32_t(kGemmTileBytes));
      iss[b] = t;
      const int ne = h.n_enum;
      const int sub = T - ne;
      for (int e = 0; e < (1 << ne); ++e) {
        long long origin = tb;
        for (int j = 0; j < ne; ++j)
          if ((e >> j) & 1) origin += 1LL << h.high[h.m - ne + j];
        int c[5];
#pragma unroll
        for (int d = 0; d < 5; ++d)
          c[d] = (d < h.tma_rank && h.tma_box[d] == 0) ? int((origin >> h.tma_start[d]) & ((1LL << h.tma_bits[d]) - 1)) : 0;
        tma_load(lbuf + (size_t(e) << sub), &args.tmap, c, h.tma_rank, &full[b]);
      }
    }
    __syncwarp();
  };
  auto sum_red = [&](int off) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < WPG; ++w) s += red[group * 16 + off + w];
    return s;
  };

  // deferred renormalisation: the previous pass's norm drift (see PassHeader)
  float corr = 1.f;
  if (h.normacc && h.pass_index > 0) {
    const double in = h.normacc[2 * h.pass_index - 2], out = h.normacc[2 * h.pass_index - 1];
    if (in > 0.0 && out > 0.0) corr = float(sqrt(in / out));
  }
  double acc_in = 0.0, acc_out = 0.0;  // this thread's norm^2 contributions (true units)
  // Scale factor: when the previous pass of this execution was a GEMM pass,
  // its output norm^2 is the state's norm^2, so one power of two for the whole
  // pass bounds every amplitude (|amp| S < 2^15): no per-tile norm reduction.
  // fp16 hi/lo then carries ~2^-22 of the STATE norm per element (absolute),
  // instead of 2^-22 of each tile's norm.  Otherwise (first pass) the scale
  // comes from each tile's 2-norm.
  float Sg = 0.f;
  if (h.normacc && h.pass_index > 0 && !(h.debug & 512)) {
    const double prev = h.normacc[2 * h.pass_index - 1];
    if (prev > 0.0) {
      const int ebits = (__float_as_int(sqrtf(float(prev))) >> 23) & 0xff;
      Sg = __int_as_float(min(max(268 - ebits, 1), 253) << 23);
      if (blockIdx.x == 0 && tid == 0) acc_in = prev * double(corr) * double(corr);
    }
  }
  // stage timestamps (SVB_GEMM_TRACE): CTA 0, stream 0, thread 0, first 8 tiles x 16 events
  unsigned long long* tr = (h.trace && blockIdx.x == 0 && group == 0 && gt == 0) ? h.trace : nullptr;
  int tev = 0;
  auto mark = [&](int it_) {
    if (tr && it_ < 8 * NG && tev < 16) tr[(it_ / NG) * 16 + tev++] = clock64();
  };
  uint32_t mpar = 0;
  if (h.debug & 48) {  // profiling: stagger the streams' start (debug 16: 300 ns, 32: 600 ns per stream)
    const unsigned long long t0 = global_ns(), d = (h.debug & 16 ? 300ull : 600ull) * group;
    while (global_ns() - t0 < d) {
    }
  }
  if (group == 0 && wig == 0)
    for (int t = 0; t < NB && t < mine; ++t) load(t);
  for (int it = group; it < mine; it += NG) {
    const int bi = it % NB, xs = (it / NB) & 1;
    const uint32_t fpar = uint32_t(xs);
    float2* buf = reinterpret_cast<float2*>(tiles + size_t(bi) * kGemmTileBytes);
    const uint32_t abase = smem_addr(buf);  // 16 KB aligned (gemm_smem_layout)
    const int* dslot = dout + (bi * 2 + xs) * kMaxOps;
    if (NB != NG)
      while (iss[bi] != it) __nanosleep(20);
    tev = 0;
    mark(it);
    if (h.debug & 8)
      mbar_wait_spin(&full[bi], fpar, true);
    else
      mbar_wait(&full[bi], fpar);
    const long long origin = orig[bi * 2 + xs];
    mark(it);  // 1: tile landed

    // ---- phase 0: linear tile -> registers (load layout), tile norm, scale,
    // ops_0, A of GEMM 1 written in place
    float S, n2in;
    {
      float2 v[NH][16];
      const PhaseDesc& p0 = args.phases[0];
#pragma unroll
      for (int k = 0; k < NH; ++k) {
        uint32_t x = tab.ld[gt7] ^ ((h0 + k) ? tab.ldr[4] : 0u);
        if (p0.map[0] == 0) {
          // register bit 0 = tile bit 0: adjacent pairs, 16-byte loads
          uint32_t basis[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) basis[i] = tab.ldr[1 + i];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i) x ^= basis[ctz_c(i)];
            const float4 q = *reinterpret_cast<const float4*>(buf + x);
            const int r = (i ^ (i >> 1)) << 1;
            v[k][r] = make_float2(q.x, q.y);
            v[k][r | 1] = make_float2(q.z, q.w);
          }
        } else {
          uint32_t basis[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) basis[i] = tab.ldr[i];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i) x ^= basis[ctz_c(i)];
            v[k][i ^ (i >> 1)] = buf[x];
          }
        }
      }
      if (Sg > 0.f) {
        group_bar<NG, NTG>(group);  // every read of the linear tile done (A is written in place)
        mark(it);                   // 2: loaded
        S = Sg;
      } else {
        float w = 0.f;
#pragma unroll
        for (int k = 0; k < NH; ++k) w += norm2_chains(v[k]);
#pragma unroll
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0) red[group * 16 + wig] = w;
        group_bar<NG, NTG>(group);  // every read of the linear tile done; partials visible
        mark(it);  // 2: loaded + norm
        n2in = sum_red(0);
        // S = 2^(14 - e), e = exponent of the tile 2-norm: |amp| S < 2^15 for the pass
        const int ebits = (__float_as_int(sqrtf(n2in)) >> 23) & 0xff;
        const int se = min(max(268 - ebits, 1), 253);
        S = n2in > 0.f ? __int_as_float(se << 23) : 1.f;
        if (gt == 0) acc_in += double(n2in) * double(corr) * double(corr);
      }
      const float Sc = S * corr;
      const uint32_t wb0 = tab.wb[0][gt7];
#pragma unroll
      for (int k = 0; k < NH; ++k) {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[k][q] = make_float2(v[k][q].x * Sc, v[k][q].y * Sc);
        for (int o = p0.op_begin; o < p0.op_end; ++o)
          gemm_diag_half(v[k], args.ops[o], pool + args.ops[o].coeff_off,
                         int(dthr[o * 128 + gt7]) | (h.has_outside ? dslot[o] : 0), h0 + k);
        gemm_write_half(v[k], abase | wb0, tab.wr[0], h0 + k);
      }
    }
    fence_proxy_async_smem();
    t5_fence_before();
    group_bar<NG, NTG>(group);
    mark(it);  // 3: A of GEMM 1 written

    for (int p = 1; p <= P; ++p) {
      const PhaseDesc& ph = args.phases[p];
      const bool ld16 = ph.flags & PH_LD16;
      // warp-uniform copies (redux results live in uniform registers): the
      // issuing thread then hands the descriptors to the tensor core without
      // a per-MMA ELECT / R2UR.BROADCAST loop
      const uint32_t abase_u = __reduce_or_sync(0xffffffffu, abase);
      const uint32_t dacc_u = __reduce_or_sync(0xffffffffu, tbase + uint32_t(group) * kColsPerGroup);
      if (gt == 0) {
        t5_fence_after();
        const uint32_t b0 = mats + uint32_t(ph.tc) * kMmaMatBytes;
        const uint32_t dacc = dacc_u;
        if (!(h.debug & 1)) {
          if constexpr (N128) {
            // Ah [Bh | Bl] (N 128: the packed B is exactly the N = 128 K-major
            // matrix [Bh | Bl]), then Al Bh into columns 0..63
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              t5_mma_ss(dacc, sw128_desc(abase + 32u * ks), t5_desc(b0 + 256u * ks, 128, 1024), ks ? 1u : 0u,
                        kIdescN128);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              t5_mma_ss(dacc, sw128_desc(abase + uint32_t(kGemmAWords * 4) + 32u * ks),
                        t5_desc(b0 + 256u * ks, 128, 1024), 1u, kIdescN64);
          } else if (h.debug & 8192) {  // per-MMA descriptors (the previous issue code, for comparison)
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ad = sw128_desc(abase + (t == 1 ? uint32_t(kGemmAWords * 4) : 0u) + 32u * ks);
                const uint64_t bd = t5_desc(b0 + (t == 2 ? 8192u : 0u) + 256u * ks, 128, 1024);
                t5_mma_ss(dacc, ad, bd, (t | ks) ? 1u : 0u);
              }
          } else {
            gemm_issue12(dacc, sw128_desc(abase_u), t5_desc(b0, 128, 1024));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_addr(&mbar[group]))
                     : "memory");
      }
      mbar_wait_spin(&mbar[group], mpar, h.debug & 4);
      mpar ^= 1;
      t5_fence_after();
      mark(it);  // GEMM p done
      if (p < P) {
        const uint32_t wb = abase | tab.wb[p][gt7];
        if (h.debug & 2)
          ;
        else if (ld16)
          gemm_phase_body<NH, true, N128, SEQ>(dcol, args, ph, pool, dthr, dslot, gt7, h0, wb, tab.wr[p]);
        else
          gemm_phase_body<NH, false, N128, SEQ>(dcol, args, ph, pool, dthr, dslot, gt7, h0, wb, tab.wr[p]);
        fence_proxy_async_smem();
        t5_fence_before();
        group_bar<NG, NTG>(group);  // A complete; every D read done before the next GEMM
        mark(it);  // A of GEMM p + 1 written
        continue;
      }
      // ---- last GEMM done: the buffer is free, so this stream's next tile
      // loads while this one is stored
      if (wig == 0 && it + NB < mine) load(it + NB);
      // undo the scale (the drift correction happens in the next pass)
      const float f = 1.f / S;
      float2* __restrict__ dst = amps + origin + tab.st[gt7];
      const bool pairs = ph.map[0] == 0;  // register bit 0 = tile bit 0: 16-byte stores
      float w;
      if (small) {
        if (ld16)
          w = gemm_store_body<NH, true, N128, int, SEQ>(dst, dcol, args, ph, pool, dthr, dslot, gt7, h0, tab.str, f, pairs);
        else
          w = gemm_store_body<NH, false, N128, int, SEQ>(dst, dcol, args, ph, pool, dthr, dslot, gt7, h0, tab.str, f, pairs);
      } else {
        if (ld16)
          w = gemm_store_body<NH, true, N128, long long, SEQ>(dst, dcol, args, ph, pool, dthr, dslot, gt7, h0, tab.str, f,
                                                         pairs);
        else
          w = gemm_store_body<NH, false, N128, long long, SEQ>(dst, dcol, args, ph, pool, dthr, dslot, gt7, h0, tab.str, f,
                                                          pairs);
      }
      acc_out += double(w);
      mark(it);  // stored
      t5_fence_before();
    }
  }
  if (h.normacc) {
#pragma unroll
    for (int o = 16; o; o >>= 1) acc_out += __shfl_xor_sync(0xffffffffu, acc_out, o);
    if (lane == 0) atomicAdd(&h.normacc[2 * h.pass_index + 1], acc_out);
    if (gt == 0) atomicAdd(&h.normacc[2 * h.pass_index], acc_in);
  }
  __syncthreads();
  if (tid < 32) {
    t5_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols) : "memory");
  }
}

}  // namespace svb
