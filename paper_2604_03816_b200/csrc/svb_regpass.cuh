// k_reg_pass -- register-resident tile pass (the production path for tiles of
// T = RB + 8 qubits).
//
// Each of the 256 compute threads holds 2^RB amplitudes of the tile in
// registers.  A pass is a sequence of *phases*; phase p fixes which RB tile
// bits are register bits (R_p) -- the other 8 tile bits are the thread index.
// Every dense op of the phase targets only register bits and runs as fully
// unrolled FMAs on registers (no address math, no shared-memory traffic);
// diagonal ops run on any bits.  Between phases the tile is transposed
// through shared memory in an XOR-swizzled layout (conflict-free for almost
// every R).  Data arrive by 1-D TMA bulk copies (producer warp, ring of
// `stages` buffers); the last phase writes its registers straight to HBM
// (coalesced when the register bits avoid the 3-4 lowest qubits), so a buffer
// is released to the producer as soon as the last phase has read it.
#pragma once
#include "svb_kernels.cuh"

namespace svb {

template <class C>
struct Swz;
template <>
struct Swz<float2> {  // 16 x 8 B per 128-B bank row
  static __device__ __forceinline__ int f(int i) { return i ^ (((i >> 4) ^ (i >> 8) ^ (i >> 12)) & 15); }
};
template <>
struct Swz<double2> {  // 8 x 16 B per 128-B bank row
  static __device__ __forceinline__ int f(int i) { return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7); }
};

template <int RB>
__host__ __device__ constexpr int deposit_mask(int x, int mask) {
  int r = 0, b = 0;
  for (int i = 0; i < RB; ++i)
    if ((mask >> i) & 1) {
      if ((x >> b) & 1) r |= 1 << i;
      ++b;
    }
  return r;
}
__host__ __device__ constexpr int popc_c(int m) { return m ? (m & 1) + popc_c(m >> 1) : 0; }

// Dense op on register bits MASK (matrix-local bit j <-> j-th lowest set bit).
template <class C, int RB, int MASK, bool HOIST = true>
__device__ __forceinline__ void reg_dense(C (&v)[1 << RB], const C* __restrict__ Ms) {
  constexpr int K = popc_c(MASK);
  constexpr int D = 1 << K;
  constexpr int REST = ((1 << RB) - 1) & ~MASK;
  // matrices up to 2q (c64 and c128) are hoisted into registers (measured:
  // per-use shared-memory broadcasts cost 12% on layered c128 at 3 streams);
  // wider ones, and every one in the 4-stream c128 kernel (128 registers),
  // are read per use (shared-memory broadcasts)
  constexpr bool kHoist = HOIST && D <= 4;
  C M[kHoist ? D * D : 1];
  if constexpr (kHoist) {
#pragma unroll
    for (int e = 0; e < D * D; ++e) M[e] = Ms[e];
  }
#pragma unroll
  for (int g = 0; g < (1 << (RB - K)); ++g) {
    const int base = deposit_mask<RB>(g, REST);
    // input-stationary order: each input feeds all D accumulators in turn
    // (operand reuse, D independent FMA chains instead of one serial chain)
    C in[D], acc[D];
#pragma unroll
    for (int j = 0; j < D; ++j) in[j] = v[base | deposit_mask<RB>(j, MASK)];
#pragma unroll
    for (int i = 0; i < D; ++i) acc[i] = czero<C>();
#pragma unroll
    for (int j = 0; j < D; ++j) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        if constexpr (kHoist) acc[i] = cfma(M[i * D + j], in[j], acc[i]);
        else acc[i] = cfma(Ms[i * D + j], in[j], acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) v[base | deposit_mask<RB>(i, MASK)] = acc[i];
  }
}

// Diagonal op.  The planner orders the table index as [thread-sourced bits |
// register-sourced bits | shard bits outside the tile]: rmap packs, per
// register index rho, the register part of the table index (one byte per
// rho, already shifted); the thread part depends only on the thread and the
// outside part only on the tile, so both are precomputed (dbase) -- see
// diag_base and k_reg_pass.  Thread bits lowest: lanes that differ in them
// read adjacent entries, so the lookups are bank-conflict free.
__device__ __forceinline__ int diag_thread_part(const OpDesc& op, int tid) {
  int dt = 0;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j)
    if (j < op.pad) dt |= ((tid >> op.srt[j]) & 1) << j;
  return dt;
}
__device__ __forceinline__ int diag_outside_part(const OpDesc& op, long long origin) {
  return op.kx ? pext_bits(origin, op.xmask) << (op.k - op.kx) : 0;
}
__device__ __forceinline__ int diag_base(const OpDesc& op, int tid, long long origin) {
  return diag_thread_part(op, tid) | diag_outside_part(op, origin);
}

// The table depends on the register index only through the bits in MASK: a
// thread loads its 2^|MASK| factors once (table index = dbase | r << kt, r the
// compact register part) and multiplies them in -- one shared-memory load per
// distinct factor instead of one per amplitude.
template <int RB, int MASK>
__host__ __device__ constexpr int pext_c(int x) {
  int r = 0, b = 0;
  for (int i = 0; i < RB; ++i)
    if ((MASK >> i) & 1) r |= ((x >> i) & 1) << b++;
  return r;
}
template <class C, int RB, int MASK>
__device__ __forceinline__ void reg_diag_mask(C (&v)[1 << RB], const C* __restrict__ table, int dbase, int kt) {
  constexpr int K = popc_c(MASK);
  C f[1 << K];
#pragma unroll
  for (int r = 0; r < (1 << K); ++r) f[r] = table[dbase | (r << kt)];
#pragma unroll
  for (int rho = 0; rho < (1 << RB); ++rho) v[rho] = cmul(v[rho], f[pext_c<RB, MASK>(rho)]);
}

template <class C, int RB>
__device__ __forceinline__ void reg_diag(C (&v)[1 << RB], const OpDesc& op, const C* __restrict__ table, int dbase) {
  switch (op.rmask) {
#define SVB_DCASE(m) \
  case m:            \
    if constexpr ((m) < (1 << RB)) reg_diag_mask<C, RB, (m)>(v, table, dbase, op.pad); \
    return;
    SVB_DCASE(0) SVB_DCASE(1) SVB_DCASE(2) SVB_DCASE(3) SVB_DCASE(4) SVB_DCASE(5) SVB_DCASE(6) SVB_DCASE(7)
    SVB_DCASE(8) SVB_DCASE(9) SVB_DCASE(10) SVB_DCASE(11) SVB_DCASE(12) SVB_DCASE(13) SVB_DCASE(14)
    SVB_DCASE(15) SVB_DCASE(16) SVB_DCASE(17) SVB_DCASE(18) SVB_DCASE(19) SVB_DCASE(20) SVB_DCASE(21)
    SVB_DCASE(22) SVB_DCASE(23) SVB_DCASE(24) SVB_DCASE(25) SVB_DCASE(26) SVB_DCASE(27) SVB_DCASE(28)
    SVB_DCASE(29) SVB_DCASE(30) SVB_DCASE(31)
#undef SVB_DCASE
    default: break;
  }
}

// Sparse 2-qubit ops (OpDesc.kx = pattern, set at launch from the exact zeros
// of the 4x4 matrix in register-local order, index = b0 + 2 b1): every row
// has 2 non-zero columns c1(i), c2(i) (controlled-U forms, CNOT-permuted
// controlled forms) or 1 (CNOT permutation with phases).  Width-2 fusion of
// CNOT layers leaves ~60 % of the fused 2q gates of a layered circuit in one
// of these forms, and QFT's fused H . CP gates are controlled-U: half (or a
// quarter) of the FP64 FMAs of a dense 4x4.
//   1: rows keep b0, mix b1      c = {i & 1, (i & 1) | 2}
//   2: rows keep b1, mix b0      c = {i & 2, (i & 2) | 1}
//   3: rows 0,1 <- {0,3}, rows 2,3 <- {1,2}
//   4: rows 0,2 <- {0,3}, rows 1,3 <- {1,2}
//   5: monomial, 1 <-> 3          c = {0, 3, 2, 1}
//   6: monomial, 2 <-> 3          c = {0, 1, 3, 2}
__host__ __device__ constexpr int sp_c1(int pat, int i) {
  return pat == 1 ? (i & 1) : pat == 2 ? (i & 2) : pat == 3 ? (i < 2 ? 0 : 1) : pat == 4 ? ((i & 1) ? 1 : 0)
       : pat == 5 ? ((i & 1) ? (i ^ 2) : i) : ((i & 2) ? (i ^ 1) : i);
}
__host__ __device__ constexpr int sp_c2(int pat, int i) {
  return pat == 1 ? ((i & 1) | 2) : pat == 2 ? ((i & 2) | 1) : pat == 3 ? (i < 2 ? 3 : 2)
       : pat == 4 ? ((i & 1) ? 2 : 3) : -1;
}
template <class C, int RB, int MASK, int PAT, bool HOIST>
__device__ __forceinline__ void reg_sparse2(C (&v)[1 << RB], const C* __restrict__ Ms) {
  constexpr int REST = ((1 << RB) - 1) & ~MASK;
  constexpr bool two = PAT <= 4;
  C M1[4], M2[two ? 4 : 1];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    M1[i] = Ms[i * 4 + sp_c1(PAT, i)];
    if constexpr (two) M2[i] = Ms[i * 4 + sp_c2(PAT, i)];
  }
#pragma unroll
  for (int g = 0; g < (1 << (RB - 2)); ++g) {
    const int base = deposit_mask<RB>(g, REST);
    C in[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) in[j] = v[base | deposit_mask<RB>(j, MASK)];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      C acc = cfma(M1[i], in[sp_c1(PAT, i)], czero<C>());
      if constexpr (two) acc = cfma(M2[i], in[sp_c2(PAT, i)], acc);
      v[base | deposit_mask<RB>(i, MASK)] = acc;
    }
  }
}
// SP: sparse patterns compiled in (0 none, 1 controlled-U forms 1-2, 2 all).
// Every variant is unrolled code for each register mask, and the size of the
// op dispatch matters (measured, qft-30 / layered-30 c128 ms: none 121 / 330,
// SP 1 106 / 325, SP 2 111 / 314 -- both without 3-qubit dense ops): the
// launch picks SP 2 only for passes holding patterns 3-6.
template <class C, int RB, int MASK, bool HOIST, int SP>
__device__ __forceinline__ void reg_dense2(C (&v)[1 << RB], const C* __restrict__ co, int pat) {
  if constexpr (SP >= 1) {
    if (pat == 1) return reg_sparse2<C, RB, MASK, 1, HOIST>(v, co);
    if (pat == 2) return reg_sparse2<C, RB, MASK, 2, HOIST>(v, co);
  }
  if constexpr (SP >= 2) {
    if (pat == 3) return reg_sparse2<C, RB, MASK, 3, HOIST>(v, co);
    if (pat == 4) return reg_sparse2<C, RB, MASK, 4, HOIST>(v, co);
    if (pat == 5) return reg_sparse2<C, RB, MASK, 5, HOIST>(v, co);
    if (pat == 6) return reg_sparse2<C, RB, MASK, 6, HOIST>(v, co);
  }
  reg_dense<C, RB, MASK, HOIST>(v, co);
}

// D3: 3-qubit dense ops compiled in (the c128 stream kernels leave them to
// the 8-thread-bit kernel: less code in the op dispatch)
// OP_CTRL ops (U0 / U1 on one register bit by the control thread bit srt[0])
// share the 1-qubit dense code: only the coefficient pointer differs.
template <class C, int RB, bool HOIST = true, int SP = 0, bool D3 = true>
__device__ __forceinline__ void reg_dense_op(C (&v)[1 << RB], const OpDesc& op, const C* pool, int gt = 0,
                                             long long origin = 0) {
  const C* co = pool + op.coeff_off +
                (op.kind == OP_CTRL
                     ? 4 * (op.srt[0] >= 0 ? (gt >> op.srt[0]) & 1 : int((origin >> op.tgt[0]) & 1))
                     : 0);
  switch (op.pad) {  // register-bit mask of the dense op
#define SVB_CASE(m) \
  case m:           \
    if constexpr ((m) < (1 << RB) && popc_c(m) == 2) reg_dense2<C, RB, (m), HOIST, SP>(v, co, op.kx); \
    else if constexpr ((m) < (1 << RB) && popc_c(m) <= (D3 ? 3 : 2)) reg_dense<C, RB, (m), HOIST>(v, co); \
    break;
    SVB_CASE(1) SVB_CASE(2) SVB_CASE(3) SVB_CASE(4) SVB_CASE(5) SVB_CASE(6) SVB_CASE(7)
    SVB_CASE(8) SVB_CASE(9) SVB_CASE(10) SVB_CASE(11) SVB_CASE(12) SVB_CASE(13) SVB_CASE(14)
    SVB_CASE(16) SVB_CASE(17) SVB_CASE(18) SVB_CASE(19) SVB_CASE(20) SVB_CASE(21) SVB_CASE(22)
    SVB_CASE(24) SVB_CASE(25) SVB_CASE(26) SVB_CASE(28)
#undef SVB_CASE
    default: break;
  }
}

template <class C, int RB>
__device__ __forceinline__ void reg_apply(C (&v)[1 << RB], const OpDesc& op, const C* pool, int dbase) {
  if (op.kind == OP_DIAG)
    reg_diag<C, RB>(v, op, pool + op.coeff_off, dbase);
  else
    reg_dense_op<C, RB>(v, op, pool);
}

// ------------------------------------------------ tensor-core GEMM phase
// v <- U v for the 32 complex columns of each row, on mma.sync m16n8k16
// (fp16 x fp16 -> fp32).  Layout (planner fuse_mma_phases): register index
// rho = m | q0 << 3 | q1 << 4 holds complex column i = c + 4 m (c = lane & 3)
// of warp row g + 8 q0 + 16 q1 (g = lane >> 2), i.e. exactly the A fragment of
// the real block form [re im] and, for the outputs, the D fragment.  Each row
// is scaled by a power of two s so that its largest component lies in
// [2^14, 2^15), split x s = h + l in fp16 (round to nearest), and
// D = h Bh + l Bh + h Bl accumulates in fp32 (relative error ~2^-22 of the
// row's largest amplitude; Bh + Bl = the fp32 matrix to ~2^-22).
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float2 unpack_half2(uint32_t x) {
  float2 f;
  asm("{\n .reg .f16 l, h;\n mov.b32 {l, h}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, h;\n}"
      : "=f"(f.x), "=f"(f.y)
      : "r"(x));
  return f;
}

// The tensor cores' fp32 accumulation shrinks magnitudes systematically
// (~1e-6 per phase measured); passes of unitary ops restore the tile's
// 2-norm at the end (PassHeader::renorm, see k_reg_pass).
__device__ __forceinline__ void mma_phase(float2 (&v)[32], const uint4* __restrict__ B, int lane) {
  // per-row power-of-two scales (rows q = q0 | q1 << 1)
  float sc[4], inv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float mx = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float2 x = v[m | (q & 1) << 3 | (q >> 1) << 4];
      mx = fmaxf(mx, fmaxf(fabsf(x.x), fabsf(x.y)));
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const int e = (__float_as_int(mx) >> 23) & 0xff;
    const int se = min(max(268 - e, 1), 253);  // 2^(14 - exponent(mx)), clamped
    sc[q] = __int_as_float(se << 23);
    inv[q] = __int_as_float((254 - se) << 23);  // exact inverse
  }
  // A fragments [q1][kk][reg]: reg r -> m = 2 kk + (r >> 1), q0 = r & 1
  uint32_t ah[2][4][4], al[2][4][4];
#pragma unroll
  for (int q1 = 0; q1 < 2; ++q1)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int q0 = r & 1, m = 2 * kk + (r >> 1);
        const float s = sc[q0 | q1 << 1];
        const float2 x = v[m | q0 << 3 | q1 << 4];
        const float xr = x.x * s, xi = x.y * s;
        const uint32_t hh = pack_half2(xr, xi);
        const float2 hf = unpack_half2(hh);
        ah[q1][kk][r] = hh;
        al[q1][kk][r] = pack_half2(xr - hf.x, xi - hf.y);
      }
  // D = A B over 8 column tiles (nt = output m), two at a time
#pragma unroll
  for (int np = 0; np < 4; ++np) {
    float d[2][2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q1 = 0; q1 < 2; ++q1)
#pragma unroll
        for (int t = 0; t < 4; ++t) d[a][q1][t] = 0.f;
    // issue order: the 4 accumulators round-robin, so dependent HMMAs are 4
    // instructions apart (hides the tensor-pipe latency at 2 warps/scheduler)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint4 b[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) b[a] = B[((2 * np + a) * 4 + kk) * 32 + lane];
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int q1 = 0; q1 < 2; ++q1) {
            const uint32_t* A = t == 1 ? al[q1][kk] : ah[q1][kk];
            const uint32_t b0 = t == 2 ? b[a].z : b[a].x, b1 = t == 2 ? b[a].w : b[a].y;
            mma_f16(d[a][q1], A[0], A[1], A[2], A[3], b0, b1);
          }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q1 = 0; q1 < 2; ++q1) {
        const int m = 2 * np + a;
        v[m | q1 << 4] = make_float2(d[a][q1][0] * inv[q1 << 1], d[a][q1][1] * inv[q1 << 1]);
        v[m | 1 << 3 | q1 << 4] = make_float2(d[a][q1][2] * inv[1 | q1 << 1], d[a][q1][3] * inv[1 | q1 << 1]);
      }
  }
}

// 2-norm^2 of a thread's amplitudes, summed over its warp (in FP32).
template <int NR>
__device__ __forceinline__ float warp_norm2(const float2 (&v)[NR]) {
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < NR; ++r) s = fmaf(v[r].x, v[r].x, fmaf(v[r].y, v[r].y, s));
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// TB = thread bits of a tile: 8 -- the 8 compute warps share one tile stream;
// 7 -- two groups of 4 warps, each with its own tile stream (tiles alternate
// between the groups) and its own named barrier, so one group's shared-memory
// transposes and conversions overlap the other's tensor-core work.
// Named barrier of one tile stream (ids 1..NG; NTHR threads each).
template <int G, int NTHR>
__device__ __forceinline__ void group_bar(int group) {
  if constexpr (G == 1) {
    asm volatile("bar.sync 1, %0;" ::"n"(NTHR) : "memory");
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "n"(NTHR) : "memory");
  }
}

// ------------------------------------- tcgen05 GEMM phase (two-stream tiles)
// With 7 thread bits each warp group owns a 128-row tile; its 128 threads
// hold one row each (32 complex amplitudes = the phase's register bits in
// matrix order).  The phase D = A B runs on the 5th-generation tensor cores:
// A (the rows, fp16 hi/lo split after per-row power-of-two scaling) is
// written to TMEM with tcgen05.st, B (the real block form of the fused
// 32x32 phase matrix, fp16 hi/lo, K-major core matrices) sits in shared
// memory, ONE thread issues the 12 tcgen05.mma.kind::f16 (M 128, N 64, K 16;
// terms h Bh + l Bh + h Bl) and commits to an mbarrier, and the rows come
// back with tcgen05.ld.  Unlike warp-level mma.sync (which holds the
// scheduler's issue slot ~8.5 cycles per HMMA on B200, tools/probes/
// mma_overlap_probe.cu), the GEMM costs the issuing warps nothing, and the
// other group's conversions and transposes overlap it.
__device__ __forceinline__ void t5_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void t5_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void t5_ld32(uint32_t taddr, uint32_t (&d)[32]) {
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

__device__ __forceinline__ void t5_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void t5_ld16(uint32_t taddr, uint32_t (&d)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
        "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
      : "r"(taddr)
      : "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_NONE, sm100 version bit
__device__ __forceinline__ uint64_t t5_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor: D f32, A/B f16, both K-major, N = 64, M = 128
constexpr uint32_t kT5Idesc = (1u << 4) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void t5_mma(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(acc), "r"(kT5Idesc)
      : "memory");
}

// Bounded wait (a fault in the async pipeline must not hang the GPU): traps
// after 4 s of wall time (%globaltimer), far above any legitimate wait.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  if (mbar_try_wait_suspend(a, parity)) return;
  const unsigned long long t0 = global_ns();
  while (!mbar_try_wait_suspend(a, parity))
    if (global_ns() - t0 > 4000000000ULL) __trap();
}

// One tcgen05 GEMM phase of a 128-row group.  tm = the group's TMEM base
// (A hi at +0, A lo at +32, D at +64 columns); lane = this thread's row.
// B: [hi 8 KB | lo 8 KB], offset(n, k) = (n/8) 1024 + (k/8) 128 + (n%8) 16 + (k%8) 2.
template <int NG, int NTG>
__device__ __forceinline__ void tc5_phase(float2 (&v)[32], uint32_t tm, int gt, uint32_t bmat, uint64_t* bar,
                                          uint32_t& par, int group) {
  const uint32_t tl = tm + (uint32_t(gt & ~31) << 16);  // this warp's lane quarter
  float mx = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) mx = fmaxf(mx, fmaxf(fabsf(v[j].x), fabsf(v[j].y)));
  const int e = (__float_as_int(mx) >> 23) & 0xff;
  const int se = min(max(268 - e, 1), 253);  // 2^(14 - exponent(mx)), clamped
  const float sc = __int_as_float(se << 23), inv = __int_as_float((254 - se) << 23);
  // convert and store in chunks of 8 columns (few live registers)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t hv[8], lv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = 8 * c + q;
      const float xr = v[j].x * sc, xi = v[j].y * sc;
      const uint32_t hh = pack_half2(xr, xi);
      const float2 hf = unpack_half2(hh);
      hv[q] = hh;
      lv[q] = pack_half2(xr - hf.x, xi - hf.y);
    }
    t5_st8(tl + 8 * c, hv);
    t5_st8(tl + 32 + 8 * c, lv);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  t5_fence_before();
  group_bar<NG, NTG>(group);
  if (gt == 0) {
    t5_fence_after();
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t a = tm + (t == 1 ? 32u : 0u) + 8u * ks;
        const uint64_t b = t5_desc(bmat + (t == 2 ? 8192u : 0u) + 256u * ks, 128, 1024);
        t5_mma(tm + 64, a, b, (t | ks) ? 1u : 0u);
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
  }
  mbar_wait_bounded(bar, par);
  par ^= 1;
  t5_fence_after();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t d[16];
    t5_ld16(tl + 64 + 16 * c, d);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q)
      v[8 * c + q] = make_float2(__uint_as_float(d[2 * q]) * inv, __uint_as_float(d[2 * q + 1]) * inv);
  }
  t5_fence_before();
}

// Shared-memory layout of k_reg_pass: barriers | coefficient pool | thread
// parts of the diagonal table indices | outside-tile parts (2S ring) | tiles.
struct RegSmem {
  size_t pool, dthr, dout, red, mats, tiles, total;
};
template <class C>
__host__ __device__ inline RegSmem reg_smem_layout(const PassHeader& h) {
  RegSmem l;
  l.pool = 128;
  l.dthr = l.pool + align_up(size_t(h.coeff_count) * sizeof(C), 128);
  l.dout = l.dthr + align_up(size_t(h.n_ops) * (size_t(1) << h.thread_bits), 128);
  l.red = l.dout + align_up(size_t(2 * h.stages) * kMaxOps * sizeof(int), 128);
  // [group][tile parity][start/end][warp] tile norms (renorm, 256 B), then the
  // tcgen05 completion barriers [group] and the TMEM base address
  l.mats = l.red + 640;  // renorm partials (<= 4 groups x 128 B), commit barriers, TMEM base
  l.tiles = l.mats + (h.mma_phases ? size_t(h.tc_count) * kMmaMatBytes : 0);
  l.total = l.tiles + size_t(h.stages) * (sizeof(C) << h.T);
  return l;
}

// Per-thread addressing of one phase.  The tile-local index of register rho
// is base | sum_i bit_i(rho) << R[i] (R ascending; base = tid with zero bits
// inserted at R).  The swizzle is GF(2)-linear, so the swizzled address is
// Swz(base) ^ (XOR of the uniform Swz(1 << R[i]) selected by rho): one LOP3
// per amplitude.
template <class C, int RB>
struct PhaseAddr {
  int base, sbase;
  int off[RB], soff[RB];
  // ph.map: register-index bit i -> tile bit map[i]; thread bit b -> map[RB + b]
  __device__ __forceinline__ PhaseAddr(const PhaseDesc& ph, int tid) {
    int b = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) b |= ((tid >> j) & 1) << ph.map[RB + j];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      off[i] = 1 << ph.map[i];
      soff[i] = Swz<C>::f(off[i]);
    }
    base = b;
    sbase = Swz<C>::f(b);
  }
  __device__ __forceinline__ int lin(int rho) const {
    int x = base;
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if ((rho >> i) & 1) x |= off[i];
    return x;
  }
  __device__ __forceinline__ int swz(int rho) const {
    int x = 0;
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if ((rho >> i) & 1) x ^= soff[i];
    return sbase ^ x;
  }
};

// Tile-local bit p -> global (shard) bit: low bits map to themselves, tile
// bit L+b to high[b].  The map is linear, so a global offset is a per-thread
// part plus a uniform part selected by rho.
__device__ __forceinline__ int gpos(int p, const PassHeader& h) { return p < h.L ? p : h.high[p - h.L]; }

__device__ __forceinline__ long long global_of(int x, const PassHeader& h) {
  long long g = x & ((1 << h.L) - 1);
  for (int b = 0; b < h.m; ++b)
    if ((x >> (h.L + b)) & 1) g += 1LL << h.high[b];
  return g;
}

template <int RB>
struct GlobalAddr {
  long long gthr;
  long long goff[RB];
  __device__ __forceinline__ long long at(int rho) const {
    long long x = gthr;
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if ((rho >> i) & 1) x += goff[i];
    return x;
  }
};

template <int TB, int NGRP>
constexpr int reg_compute_threads() {
  return (NGRP ? NGRP : kComputeThreads >> TB) << TB;
}
// Three tile streams run without a producer warp (each stream loads its own
// tiles, one stage each): 12 warps keep 3 per scheduler, which allows 168
// registers per thread instead of the 128 a 13th warp would impose.
template <int TB, int NGRP>
constexpr bool reg_no_producer() {
  return NGRP >= 3;
}
template <int TB, int NGRP>
constexpr int reg_block_threads() {
  return reg_compute_threads<TB, NGRP>() + (reg_no_producer<TB, NGRP>() ? 0 : 32);
}

// NGRP: tile streams (0 = fill 256 compute threads); 3 streams of 128 threads
// (c64 tcgen05 phases) make a 416-thread CTA.
template <class C, int RB, int TB = 8, int NGRP = 0, int SP = 0>
__global__ void __launch_bounds__(reg_block_threads<TB, NGRP>(), (sizeof(C) == 16 ? RB >= 4 : RB >= 5) ? 1 : 2)
    k_reg_pass(C* __restrict__ amps, const __grid_constant__ PassArgs<C> args) {
  constexpr int T = RB + TB;
  constexpr int NR = 1 << RB;
  constexpr int NTG = 1 << TB;                          // threads per tile stream
  constexpr int NCT = reg_compute_threads<TB, NGRP>();  // compute threads
  constexpr int NG = NCT / NTG;                         // tile streams (warp groups)
  constexpr bool kNP = reg_no_producer<TB, NGRP>();     // streams load their own tiles
  constexpr int NTH = reg_block_threads<TB, NGRP>();    // (+ the producer warp)
  constexpr int WPG = NTG / 32;                         // warps per group
  extern __shared__ __align__(1024) unsigned char smem[];
  const PassHeader& h = args.h;
  const int S = h.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // tile landed (1 arrival + tx bytes)
  uint64_t* empty = full + S;                           // tile buffer drained (NTG arrivals)
  const RegSmem lay = reg_smem_layout<C>(h);
  C* pool = reinterpret_cast<C*>(smem + lay.pool);
  unsigned char* dthr = smem + lay.dthr;  // [op][thread]: thread part of each diagonal table index
  int* dout = reinterpret_cast<int*>(smem + lay.dout);  // [2S][op]: outside-tile part, per tile
  const uint4* mats = reinterpret_cast<const uint4*>(smem + lay.mats);  // mma.sync B fragments
  float* red = reinterpret_cast<float*>(smem + lay.red);
  uint64_t* t5bar = reinterpret_cast<uint64_t*>(smem + lay.red + 512);  // [group] tcgen05 commits
  uint32_t* t5slot = reinterpret_cast<uint32_t*>(smem + lay.red + 512 + 32);
  C* tiles = reinterpret_cast<C*>(smem + lay.tiles);
  const int tid = threadIdx.x;
  constexpr bool kT5 = sizeof(C) == 8 && RB == 5 && TB == 7;  // tcgen05 GEMM phases (NG <= 3)

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NTG);
    }
    if constexpr (kT5) {
      for (int g = 0; g < NG; ++g) mbar_init(&t5bar[g], 1);
    }
    fence_mbar_init();
  }
  if constexpr (kT5) {
    if (h.mma_phases && tid < 32) {  // NG groups x 128 TMEM columns (power of two)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(t5slot)),
                   "n"(NG > 2 ? 512 : 256)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  for (int e = tid; e < h.coeff_count; e += NTH) pool[e] = pool_elem(args, e);
  if (h.mma_phases) {
    const uint4* src = reinterpret_cast<const uint4*>(h.tc_mats);
    uint4* dst = reinterpret_cast<uint4*>(smem + lay.mats);
    for (int e = tid; e < h.tc_count * (kMmaMatBytes / 16); e += NTH) dst[e] = src[e];
  }
  for (int e = tid; e < h.n_ops * NTG; e += NTH) {
    const OpDesc& op = args.ops[e / NTG];
    dthr[e] = op.kind == OP_DIAG ? (unsigned char)diag_thread_part(op, e % NTG) : 0;
  }
  if constexpr (kT5) {
    fence_proxy_async_smem();  // B operands written by the generic proxy, read by the tensor core
    t5_fence_before();
  }
  __syncthreads();
  uint32_t t5base = 0, t5par = 0;
  if constexpr (kT5) {
    t5_fence_after();
    t5base = *t5slot;
  }
  // outside-tile table bits of tile `it` (written by the producer before it
  // arms the stage's barrier; a 2S ring so a slot outlives its buffer).  The
  // whole producer warp computes it, one op per lane.
  auto publish_outside = [&](int xs, long long tile, int lane) {
    const long long o = tile_base(tile, h);
    int* slot = dout + xs * kMaxOps;
    for (int i = lane; i < h.n_ops; i += 32)
      slot[i] = args.ops[i].kind == OP_DIAG ? diag_outside_part(args.ops[i], o) : 0;
    __syncwarp();
  };

  // tile counts fit 32 bits (a shard of <= 2^34 amplitudes in >= 2^11-amplitude
  // tiles; the host checks): 32-bit loop state keeps registers free
  const int n_tiles = int(h.n_tiles);
  const int mine = int(blockIdx.x) < n_tiles ? (n_tiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  // one stream's tile load (kNP: issued by warp 0 of the stream; lane 0 arms the
  // barrier and issues the TMA, all lanes publish the outside-tile parts)
  auto stream_load = [&](int it, int st, int lane) {
    const int tile = int(blockIdx.x) + it * int(gridDim.x);
    if (h.has_outside) publish_outside(int(it % (2 * S)), tile, lane);
    C* buf = tiles + (size_t(st) << T);
    const long long tb = tile_base(tile, h);
    if (h.tma_rank > 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[st], uint32_t(sizeof(C)) << T);
        const int ne = h.n_enum;
        const int sub = T - ne;
        for (int e = 0; e < (1 << ne); ++e) {
          long long origin = tb;
          for (int j = 0; j < ne; ++j)
            if ((e >> j) & 1) origin += 1LL << h.high[h.m - ne + j];
          const long long w = origin << h.word_shift;
          int c[5];
#pragma unroll
          for (int d = 0; d < 5; ++d)
            c[d] = (d < h.tma_rank && h.tma_box[d] == 0) ? int((w >> h.tma_start[d]) & ((1LL << h.tma_bits[d]) - 1)) : 0;
          tma_load(buf + (size_t(e) << sub), &args.tmap, c, h.tma_rank, &full[st]);
        }
      }
    } else {
      const int n_chunks = 1 << h.m;
      const uint32_t chunk_bytes = uint32_t(sizeof(C)) << h.L;
      if (lane == 0) mbar_arrive_expect_tx(&full[st], chunk_bytes * uint32_t(n_chunks));
      __syncwarp();
      const uint64_t pol = policy_evict_first();
      for (int c = lane; c < n_chunks; c += 32)
        bulk_load(buf + (size_t(c) << h.L), amps + tb + chunk_offset(c, h), chunk_bytes, &full[st], pol);
    }
    __syncwarp();
  };
  if constexpr (kNP) {
    (void)stream_load;
  }

  if (!kNP && tid >= NCT) {
    // ------------------------------------------------ producer: TMA loads only
    const int lane = tid - NCT;
    if (h.tma_rank > 0) {
      // one tensor-map load per (enumerated) sub-box: a single UTMALDG per tile
      // whenever the tile's qubit runs fit a rank-5 tensor map
      if (lane != 0 && !h.has_outside) return;
      const int ne = h.n_enum;
      const int sub = T - ne;
      int s = 0, xs = 0;
      uint32_t ph = 0;  // parity of the use of buffer s
      for (long long it = 0; it < mine; ++it, xs = xs + 1 == 2 * S ? 0 : xs + 1) {
        if (it >= S) mbar_wait_sleep(&empty[s], ph ^ 1);
        if (h.has_outside) publish_outside(xs, (long long)blockIdx.x + it * gridDim.x, lane);
        if (lane == 0) mbar_arrive_expect_tx(&full[s], uint32_t(sizeof(C)) << T);
        const long long tb = tile_base((long long)blockIdx.x + it * gridDim.x, h);
        C* buf = tiles + (size_t(s) << T);
        for (int e = 0; e < (lane == 0 ? 1 << ne : 0); ++e) {
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
      if (it >= S) mbar_wait_sleep(&empty[s], uint32_t(((it - S) / S) & 1));
      __syncwarp();
      if (h.has_outside) publish_outside(int(it % (2 * S)), (long long)blockIdx.x + it * gridDim.x, lane);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], chunk_bytes * uint32_t(n_chunks));
      __syncwarp();
      const long long base = tile_base((long long)blockIdx.x + it * gridDim.x, h);
      C* buf = tiles + (size_t(s) << T);
      for (int c = lane; c < n_chunks; c += 32)
        bulk_load(buf + (size_t(c) << h.L), amps + base + chunk_offset(c, h), chunk_bytes, &full[s], pol);
    }
    return;
  }

  // -------------------------------------------------------- compute threads
  const int group = NG == 1 ? 0 : tid / NTG;
  const int gt = tid & (NTG - 1);  // thread index within the tile stream
  const int np = h.n_phases;
  // global addressing of the stores (tile-invariant) is rebuilt at the store
  // from the pass description: keeping 2 x RB 64-bit offsets live across the
  // tile loop would cost ~24 registers the tensor-core phases need
  // stage / barrier parity / outside-index slot / renorm slot of tile `it`,
  // advanced incrementally (S is a multiple of NG)
  int s = group, xs = group, tpar = 0;
  uint32_t parity = 0;
  // kNP: each stream owns the stages group, group + NG, ... (S / NG of them):
  // its first S / NG tiles load at once, and each consumed stage is refilled
  // with the tile S / NG iterations ahead (latency hidden behind that many
  // tiles of work)
  const int ahead = S;  // tiles (of this CTA) between a tile and its stage's next one
  if constexpr (kNP) {
    if ((gt >> 5) == 0)
      for (int t = group; t < S && t < mine; t += NG) stream_load(t, t, gt & 31);
  }
  for (int it = group; it < mine; it += NG) {
    const int tile = int(blockIdx.x) + it * int(gridDim.x);
    C* buf = tiles + (size_t(s) << T);
    const long long origin = tile_base(tile, h);
    float* rp = red + (group * 2 + tpar) * 16;  // renorm partials of this tile
    mbar_wait(&full[s], parity);
    C v[NR];
    for (int p = 0; p < np; ++p) {
      const PhaseDesc& ph = args.phases[p];
      const PhaseAddr<C, RB> a(ph, gt);
      const bool last = p == np - 1;
      const bool tout = last && (ph.flags & PH_TRANSPOSE_OUT);
      if (p == 0) {
        if (ph.flags & PH_TRANSPOSE_IN) {
          // linear (TMA) layout -> swizzled layout through conflict-free reads
#pragma unroll
          for (int r = 0; r < NR; ++r) v[r] = buf[r * NTG + gt];
          group_bar<NG, NTG>(group);
#pragma unroll
          for (int r = 0; r < NR; ++r) buf[Swz<C>::f(r * NTG + gt)] = v[r];
          group_bar<NG, NTG>(group);
#pragma unroll
          for (int r = 0; r < NR; ++r) v[r] = buf[a.swz(r)];
        } else {
#pragma unroll
          for (int r = 0; r < NR; ++r) v[r] = buf[a.lin(r)];
          // all reads of the linear layout finish before swizzled writes
          if (np > 1 || tout) group_bar<NG, NTG>(group);
        }
      } else {
        group_bar<NG, NTG>(group);
#pragma unroll
        for (int r = 0; r < NR; ++r) v[r] = buf[a.swz(r)];
      }
      if (last && !tout) {
        mbar_arrive(&empty[s]);  // buffer free for the next load
        if constexpr (kNP) {
          // warp 0 of the stream refills the stage with the stream's next tile
          // as soon as every thread has read it (overlaps this last phase)
          if ((gt >> 5) == 0 && it + ahead < mine) {
            mbar_wait(&empty[s], parity);
            stream_load(it + ahead, s, gt & 31);
          }
        }
      }
      if constexpr (sizeof(C) == 8 && RB == 5) {
        if (p == 0 && h.renorm) {
          const float w = warp_norm2(v);
          if ((gt & 31) == 0) rp[gt >> 5] = w;
        }
        if (ph.flags & PH_MMA) {
          if constexpr (kT5)
            tc5_phase<NG, NTG>(v, t5base + uint32_t(group) * 128u, gt,
                           smem_addr(mats) + uint32_t(ph.tc) * kMmaMatBytes, &t5bar[group], t5par, group);
          else
            mma_phase(v, mats + size_t(ph.tc) * (kMmaMatBytes / 16), tid & 31);
        }
      }
      for (int o = ph.op_begin; o < ph.op_end; ++o) {
        const OpDesc& op = args.ops[o];
        if (op.kind == OP_DIAG)
          reg_diag<C, RB>(v, op, pool + op.coeff_off,
                          int(dthr[o * NTG + gt]) | (h.has_outside ? dout[xs * kMaxOps + o] : 0));
        else
          reg_dense_op<C, RB, !(sizeof(C) == 16 && NGRP >= 4), SP, !(sizeof(C) == 16 && TB == 7)>(v, op, pool, gt,
                                                                                                 origin);
      }
      if constexpr (sizeof(C) == 8 && RB == 5) {
        if (last && h.renorm) {
          // restore the tile's 2-norm (all ops of the pass are unitary)
          const float w = warp_norm2(v);
          if ((gt & 31) == 0) rp[8 + (gt >> 5)] = w;
          group_bar<NG, NTG>(group);
          float n0 = 0.f, n1 = 0.f;
#pragma unroll
          for (int i = 0; i < WPG; ++i) {
            n0 += rp[i];
            n1 += rp[8 + i];
          }
          const float f = n1 > 0.f ? sqrtf(n0 / n1) : 1.f;
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            v[r].x *= f;
            v[r].y *= f;
          }
        }
      }
      if (!last) {
#pragma unroll
        for (int r = 0; r < NR; ++r) buf[a.swz(r)] = v[r];
      } else if (!tout) {
        // direct store from registers (coalesced: the lanes cover the bank-row bits)
        GlobalAddr<RB> last_g;
        last_g.gthr = global_of(a.base, h);
#pragma unroll
        for (int i = 0; i < RB; ++i) last_g.goff[i] = 1LL << gpos(ph.map[i], h);
        C* __restrict__ dst = amps + origin + last_g.gthr;
#pragma unroll
        for (int r = 0; r < NR; ++r) dst[last_g.at(r) - last_g.gthr] = v[r];
      } else {
        // swizzled smem, then contiguous reads -> coalesced global stores
#pragma unroll
        for (int r = 0; r < NR; ++r) buf[a.swz(r)] = v[r];
        group_bar<NG, NTG>(group);
        // per-thread global offset of the linear layout x = rho * NTG + gt
        GlobalAddr<RB> lin_g;
        lin_g.gthr = global_of(gt, h);
#pragma unroll
        for (int i = 0; i < RB; ++i) lin_g.goff[i] = 1LL << gpos(TB + i, h);
        C* __restrict__ dst = amps + origin;
#pragma unroll
        for (int r = 0; r < NR; ++r) dst[lin_g.at(r)] = buf[Swz<C>::f(r * NTG + gt)];
        mbar_arrive(&empty[s]);
        if constexpr (kNP) {
          if ((gt >> 5) == 0 && it + ahead < mine) {
            mbar_wait(&empty[s], parity);
            stream_load(it + ahead, s, gt & 31);
          }
        }
      }
    }
    s += NG;
    if (s >= S) {
      s -= S;
      parity ^= 1;
    }
    xs += NG;
    if (xs >= 2 * S) xs -= 2 * S;
    tpar ^= 1;
  }
  if constexpr (kT5) {
    if (h.mma_phases) {  // every group done with TMEM before warp 0 frees it
      asm volatile("bar.sync 7, %0;" ::"n"(NCT) : "memory");
      if (tid < 32) {
        t5_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t5base), "n"(NG > 2 ? 512 : 256)
                     : "memory");
      }
    }
  }
}

}  // namespace svb
