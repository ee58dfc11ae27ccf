// Shared host/device layout of one tile pass (kernel parameter block).
//
// A *pass* streams the whole local state once.  The state is cut into tiles
// of 2^T amplitudes: tile bits 0..L-1 are the L lowest physical qubits (a
// contiguous chunk of 2^L amplitudes), tile bits L..L+m-1 are the physical
// qubits high[0..m-1] (so a tile is 2^m chunks at strides 2^high[b]).  Every
// kernel op of the pass acts only on tile bits, so one HBM read + write of
// each amplitude applies all of them.  The whole description travels as a
// __grid_constant__ kernel parameter (< 32 KB), so a plan needs no device
// memory and is trivially CUDA-graph capturable.
#pragma once
#include <stdint.h>

namespace svb {

constexpr int kMaxOps = 48;        // kernel ops per pass
constexpr int kMaxHigh = 8;        // high (strided) tile bits
constexpr int kMaxK = 8;           // targets per kernel op
constexpr int kMaxDenseK = 6;      // dense ops up to 64x64
constexpr int kMaxDiagK = 8;       // merged diagonal tables up to 256 entries
constexpr int kCoeffBytes = 24576; // coefficient pool per pass carried in the kernel parameters
// Coefficient pool per pass the planner may fill (bytes): c64 passes keep the
// parameter-block pool (k_gemm_pass shared memory is full with four 32 KB tile
// streams and the GEMM matrices); c128 passes may grow it, the part past
// kCoeffBytes living in global memory (PassArgs::coeff_ext) and copied into
// shared memory with the rest at kernel start.  Diagonal tables of QFT-like
// circuits fill it: qft-30 c128 10 -> 5 passes.
constexpr int kPoolBytesC64 = kCoeffBytes;
constexpr int kPoolBytesC128 = 65536;
constexpr int kComputeWarps = 8;
constexpr int kComputeThreads = kComputeWarps * 32;
constexpr int kThreads = kComputeThreads + 32;   // + one TMA producer warp

// OP_PERM: a CNOT on tile bits (tgt[0] control, tgt[1] target): pairs of
// amplitudes swapped, no arithmetic (the opt-in c128 factorisation of fused
// gates; executed by the shared-memory kernel)
enum OpKind : int { OP_DENSE = 0, OP_DIAG = 1, OP_PERM = 2, OP_CTRL = 3 };
// OP_CTRL (register phases only): a 2-qubit gate that is block-diagonal in one
// qubit, applied as U0 / U1 on the target register bit (pad = its mask),
// selected by the control, which is a THREAD bit (srt[0]) -- the control
// need not be a register bit of the phase.  coeff: U0 then U1, 2x2 each.
// structure of a 1-qubit dense op's columns (planner bookkeeping of the
// factorisation): ST_GENERAL, or each column purely real / purely imaginary
enum DenseStructure : int { ST_GENERAL = 0, ST_RR = 1, ST_RI = 2, ST_IR = 3, ST_II = 4 };

struct OpDesc {
  int kind;           // OpKind
  int k;              // number of targets
  int coeff_off;      // element offset into the coefficient pool
  int pad;
  int tgt[kMaxK];     // tile-local bit acted on by matrix-local bit j
  int srt[kMaxK];     // tgt sorted ascending (zero-bit insertion order)
  // Diagonal ops only: the top kx table-index bits are shard qubits OUTSIDE
  // the tile (ascending, mask xmask).  They are constant over a tile, so a
  // diagonal gate never needs its qubits in the tile: its factor for those
  // bits is selected per tile from the tile origin.
  int kx;             // diagonal: outside-tile bits
  int rmask;          // diagonal (register phases): register indices read by the table
  unsigned long long xmask;
};

// Register-resident execution (k_reg_pass): a pass is a list of phases; in
// phase p the register bits are R[0..RB) and ops [op_begin, op_end) act on
// them (dense: OpDesc.pad = register-bit mask; diagonal: OpDesc.pad = kt,
// OpDesc.srt[0..kt) = thread bits, OpDesc.tgt viewed as 32 bytes = the
// register part of the table index for each rho).
constexpr int kMaxPhases = 32;
enum PhaseFlags : int { PH_TRANSPOSE_IN = 1, PH_TRANSPOSE_OUT = 2, PH_MMA = 4,
                        PH_LD16 = 8 /* k_gemm_pass: D read out with tcgen05.ld 16x256b */ };

struct PhaseDesc {
  int op_begin, op_end, flags, tc;  // tc >= 0: tensor-core GEMM tc between [op_begin,op_mid) and [op_mid,op_end)
  int op_mid, pad0, pad1, pad2;
  int R[8];
  // thread-local layout of the phase: map[i] = tile bit of register-index bit
  // i (i < RB), map[RB + b] = tile bit of thread-index bit b.  Register-FMA
  // phases: R ascending, then the other tile bits ascending.  mma.sync phases
  // (PH_MMA) use the m16n8k16 fragment layout, see svb_regpass.cuh.
  unsigned char map[16];
};

// k_reg_pass mma.sync phases (c64, RB 5): the fused 32x32 complex phase
// matrix as the real 64x64 block form B[k][n] (k = 2i + re/im of the input,
// n = 2j + re/im of the output), split B = Bh + Bl in fp16 and stored in
// m16n8k16 B-fragment order: [nt 0..7][kk 0..3][lane 0..31] x {bh0, bh1, bl0, bl1}.
constexpr int kMmaMatBytes = 8 * 4 * 32 * 16;
constexpr int kMaxMmaPerPass = 5;  // 5 x 16 KB + 4 tile streams x 32 KB fit 227 KB
constexpr int kGemmTileBits = 12;  // k_gemm_pass tiles: 4096 amplitudes (32 KB c64)

struct PassHeader {
  int T, L, m, n_ops;
  int high[kMaxHigh];
  int coeff_count;    // elements used in the pool
  int stages;
  long long n_tiles;
  int n_phases;       // 0: k_tile_pass (ops use tile-local targets); >0: k_reg_pass
  int reg_bits;       // RB of k_reg_pass
  int high_sorted[kMaxHigh];
  int tma_rank;       // 0: 1-D bulk copies per chunk; 1..5: one tensor load per enumerated sub-box
  int n_enum;         // high bits L+m-n_enum.. are enumerated (2^n_enum tensor loads per tile)
  int tma_start[5];   // word-bit start of each tensor dim (gap dims take coords from the origin)
  int tma_bits[5];
  int tma_box[5];     // log2 box extent (0 = box 1)
  int word_shift;     // 0 for c64 (one 8-B word per amplitude), 1 for c128
  // tile index -> shard offset of the tile origin: the tile index bits fill
  // the non-tile bits in runs: origin = sum ((tile >> src) & (2^len-1)) << dst
  int n_gap_runs;
  int gap_src[kMaxHigh + 1], gap_dst[kMaxHigh + 1], gap_len[kMaxHigh + 1];
  int tc_count;                 // fused GEMM matrices of this pass (k_gemm_pass, or
                                // k_reg_pass tensor-core phases when mma_phases)
  int has_outside;              // some diagonal op reads shard bits outside the tile
  const float* tc_mats;         // device: tc_count * kMmaMatBytes (set at launch)
  int mma_phases;               // k_reg_pass: tc_mats are mma.sync B fragments
  int renorm;                   // k_reg_pass (c64 RB 5): every op is unitary -- restore
                                // each tile's 2-norm at the end of the pass
  int thread_bits;              // k_reg_pass: 8 (one tile stream) or 7 (warp groups of 128)
  int streams;                  // k_reg_pass with 7 thread bits: 2 or 3 tile streams
  int gemm;                     // k_gemm_pass (PhaseDesc::R holds the A word table)
  int debug;                    // k_gemm_pass profiling switches (SVB_GEMM_DEBUG): 1 no MMAs,
                                // 2 no intermediate D -> A conversions (wrong results)
  unsigned long long* trace;    // k_gemm_pass stage timestamps of CTA 0 / stream 0 (or null)
  // k_gemm_pass norm bookkeeping (deferred renormalisation): pass k adds its
  // input norm^2 (after its own correction) to normacc[2k] and its output
  // norm^2 to normacc[2k + 1]; pass k + 1 multiplies its input by
  // sqrt(normacc[2k] / normacc[2k + 1]) -- the tensor cores' fp32 truncation
  // loss of pass k (~1e-6 per GEMM) -- folded into its scale factor
  double* normacc;
  int pass_index;
  int gemm_bufs;                // k_gemm_pass tile buffers (ring; >= streams)
};

// opaque 128-byte CUtensorMap (filled at launch time by the host)
struct alignas(64) TensorMapBytes {
  unsigned long long w[16];
};

template <class C>
struct PassArgs {
  TensorMapBytes tmap;
  PassHeader h;
  PhaseDesc phases[kMaxPhases];
  OpDesc ops[kMaxOps];
  C coeff[kCoeffBytes / sizeof(C)];
  // device: pool elements [kCoeffBytes / sizeof(C), coeff_count) (set at
  // launch); last, so the header, phase and op offsets of the parameter
  // block stay as they were
  const C* coeff_ext;
};

#ifdef __CUDACC__
// Pool element e: the parameter block holds the first kCoeffBytes, a c128
// pass's larger pool continues in global memory.
template <class C>
__device__ __forceinline__ C pool_elem(const PassArgs<C>& a, int e) {
  constexpr int kParam = kCoeffBytes / int(sizeof(C));
  if constexpr (kPoolBytesC64 == kCoeffBytes && sizeof(C) == 8) return a.coeff[e];  // c64: parameter block only
  else return e < kParam ? a.coeff[e] : a.coeff_ext[e - kParam];
}
#endif

}  // namespace svb
