// Native launch planner: lowers a (fused) gate list into tile passes.
//
// Input is the output of the DAG fusion pass (ref pkg/src/aqsim/dag.py:177-217:
// CUSTOM ops on an ascending qubit union, or named gates), one matrix per gate.
// Output is a sequence of passes; each pass is one launch of the tile kernel
// and one HBM round trip of the state.  The reference applies one gate per
// whole-array sweep (ref engines.py:182-185); here every gate whose qubits fit
// the pass's tile qubit set, and that no deferred gate must precede, joins the
// pass (diagonal gates commute with each other and are merged into one table).
#pragma once
#include <complex>
#include <string>
#include <vector>

#include "svb200.h"
#include "svb_types.h"

namespace svb {

using cd = std::complex<double>;

struct Gate {
  int k = 0;
  int t[kMaxK] = {0};
  bool diag = false;
  std::vector<cd> m;  // dense: 2^k x 2^k row-major; diagonal: the 2^k diagonal entries
};

struct KernelOp {
  int kind = OP_DENSE;
  int k = 0;
  int stype = 0;           // dense 1q: DenseStructure (OP_PERM: tgt[0] control, tgt[1] target)
  int tgt[kMaxK] = {0};    // tile-local bits, matrix-local bit j -> tgt[j]; diagonal ops
                           // only: tgt >= T is shard qubit tgt - T outside the tile
                           // (always the top table bits, ascending)
  std::vector<cd> coeff;
  std::vector<int> gates;  // input gates folded into this op, program order
  int ctlq = -1;           // c128 controlled op with its control OUTSIDE the tile:
                           // the control's shard qubit; k = 1 (tgt[0] = target),
                           // coeff = U0 then U1 (2x2 each), chosen per tile
};

// Register-phase encoding of a pass for k_reg_pass (see svb_regpass.cuh).
struct RegPhase {
  int R[8] = {0};           // register bit i <-> tile-local bit R[i] (ascending)
  int op_begin = 0, op_end = 0;
  int flags = 0;
  // tensor-core phases: ops [op_begin, op_mid) run on CUDA cores,
  // then the fused 2^RB x 2^RB matrix tc_mats[tc] as one tcgen05 GEMM, then
  // ops [op_mid, op_end).  tc < 0: no GEMM (op_mid == op_end).
  int op_mid = 0;
  int tc = -1;
  std::vector<int> tc_gates;  // input gates folded into the GEMM, program order
  // thread-local layout (see PhaseDesc::map); filled by build_phases
  int map[16] = {0};
  bool mma = false;           // k_reg_pass mma.sync GEMM phase (whole phase = tc_mats[tc])
  // k_gemm_pass: word address (in the A operand of this phase's GEMM) of each
  // tile bit, see svb_gemmpass.cuh; phase 0 (the load layout) has none
  unsigned short wt[16] = {0};
};
struct RegOp {
  int kind = OP_DENSE;
  int k = 0;
  int stype = 0;           // dense 1q: DenseStructure
  int mask = 0;            // dense: register-bit mask; diagonal: kt (# thread-sourced bits)
  int src[kMaxK] = {0};    // diagonal: thread bit of table bit kr + j; OP_CTRL: src[0] = control thread bit
  unsigned char rmap[32] = {0};  // diagonal: register part of the table index per rho
  int rmask = 0;                  // diagonal: register indices the table reads (its kr bits)
  int kx = 0;                     // diagonal: top kx table bits are shard qubits outside the tile
  unsigned long long xmask = 0;   //   (ascending), selected per tile from the tile origin
  std::vector<cd> coeff;   // dense: matrix permuted to ascending register bits
};

struct Pass {
  int T = 0, L = 0, m = 0;
  int high[kMaxHigh] = {0};
  std::vector<KernelOp> ops;
  double cost = 0.0;
  int num_gates = 0;
  int high_sorted[kMaxHigh] = {0};  // high[] ascending (tile_base insertion order)
  // TMA tensor-map description of the tile (in 8-byte words; c128 adds the
  // re/im bit 0).  Runs of consecutive tile bits are box dims; everything in
  // between is a box-1 dim.  The last n_enum high bits are not in the box and
  // are enumerated with one TMA load each (tile-local bits L+m-n_enum ..).
  int tma_rank = 0;
  int tma_start[5] = {0}, tma_bits[5] = {0}, tma_box[5] = {0};
  int n_enum = 0;
  int reg_bits = 0;               // > 0: executed by k_reg_pass<RB = reg_bits>
  int thread_bits = 8;            // tile bits carried by the thread index (7: warp-group streams)
  bool mma_phases = false;        // k_reg_pass with mma.sync GEMM phases (tc_mats)
  bool renorm = false;            // all ops unitary: the kernel restores each tile's norm
  int streams = 1;                // tile streams per CTA (7 thread bits: 2 or 3)
  // k_gemm_pass (c64): phases[0] = load layout + ops before the first GEMM,
  // phases[f >= 1] = GEMM tc_mats[f - 1] then element-wise diagonal ops
  bool gemm = false;
  int gemm_warps = 4;             // warps per tile stream (4: 32 amplitudes per thread, 8: 16)
  int bank_conflicts = 0;         // sum over A writes of log2(bank-conflict degree)
  std::vector<std::vector<cd>> tc_mats;  // fused phase matrices (2^RB x 2^RB, row-major)
  std::vector<RegPhase> phases;
  std::vector<RegOp> reg_ops;     // same order as ops
};

struct Plan {
  int n = 0;
  int prec = SVB_C128;
  svb_plan_options opt{};
  std::vector<Pass> passes;
};

// Tile defaults per precision: 32 KiB tiles, 512-byte contiguous chunks.
int default_tile_bits(int prec);
int default_min_low_bits(int prec);
int default_reg_bits(int prec);
double default_cost_budget(int prec);

// Parse + classify the raw ABI arrays into gates (diagonal detection).
bool make_gates(int n, int n_ops, const int* op_k, const int* op_targets, const double* op_mats,
                std::vector<Gate>& out, std::string& err);

bool build_plan(int n, int prec, const std::vector<Gate>& gates, const svb_plan_options& opt,
                Plan& out, std::string& err);

}  // namespace svb
