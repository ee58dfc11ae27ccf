// Native launch planner (see planner.h).  Host-only C++: runs without a GPU,
// which is what lets the CPU test-suite check plan legality against the oracle.
#include "planner.h"

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>

#include <algorithm>
#include <cmath>
#include <cstring>

namespace svb {

// Measured on B200 (profiles/r01_*): c64 passes are FFMA-issue bound, so the
// widest register tile (13 qubits, 32 amplitudes per thread) wins; c128 uses
// 11-qubit tiles with 8 amplitudes per thread (FP64 register pressure).

// c128: 12-qubit tiles with 16 amplitudes per thread at 1 CTA/SM (measured
// layered-30 450 ms vs 513 ms for 11-qubit tiles x 8 amplitudes at 2 CTAs/SM:
// 4 register bits hold ~3 brickwork gates per phase instead of ~2)
int default_tile_bits(int prec) { return prec == SVB_C64 ? 13 : 12; }
// contiguous low qubits of every tile: 128-B chunks (c64 16 / c128 8
// amplitudes) leave more strided tile qubits to the planner (measured:
// layered-28 c64 19 -> 13 passes, 33.3 -> 29.0 ms; layered-30 c128 21 -> 15,
// 395 -> 378 ms) at no loss of DRAM efficiency
int default_min_low_bits(int prec) { return prec == SVB_C64 ? 4 : 3; }
int default_reg_bits(int prec) { return prec == SVB_C64 ? 5 : 4; }
// c128 passes of layered circuits are FP64-bound whatever their length, so the
// budget only trims trailing short passes there (round 2, A/B on the final
// kernels: layered-33 15 -> 12 passes, 2.65 -> 2.61 s; layered-30, qft-30 and
// the Table-2 workload unchanged); c64 gemm passes lose with a longer budget
// (layered-28 15.0 -> 17.2 ms at 12)
double default_cost_budget(int prec) { return prec == SVB_C64 ? 7.0 : 12.0; }
// tile = RB + 8 qubits for the register kernel

namespace {

// ---------------------------------------------------------------- cost model
// Per-amplitude SM cycles, normalised by the pass's HBM time.  B200: HBM
// ~6.5 TB/s over 148 SMs at ~1.9 GHz = ~23 B/clk/SM; FP32 FMA 128/clk/SM,
// FP64 FMA 64/clk/SM; shared memory 128 B/clk/SM.  A pass is HBM-bound while
// the summed op cost stays below 1.0 (the default budget).
struct CostModel {
  double s, fma, mem;
  explicit CostModel(int prec) {
    s = prec == SVB_C64 ? 8.0 : 16.0;
    fma = prec == SVB_C64 ? 128.0 : 64.0;
    mem = 2.0 * s / 23.0;
  }
  // register-resident ops: FMAs plus, amortised, half a shared-memory
  // transpose per dense op (phases hold ~2 dense ops)
  double dense(int k) const {
    double flops = 4.0 * double(1 << k) / fma;
    double smem = 0.5 * 2.0 * s / 128.0;
    return (flops * 1.2 + smem) / mem;
  }
  double diag(int k) const {
    double flops = 4.0 / fma + (1.0 + k) / 64.0;
    return (flops * 1.2 + s / 128.0) / mem;
  }
  double of(const Gate& g) const { return g.diag ? diag(g.k) : dense(g.k); }
};

bool is_diagonal(int k, const double* mat) {
  const int d = 1 << k;
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c)
      if (r != c && (mat[2 * (r * d + c)] != 0.0 || mat[2 * (r * d + c) + 1] != 0.0)) return false;
  return true;
}

// Extract the bits of `x` at positions pos[0..n) into a compact index.
inline int gather_bits(int x, const int* pos, int n) {
  int r = 0;
  for (int b = 0; b < n; ++b) r |= ((x >> pos[b]) & 1) << b;
  return r;
}

// Running product of diagonal gates over a growing bit set (tile-local bits).
struct DiagAcc {
  std::vector<int> bits;   // sorted tile-local positions
  std::vector<cd> table{cd(1.0, 0.0)};
  std::vector<int> gates;
  bool empty() const { return gates.empty(); }

  int union_size(const int* tg, int k) const {
    std::vector<int> u(bits);
    for (int j = 0; j < k; ++j)
      if (std::find(u.begin(), u.end(), tg[j]) == u.end()) u.push_back(tg[j]);
    return int(u.size());
  }
  void absorb(const int* tg, int k, const std::vector<cd>& d, int gate) {
    std::vector<int> nb(bits);
    for (int j = 0; j < k; ++j)
      if (std::find(nb.begin(), nb.end(), tg[j]) == nb.end()) nb.push_back(tg[j]);
    std::sort(nb.begin(), nb.end());
    // positions of old bits / gate bits inside the new compact index
    std::vector<int> old_pos(bits.size()), g_pos(k);
    for (size_t i = 0; i < bits.size(); ++i)
      old_pos[i] = int(std::find(nb.begin(), nb.end(), bits[i]) - nb.begin());
    for (int j = 0; j < k; ++j) g_pos[j] = int(std::find(nb.begin(), nb.end(), tg[j]) - nb.begin());
    std::vector<cd> nt(size_t(1) << nb.size());
    for (size_t u = 0; u < nt.size(); ++u) {
      int oi = gather_bits(int(u), old_pos.data(), int(old_pos.size()));
      int gi = gather_bits(int(u), g_pos.data(), k);
      nt[u] = table[oi] * d[gi];
    }
    bits.swap(nb);
    table.swap(nt);
    gates.push_back(gate);
  }
  bool touches(const int* tg, int k) const {
    for (int j = 0; j < k; ++j)
      if (std::find(bits.begin(), bits.end(), tg[j]) != bits.end()) return true;
    return false;
  }
  KernelOp take() {
    KernelOp op;
    op.kind = OP_DIAG;
    op.k = int(bits.size());
    for (int j = 0; j < op.k; ++j) op.tgt[j] = bits[j];
    op.coeff = table;
    op.gates = gates;
    *this = DiagAcc();
    return op;
  }
};

size_t coeff_elems(const KernelOp& op) { return op.coeff.size(); }

// ------------------------------------------------- 2q gate factorisation (c128)
// A fused 2-qubit gate from dag.fuse is stored as a dense 4x4 matrix (16 FP64
// FMAs per amplitude in the register kernel, which is FP64-bound for c128).
// Layered circuits fuse (RZ x RZ) CNOT (G x G'), G in {H, RX, RZ}: factor
//   U = D P (A x B),  D diagonal, P in {I, CNOT 0->1, CNOT 1->0},
// normalise the rows of A and B (first non-zero entry real positive; the row
// phases move into D), and apply A, B as 1-qubit ops whose columns are purely
// real or imaginary where possible (4 instead of 8 FMAs per amplitude), P as
// a register permutation and D through the diagonal-run merge.
struct Factor2q {
  int perm = 0;                 // 0: none, 1: CNOT control bit 0 -> target 1, 2: control 1 -> target 0
  std::vector<cd> A, B;         // 2x2 row-major (local bit 0: A, local bit 1: B)
  bool a_id = false, b_id = false;
  int a_st = ST_GENERAL, b_st = ST_GENERAL;
  std::vector<cd> d;            // 4 diagonal entries (local bits 0, 1)
};

int col_structure(const std::vector<cd>& m) {
  auto kind = [&](int c) {  // 1 real, 2 imag, 0 complex (column c of a 2x2)
    bool re = true, im = true;
    for (int r = 0; r < 2; ++r) {
      re = re && std::abs(m[size_t(r) * 2 + c].imag()) <= 1e-15;
      im = im && std::abs(m[size_t(r) * 2 + c].real()) <= 1e-15;
    }
    return re ? 1 : im ? 2 : 0;
  };
  const int c0 = kind(0), c1 = kind(1);
  if (!c0 || !c1) return ST_GENERAL;
  return c0 == 1 ? (c1 == 1 ? ST_RR : ST_RI) : (c1 == 1 ? ST_IR : ST_II);
}

bool factor_2q(const std::vector<cd>& U, Factor2q& f) {
  auto permute = [](int x, int pm) {
    if (pm == 1) return x ^ ((x & 1) << 1);
    if (pm == 2) return x ^ ((x >> 1) & 1);
    return x;
  };
  for (int pm = 0; pm < 3; ++pm) {
    cd W[4][4];
    for (int x = 0; x < 4; ++x)
      for (int y = 0; y < 4; ++y) W[x][y] = U[size_t(permute(x, pm)) * 4 + y];
    // row x = (xa | xb << 1) ~ d'_x (A[xa, :] x B[xb, :]), column y = ya | yb << 1
    cd A[2][2], B[2][2];
    bool ok = true;
    for (int xa = 0; xa < 2 && ok; ++xa) {  // A rows from rows xb = 0, B rows from rows xa = 0
      int ya = 0, yb = 0;
      double best = -1;
      for (int y = 0; y < 4; ++y)
        if (std::abs(W[xa][y]) > best) {
          best = std::abs(W[xa][y]);
          ya = y & 1;
          yb = y >> 1;
        }
      if (best < 1e-12) ok = false;
      for (int j = 0; j < 2; ++j) A[xa][j] = W[xa][j | yb << 1];
      (void)ya;
    }
    for (int xb = 0; xb < 2 && ok; ++xb) {
      int ya = 0;
      double best = -1;
      for (int y = 0; y < 4; ++y)
        if (std::abs(W[xb << 1][y]) > best) {
          best = std::abs(W[xb << 1][y]);
          ya = y & 1;
        }
      if (best < 1e-12) ok = false;
      for (int j = 0; j < 2; ++j) B[xb][j] = W[xb << 1][ya | j << 1];
    }
    if (!ok) continue;
    auto normalise = [](cd (&m)[2][2]) {
      for (int r = 0; r < 2; ++r) {
        int j0 = std::abs(m[r][0]) > 1e-12 ? 0 : 1;
        const cd ph = m[r][j0] / std::abs(m[r][j0]);
        const double nrm = std::sqrt(std::norm(m[r][0]) + std::norm(m[r][1]));
        for (int j = 0; j < 2; ++j) m[r][j] /= ph * nrm;
      }
    };
    normalise(A);
    normalise(B);
    // D' per row from the largest entry, then verify the whole matrix
    cd dp[4];
    double err = 0.0;
    for (int x = 0; x < 4; ++x) {
      const int xa = x & 1, xb = x >> 1;
      int yb_ = 0;
      double best = -1;
      for (int y = 0; y < 4; ++y)
        if (std::abs(W[x][y]) > best) {
          best = std::abs(W[x][y]);
          yb_ = y;
        }
      const cd den = A[xa][yb_ & 1] * B[xb][yb_ >> 1];
      if (std::abs(den) < 1e-12) {
        err = 1.0;
        break;
      }
      dp[x] = W[x][yb_] / den;
      for (int y = 0; y < 4; ++y) err = std::max(err, std::abs(W[x][y] - dp[x] * A[xa][y & 1] * B[xb][y >> 1]));
    }
    if (err > 1e-13) continue;
    f.perm = pm;
    f.A.assign({A[0][0], A[0][1], A[1][0], A[1][1]});
    f.B.assign({B[0][0], B[0][1], B[1][0], B[1][1]});
    auto is_id = [](const std::vector<cd>& m) {
      return std::abs(m[0] - 1.0) <= 1e-15 && std::abs(m[3] - 1.0) <= 1e-15 && std::abs(m[1]) <= 1e-15 &&
             std::abs(m[2]) <= 1e-15;
    };
    f.a_id = is_id(f.A);
    f.b_id = is_id(f.B);
    f.a_st = col_structure(f.A);
    f.b_st = col_structure(f.B);
    // U = D P (A x B): d[perm(x)] = d'_x
    f.d.assign(4, cd());
    for (int x = 0; x < 4; ++x) f.d[permute(x, pm)] = dp[x];
    return true;
  }
  return false;
}

// FP64 FMAs per amplitude of the factored form (diagonal counted as a
// complex multiply; it usually merges with neighbouring diagonal runs)
double factored_cost(const Factor2q& f) {
  auto one = [](bool id, int st) { return id ? 0.0 : st == ST_GENERAL ? 8.0 : 4.0; };
  return one(f.a_id, f.a_st) + one(f.b_id, f.b_st) + 4.0;
}

// Transposes around the first / last phase: the TMA buffer (linear tile
// layout) is read, and the last phase stores to HBM, directly in the phase's
// layout only when the lane bits cover the bank-row index bits (conflict-free
// shared-memory reads, coalesced stores); otherwise through a swizzled
// shared-memory transpose.
void set_layout_flags(RegPhase& rp, int RB, int prec, bool first, bool last) {
  const int low_conflict = prec == SVB_C64 ? 4 : 3;  // bank-row index bits
  int lanes = 0;  // tile bits of the lanes of one shared-memory wavefront
  for (int b = 0; b < low_conflict; ++b) lanes |= 1 << rp.map[RB + b];
  // one missing bank bit costs a 2-way conflict on one read / 64-B store
  // segments, cheaper than a transpose (two extra tile traversals); SVB
  // measured: a single-gate c64 pass touching qubit 3 ran at 63 % of HBM
  // with the transposes
  const int missing = low_conflict - __builtin_popcount(lanes & ((1 << low_conflict) - 1));
  const bool low = missing > 1;
  rp.flags &= ~(PH_TRANSPOSE_IN | PH_TRANSPOSE_OUT);
  if (first && low) rp.flags |= PH_TRANSPOSE_IN;
  if (last && low) rp.flags |= PH_TRANSPOSE_OUT;
}

// Partition a lowered pass into register phases (k_reg_pass).  Phases are
// list-scheduled: each phase scans the remaining ops in order and takes every
// op whose predecessors (earlier ops on a shared bit, diagonal pairs excepted)
// are already scheduled and whose bits fit the phase's RB register bits
// (diagonal ops fit any phase).  Ops are reordered into phase order.
// Returns false when the pass must use the shared-memory kernel instead.
bool build_phases(Pass& p, int RB, int prec, int TB = 8, bool allow_ctrl = false) {
  // instantiated register kernels: c64 RB 3..5, c128 RB 3..4 (8 thread bits);
  // the tensor-core kernel: c64 RB 5 with 7 thread bits
  if (TB == 8 && (RB < 3 || RB > (prec == SVB_C64 ? 5 : 4))) return false;
  // 7 thread bits: k_reg_pass<float2, 5, 7> (tcgen05 phases), k_reg_pass<double2, 4, 7>
  if (TB == 7 && !((RB == 5 && prec == SVB_C64) || (RB == 4 && prec == SVB_C128))) return false;
  if (p.T != RB + TB) return false;
  for (const KernelOp& op : p.ops)
    if (op.kind == OP_DENSE && op.k > std::min(RB, 3)) return false;
  // the c128 stream kernels carry no 3-qubit dense code (op-dispatch size,
  // see reg_dense_op): such passes take the 8-thread-bit kernel
  if (prec == SVB_C128 && TB == 7)
    for (const KernelOp& op : p.ops)
      if (op.kind == OP_DENSE && op.k > 2) return false;
  for (const KernelOp& op : p.ops)
    if (op.kind == OP_DIAG && op.k > kMaxK) return false;
  // factorised c128 ops (CNOT permutations) run on the shared-memory kernel:
  // register-kernel support cost ~10 % on every c128 pass (measured)
  for (const KernelOp& op : p.ops)
    if (op.kind == OP_PERM) return false;
  std::vector<int> pending(p.ops.size());
  for (size_t i = 0; i < p.ops.size(); ++i) pending[i] = int(i);
  std::vector<std::vector<int>> sets, members;
  // Controlled 2q ops (block-diagonal in one qubit, exact zeros): only the
  // target must be a register bit -- the control selects U0 / U1 per thread
  // (OP_CTRL) -- and the control orders like a diagonal touch (a controlled-U
  // commutes with diagonals on its control).  ctl[i] = local index of the
  // control in tgt, or -1.
  std::vector<int> ctl(p.ops.size(), -1);
  if (allow_ctrl)
    for (size_t i = 0; i < p.ops.size(); ++i) {
      const KernelOp& op = p.ops[i];
      if (op.kind != OP_DENSE || op.k != 2 || op.coeff.size() != 16) continue;
      for (int b = 0; b < 2 && ctl[i] < 0; ++b) {
        bool bd = true;
        for (int r = 0; r < 4 && bd; ++r)
          for (int c = 0; c < 4 && bd; ++c)
            if (((r >> b) & 1) != ((c >> b) & 1)) bd = op.coeff[size_t(r) * 4 + c] == cd();
        if (bd && op.tgt[b] < p.T && op.tgt[1 - b] < p.T) ctl[i] = b;
      }
    }
  // bits an op needs in the register set / bits it touches like a dense op /
  // bits it touches like a diagonal (for the ordering blocks)
  auto need_bits = [&](int i) {
    const KernelOp& op = p.ops[i];
    int b = 0;
    if (op.kind == OP_DIAG) return b;
    for (int j = 0; j < op.k; ++j)
      if (op.tgt[j] < p.T && j != ctl[i]) b |= 1 << op.tgt[j];
    return b;
  };
  auto diagish_bits = [&](int i) {
    const KernelOp& op = p.ops[i];
    int b = 0;
    for (int j = 0; j < op.k; ++j)
      if (op.tgt[j] < p.T && (op.kind == OP_DIAG || j == ctl[i])) b |= 1 << op.tgt[j];
    return b;
  };
  // dense ops a phase with register set `mask` (tile bits) would absorb
  auto absorbed = [&](const std::vector<int>& pend, int mask) {
    int dense = 0, all_block = 0, dense_block = 0;
    for (int i : pend) {
      const KernelOp& op = p.ops[i];
      const int nb = need_bits(i), db = diagish_bits(i);
      const bool blocked = ((nb | db) & all_block) || (nb & dense_block);
      const bool take = !blocked && (op.kind == OP_DIAG || (nb & ~mask) == 0);
      if (take) {
        dense += op.kind != OP_DIAG;
      } else {
        all_block |= nb;
        dense_block |= db;
      }
    }
    return dense;
  };
  // One phase from `pend` with register set `fixed` (-1: first fit): the
  // register bits, the ops it absorbs, the ops left.
  struct PhaseStep {
    std::vector<int> R, took, rest;
  };
  auto phase_with = [&](const std::vector<int>& pend, int fixed) {
    PhaseStep ps;
    std::vector<char> block_all(p.T, 0), block_dense(p.T, 0);
    if (fixed >= 0)
      for (int b = 0; b < p.T; ++b)
        if ((fixed >> b) & 1) ps.R.push_back(b);
    for (int i : pend) {
      const KernelOp& op = p.ops[i];
      const int nb = need_bits(i), db = diagish_bits(i);
      bool blocked = false;
      for (int b = 0; b < p.T && !blocked; ++b)
        blocked = (((nb | db) >> b) & 1 && block_all[b]) || ((nb >> b) & 1 && block_dense[b]);
      bool take = false;
      if (!blocked) {
        if (op.kind == OP_DIAG) {
          take = true;
        } else if (fixed >= 0) {
          take = (nb & ~fixed) == 0;
        } else {
          std::vector<int> u = ps.R;
          for (int b = 0; b < p.T; ++b)
            if ((nb >> b) & 1 && std::find(u.begin(), u.end(), b) == u.end()) u.push_back(b);
          if (int(u.size()) <= RB) {
            ps.R.swap(u);
            take = true;
          }
        }
      }
      if (take) {
        ps.took.push_back(i);
      } else {
        ps.rest.push_back(i);
        for (int b = 0; b < p.T; ++b) {
          if ((nb >> b) & 1) block_all[b] = 1;
          if ((db >> b) & 1) block_dense[b] = 1;
        }
      }
    }
    return ps;
  };
  // Candidate register sets for a phase: every RB-subset of the bits the
  // pending dense ops touch, ranked by the dense ops they absorb (fewer phases
  // = fewer transposes / GEMMs); first fit when <= RB bits are in play.
  auto candidates = [&](const std::vector<int>& pend, int keep) {
    std::vector<std::pair<int, int>> got;  // (absorbed, mask)
    int cand = 0;
    for (int i : pend)
      if (p.ops[i].kind != OP_DIAG) cand |= need_bits(i);
    if (__builtin_popcount(cand) > RB && __builtin_popcount(cand) <= 16) {
      std::vector<int> cb;
      for (int b = 0; b < p.T; ++b)
        if ((cand >> b) & 1) cb.push_back(b);
      const int nb = int(cb.size());
      std::vector<int> sel(RB);
      for (int i = 0; i < RB; ++i) sel[i] = i;
      while (true) {  // all RB-subsets of cb, lexicographic
        int mask = 0;
        for (int i = 0; i < RB; ++i) mask |= 1 << cb[sel[i]];
        got.push_back({absorbed(pend, mask), mask});
        int i = RB - 1;
        while (i >= 0 && sel[i] == nb - RB + i) --i;
        if (i < 0) break;
        ++sel[i];
        for (int j = i + 1; j < RB; ++j) sel[j] = sel[j - 1] + 1;
      }
      // most absorbed first; lexicographic order breaks ties (the greedy choice)
      std::stable_sort(got.begin(), got.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
      if (int(got.size()) > keep) got.resize(keep);
    } else {
      got.push_back({0, -1});
    }
    return got;
  };
  // greedy sequence
  {
    std::vector<int> pend = pending;
    while (!pend.empty()) {
      PhaseStep ps = phase_with(pend, candidates(pend, 1)[0].second);
      sets.push_back(ps.R);
      members.push_back(ps.took);
      pend.swap(ps.rest);
    }
  }
  // beam over register-set choices (width 4, 4 candidates per phase), kept
  // when it needs fewer phases -- each phase is a shared-memory transpose
  // (c128) or a GEMM (c64); ~1.5-2 ms per phase at 30 q c128 (measured)
  if (sets.size() >= 3) {
    struct Node {
      std::vector<int> pend;
      std::vector<std::vector<int>> sets, members;
    };
    std::vector<Node> beam(1);
    beam[0].pend = pending;
    while (!beam.empty() && beam[0].sets.size() + 1 < sets.size()) {
      std::vector<Node> next;
      for (const Node& nd : beam)
        for (const auto& c : candidates(nd.pend, 4)) {
          PhaseStep ps = phase_with(nd.pend, c.second);
          if (ps.took.empty()) continue;
          Node ch;
          ch.sets = nd.sets;
          ch.members = nd.members;
          ch.sets.push_back(ps.R);
          ch.members.push_back(ps.took);
          ch.pend.swap(ps.rest);
          next.push_back(std::move(ch));
        }
      auto dense_left = [&](const Node& nd) {
        int d = 0;
        for (int i : nd.pend) d += p.ops[i].kind != OP_DIAG;
        return d;
      };
      std::stable_sort(next.begin(), next.end(), [&](const Node& x, const Node& y) {
        const int dx = dense_left(x), dy = dense_left(y);
        return dx != dy ? dx < dy : x.pend.size() < y.pend.size();
      });
      beam.clear();
      for (Node& ch : next) {
        bool dup = false;
        for (const Node& b : beam) dup = dup || b.pend == ch.pend;
        if (!dup) beam.push_back(std::move(ch));
        if (beam.size() == 4) break;
      }
      const Node* done = nullptr;
      for (const Node& nd : beam)
        if (nd.pend.empty()) done = &nd;
      if (done) {
        if (done->sets.size() < sets.size()) {
          sets = done->sets;
          members = done->members;
        }
        break;
      }
    }
  }
  pending.clear();
  if (int(sets.size()) > kMaxPhases) return false;
  // reorder ops into phase order
  std::vector<KernelOp> ordered;
  std::vector<int> ctl_o;
  std::vector<std::pair<int, int>> ranges;
  for (auto& mem : members) {
    const int b = int(ordered.size());
    for (int i : mem) {
      ordered.push_back(p.ops[i]);
      ctl_o.push_back(ctl[i]);
    }
    ranges.emplace_back(b, int(ordered.size()));
  }
  p.ops.swap(ordered);

  const int low_conflict = prec == SVB_C64 ? 4 : 3;  // bank-row index bits
  p.phases.clear();
  p.reg_ops.assign(p.ops.size(), RegOp());
  for (size_t ph = 0; ph < sets.size(); ++ph) {
    std::vector<int> R = sets[ph];
    // fill free register bits: prefer bits of this phase's diagonal ops (fewer
    // thread-sourced table bits), then the highest tile bits (coalescing)
    for (int i = ranges[ph].first; i < ranges[ph].second && int(R.size()) < RB; ++i) {
      const KernelOp& op = p.ops[i];
      if (op.kind != OP_DIAG) continue;
      for (int j = op.k - 1; j >= 0 && int(R.size()) < RB; --j)
        if (op.tgt[j] >= low_conflict && op.tgt[j] < p.T && std::find(R.begin(), R.end(), op.tgt[j]) == R.end())
          R.push_back(op.tgt[j]);
    }
    for (int b = p.T - 1; b >= 0 && int(R.size()) < RB; --b)
      if (std::find(R.begin(), R.end(), b) == R.end()) R.push_back(b);
    std::sort(R.begin(), R.end());
    RegPhase rp;
    rp.op_mid = ranges[ph].second;
    for (int i = 0; i < RB; ++i) rp.R[i] = R[i];
    rp.op_begin = ranges[ph].first;
    rp.op_end = ranges[ph].second;
    // register-FMA layout: register-index bit i <-> R[i], thread bits <-> the
    // other tile bits ascending -- except that the first low_conflict lanes
    // take tile bits of distinct residues mod low_conflict when the ascending
    // order would not: the shared-memory swizzle XORs tile bits q into bank
    // bit q mod low_conflict, so lanes whose tile bits share a residue hit the
    // same banks (an 8-way conflict for lane bits {0, 3, 6} in c128, measured
    // 19 % extra wavefronts once controlled ops freed the low bits)
    for (int i = 0; i < RB; ++i) rp.map[i] = R[i];
    {
      std::vector<int> th;
      for (int q = 0; q < p.T; ++q)
        if (std::find(R.begin(), R.end(), q) == R.end()) th.push_back(q);
      std::vector<int> lanes, rest;
      int seen = 0;
      for (int q : th) {
        const int r = q % low_conflict;
        if (int(lanes.size()) < low_conflict && !((seen >> r) & 1)) {
          lanes.push_back(q);
          seen |= 1 << r;
        } else {
          rest.push_back(q);
        }
      }
      // (c128 only: the c64 tensor-core phases need the ascending order)
      if (int(lanes.size()) < low_conflict || prec != SVB_C128) {  // plain ascending order
        lanes.clear();
        rest = th;
      }
      int j = 0;
      for (int q : lanes) rp.map[RB + j++] = q;
      for (int q : rest) rp.map[RB + j++] = q;
    }
    set_layout_flags(rp, RB, prec, ph == 0, ph + 1 == sets.size());
    auto reg_of = [&](int t) {
      for (int i = 0; i < RB; ++i)
        if (R[i] == t) return i;
      return -1;
    };
    auto thread_bit_of = [&](int t) {
      for (int j = 0; j < p.T - RB; ++j)
        if (rp.map[RB + j] == t) return j;
      return -1;
    };
    for (int i = rp.op_begin; i < rp.op_end; ++i) {
      const KernelOp& op = p.ops[i];
      RegOp& ro = p.reg_ops[i];
      ro.kind = op.kind;
      ro.k = op.k;
      if (op.kind == OP_DIAG) {
        // new table index = [thread bits asc. | register-sourced bits asc. by register
        //                    | shard bits outside the tile, asc.]: lanes of a warp that
        // differ in thread bits read adjacent table entries (no bank conflicts)
        std::vector<std::pair<int, int>> regb, thrb, extb;  // (register idx / thread bit / qubit, op bit)
        for (int b = 0; b < op.k; ++b) {
          if (op.tgt[b] >= p.T) {
            extb.push_back({op.tgt[b] - p.T, b});
            continue;
          }
          const int r = reg_of(op.tgt[b]);
          if (r >= 0)
            regb.push_back({r, b});
          else
            thrb.push_back({thread_bit_of(op.tgt[b]), b});
        }
        std::sort(regb.begin(), regb.end());
        std::sort(thrb.begin(), thrb.end());
        std::sort(extb.begin(), extb.end());
        const int kr = int(regb.size()), kt = int(thrb.size()), kx = int(extb.size());
        ro.mask = kt;  // stored in OpDesc.pad
        for (int j = 0; j < kt; ++j) ro.src[j] = thrb[j].first;
        ro.rmask = 0;
        for (int j = 0; j < kr; ++j) ro.rmask |= 1 << regb[j].first;
        ro.kx = kx;
        ro.xmask = 0;
        for (int j = 0; j < kx; ++j) ro.xmask |= 1ULL << extb[j].first;
        for (int rho = 0; rho < (1 << RB); ++rho) {
          int d = 0;
          for (int j = 0; j < kr; ++j) d |= ((rho >> regb[j].first) & 1) << (kt + j);
          ro.rmap[rho] = static_cast<unsigned char>(d);
        }
        ro.coeff.assign(op.coeff.size(), cd());
        for (size_t nidx = 0; nidx < op.coeff.size(); ++nidx) {
          int old = 0;
          for (int j = 0; j < kt; ++j) old |= ((int(nidx) >> j) & 1) << thrb[j].second;
          for (int j = 0; j < kr; ++j) old |= ((int(nidx) >> (kt + j)) & 1) << regb[j].second;
          for (int j = 0; j < kx; ++j) old |= ((int(nidx) >> (kr + kt + j)) & 1) << extb[j].second;
          ro.coeff[nidx] = op.coeff[old];
        }
      } else if (op.kind == OP_DENSE && op.ctlq >= 0) {
        // controlled op with its control outside the tile (chosen per tile)
        const int rt = reg_of(op.tgt[0]);
        if (rt < 0) return false;  // cannot happen by construction
        ro.kind = OP_CTRL;
        ro.k = 1;
        ro.mask = 1 << rt;
        ro.src[0] = -1 - op.ctlq;
        ro.coeff = op.coeff;
      } else if (op.kind == OP_DENSE && ctl_o[i] >= 0 && reg_of(op.tgt[ctl_o[i]]) < 0) {
        // controlled op with its control on a thread bit: U0 / U1 on the target
        const int cb = ctl_o[i], tb = 1 - cb;
        const int rt = reg_of(op.tgt[tb]);
        if (rt < 0) return false;  // cannot happen by construction
        ro.kind = OP_CTRL;
        ro.k = 1;
        ro.mask = 1 << rt;
        ro.src[0] = thread_bit_of(op.tgt[cb]);
        ro.coeff.assign(8, cd());
        for (int v = 0; v < 2; ++v)
          for (int x = 0; x < 2; ++x)
            for (int y = 0; y < 2; ++y)
              ro.coeff[size_t(v) * 4 + x * 2 + y] =
                  op.coeff[size_t((v << cb) | (x << tb)) * 4 + ((v << cb) | (y << tb))];
      } else if (op.kind == OP_PERM) {
        const int rc = reg_of(op.tgt[0]), rt = reg_of(op.tgt[1]);
        if (rc < 0 || rt < 0) return false;
        ro.mask = (1 << rc) | (1 << rt);
        ro.src[0] = rc;
        ro.src[1] = rt;
      } else {
        int ri[kMaxK];
        ro.stype = op.stype;
        for (int j = 0; j < op.k; ++j) {
          ri[j] = reg_of(op.tgt[j]);
          if (ri[j] < 0) return false;  // cannot happen by construction
          ro.mask |= 1 << ri[j];
        }
        // new local bit j' <-> j'-th lowest register bit; pos[j] = rank of ri[j]
        int pos[kMaxK];
        for (int j = 0; j < op.k; ++j) {
          pos[j] = 0;
          for (int j2 = 0; j2 < op.k; ++j2) pos[j] += ri[j2] < ri[j];
        }
        const int D = 1 << op.k;
        auto old_index = [&](int a) {
          int o = 0;
          for (int j = 0; j < op.k; ++j) o |= ((a >> pos[j]) & 1) << j;
          return o;
        };
        ro.coeff.assign(size_t(D) * D, cd());
        for (int a = 0; a < D; ++a)
          for (int b = 0; b < D; ++b) ro.coeff[size_t(a) * D + b] = op.coeff[size_t(old_index(a)) * D + old_index(b)];
      }
    }
    p.phases.push_back(rp);
  }
  p.reg_bits = RB;
  p.thread_bits = TB;
  return true;
}

// Expand a phase op (register encoding) to a 2^RB x 2^RB matrix.
std::vector<cd> reg_op_matrix(const RegOp& ro, int RB) {
  const int D = 1 << RB;
  std::vector<cd> m(size_t(D) * D, cd());
  if (ro.kind == OP_DIAG) {
    for (int r = 0; r < D; ++r) m[size_t(r) * D + r] = ro.coeff[ro.rmap[r]];
    return m;
  }
  std::vector<int> pos;
  for (int i = 0; i < RB; ++i)
    if ((ro.mask >> i) & 1) pos.push_back(i);
  const int k = int(pos.size()), d = 1 << k;
  for (int ro_ = 0; ro_ < D; ++ro_)
    for (int ri = 0; ri < D; ++ri) {
      if ((ro_ & ~ro.mask) != (ri & ~ro.mask)) continue;
      int a = 0, b = 0;
      for (int j = 0; j < k; ++j) {
        a |= ((ro_ >> pos[j]) & 1) << j;
        b |= ((ri >> pos[j]) & 1) << j;
      }
      m[size_t(ro_) * D + ri] = ro.coeff[size_t(a) * d + b];
    }
  return m;
}

// Turn up to max_mma whole register phases (c64, RB 5, 8 thread bits) whose
// ops all act on register bits only into one fused 32x32 matrix each,
// executed by k_reg_pass as a warp-level tensor-core GEMM (mma.sync m16n8k16,
// fp16 hi/lo split with per-row power-of-two scaling).  The GEMM phase uses the
// fragment layout: with the phase's register set R ascending (the matrix-local
// bit order) and the other 8 tile bits r0..r7 ascending,
//   register-index bits 0..4 <-> R[2], R[3], R[4], r3, r4
//   thread-index bits  0..7 <-> R[0], R[1], r0, r1, r2, r5, r6, r7
// so lane = 4 g + c holds complex columns i = c + 4 m (m = register bits 0..2)
// of the rows g, g + 8, g + 16, g + 24 (register bits 3, 4) of its warp.
void fuse_mma_phases(Pass& p, int min_dense, int max_mma, int prec) {
  const int RB = p.reg_bits;
  const int TB = p.thread_bits;
  if (RB != 5 || (TB != 8 && TB != 7) || prec != SVB_C64) return;
  const int D = 1 << RB;
  struct Cand { int dense, phase; };
  std::vector<Cand> cands;
  for (int f = 0; f < int(p.phases.size()); ++f) {
    const RegPhase& ph = p.phases[f];
    int dense = 0;
    bool ok = ph.op_end > ph.op_begin;
    for (int i = ph.op_begin; i < ph.op_end && ok; ++i) {
      const RegOp& ro = p.reg_ops[i];
      if (ro.kind == OP_DENSE) ++dense;
      else ok = ro.mask == 0 && ro.kx == 0;  // diagonal on register bits only
    }
    if (ok && dense >= 1) cands.push_back({dense, f});
  }
  // a pass goes to the tensor cores when one of its phases holds min_dense
  // dense ops; then every register-only phase does (measured: single-op
  // phases in a tensor-core pass are cheaper as GEMMs, layered-28 25.0 ->
  // 24.3 ms; an HBM-bound pass of single ops stays on the FMA pipes)
  bool any = false;
  for (const Cand& c : cands) any = any || c.dense >= min_dense;
  if (!any) return;
  std::sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {
    return x.dense != y.dense ? x.dense > y.dense : x.phase < y.phase;
  });
  if (int(cands.size()) > max_mma) cands.resize(max_mma);
  std::vector<char> chosen(p.phases.size(), 0);
  for (const Cand& c : cands) chosen[c.phase] = 1;
  std::vector<KernelOp> ops;
  std::vector<RegOp> rops;
  p.tc_mats.clear();
  for (int f = 0; f < int(p.phases.size()); ++f) {
    RegPhase& ph = p.phases[f];
    const int b = ph.op_begin, e = ph.op_end;
    ph.op_begin = int(ops.size());
    if (chosen[f]) {
      std::vector<cd> U(size_t(D) * D, cd());
      for (int r = 0; r < D; ++r) U[size_t(r) * D + r] = 1.0;
      for (int i = b; i < e; ++i) {
        const std::vector<cd> M = reg_op_matrix(p.reg_ops[i], RB);
        std::vector<cd> nu(size_t(D) * D, cd());
        for (int r = 0; r < D; ++r)
          for (int q = 0; q < D; ++q) {
            const cd mrq = M[size_t(r) * D + q];
            if (mrq == cd()) continue;
            for (int t = 0; t < D; ++t) nu[size_t(r) * D + t] += mrq * U[size_t(q) * D + t];
          }
        U.swap(nu);
        for (int g : p.ops[i].gates) ph.tc_gates.push_back(g);
      }
      ph.tc = int(p.tc_mats.size());
      p.tc_mats.push_back(std::move(U));
      ph.mma = true;
      ph.flags |= PH_MMA;
      if (TB == 7) {
        // tcgen05 phases (two-stream kernel): thread = one 32-amplitude row in
        // matrix order, i.e. the register-FMA layout built by build_phases
        ph.op_mid = ph.op_end = int(ops.size());
        continue;
      }
      // row bits: g0, g1 (lanes 2, 3) complete the bank positions of the
      // half-warp together with R[0], R[1] (lanes 0, 1): tile bit t lands on
      // bank-row position t mod 4 under the XOR swizzle, and on t itself in
      // the linear TMA layout -- prefer exactly {0..3}, else distinct
      // residues; g2 (lane 4) then prefers bit 4 (256-B coalesced stores)
      std::vector<int> rows;
      for (int q = 0; q < p.T; ++q)
        if (std::find(ph.R, ph.R + RB, q) == ph.R + RB) rows.push_back(q);
      std::vector<int> pick;
      auto take_row = [&](int q) {
        rows.erase(std::find(rows.begin(), rows.end(), q));
        pick.push_back(q);
      };
      int used = (1 << (ph.R[0] & 3)) | (1 << (ph.R[1] & 3));
      for (int want = 0; want < 2; ++want) {
        int best = -1;
        for (int q : rows) {
          const bool fresh = !((used >> (q & 3)) & 1);
          const int score = (fresh ? 2 : 0) + (q < 4 ? 1 : 0);
          const int bscore = best < 0 ? -1 : (!((used >> (best & 3)) & 1) ? 2 : 0) + (best < 4 ? 1 : 0);
          if (score > bscore) best = q;
        }
        used |= 1 << (best & 3);
        take_row(best);
      }
      take_row(std::find(rows.begin(), rows.end(), 4) != rows.end() ? 4 : rows[0]);
      // warp bits: the remaining rows (3 with one tile stream, 2 with two)
      const int lay[13] = {ph.R[2], ph.R[3], ph.R[4], rows[0], rows[1],
                           ph.R[0], ph.R[1], pick[0], pick[1], pick[2], rows[2], rows[3],
                           TB == 8 ? rows[4] : 0};
      for (int i = 0; i < 13; ++i) ph.map[i] = lay[i];
      set_layout_flags(ph, RB, prec, f == 0, f + 1 == int(p.phases.size()));
    } else {
      for (int i = b; i < e; ++i) {
        ops.push_back(p.ops[i]);
        rops.push_back(p.reg_ops[i]);
      }
    }
    ph.op_mid = ph.op_end = int(ops.size());
  }
  p.ops.swap(ops);
  p.reg_ops.swap(rops);
  p.mma_phases = true;
  // all ops of the pass unitary (|U^dagger U - 1| <= 1e-9, diagonal |z| = 1):
  // the tile 2-norm is invariant and the kernel restores it
  auto unitary = [](const std::vector<cd>& m, int d) {
    for (int r = 0; r < d; ++r)
      for (int t = 0; t < d; ++t) {
        cd acc = 0.0;
        for (int q = 0; q < d; ++q) acc += std::conj(m[size_t(q) * d + r]) * m[size_t(q) * d + t];
        if (std::abs(acc - (r == t ? cd(1.0) : cd(0.0))) > 1e-9) return false;
      }
    return true;
  };
  bool ok = true;
  for (const auto& U : p.tc_mats) ok = ok && unitary(U, D);
  for (const KernelOp& op : p.ops) {
    if (op.kind == OP_DIAG) {
      for (const cd& z : op.coeff) ok = ok && std::abs(std::abs(z) - 1.0) <= 1e-9;
    } else {
      ok = ok && unitary(op.coeff, 1 << op.k);
    }
  }
  p.renorm = ok;
}

// ------------------------------------------------------------ k_gemm_pass
constexpr int kGemmDefaultWarps = 4;  // measured: 8 warps (64 registers, spills) 17.4 vs 16.0 ms
// A-operand word of each tile bit in a phase layout (register bits j0..j4 =
// map[0..4], row bits m0..m6 = map[5..11]); word = m 32 + ((j >> 2) ^ (m & 7)) 4
// + (j & 3), the K-major SWIZZLE_128B canonical layout of svb_gemmpass.cuh.
void gemm_word_table(const int* map, unsigned short* wt) {
  static const unsigned short jw[5] = {1, 2, 4, 8, 16};
  static const unsigned short mw[7] = {32 | 4, 64 | 8, 128 | 16, 256, 512, 1024, 2048};
  for (int i = 0; i < 16; ++i) wt[i] = 0;
  for (int i = 0; i < 5; ++i) wt[map[i]] = jw[i];
  for (int b = 0; b < 7; ++b) wt[map[5 + b]] = mw[b];
}

int gf2_rank(std::vector<int> v) {
  int r = 0;
  for (int bit = 31; bit >= 0; --bit) {
    int piv = -1;
    for (size_t i = r; i < v.size(); ++i)
      if ((v[i] >> bit) & 1) {
        piv = int(i);
        break;
      }
    if (piv < 0) continue;
    std::swap(v[r], v[piv]);
    for (size_t i = 0; i < v.size(); ++i)
      if (int(i) != r && ((v[i] >> bit) & 1)) v[i] ^= v[r];
    ++r;
  }
  return r;
}

// Shared-memory wavefronts of one warp instruction: lanes l = 0..31 access
// `bytes` at byte address addr[l]; the warp is served in groups of 128 / bytes
// lanes, each group in as many wavefronts as its most-loaded bank has
// distinct 4-byte words.  Returns log2(wavefronts / ideal).
int smem_excess(const std::vector<long long>& addr, int bytes) {
  const int per = 128 / bytes;
  int total = 0;
  long long words[128];
  for (int g0 = 0; g0 < 32; g0 += per) {
    int nw = 0;
    for (int l = g0; l < g0 + per; ++l)
      for (int w = 0; w < bytes / 4; ++w) words[nw++] = addr[l] / 4 + w;
    std::sort(words, words + nw);
    nw = int(std::unique(words, words + nw) - words);
    int cnt[32] = {0}, mx = 0;
    for (int i = 0; i < nw; ++i) mx = std::max(mx, ++cnt[words[i] & 31]);
    total += mx;
  }
  const int ideal = 32 * bytes / 128;
  int lg = 0;
  while ((ideal << lg) < total) ++lg;
  return lg;
}

// tile index of the element in register `rho` of lane `lane` (warp 0) of a thread layout
long long lane_elem(const int* map, int lane, int rho) {
  long long x = 0;
  for (int i = 0; i < 5; ++i)
    if ((rho >> i) & 1) x |= 1LL << map[i];
  for (int b = 0; b < 5; ++b)
    if ((lane >> b) & 1) x |= 1LL << map[5 + b];
  return x;
}

// A writes (STS.32 of f16x2 words) from thread layout `cur` into the A layout `nxt`
int gemm_write_conflict(const int* cur, const int* nxt) {
  unsigned short wt[16];
  gemm_word_table(nxt, wt);
  std::vector<long long> addr(32);
  for (int l = 0; l < 32; ++l) {
    const long long x = lane_elem(cur, l, 0);
    int w = 0;
    for (int t = 0; t < kGemmTileBits; ++t)
      if ((x >> t) & 1) w ^= wt[t];
    addr[l] = 4LL * w;
  }
  return smem_excess(addr, 4);
}

// Loads of the linear TMA tile in the load layout (16-byte pairs when register
// bit 0 is tile bit 0, else 8-byte amplitudes)
int gemm_load_conflict(const int* map0) {
  const int bytes = map0[0] == 0 ? 16 : 8;
  std::vector<long long> addr(32);
  for (int l = 0; l < 32; ++l) addr[l] = 8 * lane_elem(map0, l, 0);
  return smem_excess(addr, bytes);
}

// log2 of the extra 128-B segments of the final global stores (tile bits
// below L are contiguous; anything above lands in another segment)
int gemm_store_cost(const int* map, int L) {
  const int bytes = map[0] == 0 ? 16 : 8;
  long long seg[32];
  for (int l = 0; l < 32; ++l) {
    const long long x = lane_elem(map, l, 0);
    const long long lo = x & ((1LL << L) - 1), hi = x >> L;
    seg[l] = (hi << 40) | ((8 * lo) / 128);
  }
  std::sort(seg, seg + 32);
  const int ns = int(std::unique(seg, seg + 32) - seg);
  const int ideal = 32 * bytes / 128;
  int lg = 0;
  while ((ideal << lg) < ns) ++lg;
  return lg;
}

// Thread layout of a GEMM phase's D read-out: 32x32b -> thread = row (m0..m6),
// registers = columns j0..j4; 16x256b -> registers j2 j3 j4 m3 m4, lanes
// j0 j1 m0 m1 m2, warps m5 m6 (see gemm_read_half)
void gemm_thread_map(const int* alay, bool ld16, int* map) {
  if (!ld16) {
    for (int i = 0; i < 12; ++i) map[i] = alay[i];
    return;
  }
  const int m[12] = {alay[2], alay[3], alay[4], alay[5 + 3], alay[5 + 4],
                     alay[0], alay[1], alay[5 + 0], alay[5 + 1], alay[5 + 2], alay[5 + 5], alay[5 + 6]};
  for (int i = 0; i < 12; ++i) map[i] = m[i];
}

// A layout of GEMM phase f (j0..j4 = register qubits, m0..m6 = rows) given the
// lanes of the writing layout: previous lanes that are register qubits go to
// j0, j1 (bank bits 0, 1) and then to j2..j4, those that are row qubits to
// m0..m2 (bank bits 2..4 -- XOR-paired with j2..j4, so a pair never shares a
// bank bit).  `j01` (optional) claims j0, j1 first (low qubits on the lanes of
// a 16x256b read-out); the free lane rows take the qubits in `pref`.
void gemm_layout(const int* prev_lanes, const int* R, const std::vector<int>& pref, const std::vector<int>* j01,
                 int* alay) {
  const int T = kGemmTileBits;
  std::vector<int> inR(T, 0);
  for (int i = 0; i < 5; ++i) inR[R[i]] = 1;
  std::vector<int> X, Y;
  for (int b = 0; b < 5; ++b) (inR[prev_lanes[b]] ? X : Y).push_back(prev_lanes[b]);
  int j[5] = {-1, -1, -1, -1, -1}, m[7] = {-1, -1, -1, -1, -1, -1, -1};
  std::vector<int> used(T, 0);
  int s = 0;
  if (j01)
    for (int t : *j01)
      if (s < 2 && inR[t] && !used[t]) {
        j[s++] = t;
        used[t] = 1;
      }
  for (int t : X)
    if (s < 2 && !used[t]) {
      j[s++] = t;
      used[t] = 1;
    }
  bool slot_used[3] = {false, false, false};  // bank bits 2..4
  int yi = 0;
  for (int t : Y)
    if (yi < 3) {
      m[yi] = t;
      used[t] = 1;
      slot_used[yi++] = true;
    }
  for (int t : X) {
    if (used[t]) continue;
    for (int sl = 0; sl < 3; ++sl)
      if (!slot_used[sl] && j[2 + sl] < 0) {
        j[2 + sl] = t;
        used[t] = 1;
        slot_used[sl] = true;
        break;
      }
  }
  for (int i = 0; i < 5; ++i)
    if (j[i] < 0)
      for (int q = 0; q < 5; ++q)
        if (!used[R[q]]) {
          j[i] = R[q];
          used[R[q]] = 1;
          break;
        }
  for (int t : Y)
    if (!used[t])
      for (int i = 0; i < 7; ++i)
        if (m[i] < 0) {
          m[i] = t;
          used[t] = 1;
          break;
        }
  for (int i = 0; i < 7; ++i) {
    if (m[i] >= 0) continue;
    int pick = -1;
    if (i < 5)
      for (int t : pref)
        if (!used[t] && !inR[t]) {
          pick = t;
          break;
        }
    if (pick < 0)
      for (int t = 0; t < T; ++t)
        if (!used[t] && !inR[t]) {
          pick = t;
          break;
        }
    m[i] = pick;
    used[pick] = 1;
  }
  for (int i = 0; i < 5; ++i) alay[i] = j[i];
  for (int b = 0; b < 7; ++b) alay[5 + b] = m[b];
}

// Lower a pass (12-qubit tile, unitary ops) for k_gemm_pass: list-schedule
// register phases (build_phases), fold each phase's dense ops and register-
// only diagonal ops into one 32x32 matrix, move diagonal ops on row / outside
// bits before or after the GEMM they commute with, and choose every phase's
// qubit order for conflict-free A writes and coalesced loads / stores.
// Returns false (pass left unchanged) when the pass does not fit the kernel.
bool build_gemm_pass(Pass& p, int streams, int warps) {
  const int T = kGemmTileBits;
  if (p.T != T) return false;
  for (const KernelOp& op : p.ops) {  // unitary ops only (the kernel rescales by the tile norm)
    const int d = 1 << op.k;
    if (op.kind == OP_DIAG) {
      for (const cd& z : op.coeff)
        if (std::abs(std::abs(z) - 1.0) > 1e-9) return false;
      continue;
    }
    for (int r = 0; r < d; ++r)
      for (int t = 0; t < d; ++t) {
        cd acc = 0.0;
        for (int q = 0; q < d; ++q) acc += std::conj(op.coeff[size_t(q) * d + r]) * op.coeff[size_t(q) * d + t];
        if (std::abs(acc - (r == t ? cd(1.0) : cd(0.0))) > 1e-9) return false;
      }
  }
  Pass q = p;
  if (!build_phases(q, 5, SVB_C64, 7)) return false;
  struct GP {
    int R[5];
    std::vector<cd> U;  // ascending-R index space
    std::vector<int> post, gates;
  };
  std::vector<int> pre0;
  std::vector<GP> gps;
  const int D = 32;
  auto bits_of = [&](const KernelOp& op) {
    unsigned long long b = 0;  // tile bits 0..T-1, outside-tile qubits at T + q
    for (int j = 0; j < op.k; ++j) b |= 1ULL << std::min(op.tgt[j], 63);
    return b;
  };
  for (const RegPhase& ph : q.phases) {
    const int* R = ph.R;
    int rmask = 0;
    for (int i = 0; i < 5; ++i) rmask |= 1 << R[i];
    auto rpos = [&](int t) {
      for (int i = 0; i < 5; ++i)
        if (R[i] == t) return i;
      return -1;
    };
    std::vector<unsigned long long> dense_bits;
    for (int i = ph.op_begin; i < ph.op_end; ++i)
      dense_bits.push_back(q.ops[i].kind == OP_DENSE ? bits_of(q.ops[i]) : 0ULL);
    bool any_dense = false;
    for (auto b : dense_bits) any_dense = any_dense || b;
    if (!any_dense) {
      for (int i = ph.op_begin; i < ph.op_end; ++i) (gps.empty() ? pre0 : gps.back().post).push_back(i);
      continue;
    }
    // segments: ops fold into the open GEMM; a diagonal op on row / outside
    // qubits moves after it (commutes with the phase's later dense ops) or
    // before it (commutes with the dense ops folded so far), else the GEMM is
    // closed there and the op runs between it and the next one (same columns)
    auto fresh = [&]() {
      GP g;
      for (int i = 0; i < 5; ++i) g.R[i] = R[i];
      g.U.assign(size_t(D) * D, cd());
      for (int r = 0; r < D; ++r) g.U[size_t(r) * D + r] = 1.0;
      return g;
    };
    GP g = fresh();
    unsigned long long folded = 0;  // dense qubits folded into the open GEMM
    std::vector<int> pre;
    for (int i = ph.op_begin; i < ph.op_end; ++i) {
      const KernelOp& op = q.ops[i];
      const unsigned long long b = bits_of(op);
      const bool reg_only = (b & ~(unsigned long long)rmask) == 0;
      if (op.kind == OP_DIAG && !reg_only) {
        unsigned long long after = 0;
        for (int k = i + 1; k < ph.op_end; ++k) after |= dense_bits[k - ph.op_begin];
        if ((b & after) == 0) {
          g.post.push_back(i);
        } else if ((b & folded) == 0) {
          pre.push_back(i);
        } else {
          for (int k : pre) (gps.empty() ? pre0 : gps.back().post).push_back(k);
          pre.clear();
          g.post.push_back(i);
          gps.push_back(std::move(g));
          g = fresh();
          folded = 0;
        }
        continue;
      }
      if (op.kind == OP_DENSE) folded |= b;
      // fold into U: M (in ascending-R index space) times U
      int pos[kMaxK];
      for (int j = 0; j < op.k; ++j) pos[j] = rpos(op.tgt[j]);
      std::vector<cd> nu(size_t(D) * D, cd());
      const int d = 1 << op.k;
      int omask = 0;
      for (int j = 0; j < op.k; ++j) omask |= 1 << pos[j];
      for (int r = 0; r < D; ++r) {
        int a = 0;
        for (int j = 0; j < op.k; ++j) a |= ((r >> pos[j]) & 1) << j;
        for (int bb = 0; bb < d; ++bb) {
          cd mrb;
          if (op.kind == OP_DIAG) {
            if (bb != a) continue;
            mrb = op.coeff[a];
          } else {
            mrb = op.coeff[size_t(a) * d + bb];
          }
          if (mrb == cd()) continue;
          int c = r & ~omask;
          for (int j = 0; j < op.k; ++j) c |= ((bb >> j) & 1) << pos[j];
          for (int s = 0; s < D; ++s) nu[size_t(r) * D + s] += mrb * g.U[size_t(c) * D + s];
        }
      }
      g.U.swap(nu);
      for (int gi : op.gates) g.gates.push_back(gi);
    }
    for (int i : pre) (gps.empty() ? pre0 : gps.back().post).push_back(i);
    gps.push_back(std::move(g));
  }
  const int P = int(gps.size());
  if (P < 1 || P > kMaxMmaPerPass || P + 1 > kMaxPhases) return false;

  // ---- layouts.  Load lanes: tile qubits 1, 2, 3 (conflict-free 16-byte
  // loads with tile qubit 0 in register bit 0) plus two more; then each GEMM
  // phase greedily (A layout from the writing lanes) with a 32x32b or 16x256b
  // D read-out.  Cost: smem wavefronts of the loads and A writes, 128-B
  // segments of the final stores (doubled: global).
  const std::vector<int> low = {0, 1, 2, 3};
  auto pref_for = [&](int f) {  // qubits the lanes of GEMM phase f should carry
    std::vector<int> pr;
    if (f < P) {
      for (int i = 0; i < 5; ++i) pr.push_back(gps[f].R[i]);  // gps[f] is GEMM phase f + 1
    } else {
      pr = low;
    }
    return pr;
  };
  int best_cost = 1 << 30;
  std::vector<std::vector<int>> best_maps, best_alay;
  std::vector<int> best_ld16;
  // read-out shape choices: the last phase's (store coalescing) always, the
  // intermediate ones only for short passes (planning time)
  const int n_shape = P <= 2 ? (1 << P) : 2;
  for (int a = 0; a < T; ++a)
    for (int b = a + 1; b < T; ++b) {
      if (a <= 3 || b <= 3) continue;  // lanes = {1, 2, 3, a, b}
      for (int shape = 0; shape < n_shape * 2; ++shape) {
        std::vector<std::vector<int>> mp(P + 1, std::vector<int>(16, 0)), al(P + 1, std::vector<int>(16, 0));
        std::vector<int> ld16(P + 1, 0);
        // load layout: register bit 0 = tile qubit 0, lanes 1 2 3 a b
        std::vector<int> rest;
        for (int t = 0; t < T; ++t)
          if (t != 0 && t != 1 && t != 2 && t != 3 && t != a && t != b) rest.push_back(t);
        const int m0[12] = {0, rest[0], rest[1], rest[2], rest[3], 1, 2, 3, a, b, rest[4], rest[5]};
        for (int i = 0; i < 12; ++i) mp[0][i] = m0[i];
        int cost = gemm_load_conflict(mp[0].data());
        for (int f = 1; f <= P; ++f) {
          const bool last = f == P;
          ld16[f] = n_shape == 2 ? (last ? (shape & 1) : 0) : ((shape >> (f - 1)) & 1);
          const bool lowj = last && ld16[f] && (shape >> (n_shape == 2 ? 1 : P)) & 1;
          gemm_layout(&mp[f - 1][5], gps[f - 1].R, pref_for(f), lowj ? &low : nullptr, al[f].data());
          gemm_thread_map(al[f].data(), ld16[f], mp[f].data());
          cost += 2 * gemm_write_conflict(mp[f - 1].data(), al[f].data());
        }
        cost += 3 * gemm_store_cost(mp[P].data(), p.L);
        if (cost < best_cost) {
          best_cost = cost;
          best_maps = mp;
          best_alay = al;
          best_ld16 = ld16;
        }
      }
    }
  const std::vector<std::vector<int>>& maps = best_maps;
  int conflicts = 0;
  for (int f = 1; f <= P; ++f) conflicts += gemm_write_conflict(maps[f - 1].data(), best_alay[f].data());

  // ---- assemble: ops in execution order, phases, GEMM matrices in layout order
  std::vector<int> order;
  std::vector<std::pair<int, int>> ranges;
  ranges.push_back({0, int(pre0.size())});
  for (int i : pre0) order.push_back(i);
  for (int f = 0; f < P; ++f) {
    const int b0 = int(order.size());
    for (int i : gps[f].post) order.push_back(i);
    ranges.push_back({b0, int(order.size())});
  }
  std::vector<KernelOp> ops;
  for (int i : order) ops.push_back(q.ops[i]);
  p.ops.swap(ops);
  p.reg_ops.assign(p.ops.size(), RegOp());
  p.phases.clear();
  p.tc_mats.clear();
  for (int f = 0; f <= P; ++f) {
    RegPhase rp;
    const int* mp = maps[f].data();
    for (int i = 0; i < 16; ++i) rp.map[i] = i < T ? mp[i] : 0;
    // R = the GEMM's column qubits in matrix order (the A layout's j0..j4);
    // the load phase has no GEMM: its register qubits
    for (int i = 0; i < 5; ++i) rp.R[i] = f == 0 ? mp[i] : best_alay[f][i];
    rp.op_begin = ranges[f].first;
    rp.op_end = ranges[f].second;
    if (f == 0) {
      rp.op_mid = rp.op_end;  // ops before any GEMM
      rp.tc = -1;
    } else {
      rp.op_mid = rp.op_begin;  // GEMM first, then the diagonal ops
      rp.tc = f - 1;
      if (best_ld16[f]) rp.flags |= PH_LD16;
      const int* al = best_alay[f].data();
      gemm_word_table(al, rp.wt);
      rp.tc_gates = gps[f - 1].gates;
      // U in the A layout's column order: column bit i <-> tile bit al[i]
      const int* R = gps[f - 1].R;
      int to_asc[5];
      for (int i = 0; i < 5; ++i)
        for (int k = 0; k < 5; ++k)
          if (R[k] == al[i]) to_asc[i] = k;
      auto conv = [&](int x) {
        int y = 0;
        for (int i = 0; i < 5; ++i) y |= ((x >> i) & 1) << to_asc[i];
        return y;
      };
      std::vector<cd> U(size_t(D) * D);
      for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) U[size_t(r) * D + c] = gps[f - 1].U[size_t(conv(r)) * D + conv(c)];
      p.tc_mats.push_back(std::move(U));
    }
    // diagonal ops in this layout: table index = [thread bits | register bits | outside bits]
    for (int i = rp.op_begin; i < rp.op_end; ++i) {
      const KernelOp& op = p.ops[i];
      RegOp& ro = p.reg_ops[i];
      ro.kind = op.kind;
      ro.k = op.k;
      std::vector<std::pair<int, int>> regb, thrb, extb;
      for (int b = 0; b < op.k; ++b) {
        const int t = op.tgt[b];
        if (t >= T) {
          extb.push_back({t - T, b});
          continue;
        }
        int where = -1;
        for (int k = 0; k < T; ++k)
          if (mp[k] == t) where = k;
        if (where < 5)
          regb.push_back({where, b});
        else
          thrb.push_back({where - 5, b});
      }
      std::sort(regb.begin(), regb.end());
      std::sort(thrb.begin(), thrb.end());
      std::sort(extb.begin(), extb.end());
      const int kr = int(regb.size()), kt = int(thrb.size()), kx = int(extb.size());
      ro.mask = kt;
      for (int j = 0; j < kt; ++j) ro.src[j] = thrb[j].first;
      ro.rmask = 0;
      for (int j = 0; j < kr; ++j) ro.rmask |= 1 << regb[j].first;
      ro.kx = kx;
      ro.xmask = 0;
      for (int j = 0; j < kx; ++j) ro.xmask |= 1ULL << extb[j].first;
      for (int rho = 0; rho < 32; ++rho) {
        int d = 0;
        for (int j = 0; j < kr; ++j) d |= ((rho >> regb[j].first) & 1) << (kt + j);
        ro.rmap[rho] = static_cast<unsigned char>(d);
      }
      ro.coeff.assign(op.coeff.size(), cd());
      for (size_t nidx = 0; nidx < op.coeff.size(); ++nidx) {
        int old = 0;
        for (int j = 0; j < kt; ++j) old |= ((int(nidx) >> j) & 1) << thrb[j].second;
        for (int j = 0; j < kr; ++j) old |= ((int(nidx) >> (kt + j)) & 1) << regb[j].second;
        for (int j = 0; j < kx; ++j) old |= ((int(nidx) >> (kr + kt + j)) & 1) << extb[j].second;
        ro.coeff[nidx] = op.coeff[old];
      }
    }
    p.phases.push_back(rp);
  }
  p.reg_bits = 5;
  p.thread_bits = 7;
  p.streams = streams >= 2 && streams <= 4 ? streams : 4;
  p.gemm_warps = warps == 4 ? 4 : warps == 8 ? 8 : kGemmDefaultWarps;
  p.gemm = true;
  p.mma_phases = false;
  p.renorm = true;
  p.bank_conflicts = conflicts;
  return true;
}

}  // namespace

// Decide the TMA tensor-map shape of a pass and the tile-local order of its
// high bits (see Pass).  Includes as many runs of consecutive tile bits in the
// box as fit a rank-5 tensor map; the remaining high bits are enumerated.
void plan_tma(Pass& p, int n, int prec) {
  const int sh = prec == SVB_C128 ? 1 : 0;
  const int nw = n + sh;
  std::vector<std::pair<int, int>> runs;  // qubit-space [start, len)
  runs.push_back({0, p.L});
  for (int b = 0; b < p.m; ++b) {
    const int q = p.high[b];
    if (runs.back().first + runs.back().second == q)
      runs.back().second++;
    else
      runs.push_back({q, 1});
  }
  struct Dim { int start, bits, box; };
  // dims for the subset `inc` (bit r set: run r is a box dim; run 0 always)
  auto dims_for = [&](unsigned inc) {
    std::vector<Dim> d;
    int c = 0;
    for (int r = 0; r < int(runs.size()); ++r) {
      if (!((inc >> r) & 1)) continue;
      int st = runs[r].first == 0 ? 0 : runs[r].first + sh;
      int len = runs[r].second + (runs[r].first == 0 ? sh : 0);
      if (st > c) d.push_back({c, st - c, 0});
      while (len > 0) {
        int piece = std::min(len, 8);
        d.push_back({st, piece, piece});
        st += piece;
        len -= piece;
      }
      c = st;
    }
    if (c < nw) d.push_back({c, nw - c, 0});
    return d;
  };
  // choose the subset of runs that fits rank 5 with the fewest enumerated bits
  const int nr = int(runs.size());
  unsigned best = 0;
  int best_excl = 1 << 30;
  for (unsigned inc = 1; inc < (1u << nr); inc += 2) {  // run 0 always included
    if (int(dims_for(inc).size()) > 5) continue;
    int excl = 0;
    for (int r = 0; r < nr; ++r)
      if (!((inc >> r) & 1)) excl += runs[r].second;
    if (excl < best_excl) {
      best_excl = excl;
      best = inc;
    }
  }
  if (best == 0 || best_excl > 6) {  // no usable tensor map: 1-D bulk copies per chunk
    p.tma_rank = 0;
    p.n_enum = 0;
  } else {
    std::vector<Dim> d = dims_for(best);
    p.tma_rank = int(d.size());
    for (int i = 0; i < p.tma_rank; ++i) {
      p.tma_start[i] = d[i].start;
      p.tma_bits[i] = d[i].bits;
      p.tma_box[i] = d[i].box;
    }
    // tile-local order: included high runs first, enumerated ones last
    std::vector<int> inc, exc;
    for (int r = 1; r < nr; ++r)
      for (int j = 0; j < runs[r].second; ++j) (((best >> r) & 1) ? inc : exc).push_back(runs[r].first + j);
    int b = 0;
    for (int q : inc) p.high[b++] = q;
    for (int q : exc) p.high[b++] = q;
    p.n_enum = int(exc.size());
  }
  for (int b = 0; b < p.m; ++b) p.high_sorted[b] = p.high[b];
  std::sort(p.high_sorted, p.high_sorted + p.m);
}

bool make_gates(int n, int n_ops, const int* op_k, const int* op_targets, const double* op_mats,
                std::vector<Gate>& out, std::string& err) {
  out.clear();
  out.reserve(n_ops);
  size_t off = 0;
  for (int i = 0; i < n_ops; ++i) {
    Gate g;
    g.k = op_k[i];
    if (g.k < 1 || g.k > kMaxDenseK) {
      err = "gate " + std::to_string(i) + ": arity " + std::to_string(g.k) +
            " outside supported range 1.." + std::to_string(kMaxDenseK);
      return false;
    }
    if (g.k > n) {
      err = "gate " + std::to_string(i) + ": arity exceeds qubit count";
      return false;
    }
    for (int j = 0; j < g.k; ++j) {
      int t = op_targets[i * SVB_MAX_TARGETS + j];
      if (t < 0 || t >= n) {
        err = "target out of range for " + std::to_string(n) + " qubits at gate " + std::to_string(i);
        return false;
      }
      for (int j2 = 0; j2 < j; ++j2)
        if (g.t[j2] == t) {
          err = "duplicate target at gate " + std::to_string(i);
          return false;
        }
      g.t[j] = t;
    }
    const int d = 1 << g.k;
    const double* mat = op_mats + off;
    off += size_t(2) * d * d;
    g.diag = is_diagonal(g.k, mat);
    if (g.diag) {
      g.m.resize(d);
      for (int r = 0; r < d; ++r) g.m[r] = cd(mat[2 * (r * d + r)], mat[2 * (r * d + r) + 1]);
    } else {
      g.m.resize(size_t(d) * d);
      for (int e = 0; e < d * d; ++e) g.m[e] = cd(mat[2 * e], mat[2 * e + 1]);
    }
    out.push_back(std::move(g));
  }
  return true;
}

bool build_plan_merged(int n, int prec, const std::vector<Gate>& gates, const svb_plan_options& opt_in,
                       Plan& plan, std::string& err, bool ctlx = true) {
  if (n < 1 || n > 62) {
    err = "n_local must be in 1..62";
    return false;
  }
  if (prec != SVB_C64 && prec != SVB_C128) {
    err = "precision must be SVB_C64 or SVB_C128";
    return false;
  }
  svb_plan_options opt = opt_in;
  // c64 tensor cores (default): passes with >= 2 dense gates run on
  // k_gemm_pass (every dense op in tcgen05 GEMMs with shared-memory operands);
  // tensor_cores == 2: the k_reg_pass tensor-core phases (tcgen05 with A in
  // TMEM on 12-qubit tiles, warp-level mma.sync on 13-qubit tiles);
  // tensor_cores == -1: FMA pipes only
  const bool use_gemm = prec == SVB_C64 && (opt.tensor_cores == 0 || opt.tensor_cores == 1) &&
                        !opt.no_reg_phases && (opt.tile_bits == 0 || opt.tile_bits == kGemmTileBits) &&
                        (opt.reg_bits == 0 || opt.reg_bits == 5) && opt.streams != 1;
  const bool use_mma = prec == SVB_C64 && opt.tensor_cores >= 0 && !opt.no_reg_phases &&
                       (opt.reg_bits == 0 || opt.reg_bits == 5);
  // c64 tensor-core phases: 12-qubit tiles in warp-group streams (measured
  // layered-28 33.2 ms vs 43.3 ms for 13-qubit tiles with mma.sync phases)
  int T = opt.tile_bits > 0 ? opt.tile_bits
          : ((use_gemm || (use_mma && opt.streams != 1)) ? 12
             : (prec == SVB_C128 && opt.streams != 1 && (opt.reg_bits == 0 || opt.reg_bits == 4)) ? 11
                                                                                                : default_tile_bits(prec));
  // 64 KiB tiles at most (two-stage TMA ring must fit shared memory)
  if (T > (prec == SVB_C64 ? 13 : 12)) T = prec == SVB_C64 ? 13 : 12;
  if (T > n) T = n;
  int Lmin = opt.min_low_bits > 0 ? opt.min_low_bits : default_min_low_bits(prec);
  if (Lmin > T) Lmin = T;
  if (Lmin < T - kMaxHigh) Lmin = T - kMaxHigh;
  if (prec == SVB_C64 && Lmin < 1) Lmin = 1;  // chunks must be >= 16 bytes
  int mmax = T - Lmin;
  // Wide-chunk alternative (1 KiB contiguous runs: 7 low bits c64, 6 c128):
  // a pass whose strided tile qubits are scattered reads 2^L-amplitude chunks
  // all over the shard, and at 128 B (the default L) HBM runs at 20-50 % of
  // its bandwidth (measured on random-target circuits, paper Table 2: n = 30
  // c64 69 -> 47 ms, c128 432 -> 302 ms with 1 KiB chunks).  Used for a pass
  // when it absorbs >= 90 % of the gates the default candidate does.
  const int Lbase = Lmin;
  const int Lwide = opt.min_low_bits > 0 ? Lbase : std::min(T - 2, prec == SVB_C64 ? 7 : 6);
  const int max_ops = (opt.max_ops_per_pass > 0 && opt.max_ops_per_pass < kMaxOps)
                          ? opt.max_ops_per_pass : kMaxOps;
  const double default_budget =
      opt.cost_budget == 0.0 ? default_cost_budget(prec) : opt.cost_budget;
  double budget = default_budget;  // the tail merge below lifts it
  const size_t pool_cap = prec == SVB_C64 ? size_t(kPoolBytesC64) / 8 : size_t(kPoolBytesC128) / 16;
  const CostModel cm(prec);

  plan.n = n;
  plan.prec = prec;
  plan.opt = opt;
  plan.passes.clear();

  // c128: 2q gates that are block-diagonal in one qubit (controlled-U, exact
  // zeros) need only their target in the tile -- the control may be a shard
  // qubit outside it (U0 / U1 chosen per tile), and it orders like a diagonal
  // touch.  gctl[i] = local index of that control, or -1.
  std::vector<int> gctl(gates.size(), -1);
  if (ctlx && prec == SVB_C128 && !std::getenv("SVB_NO_CTRLX"))
    for (size_t i = 0; i < gates.size(); ++i) {
      const Gate& g = gates[i];
      if (g.diag || g.k != 2 || g.m.size() != 16) continue;
      for (int b = 0; b < 2 && gctl[i] < 0; ++b) {
        bool bd = true;
        for (int r = 0; r < 4 && bd; ++r)
          for (int c = 0; c < 4 && bd; ++c)
            if (((r >> b) & 1) != ((c >> b) & 1)) bd = g.m[size_t(r) * 4 + c] == cd();
        if (bd) gctl[i] = b;
      }
    }
  for (size_t i = 0; i < gates.size(); ++i) {
    int high_needed = 0;  // diagonal gates need no tile qubits (bits outside the tile are per-tile constants)
    if (!gates[i].diag)
      for (int j = 0; j < gates[i].k; ++j) high_needed += gates[i].t[j] >= Lmin && j != gctl[i];
    if (high_needed > mmax) {
      err = "gate " + std::to_string(i) + " needs more strided tile bits than the tile allows";
      return false;
    }
  }

  std::vector<int> pending(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) pending[i] = int(i);

  // One greedy scan over the pending gates.  `allowed` (optional) restricts the
  // strided tile qubits to a window; the result is the pass it would build.
  struct Scan {
    std::vector<int> taken, deferred;
    std::vector<char> in_high;
    double cost = 0.0;
  };
  auto scan = [&](const std::vector<int>& pend, const std::vector<char>* allowed) {
    Scan r;
    std::vector<char> block_all(n, 0), block_dense(n, 0);
    r.in_high.assign(n, 0);
    int n_high = 0;
    // Mirror of the diagonal-run merge done at lowering time, so that a
    // diagonal gate joining an open run is charged only its marginal cost and
    // the coefficient pool is accounted for with the merged table sizes.
    std::vector<int> acc_bits;
    bool acc_open = false;
    size_t closed_pool = 0;
    int n_kops = 0;  // kernel ops after merging (what max_ops bounds)
    const bool merging = !opt.no_diag_merge;
    for (int gi : pend) {
      const Gate& g = gates[gi];
      const int gc = gctl[gi];  // a control that may stay outside the tile
      bool blocked = false;
      for (int j = 0; j < g.k && !blocked; ++j)
        blocked = block_all[g.t[j]] || (!g.diag && j != gc && block_dense[g.t[j]]);
      bool take = false;
      if (!blocked) {
        int extra = 0;
        bool outside = false;
        for (int j = 0; j < g.k; ++j)
          if (!g.diag && j != gc && g.t[j] >= Lmin && !r.in_high[g.t[j]]) {
            ++extra;
            outside |= allowed && !(*allowed)[g.t[j]];
          }
        double c;
        size_t new_closed = closed_pool;
        std::vector<int> new_acc = acc_bits;
        bool new_open = acc_open;
        int new_kops = n_kops + 1;
        if (!merging) {
          c = cm.of(g);
          new_closed += g.m.size();
        } else if (g.diag) {
          std::vector<int> u = acc_bits;
          for (int j = 0; j < g.k; ++j)
            if (std::find(u.begin(), u.end(), g.t[j]) == u.end()) u.push_back(g.t[j]);
          if (acc_open && int(u.size()) <= kMaxDiagK) {
            c = cm.diag(int(u.size())) - cm.diag(int(acc_bits.size()));
            new_acc = u;
            new_kops = n_kops;
          } else {
            if (acc_open) new_closed += size_t(1) << acc_bits.size();
            c = cm.diag(g.k);
            new_acc.assign(g.t, g.t + g.k);
          }
          new_open = true;
        } else {
          c = cm.dense(g.k);
          new_closed += g.m.size();
          bool touches = false;
          for (int j = 0; j < g.k; ++j)
            touches |= std::find(acc_bits.begin(), acc_bits.end(), g.t[j]) != acc_bits.end();
          if (acc_open && touches) {
            new_closed += size_t(1) << acc_bits.size();
            new_acc.clear();
            new_open = false;
          }
        }
        const size_t new_pool = new_closed + (new_open ? (size_t(1) << new_acc.size()) : 0);
        take = !outside && n_high + extra <= mmax && new_kops <= max_ops && new_pool <= pool_cap &&
               (r.taken.empty() || budget < 0 || r.cost + c <= budget);
        if (take) {
          for (int j = 0; j < g.k; ++j)
            if (!g.diag && j != gc && g.t[j] >= Lmin && !r.in_high[g.t[j]]) {
              r.in_high[g.t[j]] = 1;
              ++n_high;
            }
          r.cost += c;
          n_kops = new_kops;
          closed_pool = new_closed;
          acc_bits = new_acc;
          acc_open = new_open;
          r.taken.push_back(gi);
        }
      }
      if (!take) {
        r.deferred.push_back(gi);
        for (int j = 0; j < g.k; ++j) ((g.diag || j == gc) ? block_dense : block_all)[g.t[j]] = 1;
      }
    }
    return r;
  };

  // candidate passes: the unrestricted greedy scan, and one scan per window
  // of consecutive strided qubits; keep the one absorbing the most gates
  auto best_scan = [&](const std::vector<int>& pend) {
    Scan best = scan(pend, nullptr);
    if (mmax > 0 && !opt.no_window_search) {
      std::vector<char> allowed(n, 0);
      for (int a = Lmin; a + mmax <= n; ++a) {
        std::fill(allowed.begin(), allowed.end(), 0);
        for (int q = a; q < a + mmax; ++q) allowed[q] = 1;
        Scan cand = scan(pend, &allowed);
        if (cand.taken.size() > best.taken.size() ||
            (cand.taken.size() == best.taken.size() && cand.cost < best.cost))
          best = std::move(cand);
      }
    }
    return best;
  };
  std::vector<std::vector<int>> taken_of;  // the gates of each emitted pass (circuit order)

  // Lower one scan result to a pass and append it (false + err on failure)
  auto emit = [&](Scan& best) -> bool {
    std::vector<int>& taken = best.taken;
    std::vector<char>& in_high = best.in_high;

    // ---- tile qubit set: low Lmin qubits + chosen high ones, filled upward
    Pass p;
    p.T = T;
    std::vector<char> inq(n, 0);
    for (int q = 0; q < Lmin; ++q) inq[q] = 1;
    int cnt = Lmin;
    for (int q = Lmin; q < n; ++q)
      if (in_high[q]) {
        inq[q] = 1;
        ++cnt;
      }
    for (int q = 0; q < n && cnt < T; ++q)
      if (!inq[q]) {
        inq[q] = 1;
        ++cnt;
      }
    int L = 0;
    while (L < n && inq[L]) ++L;
    if (L > T) L = T;
    p.L = L;
    p.m = 0;
    for (int q = L; q < n; ++q)
      if (inq[q]) p.high[p.m++] = q;
    if (p.L + p.m != T || p.m > kMaxHigh) {
      err = "internal planner error: tile set";
      return false;
    }
    plan_tma(p, n, prec);
    auto local = [&](int q) {
      if (q < p.L) return q;
      for (int b = 0; b < p.m; ++b)
        if (p.high[b] == q) return p.L + b;
      return -1;
    };

    // ---- lower to kernel ops, merging diagonal runs
    // diagonal gates: qubits outside the tile are encoded as T + qubit
    auto dloc = [&](int q) {
      const int l = local(q);
      return l >= 0 ? l : p.T + q;
    };
    auto lower_plain = [&](int gi) {
      const Gate& g = gates[gi];
      if (!g.diag && gctl[gi] >= 0 && local(g.t[gctl[gi]]) < 0) {
        // controlled op, control outside the tile: U0 / U1 on the target
        const int cb = gctl[gi], tb = 1 - cb;
        KernelOp op;
        op.kind = OP_DENSE;
        op.k = 1;
        op.tgt[0] = local(g.t[tb]);
        op.ctlq = g.t[cb];
        op.coeff.assign(8, cd());
        for (int v = 0; v < 2; ++v)
          for (int x = 0; x < 2; ++x)
            for (int y = 0; y < 2; ++y)
              op.coeff[size_t(v) * 4 + x * 2 + y] = g.m[size_t((v << cb) | (x << tb)) * 4 + ((v << cb) | (y << tb))];
        op.gates.push_back(gi);
        return op;
      }
      if (g.diag) {  // sorted table bits (shard bits outside the tile last)
        int tg[kMaxK];
        for (int j = 0; j < g.k; ++j) tg[j] = dloc(g.t[j]);
        DiagAcc one;
        one.absorb(tg, g.k, g.m, gi);
        return one.take();
      }
      KernelOp op;
      op.kind = g.diag ? OP_DIAG : OP_DENSE;
      op.k = g.k;
      for (int j = 0; j < g.k; ++j) op.tgt[j] = local(g.t[j]);
      op.coeff = g.m;
      op.gates.push_back(gi);
      return op;
    };
    std::vector<KernelOp> ops;
    bool merge = !opt.no_diag_merge;
    // c128, on request (no_factor == -1): fused 2q gates as D P (A x B) when
    // that has fewer FMAs (see factor_2q).  Off by default: width-2 fusion of
    // layered circuits also absorbs the NEXT layer's 1q gates, (A' x B') D P
    // (A x B), so only ~1/6 of the gates factor, and the extra ops / diagonal
    // tables made layered-30 c128 slower (374 vs 330 ms measured)
    bool factor = prec == SVB_C128 && opt.no_factor == -1 && merge;
    for (int attempt = 0; attempt < 2 && merge; ++attempt) {
      ops.clear();
      DiagAcc acc;
      for (int gi : taken) {
        const Gate& g = gates[gi];
        int tg[kMaxK];
        for (int j = 0; j < g.k; ++j) tg[j] = g.diag ? dloc(g.t[j]) : local(g.t[j]);
        if (g.diag) {
          if (!acc.empty() && acc.union_size(tg, g.k) > kMaxDiagK) ops.push_back(acc.take());
          acc.absorb(tg, g.k, g.m, gi);
          continue;
        }
        Factor2q fz;
        const bool cx = gctl[gi] >= 0 && local(g.t[gctl[gi]]) < 0;  // control outside the tile
        if (cx) {
          // close an open diagonal run the gate touches on either qubit (the
          // pass scan's op-count and pool model does the same)
          int tt[2] = {local(g.t[1 - gctl[gi]]), dloc(g.t[gctl[gi]])};
          if (!acc.empty() && acc.touches(tt, 2)) ops.push_back(acc.take());
          ops.push_back(lower_plain(gi));
          continue;
        }
        if (factor && g.k == 2 && factor_2q(g.m, fz) && factored_cost(fz) < 16.0) {
          if (!acc.empty() && acc.touches(tg, g.k)) ops.push_back(acc.take());
          for (int side = 0; side < 2; ++side) {
            const bool id = side ? fz.b_id : fz.a_id;
            if (id) continue;
            KernelOp o;
            o.kind = OP_DENSE;
            o.k = 1;
            o.tgt[0] = tg[side];
            o.coeff = side ? fz.B : fz.A;
            o.stype = side ? fz.b_st : fz.a_st;
            o.gates.push_back(gi);
            ops.push_back(o);
          }
          if (fz.perm) {
            KernelOp o;
            o.kind = OP_PERM;
            o.k = 2;
            o.tgt[0] = fz.perm == 1 ? tg[0] : tg[1];  // control
            o.tgt[1] = fz.perm == 1 ? tg[1] : tg[0];  // target
            o.gates.push_back(gi);
            ops.push_back(o);
          }
          // D opens (or joins) a diagonal run
          if (!acc.empty() && acc.union_size(tg, 2) > kMaxDiagK) ops.push_back(acc.take());
          acc.absorb(tg, 2, fz.d, gi);
          continue;
        }
        if (!acc.empty() && acc.touches(tg, g.k)) ops.push_back(acc.take());
        ops.push_back(lower_plain(gi));
      }
      if (!acc.empty()) ops.push_back(acc.take());
      size_t used = 0;
      for (auto& o : ops) used += coeff_elems(o);
      if (used <= pool_cap && int(ops.size()) <= kMaxOps) break;
      if (factor) {
        factor = false;  // factorised ops overflow the pass: retry plain
        continue;
      }
      merge = false;  // merged tables grew past the pool
    }
    if (!merge) {
      ops.clear();
      for (int gi : taken) ops.push_back(lower_plain(gi));
    }
    if (int(ops.size()) > kMaxOps) {
      err = "internal planner error: kernel ops per pass";
      return false;
    }
    p.ops = std::move(ops);
    p.num_gates = int(taken.size());
    plan.passes.push_back(std::move(p));
    taken_of.push_back(taken);
    return true;
  };

  // Kernel choice and phase encoding of one lowered pass (k_gemm_pass layout
  // search, register phases, ...): independent per pass, so it runs for all
  // passes at once on the host's cores after the pass partition is fixed
  // (layered-28 c64 planning 14 -> ~4 ms: the GEMM layout search is ~1 ms
  // per pass)
  auto select_kernel = [&](Pass& p) {
    int n_dense = 0;
    for (const KernelOp& o : p.ops) n_dense += o.kind == OP_DENSE;
    const int min_dense = opt.tc_min_dense > 0 ? opt.tc_min_dense : 2;
    if (use_gemm && p.T == kGemmTileBits && n_dense >= min_dense && build_gemm_pass(p, opt.streams, opt.gemm_warps)) {
      // k_gemm_pass (lowered above)
    } else if (use_mma && opt.streams != 1 && p.T == 12 && build_phases(p, 5, prec, 7)) {
      // 12-qubit tiles: warp groups with their own tile streams (k_reg_pass TB 7)
      fuse_mma_phases(p, opt.tc_min_dense > 0 ? opt.tc_min_dense : 2, kMaxMmaPerPass, prec);
      // four streams by default (measured layered-28 25.0 ms vs 25.8 with
      // three and 29.7 with two: more warp groups hide the per-phase TMEM /
      // MMA / barrier latency; 16 warps keep 128 registers per thread)
      // (a pass without tensor-core phases is HBM-bound: three streams keep
      // more of each SM's shared memory for loads in flight -- single-gate
      // pass 93 % of HBM vs 80 % with four)
      p.streams = opt.streams == 2 ? 2 : opt.streams == 3 ? 3 : opt.streams == 4 ? 4 : (p.mma_phases ? 4 : 3);
    } else if (prec == SVB_C128 && opt.streams != 1 && (opt.reg_bits == 0 || opt.reg_bits == 4) && p.T == 11 &&
               build_phases(p, 4, prec, 7, !std::getenv("SVB_NO_CTRL"))) {
      // c128 default: tile streams of 11-qubit tiles, 16 amplitudes x 128
      // threads each (measured layered-30 395 ms with two vs 422 ms for one
      // stream of 12-qubit tiles: one group's transposes overlap another's
      // FP64 work)
      // three producer-free streams by default (measured layered-30 332 ms vs
      // 379 ms with two, qft-30 121 vs 131 ms)
      p.streams = opt.streams == 2 ? 2 : opt.streams == 4 ? 4 : 3;
    } else {
      int RB = opt.reg_bits > 0 ? opt.reg_bits : default_reg_bits(prec);
      if (p.T < RB + 8) RB = p.T - 8;  // small states: narrower register tile
      if (!opt.no_reg_phases && !build_phases(p, RB, prec, 8, prec == SVB_C128 && !std::getenv("SVB_NO_CTRL"))) {
        p.phases.clear();
        p.reg_ops.clear();
        p.reg_bits = 0;
      } else if (use_mma && p.reg_bits == 5 && p.T == 13) {
        fuse_mma_phases(p, opt.tc_min_dense > 0 ? opt.tc_min_dense : 2, kMaxMmaPerPass, prec);
      }
    }
    p.cost = 0.0;
    for (auto& o : p.ops) p.cost += o.kind == OP_DIAG ? cm.diag(o.k) : cm.dense(o.k);
  };

  // runs of consecutive strided qubits a scan chose (a window search result
  // is one run; scattered random targets give many)
  auto high_runs = [&](const Scan& sc) {
    int runs = 0;
    for (int q = Lbase; q < n; ++q)
      runs += sc.in_high[q] && (q == Lbase || !sc.in_high[q - 1]);
    return runs;
  };
  // The greedy step: the most-gates candidate, or its wide-chunk alternative.
  // Returns the scan and the low-run length it was planned with.
  auto greedy_step = [&](const std::vector<int>& pend) {
    Scan best = best_scan(pend);
    int L_used = Lbase;
    if (Lwide > Lbase) {
      Lmin = Lwide;
      mmax = T - Lmin;
      Scan wide = best_scan(pend);
      // scattered strided qubits (> 2 runs) cost 3-7x the HBM time at 128-B
      // chunks (measured): the wide candidate wins at >= 40 % of the gates;
      // window-shaped candidates keep the default unless it is >= 90 %
      const size_t need = high_runs(best) > 2 ? 4 : 9;
      if (!wide.taken.empty() && wide.taken.size() * 10 >= best.taken.size() * need) {
        best = std::move(wide);
        L_used = Lwide;
      }
      Lmin = Lbase;
      mmax = T - Lmin;
    }
    return std::make_pair(std::move(best), L_used);
  };
  // Pass sequence: a small beam search over the greedy step and every
  // window-shaped candidate (measured on the 1-D layered circuits: the
  // most-gates-now choice can cost a pass later; beam width 4 x 4
  // candidates).  Planning only: the kernels see the same kind of passes.
  std::vector<std::pair<Scan, int>> seq;
  {
    std::vector<int> pend = pending;
    while (!pend.empty()) {
      auto st = greedy_step(pend);
      pend = st.first.deferred;
      seq.push_back(std::move(st));
    }
  }
  // the beam's sequence replaces the greedy one only when it needs fewer
  // passes (same count: the greedy plan, measured no slower)
  const bool use_beam = !opt.no_window_search && mmax > 0 && n >= 20 && gates.size() >= 32 && seq.size() >= 3;
  if (use_beam) {
    struct Node {
      std::vector<int> pend;
      std::vector<std::pair<Scan, int>> path;
      double cost = 0.0;
    };
    std::vector<Node> beam(1);
    beam[0].pend = pending;
    constexpr int kWidth = 4, kCand = 4;
    while (true) {
      const Node* done = nullptr;
      for (const Node& nd : beam)
        if (nd.pend.empty() && (!done || nd.cost < done->cost)) done = &nd;
      if (done) {
        if (done->path.size() < seq.size()) seq = done->path;
        break;
      }
      if (beam[0].path.size() + 1 >= seq.size()) break;  // cannot beat the greedy count
      std::vector<Node> next;
      for (const Node& nd : beam) {
        std::vector<std::pair<Scan, int>> cand;
        cand.push_back(greedy_step(nd.pend));
        std::vector<char> allowed(n, 0);
        for (int a = Lbase; a + mmax <= n; ++a) {
          std::fill(allowed.begin(), allowed.end(), 0);
          for (int q = a; q < a + mmax; ++q) allowed[q] = 1;
          Scan sc = scan(nd.pend, &allowed);
          if (!sc.taken.empty()) cand.push_back(std::make_pair(std::move(sc), Lbase));
        }
        std::stable_sort(cand.begin() + 1, cand.end(), [](const auto& x, const auto& y) {
          return x.first.taken.size() > y.first.taken.size();
        });
        int used = 0;
        for (auto& c : cand) {
          if (c.first.taken.empty() || used++ >= kCand) continue;
          Node ch;
          ch.pend = c.first.deferred;
          ch.cost = nd.cost + c.first.cost;
          ch.path = nd.path;
          ch.path.push_back(c);
          next.push_back(std::move(ch));
        }
      }
      // fewest gates left first; duplicates (same remaining set) collapse
      std::stable_sort(next.begin(), next.end(), [](const Node& x, const Node& y) {
        return x.pend.size() != y.pend.size() ? x.pend.size() < y.pend.size() : x.cost < y.cost;
      });
      beam.clear();
      for (Node& ch : next) {
        bool dup = false;
        for (const Node& b : beam) dup = dup || b.pend == ch.pend;
        if (!dup) beam.push_back(std::move(ch));
        if (int(beam.size()) == kWidth) break;
      }
      if (beam.empty()) {
        err = "internal planner error: empty beam";
        return false;
      }
    }
  }
  for (auto& st : seq) {
    Lmin = st.second;
    mmax = T - Lmin;
    const bool ok = emit(st.first);
    Lmin = Lbase;
    mmax = T - Lmin;
    if (!ok) return false;
  }
  pending.clear();

  // Tail merge: the greedy scan can leave a last pass with a handful of gates
  // (QFT-30 c128 and layered-33 c128 ended with a one-gate pass -- a full HBM
  // round trip for one gate).  Re-plan the gates of the last k passes with the
  // cost budget lifted (the tile, op and coefficient limits still hold) and
  // keep the result when it needs fewer than k passes.
  for (int k = 2; k <= 4 && budget >= 0 && int(plan.passes.size()) >= k; ++k) {
    const size_t P = plan.passes.size();
    if (taken_of[P - 1].size() > taken_of[P - 2].size() / 2 + 2) break;  // no short tail
    std::vector<int> tail;
    for (size_t q = P - k; q < P; ++q) tail.insert(tail.end(), taken_of[q].begin(), taken_of[q].end());
    std::sort(tail.begin(), tail.end());  // circuit order (every scan keeps circuit order)
    budget = -1.0;
    // the first re-planned pass tries every window (the most-gates choice is
    // what left the tail), the rest are greedy
    std::vector<Scan> re;
    std::vector<char> allowed(n, 0);
    for (int a = Lmin - 1; a + mmax <= n && re.empty(); ++a) {
      if (a >= Lmin) {
        std::fill(allowed.begin(), allowed.end(), 0);
        for (int q = a; q < a + mmax; ++q) allowed[q] = 1;
      } else if (mmax == 0 || opt.no_window_search) {
        a = n;  // unrestricted only
      }
      std::vector<Scan> cand{scan(tail, a >= Lmin && a < n ? &allowed : nullptr)};
      while (!cand.back().deferred.empty() && int(cand.size()) < k - 1) cand.push_back(best_scan(cand.back().deferred));
      if (cand.back().deferred.empty()) re = std::move(cand);
    }
    budget = default_budget;
    if (re.empty()) continue;
    std::vector<Pass> keep(std::make_move_iterator(plan.passes.end() - k), std::make_move_iterator(plan.passes.end()));
    std::vector<std::vector<int>> keep_t(taken_of.end() - k, taken_of.end());
    plan.passes.resize(P - k);
    taken_of.resize(P - k);
    bool ok = true;
    for (Scan& sc : re) ok = ok && emit(sc);
    if (!ok) {  // lowering refused a merged pass: restore the originals
      plan.passes.resize(P - k);
      taken_of.resize(P - k);
      for (auto& x : keep) plan.passes.push_back(std::move(x));
      for (auto& x : keep_t) taken_of.push_back(std::move(x));
      err.clear();
    }
    break;
  }
  {
    const int np_ = int(plan.passes.size());
    const int hw = int(std::thread::hardware_concurrency());
    const int nt = std::max(1, std::min({np_, hw > 0 ? hw : 1, 16}));
    if (std::getenv("SVB_PLAN_TIMING")) {
      for (Pass& p : plan.passes) {
        auto t0 = std::chrono::steady_clock::now();
        select_kernel(p);
        auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "select_kernel %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
      }
    } else if (!use_gemm || nt <= 1 || np_ < 4) {  // register-phase encodings are cheap: serial
      for (Pass& p : plan.passes) select_kernel(p);
    } else {
      std::atomic<int> next{0};
      std::vector<std::thread> pool;
      for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
          for (int i = next++; i < np_; i = next++) select_kernel(plan.passes[i]);
        });
      for (auto& th : pool) th.join();
    }
  }
  // outside-tile controls exist only in register-phase kernels: a pass that
  // ended on another kernel re-plans the whole circuit without them
  for (const Pass& ps : plan.passes)
    for (const KernelOp& o : ps.ops)
      if (o.ctlq >= 0 && (ps.phases.empty() || ps.gemm)) {
        if (!ctlx) {
          err = "internal planner error: outside control in a non-register pass";
          return false;
        }
        plan.passes.clear();
        return build_plan_merged(n, prec, gates, opt_in, plan, err, false);
      }
  return true;
}


// ---- peephole gate merge (before pass building)
// Unfused input (the paper's Table-2 circuits: 10n random single-qubit gates,
// run gate by gate by the reference's bench-scaling, ref cli.py:304-337) has
// runs of dense gates on the same qubits.  Each dense gate is multiplied into
// the previous dense gate when that gate is the last one on all of its qubits
// and the union stays <= 2 qubits; a 2-qubit gate also absorbs open 1-qubit
// gates on its qubits.  Diagonal gates are never merge targets (a dense
// factor would make a CP gate need both qubits in the tile).  The product is
// the same operator up to rounding (~1e-16 per merge).
namespace {
// g's matrix acting on the qubit list tgt (g.t a subset of tgt), local bit j <-> tgt[j]
std::vector<cd> expand_on(const Gate& g, const int* tgt, int k) {
  const int D = 1 << k, d = 1 << g.k;
  int pos[kMaxK];
  for (int j = 0; j < g.k; ++j)
    for (int i = 0; i < k; ++i)
      if (tgt[i] == g.t[j]) pos[j] = i;
  int gmask = 0;
  for (int j = 0; j < g.k; ++j) gmask |= 1 << pos[j];
  std::vector<cd> m(size_t(D) * D, cd());
  for (int r = 0; r < D; ++r)
    for (int c = 0; c < D; ++c) {
      if ((r & ~gmask) != (c & ~gmask)) continue;
      int a = 0, b = 0;
      for (int j = 0; j < g.k; ++j) {
        a |= ((r >> pos[j]) & 1) << j;
        b |= ((c >> pos[j]) & 1) << j;
      }
      m[size_t(r) * D + c] = g.diag ? (a == b ? g.m[a] : cd()) : g.m[size_t(a) * d + b];
    }
  return m;
}
std::vector<cd> matmul(const std::vector<cd>& x, const std::vector<cd>& y, int D) {
  std::vector<cd> z(size_t(D) * D, cd());
  for (int r = 0; r < D; ++r)
    for (int q = 0; q < D; ++q) {
      const cd a = x[size_t(r) * D + q];
      if (a == cd()) continue;
      for (int c = 0; c < D; ++c) z[size_t(r) * D + c] += a * y[size_t(q) * D + c];
    }
  return z;
}
}  // namespace

std::vector<Gate> merge_gates(const std::vector<Gate>& in, int n, std::vector<std::vector<int>>& orig) {
  std::vector<Gate> out;
  std::vector<char> dead;
  orig.clear();
  std::vector<int> last(n, -1);  // qubit -> index in `out` of the last gate touching it
  for (size_t i = 0; i < in.size(); ++i) {
    const Gate& g = in[i];
    if (!g.diag && g.k <= 2) {
      const int c = last[g.t[0]];
      bool same = c >= 0 && !out[c].diag;
      for (int j = 1; j < g.k; ++j) same = same && last[g.t[j]] == c;
      if (same) {  // every qubit of g: last touched by the dense gate c
        Gate& h = out[c];
        bool sub = true;  // g's qubits within h's
        for (int j = 0; j < g.k; ++j) sub = sub && std::find(h.t, h.t + h.k, g.t[j]) != h.t + h.k;
        if (sub) {
          h.m = matmul(expand_on(g, h.t, h.k), h.m, 1 << h.k);
          orig[c].push_back(int(i));
          continue;
        }
      }
      if (g.k == 2) {  // absorb open 1q gates on g's qubits
        Gate ng = g;
        std::vector<int> src;
        for (int j = 0; j < 2; ++j) {
          const int c1 = last[g.t[j]];
          if (c1 >= 0 && !out[c1].diag && out[c1].k == 1) {
            ng.m = matmul(ng.m, expand_on(out[c1], g.t, 2), 4);
            dead[c1] = 1;
            src.insert(src.end(), orig[c1].begin(), orig[c1].end());
          }
        }
        if (!src.empty()) {
          std::sort(src.begin(), src.end());
          src.push_back(int(i));
          out.push_back(ng);
          dead.push_back(0);
          orig.push_back(src);
          for (int j = 0; j < 2; ++j) last[g.t[j]] = int(out.size()) - 1;
          continue;
        }
      }
    }
    out.push_back(g);
    dead.push_back(0);
    orig.push_back({int(i)});
    for (int j = 0; j < g.k; ++j) last[g.t[j]] = int(out.size()) - 1;
  }
  std::vector<Gate> res;
  std::vector<std::vector<int>> ores;
  for (size_t i = 0; i < out.size(); ++i)
    if (!dead[i]) {
      res.push_back(std::move(out[i]));
      ores.push_back(std::move(orig[i]));
    }
  orig.swap(ores);
  return res;
}

bool build_plan(int n, int prec, const std::vector<Gate>& gates_in, const svb_plan_options& opt_in,
                Plan& plan, std::string& err) {
  std::vector<std::vector<int>> orig;
  std::vector<Gate> merged;
  if (!opt_in.no_gate_merge) merged = merge_gates(gates_in, n, orig);
  const std::vector<Gate>& gates = opt_in.no_gate_merge ? gates_in : merged;
  if (!build_plan_merged(n, prec, gates, opt_in, plan, err)) {
    // outside-tile controls change the pass partition; if that partition
    // cannot be lowered, plan without them before giving up
    std::string err2;
    plan.passes.clear();
    if (!build_plan_merged(n, prec, gates, opt_in, plan, err2, false)) return false;
    err.clear();
  }
  if (opt_in.no_gate_merge) return true;
  // input-gate indices everywhere (pass_gates, reports, tests)
  auto remap = [&](std::vector<int>& v) {
    std::vector<int> r;
    for (int g : v) r.insert(r.end(), orig[g].begin(), orig[g].end());
    std::sort(r.begin(), r.end());
    v.swap(r);
  };
  for (Pass& p : plan.passes) {
    int ng = 0;
    std::vector<int> seen;
    auto note = [&](const std::vector<int>& v) {
      for (int g : v)
        if (std::find(seen.begin(), seen.end(), g) == seen.end()) seen.push_back(g);
    };
    for (KernelOp& op : p.ops) {
      note(op.gates);
      remap(op.gates);
    }
    for (RegPhase& ph : p.phases) {
      note(ph.tc_gates);
      remap(ph.tc_gates);
    }
    for (int g : seen) ng += int(orig[g].size());
    p.num_gates = ng;
  }
  return true;
}

}  // namespace svb
