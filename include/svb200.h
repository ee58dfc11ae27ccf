/*
 * svb200.h -- C ABI of the B200 state-vector engine (libsvb200.so).
 *
 * The reference package (aqsim, pure Python/NumPy) has no FFI; its plugin
 * boundary is the Python ``Engine`` class (ref pkg/src/aqsim/engines.py:110-187).
 * This ABI sits *under* that boundary: the Python ``B200Engine``
 * (paper_2604_03816_b200/engine.py) binds it with ctypes, and any other host
 * (C, C++, another FFI) can bind the same symbols.  Each entry point names the
 * reference symbol whose work it replaces.
 *
 * Conventions (identical to the reference):
 *   - amplitudes are interleaved complex (float2 for SVB_C64, double2 for
 *     SVB_C128), 2^n_local contiguous elements, little-endian index: bit t of
 *     the index is (local physical) qubit t;
 *   - a k-qubit matrix is 2^k x 2^k, row-major, interleaved complex128
 *     (re, im doubles), and its local bit j acts on targets[j];
 *     for SVB_C64 states the matrix is rounded to complex64 before use,
 *     exactly as ref engines.py:157 does;
 *   - device pointers are borrowed, never freed or reallocated;
 *   - ``stream`` is a cudaStream_t (NULL = legacy default stream); every call
 *     is stream-ordered and asynchronous unless it returns host data.
 *
 * Errors: every int-returning call returns SVB_OK (0) or a negative status;
 * svb_last_error() returns a thread-local message for the last failure.
 */
#ifndef SVB200_H_
#define SVB200_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVB_ABI_VERSION 2
#define SVB_MAX_TARGETS 8   /* per gate; ref allows any k, fusion emits k <= 3 */

enum svb_precision { SVB_C64 = 0, SVB_C128 = 1 };

enum svb_status {
  SVB_OK = 0,
  SVB_EINVAL = -1,       /* bad argument      -> Python ValueError        */
  SVB_ECUDA = -2,        /* CUDA runtime error -> RuntimeError            */
  SVB_ENOMEM = -3,       /* allocation refused -> AllocationError         */
  SVB_EUNSUPPORTED = -4  /* shape outside what the kernels support        */
};

typedef struct svb_plan svb_plan;

/* Planner knobs; zero-initialise for defaults. */
typedef struct svb_plan_options {
  int tile_bits;        /* qubits per shared-memory tile (0: 13 for c64, 12 for c128) */
  int min_low_bits;     /* contiguous low qubits always in the tile (0: 128-B chunks) */
  int max_ops_per_pass; /* 0: 48 (kernel limit)                                      */
  double cost_budget;   /* modelled compute per pass as a multiple of the pass's HBM
                           time; 0: default (7.0 c64, 5.0 c128), <0: unlimited       */
  int no_diag_merge;    /* 1: do not merge diagonal runs into one table              */
  int stages;           /* TMA pipeline depth per CTA (0: deepest ring that keeps the
                           CTAs per SM of a 2-stage ring)                         */
  int reg_bits;         /* amplitudes per thread = 2^reg_bits (0: 5 for c64, 4 c128) */
  int no_reg_phases;    /* 1: force the shared-memory-per-op kernel (k_tile_pass)    */
  int tensor_cores;     /* c64 only: 0 = default = 1: passes with >= tc_min_dense dense
                           gates run k_gemm_pass (every dense op in tcgen05 GEMMs,
                           both operands in shared memory); 2 = tensor-core phases
                           inside k_reg_pass (A in TMEM / warp-level mma.sync);
                           -1 = FMA pipes only */
  int tc_min_dense;     /* dense gates a phase needs to become a GEMM (0: 2)         */
  int no_window_search; /* 1: plain program-order greedy pass building             */
  int streams;          /* tile streams per CTA for register phases: 2..4 = warp
                           groups of 128 threads (7 thread bits; 3-4 without a
                           producer warp), 1 = one stream of 256; 0 = default
                           (4 for c64 tensor-core phases, 3 for c128)           */
  int gemm_warps;       /* k_gemm_pass warps per tile stream: 4 or 8 (0: default 4) */
  int no_factor;        /* c128: -1 = factor fused 2q gates as D P (A x B) where cheaper
                           (structured 1q ops + CNOT permutation); 0/1 = keep them dense */
  int no_gate_merge;    /* 1: keep every input gate a separate op (default: a dense gate
                           is multiplied into the previous dense gate on the same <= 2
                           qubits when nothing in between touches them) */
} svb_plan_options;

/* Per-pass description (for tests, profiling and the sharded driver). */
typedef struct svb_pass_info {
  int tile_bits;        /* T */
  int low_bits;         /* L: tile = 2^m chunks of 2^L contiguous amplitudes */
  int num_high;         /* m */
  int high[8];          /* physical qubits of tile bits L..L+m-1, ascending */
  int num_kernel_ops;   /* ops the kernel applies (after diagonal merging) */
  int num_gates;        /* input gates covered by this pass */
  double est_cost;      /* planner cost estimate (fraction of HBM time) */
  int reg_bits;         /* > 0: register-phase kernel with 2^reg_bits amps per thread */
  int num_phases;       /* register phases (0 for the shared-memory kernel) */
  int num_tc;           /* phases executed as tensor-core GEMMs */
  int kernel;           /* SVB_KERNEL_TILE / _REG / _REG_TC / _GEMM */
  int streams;          /* tile streams per CTA (warp groups of 128 threads) */
  int bank_conflicts;   /* k_gemm_pass: sum of log2 bank-conflict degrees of the A writes */
} svb_pass_info;

enum {
  SVB_KERNEL_TILE = 0,   /* k_tile_pass: shared-memory ops                         */
  SVB_KERNEL_REG = 1,    /* k_reg_pass: register phases on the FMA pipes            */
  SVB_KERNEL_REG_TC = 2, /* k_reg_pass with tensor-core phases (A in TMEM / mma.sync) */
  SVB_KERNEL_GEMM = 3    /* k_gemm_pass: tcgen05 GEMMs, both operands in shared memory */
};

int svb_abi_version(void);
/* Profiling aid: stage timestamps (clock64) of the last k_gemm_pass launch
   (CTA 0, tile stream 0, first 8 tiles x 16 events) when the process runs
   with SVB_GEMM_TRACE set; returns the number of entries copied (0: off). */
int svb_debug_trace(unsigned long long* out, int n);
const char* svb_last_error(void);

/* Device facts (needs a GPU). */
int svb_device_sm_count(int* out);

/* |basis> preparation -- replaces Engine.init_state (ref engines.py:130-140).
 * Writes 0 everywhere and 1 at index_of_one (pass -1 for an all-zero shard). */
int svb_fill_basis(void* amps, int n_local, int prec, long long index_of_one, void* stream);

/* One gate, one HBM pass -- replaces Engine.apply_gate -> _apply_single /
 * _apply_multi (ref engines.py:152-162, kernels 62-105).  Exactly diagonal
 * matrices take the diagonal kernel path. */
int svb_apply_gate(void* amps, int n_local, int prec, int k, const int* targets,
                   const double* matrix, void* stream);

/* Launch plans -- replace the per-gate loop of Engine.run_circuit
 * (ref engines.py:174-187) for a fused circuit (ref dag.py:177-217 output).
 * op_k[i] = arity of gate i; op_targets holds SVB_MAX_TARGETS ints per gate
 * (first op_k[i] used); op_mats concatenates the 2^k x 2^k complex128
 * matrices (2 * 4^k doubles per gate).  Planning is host-only (no GPU). */
int svb_plan_create(int n_local, int prec, int n_ops, const int* op_k, const int* op_targets,
                    const double* op_mats, const svb_plan_options* opts, svb_plan** out);
int svb_plan_num_passes(const svb_plan* plan);
int svb_plan_pass_info(const svb_plan* plan, int pass, svb_pass_info* out);
/* Input-gate indices of pass `pass`, in the order the kernel applies them. */
int svb_plan_pass_gates(const svb_plan* plan, int pass, int* out, int cap);
/* Kernel op i of pass `pass`: kind 0 dense / 1 diagonal, tile-local targets,
 * coefficients as complex128 (dense 4^k, diagonal 2^k entries). */
int svb_plan_kernel_op(const svb_plan* plan, int pass, int i, int* kind, int* k, int* tile_targets,
                       double* coeffs, int coeff_cap);
/* Register phase `phase` of pass `pass`: R[8] register bits, op range, flags;
 * op_mid / tc describe a tensor-core GEMM between ops [op_begin, op_mid) and
 * [op_mid, op_end) (tc = -1: none). */
int svb_plan_phase(const svb_plan* plan, int pass, int phase, int* R, int* op_begin, int* op_end,
                   int* flags);
int svb_plan_phase_tc(const svb_plan* plan, int pass, int phase, int* op_mid, int* tc);
/* Fused GEMM matrix `tc` of pass `pass` (2^reg_bits x 2^reg_bits complex128,
 * row-major, register-bit order) for tests. */
int svb_plan_tc_matrix(const svb_plan* plan, int pass, int tc, double* out, int cap);
/* Register-phase encoding of kernel op i.  Dense: *mask = register-bit mask.
 * Diagonal: table index = [thread bits | register bits | outside-tile bits];
 * *mask = kt, src[0..kt) = thread bits of table bits 0..kt; src must hold
 * 2 * SVB_MAX_TARGETS ints: src[8..15] viewed as 32 bytes map each rho to
 * the register part of the table index (already shifted by kt). */
int svb_plan_phase_op(const svb_plan* plan, int pass, int i, int* kind, int* k, int* mask, int* src,
                      double* coeffs, int coeff_cap);
/* Thread-local layout of register phase `phase`: map16[i] = tile bit of
 * register-index bit i (i < reg_bits), map16[reg_bits + b] = tile bit of
 * thread-index bit b; *mma = 1 for a tensor-core (mma.sync) GEMM phase. */
int svb_plan_phase_map(const svb_plan* plan, int pass, int phase, int* map16, int* mma);
/* Diagonal op i: the top *kx table-index bits are shard qubits outside the
 * tile (set bits of *xmask, ascending), constant over a tile.  svb_plan_kernel_op
 * reports such a target as tile_bits + qubit. */
int svb_plan_phase_op_ext(const svb_plan* plan, int pass, int i, int* kx, unsigned long long* xmask);
int svb_plan_execute(svb_plan* plan, void* amps, void* stream);
int svb_plan_execute_range(svb_plan* plan, void* amps, int first_pass, int num_passes, void* stream);
void svb_plan_destroy(svb_plan* plan);

/* FP64-accumulated reductions -- replace StateVector.norm_squared
 * (ref circuit.py:200-201) and the overlap inside state_fidelity
 * (ref engines.py:340-346).  Results are written to host memory; the call
 * synchronises `stream`.  out2 = {re, im} of sum conj(a[i]) * b[i]. */
int svb_dot(const void* a, const void* b, int n_local, int prec, double* out2, void* stream);
/* <a|b> with a and b in possibly different precisions, both promoted to
   complex128 as ref engines.py:340-346 (state_fidelity) does. */
int svb_dot_mixed(const void* a, int prec_a, const void* b, int prec_b, int n_local, double* out2, void* stream);
int svb_norm2(const void* a, int n_local, int prec, double* out, void* stream);

/* |amp|^2 as float64 -- replaces StateVector.probabilities (ref circuit.py:203-205)
 * for a slice [offset, offset+count) of the shard. */
int svb_probabilities(const void* amps, int prec, long long offset, long long count,
                      double* out_device, void* stream);

/* Measurement sampling on the device -- replaces the host path of sample /
 * sample_from_probabilities (ref engines.py:307-337): per-block FP64 sums of
 * |amp|^2 (blocks of 2^log_block amplitudes), then for each target x (= the
 * host's Philox draw times the total) the index numpy.searchsorted(cdf, x,
 * side="right") would return, given the inclusive block prefix sums. */
int svb_block_sums(const void* amps, int n_local, int prec, int log_block, double* out_device, void* stream);
int svb_sample_search(const void* amps, int n_local, int prec, int log_block, const double* block_cum,
                      const double* targets, long long shots, long long* out_indices, void* stream);

/* Global-qubit swap between shards -- replaces nothing in the reference (which
 * has no multi-device path); it is the exchange step of the north star's
 * sharding.  Swaps two equal byte ranges in place in ONE
 * kernel: each 16-byte element pair is read and written by one thread, so no
 * staging buffer and no second copy.  `a` and `b` may live on different GPUs
 * (peer access enabled with svb_enable_peer_access, or a peer buffer mapped
 * with svb_ipc_import): the loads/stores of the remote side travel over
 * NVLink.  The kernel runs on the current device's `stream`; bytes % 16 == 0. */
int svb_swap_blocks(void* a, void* b, long long bytes, void* stream);
/* cudaDeviceEnablePeerAccess(peer) from `device` (already-enabled is OK). */
int svb_enable_peer_access(int device, int peer);
/* CUDA IPC of a device buffer between the processes of one node (torchrun
 * ranks): export writes a 64-byte handle of the allocation holding `ptr` and
 * ptr's offset in it; import maps a peer's allocation into this process and
 * returns ptr (base + offset) and the base to close later. */
int svb_ipc_export(const void* ptr, void* handle64, long long* offset);
int svb_ipc_import(const void* handle64, long long offset, void** ptr, void** base);
int svb_ipc_close(void* base);

#ifdef __cplusplus
}
#endif
#endif /* SVB200_H_ */
