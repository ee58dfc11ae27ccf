// extern "C" entry points of libsvb200.so (declared in include/svb200.h).
//
// Thin host layer: argument validation, plan objects (planner.cpp) turned
// into __grid_constant__ kernel parameter blocks, launch geometry (persistent
// grid = SMs x resident CTAs), error mapping.  No device memory is owned by a
// plan; reductions use a per-device scratch buffer allocated once.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "planner.h"
#include "svb200.h"
#include "svb_kernels.cuh"
#include "svb_regpass.cuh"
#include "svb_instances.h"

using namespace svb;

namespace {

// Shared-window address where a kernel's dynamic shared memory starts (no
// static shared memory here, like the tile-pass kernels).
__global__ void k_smem_base(uint32_t* out) {
  extern __shared__ unsigned char s_dyn[];
  *out = smem_addr(s_dyn);
}

thread_local std::string g_err;
unsigned long long* g_trace = nullptr;  // SVB_GEMM_TRACE buffer (managed memory)

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(SVB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define SVB_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

bool valid_prec(int p) { return p == SVB_C64 || p == SVB_C128; }

struct DeviceFacts {
  int sm_count = 0;
  int max_smem = 0;
  int ctas_per_sm_c64 = 0;
  int ctas_per_sm_c128 = 0;
  uint32_t dyn_smem_base = 0;  // shared-window address of dynamic shared memory
  bool attrs_set = false;
  // reduction scratch (device partials + pinned host copy), allocated once:
  // stream-ordered cudaMallocAsync next to a 100+ GiB torch allocation was
  // measured taking 10-1000 ms per call
  double2* red_dev = nullptr;
  double2* red_host = nullptr;
  long long red_cap = 0;
  std::mutex red_mu;
};
std::mutex g_dev_mu;
DeviceFacts g_dev[64];

int device_facts(DeviceFacts** out) {
  int dev = 0;
  SVB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(SVB_EUNSUPPORTED, "device index out of range");
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceFacts& f = g_dev[dev];
  if (!f.attrs_set) {
    SVB_CUDA(cudaDeviceGetAttribute(&f.sm_count, cudaDevAttrMultiProcessorCount, dev));
    int max_optin = 0;
    SVB_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    f.max_smem = max_optin;
    const void* fns[] = {(const void*)k_tile_pass<float2, 2>,  (const void*)k_tile_pass<float2, 3>,
                         (const void*)k_tile_pass<float2, 6>,  (const void*)k_tile_pass<double2, 2>,
                         (const void*)k_tile_pass<double2, 3>, (const void*)k_tile_pass<double2, 6>,
                         (const void*)k_reg_pass<float2, 3>,   (const void*)k_reg_pass<float2, 4>,
                         (const void*)k_reg_pass<float2, 5>,   (const void*)k_gemm_pass<4, 4, true>,
                         (const void*)k_gemm_pass<4, 4, false>, (const void*)k_gemm_pass<3, 4, true>,
                         (const void*)k_gemm_pass<5, 4, false>,
                         (const void*)k_gemm_pass<2, 4, true>, (const void*)k_gemm_pass<4, 8, true>,
                         (const void*)k_reg_pass<float2, 5, 7>, (const void*)k_reg_pass<double2, 4, 7>,
                         (const void*)k_reg_pass<float2, 5, 7, 3>, (const void*)k_reg_pass<double2, 4, 7, 3>,
                         (const void*)k_reg_pass<double2, 4, 7, 4>,
                         (const void*)k_reg_pass<double2, 4, 7, 3, 1>, (const void*)k_reg_pass<double2, 4, 7, 3, 2>,
                         (const void*)k_reg_pass<float2, 5, 7, 4>,
                         (const void*)k_reg_pass<double2, 3>,  (const void*)k_reg_pass<double2, 4>};
    for (const void* fn : fns)
      SVB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin));
    {  // where dynamic shared memory starts (k_gemm_pass aligns its tiles in that window)
      uint32_t* d = nullptr;
      SVB_CUDA(cudaMalloc(&d, sizeof(uint32_t)));
      k_smem_base<<<1, 1, 1024>>>(d);
      SVB_CUDA(cudaGetLastError());
      SVB_CUDA(cudaMemcpy(&f.dyn_smem_base, d, sizeof(uint32_t), cudaMemcpyDeviceToHost));
      cudaFree(d);
    }
    f.attrs_set = true;
  }
  *out = &f;
  return SVB_OK;
}

template <class C>
void fill_args(const Pass& p, int stages, int n_local_for_args, PassArgs<C>& a, std::vector<C>& ext) {
  std::memset(&a.h, 0, sizeof(a.h));
  a.coeff_ext = nullptr;
  ext.clear();
  // pool elements past the parameter block go to `ext` (global memory at launch)
  constexpr int kParam = kCoeffBytes / int(sizeof(C));
  auto put = [&](int off, const cd& z) {
    C c;
    c.x = static_cast<decltype(c.x)>(z.real());
    c.y = static_cast<decltype(c.x)>(z.imag());
    if (off < kParam) a.coeff[off] = c;
    else ext.push_back(c);
  };
  a.h.T = p.T;
  a.h.L = p.L;
  a.h.m = p.m;
  a.h.n_ops = int(p.ops.size());
  for (int b = 0; b < p.m; ++b) {
    a.h.high[b] = p.high[b];
    a.h.high_sorted[b] = p.high_sorted[b];
  }
  a.h.tma_rank = p.tma_rank;
  a.h.n_enum = p.n_enum;
  for (int d = 0; d < 5; ++d) {
    a.h.tma_start[d] = p.tma_start[d];
    a.h.tma_bits[d] = p.tma_bits[d];
    a.h.tma_box[d] = p.tma_box[d];
  }
  a.h.word_shift = sizeof(C) == 16 ? 1 : 0;
  {  // runs of non-tile bits (ascending), consumed from the tile index low bits up
    std::vector<char> in_tile(64, 0);
    for (int q = 0; q < p.L; ++q) in_tile[q] = 1;
    for (int b = 0; b < p.m; ++b) in_tile[p.high[b]] = 1;
    int src = 0, nr = 0;
    for (int q = 0; q < n_local_for_args;) {
      if (in_tile[q]) {
        ++q;
        continue;
      }
      int len = 0;
      while (q + len < n_local_for_args && !in_tile[q + len]) ++len;
      a.h.gap_src[nr] = src;
      a.h.gap_dst[nr] = q;
      a.h.gap_len[nr] = len;
      ++nr;
      src += len;
      q += len;
    }
    a.h.n_gap_runs = nr;
  }
  a.h.stages = stages;
  a.h.n_phases = int(p.phases.size());
  a.h.reg_bits = p.reg_bits;
  a.h.tc_count = (p.mma_phases || p.gemm) ? int(p.tc_mats.size()) : 0;
  a.h.mma_phases = p.mma_phases ? 1 : 0;
  a.h.thread_bits = p.phases.empty() ? 8 : p.thread_bits;
  a.h.streams = p.phases.empty() ? 1 : p.streams;
  a.h.renorm = p.renorm ? 1 : 0;
  a.h.gemm = p.gemm ? (p.gemm_warps == 8 ? 8 : 4) : 0;
  if (p.gemm) a.h.tc_count = int(p.tc_mats.size());
  a.h.tc_mats = nullptr;
  int off = 0;
  if (!p.phases.empty()) {
    for (size_t f = 0; f < p.phases.size(); ++f) {
      PhaseDesc& d = a.phases[f];
      std::memset(&d, 0, sizeof(d));
      d.op_begin = p.phases[f].op_begin;
      d.op_end = p.phases[f].op_end;
      d.op_mid = p.phases[f].op_mid;
      d.tc = p.phases[f].tc;
      d.flags = p.phases[f].flags;
      for (int i = 0; i < 8; ++i) d.R[i] = p.phases[f].R[i];
      if (p.gemm) std::memcpy(d.R, p.phases[f].wt, sizeof(d.R));  // A word table (16 x u16)
      for (int i = 0; i < 16; ++i) d.map[i] = static_cast<unsigned char>(p.phases[f].map[i]);
    }
    for (size_t i = 0; i < p.reg_ops.size(); ++i) {
      const RegOp& ro = p.reg_ops[i];
      OpDesc& d = a.ops[i];
      std::memset(&d, 0, sizeof(d));
      d.kind = ro.kind;
      d.k = ro.k;
      d.coeff_off = off;
      d.pad = ro.mask;
      if (ro.kind == OP_DENSE && ro.k == 2 && ro.coeff.size() == 16 && !std::getenv("SVB_NO_SPARSE2")) {
        // sparse 2q pattern from the exact zeros (register-local order; see
        // reg_sparse2): monomial forms first, they also fit the 2-column ones
        static const int order[6] = {5, 6, 1, 2, 3, 4};
        for (int pat : order) {
          bool ok = true;
          for (int r = 0; r < 4 && ok; ++r)
            for (int c = 0; c < 4 && ok; ++c)
              if (c != sp_c1(pat, r) && c != sp_c2(pat, r)) ok = ro.coeff[size_t(r) * 4 + c] == cd();
          if (ok) {
            d.kx = pat;
            break;
          }
        }
      }
      if (ro.kind == OP_CTRL) {  // control thread bit, or (srt[0] = -1) shard qubit tgt[0] outside the tile
        d.srt[0] = ro.src[0] >= 0 ? ro.src[0] : -1;
        d.tgt[0] = ro.src[0] >= 0 ? 0 : -1 - ro.src[0];
      }
      if (ro.kind == OP_DIAG) {
        std::memcpy(d.tgt, ro.rmap, sizeof(ro.rmap));
        for (int j = 0; j < ro.mask; ++j) d.srt[j] = ro.src[j];
        d.kx = ro.kx;
        d.rmask = ro.rmask;
        d.xmask = ro.xmask;
        if (ro.kx) a.h.has_outside = 1;
      }
      for (const cd& z : ro.coeff) put(off++, z);
    }
    a.h.coeff_count = off;
    return;
  }
  for (size_t i = 0; i < p.ops.size(); ++i) {
    const KernelOp& ko = p.ops[i];
    OpDesc& d = a.ops[i];
    std::memset(&d, 0, sizeof(d));
    d.kind = ko.kind;
    d.k = ko.k;
    d.coeff_off = off;
    for (int j = 0; j < ko.k; ++j) {
      if (ko.kind == OP_DIAG && ko.tgt[j] >= p.T) {  // shard bit outside the tile
        ++d.kx;
        d.xmask |= 1ULL << (ko.tgt[j] - p.T);
        continue;
      }
      d.tgt[j] = d.srt[j] = ko.tgt[j];
    }
    std::sort(d.srt, d.srt + ko.k - d.kx);
    for (const cd& z : ko.coeff) put(off++, z);
  }
  a.h.coeff_count = off;
}

}  // namespace

struct svb_plan {
  Plan plan;
  int stages = 3;
  std::vector<PassArgs<float2>> args64;
  std::vector<PassArgs<double2>> args128;
  // tensor-core GEMM matrices of every pass, packed for the kernels (host copy
  // built at plan time; uploaded once per device on first execution)
  std::vector<float> tc_host;
  std::vector<size_t> tc_offset;  // per pass, in floats
  float* tc_dev = nullptr;
  int tc_dev_id = -1;
  // coefficient pool past the parameter block, per pass (c128 passes with
  // large diagonal tables); packed host copy, uploaded with the GEMM matrices
  std::vector<unsigned char> ext_host;
  std::vector<size_t> ext_offset;  // per pass, bytes (SIZE_MAX: none)
  unsigned char* ext_dev = nullptr;
  int ext_dev_id = -1;
  // execute_range writes the launch-time fields (tensor map of the state, TMA
  // ring depth) into the cached parameter blocks: one launcher at a time
  std::mutex mu;
  // k_gemm_pass norm accumulators (2 doubles per pass), per (device, stream)
  std::map<std::pair<int, cudaStream_t>, double*> normacc;

  ~svb_plan() {
    if (tc_dev) cudaFree(tc_dev);
    if (ext_dev) cudaFree(ext_dev);
    for (auto& kv : normacc) cudaFree(kv.second);
  }
};

namespace {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor map over the whole shard viewed as 8-byte words, dims as planned.
bool encode_tile_map(const PassHeader& h, void* amps, TensorMapBytes* out) {
  auto enc = tensor_map_encoder();
  if (!enc || h.tma_rank < 1) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  for (int d = 0; d < h.tma_rank; ++d) {
    dims[d] = cuuint64_t(1) << h.tma_bits[d];
    box[d] = 1u << h.tma_box[d];
    estr[d] = 1;
    if (d > 0) strides[d - 1] = (cuuint64_t(1) << h.tma_start[d]) * 8;
  }
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_UINT64, cuuint32_t(h.tma_rank),
                   amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <class C>
int launch_pass(PassArgs<C>& a, int n_local, C* amps, cudaStream_t stream) {
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  if (a.h.n_phases > 0 && a.h.tma_rank > 0 && !encode_tile_map(a.h, amps, &a.tmap)) {
    // tensor map refused (should not happen for planned shapes): 1-D bulk copies
    a.h.tma_rank = 0;
  }
  auto smem_of = [&]() {
    return a.h.n_phases > 0 ? reg_smem_layout<C>(a.h).total : tile_pass_smem_bytes<C>(a.h);
  };
  static_assert(sizeof(PassArgs<C>) <= 32764, "kernel parameter block too large");
  if constexpr (sizeof(C) == 8) {
    if (a.h.gemm) {
      if (a.h.tma_rank < 1) return fail(SVB_EUNSUPPORTED, "k_gemm_pass needs a tensor map");
      static const int dbg = [] {
        const char* e = std::getenv("SVB_GEMM_DEBUG");
        return e ? std::atoi(e) : 0;
      }();
      a.h.debug = dbg;
      static unsigned long long* trace = [] {
        unsigned long long* t = nullptr;
        if (std::getenv("SVB_GEMM_TRACE") && cudaMallocManaged(&t, 128 * sizeof(unsigned long long)) == cudaSuccess)
          std::memset(t, 0, 128 * sizeof(unsigned long long));
        return t;
      }();
      a.h.trace = trace;
      g_trace = trace;
      const int wpg = a.h.gemm == 8 ? 8 : 4;  // warps per tile stream
      int ng = wpg == 8 ? 4 : a.h.streams == 2 ? 2 : a.h.streams == 3 ? 3 : 4;
      // five tile streams (passes with <= 3 GEMMs fit shared memory) only on
      // request, SVB_GEMM_DEBUG bit 2048: measured 16.9 vs 16.4 ms -- the
      // 96-register budget of 640 threads (spills, one TMEM half in flight)
      // costs more than the fifth tile in flight gains
      if (ng == 4 && wpg == 4 && (dbg & 2048)) {
        a.h.gemm_bufs = 5;
        if (gemm_smem_layout(a.h, 5, f->dyn_smem_base).total <= size_t(f->max_smem)) ng = 5;
      }
      // SVB_GEMM_DEBUG bit 256: the 8-MMA (N = 128 hi product) variant, for comparison
      // (measured slower: 17.1 vs 16.2 ms, the doubled TMEM read-out costs more)
      void (*gfn)(float2*, PassArgs<float2>) =
          wpg == 8 ? k_gemm_pass<4, 8, true>
          : ng == 5 ? k_gemm_pass<5, 4, false>
          : ng == 2 ? k_gemm_pass<2, 4, true>
          : ng == 3 ? k_gemm_pass<3, 4, true>
          : (dbg & 256) ? k_gemm_pass<4, 4, true> : k_gemm_pass<4, 4, false>;
      // a spare tile buffer when shared memory allows (loads issued one tile
      // slot ahead; measured neutral at four streams) -- only on request,
      // SVB_GEMM_DEBUG bit 4096
      a.h.gemm_bufs = ng;
      if ((dbg & 4096) && gemm_smem_layout(a.h, ng, f->dyn_smem_base).total <= size_t(f->max_smem)) {
        a.h.gemm_bufs = ng + 1;
        if (gemm_smem_layout(a.h, ng, f->dyn_smem_base).total > size_t(f->max_smem)) a.h.gemm_bufs = ng;
      }
      // a pass whose coefficient pool and GEMM matrices leave no room for four
      // tile buffers runs with three (then two) tile streams
      while (wpg == 4 && ng > 2 && gemm_smem_layout(a.h, ng, f->dyn_smem_base).total > size_t(f->max_smem)) {
        ng = ng == 5 ? 4 : ng - 1;
        a.h.gemm_bufs = ng;
        gfn = ng == 4 ? k_gemm_pass<4, 4, false> : ng == 3 ? k_gemm_pass<3, 4, true> : k_gemm_pass<2, 4, true>;
      }
      const size_t smem_g = gemm_smem_layout(a.h, ng, f->dyn_smem_base).total;
      if (smem_g > size_t(f->max_smem)) return fail(SVB_EUNSUPPORTED, "gemm pass exceeds shared memory");
      long long grid = std::min<long long>(a.h.n_tiles, (long long)f->sm_count);
      if (grid < 1) grid = 1;
      gfn<<<(unsigned)grid, ng * wpg * 32, smem_g, stream>>>(reinterpret_cast<float2*>(amps),
                                                       reinterpret_cast<const PassArgs<float2>&>(a));
      SVB_CUDA(cudaGetLastError());
      return SVB_OK;
    }
  }
  void (*fn)(C*, PassArgs<C>);
  if (a.h.n_phases > 0) {
    if constexpr (sizeof(C) == 8) {
      if (a.h.reg_bits < 3 || a.h.reg_bits > 5) return fail(SVB_EUNSUPPORTED, "c64 reg_bits must be 3..5");
      if (a.h.thread_bits == 7 && a.h.reg_bits != 5) return fail(SVB_EUNSUPPORTED, "two-stream tiles need reg_bits 5");
      fn = a.h.thread_bits == 7 ? (a.h.streams == 4 ? k_reg_pass<C, 5, 7, 4>
                                   : a.h.streams == 3 ? k_reg_pass<C, 5, 7, 3> : k_reg_pass<C, 5, 7>)
           : a.h.reg_bits == 5  ? k_reg_pass<C, 5>
           : a.h.reg_bits == 4  ? k_reg_pass<C, 4>
                                : k_reg_pass<C, 3>;
    } else {
      if (a.h.reg_bits < 3 || a.h.reg_bits > 4 || (a.h.thread_bits == 7 && a.h.reg_bits != 4))
        return fail(SVB_EUNSUPPORTED, "c128 reg_bits must be 3..4 (two streams: 4)");
      // sparse 2q patterns (OpDesc.kx, fill_args): the three-stream kernel
      // with only the controlled-U forms unless the pass holds others
      int sp = 0;
      for (int i = 0; i < a.h.n_ops; ++i)
        if (a.ops[i].kind == OP_DENSE && a.ops[i].k == 2) sp = std::max(sp, a.ops[i].kx == 0 ? 0 : a.ops[i].kx <= 2 ? 1 : 2);
      fn = a.h.thread_bits == 7 ? (a.h.streams == 4   ? k_reg_pass<C, 4, 7, 4>
                                   : a.h.streams == 3 ? (sp == 2 ? k_reg_pass<C, 4, 7, 3, 2> : k_reg_pass<C, 4, 7, 3, 1>)
                                                      : k_reg_pass<C, 4, 7>)
           : a.h.reg_bits == 4  ? k_reg_pass<C, 4>
                                : k_reg_pass<C, 3>;
    }
  } else {
    int kmax = 0;
    for (int i = 0; i < a.h.n_ops; ++i)
      if (a.ops[i].kind == OP_DENSE) kmax = std::max(kmax, a.ops[i].k);
    fn = kmax <= 2 ? k_tile_pass<C, 2> : kmax <= 3 ? k_tile_pass<C, 3> : k_tile_pass<C, 6>;
  }
  // k_reg_pass: 128 threads per tile stream (7 thread bits) or 256, + producer warp
  // (three streams have no producer warp: each loads its own tiles)
  const int block = a.h.n_phases > 0 && a.h.thread_bits == 7 && a.h.streams >= 3 ? a.h.streams * 128 : kThreads;
  if (a.h.stages == 0) {
    // Automatic TMA ring depth: the deepest ring that keeps the CTAs per SM of
    // a 2-stage ring (measured: resident warps matter more than ring depth --
    // qft-30 c128 141 ms at 2 stages / 2 CTAs vs 192 ms at 3 stages / 1 CTA).
    a.h.stages = 2;
    int occ2 = 0, occ = 0;
    SVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, fn, block, smem_of()));
    while (a.h.stages < 6) {
      ++a.h.stages;
      occ = 0;
      if (smem_of() <= size_t(f->max_smem))
        SVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem_of()));
      if (occ < occ2) {
        --a.h.stages;
        break;
      }
    }
  }
  // deepest TMA ring that fits the opt-in shared memory (>= 2 stages); two
  // tile streams (7 thread bits) own alternate stages, so the ring is even
  while (a.h.stages > 2 && smem_of() > size_t(f->max_smem)) --a.h.stages;
  if (a.h.n_phases > 0 && a.h.thread_bits == 7) {  // stage s belongs to stream s % streams
    const int g = a.h.streams >= 3 ? a.h.streams : 2;
    // 3-4 producer-free streams: one stage each; SVB_REG_STAGES=2 gives each
    // two (the next tile loads while this one computes) when shared memory
    // allows
    static const int per = [] {
      const char* e = std::getenv("SVB_REG_STAGES");
      return e ? std::max(1, std::min(2, std::atoi(e))) : 1;  // measured neutral (qft-30: 133 vs 132 ms)
    }();
    a.h.stages = a.h.streams >= 3 ? a.h.streams * per : std::max(g, a.h.stages / g * g);
    while (a.h.stages > g && smem_of() > size_t(f->max_smem)) a.h.stages -= g;
  }
  const size_t smem = smem_of();
  if (a.h.n_tiles >= (1LL << 31)) return fail(SVB_EUNSUPPORTED, "more than 2^31 tiles per shard");
  int per_sm = 0;
  SVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
  if (per_sm < 1) return fail(SVB_EUNSUPPORTED, "tile pass does not fit on an SM (shared memory)");
  const long long n_tiles = a.h.n_tiles;
  long long grid = std::min<long long>(n_tiles, (long long)f->sm_count * per_sm);
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, block, smem, stream>>>(amps, a);
  SVB_CUDA(cudaGetLastError());
  (void)n_local;
  return SVB_OK;
}

// mma.sync m16n8k16 B fragments of the real block form of a 32x32 complex
// phase matrix U (v_out = U v_in): B[2i + a][2j + b] with
// B[2i][2j] = Re U[j][i], B[2i+1][2j] = -Im U[j][i], B[2i][2j+1] = Im U[j][i],
// B[2i+1][2j+1] = Re U[j][i]; split B = Bh + Bl (fp16, round to nearest).
// Fragment (nt, kk), lane = 4 g + c: b0 = B[16kk + 2c + {0,1}][8nt + g],
// b1 = B[16kk + 8 + 2c + {0,1}][8nt + g] (lower k in the low half).
void pack_mma(const std::vector<cd>& U, std::vector<float>& out) {
  auto Bv = [&](int k, int n) -> double {
    const int i = k >> 1, a = k & 1, j = n >> 1, b = n & 1;
    const cd u = U[size_t(j) * 32 + i];
    if (a == 0) return b == 0 ? u.real() : u.imag();
    return b == 0 ? -u.imag() : u.real();
  };
  auto split = [](double x, uint16_t& h, uint16_t& l) {
    const float f = float(x);
    const __half hh = __float2half_rn(f);
    const __half ll = __float2half_rn(f - __half2float(hh));
    std::memcpy(&h, &hh, 2);
    std::memcpy(&l, &ll, 2);
  };
  const size_t base = out.size();
  out.resize(base + kMmaMatBytes / 4);
  uint32_t* w = reinterpret_cast<uint32_t*>(out.data() + base);
  for (int nt = 0; nt < 8; ++nt)
    for (int kk = 0; kk < 4; ++kk)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, c = lane & 3, n = 8 * nt + g;
        uint16_t h[4], l[4];
        split(Bv(16 * kk + 2 * c, n), h[0], l[0]);
        split(Bv(16 * kk + 2 * c + 1, n), h[1], l[1]);
        split(Bv(16 * kk + 8 + 2 * c, n), h[2], l[2]);
        split(Bv(16 * kk + 8 + 2 * c + 1, n), h[3], l[3]);
        uint32_t* q = w + ((nt * 4 + kk) * 32 + lane) * 4;
        q[0] = uint32_t(h[0]) | (uint32_t(h[1]) << 16);
        q[1] = uint32_t(h[2]) | (uint32_t(h[3]) << 16);
        q[2] = uint32_t(l[0]) | (uint32_t(l[1]) << 16);
        q[3] = uint32_t(l[2]) | (uint32_t(l[3]) << 16);
      }
}

// tcgen05 (kind::f16, K-major, SWIZZLE_NONE) B operand of the same block form:
// [Bh | Bl], 64 (n) x 64 (k) fp16 each, byte offset
// (n / 8) 1024 + (k / 8) 128 + (n % 8) 16 + (k % 8) 2.
void pack_t5(const std::vector<cd>& U, std::vector<float>& out) {
  auto Bv = [&](int k, int n) -> double {
    const int i = k >> 1, a = k & 1, j = n >> 1, b = n & 1;
    const cd u = U[size_t(j) * 32 + i];
    if (a == 0) return b == 0 ? u.real() : u.imag();
    return b == 0 ? -u.imag() : u.real();
  };
  const size_t base = out.size();
  out.resize(base + kMmaMatBytes / 4);
  unsigned char* w = reinterpret_cast<unsigned char*>(out.data() + base);
  for (int n = 0; n < 64; ++n)
    for (int k = 0; k < 64; ++k) {
      const float f = float(Bv(k, n));
      const __half hh = __float2half_rn(f);
      const __half ll = __float2half_rn(f - __half2float(hh));
      const size_t off = size_t(n / 8) * 1024 + size_t(k / 8) * 128 + size_t(n % 8) * 16 + size_t(k % 8) * 2;
      std::memcpy(w + off, &hh, 2);
      std::memcpy(w + 8192 + off, &ll, 2);
    }
}

void pack_tc(svb_plan* p) {
  p->tc_host.clear();
  p->tc_offset.assign(p->plan.passes.size(), 0);
  for (size_t i = 0; i < p->plan.passes.size(); ++i) {
    const Pass& ps = p->plan.passes[i];
    p->tc_offset[i] = p->tc_host.size();
    if (ps.mma_phases || ps.gemm) {
      for (const auto& U : ps.tc_mats) {
        if (ps.thread_bits == 7)
          pack_t5(U, p->tc_host);
        else
          pack_mma(U, p->tc_host);
      }
      continue;
    }
  }
}

template <class C>
void point_ext(svb_plan* p, std::vector<PassArgs<C>>& args) {
  for (size_t i = 0; i < args.size(); ++i)
    args[i].coeff_ext = p->ext_offset[i] == SIZE_MAX ? nullptr : reinterpret_cast<const C*>(p->ext_dev + p->ext_offset[i]);
}

int upload_ext(svb_plan* p) {
  if (p->ext_host.empty()) return SVB_OK;
  int dev = 0;
  SVB_CUDA(cudaGetDevice(&dev));
  if (p->ext_dev && p->ext_dev_id == dev) return SVB_OK;
  if (p->ext_dev) cudaFree(p->ext_dev);
  p->ext_dev = nullptr;
  SVB_CUDA(cudaMalloc(&p->ext_dev, p->ext_host.size()));
  SVB_CUDA(cudaMemcpy(p->ext_dev, p->ext_host.data(), p->ext_host.size(), cudaMemcpyHostToDevice));
  p->ext_dev_id = dev;
  point_ext(p, p->args64);
  point_ext(p, p->args128);
  return SVB_OK;
}

int upload_tc(svb_plan* p) {
  if (int rc = upload_ext(p)) return rc;
  if (p->tc_host.empty()) return SVB_OK;
  int dev = 0;
  SVB_CUDA(cudaGetDevice(&dev));
  if (p->tc_dev && p->tc_dev_id == dev) return SVB_OK;
  if (p->tc_dev) cudaFree(p->tc_dev);
  p->tc_dev = nullptr;
  SVB_CUDA(cudaMalloc(&p->tc_dev, p->tc_host.size() * sizeof(float)));
  SVB_CUDA(cudaMemcpy(p->tc_dev, p->tc_host.data(), p->tc_host.size() * sizeof(float), cudaMemcpyHostToDevice));
  p->tc_dev_id = dev;
  for (size_t i = 0; i < p->args64.size(); ++i)
    p->args64[i].h.tc_mats = p->args64[i].h.tc_count ? p->tc_dev + p->tc_offset[i] : nullptr;
  return SVB_OK;
}

template <class C>
int exec_range(svb_plan* p, std::vector<PassArgs<C>>& args, void* amps, int first, int count, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(p->mu);
  if (int rc = upload_tc(p)) return rc;
  double* acc = nullptr;
  if constexpr (sizeof(C) == 8) {
    bool any = false;
    for (const Pass& ps : p->plan.passes) any = any || ps.gemm;
    // SVB_NO_RENORM=1: no deferred renormalisation (and a per-tile scale in
    // every pass) -- exposes the raw fp16-split / fp32-accumulation error
    if (any && !std::getenv("SVB_NO_RENORM")) {
      int dev = 0;
      SVB_CUDA(cudaGetDevice(&dev));
      double*& buf = p->normacc[{dev, s}];
      if (!buf) SVB_CUDA(cudaMalloc(&buf, sizeof(double) * 2 * p->plan.passes.size()));
      acc = buf;
      // a new execution starts from pass 0: fresh accumulators (a range that
      // continues an execution keeps the earlier passes' sums)
      if (first == 0) SVB_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * 2 * p->plan.passes.size(), s));
    }
  }
  for (int i = first; i < first + count; ++i) {
    args[i].h.normacc = acc;
    args[i].h.pass_index = i;
    int rc = launch_pass<C>(args[i], p->plan.n, static_cast<C*>(amps), s);
    if (rc) return rc;
  }
  return SVB_OK;
}

template <class CA, class CB = CA>
int dot_impl(const void* a, const void* b, long long n, double* out2, cudaStream_t s) {
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  const int threads = 512;
  long long grid = std::min<long long>((n + threads - 1) / threads, (long long)f->sm_count * 4);
  if (grid < 1) grid = 1;
  std::lock_guard<std::mutex> lk(f->red_mu);
  if (f->red_cap < grid) {
    if (f->red_dev) cudaFree(f->red_dev);
    if (f->red_host) cudaFreeHost(f->red_host);
    f->red_dev = nullptr;
    f->red_host = nullptr;
    f->red_cap = 0;
    SVB_CUDA(cudaMalloc(&f->red_dev, sizeof(double2) * grid));
    SVB_CUDA(cudaMallocHost(&f->red_host, sizeof(double2) * grid));
    f->red_cap = grid;
  }
  k_dot<CA, CB><<<(unsigned)grid, threads, 0, s>>>(static_cast<const CA*>(a), static_cast<const CB*>(b), n,
                                                  f->red_dev);
  SVB_CUDA(cudaGetLastError());
  SVB_CUDA(cudaMemcpyAsync(f->red_host, f->red_dev, sizeof(double2) * grid, cudaMemcpyDeviceToHost, s));
  SVB_CUDA(cudaStreamSynchronize(s));
  double re = 0.0, im = 0.0;
  for (long long i = 0; i < grid; ++i) {
    re += f->red_host[i].x;
    im += f->red_host[i].y;
  }
  out2[0] = re;
  out2[1] = im;
  return SVB_OK;
}

}  // namespace

extern "C" {

int svb_abi_version(void) { return SVB_ABI_VERSION; }

int svb_debug_trace(unsigned long long* out, int n) {
  if (!out || n < 0) return fail(SVB_EINVAL, "bad argument");
  if (!g_trace) return 0;
  cudaDeviceSynchronize();
  const int m = std::min(n, 128);
  std::memcpy(out, g_trace, sizeof(unsigned long long) * m);
  return m;
}

const char* svb_last_error(void) { return g_err.c_str(); }

int svb_device_sm_count(int* out) {
  if (!out) return fail(SVB_EINVAL, "null out");
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  *out = f->sm_count;
  return SVB_OK;
}

int svb_fill_basis(void* amps, int n_local, int prec, long long index_of_one, void* stream) {
  if (!amps) return fail(SVB_EINVAL, "null amplitudes");
  if (n_local < 1 || n_local > 62) return fail(SVB_EINVAL, "num_qubits must be >= 1");
  if (!valid_prec(prec)) return fail(SVB_EINVAL, "bad precision");
  const long long n = 1LL << n_local;
  if (index_of_one >= n) return fail(SVB_EINVAL, "index_of_one outside the shard");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  const long long words = n * (prec == SVB_C64 ? 8 : 16) / 16;
  long long grid = std::min<long long>((words + 255) / 256, (long long)f->sm_count * 8);
  if (grid < 1) grid = 1;
  if (prec == SVB_C64) {
    k_fill_zero<float2><<<(unsigned)grid, 256, 0, s>>>(static_cast<float2*>(amps), n);
    if (index_of_one >= 0) k_set_one<float2><<<1, 1, 0, s>>>(static_cast<float2*>(amps), index_of_one);
  } else {
    k_fill_zero<double2><<<(unsigned)grid, 256, 0, s>>>(static_cast<double2*>(amps), n);
    if (index_of_one >= 0) k_set_one<double2><<<1, 1, 0, s>>>(static_cast<double2*>(amps), index_of_one);
  }
  SVB_CUDA(cudaGetLastError());
  return SVB_OK;
}

int svb_plan_create(int n_local, int prec, int n_ops, const int* op_k, const int* op_targets,
                    const double* op_mats, const svb_plan_options* opts, svb_plan** out) {
  if (!out) return fail(SVB_EINVAL, "null out");
  *out = nullptr;
  if (n_local < 1) return fail(SVB_EINVAL, "num_qubits must be >= 1");
  if (!valid_prec(prec)) return fail(SVB_EINVAL, "bad precision");
  if (n_ops < 0 || (n_ops > 0 && (!op_k || !op_targets || !op_mats)))
    return fail(SVB_EINVAL, "bad gate arrays");
  svb_plan_options o{};
  if (opts) o = *opts;
  std::vector<Gate> gates;
  std::string err;
  if (!make_gates(n_local, n_ops, op_k, op_targets, op_mats, gates, err)) return fail(SVB_EINVAL, err);
  std::unique_ptr<svb_plan> p(new svb_plan());
  if (!build_plan(n_local, prec, gates, o, p->plan, err)) return fail(SVB_EUNSUPPORTED, err);
  p->stages = o.stages > 0 ? std::max(2, std::min(o.stages, 6)) : 0;  // 0: chosen at first launch
  pack_tc(p.get());
  const int np = int(p->plan.passes.size());
  const long long n_tiles = 1LL << (n_local - (np ? p->plan.passes[0].T : 0));
  p->ext_offset.assign(np, SIZE_MAX);
  auto keep_ext = [&](int i, const auto& ext) {
    if (ext.empty()) return;
    p->ext_offset[i] = p->ext_host.size();
    const auto* b = reinterpret_cast<const unsigned char*>(ext.data());
    p->ext_host.insert(p->ext_host.end(), b, b + ext.size() * sizeof(ext[0]));
    while (p->ext_host.size() % 256) p->ext_host.push_back(0);
  };
  if (prec == SVB_C64) {
    p->args64.resize(np);
    std::vector<float2> ext;
    for (int i = 0; i < np; ++i) {
      fill_args<float2>(p->plan.passes[i], p->stages, n_local, p->args64[i], ext);
      p->args64[i].h.n_tiles = n_tiles;
      keep_ext(i, ext);
    }
  } else {
    p->args128.resize(np);
    std::vector<double2> ext;
    for (int i = 0; i < np; ++i) {
      fill_args<double2>(p->plan.passes[i], p->stages, n_local, p->args128[i], ext);
      p->args128[i].h.n_tiles = n_tiles;
      keep_ext(i, ext);
    }
  }
  *out = p.release();
  return SVB_OK;
}

int svb_plan_num_passes(const svb_plan* plan) {
  if (!plan) return fail(SVB_EINVAL, "null plan");
  return int(plan->plan.passes.size());
}

int svb_plan_pass_info(const svb_plan* plan, int pass, svb_pass_info* out) {
  if (!plan || !out) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  std::memset(out, 0, sizeof(*out));
  out->tile_bits = p.T;
  out->low_bits = p.L;
  out->num_high = p.m;
  for (int b = 0; b < p.m; ++b) out->high[b] = p.high[b];
  out->num_kernel_ops = int(p.ops.size());
  out->num_gates = p.num_gates;
  out->est_cost = p.cost;
  out->reg_bits = p.reg_bits;
  out->num_phases = int(p.phases.size());
  out->num_tc = (p.mma_phases || p.gemm) ? int(p.tc_mats.size()) : 0;
  out->kernel = p.gemm ? SVB_KERNEL_GEMM : p.mma_phases ? SVB_KERNEL_REG_TC : p.phases.empty() ? SVB_KERNEL_TILE : SVB_KERNEL_REG;
  out->streams = p.phases.empty() ? 1 : p.streams;
  out->bank_conflicts = p.bank_conflicts;
  return SVB_OK;
}

int svb_plan_phase_tc(const svb_plan* plan, int pass, int phase, int* op_mid, int* tc) {
  if (!plan || !op_mid || !tc) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (phase < 0 || phase >= int(p.phases.size())) return fail(SVB_EINVAL, "phase index out of range");
  *op_mid = p.phases[phase].op_mid;
  *tc = p.phases[phase].tc;
  return SVB_OK;
}

int svb_plan_tc_matrix(const svb_plan* plan, int pass, int tc, double* out, int cap) {
  if (!plan || !out) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (tc < 0 || tc >= int(p.tc_mats.size())) return fail(SVB_EINVAL, "tc index out of range");
  const auto& U = p.tc_mats[tc];
  if (int(U.size()) > cap) return fail(SVB_EINVAL, "capacity too small");
  for (size_t e = 0; e < U.size(); ++e) {
    out[2 * e] = U[e].real();
    out[2 * e + 1] = U[e].imag();
  }
  return int(U.size());
}

int svb_plan_phase(const svb_plan* plan, int pass, int phase, int* R, int* op_begin, int* op_end, int* flags) {
  if (!plan || !R || !op_begin || !op_end || !flags) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (phase < 0 || phase >= int(p.phases.size())) return fail(SVB_EINVAL, "phase index out of range");
  const RegPhase& ph = p.phases[phase];
  for (int i = 0; i < 8; ++i) R[i] = ph.R[i];
  *op_begin = ph.op_begin;
  *op_end = ph.op_end;
  *flags = ph.flags;
  return SVB_OK;
}

int svb_plan_phase_op(const svb_plan* plan, int pass, int i, int* kind, int* k, int* mask, int* src,
                      double* coeffs, int coeff_cap) {
  if (!plan || !kind || !k || !mask || !src) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (i < 0 || i >= int(p.reg_ops.size())) return fail(SVB_EINVAL, "op index out of range");
  const RegOp& op = p.reg_ops[i];
  *kind = op.kind;
  *k = op.k;
  *mask = op.mask;
  for (int j = 0; j < kMaxK; ++j) src[j] = op.src[j];
  if (op.kind == OP_DIAG) std::memcpy(src + kMaxK, op.rmap, sizeof(op.rmap));  // src[8..15]
  if (coeffs) {
    if (int(op.coeff.size()) > coeff_cap) return fail(SVB_EINVAL, "coefficient capacity too small");
    for (size_t e = 0; e < op.coeff.size(); ++e) {
      coeffs[2 * e] = op.coeff[e].real();
      coeffs[2 * e + 1] = op.coeff[e].imag();
    }
  }
  return int(op.coeff.size());
}

int svb_plan_phase_map(const svb_plan* plan, int pass, int phase, int* map16, int* mma) {
  if (!plan || !map16 || !mma) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (phase < 0 || phase >= int(p.phases.size())) return fail(SVB_EINVAL, "phase index out of range");
  for (int i = 0; i < 16; ++i) map16[i] = p.phases[phase].map[i];
  *mma = p.phases[phase].mma ? 1 : 0;
  return SVB_OK;
}

int svb_plan_phase_op_ext(const svb_plan* plan, int pass, int i, int* kx, unsigned long long* xmask) {
  if (!plan || !kx || !xmask) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (i < 0 || i >= int(p.reg_ops.size())) return fail(SVB_EINVAL, "op index out of range");
  *kx = p.reg_ops[i].kx;
  *xmask = p.reg_ops[i].xmask;
  return SVB_OK;
}

int svb_plan_pass_gates(const svb_plan* plan, int pass, int* out, int cap) {
  if (!plan || !out) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  int w = 0;
  const Pass& ps = plan->plan.passes[pass];
  // a factorised gate (c128 D P (A x B)) is several kernel ops: listed once,
  // at its first op (its ops follow every earlier gate's on shared qubits)
  std::vector<int> seen;
  auto emit = [&](int g) {
    if (std::find(seen.begin(), seen.end(), g) != seen.end()) return true;
    seen.push_back(g);
    if (w >= cap) return false;
    out[w++] = g;
    return true;
  };
  if (ps.phases.empty()) {
    for (const KernelOp& op : ps.ops)
      for (int g : op.gates)
        if (!emit(g)) return fail(SVB_EINVAL, "output capacity too small");
    return w;
  }
  for (const RegPhase& ph : ps.phases) {
    for (int i = ph.op_begin; i < ph.op_mid; ++i)
      for (int g : ps.ops[i].gates)
        if (!emit(g)) return fail(SVB_EINVAL, "output capacity too small");
    for (int g : ph.tc_gates)
      if (!emit(g)) return fail(SVB_EINVAL, "output capacity too small");
    for (int i = ph.op_mid; i < ph.op_end; ++i)
      for (int g : ps.ops[i].gates)
        if (!emit(g)) return fail(SVB_EINVAL, "output capacity too small");
  }
  return w;
}

int svb_plan_kernel_op(const svb_plan* plan, int pass, int i, int* kind, int* k, int* tile_targets,
                       double* coeffs, int coeff_cap) {
  if (!plan || !kind || !k || !tile_targets) return fail(SVB_EINVAL, "null argument");
  if (pass < 0 || pass >= int(plan->plan.passes.size())) return fail(SVB_EINVAL, "pass index out of range");
  const Pass& p = plan->plan.passes[pass];
  if (i < 0 || i >= int(p.ops.size())) return fail(SVB_EINVAL, "op index out of range");
  const KernelOp& op = p.ops[i];
  *kind = op.ctlq >= 0 ? OP_CTRL : op.kind;  // controlled op, control = shard qubit tile_targets[1]
  *k = op.k;
  for (int j = 0; j < op.k; ++j) tile_targets[j] = op.tgt[j];
  if (op.ctlq >= 0) tile_targets[1] = op.ctlq;
  if (coeffs) {
    if (int(op.coeff.size()) > coeff_cap) return fail(SVB_EINVAL, "coefficient capacity too small");
    for (size_t e = 0; e < op.coeff.size(); ++e) {
      coeffs[2 * e] = op.coeff[e].real();
      coeffs[2 * e + 1] = op.coeff[e].imag();
    }
  }
  return int(op.coeff.size());
}

int svb_plan_execute_range(svb_plan* plan, void* amps, int first_pass, int num_passes, void* stream) {
  if (!plan || !amps) return fail(SVB_EINVAL, "null argument");
  const int np = int(plan->plan.passes.size());
  if (first_pass < 0 || num_passes < 0 || first_pass + num_passes > np)
    return fail(SVB_EINVAL, "pass range out of bounds");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (plan->plan.prec == SVB_C64) return exec_range<float2>(plan, plan->args64, amps, first_pass, num_passes, s);
  return exec_range<double2>(plan, plan->args128, amps, first_pass, num_passes, s);
}

int svb_plan_execute(svb_plan* plan, void* amps, void* stream) {
  if (!plan) return fail(SVB_EINVAL, "null plan");
  return svb_plan_execute_range(plan, amps, 0, int(plan->plan.passes.size()), stream);
}

void svb_plan_destroy(svb_plan* plan) { delete plan; }

int svb_apply_gate(void* amps, int n_local, int prec, int k, const int* targets, const double* matrix,
                   void* stream) {
  if (!amps || !targets || !matrix) return fail(SVB_EINVAL, "null argument");
  if (k < 1 || k > SVB_MAX_TARGETS) return fail(SVB_EINVAL, "bad arity");
  int tg[SVB_MAX_TARGETS] = {0};
  for (int j = 0; j < k; ++j) tg[j] = targets[j];
  svb_plan* p = nullptr;
  int rc = svb_plan_create(n_local, prec, 1, &k, tg, matrix, nullptr, &p);
  if (rc) return rc;
  rc = svb_plan_execute(p, amps, stream);
  svb_plan_destroy(p);
  return rc;
}

int svb_dot(const void* a, const void* b, int n_local, int prec, double* out2, void* stream) {
  if (!a || !b || !out2) return fail(SVB_EINVAL, "null argument");
  if (n_local < 0 || n_local > 62 || !valid_prec(prec)) return fail(SVB_EINVAL, "bad shape");
  const long long n = 1LL << n_local;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return prec == SVB_C64 ? dot_impl<float2>(a, b, n, out2, s) : dot_impl<double2>(a, b, n, out2, s);
}

int svb_dot_mixed(const void* a, int prec_a, const void* b, int prec_b, int n_local, double* out2, void* stream) {
  if (!a || !b || !out2) return fail(SVB_EINVAL, "null argument");
  if (n_local < 0 || n_local > 62 || !valid_prec(prec_a) || !valid_prec(prec_b)) return fail(SVB_EINVAL, "bad shape");
  const long long n = 1LL << n_local;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (prec_a == SVB_C64)
    return prec_b == SVB_C64 ? dot_impl<float2>(a, b, n, out2, s) : dot_impl<float2, double2>(a, b, n, out2, s);
  return prec_b == SVB_C64 ? dot_impl<double2, float2>(a, b, n, out2, s) : dot_impl<double2>(a, b, n, out2, s);
}

int svb_norm2(const void* a, int n_local, int prec, double* out, void* stream) {
  if (!out) return fail(SVB_EINVAL, "null argument");
  double z[2];
  int rc = svb_dot(a, a, n_local, prec, z, stream);
  if (rc) return rc;
  *out = z[0];
  return SVB_OK;
}

int svb_block_sums(const void* amps, int n_local, int prec, int log_block, double* out_device, void* stream) {
  if (!amps || !out_device) return fail(SVB_EINVAL, "null argument");
  if (!valid_prec(prec) || log_block < 0 || log_block > n_local || n_local > 62)
    return fail(SVB_EINVAL, "bad shape");
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long nb = 1LL << (n_local - log_block);
  const unsigned grid = unsigned(std::min<long long>(nb, (long long)f->sm_count * 8));
  if (prec == SVB_C64)
    k_block_sums<float2><<<grid, 256, 0, s>>>(static_cast<const float2*>(amps), nb, log_block, out_device);
  else
    k_block_sums<double2><<<grid, 256, 0, s>>>(static_cast<const double2*>(amps), nb, log_block, out_device);
  SVB_CUDA(cudaGetLastError());
  return SVB_OK;
}

int svb_sample_search(const void* amps, int n_local, int prec, int log_block, const double* block_cum,
                      const double* targets, long long shots, long long* out_indices, void* stream) {
  if (!amps || !block_cum || !targets || !out_indices || shots < 0) return fail(SVB_EINVAL, "bad argument");
  if (!valid_prec(prec) || log_block < 0 || log_block > n_local || n_local > 62)
    return fail(SVB_EINVAL, "bad shape");
  if (shots == 0) return SVB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long nb = 1LL << (n_local - log_block);
  const unsigned grid = unsigned((shots + 255) / 256);
  if (prec == SVB_C64)
    k_sample_search<float2><<<grid, 256, 0, s>>>(static_cast<const float2*>(amps), nb, log_block, block_cum,
                                                 targets, shots, out_indices);
  else
    k_sample_search<double2><<<grid, 256, 0, s>>>(static_cast<const double2*>(amps), nb, log_block, block_cum,
                                                  targets, shots, out_indices);
  SVB_CUDA(cudaGetLastError());
  return SVB_OK;
}

int svb_probabilities(const void* amps, int prec, long long offset, long long count, double* out_device,
                      void* stream) {
  if (!amps || !out_device || offset < 0 || count < 0) return fail(SVB_EINVAL, "bad argument");
  if (!valid_prec(prec)) return fail(SVB_EINVAL, "bad precision");
  if (count == 0) return SVB_OK;
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long long grid = std::min<long long>((count + 255) / 256, (long long)f->sm_count * 8);
  if (prec == SVB_C64)
    k_probabilities<float2><<<(unsigned)grid, 256, 0, s>>>(static_cast<const float2*>(amps) + offset, count,
                                                            out_device);
  else
    k_probabilities<double2><<<(unsigned)grid, 256, 0, s>>>(static_cast<const double2*>(amps) + offset, count,
                                                             out_device);
  SVB_CUDA(cudaGetLastError());
  return SVB_OK;
}

int svb_swap_blocks(void* a, void* b, long long bytes, void* stream) {
  if (!a || !b) return fail(SVB_EINVAL, "null argument");
  if (bytes < 0 || (bytes & 15) || (reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
    return fail(SVB_EINVAL, "swap ranges must be 16-byte aligned multiples of 16 bytes");
  if (bytes == 0) return SVB_OK;
  DeviceFacts* f = nullptr;
  int rc = device_facts(&f);
  if (rc) return rc;
  const long long n = bytes / 16;
  const int threads = 512;
  // 4 CTAs of 512 per SM, each thread 4 pairs in flight: ~64 KB of remote
  // loads outstanding per SM
  long long grid = std::min<long long>((n + 4LL * threads - 1) / (4LL * threads), (long long)f->sm_count * 4);
  if (grid < 1) grid = 1;
  k_swap<4><<<unsigned(grid), threads, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint4*>(a),
                                                                            static_cast<uint4*>(b), n);
  SVB_CUDA(cudaGetLastError());
  return SVB_OK;
}

int svb_enable_peer_access(int device, int peer) {
  int cur = 0;
  SVB_CUDA(cudaGetDevice(&cur));
  if (device == peer) return SVB_OK;
  int can = 0;
  SVB_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return fail(SVB_EUNSUPPORTED, "no peer access between these devices");
  SVB_CUDA(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(SVB_ECUDA, cudaGetErrorString(e));
  return SVB_OK;
}

int svb_ipc_export(const void* ptr, void* handle64, long long* offset) {
  if (!ptr || !handle64 || !offset) return fail(SVB_EINVAL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  // driver entry point fetched at run time: the library must load on hosts
  // without libcuda (the CPU test-suite)
  static PFN_cuMemGetAddressRange_v3020 range_fn = [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    return cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &r) == cudaSuccess &&
                   r == cudaDriverEntryPointSuccess
               ? reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(q)
               : nullptr;
  }();
  if (!range_fn) return fail(SVB_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(SVB_EINVAL, "pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  SVB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle64, &h, 64);
  *offset = static_cast<long long>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return SVB_OK;
}

int svb_ipc_import(const void* handle64, long long offset, void** ptr, void** base) {
  if (!handle64 || !ptr || !base || offset < 0) return fail(SVB_EINVAL, "bad argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void* b = nullptr;
  SVB_CUDA(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
  *base = b;
  *ptr = static_cast<char*>(b) + offset;
  return SVB_OK;
}

int svb_ipc_close(void* base) {
  if (!base) return fail(SVB_EINVAL, "null argument");
  SVB_CUDA(cudaIpcCloseMemHandle(base));
  return SVB_OK;
}

}  // extern "C"
