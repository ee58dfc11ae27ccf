// sm_100a device code of the B200 state-vector engine.
//
// k_tile_pass -- the workhorse: one launch = one HBM pass over the local state
// applying every kernel op of a planned pass (replaces the per-gate numpy
// sweeps of ref engines.py:62-105).  Persistent CTAs (one per SM) walk the
// tiles; a dedicated producer warp moves each tile HBM -> shared memory with
// 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx, SASS UBLKCP) into
// a ring of `stages` buffers and writes finished tiles back with bulk stores,
// while 8 compute warps apply the ops in shared memory.  Loads of tile i+1..
// i+S-1 and the store of tile i-1 overlap the math on tile i.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "svb_types.h"

namespace svb {

// ------------------------------------------------------------------ PTX glue
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the waiting thread is suspended in
// hardware until the phase completes (or the hint expires), so waiting warps
// take no issue slots from the compute warps sharing their scheduler.
__device__ __forceinline__ bool mbar_try_wait_suspend(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  while (!mbar_try_wait_suspend(a, parity)) {
  }
}
// Producer-side wait (same primitive; kept as a separate name for call sites
// that previously backed off with nanosleep).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
// Multi-dimensional TMA load (SASS UTMALDG) of one box into shared memory.
__device__ __forceinline__ void tma_load(void* sdst, const void* tmap, const int* c, int rank, uint64_t* bar) {
  const uint32_t d = smem_addr(sdst), b = smem_addr(bar);
  const uint64_t m = reinterpret_cast<uint64_t>(tmap);
  switch (rank) {
    case 1:
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(d), "l"(m), "r"(c[0]), "r"(b) : "memory");
      break;
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b) : "memory");
      break;
    default:
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
      break;
  }
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------ complex math
__device__ __forceinline__ float2 cfma(float2 m, float2 v, float2 acc) {
  acc.x = fmaf(m.x, v.x, acc.x);
  acc.x = fmaf(-m.y, v.y, acc.x);
  acc.y = fmaf(m.x, v.y, acc.y);
  acc.y = fmaf(m.y, v.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cfma(double2 m, double2 v, double2 acc) {
  acc.x = fma(m.x, v.x, acc.x);
  acc.x = fma(-m.y, v.y, acc.x);
  acc.y = fma(m.x, v.y, acc.y);
  acc.y = fma(m.y, v.x, acc.y);
  return acc;
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <class C>
__device__ __forceinline__ C czero();
template <>
__device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }
template <>
__device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }

__device__ __forceinline__ int insert_zero(int x, int p) { return ((x >> p) << (p + 1)) | (x & ((1 << p) - 1)); }

// ----------------------------------------------------------- op application
// Dense k-qubit op on one shared-memory tile.  Each compute thread owns whole
// groups of 2^K amplitudes (the K target bits varied, others fixed); for
// K <= 2 the matrix lives in registers, otherwise it is read (broadcast) from
// the shared coefficient pool.
template <class C, int K>
__device__ __forceinline__ void tile_dense(C* __restrict__ buf, const OpDesc& op, const C* __restrict__ pool,
                                           int T, int tid) {
  constexpr int D = 1 << K;
  constexpr bool kRegM = K <= 2;
  C M[kRegM ? D * D : 1];
  const C* Ms = pool + op.coeff_off;
  if (kRegM) {
#pragma unroll
    for (int e = 0; e < D * D; ++e) M[e] = Ms[e];
  }
  int off[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    int o = 0;
#pragma unroll
    for (int b = 0; b < K; ++b)
      if ((j >> b) & 1) o |= 1 << op.tgt[b];
    off[j] = o;
  }
  int srt[K];
#pragma unroll
  for (int b = 0; b < K; ++b) srt[b] = op.srt[b];
  const int G = 1 << (T - K);
  for (int g = tid; g < G; g += kComputeThreads) {
    int base = g;
#pragma unroll
    for (int b = 0; b < K; ++b) base = insert_zero(base, srt[b]);
    C v[D];
    if constexpr (K <= 4) {
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = buf[base + off[j]];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        C acc = czero<C>();
#pragma unroll
        for (int j = 0; j < D; ++j) acc = cfma(kRegM ? M[i * D + j] : Ms[i * D + j], v[j], acc);
        buf[base + off[i]] = acc;
      }
    } else {  // rare wide CUSTOM gates: keep code size and compile time bounded
      for (int j = 0; j < D; ++j) v[j] = buf[base + off[j]];
      for (int i = 0; i < D; ++i) {
        C acc = czero<C>();
#pragma unroll 4
        for (int j = 0; j < D; ++j) acc = cfma(Ms[i * D + j], v[j], acc);
        buf[base + off[i]] = acc;
      }
    }
  }
}

// Bits of `x` selected by `mask`, packed ascending (software PEXT).
__device__ __forceinline__ int pext_bits(long long x, unsigned long long mask) {
  int r = 0, b = 0;
  while (mask) {
    const int q = __ffsll((long long)mask) - 1;
    r |= int((x >> q) & 1) << b++;
    mask &= mask - 1;
  }
  return r;
}

// Diagonal op (a merged run of diagonal gates): amp[e] *= table[bits of e at
// tgt | shard bits of the tile origin at xmask].
template <class C>
__device__ __forceinline__ void tile_diag(C* __restrict__ buf, const OpDesc& op, const C* __restrict__ pool,
                                          int T, int tid, long long origin) {
  const C* table = pool + op.coeff_off;
  const int k = op.k - op.kx;
  int tg[kMaxK];
#pragma unroll
  for (int b = 0; b < kMaxK; ++b) tg[b] = b < k ? op.tgt[b] : 0;
  const int dx = op.kx ? pext_bits(origin, op.xmask) << k : 0;
  const int N = 1 << T;
  for (int e = tid; e < N; e += kComputeThreads) {
    int d = dx;
#pragma unroll
    for (int b = 0; b < kMaxK; ++b)
      if (b < k) d |= ((e >> tg[b]) & 1) << b;
    buf[e] = cmul(buf[e], table[d]);
  }
}

// KMAX bounds the dense arity compiled into a kernel variant, so the common
// (fused width <= 2) variant carries no register pressure from wide gates.
// CNOT on tile bits tgt[0] (control) -> tgt[1] (target): swap pairs in place.
template <class C>
__device__ __forceinline__ void tile_perm(C* __restrict__ buf, const OpDesc& op, int T, int tid) {
  const int c = op.tgt[0], t = op.tgt[1];
  const int lo = c < t ? c : t, hi = c < t ? t : c;
  for (int e = tid; e < (1 << (T - 2)); e += kComputeThreads) {
    const int base = insert_zero(insert_zero(e, lo), hi) | (1 << c);
    const C a = buf[base], b = buf[base | (1 << t)];
    buf[base] = b;
    buf[base | (1 << t)] = a;
  }
}

template <class C, int KMAX>
__device__ __forceinline__ void tile_apply(C* buf, const OpDesc& op, const C* pool, int T, int tid,
                                           long long origin) {
  if (op.kind == OP_DIAG) {
    tile_diag<C>(buf, op, pool, T, tid, origin);
    return;
  }
  if (op.kind == OP_PERM) {
    tile_perm<C>(buf, op, T, tid);
    return;
  }
  switch (op.k) {
    case 1: tile_dense<C, 1>(buf, op, pool, T, tid); break;
    case 2: tile_dense<C, 2>(buf, op, pool, T, tid); break;
    case 3: if constexpr (KMAX >= 3) tile_dense<C, 3>(buf, op, pool, T, tid); break;
    case 4: if constexpr (KMAX >= 4) tile_dense<C, 4>(buf, op, pool, T, tid); break;
    case 5: if constexpr (KMAX >= 5) tile_dense<C, 5>(buf, op, pool, T, tid); break;
    default: if constexpr (KMAX >= 6) tile_dense<C, 6>(buf, op, pool, T, tid); break;
  }
}

__device__ __forceinline__ long long tile_base(long long tile, const PassHeader& h) {
  long long g = 0;
  for (int r = 0; r < h.n_gap_runs; ++r)
    g |= ((tile >> h.gap_src[r]) & ((1LL << h.gap_len[r]) - 1)) << h.gap_dst[r];
  return g;
}
__device__ __forceinline__ long long chunk_offset(int c, const PassHeader& h) {
  long long o = 0;
  for (int b = 0; b < h.m; ++b)
    if ((c >> b) & 1) o += 1LL << h.high[b];
  return o;
}

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <class C>
__host__ __device__ inline size_t tile_pass_smem_bytes(const PassHeader& h) {
  return 128 + align_up(size_t(h.coeff_count) * sizeof(C), 128) + size_t(h.stages) * (sizeof(C) << h.T);
}

// ------------------------------------------------------------------ kernel
template <class C, int KMAX>
__global__ void __launch_bounds__(kThreads, 1) k_tile_pass(C* __restrict__ amps, const __grid_constant__ PassArgs<C> args) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const PassHeader& h = args.h;
  const int S = h.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // tile landed   (1 arrival + tx)
  uint64_t* done = full + S;                            // tile computed (256 arrivals)
  C* pool = reinterpret_cast<C*>(smem + 128);
  C* tiles = reinterpret_cast<C*>(smem + 128 + align_up(size_t(h.coeff_count) * sizeof(C), 128));
  const int tile_elems = 1 << h.T;
  const int tid = threadIdx.x;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], kComputeThreads);
    }
    fence_mbar_init();
  }
  for (int e = tid; e < h.coeff_count; e += kThreads) pool[e] = pool_elem(args, e);
  __syncthreads();

  const long long n_tiles = h.n_tiles;
  const long long mine = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (tid >= kComputeThreads) {
    // ---------------- producer warp: TMA bulk loads / stores
    const int lane = tid - kComputeThreads;
    const int n_chunks = 1 << h.m;
    const uint32_t chunk_bytes = uint32_t(sizeof(C)) << h.L;
    const uint64_t pol = policy_evict_first();
    auto tile_of = [&](long long it) { return (long long)blockIdx.x + it * gridDim.x; };
    auto store_tile = [&](long long it) {
      const int s = int(it % S);
      const long long base = tile_base(tile_of(it), h);
      C* buf = tiles + size_t(s) * tile_elems;
      for (int c = lane; c < n_chunks; c += 32)
        bulk_store(amps + base + chunk_offset(c, h), buf + (size_t(c) << h.L), chunk_bytes, pol);
      bulk_commit();
    };
    for (long long it = 0; it < mine; ++it) {
      const int s = int(it % S);
      if (it >= S) {
        mbar_wait(&done[s], uint32_t(((it - S) / S) & 1));
        store_tile(it - S);
        bulk_wait_read_all();  // buffer s drained before it is refilled
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[s], chunk_bytes * uint32_t(n_chunks));
      __syncwarp();
      const long long base = tile_base(tile_of(it), h);
      C* buf = tiles + size_t(s) * tile_elems;
      for (int c = lane; c < n_chunks; c += 32)
        bulk_load(buf + (size_t(c) << h.L), amps + base + chunk_offset(c, h), chunk_bytes, &full[s], pol);
    }
    for (long long it = (mine > S ? mine - S : 0); it < mine; ++it) {
      const int s = int(it % S);
      mbar_wait(&done[s], uint32_t((it / S) & 1));
      store_tile(it);
    }
    bulk_wait_all();
  } else {
    // ---------------- compute warps
    for (long long it = 0; it < mine; ++it) {
      const int s = int(it % S);
      mbar_wait(&full[s], uint32_t((it / S) & 1));
      C* buf = tiles + size_t(s) * tile_elems;
      const long long origin = tile_base((long long)blockIdx.x + it * gridDim.x, h);
      for (int o = 0; o < h.n_ops; ++o) {
        if (o) compute_bar();
        tile_apply<C, KMAX>(buf, args.ops[o], pool, h.T, tid, origin);
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the bulk store
      mbar_arrive(&done[s]);
    }
  }
}

// --------------------------------------------------------------- utilities
template <class C>
__global__ void k_fill_zero(C* __restrict__ amps, long long n_amps) {
  // 16-byte stores: 2 c64 or 1 c128 amplitude per word
  constexpr int per = 16 / sizeof(C);
  const long long words = n_amps / per;
  uint4* w = reinterpret_cast<uint4*>(amps);
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x)
    w[i] = z;
}

template <class C>
__global__ void k_set_one(C* amps, long long one) {
  C v = czero<C>();
  v.x = 1;
  amps[one] = v;
}

// <a|b> partial sums in FP64; a and b may differ in precision (both are
// promoted to complex128 first, as ref engines.py:340-346 promotes states)
// In-place swap of two equal ranges (global-qubit exchange between shards):
// each 16-byte pair is loaded and stored by one thread, either side may be a
// peer GPU's memory (NVLink loads/stores).  Four independent pairs per thread
// per iteration keep enough remote loads in flight to cover NVLink latency.
template <int U = 4>
__global__ void __launch_bounds__(512) k_swap(uint4* __restrict__ a, uint4* __restrict__ b, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = a[i + u * stride];
      y[u] = b[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[i + u * stride] = y[u];
      b[i + u * stride] = x[u];
    }
  }
  for (; i < n; i += stride) {
    const uint4 x = a[i], y = b[i];
    a[i] = y;
    b[i] = x;
  }
}

template <class CA, class CB = CA>
__global__ void k_dot(const CA* __restrict__ a, const CB* __restrict__ b, long long n, double2* __restrict__ partial) {
  double re = 0.0, im = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const CA x = a[i];
    const CB y = b[i];
    const double xr = x.x, xi = x.y, yr = y.x, yi = y.y;
    re += xr * yr + xi * yi;  // conj(x) * y
    im += xr * yi - xi * yr;
  }
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  __shared__ double2 red[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = make_double2(re, im);
  __syncthreads();
  if (w == 0) {
    double2 v = l < (blockDim.x >> 5) ? red[l] : make_double2(0.0, 0.0);
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    if (l == 0) partial[blockIdx.x] = v;
  }
}

// Sum of |amp|^2 (FP64) over each block of 2^lb amplitudes; one CTA per block.
template <class C>
__global__ void k_block_sums(const C* __restrict__ a, long long n_blocks, int lb, double* __restrict__ out) {
  __shared__ double red[32];
  for (long long b = blockIdx.x; b < n_blocks; b += gridDim.x) {
    const C* p = a + (b << lb);
    double acc = 0.0;
    for (int i = threadIdx.x; i < (1 << lb); i += blockDim.x) {
      const double r = p[i].x, m = p[i].y;
      acc += r * r + m * m;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) out[b] = v;
    }
    __syncthreads();
  }
}

// Inverse-CDF search (numpy searchsorted side='right' on the cumulative
// |amp|^2): block by binary search over the inclusive block prefix, then a
// sequential scan inside the block.  One thread per draw.
template <class C>
__global__ void k_sample_search(const C* __restrict__ a, long long n_blocks, int lb,
                                const double* __restrict__ block_cum, const double* __restrict__ x,
                                long long shots, long long* __restrict__ out) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= shots) return;
  const double t = x[s];
  long long lo = 0, hi = n_blocks;  // first block with block_cum > t
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (block_cum[mid] > t) hi = mid; else lo = mid + 1;
  }
  if (lo >= n_blocks) {
    out[s] = (n_blocks << lb) - 1;
    return;
  }
  double cum = lo > 0 ? block_cum[lo - 1] : 0.0;
  const C* p = a + (lo << lb);
  long long idx = (lo << lb) + (1 << lb) - 1;
  for (int i = 0; i < (1 << lb); ++i) {
    const double r = p[i].x, m = p[i].y;
    cum += r * r + m * m;
    if (cum > t) {
      idx = (lo << lb) + i;
      break;
    }
  }
  out[s] = idx;
}

template <class C>
__global__ void k_probabilities(const C* __restrict__ a, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const C x = a[i];
    const double r = x.x, m = x.y;
    out[i] = r * r + m * m;
  }
}

}  // namespace svb
