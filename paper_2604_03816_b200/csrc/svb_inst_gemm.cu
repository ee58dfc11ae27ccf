// Explicit instantiations (see svb_instances.h).
#include "svb_gemmpass.cuh"

namespace svb {
template __global__ void k_gemm_pass<4, 4, true>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_gemm_pass<4, 4, false>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_gemm_pass<5, 4, false>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_gemm_pass<3, 4, true>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_gemm_pass<2, 4, true>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_gemm_pass<4, 8, true>(float2*, const __grid_constant__ PassArgs<float2>);
}  // namespace svb
