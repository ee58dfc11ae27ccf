// Explicit instantiations of the tile-pass kernels, one translation unit per
// group (svb_inst_*.cu) so the library compiles in parallel; svb_capi.cu
// sees only these declarations.
#pragma once
#include "svb_gemmpass.cuh"

namespace svb {
extern template __global__ void k_tile_pass<float2, 2>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_tile_pass<float2, 3>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_tile_pass<float2, 6>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_tile_pass<double2, 2>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_tile_pass<double2, 3>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_tile_pass<double2, 6>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<float2, 3>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_reg_pass<float2, 4>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_reg_pass<float2, 5>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_reg_pass<float2, 5, 7>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_reg_pass<float2, 5, 7, 3>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_reg_pass<float2, 5, 7, 4>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_reg_pass<double2, 3>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<double2, 4>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<double2, 4, 7>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<double2, 4, 7, 3>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<double2, 4, 7, 3, 1>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<double2, 4, 7, 3, 2>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_reg_pass<double2, 4, 7, 4>(double2*, const __grid_constant__ PassArgs<double2>);
extern template __global__ void k_gemm_pass<4, 4, true>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_gemm_pass<4, 4, false>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_gemm_pass<5, 4, false>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_gemm_pass<3, 4, true>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_gemm_pass<2, 4, true>(float2*, const __grid_constant__ PassArgs<float2>);
extern template __global__ void k_gemm_pass<4, 8, true>(float2*, const __grid_constant__ PassArgs<float2>);
}  // namespace svb
