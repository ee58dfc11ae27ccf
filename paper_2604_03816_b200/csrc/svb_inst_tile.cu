// Explicit instantiations (see svb_instances.h).
#include "svb_gemmpass.cuh"

namespace svb {
template __global__ void k_tile_pass<float2, 2>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_tile_pass<float2, 3>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_tile_pass<float2, 6>(float2*, const __grid_constant__ PassArgs<float2>);
template __global__ void k_tile_pass<double2, 2>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_tile_pass<double2, 3>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_tile_pass<double2, 6>(double2*, const __grid_constant__ PassArgs<double2>);
}  // namespace svb
