// Explicit instantiations (see svb_instances.h).
#include "svb_gemmpass.cuh"

namespace svb {
template __global__ void k_reg_pass<double2, 3>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_reg_pass<double2, 4>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_reg_pass<double2, 4, 7>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_reg_pass<double2, 4, 7, 3>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_reg_pass<double2, 4, 7, 3, 1>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_reg_pass<double2, 4, 7, 3, 2>(double2*, const __grid_constant__ PassArgs<double2>);
template __global__ void k_reg_pass<double2, 4, 7, 4>(double2*, const __grid_constant__ PassArgs<double2>);
}  // namespace svb
