// Instantiations of the lane-per-point state pass (lane_kernels.cuh), kept in
// their own translation unit: compile-time walks for the BASELINE workloads'
// (H', γ) — c1 (10, 4), c2 (12, 4), c3/c4 (14, 5) — and the run-time-H' walk
// for every other shape with 2 ≤ γ ≤ 6, 2 ≤ H' ≤ 16.
#include "bsc_engine.hpp"
#include "lane_kernels.cuh"

namespace bscgpu {

const void* lane_fn(int gamma, int hprime) {
  if (gamma == 4 && hprime == 10) return (const void*)lane_states_fixed_kernel<4, 10>;
  if (gamma == 4 && hprime == 12) return (const void*)lane_states_fixed_kernel<4, 12>;
  if (gamma == 5 && hprime == 14) return (const void*)lane_states_fixed_kernel<5, 14>;
  switch (gamma) {
    case 2: return (const void*)lane_states_kernel<2>;
    case 3: return (const void*)lane_states_kernel<3>;
    case 4: return (const void*)lane_states_kernel<4>;
    case 5: return (const void*)lane_states_kernel<5>;
    default: return (const void*)lane_states_kernel<6>;
  }
}

int lane_smem(int gamma, int hprime) {
  if (gamma == 4 && hprime == 10) return LaneShape<10, 4>::SLOTS * 256;
  if (gamma == 4 && hprime == 12) return LaneShape<12, 4>::SLOTS * 256;
  if (gamma == 5 && hprime == 14) return LaneShape<14, 5>::SLOTS * 256;
  return lane_smem_bytes(hprime, gamma);
}

}  // namespace bscgpu
