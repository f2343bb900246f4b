// Instantiations of the lane-per-point state pass (lane_kernels.cuh), kept in
// their own translation unit: compile-time walks for the BASELINE workloads'
// (H', γ) — c1 (10, 4), c2 (12, 4), c3/c4 (14, 5) — and the run-time-H' walk
// for every other shape with 2 ≤ γ ≤ 6, 2 ≤ H' ≤ 16.
#include "bsc_engine.hpp"
#include "lane_kernels.cuh"
#include "select_kernels.cuh"
#include "finish_slice_kernels.cuh"

namespace bscgpu {

const void* lane_fn(int gamma, int hprime) {
  if (gamma == 4 && hprime == 10) return (const void*)lane_states_fixed_kernel<4, 10, 2>;
  if (gamma == 4 && hprime == 12) return (const void*)lane_states_fixed_kernel<4, 12, 2>;
  if (gamma == 5 && hprime == 14) return (const void*)lane_states_fixed_kernel<5, 14, 1>;
  switch (gamma) {
    case 2: return (const void*)lane_states_kernel<2>;
    case 3: return (const void*)lane_states_kernel<3>;
    case 4: return (const void*)lane_states_kernel<4>;
    case 5: return (const void*)lane_states_kernel<5>;
    default: return (const void*)lane_states_kernel<6>;
  }
}

// the thread-per-point selection pass for H' (2 ≤ H' ≤ 16)
const void* select_fn(int hprime) {
  switch (hprime) {
#define SEL_CASE(v) \
  case v:           \
    return (const void*)select_kernel<v>;
    SEL_CASE(2) SEL_CASE(3) SEL_CASE(4) SEL_CASE(5) SEL_CASE(6) SEL_CASE(7) SEL_CASE(8) SEL_CASE(9)
    SEL_CASE(10) SEL_CASE(11) SEL_CASE(12) SEL_CASE(13) SEL_CASE(14) SEL_CASE(15) SEL_CASE(16)
#undef SEL_CASE
    default:
      return nullptr;
  }
}
int select_smem(int latents) { return select_smem_bytes(latents); }

// the finish pass with the singleton weights of MAXJ·32 ≥ H units in registers
const void* finish_fn(int maxj) {
  switch (maxj) {
    case 1: return (const void*)lane_finish_kernel<1>;
    case 2: return (const void*)lane_finish_kernel<2>;
    case 4: return (const void*)lane_finish_kernel<4>;
    case 6: return (const void*)lane_finish_kernel<6>;
    case 8: return (const void*)lane_finish_kernel<8>;
    case 10: return (const void*)lane_finish_kernel<10>;
    case 12: return (const void*)lane_finish_kernel<12>;
    case 16: return (const void*)lane_finish_kernel<16>;
    case 24: return (const void*)lane_finish_kernel<24>;
    default: return (const void*)lane_finish_kernel<32>;
  }
}

const void* finish_slice_fn(int pt) {
  return pt == 32 ? (const void*)lane_finish_slice_kernel<32> : (const void*)lane_finish_slice_kernel<16>;
}
int finish_slice_smem(int pt, int latents, int hp_padded, int hprime) {
  return finish_slice_smem_bytes(pt, latents, hp_padded, hprime);
}

// warps (32-point tiles) per CTA of lane_fn's kernel
int lane_wpc(int gamma, int hprime) { return gamma == 4 && (hprime == 10 || hprime == 12) ? 2 : 1; }

// dynamic shared memory per CTA
int lane_smem(int gamma, int hprime) {
  const int w = lane_wpc(gamma, hprime);
  if (gamma == 4 && hprime == 10) return w * LaneShape<10, 4>::SLOTS * 256;
  if (gamma == 4 && hprime == 12) return w * LaneShape<12, 4>::SLOTS * 256;
  if (gamma == 5 && hprime == 14) return w * LaneShape<14, 5>::SLOTS * 256;
  return lane_smem_bytes(hprime, gamma);
}

}  // namespace bscgpu
