// Warp-level candidate selection shared by the multi-valued and the
// max-causes enumerators: top-H′ of register-resident scores by (score desc,
// index asc), bit-exact against the reference's stable_sort
// (truncation.cpp:38-57). Scores come from the fast DMMA product; when the
// H′-th and (H′+1)-th scores are closer than twice the error bound `eps`, the
// band around the threshold is re-scored exactly (`exact(h)`: the oracle's
// left-to-right dot product and score arithmetic) and re-ranked. The result
// is sorted ascending into cand[0..H′).
#pragma once
#include "bsc_kernels.cuh"

namespace bscgpu {

template <int MAXJ, class ExactScore>
__device__ __forceinline__ void warp_select(double (&f)[MAXJ], uint32_t removed, double eps, int H, int HP,
                                            int lane, double* pool_v, int* pool_i, uint32_t* cand,
                                            ExactScore exact) {
  if (HP < H) {
    double t, nv;
    top_k<MAXJ>(f, removed, HP, H, lane, pool_v, pool_i, cand, t, nv);
    if (!(t - nv > 2.0 * eps)) {
      uint32_t rem2 = 0;
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) {
        const int h = lane + 32 * j;
        if (h >= H) {
          rem2 |= 1u << j;
        } else if (f[j] > t + 2.0 * eps) {
          f[j] = INFINITY;
        } else if (f[j] < t - 2.0 * eps) {
          f[j] = -INFINITY;
        } else {
          f[j] = exact(h);
        }
      }
      for (int r = 0; r < HP; ++r) {
        double wv;
        int wi;
        select_round<MAXJ>(f, rem2, lane, wv, wi);
        if ((wi & 31) == lane) rem2 |= 1u << (wi >> 5);
        if (lane == 0) cand[r] = static_cast<uint32_t>(wi);
      }
    }
  } else {
    for (int p = lane; p < HP; p += 32) cand[p] = static_cast<uint32_t>(p);
  }
  __syncwarp();
  // candidates ascending (truncation.cpp:55): rank by count of smaller picks
  uint32_t mine[2] = {0xffffffffu, 0xffffffffu};
  int pos[2] = {-1, -1};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int p = lane + 32 * s;
    if (p < HP) {
      mine[s] = cand[p];
      int rk = 0;
      for (int q = 0; q < HP; ++q) rk += cand[q] < mine[s];
      pos[s] = rk;
    }
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 2; ++s)
    if (pos[s] >= 0) cand[pos[s]] = mine[s];
  __syncwarp();
}

}  // namespace bscgpu
