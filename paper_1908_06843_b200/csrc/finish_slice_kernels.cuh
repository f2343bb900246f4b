// Finish pass of the lane path fused with the ⟨S⟩ᵀ slicer (sm_100a).
//
// Reference: the tail of the per-point loop of LinearDiscreteModel::estep_impl
// (linear_discrete.cpp:272-304 at T = 1: log Z, the normalised ⟨s_n⟩, the
// candidate pairs of Σ⟨s sᵀ⟩) and the accumulation of Σ⟨s⟩ (:296-299), whose
// product with Y the int8 tensor-core GEMM of ozaki_gemm.cuh forms.
//
// lane_finish_kernel writes the N × H fp64 ⟨S⟩ rows to HBM and
// oz_slice_cols_kernel reads them back to cut them into int8 slices. Here the
// rows never leave the SM: a CTA owns blocks of 128 consecutive points and
// walks them in sub-tiles of PT points whose rows sit in shared memory
// ([PT][Hp] fp64):
//   phase A  warp per point (as lane_finish_kernel): the B = Y·W row arrives by
//            cp.async and is overwritten in place by the unnormalised singleton
//            weights e^{rel_h − shift}; the candidates' entries take their
//            marginals from the state pass; 1/Z goes to a per-row factor; the
//            candidate pairs go to Σ⟨ssᵀ⟩ in fixed point (pair_fx_add).
//            Points the fallback launch handled arrive as finished ⟨s⟩ rows
//            (factor 1); rows past N are zero.
//   phase B  thread per (unit h, 16 points): the values of column h, scaled by their
//            row factors, are cut into the 8 base-128 digits of ⌊x·2⁵⁶/scale⌋
//            (x ≥ 0: no sign), transposed with byte permutes and stored as 16
//            contiguous bytes per slice — the K-blocked operand layout
//            [slice][point/64][h][64] of the Yᵀ⟨S⟩ GEMM — while the column sums
//            Σ_n⟨s_nh⟩ of the 128-point block accumulate in a fixed order.
// HBM traffic per point: the B row in (8·Hp B), the slices out (8·Hp B).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lane_kernels.cuh"

namespace bscgpu {

struct FinishSliceArgs {
  FinishArgs f;            // f.ES: rows the fallback launch wrote for its points
  int8_t* ess;             // ⟨S⟩ᵀ slices [8][npc/64][Hp][64]
  long long slice_stride;  // Hp · npc
  double* colsum;          // [blocks of 128 points][Hp]
  double inv56;            // 2⁵⁶ / slice scale (a power of two)
};


constexpr int kFsBlock = 128;  // points per column-sum block (oz_colsum_reduce_kernel's rows)

// threads per CTA: 256 with 32-point sub-tiles (two CTAs per SM), 512 with the 16-point sub-tiles of
// H > 800 (one CTA per SM fits: 16 warps instead of 8)
__host__ __device__ constexpr int fs_threads(int pt) { return pt == 32 ? 256 : 512; }

__host__ __device__ inline int finish_slice_smem_bytes(int pt, int H, int Hp, int hp) {
  // ⟨S⟩ tile, diag(G), row factors, pq, per-warp Σ log Z, and the sub-tile's lane outputs [field][pt + 2]
  return 8 * (pt * Hp + ((H + 1) & ~1) + pt) + 512 + 8 * (fs_threads(pt) / 32) + 8 * lane_out_fields(hp) * (pt + 2);
}

// the four 7-bit digits of t (< 2²⁸) spread to the bytes of a word, digit k at byte k
__device__ __forceinline__ uint32_t spread7(uint32_t t) {
  return (t & 0x7fu) | ((t << 1) & 0x7f00u) | ((t << 2) & 0x7f0000u) | ((t << 3) & 0x7f000000u);
}

template <int PT>
__global__ void __launch_bounds__(fs_threads(PT), PT == 32 ? 2 : 1) lane_finish_slice_kernel(FinishSliceArgs a) {
  constexpr int kFsThreads = fs_threads(PT);
  static_assert(PT == 32 || PT == 16, "sub-tile of 16 or 32 points");
  constexpr int NW = kFsThreads / 32, RPW = PT / NW;  // rows per warp and sub-tile
  constexpr int NH = PT / 16;                         // 16-point halves per unit and sub-tile (phase B items)
  // phase B passes: the 32-point variant is only taken while its tile fits beside a second CTA's
  // (Hp ≤ ~800), the 16-point variant covers Hp ≤ 1024
  constexpr int ITS = PT == 32 ? 7 : 2;
  extern __shared__ __align__(16) double fsm[];
  const FinishArgs& f = a.f;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int H = f.H, Hp = f.Hp, hp = f.hp, nm = hp * (hp + 1) / 2;
  double* tile = fsm;                          // [PT][Hp]
  double* gd = tile + PT * Hp;                 // diag(G)
  double* rs = gd + ((H + 1) & ~1);            // per-row factor (1/Z, 1, or 0)
  uint16_t* pq = reinterpret_cast<uint16_t*>(rs + PT);  // moment entry o → (p, q)
  double* red = reinterpret_cast<double*>(pq + 256);
  // the sub-tile's lane-pass outputs (shift, Σ multi-active weights, moments), staged [field][PT + 2]:
  // a point's fields sit 256 bytes apart in the [field][32 points] tiles of the lane pass, so reading
  // them per point from global memory cost 32 L1 wavefronts per load instruction
  constexpr int MP = PT + 2;
  double* momt = red + NW;
  const int nf = lane_out_fields(hp);
  for (int i = threadIdx.x; i < H; i += kFsThreads) gd[i] = f.gdiag[i];
  for (int o = threadIdx.x; o < nm; o += kFsThreads) {
    int idx = o, p = 0;
    while (idx >= hp - p) {
      idx -= hp - p;
      ++p;
    }
    pq[o] = static_cast<uint16_t>(p | ((p + idx) << 8));
  }
  __syncthreads();
  const long long nblk = (static_cast<long long>(f.N) + kFsBlock - 1) / kFsBlock;
  const int row16 = Hp / 2;  // 16-byte pieces per row
  double lse_acc = 0.0;
  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    double cs[ITS];  // column sums of the items this thread owns
#pragma unroll
    for (int it = 0; it < ITS; ++it) cs[it] = 0.0;
    for (int st = 0; st < kFsBlock / PT; ++st) {
      const long long n0 = blk * kFsBlock + st * PT;
      // ---- phase A: this warp's rows r = wib + NW·i
      int mode[RPW];
      if (n0 < f.N) {  // (a sub-tile wholly past the chunk only pads the slices: its lane tile does not exist)
        const double* src = f.out + (n0 >> 5) * nf * 32 + (n0 & 31);
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(momt));
        for (int idx = threadIdx.x; idx < nf * (PT / 2); idx += kFsThreads) {
          const int fld = idx / (PT / 2), pc = idx % (PT / 2);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + (fld * MP + 2 * pc) * 8),
                       "l"(src + fld * 32 + 2 * pc)
                       : "memory");
        }
      }
      double y2v[RPW];
#pragma unroll
      for (int i = 0; i < RPW; ++i) {  // (all of this warp's modes and ‖y‖² in flight before the first is used)
        const long long n = n0 + wib + NW * i;
        mode[i] = n < f.N ? f.pmode[n] : -1;
        y2v[i] = n < f.N ? f.y2[n] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int r = wib + NW * i;
        const long long n = n0 + r;
        if (n < f.N) {
          const bool lanept = mode[i] == kModeShift || mode[i] == kModeMax;
          const double* src = (lanept ? f.B : f.ES) + n * Hp;
          const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(tile + r * Hp));
          for (int c = lane; c < row16; c += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + c * 16), "l"(src + 2 * c) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      // this warp's rows of the CTA's next sub-tile: on their way into L2 meanwhile
      const long long nn0 = st + 1 < kFsBlock / PT ? n0 + PT : (blk + gridDim.x) * kFsBlock;
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const long long n = nn0 + wib + NW * i;
        if (n < f.N)
          for (int l = lane; l < (Hp * 8 + 127) / 128; l += 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(f.B + n * Hp + l * 16));
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // (the lane outputs were fetched by all threads)
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int r = wib + NW * i;
        const long long n = n0 + r;
        double* row = tile + r * Hp;
        if (mode[i] < 0) {  // past the chunk: a zero row
          for (int h = lane; h < Hp; h += 32) row[h] = 0.0;
          if (lane == 0) rs[r] = 0.0;
          continue;
        }
        if (mode[i] != kModeShift && mode[i] != kModeMax) {  // finished by the fallback launch
          if (lane == 0) rs[r] = 1.0;
          continue;
        }
        const double shift = momt[r], zm = momt[MP + r];
        const uint32_t cmine = lane < hp ? f.cand[n * hp + lane] : 0u;
        // (Dropping the weights below e^-48 of the point's largest and compacting the rest by
        // ballot was measured slower — early EM iterations keep most units inside the window —
        // profiles/r02_variants.txt.)
        double zs = 0.0;
#pragma unroll 4
        for (int h = lane; h < H; h += 32) {
          // rel = fma(inv2s, 2b − G_hh, dlp), the selection pass's rounding: shift ≥ rel
          const double e = exp_nonpos_ftz(__fma_rn(f.inv2s, __fma_rn(2.0, row[h], -gd[h]), f.dlp) - shift);
          row[h] = e;
          zs += e;
        }
        zs = warp_sum(zs) + exp_nonpos(-shift);  // + the zero state
        const double z1 = zs + zm;
        const double inv_z = 1.0 / z1;
        if (lane == 0) {
          lse_acc += (f.base0 - y2v[i] * f.inv2s) + (shift + log(z1));
          rs[r] = inv_z;
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          const int o = lane + 32 * t;
          if (32 * t >= nm) break;  // (warp-uniform)
          const bool on = o < nm;
          const int p = on ? pq[o] & 0xff : 0, q = on ? pq[o] >> 8 : 0;
          const uint32_t cp = __shfl_sync(0xffffffffu, cmine, p), cq = __shfl_sync(0xffffffffu, cmine, q);
          if (!on) continue;
          const double v = momt[(2 + o) * MP + r];
          if (q == p)
            row[cp] = v;  // candidate marginal (unnormalised, as the singleton weights)
          else
            pair_fx_add(f.ssT + static_cast<long long>(cp) * H + cq, v * inv_z, f.fx_scale);
        }
      }
      __syncthreads();
      // ---- phase B: item t = threadIdx.x + threads·it is (unit h, 16-point half) = (t / NH, t % NH)
      const long long kpt = n0;  // first point of the sub-tile within the chunk
      const long long kb = kpt / 64;
      const int boff = static_cast<int>(kpt % 64);
#pragma unroll
      for (int it = 0; it < ITS; ++it) {
        const int t = threadIdx.x + kFsThreads * it;
        const int h = t / NH, g0 = (t % NH) * 4;  // g0: first 4-point group of this half
        if (h >= Hp) break;
        double csum = cs[it];
        uint32_t w[8][4];
        if (h < H) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int p = 4 * (g0 + g) + e;
              const double x = tile[p * Hp + h] * rs[p];
              csum += x;
              const unsigned long long m = static_cast<unsigned long long>(x * a.inv56);
              hi[e] = spread7(static_cast<uint32_t>(m >> 28));         // digits 0-3: digit i at byte 3 − i
              lo[e] = spread7(static_cast<uint32_t>(m) & 0xfffffffu);  // digits 4-7: digit i at byte 7 − i
            }
            // 4 × 4 byte transposes: word of slice i = that digit of points 4g … 4g+3
            const uint32_t h01l = __byte_perm(hi[0], hi[1], 0x5140), h01h = __byte_perm(hi[0], hi[1], 0x7362);
            const uint32_t h23l = __byte_perm(hi[2], hi[3], 0x5140), h23h = __byte_perm(hi[2], hi[3], 0x7362);
            w[3][g] = __byte_perm(h01l, h23l, 0x5410);
            w[2][g] = __byte_perm(h01l, h23l, 0x7632);
            w[1][g] = __byte_perm(h01h, h23h, 0x5410);
            w[0][g] = __byte_perm(h01h, h23h, 0x7632);
            const uint32_t l01l = __byte_perm(lo[0], lo[1], 0x5140), l01h = __byte_perm(lo[0], lo[1], 0x7362);
            const uint32_t l23l = __byte_perm(lo[2], lo[3], 0x5140), l23h = __byte_perm(lo[2], lo[3], 0x7362);
            w[7][g] = __byte_perm(l01l, l23l, 0x5410);
            w[6][g] = __byte_perm(l01l, l23l, 0x7632);
            w[5][g] = __byte_perm(l01h, l23h, 0x5410);
            w[4][g] = __byte_perm(l01h, l23h, 0x7632);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int g = 0; g < 4; ++g) w[i][g] = 0u;
        }
        // (with two halves per unit, neighbouring lanes fill the two 16-byte halves of one 32-byte sector)
        int8_t* o = a.ess + (kb * Hp + h) * 64 + boff + 4 * g0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<uint4*>(o + i * a.slice_stride) = make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
        cs[it] = csum;
      }
      __syncthreads();
    }
    // Σ_n⟨s_nh⟩ of the block: the halves of a unit sit in neighbouring lanes
#pragma unroll
    for (int it = 0; it < ITS; ++it) {
      const int t = threadIdx.x + kFsThreads * it;
      double v = cs[it];
      if (NH == 2) v += __shfl_xor_sync(0xffffffffu, v, 1);
      const int h = t / NH;
      if (t % NH == 0 && h < H) a.colsum[blk * Hp + h] = v;
    }
  }
  if (lane == 0) red[wib] = lse_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int w = 0; w < NW; ++w) l += red[w];
    f.cta_scalars[2 * blockIdx.x] = l;
    f.cta_scalars[2 * blockIdx.x + 1] = 0.0;
  }
}

}  // namespace bscgpu
