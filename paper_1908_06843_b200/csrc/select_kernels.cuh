// Thread-per-point selection pass of the lane path (sm_100a).
//
// Reference: the per-point head of LinearDiscreteModel::estep_impl
// (linear_discrete.cpp:240-253: b = Wᵀy, the selection scores of :248-249) and
// select_candidates (truncation.cpp:38-57: stable sort of all H scores,
// descending, ties to the lower index, first H' kept, sorted ascending).
//
// One THREAD per data point, 32 consecutive points per warp (the record tile of
// lane_kernels.cuh), so the per-point scan over the H scores is scalar code with
// no shuffles: the B = Y·W rows of the warp's 32 points are staged through
// shared memory 32 columns at a time (cp.async, double-buffered, 16-byte pieces
// XOR-swizzled so that the 32 row reads of a warp hit distinct banks), and every
// thread keeps a sorted register list of its best H'+1 keys.
//
// Keys: the order-preserving 64-bit image of the score with its lowest 10 bits
// replaced by 1023 − h, so one unsigned compare orders by score and breaks
// exact ties toward the lower index (the reference's stable sort). The dropped
// bits move a score by < 2⁻⁴² relative; they enter the gap test below, like the
// error of the fast b. A point is proven exact when the gap between its H'-th
// and (H'+1)-th scores exceeds 2ε + δ (ε: |b_fast − b_oracle| propagated,
// bsc_engine.cu fill_enum_args; δ: the key truncation). Points that are not
// (near-ties, non-finite terms, the multiplicative range guard) are marked
// kModeFallback and redone by the warp-per-point pass with the exact re-rank.
//
// Outputs per point: the candidates (ascending), the record (shift bound, the
// singleton maximum, u, e^u, P, e^P — lane_kernels.cuh layout) and the point
// mode; Σ‖y‖² per CTA in a fixed order. The singleton weights of all H units
// are not written here: lane_finish_kernel computes them from the B row once
// the point's shift is final.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "bsc_kernels.cuh"

namespace bscgpu {

constexpr int kSelWarps = 4;                  // points per CTA = 32 · kSelWarps
constexpr int kSelCols = 16;                  // B columns per staged chunk
constexpr int kSelQueue = kSelCols;           // key queue slots per lane (merged after every chunk)
constexpr int kSelStageBytes = 32 * kSelCols * 8;  // 32 rows × 16 columns fp64
constexpr int kSelWarpBytes = 2 * kSelStageBytes + kSelQueue * 256;  // 2 stages + the key queue

__host__ __device__ inline int select_smem_bytes(int H) {
  return 8 * ((H + 1) & ~1) + 16 + kSelWarps * kSelWarpBytes;
}

// Selection key: the score with its lowest 10 mantissa bits replaced by an index
// code, h for negative scores and 1023 − h otherwise, so that as a DOUBLE the
// key orders by score and, among scores equal in their upper 42 bits, puts the
// lower index first (the reference's stable sort). Keys compare and sort with
// fp64 min/max (DMNMX, the FP64 pipe) instead of 64-bit integer compare/select
// chains on the ALU pipe.
__device__ __forceinline__ double sel_key(double f, int h) {
  const int hi = __double2hiint(f);
  const unsigned code = static_cast<unsigned>(hi < 0 ? h : 1023 - h);  // (only the low word changes)
  return __hiloint2double(hi, static_cast<int>((static_cast<unsigned>(__double2loint(f)) & ~1023u) | code));
}
__device__ __forceinline__ int key_index(double k) {
  const long long kb = __double_as_longlong(k);
  const int low = static_cast<int>(kb & 1023);
  return kb < 0 ? low : 1023 - low;
}
__device__ __forceinline__ double key_score(double k) {  // the score with the code bits cleared
  return __longlong_as_double(__double_as_longlong(k) & ~1023LL);
}

template <int HP>
__global__ void __launch_bounds__(32 * kSelWarps, 4) select_kernel(EnumArgs a) {
  constexpr int K = HP + 1;  // the H' best and the next one (gap test)
  constexpr int NP = HP * (HP - 1) / 2;
  extern __shared__ __align__(16) double ssm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int H = a.H, Hp = a.Hp, GM = a.gamma;
  double* gd = ssm;  // diag(G), this CTA
  double* sbound = ssm + ((H + 1) & ~1);
  char* stage = reinterpret_cast<char*>(sbound + 2) + wib * kSelWarpBytes;
  double* queue = reinterpret_cast<double*>(stage + 2 * kSelStageBytes) + lane;  // [slot][32 lanes]
  for (int i = threadIdx.x; i < H; i += blockDim.x) gd[i] = a.gdiag[i];
  if (wib == 0) {
    double bd = 0.0, gm = 0.0;  // max_h ‖W_h‖ (selection error bound), max_h G_hh
    for (int h = lane; h < H; h += 32) {
      bd = fmax(bd, a.wnorm[h]);
      gm = fmax(gm, a.gdiag[h]);
    }
    bd = warp_max(bd);
    gm = warp_max(gm);
    if (lane == 0) {
      sbound[0] = bd;
      sbound[1] = gm;
    }
  }
  __syncthreads();
  const double bound = sbound[0], gmax = sbound[1];

  double y2_acc = 0.0;
  // persistent over CTA tiles of 32·kSelWarps points; warp wib owns points [n0, n0 + 32)
  for (long long ct = blockIdx.x; ct * 32 * kSelWarps < a.N; ct += gridDim.x) {
    const long long n0 = (ct * kSelWarps + wib) * 32;
    if (n0 >= a.N) continue;
    const long long n = n0 + lane;
    const bool live = n < a.N;
    const int nrows = static_cast<int>(min(32LL, a.N - n0));
    const int nch = (Hp + kSelCols - 1) / kSelCols;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    // stage s ← columns [16c, 16c+16) of the tile's rows (16-byte piece j of row r
    // at r·128 + (j ^ (r & 7))·16: a row read by its lane hits distinct banks)
    auto issue = [&](int c, int s) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + (lane >> 3), j = lane & 7;
        const int col = c * kSelCols + 2 * j;
        if (r < nrows && col < Hp) {
          const uint32_t d = sbase + s * kSelStageBytes + r * 128 + ((j ^ (r & 7)) << 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                       "l"(a.B + (n0 + r) * Hp + col)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0, 0);

    // The best K keys so far, descending. A column's key is only queued when it
    // beats the list's current K-th key (the threshold only rises: a valid lower
    // bound of the final K-th), and the queue is merged into the list once per
    // chunk, so the insertion network runs ~K·(1 + ln(H/16K)) times per point
    // instead of at every column where any lane of the warp would insert.
    // (Measured and rejected, profiles/r02_variants.txt: thresholds warm-started from
    // the previous iteration's candidates with merges deferred until the queue fills.)
    double L[K];
#pragma unroll
    for (int j = 0; j < K; ++j) L[j] = -INFINITY;
    double tau = -INFINITY, probe = 0.0;
    const double log_pi = a.log_pi, inv2s = a.inv2s;
    int cnt = 0;
    auto merge = [&]() {
      // L'[j] = c_j ? (c_{j−1} ? L[j−1] : k) : L[j], c_j = k > L[j]
      const int rounds = __reduce_max_sync(0xffffffffu, cnt);
      for (int i = 0; i < rounds; ++i) {
        const double k = i < cnt ? queue[i * 32] : -INFINITY;
        bool c_prev = k > L[0];
        const double l0 = L[0];
        L[0] = c_prev ? k : l0;
        double up = l0;  // old L[j−1]
#pragma unroll
        for (int j = 1; j < K; ++j) {
          const bool cj = k > L[j];
          const double old = L[j];
          L[j] = cj ? (c_prev ? up : k) : old;
          up = old;
          c_prev = cj;
        }
      }
      cnt = 0;
      tau = L[K - 1];
    };
    for (int c = 0; c < nch; ++c) {
      if (c + 1 < nch) {
        issue(c + 1, (c + 1) & 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      const char* row = stage + (c & 1) * kSelStageBytes + lane * 128;
      const int h0 = c * kSelCols;
      auto score = [&](auto checked) {
#pragma unroll
        for (int j = 0; j < kSelCols / 2; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(row + ((j ^ (lane & 7)) << 4));
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int h = h0 + 2 * j + u;
            if (!decltype(checked)::value || h < H) {
              const double t = __fma_rn(2.0, u ? v.y : v.x, -gd[h]);  // = 2b − G_hh (2b is exact)
              const double f = __dadd_rn(log_pi, __dmul_rn(t, inv2s));  // linear_discrete.cpp:248-249, unfused
              probe = __fma_rn(f, 0.0, probe);                          // NaN once any score is not finite
              const double k = sel_key(f, h);
              if (k > tau) queue[(cnt++) * 32] = k;
            }
          }
        }
      };
      if (h0 + kSelCols <= H)  // a full chunk: one straight-line block of 16 columns, no per-column test
        score(std::false_type{});
      else
        score(std::true_type{});
      __syncwarp();
      merge();
      __syncwarp();
    }

    int mode = kModeDone;
    if (live) {
      const double y2 = a.y2[n];
      const bool bad = !(probe == 0.0);
      int cand[HP];
      bool exact = true;
      if (HP < H) {
#pragma unroll
        for (int j = 0; j < HP; ++j) cand[j] = key_index(L[j]);
        // |f_fast − f_exact| ≤ eps: the b error (eps_dot·‖W_h‖·‖y‖) propagated
        // through ×2, −G, ×inv2s, +log π, plus the rounding of those operations
        // relative to mag ≥ max_h (|f_h| + inv2s(2|b_h| + G_hh)) + |log π|, with
        // |b_h| ≤ ‖W_h‖‖y‖ (Cauchy–Schwarz) and |f_h| ≤ |log π| + inv2s(2|b_h| + G_hh)
        const double bmax = bound * sqrt(y2) * 1.0001;
        const double mag = 2.0 * fabs(log_pi) + 2.0 * inv2s * (2.0 * bmax + gmax) * 1.0001;
        const double eps = 2.5 * inv2s * a.eps_dot * bound * sqrt(y2) * 1.0001 + 0x1.0p-46 * mag;
        const double t = key_score(L[HP - 1]), nv = key_score(L[HP]);
        const double delta = 0x1.0p-40 * (fabs(t) + fabs(nv));  // the 10 code bits of both keys
        exact = t - nv > 2.0 * eps + delta;
      } else {
#pragma unroll
        for (int j = 0; j < HP; ++j) cand[j] = j;
      }
      if (bad) {
        atomicOr(a.err, kErrNonFiniteScore);
      } else {
        // ascending (truncation.cpp:55): odd-even transposition network
#pragma unroll
        for (int r = 0; r < HP; ++r)
#pragma unroll
          for (int j = r & 1; j + 1 < HP; j += 2) {
            const int lo = min(cand[j], cand[j + 1]), hi = max(cand[j], cand[j + 1]);
            cand[j] = lo;
            cand[j + 1] = hi;
          }
        uint32_t* co = a.cand_out + n * HP;
#pragma unroll
        for (int j = 0; j < HP; ++j) co[j] = static_cast<uint32_t>(cand[j]);
        y2_acc += y2;
        mode = kModeFallback;
        if (exact) {
          // unary / pairwise log-joint terms relative to the zero state (as the
          // warp pass): u_p = dlp + inv2s(2b − G_pp), P_pq = −2 inv2s G_pq
          double* rt = a.rec + (n >> 5) * lane_rec_fields(HP) * 32 + (n & 31);
          const double* brow = a.B + n * Hp;
          double umax = -INFINITY, uabs = 0.0, pmax = -INFINITY, pabs = 0.0;
          bool fin = true;
#pragma unroll
          for (int p = 0; p < HP; ++p) {
            const double u = __fma_rn(inv2s, __fma_rn(2.0, brow[cand[p]], -gd[cand[p]]), a.dlp);
            fin = fin && isfinite(u);
            umax = fmax(umax, u);
            uabs = fmax(uabs, fabs(u));
            rt[(4 + p) * 32] = u;
            rt[(4 + HP + p) * 32] = exp_nonpos(u);  // used only when |u| ≤ 300 (mult_ok)
          }
          int e = 0;
#pragma unroll
          for (int p = 0; p < HP; ++p) {
            const long long go = static_cast<long long>(cand[p]) * Hp;
#pragma unroll
            for (int q = p + 1; q < HP; ++q, ++e) {
              // (P and e^P gathered from per-E-step H × H tables instead: measured slower, r02_variants.txt)
              const double v = -2.0 * inv2s * __ldg(a.G + go + cand[q]);
              const double ev = exp_nonpos(v);
              fin = fin && isfinite(v);
              pmax = fmax(pmax, v);
              pabs = fmax(pabs, fabs(v));
              rt[(4 + 2 * HP + e) * 32] = v;
              rt[(4 + 2 * HP + NP + e) * 32] = ev;
            }
          }
          // q(S) = q(A)·e^{u_z}·e^{coup(S)} stays in fp64 range when |u| ≤ 300 and
          // (γ−1)|P| ≤ 300; the shift needs no maximum: an upper bound within e^300
          // of it loses nothing to underflow (bsc_kernels.cuh, phase 3)
          // the largest singleton log-joint (and the zero state, rel 0): the top
          // selection score's unit is a candidate, and rel = u is monotone in f
          const double mx = fmax(0.0, umax);
          const bool mult_ok = fin && a.weight_mode != 2 && uabs <= 300.0 && (GM - 1) * pabs <= 300.0;
          if (!fin) atomicOr(a.err, kErrNonFiniteLogJoint);
          if (mult_ok) {
            const double ub = GM * fmax(umax, 0.0) + 0.5 * GM * (GM - 1) * fmax(pmax, 0.0);
            const bool skip_rel = a.weight_mode == 0 && ub - mx <= 300.0;
            rt[0] = fmax(mx, ub);
            rt[64] = mx;
            mode = skip_rel ? kModeShift : kModeMax;
          }
        }
      }
      a.pmode[n] = mode;
      if (mode == kModeFallback) atomicAdd(a.err + 1, 1);
    }
  }
  // per-CTA Σ‖y_n‖² in a fixed order (warp tree, then warps in index order)
  y2_acc = warp_sum(y2_acc);
  __syncthreads();
  if (lane == 0) ssm[wib] = y2_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kSelWarps; ++w) s += ssm[w];
    a.warp_scalars[2 * blockIdx.x] = 0.0;
    a.warp_scalars[2 * blockIdx.x + 1] = s;
  }
}

}  // namespace bscgpu
