// M-step kernels (linear_discrete.cpp:336-408): ridge, blocked Cholesky of
// Σ⟨ssᵀ⟩ + ridge·I (panel factor + row-wise triangular solves here, trailing
// updates on the DMMA GEMM), and the σ²/π updates.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "dgemm.cuh"

namespace bscgpu {

constexpr int kCholNb = 64;
#ifndef SOLVE_CHAIN_UNROLL
#define SOLVE_CHAIN_UNROLL 4  // unroll of the solves' dependent chain loop (1 / 4 / 8 measured: profiles/r02_variants.txt)
#endif
constexpr int kSolveChainUnroll = SOLVE_CHAIN_UNROLL;

// Device-side scalars of one EM iteration (kept resident; the host reads
// back only what the StepResult API needs).
struct MstepScalars {
  double trace, ridge;
  int chol_failed;  // LLT failure ⇒ keep the previous dictionary (:360-362)
  int pad;
  double t2, t3;
  double sigma2, pi;
};

// Bm = Σ⟨ssᵀ⟩ + ridge·I with ridge = 1e-9·trace/H (:349-353); Xr = Σ y⟨s⟩ᵀ.
// Two launches (`parts`): the factor's input, which needs only the E-step's
// moment sums, and the right-hand side, which needs the Yᵀ⟨S⟩ product.
constexpr int kPrepareFactor = 1, kPrepareRhs = 2;
__global__ void mstep_prepare_kernel(const double* __restrict__ stats, long long off_ssT, int D, int H,
                                     int ldb, double* __restrict__ Bm, double* __restrict__ X, int ldx,
                                     MstepScalars* sc, int parts) {
  if (parts & kPrepareRhs) {
    const long long DH = (long long)D * H;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < DH;
         e += (long long)gridDim.x * blockDim.x) {
      const int d = static_cast<int>(e / H), h = static_cast<int>(e % H);
      X[(long long)d * ldx + h] = stats[e];
    }
  }
  if (!(parts & kPrepareFactor)) return;
  __shared__ double tr;
  if (threadIdx.x < 32) {
    double acc = 0.0;
    for (int h = threadIdx.x; h < H; h += 32) acc += stats[off_ssT + (long long)h * H + h];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) tr = acc;
  }
  __syncthreads();
  const double trace = tr;
  const double ridge = 1e-9 * trace / static_cast<double>(H);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->trace = trace;
    sc->ridge = ridge;
    sc->chol_failed = trace > 0.0 ? 0 : 1;
  }
  const long long HH = (long long)H * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < HH; e += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(e / H), j = static_cast<int>(e % H);
    double v = stats[off_ssT + e];
    if (i == j) v += ridge;
    Bm[(long long)i * ldb + j] = v;
  }
}

// Right-looking Cholesky of the kb×kb diagonal block at (k0,k0) in shared
// memory (a partial last block is padded with the identity). One column per
// step: pivot (one thread), scale, rank-1 update of the trailing triangle by a
// 16×16 thread grid (each thread a fixed 4×4 set of entries).
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ A, int lda, int k0, int kb,
                                                         MstepScalars* sc) {
  __shared__ double L[kCholNb][kCholNb + 1];
  __shared__ int fail;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < kCholNb * kCholNb; e += blockDim.x) {
    const int i = e / kCholNb, j = e % kCholNb;
    L[i][j] = (i < kb && j < kb) ? A[(long long)(k0 + i) * lda + k0 + j] : (i == j ? 1.0 : 0.0);
  }
  if (tid == 0) fail = sc->chol_failed;
  __syncthreads();
  // Two barriers per column: every thread derives 1/√d itself and scales the
  // column entries it needs on the fly (the same product the stored scaled
  // entry holds), so each entry sees exactly the operations of the classic
  // scale-then-update loop.
  for (int j = 0; j < kCholNb; ++j) {
    double d = L[j][j];
    const bool bad = !(d > 0.0) || !isfinite(d);
    if (bad) d = 1.0;
    d = sqrt(d);
    const double rinv = 1.0 / d;
    double li[4], lk[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      li[a] = L[ty + 16 * a][j] * rinv;
      lk[a] = L[tx + 16 * a][j] * rinv;
    }
    __syncthreads();  // column j read by everyone before it is overwritten
    if (tid == 0) {
      if (bad) fail = 1;
      L[j][j] = d;
    }
    if (tid > j && tid < kCholNb) L[tid][j] *= rinv;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * a, k = tx + 16 * b;
        if (k > j && i >= k) L[i][k] -= li[a] * lk[b];
      }
    __syncthreads();
  }
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    const int i = e / kb, j = e % kb;
    A[(long long)(k0 + i) * lda + k0 + j] = j <= i ? L[i][j] : 0.0;
  }
  if (tid == 0 && fail) sc->chol_failed = 1;
}

// Warp-per-row triangular solves (right-looking, one column per step, the
// pivot broadcast by a shuffle): lane l holds entries l + 32·s of its row.
// Same operation order as the column-by-column substitution, so a row solve
// costs ~n dependent shuffle+FMA steps instead of n² serial FMAs per thread.

// Cholesky panel: rows [r0, r0+nrows) of Bm at columns [k0, k0+kb) ← X·L_kk⁻ᵀ.
// L_kk is staged per CTA in shared memory, transposed (U = L_kkᵀ).
__global__ void __launch_bounds__(256) trsm_panel_warp_kernel(double* __restrict__ Bm, int ldb, int k0, int kb, int r0,
                                                              int nrows) {
  __shared__ double U[kCholNb][kCholNb + 1];
  __shared__ double rinv[kCholNb];
  for (int e = threadIdx.x; e < kCholNb * kCholNb; e += blockDim.x) {
    const int c = e / kCholNb, t = e % kCholNb;  // U[c][t] = L[t][c]
    U[c][t] = (c < kb && t < kb && t >= c) ? Bm[(long long)(k0 + t) * ldb + k0 + c] : 0.0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kb; c += blockDim.x) rinv[c] = 1.0 / U[c][c];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= r0 + nrows) return;
  double* xr = Bm + (long long)row * ldb + k0;
  double x0 = lane < kb ? xr[lane] : 0.0, x1 = lane + 32 < kb ? xr[lane + 32] : 0.0;
  for (int c = 0; c < kb; ++c) {
    double xc;
    if (c < 32) {
      if (lane == c) x0 *= rinv[c];
      xc = __shfl_sync(0xffffffffu, x0, c);
      if (lane > c) x0 -= xc * U[c][lane];
      x1 -= xc * U[c][lane + 32];
    } else {
      if (lane == c - 32) x1 *= rinv[c];
      xc = __shfl_sync(0xffffffffu, x1, c - 32);
      if (lane + 32 > c) x1 -= xc * U[c][lane + 32];
    }
  }
  if (lane < kb) xr[lane] = x0;
  if (lane + 32 < kb) xr[lane + 32] = x1;
}

// U = Lᵀ (lower factor in Bm → upper rows, zeros elsewhere).
__global__ void transpose_lower_kernel(const double* __restrict__ Bm, int ldb, int H, double* __restrict__ U) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, t0 = blockIdx.y * 32;  // U[c][t] = L[t][c], t ≥ c
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int t = t0 + r, c = c0 + threadIdx.x;
    tile[r][threadIdx.x] = (t < H && c < H && t >= c) ? Bm[(long long)t * ldb + c] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int c = c0 + r, t = t0 + threadIdx.x;
    if (c < H && t < ldb) U[(long long)c * ldb + t] = t < H ? tile[threadIdx.x][r] : 0.0;
  }
}

// Rows of X (nrows × n, leading dim ldx) against the full factor:
//   FWD: X·Lᵀ = X with T = U = Lᵀ (row c of T = column c of L)
//   BWD: X·L  = X with T = L
// S = register slots per lane (n ≤ 32·S). The rows of T are consumed in
// order by every warp of the CTA: blocks of `rb` rows are staged in shared
// memory with cp.async, double-buffered, so each step reads the pivot row at
// shared-memory latency. Shared layout: rinv[n (padded)] | buf[2][rb·ldt].
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {  // f(integral_constant<I>) … f(<N-1>), unrolled by construction
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

template <int S, bool FWD>
__global__ void __launch_bounds__(128) solve_rows_kernel(const double* __restrict__ T, int ldt, int n,
                                                         double* __restrict__ X, int ldx, int nrows, int rb) {
  extern __shared__ __align__(16) double msm[];
  const int npad = (n + 1) & ~1;
  double* rinv = msm;
  double* buf0 = msm + npad;
  double* buf1 = buf0 + (size_t)rb * ldt;
  for (int c = threadIdx.x; c < n; c += blockDim.x) rinv[c] = 1.0 / T[(long long)c * ldt + c];
  const int nblk = (n + rb - 1) / rb;
  auto stage = [&](int blk, double* dst) {  // rows of block blk (in consumption order)
    const int b = FWD ? blk : nblk - 1 - blk;
    const int r0 = b * rb, rows = (r0 + rb <= n ? rb : n - r0);
    // whole rows, same stride on both sides: one contiguous range of 16-byte chunks
    const double* src = T + (long long)r0 * ldt;
    const int chunks = rows * (ldt / 2);
    for (int e = threadIdx.x; e < chunks; e += blockDim.x) cp_async16(dst + 2 * e, src + 2 * e, true);
    cp_async_commit();
  };
  stage(0, buf0);
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool active = row < nrows;
  double* xr = X + (long long)(active ? row : 0) * ldx;
  double x[S];
#pragma unroll
  for (int s = 0; s < S; ++s) x[s] = (active && lane + 32 * s < n) ? xr[lane + 32 * s] : 0.0;
  int blk = 0, cur_r0 = FWD ? 0 : (nblk - 1) * rb;
  double* cur = buf0;
  double* nxt = buf1;
  int blk_end = FWD ? -1 : 0x7fffffff;  // first c beyond the staged block (FWD) / below it (BWD)
  auto advance = [&](int c) {
    // make the block holding row c current (c leaves the staged range)
    if (blk > 0) {
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
    cp_async_wait<0>();
    __syncthreads();
    if (blk + 1 < nblk) stage(blk + 1, nxt);
    const int b = FWD ? blk : nblk - 1 - blk;
    cur_r0 = b * rb;
    blk_end = FWD ? cur_r0 + rb : cur_r0 - 1;
    ++blk;
  };
  // Columns are taken in segments (the run of one 32-column slot inside the staged row
  // block): first the dependent chain alone — pivot, broadcast, the update of the slot's own
  // remaining lanes — then the segment's updates of every other slot, which nothing in the
  // segment waits on. Each entry still receives its column updates in ascending (descending)
  // column order, so the result is the bits of the column-at-a-time loop.
  if (FWD) {
    static_for<0, S>([&](auto si) {
      constexpr int s = decltype(si)::value;
      const int cend = n - 32 * s < 32 ? n - 32 * s : 32;
      int cc = 0;
      while (cc < cend) {
        if (32 * s + cc >= blk_end) advance(32 * s + cc);
        const int seg_end = blk_end - 32 * s < cend ? blk_end - 32 * s : cend;
        const double* tb = cur + ((ptrdiff_t)32 * s - cur_r0) * ldt;  // row of column 32·s
#pragma unroll kSolveChainUnroll
        for (int q = cc; q < seg_end; ++q) {
          const double* tr = tb + (ptrdiff_t)q * ldt;
          if (lane == q) x[s] *= rinv[32 * s + q];
          const double xc = __shfl_sync(0xffffffffu, x[s], q);
          if (lane > q && lane < cend) x[s] -= xc * tr[lane + 32 * s];
        }
        if (s + 1 < S)
          for (int q = cc; q < seg_end; ++q) {
            const double* tr = tb + (ptrdiff_t)q * ldt;
            const double xc = __shfl_sync(0xffffffffu, x[s], q);
#pragma unroll
            for (int s2 = s + 1; s2 < S; ++s2)
              if (lane + 32 * s2 < n) x[s2] -= xc * tr[lane + 32 * s2];
          }
        cc = seg_end;
      }
    });
  } else {
    static_for<0, S>([&](auto si) {
      constexpr int s = S - 1 - decltype(si)::value;
      const int cend = n - 32 * s < 32 ? n - 32 * s : 32;
      int cc = cend - 1;
      while (cc >= 0) {
        if (32 * s + cc <= blk_end) advance(32 * s + cc);
        const int seg_lo = cur_r0 - 32 * s > 0 ? cur_r0 - 32 * s : 0;
        const double* tb = cur + ((ptrdiff_t)32 * s - cur_r0) * ldt;
#pragma unroll kSolveChainUnroll
        for (int q = cc; q >= seg_lo; --q) {
          const double* tr = tb + (ptrdiff_t)q * ldt;
          if (lane == q) x[s] *= rinv[32 * s + q];
          const double xc = __shfl_sync(0xffffffffu, x[s], q);
          if (lane < q) x[s] -= xc * tr[lane + 32 * s];
        }
        if (s > 0)
          for (int q = cc; q >= seg_lo; --q) {
            const double* tr = tb + (ptrdiff_t)q * ldt;
            const double xc = __shfl_sync(0xffffffffu, x[s], q);
#pragma unroll
            for (int s2 = 0; s2 < s; ++s2) x[s2] -= xc * tr[lane + 32 * s2];
          }
        cc = seg_lo - 1;
      }
    });
  }
  if (active) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (lane + 32 * s < n) xr[lane + 32 * s] = x[s];
  }
}

// W ← X unless the factorisation failed (then the previous W is kept).
__global__ void commit_w_kernel(const double* __restrict__ X, int ldx, double* __restrict__ W, int ldw, int D,
                                int H, const MstepScalars* sc) {
  if (sc->chol_failed) return;
  const long long DH = (long long)D * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < DH; e += (long long)gridDim.x * blockDim.x) {
    const int d = static_cast<int>(e / H), h = static_cast<int>(e % H);
    W[(long long)d * ldw + h] = X[(long long)d * ldx + h];
  }
}

// Partial sums of t2 = Σ W'∘Σy⟨s⟩ᵀ and t3 = Σ (W'ᵀW')∘Σ⟨ssᵀ⟩ (:366-368):
// one pair per CTA, folded in fixed order by mstep_scalars_kernel.
constexpr int kTraceCtas = 64;
__global__ void mstep_traces_kernel(const double* __restrict__ W, int ldw, const double* __restrict__ G, int ldg,
                                    const double* __restrict__ stats, long long off_ssT, int D, int H,
                                    double* __restrict__ partial) {
  __shared__ double red[2][32];
  double t2 = 0.0, t3 = 0.0;
  const long long DH = (long long)D * H, HH = (long long)H * H;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < DH; e += stride)
    t2 += W[(e / H) * ldw + e % H] * stats[e];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < HH; e += stride)
    t3 += G[(e / H) * ldg + e % H] * stats[off_ssT + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t2 += __shfl_xor_sync(0xffffffffu, t2, o);
    t3 += __shfl_xor_sync(0xffffffffu, t3, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = t2;
    red[1][threadIdx.x >> 5] = t3;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
  }
}

// σ²' = max((t1 − 2t2 + t3)/(N·D), 1e-12) and, for bsc / tsc,
// π' = clip(Σ_v counts_v/(N·H), 1e-6, 1−1e-6) (linear_discrete.cpp:369-381:
// bsc counts(0,0), tsc counts(0,0) + counts(0,1)); dsc probabilities are
// finished on the host from the counts. Tail layout: counts[V], y2, logZ, N.
// The iteration's host-visible result goes straight into one pinned, device-mapped block
// (kHostResult* offsets): the scalars, the E-step error flags and the statistics tail (F among
// them), so the host needs a stream synchronisation and no copy.
constexpr int kHostResultErr = 64, kHostResultTail = 72;
static_assert(sizeof(MstepScalars) <= kHostResultErr, "host result layout");
__global__ void mstep_scalars_kernel(const double* __restrict__ stats, long long off_tail, int D, int H, int V,
                                     const double* __restrict__ partial, MstepScalars* sc,
                                     const int* __restrict__ err, char* __restrict__ host_result) {
  double t2 = 0.0, t3 = 0.0;
  for (int c = 0; c < kTraceCtas; ++c) {
    t2 += partial[2 * c];
    t3 += partial[2 * c + 1];
  }
  sc->t2 = t2;
  sc->t3 = t3;
  const double n = stats[off_tail + V + 2];
  const double t1 = stats[off_tail + V];
  const double s2 = (t1 - 2.0 * sc->t2 + sc->t3) / (n * static_cast<double>(D));
  sc->sigma2 = s2 < 1e-12 ? 1e-12 : s2;
  double cnt = stats[off_tail];
  for (int k = 1; k < V; ++k) cnt += stats[off_tail + k];
  double p = cnt / (n * static_cast<double>(H));
  p = p < 1e-6 ? 1e-6 : p;
  p = (1.0 - 1e-6) < p ? (1.0 - 1e-6) : p;
  sc->pi = p;
  *reinterpret_cast<MstepScalars*>(host_result) = *sc;
  *reinterpret_cast<int*>(host_result + kHostResultErr) = *err;
  double* tail = reinterpret_cast<double*>(host_result + kHostResultTail);
  for (int k = 0; k < V + 3; ++k) tail[k] = stats[off_tail + k];
  __threadfence_system();
}

}  // namespace bscgpu
