// M-step kernels (linear_discrete.cpp:336-408): ridge, blocked Cholesky of
// Σ⟨ssᵀ⟩ + ridge·I (panel factor + row-wise triangular solves here, trailing
// updates on the DMMA GEMM), and the σ²/π updates.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bscgpu {

constexpr int kCholNb = 64;

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
__global__ void mstep_prepare_kernel(const double* __restrict__ stats, long long off_ssT, int D, int H,
                                     int ldb, double* __restrict__ Bm, double* __restrict__ X, int ldx,
                                     MstepScalars* sc) {
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
  const long long DH = (long long)D * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < DH; e += (long long)gridDim.x * blockDim.x) {
    const int d = static_cast<int>(e / H), h = static_cast<int>(e % H);
    X[(long long)d * ldx + h] = stats[e];
  }
}

// Right-looking Cholesky of the kb×kb diagonal block at (k0,k0) in shared
// memory (a partial last block is padded with the identity). One column per
// step: pivot (one thread), scale, rank-1 update of the trailing triangle by a
// 16×16 thread grid (each thread a fixed 4×4 set of entries).
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* __restrict__ A, int lda, int k0, int kb,
                                                         MstepScalars* sc) {
  __shared__ double L[kCholNb][kCholNb + 1];
  __shared__ double rinv;
  __shared__ int fail;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  for (int e = tid; e < kCholNb * kCholNb; e += blockDim.x) {
    const int i = e / kCholNb, j = e % kCholNb;
    L[i][j] = (i < kb && j < kb) ? A[(long long)(k0 + i) * lda + k0 + j] : (i == j ? 1.0 : 0.0);
  }
  if (tid == 0) fail = sc->chol_failed;
  __syncthreads();
  for (int j = 0; j < kCholNb; ++j) {
    if (tid == 0) {
      double d = L[j][j];
      if (!(d > 0.0) || !isfinite(d)) {
        fail = 1;
        d = 1.0;
      }
      d = sqrt(d);
      L[j][j] = d;
      rinv = 1.0 / d;
    }
    __syncthreads();
    if (tid > j && tid < kCholNb) L[tid][j] *= rinv;
    __syncthreads();
    double li[4], lk[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      li[a] = L[ty + 16 * a][j];
      lk[a] = L[tx + 16 * a][j];
    }
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

// Row-wise triangular solves against the kb×kb lower block Lkk stored at
// (k0,k0) of L (leading dim ldl), applied to rows [r0, r0+nrows) of X at
// columns [c0, c0+kb); one thread per row, the row held in registers (the
// 64-wide block is fully unrolled, padded with the identity past kb):
//   FWD_T:  x · Lkkᵀ = x_in  (forward substitution)   — Cholesky panel / Z = R·L⁻ᵀ
//   BWD  :  x · Lkk  = x_in  (backward substitution)  — X = Z·L⁻¹
template <bool FWD_T>
__global__ void __launch_bounds__(128) trsm_rows_kernel(const double* __restrict__ Lm, int ldl, int k0, int kb,
                                                        double* __restrict__ X, int ldx, int r0, int nrows, int c0) {
  __shared__ double L[kCholNb][kCholNb + 1];
  __shared__ double rinv[kCholNb];
  const int tid = threadIdx.x;
  for (int e = tid; e < kCholNb * kCholNb; e += blockDim.x) {
    const int i = e / kCholNb, j = e % kCholNb;
    L[i][j] = (i < kb && j < kb) ? Lm[(long long)(k0 + i) * ldl + k0 + j] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int c = tid; c < kCholNb; c += blockDim.x) rinv[c] = 1.0 / L[c][c];
  __syncthreads();
  const int row = r0 + blockIdx.x * blockDim.x + tid;
  if (row >= r0 + nrows) return;
  double* xr = X + (long long)row * ldx + c0;
  double x[kCholNb];
#pragma unroll
  for (int c = 0; c < kCholNb; ++c) x[c] = c < kb ? xr[c] : 0.0;
  if (FWD_T) {
#pragma unroll
    for (int c = 0; c < kCholNb; ++c) {
      x[c] *= rinv[c];
#pragma unroll
      for (int t = c + 1; t < kCholNb; ++t) x[t] -= x[c] * L[t][c];
    }
  } else {
#pragma unroll
    for (int c = kCholNb - 1; c >= 0; --c) {
      x[c] *= rinv[c];
#pragma unroll
      for (int t = 0; t < c; ++t) x[t] -= x[c] * L[c][t];
    }
  }
#pragma unroll
  for (int c = 0; c < kCholNb; ++c)
    if (c < kb) xr[c] = x[c];
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
__global__ void mstep_scalars_kernel(const double* __restrict__ stats, long long off_tail, int D, int H, int V,
                                     const double* __restrict__ partial, MstepScalars* sc) {
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
}

}  // namespace bscgpu
