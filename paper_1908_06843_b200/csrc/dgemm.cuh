// fp64 tensor-core GEMM for sm_100a (DMMA.8x8x4 via mma.sync m8n8k4.f64).
//
// tcgen05 has no f64 kind, so the fp64 contractions of the BSC E/M-step
// (Y·W, Yᵀ·⟨S⟩, Gram and M-step products) run on the warp-level DMMA pipe,
// which on B200 delivers the same ≈37 TFLOP/s as the DFMA peak
// (profiles/r01_fp64_peaks.json) with a quarter of the issue slots.
//
//   C[M×N] = alpha · op(A)[M×K] · op(B)[K×N] + beta · C
//
// A_ROW: A is stored M×K row-major (lda); otherwise K×M row-major (Aᵀ).
// B_ROW: B is stored K×N row-major (ldb); otherwise N×K row-major (Bᵀ).
// Split-K: blockIdx.z takes K range [z·kchunk, min(K,(z+1)·kchunk)) and writes
// its partial to C + z·c_split_stride (a workspace reduced in fixed order).
// Tiles are staged global→shared with cp.async (16 B = 2 doubles, zero-filled
// past the edges) through a STAGES-deep ring; requirements: lda/ldb/ldc even,
// K and kchunk even, M and N even, base pointers 16 B aligned.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bscgpu {

struct GemmArgs {
  int M, N, K;
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
  double alpha, beta;
  int kchunk;
  long long c_split_stride;
  double* colsum = nullptr;  // optional [splits][N]: Σ_k B[k, n] per split (B_ROW only)
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM, int WN, bool A_ROW, bool B_ROW, int STAGES>
struct DgemmCfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  // Leading dims padded to ≡ 4 (mod 16) doubles: the m8n8k4 fragment pattern
  // (4 rows × 4 cols per half-warp) then hits 16 distinct 8-byte banks.
  static constexpr int kLdA = A_ROW ? BK + 4 : BM + 4;
  static constexpr int kLdB = B_ROW ? BN + 4 : BK + 4;
  static constexpr int kSizeA = A_ROW ? BM * kLdA : BK * kLdA;
  static constexpr int kSizeB = B_ROW ? BK * kLdB : BN * kLdB;
  static constexpr int kStageDoubles = kSizeA + kSizeB;
  static constexpr int kSmemBytes = STAGES * kStageDoubles * 8;
  static_assert(kLdA % 16 == 4 && kLdB % 16 == 4, "bank-conflict-free padding");
  static_assert(BK % 4 == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shape");
};

template <int BM, int BN, int BK, int WM, int WN, bool A_ROW, bool B_ROW, int STAGES>
__global__ void __launch_bounds__(DgemmCfg<BM, BN, BK, WM, WN, A_ROW, B_ROW, STAGES>::kThreads)
    dgemm_kernel(GemmArgs g) {
  using Cfg = DgemmCfg<BM, BN, BK, WM, WN, A_ROW, B_ROW, STAGES>;
  constexpr int MI = WM / 8, NI = WN / 8;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % Cfg::kWarpsM, wn = warp / Cfg::kWarpsM;
  const int m_base = blockIdx.y * BM, n_base = blockIdx.x * BN;
  const int k_begin = blockIdx.z * g.kchunk;
  const int k_end = min(g.K, k_begin + g.kchunk);
  const int ktiles = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;

  auto load_tile = [&](int stage, int kt) {
    double* As = smem + stage * Cfg::kStageDoubles;
    double* Bs = As + Cfg::kSizeA;
    const int k0 = k_begin + kt * BK;
    constexpr int kChunksA = BM * BK / 2, kChunksB = BN * BK / 2;
    for (int c = tid; c < kChunksA; c += Cfg::kThreads) {
      int r, cc;
      const double* src;
      double* dst;
      bool ok;
      if constexpr (A_ROW) {  // As[m][k]
        r = c / (BK / 2);
        cc = (c % (BK / 2)) * 2;
        const int gm = m_base + r, gk = k0 + cc;
        ok = gm < g.M && gk < k_end;
        src = ok ? g.A + (long long)gm * g.lda + gk : g.A;
        dst = As + r * Cfg::kLdA + cc;
      } else {  // As[k][m]
        r = c / (BM / 2);
        cc = (c % (BM / 2)) * 2;
        const int gk = k0 + r, gm = m_base + cc;
        ok = gk < k_end && gm < g.M;
        src = ok ? g.A + (long long)gk * g.lda + gm : g.A;
        dst = As + r * Cfg::kLdA + cc;
      }
      cp_async16(dst, src, ok);
    }
    for (int c = tid; c < kChunksB; c += Cfg::kThreads) {
      int r, cc;
      const double* src;
      double* dst;
      bool ok;
      if constexpr (B_ROW) {  // Bs[k][n]
        r = c / (BN / 2);
        cc = (c % (BN / 2)) * 2;
        const int gk = k0 + r, gn = n_base + cc;
        ok = gk < k_end && gn < g.N;
        src = ok ? g.B + (long long)gk * g.ldb + gn : g.B;
        dst = Bs + r * Cfg::kLdB + cc;
      } else {  // Bs[n][k]
        r = c / (BK / 2);
        cc = (c % (BK / 2)) * 2;
        const int gn = n_base + r, gk = k0 + cc;
        ok = gn < g.N && gk < k_end;
        src = ok ? g.B + (long long)gn * g.ldb + gk : g.B;
        dst = Bs + r * Cfg::kLdB + cc;
      }
      cp_async16(dst, src, ok);
    }
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fc = lane & 3;  // fragment row / k index
  const bool colsum_cta = g.colsum != nullptr && blockIdx.y == 0;
  double cs = 0.0;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch tile kt + STAGES - 1 into the slot freed by tile kt - 1
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) load_tile(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* As = smem + (kt % STAGES) * Cfg::kStageDoubles;
    const double* Bs = As + Cfg::kSizeA;
    if constexpr (B_ROW) {
      if (colsum_cta) {  // Σ_k B[k, n] of this split (e.g. Σ_n ⟨s_n⟩ beside Yᵀ⟨S⟩)
#pragma unroll
        for (int r = tid / BN; r < BK; r += Cfg::kThreads / BN) cs += Bs[r * Cfg::kLdB + tid % BN];
      }
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int m = wm * WM + i * 8 + fr;
        a[i] = A_ROW ? As[m * Cfg::kLdA + kk + fc] : As[(kk + fc) * Cfg::kLdA + m];
      }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int n = wn * WN + j * 8 + fr;
        b[j] = B_ROW ? Bs[(kk + fc) * Cfg::kLdB + n] : Bs[n * Cfg::kLdB + kk + fc];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  double* C = g.C + (long long)blockIdx.z * g.c_split_stride;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int m = m_base + wm * WM + i * 8 + fr;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int n = n_base + wn * WN + j * 8 + fc * 2;
      if (n >= g.N) continue;
      double2* dst = reinterpret_cast<double2*>(C + (long long)m * g.ldc + n);
      double2 v;
      v.x = g.alpha * acc[i][j][0];
      v.y = g.alpha * acc[i][j][1];
      if (g.beta != 0.0) {
        const double2 o = *dst;
        v.x += g.beta * o.x;
        v.y += g.beta * o.y;
      }
      *dst = v;
    }
  }
  if constexpr (B_ROW) {
    if (colsum_cta) {  // fold the row groups in fixed order → colsum[z][n]
      __syncthreads();
      double* red = smem;
      red[tid] = cs;
      __syncthreads();
      if (tid < BN) {
        double s = 0.0;
        for (int r = 0; r < Cfg::kThreads / BN; ++r) s += red[r * BN + tid];
        const int n = n_base + tid;
        if (n < g.N) g.colsum[(long long)blockIdx.z * g.N + n] = s;
      }
    }
  }
}

// Host-side launcher for one tile configuration.
template <int BM, int BN, int BK, int WM, int WN, bool A_ROW, bool B_ROW, int STAGES>
inline cudaError_t launch_dgemm(const GemmArgs& g, int splits, cudaStream_t stream) {
  using Cfg = DgemmCfg<BM, BN, BK, WM, WN, A_ROW, B_ROW, STAGES>;
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, A_ROW, B_ROW, STAGES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, splits);
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, stream>>>(g);
  return cudaGetLastError();
}

}  // namespace bscgpu
