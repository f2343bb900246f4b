// fp64 GEMM on the sm_100a integer tensor cores (tcgen05.mma kind::i8) by
// exact int8 slicing (the Ozaki scheme).
//
// Every row of A (and every column of B) is scaled by a power of two 2^e with
// max|x| < 2^e and cut into S = 8 signed 7-bit slices:
//     x = 2^e · Σ_{i<S} a_i · 2^{-7(i+1)} + r,   a_i ∈ [-127, 127],  |r| < 2^{e-56}
// (truncation toward zero; every step is exact in fp64). The product is then
//     A·B ≈ diag(sa) · Σ_{g<S} 2^{-7(g+2)} · (Σ_{i+j=g} A_i · B_j) · diag(sb)
// where each inner sum is an exact int32 accumulation on the tensor cores
// (|A_i B_j| ≤ 127² per term; ≤ 8·K_job·127² < 2^31 for K_job ≤ 16384) and the
// eight group sums are combined in fp64 in the epilogue. Dropped terms
// (i+j ≥ S) and the slicing remainders bound the error per output by
//     |ΔC| ≤ K · 11·2^{-56} · sa_m · sb_n  ≤  K · 2^{-50.5} · max_k|a_mk| · max_k|b_kn|
// which is of the order of (and never worse than K/u times) the rounding bound
// of an fp64 DGEMM, γ_K Σ|a||b|.
//
// Kernel layout (one CTA per SM, persistent over jobs = (k-split, m-tile, n-tile)):
//   warp 0: TMA producer — B tile (S slices, 128 rows × 64 k) + A tiles
//           (one slice, 128 rows × 64 k) through mbarrier rings;
//   warp 1: TMEM allocation (512 columns = 4 group accumulators × 128) and the
//           single-thread tcgen05.mma issue; each tile runs in two passes over
//           K, groups 4-7 (26 slice products) then 0-3 (10 products);
//   warps 2-9: epilogue — tcgen05.ld of the 4 int32 groups of a pass, fp64
//           combine (smallest weights first) across both passes, scale, store
//           (or accumulate) to C.
// The 128-column tile matters: on B200 a kind::i8 M=128 K=32 MMA costs the same
// ~80 cycles for N = 32, 64 or 128 (N = 256: 1.55×; tools/ozaki_test probes),
// so N = 128 halves the issue time of N = 64 per output column.
// Operands are K-major int8, 64-byte swizzled (TMA SWIZZLE_64B ↔ UMMA
// SWIZZLE_64B, SBO = 512 B), K advanced by 32 bytes per MMA inside the row.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace bscgpu {
namespace oz {

constexpr int S = 8;                    // slices
constexpr int BM = 128, BN = 128, BK = 64;
constexpr int GPP = 4, NPASS = 2;       // 4 group accumulators × 128 TMEM columns per pass
// A ring: 10 stages, or 8 beside the epilogue's staging tiles (the variant with TMA stores)
__host__ __device__ constexpr int a_stages(bool tma_store) { return tma_store ? 8 : 10; }
constexpr int B_STAGES = 2;
constexpr int A_BYTES = BM * BK;        // 8 KB: one slice
constexpr int B_BYTES = S * BN * BK;    // 64 KB: all slices
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (2 + EPI_WARPS);  // producer, MMA, 8 epilogue warps (2 per TMEM lane quadrant)
constexpr int EPI_COLS = BN / 2;        // columns per epilogue thread
constexpr int C_COLS = 8;                         // output columns per staged epilogue piece (64-byte rows)
constexpr int C_WARP_BYTES = 32 * C_COLS * 8;     // one warp's staging tile: 32 rows × 8 columns fp64
constexpr int C_BYTES = EPI_WARPS * C_WARP_BYTES;
__host__ __device__ constexpr int smem_bytes(bool tma_store) {
  return a_stages(tma_store) * A_BYTES + B_STAGES * B_BYTES + (tma_store ? C_BYTES : 0) + 1024 + 256;
}
constexpr int MAX_KJOB = 16384;         // int32 headroom per job (see above)
constexpr int MAX_KROW = 1024;          // longest row the row slicer holds in registers
static_assert(smem_bytes(true) <= 227 * 1024 && smem_bytes(false) <= 227 * 1024, "shared memory");
static_assert(GPP * BN <= 512 && GPP * NPASS == S, "TMEM groups");

struct Args {
  int M, N;             // valid output rows / cols
  int K;                // K extent (elements) of the whole product
  int kchunk;           // K per job, a multiple of BK (≤ MAX_KJOB)
  int m_tiles, n_tiles, k_splits;
  const double* sa;     // row scales of A, [k_split][sa_stride]
  long long sa_stride;  // 0: one vector for every split
  const double* sb;     // column scales of B
  long long sb_stride;
  double* C;
  long long ldc;
  long long c_split_stride;  // partial slot stride per k-split
  int accumulate;            // C += result (else C = result)
  int tma_store;             // the epilogue stores C through the tensor map tc (set by launch_gemm)
  int blk_a, blk_b;          // operand layout: 0 rows [S][rows][ld], 1 K-blocked [S][k/BK][rows][BK]
};

// One sliced operand: slice s, row r, k at
//   rows layout:      base + s·slice_stride + r·ld + k
//   K-blocked layout: base + s·slice_stride + ((k / BK)·ld + r)·BK + k % BK   (ld = allocated rows)
// The K-blocked layout keeps every TMA box (BK × rows) one contiguous run,
// which matters when k is the point index (rows ~N bytes apart otherwise).
struct Operand {
  const int8_t* base;
  long long slice_stride;
  long long ld;
  int rows;      // valid rows (TMA zero-fills past them)
  int blocked;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_op(uint32_t dst, const CUtensorMap* map, bool blocked, int k, int row,
                                            int slice, uint32_t bar) {
  if (blocked)
    tma_load_4d(dst, map, 0, row, k / BK, slice, bar);
  else
    tma_load_3d(dst, map, k, row, slice, bar);
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// K-major operand, 64-byte swizzle (rows of BK = 64 int8), 8-row groups 512 B
// apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(4) << 61);
}
// kind::i8: D s32 (bits 4-5 = 2), A/B signed (bits 7-9, 10-12 = 1), K-major, N>>3 at 17, M>>4 at 24.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                            (static_cast<uint32_t>(BM >> 4) << 24);

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// (double)x without I2F: the int32 as the low word of 2^52 + 2^31 + x, minus that constant — one
// logic op and one exact fp64 add. I2F.F64 issues at a quarter of the FP64 rate (conversion unit):
// 65,536 conversions per pass and SM sat on the TMEM drain (c2 Y·W 0.82 -> 0.79 ms).
__device__ __forceinline__ double i32_to_f64(int x) {
  return __hiloint2double(0x43300000, x ^ static_cast<int>(0x80000000u)) - 4503601774854144.0;
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// ---------------------------------------------------------------- the GEMM
template <bool TMA_STORE>
__global__ void __launch_bounds__(THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb8,
                   const __grid_constant__ CUtensorMap tb4, const __grid_constant__ CUtensorMap tc, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  constexpr int A_STAGES = a_stages(TMA_STORE);
  uint8_t* sB = smem + A_STAGES * A_BYTES;
  uint8_t* sC = sB + B_STAGES * B_BYTES;  // (1024-byte aligned: the stage sizes are multiples of 1024)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + (TMA_STORE ? C_BYTES : 0));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * A_STAGES + 2 * B_STAGES + 2);
  const uint32_t full_a = smem_u32(bars), empty_a = full_a + 8 * A_STAGES;
  const uint32_t full_b = empty_a + 8 * A_STAGES, empty_b = full_b + 8 * B_STAGES;
  const uint32_t tfull = empty_b + 8 * B_STAGES, tempty = tfull + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < A_STAGES; ++i) mbar_init(full_a + 8 * i, 1), mbar_init(empty_a + 8 * i, 1);
    for (int i = 0; i < B_STAGES; ++i) mbar_init(full_b + 8 * i, 1), mbar_init(empty_b + 8 * i, 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int per_split = a.m_tiles * a.n_tiles;
  const int jobs = per_split * a.k_splits;

  if (warp == 0) {
    if (lane == 0) {
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      for (int job = blockIdx.x; job < jobs; job += gridDim.x) {
        const int nt = job % a.n_tiles, mt = (job / a.n_tiles) % a.m_tiles, ks = job / per_split;
        const int k0 = ks * a.kchunk;
        const int nkb = (min(a.kchunk, a.K - k0) + BK - 1) / BK;
        for (int p = 0; p < NPASS; ++p) {
          const int gbase = (NPASS - 1 - p) * GPP;  // high groups first
          const int nA = min(S, gbase + GPP);       // A slices 0 … nA−1 take part
          const bool all_b = nA == S;               // B slices 0 … nA−1 likewise
          for (int kb = 0; kb < nkb; ++kb) {
            const int kc = k0 + kb * BK;
            mbar_wait(empty_b + 8 * bs, bph ^ 1);
            mbar_expect_tx(full_b + 8 * bs, all_b ? B_BYTES : B_BYTES / 2);
            tma_load_op(smem_u32(sB + bs * B_BYTES), all_b ? &tb8 : &tb4, a.blk_b, kc, nt * BN, 0, full_b + 8 * bs);
            if (++bs == B_STAGES) bs = 0, bph ^= 1;
            for (int i = 0; i < nA; ++i) {
              mbar_wait(empty_a + 8 * as, aph ^ 1);
              mbar_expect_tx(full_a + 8 * as, A_BYTES);
              tma_load_op(smem_u32(sA + as * A_BYTES), &ta, a.blk_a, kc, mt * BM, i, full_a + 8 * as);
              if (++as == A_STAGES) as = 0, aph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int as = 0, bs = 0, u = 0;
      uint32_t aph = 0, bph = 0;
      for (int job = blockIdx.x; job < jobs; job += gridDim.x) {
        const int ks = job / per_split;
        const int k0 = ks * a.kchunk;
        const int nkb = (min(a.kchunk, a.K - k0) + BK - 1) / BK;
        for (int p = 0; p < NPASS; ++p, ++u) {
          const int gbase = (NPASS - 1 - p) * GPP;
          const int nA = min(S, gbase + GPP);
          if (u > 0) mbar_wait(tempty, (u - 1) & 1);  // the epilogue drained the previous pass
          tc_fence_after();
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(full_b + 8 * bs, bph);
            const uint32_t b_base = smem_u32(sB + bs * B_BYTES);
            for (int i = 0; i < nA; ++i) {
              mbar_wait(full_a + 8 * as, aph);
              tc_fence_after();
              const uint64_t da = sdesc(smem_u32(sA + as * A_BYTES));
              // groups g = i + j in [gbase, gbase + GPP): i = 0 comes first and opens all of them
              const int j0 = max(0, gbase - i), j1 = min(S - 1 - i, gbase + GPP - 1 - i);
              for (int j = j0; j <= j1; ++j) {
                const uint64_t db = sdesc(b_base + j * BN * BK);
                const uint32_t d = tmem + (i + j - gbase) * BN;
#pragma unroll
                for (int kk = 0; kk < BK / 32; ++kk)
                  mma_i8(d, da + 2 * kk, db + 2 * kk, kIdesc, (kb | i | kk) != 0);
              }
              tc_commit(empty_a + 8 * as);
              if (++as == A_STAGES) as = 0, aph ^= 1;
            }
            tc_commit(empty_b + 8 * bs);
            if (++bs == B_STAGES) bs = 0, bph ^= 1;
          }
          tc_commit(tfull);
        }
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;                  // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;        // which half of the BN columns
    const int row = q * 32 + lane;
    const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + half * EPI_COLS;
    int u = 0;
    for (int job = blockIdx.x; job < jobs; job += gridDim.x) {
      const int nt = job % a.n_tiles, mt = (job / a.n_tiles) % a.m_tiles, ks = job / per_split;
      double acc[EPI_COLS];
#pragma unroll
      for (int c = 0; c < EPI_COLS; ++c) acc[c] = 0.0;
#pragma unroll
      for (int p = 0; p < NPASS; ++p, ++u) {
        const int gbase = (NPASS - 1 - p) * GPP;
        mbar_wait(tfull, u & 1);
        tc_fence_after();
#pragma unroll
        for (int gl = GPP - 1; gl >= 0; --gl) {  // smallest weights first
          const double w = ldexp(1.0, -7 * (gbase + gl + 2));
#pragma unroll
          for (int h = 0; h < EPI_COLS / 16; ++h) {  // (16 columns per load: ptxas keeps several loads in flight)
            int v[16];
            tmem_ld16(tbase + gl * BN + h * 16, v);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 16; ++x) acc[h * 16 + x] = fma(i32_to_f64(v[x]), w, acc[h * 16 + x]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
      const int m = mt * BM + row;
      if constexpr (TMA_STORE) {
        // A thread owns one output row (its TMEM lane), so storing from the accumulators makes every
        // warp store touch 32 rows: 8,192 L1 wavefronts per tile, on the path the tensor cores read
        // their shared-memory operands through (probes: this block cost 0.19 ms of the c2 Y·W launch
        // although it runs beside the next tile's MMAs). Instead the scaled values are staged 8 columns
        // at a time in a swizzled 32 × 64-byte tile per warp and leave through the TMA unit, which
        // also clips the ragged edges.
        int ln = lane, wp = warp;
        asm volatile("" : "+r"(ln), "+r"(wp));  // (derived addresses are formed here, not held across the drain loops)
        const int c0 = nt * BN + ((wp - 2) >> 2) * EPI_COLS;
        const double sam = m < a.M ? a.sa[ks * a.sa_stride + m] : 0.0;
        const double* sb = a.sb + ks * a.sb_stride + c0;
        uint8_t* wrow = sC + (wp - 2) * C_WARP_BYTES + ln * (C_COLS * 8);
        const uint32_t wtile = smem_u32(sC + (wp - 2) * C_WARP_BYTES);
        const int sw = (ln >> 1) & 3;  // SWIZZLE_64B: 16-byte piece j of row r at (j ^ ((r >> 1) & 3))
#pragma unroll
        for (int ch = 0; ch < EPI_COLS / C_COLS; ++ch) {
          if (c0 + ch * C_COLS < a.N) {  // (warp-uniform)
            if (ch > 0) {
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < C_COLS / 2; ++j) {
              const int c = ch * C_COLS + 2 * j;
              const double s0 = c0 + c < a.N ? sb[c] : 0.0, s1 = c0 + c + 1 < a.N ? sb[c + 1] : 0.0;
              *reinterpret_cast<double2*>(wrow + ((j ^ sw) << 4)) =
                  make_double2(acc[c] * sam * s0, acc[c + 1] * sam * s1);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (ln == 0) {
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                  "cp.async.bulk.commit_group;" ::"l"(reinterpret_cast<uint64_t>(&tc)),
                  "r"(c0 + ch * C_COLS), "r"(mt * BM + (wp & 3) * 32), "r"(ks), "r"(wtile)
                  : "memory");
            }
          }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      } else if (m < a.M) {  // (the variant without the TMA store: accumulating launches, odd strides)
        const double sam = a.sa[ks * a.sa_stride + m];
        const int c0 = nt * BN + half * EPI_COLS;
        const double* sb = a.sb + ks * a.sb_stride + c0;
        double* crow = a.C + ks * a.c_split_stride + static_cast<long long>(m) * a.ldc + c0;
        const int nvalid = a.N - c0;
        if (nvalid >= EPI_COLS && ((a.ldc | c0) & 1) == 0) {
#pragma unroll
          for (int c = 0; c < EPI_COLS; c += 2) {
            double2 v = make_double2(acc[c] * sam * sb[c], acc[c + 1] * sam * sb[c + 1]);
            if (a.accumulate) {
              const double2 o = *reinterpret_cast<const double2*>(crow + c);
              v.x += o.x;
              v.y += o.y;
            }
            *reinterpret_cast<double2*>(crow + c) = v;
          }
        } else {
#pragma unroll
          for (int c = 0; c < EPI_COLS; ++c) {
            if (c < nvalid) {
              const double v = acc[c] * sam * sb[c];
              crow[c] = a.accumulate ? crow[c] + v : v;
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- slicing
__device__ __forceinline__ double pow2_above(double m) {  // 2^e with m < 2^e (1 for m == 0)
  return m > 0.0 ? ldexp(1.0, ilogb(m) + 1) : 1.0;
}
// The slices of x = scale·r (|r| < 1): a_i = sign(x)·⌊|r|·2^{7(i+1)}⌋ mod 2^7, i.e.
// the base-128 digits of m = ⌊|r|·2⁵⁶⌋ (< 2⁵⁶) with x's sign — the same digits
// as truncating r·2⁷ step by step, from one exact product and one conversion.
// inv56 = 2⁵⁶ / scale (a power of two).
__device__ __forceinline__ void slice8(double x, double inv56, int8_t (&o)[S]) {
  const unsigned long long m = static_cast<unsigned long long>(fabs(x) * inv56);
  const bool neg = x < 0.0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const int v = static_cast<int>((m >> (7 * (S - 1 - i))) & 127u);
    o[i] = static_cast<int8_t>(neg ? -v : v);
  }
}

// Rows of X (R × K, row-major, ldx) → out[S][R][Kp] with a per-row scale
// (one warp per row, the row read once into registers: NIT·128 ≥ Kp columns;
// columns K..Kp-1 written as zero; Kp % 4 == 0, ldx even).
template <int NIT>
__global__ void __launch_bounds__(256) oz_slice_rows_kernel(const double* __restrict__ X, long long ldx, int R, int K,
                                                            int Kp, int8_t* __restrict__ out, long long slice_stride,
                                                            double* __restrict__ scale) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= R) return;
  const double* x = X + static_cast<long long>(row) * ldx;
  double v[NIT][4];
  double m = 0.0;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int k = it * 128 + lane * 4;
#pragma unroll
    for (int e = 0; e < 4; e += 2) {
      double2 p = make_double2(0.0, 0.0);
      if (k + e + 1 < K) {
        p = __ldcs(reinterpret_cast<const double2*>(x + k + e));
      } else if (k + e < K) {
        p.x = x[k + e];
      }
      v[it][e] = p.x;
      v[it][e + 1] = p.y;
      m = fmax(m, fmax(fabs(p.x), fabs(p.y)));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const double sc = pow2_above(m), inv = ldexp(1.0 / sc, 56);
  if (lane == 0) scale[row] = sc;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int k = it * 128 + lane * 4;
    if (k >= Kp) break;
    uint32_t w[S] = {};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int8_t o[S];
      slice8(v[it][e], inv, o);
#pragma unroll
      for (int i = 0; i < S; ++i) w[i] |= static_cast<uint32_t>(static_cast<uint8_t>(o[i])) << (8 * e);
    }
#pragma unroll
    for (int i = 0; i < S; ++i)
      *reinterpret_cast<uint32_t*>(out + i * slice_stride + static_cast<long long>(row) * Kp + k) = w[i];
  }
}

inline cudaError_t slice_rows(const double* X, long long ldx, int R, int K, int Kp, int8_t* out,
                              long long slice_stride, double* scale, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((R + 7) / 8);
  switch ((Kp + 127) / 128) {
    case 1: oz_slice_rows_kernel<1><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 2: oz_slice_rows_kernel<2><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 3: oz_slice_rows_kernel<3><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 4: oz_slice_rows_kernel<4><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 5: oz_slice_rows_kernel<5><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 6: oz_slice_rows_kernel<6><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 7: oz_slice_rows_kernel<7><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    case 8: oz_slice_rows_kernel<8><<<grid, 256, 0, s>>>(X, ldx, R, K, Kp, out, slice_stride, scale); break;
    default: return cudaErrorInvalidValue;  // Kp > 1024: the engine keeps such shapes on DMMA
  }
  return cudaGetLastError();
}

// Σ over `rows` partial rows (stride ldp) per column h < H, one warp per
// column: lane-strided sums then a shuffle tree (a fixed order).
__global__ void oz_colsum_reduce_kernel(const double* __restrict__ part, int rows, int ldp, int H,
                                        double* __restrict__ out, double* __restrict__ out_diag, int diag_ld) {
  const int h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (h >= H) return;
  double s = 0.0;
  for (int z = lane; z < rows; z += 32) s += part[static_cast<long long>(z) * ldp + h];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    out[h] = s;
    if (out_diag) out_diag[static_cast<long long>(h) * diag_ld + h] = s;
  }
}

// Column maxima of X (Krows × R, row-major): atomically folded into
// colmax_bits[R] (non-negative doubles order like their bit patterns).
__global__ void oz_colmax_kernel(const double* __restrict__ X, long long ldx, long long Krows, int R,
                                 unsigned long long* __restrict__ colmax_bits) {
  const int r = blockIdx.x * 32 + (threadIdx.x & 31);
  double m = 0.0;
  if (r < R)
    for (long long k = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5); k < Krows;
         k += static_cast<long long>(gridDim.y) * (blockDim.x >> 5))
      m = fmax(m, fabs(X[k * ldx + r]));
  __shared__ double sm[32][33];
  sm[threadIdx.x >> 5][threadIdx.x & 31] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, sm[w][threadIdx.x]);
    if (r < R) atomicMax(colmax_bits + r, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}
__global__ void oz_scale_from_max_kernel(const unsigned long long* __restrict__ colmax_bits, int R, int Rp,
                                         double fixed, double* __restrict__ scale) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < Rp) scale[r] = fixed > 0.0 ? fixed : (r < R ? pow2_above(__longlong_as_double(colmax_bits[r])) : 1.0);
}

// Columns of X (Krows × R, row-major, ldx) → out[S][Kp/BK][Rp][BK] (K-blocked, Kp % BK == 0)
// with per-column scales scale[Rp]. Tile: 32 columns × 128 rows per CTA
// (256 threads). Optionally writes the CTA's column sums of X to
// colsum[blockIdx.y][Rp] (fixed order: 16 rows per thread, then 8 threads).
__global__ void __launch_bounds__(256) oz_slice_cols_kernel(const double* __restrict__ X, long long ldx,
                                                           long long Krows, int R, int Rp, long long Kp,
                                                           const double* __restrict__ scale,
                                                           int8_t* __restrict__ out, long long slice_stride,
                                                           double* __restrict__ colsum,
                                                           const double* __restrict__ rowscale = nullptr) {
  __shared__ uint32_t sT[S][32][33];
  __shared__ double ssum[8][33];
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + lane;
  const long long k0 = static_cast<long long>(blockIdx.y) * 128;
  const double inv = ldexp(r < Rp ? 1.0 / scale[r] : 1.0, 56);
  double xv[16];  // all 16 loads in flight before any slicing
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const long long k = k0 + ty * 16 + e;
    xv[e] = (r < R && k < Krows) ? __ldcs(X + k * ldx + r) : 0.0;
  }
  if (rowscale) {  // per-row factors of this CTA's 128 rows, staged once
    __shared__ double srs[128];
    if (threadIdx.x < 128) srs[threadIdx.x] = k0 + threadIdx.x < Krows ? rowscale[k0 + threadIdx.x] : 1.0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) xv[e] *= srs[ty * 16 + e];
  }
  double csum = 0.0;
#pragma unroll
  for (int w4 = 0; w4 < 4; ++w4) {  // 4 words = 16 rows per thread
    uint32_t wd[S] = {};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double x = xv[w4 * 4 + e];
      csum += x;
      int8_t o[S];
      slice8(x, inv, o);
#pragma unroll
      for (int i = 0; i < S; ++i) wd[i] |= static_cast<uint32_t>(static_cast<uint8_t>(o[i])) << (8 * e);
    }
#pragma unroll
    for (int i = 0; i < S; ++i) sT[i][lane][ty * 4 + w4] = wd[i];
  }
  ssum[ty][lane] = csum;
  __syncthreads();
  if (colsum && ty == 0 && r < R) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += ssum[w][lane];
    colsum[static_cast<long long>(blockIdx.y) * Rp + r] = s;
  }
  // write: per slice, 32 rows × 32 words (128 B) — a warp writes one row
  for (int idx = threadIdx.x; idx < S * 32 * 32; idx += 256) {
    const int i = idx >> 10, rr = (idx >> 5) & 31, w = idx & 31;
    const int orow = blockIdx.x * 32 + rr;
    const long long k = k0 + w * 4;
    if (orow < Rp && k < Kp)
      *reinterpret_cast<uint32_t*>(out + i * slice_stride + ((k / BK) * Rp + orow) * BK + (k % BK)) = sT[i][rr][w];
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// TMA map of an operand: box = BK k × box_rows × box_slices, 64-byte swizzle;
// K elements valid along k (TMA zero-fills past K and past the valid rows).
inline bool make_map(CUtensorMap* map, const Operand& op, uint64_t K, uint32_t box_rows, uint32_t box_slices) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint32_t estr[4] = {1, 1, 1, 1};
  if (op.blocked) {
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(BK), static_cast<cuuint64_t>(op.rows), (K + BK - 1) / BK,
                          static_cast<cuuint64_t>(S)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(BK), static_cast<cuuint64_t>(op.ld) * BK,
                             static_cast<cuuint64_t>(op.slice_stride)};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(BK), box_rows, 1, box_slices};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(op.base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t dims[3] = {K, static_cast<cuuint64_t>(op.rows), static_cast<cuuint64_t>(S)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(op.ld), static_cast<cuuint64_t>(op.slice_stride)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(BK), box_rows, box_slices};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(op.base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C (+)= A·B over K with A slices (rows scaled by sa) and B slices (rows of Bᵀ
// scaled by sb); K is split into jobs of args.kchunk (multiple of BK).
inline cudaError_t launch_gemm(const Operand& A, const Operand& B, int M, int N, int K, Args args, int num_sms,
                               cudaStream_t s) {
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(oz_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(true));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(oz_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(false));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  CUtensorMap ta, tb8, tb4, tc;
  if (!make_map(&ta, A, K, BM, 1) || !make_map(&tb8, B, K, BN, S) || !make_map(&tb4, B, K, BN, S / 2))
    return cudaErrorInvalidValue;
  {
    // C as a 3-d fp64 tensor (columns, rows, k-splits) for the epilogue's TMA stores: boxes of
    // C_COLS columns × 32 rows, 64-byte swizzle; used when C is overwritten and its strides
    // are multiples of 16 bytes (else the kernel stores from registers)
    const int splits = args.kchunk > 0 ? (K + args.kchunk - 1) / args.kchunk : 1;
    const unsigned long long row_bytes = static_cast<unsigned long long>(args.ldc) * 8;
    const unsigned long long split_bytes =
        splits > 1 ? static_cast<unsigned long long>(args.c_split_stride) * 8 : row_bytes * static_cast<unsigned long long>(M);
    // (split-K launches have long tiles and a small output: they keep the 10-stage A ring instead)
    args.tma_store = splits == 1 && !args.accumulate && row_bytes % 16 == 0 && split_bytes % 16 == 0 &&
                     (reinterpret_cast<uintptr_t>(args.C) & 15) == 0 && encode_fn() != nullptr;
    if (args.tma_store) {
      cuuint64_t dims[3] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(splits)};
      cuuint64_t strides[2] = {row_bytes, split_bytes};
      cuuint32_t box[3] = {C_COLS, 32, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      if (encode_fn()(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, args.C, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        args.tma_store = 0;
    }
    if (!args.tma_store) tc = ta;  // (unused)
  }
  args.blk_a = A.blocked;
  args.blk_b = B.blocked;
  args.M = M;
  args.N = N;
  args.K = K;
  args.m_tiles = (M + BM - 1) / BM;
  args.n_tiles = (N + BN - 1) / BN;
  if (args.kchunk <= 0) args.kchunk = ((K + BK - 1) / BK) * BK;
  args.k_splits = (K + args.kchunk - 1) / args.kchunk;
  const int jobs = args.m_tiles * args.n_tiles * args.k_splits;
  int grid = jobs < num_sms ? jobs : num_sms;
  if (jobs > num_sms) {  // whole n-tile groups per CTA so neighbours share the A tile in L2
    grid = (num_sms / args.n_tiles) * args.n_tiles;
    if (grid <= 0) grid = num_sms;
  }
  if (args.tma_store)
    oz_gemm_kernel<true><<<grid, THREADS, smem_bytes(true), s>>>(ta, tb8, tb4, tc, args);
  else
    oz_gemm_kernel<false><<<grid, THREADS, smem_bytes(false), s>>>(ta, tb8, tb4, tc, args);
  return cudaGetLastError();
}

}  // namespace oz
}  // namespace bscgpu
