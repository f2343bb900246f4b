// Lane-per-point state pass of the BSC E-step (sm_100a).
//
// Reference: the per-state loop of LinearDiscreteModel::estep_impl
// (linear_discrete.cpp:256-303) — log-joint, posterior q, ⟨s⟩ and ⟨s sᵀ⟩ over
// the multi-active states of truncation.cpp:95-169 — for the points whose
// log-joint terms pass the range guard of the multiplicative weights (the
// common case; the rest keep the warp-per-point path of bsc_kernels.cuh).
//
// Split of the work (one E-step chunk):
//   select  select_kernel<H'> (select_kernels.cuh): thread per point — scores,
//           top-H' with a gap proof, unary/pairwise terms u, P. A point that
//           passes the guard is *deferred*: its u, e^u, P, e^P and scalars go to
//           a record tile. Anything else (near-ties, terms outside the range
//           guard) is marked and counted for the fallback launch
//           (enumerate_kernel<…, kPassFallback>, warp per point, bsc_kernels.cuh).
//   states  lane_states_fixed_kernel<γ, H', W> for the BASELINE shapes (below),
//           lane_states_kernel<γ> otherwise: one LANE per deferred point, 32
//           points per warp walking the same depth-first state tree in lockstep,
//           so every index, loop bound and table offset is warp-uniform and all
//           that is left per state is the arithmetic: q(A∪{z}) = q(A)·e^{u_z}·c(A,z),
//           c(A∪{z},w) = c(A,w)·e^{P_zw}, subtree sums, and the moment updates.
//           Per-point arrays live in shared memory as [slot][32 lanes] (one
//           conflict-free 256-byte row per slot).
//   finish  lane_finish_slice_kernel<PT> (finish_slice_kernels.cuh) on the sliced
//           path: log Z, the singleton weights of all H units, the candidate
//           marginals and the candidate pairs of Σ⟨ssᵀ⟩, with the ⟨s⟩ rows cut into
//           the int8 operand of Yᵀ⟨S⟩ in shared memory; lane_finish_kernel (below)
//           writes fp64 ⟨s⟩ rows instead (BSC_GEMM=dmma, BSC_FUSED_FINISH=0).
//
// Moments by subtree sums (post-order): sub(A) = q(A) + Σ_children sub(child);
// ⟨s_p⟩ = Σ_{A: max A = p} sub(A), ⟨s_p s_q⟩ = Σ_{A: max A = q, p∈A} sub(A).
// The depth-first order is the reference's prefix-first pattern order
// (truncation.cpp:116-147), so the tree is exactly its state set.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "bsc_kernels.cuh"

namespace bscgpu {

// Record tile (per 32 consecutive points of a chunk), doubles [field][32]
// (lane_rec_fields, bsc_kernels.cuh):
//   0 shift (mode 1)   1 zs1 (zero + singleton weights relative to mxs)   2 mxs
//   3 pad   4.. u[H']   .. e^u[H']   .. P[np]   .. e^P[np]      (np = H'(H'−1)/2)
// Output tile: 0 shift   1 Σ multi-active weights   2.. M[nm]  (nm = H'(H'+1)/2,
// upper triangle with diagonal, row-major: ⟨s_p⟩ on the diagonal)
__host__ __device__ inline int lane_out_fields(int hp) { return 2 + hp * (hp + 1) / 2; }
// shared memory per warp of lane_states_kernel<GM>
__host__ __device__ inline int lane_smem_bytes(int hp, int gm) {
  const int np = hp * (hp - 1) / 2, nm = hp * (hp + 1) / 2;
  return (hp + np + (gm > 2 ? gm - 2 : 0) * hp + nm) * 256;
}

// point modes (EnumArgs::pmode): kModeDone / kModeShift (shift = the bound
// in the record) / kModeMax (shift = exact maximum, computed here) /
// kModeFallback (bsc_kernels.cuh)

struct LaneArgs {
  int N, hp;
  const double* rec;
  double* out;
  const int* pmode;
};

// per-lane shared arrays: element i of the calling lane's array at byte offset i·256
__device__ __forceinline__ double lds_(const char* p, int i) { return *reinterpret_cast<const double*>(p + i * 256); }
__device__ __forceinline__ void sts_(char* p, int i, double v) { *reinterpret_cast<double*>(p + i * 256) = v; }

// strict upper triangle (p < q): pidx = prow(p) + q;  with diagonal (p ≤ q): tri = mrow(p) + q
__device__ __forceinline__ int prow_(int p, int hp) { return p * (2 * hp - p - 1) / 2 - p - 1; }
__device__ __forceinline__ int mrow_(int p, int hp) { return p * (2 * hp - p + 1) / 2 - p; }

// Weight pass below node A (|A| = K, max x, weight qA, members path[0..K)):
// returns Σ_children sub(child) and adds every descendant's subtree sum into
// the moment array M. c(A, w) is e^P row x for K = 1, else cv level K−2.
template <int K, int GM>
__device__ __forceinline__ double wnode(const char* eu, const char* eP, char* cv, char* M, int hp, double qA, int x,
                                        int (&path)[8]) {
  double ch = 0.0;
  int mrow[K];
#pragma unroll
  for (int i = 0; i < K; ++i) mrow[i] = mrow_(path[i], hp);
  const int px = prow_(x, hp);
  if constexpr (K + 1 < GM) {
    for (int z = x + 1; z < hp; ++z) {
      const double c = K == 1 ? lds_(eP, px + z) : lds_(cv, (K - 2) * hp + z);
      const double qz = qA * lds_(eu, z) * c;
      const int pz = prow_(z, hp);
      for (int w = z + 1; w < hp; ++w) {
        const double cw = K == 1 ? lds_(eP, px + w) : lds_(cv, (K - 2) * hp + w);
        sts_(cv, (K - 1) * hp + w, cw * lds_(eP, pz + w));
      }
      path[K] = z;
      const double s = qz + wnode<K + 1, GM>(eu, eP, cv, M, hp, qz, z, path);
      const int zz = mrow_(z, hp) + z;
      double m[K + 1];
      m[K] = lds_(M, zz);
#pragma unroll
      for (int i = 0; i < K; ++i) m[i] = lds_(M, mrow[i] + z);
      sts_(M, zz, m[K] + s);
#pragma unroll
      for (int i = 0; i < K; ++i) sts_(M, mrow[i] + z, m[i] + s);
      ch += s;
    }
  } else {
    // leaves, two per iteration (their moment entries are distinct)
    int z = x + 1;
    for (; z + 1 < hp; z += 2) {
      const double c0 = K == 1 ? lds_(eP, px + z) : lds_(cv, (K - 2) * hp + z);
      const double c1 = K == 1 ? lds_(eP, px + z + 1) : lds_(cv, (K - 2) * hp + z + 1);
      const double e0 = lds_(eu, z), e1 = lds_(eu, z + 1);
      const int zz0 = mrow_(z, hp) + z, zz1 = mrow_(z + 1, hp) + z + 1;
      double m0[K + 1], m1[K + 1];
      m0[K] = lds_(M, zz0);
      m1[K] = lds_(M, zz1);
#pragma unroll
      for (int i = 0; i < K; ++i) {
        m0[i] = lds_(M, mrow[i] + z);
        m1[i] = lds_(M, mrow[i] + z + 1);
      }
      const double s0 = qA * e0 * c0, s1 = qA * e1 * c1;
      sts_(M, zz0, m0[K] + s0);
      sts_(M, zz1, m1[K] + s1);
#pragma unroll
      for (int i = 0; i < K; ++i) {
        sts_(M, mrow[i] + z, m0[i] + s0);
        sts_(M, mrow[i] + z + 1, m1[i] + s1);
      }
      ch += s0 + s1;
    }
    if (z < hp) {
      const double c0 = K == 1 ? lds_(eP, px + z) : lds_(cv, (K - 2) * hp + z);
      const double s0 = qA * lds_(eu, z) * c0;
      const int zz0 = mrow_(z, hp) + z;
      sts_(M, zz0, lds_(M, zz0) + s0);
#pragma unroll
      for (int i = 0; i < K; ++i) sts_(M, mrow[i] + z, lds_(M, mrow[i] + z) + s0);
      ch += s0;
    }
  }
  return ch;
}

// Maximum log-joint (relative to the zero state) below node A: the additive
// twin of wnode (rel(A∪{z}) = rel(A) + u_z + Σ_{a∈A} P_az), for the points
// whose cheap upper bound was too loose to use as the shift (mode 2).
template <int K, int GM>
__device__ __forceinline__ double mnode(const char* U, const char* P, char* cv, int hp, double relA, int x) {
  double m = -INFINITY;
  const int px = prow_(x, hp);
  for (int z = x + 1; z < hp; ++z) {
    const double c = K == 1 ? lds_(P, px + z) : lds_(cv, (K - 2) * hp + z);
    const double rz = relA + lds_(U, z) + c;
    m = fmax(m, rz);
    if constexpr (K + 1 < GM) {
      const int pz = prow_(z, hp);
      for (int w = z + 1; w < hp; ++w) {
        const double cw = K == 1 ? lds_(P, px + w) : lds_(cv, (K - 2) * hp + w);
        sts_(cv, (K - 1) * hp + w, cw + lds_(P, pz + w));
      }
      m = fmax(m, mnode<K + 1, GM>(U, P, cv, hp, rz, z));
    }
  }
  return m;
}

// ---------------------------------------------------------------------------
// Compile-time shapes (the BASELINE workloads' H', γ ≥ 3): the same tree walk,
// restructured so the deepest level runs out of registers with constant
// shared-memory offsets.
//
// Node A at depth K = γ−2 (its children are the leaf parents), max x, members
// a_1..a_K: with ce[w] = e^{u_w}·c(A,w) (a register vector, w > x)
//   child  B = A∪{Z}:   q_B = q_A·ce[Z]
//   leaf   B∪{w}, w>Z:  q = q_B·ce[w]·e^{P_Zw}
// Every descendant of A contains all of A's members, so its contribution to
// M[a_i][z] is the same for each i, and equals its contribution to M[z][z]
// (z its maximum): one register accumulator R[z] per column collects them and
// is flushed once per A into M[z][z] and the K member rows. Only the leaf-
// parent row M[Z][w] is updated per leaf — at a constant offset. Levels above
// run over z at run time (coupling rows built by a dispatched unrolled block).
#ifndef LANE_EPS_ROW
#define LANE_EPS_ROW (HP / 2 - 1)  // first e^P row still staged when e^P is read through L1
#endif
#ifndef LANE_EPG_MIN_PAIRS
#define LANE_EPG_MIN_PAIRS 60  // e^P read through L1 when H'(H'-1)/2 exceeds this
#endif
template <int HP, int GM>
struct LaneShape {
  static_assert(GM >= 3, "compile-time walk needs gamma >= 3");
  static constexpr int NP = HP * (HP - 1) / 2, NM = HP * (HP + 1) / 2;
  // γ = 4: the coupling row of a deepest node {r, z} is never stored. The part its entries share,
  // e^{u_w}·e^{P_rw}, is held in registers per root r, and the node forms
  // ce[w] = e^{u_w}·e^{P_rw}·e^{P_zw} in a block dispatched on z (compile-time e^P offsets), which
  // saves the row's write, its read back and its H'−2 slots per lane: 121 -> 111 at (12, 4), 8
  // resident warps per SM instead of 7 (two warps per CTA, lane_engine.cu).
  static constexpr bool HOIST = GM == 4;
  static constexpr int CV_LEVELS = HOIST ? 0 : GM - 3;  // stored coupling rows (depths 2 .. γ−2)
  // e^P staged in shared memory, or (EP_GLOBAL) read from the record tile ([pair][32 lanes])
  // through the read-only path, leaving the slots to e^u, the coupling rows and M. Measured:
  // (14, 5) 3 -> 5 warps/SM, state pass 20.0 -> 12.6 ms at c3; (12, 4) fully unstaged reached
  // 8 warps/SM but 0.45 -> 0.48 ms at c2. With the heavily read rows staged (EPS_ROW below):
  // c3 10.6 ms, c2 0.423 ms (7 warps/SM); (10, 4) stays fully staged.
  static constexpr bool EP_GLOBAL = NP > LANE_EPG_MIN_PAIRS;
  static constexpr int O_EU = 0, O_EP = HP, O_CV = O_EP + (EP_GLOBAL ? 0 : NP);
  // coupling row c (written by depth-(c+1) nodes for their children) only ever holds
  // w ≥ c + 2 (a depth-K node's child is ≥ K): rows packed without those slots, so
  // (14, 5) fits 6 warps per SM. cvb(c) + w is the slot of entry w of row c.
  __host__ __device__ static constexpr int cv_start(int c) { return c <= 0 ? O_CV : cv_start(c - 1) + HP - (c - 1) - 2; }
  __host__ __device__ static constexpr int cvb(int c) { return cv_start(c) - (c + 2); }
  // EP_GLOBAL: the e^P rows p ≥ EPS_ROW (pairs from EPS_FIRST on) are still staged. A
  // deepest-level node with maximum x reads rows x+1 … H'−1, so row p is read by the C(p, γ−2)
  // nodes below it: at (14, 5) rows 6-12 take 94 % of those reads in 28 slots (5 warps/SM).
  static constexpr int EPS_ROW = EP_GLOBAL ? LANE_EPS_ROW : HP;
  static constexpr int EPS_FIRST = EPS_ROW * (2 * HP - EPS_ROW - 1) / 2;
  static constexpr int EPS_N = EP_GLOBAL ? NP - EPS_FIRST : 0;
  static constexpr int O_EPS = cv_start(CV_LEVELS);
  static constexpr int O_M = O_EPS + EPS_N;
  // element i of this lane's e^P (E: record tile or the staged slots, stride 32 doubles;
  // S: this lane's slot 0). i is warp-uniform, so the split branch never diverges.
  __device__ static __forceinline__ double ep(const double* S, const double* E, int i) {
    if constexpr (EP_GLOBAL)
      return i >= EPS_FIRST ? S[(O_EPS + i - EPS_FIRST) * 32] : __ldg(E + i * 32);
    else
      return E[i * 32];
  }
  static constexpr int SLOTS = O_M + NM;
  // The leaf-parent rows M[Z][·] with Z ≥ MR_ROW accumulate in registers over the whole walk
  // (deep_child's indices are compile-time) and are added to the shared-memory triangle at the
  // end: row Z is visited by the C(Z, γ−2) deepest nodes below it, so the last six rows
  // (21 entries) take 85 % of the leaf updates at (12, 4) and 87 % at (14, 5), and a leaf
  // there costs one shared-memory read (e^P) instead of two reads and a write.
#ifndef LANE_MR_ROWS
#define LANE_MR_ROWS 6
#endif
  static constexpr int MR_ROW = HP - 1 - (LANE_MR_ROWS < HP - 1 ? LANE_MR_ROWS : HP - 1);
  static constexpr int MR_FIRST = MR_ROW * (2 * HP - MR_ROW - 1) / 2;
  static constexpr int NMR = NP - MR_FIRST > 0 ? NP - MR_FIRST : 1;
  __host__ __device__ static constexpr int pidx(int p, int q) { return p * (2 * HP - p - 1) / 2 + (q - p - 1); }
  __host__ __device__ static constexpr int tri(int p, int q) { return p * (2 * HP - p + 1) / 2 + (q - p); }
};

// lane-private slot i of the per-warp [slot][32] arrays (S = base + lane)
#define LS(i) S[(i) * 32]

// Coupling row of child A∪{Z} (node A at depth K < γ−2): cv[K−1][w] =
// c(A,w)·e^{P_Zw}, w > Z; c(A,·) = e^P row x (runtime, xrow) for K = 1, else cv[K−2].
template <int HP, int GM, int K, int Z>
__device__ __forceinline__ void cv_block(double* S, const double* __restrict__ E, int xrow) {
  using F = LaneShape<HP, GM>;
  constexpr int NW = HP - 1 - Z > 0 ? HP - 1 - Z : 1;
  double v[NW];
#pragma unroll
  for (int w = Z + 1; w < HP; ++w) {
    const double cw = K == 1 ? F::ep(S, E, xrow + w) : LS(F::cvb(K - 2) + w);
    v[w - Z - 1] = cw * F::ep(S, E, F::pidx(Z, w));
  }
#pragma unroll
  for (int w = Z + 1; w < HP; ++w) LS(F::cvb(K - 1) + w) = v[w - Z - 1];
}

#define LANE_CASES(M_)                                                                                      \
  M_(0) M_(1) M_(2) M_(3) M_(4) M_(5) M_(6) M_(7) M_(8) M_(9) M_(10) M_(11) M_(12) M_(13) M_(14) M_(15)

template <int HP, int GM, int K>
__device__ __forceinline__ void cv_dispatch(int z, double* S, const double* __restrict__ E, int xrow) {
  switch (z) {
#define LANE_CV_CASE(v)                                                       \
  case v:                                                                     \
    if constexpr (v < HP - 1) cv_block<HP, GM, K, (v < HP - 1 ? v : 0)>(S, E, xrow); \
    break;
    LANE_CASES(LANE_CV_CASE)
#undef LANE_CV_CASE
    default:
      break;
  }
}

// HOIST (γ = 4): ce[w] = pc[w]·e^{P_Zw}, w > Z, of the deepest node {r, Z} (pc = e^{u_w}·e^{P_rw}).
template <int HP, int GM, int Z>
__device__ __forceinline__ void ce_block(double* S, const double* __restrict__ E, const double (&pc)[HP], double (&ce)[HP]) {
  using F = LaneShape<HP, GM>;
#pragma unroll
  for (int w = Z + 1; w < HP; ++w) ce[w] = pc[w] * F::ep(S, E, F::pidx(Z, w));
}
template <int HP, int GM>
__device__ __forceinline__ void ce_dispatch(int z, double* S, const double* __restrict__ E, const double (&pc)[HP],
                                            double (&ce)[HP]) {
  switch (z) {
#define LANE_CE_CASE(v)                                                         \
  case v:                                                                       \
    if constexpr (v < HP - 1) ce_block<HP, GM, (v < HP - 1 ? v : 0)>(S, E, pc, ce); \
    break;
    LANE_CASES(LANE_CE_CASE)
#undef LANE_CE_CASE
    default:
      break;
  }
}

// Child A∪{Z} of the deepest node A and its leaves.
template <int HP, int GM, int Z>
__device__ __forceinline__ void deep_child(double* S, const double* __restrict__ E, double qA, const double (&ce)[HP], double (&R)[HP],
                                           double (&MR)[LaneShape<HP, GM>::NMR], double& ch) {
  using F = LaneShape<HP, GM>;
  const double qz = qA * ce[Z];
  double s = qz;
  if constexpr (Z < HP - 1) {
    constexpr int NW = HP - 1 - Z;
    double q[NW], m[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const int w = Z + 1 + j;
      q[j] = qz * ce[w] * F::ep(S, E, F::pidx(Z, w));
      if constexpr (Z < F::MR_ROW) m[j] = LS(F::O_M + F::tri(Z, w));
    }
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const int w = Z + 1 + j;
      if constexpr (Z < F::MR_ROW)
        LS(F::O_M + F::tri(Z, w)) = m[j] + q[j];
      else
        MR[F::pidx(Z, w) - F::MR_FIRST] += q[j];
      R[w] += q[j];
      s += q[j];
    }
  }
  R[Z] += s;
  ch += s;
}

template <int HP, int GM, int Z>
__device__ __forceinline__ void deep_pred(double* S, const double* __restrict__ E, double qA, int x, const double (&ce)[HP], double (&R)[HP],
                                          double (&MR)[LaneShape<HP, GM>::NMR], double& ch) {
  if (Z > x) deep_child<HP, GM, Z>(S, E, qA, ce, R, MR, ch);
  if constexpr (Z + 1 < HP) deep_pred<HP, GM, Z + 1>(S, E, qA, x, ce, R, MR, ch);
}

// Duff-style dispatch on the node maximum x: case x falls through the
// unrolled blocks Z = x+1 … H'−1 (one uniform indirect branch per node).
#define LANE_FT_CASES(BLOCK)                                                                                     \
  BLOCK(0, 1) BLOCK(1, 2) BLOCK(2, 3) BLOCK(3, 4) BLOCK(4, 5) BLOCK(5, 6) BLOCK(6, 7) BLOCK(7, 8) BLOCK(8, 9)     \
  BLOCK(9, 10) BLOCK(10, 11) BLOCK(11, 12) BLOCK(12, 13) BLOCK(13, 14) BLOCK(14, 15)

// Node A (|A| = K ≤ γ−2, max x, weight qA, members path[0..K)): walks its
// children, returns Σ_children sub(child).
template <int HP, int GM, int K>
__device__ __forceinline__ double fnode(double* S, const double* __restrict__ E, double qA, int x, int (&path)[8],
                                        double (&MR)[LaneShape<HP, GM>::NMR], const double (&pc)[HP]) {
  using F = LaneShape<HP, GM>;
  int orow[K + 1];
#pragma unroll
  for (int i = 0; i < K; ++i) orow[i] = F::O_M + mrow_(path[i], HP);
  const int xrow = prow_(x, HP);
  double ch = 0.0;
  if constexpr (K == GM - 2) {
    double ce[HP], R[HP];
#pragma unroll
    for (int w = 0; w < HP; ++w) R[w] = 0.0;
    if constexpr (GM < 5) {
      // predicated unrolled blocks (fewer, shorter nodes: cheaper than the indirect branch)
      if constexpr (F::HOIST && K == 2) {
#pragma unroll
        for (int w = 0; w < HP; ++w) ce[w] = 0.0;
        ce_dispatch<HP, GM>(x, S, E, pc, ce);
      } else {
#pragma unroll
        for (int w = 0; w < HP; ++w) {
          ce[w] = 0.0;
          if (w > x) ce[w] = LS(F::O_EU + w) * (K == 1 ? F::ep(S, E, xrow + w) : LS(F::cvb(K - 2) + w));
        }
      }
      deep_pred<HP, GM, (K < HP ? K : 0)>(S, E, qA, x, ce, R, MR, ch);
#pragma unroll
      for (int z = 0; z < HP; ++z) {
        if (z > x) {
          double m[K + 1];
          m[K] = LS(F::O_M + F::tri(z, z));
#pragma unroll
          for (int i = 0; i < K; ++i) m[i] = S[(orow[i] + z) * 32];
          LS(F::O_M + F::tri(z, z)) = m[K] + R[z];
#pragma unroll
          for (int i = 0; i < K; ++i) S[(orow[i] + z) * 32] = m[i] + R[z];
        }
      }
    } else {
    // ce[w] = e^{u_w}·c(A,w), w > x
      switch (x) {
  #define LANE_CE(c_, Z_)                                                                        \
    case c_:                                                                                     \
      if constexpr (Z_ < HP) {                                                                   \
        constexpr int Zc = Z_ < HP ? Z_ : 0;                                                     \
        ce[Zc] = LS(F::O_EU + Zc) * (K == 1 ? F::ep(S, E, xrow + Zc) : LS(F::cvb(K - 2) + Zc)); \
      }                                                                                          \
      [[fallthrough]];
        LANE_FT_CASES(LANE_CE)
  #undef LANE_CE
        default:
          break;
      }
      switch (x) {
  #define LANE_DC(c_, Z_)                                                     \
    case c_:                                                                  \
      if constexpr (Z_ < HP) deep_child<HP, GM, (Z_ < HP ? Z_ : 0)>(S, E, qA, ce, R, MR, ch); \
      [[fallthrough]];
        LANE_FT_CASES(LANE_DC)
  #undef LANE_DC
        default:
          break;
      }
      // flush the column accumulators: M[z][z] and the members' rows, z > x
      switch (x) {
  #define LANE_FL(c_, Z_)                                                           \
    case c_:                                                                        \
      if constexpr (Z_ < HP) {                                                      \
        constexpr int Zc = Z_ < HP ? Z_ : 0;                                        \
        double m[K + 1];                                                            \
        m[K] = LS(F::O_M + F::tri(Zc, Zc));                                         \
        _Pragma("unroll") for (int i = 0; i < K; ++i) m[i] = S[(orow[i] + Zc) * 32]; \
        LS(F::O_M + F::tri(Zc, Zc)) = m[K] + R[Zc];                                 \
        _Pragma("unroll") for (int i = 0; i < K; ++i) S[(orow[i] + Zc) * 32] = m[i] + R[Zc]; \
      }                                                                             \
      [[fallthrough]];
        LANE_FT_CASES(LANE_FL)
  #undef LANE_FL
        default:
          break;
      }
    }
  } else {
    // children at the deepest level form their own coupling factors; with HOIST (γ = 4, this
    // node a root) the part they share, e^{u_w}·e^{P_xw}, stays in registers
    auto children = [&](const double (&pcx)[HP]) {
      for (int z = x + 1; z < HP; ++z) {
        const double c = K == 1 ? F::ep(S, E, xrow + z) : S[(F::cvb(K - 2) + z) * 32];
        const double qz = qA * S[(F::O_EU + z) * 32] * c;
        if constexpr (!(F::HOIST && K + 1 == GM - 2)) cv_dispatch<HP, GM, K>(z, S, E, xrow);
        path[K] = z;
        const double s = qz + fnode<HP, GM, (K + 1 < GM - 1 ? K + 1 : K)>(S, E, qz, z, path, MR, pcx);
        const int zz = F::O_M + mrow_(z, HP) + z;
        double m[K + 1];
        m[K] = S[zz * 32];
#pragma unroll
        for (int i = 0; i < K; ++i) m[i] = S[(orow[i] + z) * 32];
        S[zz * 32] = m[K] + s;
#pragma unroll
        for (int i = 0; i < K; ++i) S[(orow[i] + z) * 32] = m[i] + s;
        ch += s;
      }
    };
    if constexpr (F::HOIST && K == 1) {
      double pcn[HP];
#pragma unroll
      for (int w = 0; w < HP; ++w) {
        pcn[w] = 0.0;
        if (w > x + 1) pcn[w] = LS(F::O_EU + w) * F::ep(S, E, xrow + w);
      }
      children(pcn);
    } else {
      children(pc);
    }
  }
  return ch;
}
#undef LS

// One warp per CTA, one tile of 32 consecutive points of the chunk; lane l
// owns point 32·tile + l. Run-time H' (generic tree walk, wnode).
template <int GM>
__global__ void __launch_bounds__(32) lane_states_kernel(LaneArgs a) {
  extern __shared__ __align__(16) double lsm[];
  const int lane = threadIdx.x;
  const int hp = a.hp, np = hp * (hp - 1) / 2, nm = hp * (hp + 1) / 2;
  const long long tile = blockIdx.x;
  const long long n = tile * 32 + lane;
  const int mode = n < a.N ? a.pmode[n] : kModeDone;
  const bool live = mode == kModeShift || mode == kModeMax;
  if (!__any_sync(0xffffffffu, live)) return;
  char* base = reinterpret_cast<char*>(lsm) + lane * 8;
  char* eu = base;
  char* eP = eu + hp * 256;
  char* cv = eP + np * 256;
  char* M = cv + (GM > 2 ? GM - 2 : 0) * hp * 256;
  const double* rt = a.rec + tile * lane_rec_fields(hp) * 32 + lane;
  const int fu = 4, feu = 4 + hp, fP = 4 + 2 * hp, feP = 4 + 2 * hp + np;
  int path[8];

  double shift = live ? rt[0] : 0.0;
  if (__any_sync(0xffffffffu, mode == kModeMax)) {
    // exact maximum over the multi-active states (u staged in the M region)
    for (int p = 0; p < hp; ++p) sts_(M, p, live ? rt[(fu + p) * 32] : 0.0);
    for (int e = 0; e < np; ++e) sts_(eP, e, live ? rt[(fP + e) * 32] : 0.0);
    double m = -INFINITY;
    for (int r = 0; r < hp; ++r) {
      const double ur = lds_(M, r);
      m = fmax(m, fmax(ur, mnode<1, GM>(M, eP, cv, hp, ur, r)));
    }
    if (mode == kModeMax) shift = fmax(rt[2 * 32], m);
  }
  for (int p = 0; p < hp; ++p) sts_(eu, p, live ? rt[(feu + p) * 32] : 0.0);
  for (int e = 0; e < np; ++e) sts_(eP, e, live ? rt[(feP + e) * 32] : 0.0);
  for (int i = 0; i < nm; ++i) sts_(M, i, 0.0);
  double zm = 0.0;
  for (int r = 0; r < hp; ++r) {
    const double qr = live ? exp_nonpos(rt[(fu + r) * 32] - shift) : 0.0;
    path[0] = r;
    const double ch = wnode<1, GM>(eu, eP, cv, M, hp, qr, r, path);
    const int rr = mrow_(r, hp) + r;
    sts_(M, rr, lds_(M, rr) + qr + ch);
    zm += ch;
  }
  if (live) {
    double* ot = a.out + tile * lane_out_fields(hp) * 32 + lane;
    ot[0] = shift;
    ot[32] = zm;
    for (int i = 0; i < nm; ++i) ot[(2 + i) * 32] = lds_(M, i);
  }
}

// The compile-time walk for H' = HP, γ = GM (layout LaneShape<HP, GM>).
// WPC warps per CTA (independent tiles; no CTA-wide synchronisation): two where that lets one
// more warp fit beside the 1 KB of shared memory the system reserves per CTA.
template <int GM, int HP, int WPC>
__global__ void __launch_bounds__(32 * WPC, 1) lane_states_fixed_kernel(LaneArgs a) {
  using F = LaneShape<HP, GM>;
  extern __shared__ __align__(16) double lsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long tile = static_cast<long long>(blockIdx.x) * WPC + wib;
  const long long n = tile * 32 + lane;
  const int mode = n < a.N ? a.pmode[n] : kModeDone;
  const bool live = mode == kModeShift || mode == kModeMax;
  if (!__any_sync(0xffffffffu, live)) return;
  double* S = lsm + wib * (F::SLOTS * 32) + lane;
  char* base = reinterpret_cast<char*>(lsm) + wib * (F::SLOTS * 256) + lane * 8;
  const double* rt = a.rec + tile * lane_rec_fields(HP) * 32 + lane;
  constexpr int fu = 4, feu = 4 + HP, fP = 4 + 2 * HP, feP = 4 + 2 * HP + F::NP;

  double ur[HP];
#pragma unroll
  for (int r = 0; r < HP; ++r) ur[r] = live ? rt[(fu + r) * 32] : 0.0;
  double shift = live ? rt[0] : 0.0;
  if (__any_sync(0xffffffffu, mode == kModeMax)) {
    // exact maximum: u and the coupling sums staged in the M region
    char* U = base + F::O_M * 256;
    char* cvm = U + HP * 256;
    const char* eP = reinterpret_cast<const char*>(rt + fP * 32);  // P from the record tile
#pragma unroll
    for (int p = 0; p < HP; ++p) sts_(U, p, ur[p]);
    double m = -INFINITY;
    for (int r = 0; r < HP; ++r) {
      const double u = lds_(U, r);
      m = fmax(m, fmax(u, mnode<1, GM>(U, eP, cvm, HP, u, r)));
    }
    if (mode == kModeMax) shift = fmax(rt[2 * 32], m);
  }
#pragma unroll
  for (int p = 0; p < HP; ++p) S[(F::O_EU + p) * 32] = live ? rt[(feu + p) * 32] : 0.0;
  // e^P of this lane's point (dead lanes: unused values)
  const double* E = rt + feP * 32;
  if constexpr (!F::EP_GLOBAL) {
    for (int e = 0; e < F::NP; ++e) S[(F::O_EP + e) * 32] = live ? rt[(feP + e) * 32] : 0.0;
    E = S + F::O_EP * 32;
  } else {
    for (int e = 0; e < F::EPS_N; ++e) S[(F::O_EPS + e) * 32] = live ? rt[(feP + F::EPS_FIRST + e) * 32] : 0.0;
  }
  for (int i = 0; i < F::NM; ++i) S[(F::O_M + i) * 32] = 0.0;
  int path[8];
  double zm = 0.0;
  double MR[F::NMR];
#pragma unroll
  for (int i = 0; i < F::NMR; ++i) MR[i] = 0.0;
  double pc0[HP];  // (unused by the root level)
#pragma unroll
  for (int i = 0; i < HP; ++i) pc0[i] = 0.0;
#pragma unroll 1
  for (int r = 0; r < HP; ++r) {
    double u = ur[0];
#pragma unroll
    for (int j = 1; j < HP; ++j) u = r == j ? ur[j] : u;
    const double qr = live ? exp_nonpos(u - shift) : 0.0;
    path[0] = r;
    const double ch = fnode<HP, GM, 1>(S, E, qr, r, path, MR, pc0);
    const int rr = F::O_M + mrow_(r, HP) + r;
    S[rr * 32] += qr + ch;
    zm += ch;
  }
  // the register-held leaf-parent rows join the triangle
#pragma unroll
  for (int p = F::MR_ROW; p < HP - 1; ++p)
#pragma unroll
    for (int q = p + 1; q < HP; ++q) S[(F::O_M + F::tri(p, q)) * 32] += MR[F::pidx(p, q) - F::MR_FIRST];
  if (live) {
    double* ot = a.out + tile * lane_out_fields(HP) * 32 + lane;
    ot[0] = shift;
    ot[32] = zm;
    for (int i = 0; i < F::NM; ++i) ot[(2 + i) * 32] = S[(F::O_M + i) * 32];
  }
}

struct FinishArgs {
  int N, H, Hp, hp;
  const double* out;
  const int* pmode;
  const uint32_t* cand;  // N × hp, ascending
  const double* y2;
  const double* B;       // N × Hp rows of Y·W (singleton terms)
  const double* gdiag;   // diag(G)
  double* ES;
  double* ssT;           // H × H; strict upper triangle accumulated as fixed point (pair_fx_add)
  double* cta_scalars;   // [gridDim.x][2] Σ log Z_n (deferred points), 0
  double base0, inv2s, dlp;
  double fx_scale;       // 2^k of the fixed-point pair accumulation
};

// Warp per deferred point (linear_discrete.cpp:272-304 at T = 1): the singleton
// weights of all H units relative to the point's shift (recomputed from the B
// row, as the selection pass leaves them), log Z = base + shift + log(z)
// (core.cpp:36-45), the normalised ⟨s_n⟩ row (candidates take their marginals
// from the state pass) and the candidate pairs of Σ⟨ssᵀ⟩ (fixed point:
// order-independent, so the statistics are bitwise reproducible).
template <int MAXJ>
__global__ void __launch_bounds__(256) lane_finish_kernel(FinishArgs a) {
  __shared__ double red[8];
  __shared__ uint16_t pq[256];  // moment entry o → (p, q), p ≤ q (row-major upper triangle with diagonal)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int hp = a.hp, nm = hp * (hp + 1) / 2;
  for (int o = threadIdx.x; o < nm; o += blockDim.x) {
    int idx = o, p = 0;
    while (idx >= hp - p) {
      idx -= hp - p;
      ++p;
    }
    pq[o] = static_cast<uint16_t>(p | ((p + idx) << 8));
  }
  __syncthreads();
  const int row_lines = (a.Hp * 8 + 127) / 128;
  double lse_acc = 0.0;
  for (int n = blockIdx.x * (blockDim.x >> 5) + wib; n < a.N; n += nwarps) {
    // the B rows of the next two points of this warp: into L2, and the next one into L1
    if (n + 2 * nwarps < a.N)
      for (int l = lane; l < row_lines; l += 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.B + (long long)(n + 2 * nwarps) * a.Hp + l * 16));
    if (n + nwarps < a.N)
      for (int l = lane; l < row_lines; l += 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.B + (long long)(n + nwarps) * a.Hp + l * 16));
    const int mode = a.pmode[n];
    if (mode != kModeShift && mode != kModeMax) continue;
    const long long tile = n >> 5;
    const double* ot = a.out + tile * lane_out_fields(hp) * 32 + (n & 31);
    const double shift = ot[0], zm = ot[32];
    const double* brow = a.B + (long long)n * a.Hp;
    double e[MAXJ];
    double zs = 0.0;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      e[j] = 0.0;
      if (h < a.H) {
        // rel = fma(inv2s, 2b − G_hh, dlp), the selection pass's rounding: shift ≥ rel
        e[j] = exp_nonpos(__fma_rn(a.inv2s, __fma_rn(2.0, brow[h], -a.gdiag[h]), a.dlp) - shift);
        zs += e[j];
      }
    }
    zs = warp_sum(zs) + exp_nonpos(-shift);  // + the zero state
    const double z1 = zs + zm;
    const double inv_z = 1.0 / z1;
    if (lane == 0) lse_acc += (a.base0 - a.y2[n] * a.inv2s) + (shift + log(z1));
    double* esrow = a.ES + (long long)n * a.Hp;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < a.H) esrow[h] = e[j] * inv_z;
    }
    __syncwarp();
    const uint32_t* cn = a.cand + (long long)n * hp;
    // the moment entries this lane finishes: lane, lane + 32, …
    for (int o = lane; o < nm; o += 32) {
      const int p = pq[o] & 0xff, q = pq[o] >> 8;
      const double v = ot[(2 + o) * 32] * inv_z;
      if (q == p)
        esrow[cn[p]] = v;
      else
        pair_fx_add(a.ssT + (long long)cn[p] * a.H + cn[q], v, a.fx_scale);
    }
    __syncwarp();
  }
  if (lane == 0) red[wib] = lse_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) l += red[w];
    a.cta_scalars[2 * blockIdx.x] = l;
    a.cta_scalars[2 * blockIdx.x + 1] = 0.0;
  }
}

}  // namespace bscgpu
