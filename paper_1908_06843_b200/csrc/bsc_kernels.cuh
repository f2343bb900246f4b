// Hand-written sm_100a kernels of the BSC truncated-EM E/M-step.
//
// Reference path: LinearDiscreteModel::estep_impl (linear_discrete.cpp:202-325)
// and ::mstep (:336-408) of /root/reference/proj/src. Layout in HBM (all fp64,
// leading dims padded to multiples of 8 doubles, pads zero):
//   Y  N × Dp   data points (one per row), resident for the whole run
//   W  D × Hp   dictionary
//   G  H × H    Gram WᵀW, every entry summed left-to-right over d exactly as
//               the reference's Eigen product (oracle order), so selection
//               scores are reproducible bit for bit
//   B  N × Hp   Y·W (DMMA GEMM)
//   ES N × Hp   posterior means ⟨s_n⟩ (dense: singletons span all H units)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bscgpu {

constexpr int kMaxHprime = 64;  // candidate positions fit a uint64 mask

// lane path (lane_kernels.cuh): record tile fields per point and point modes
__host__ __device__ inline int lane_rec_fields(int hp) { return 4 + 2 * hp + hp * (hp - 1); }
enum : int { kModeDone = 0, kModeShift = 1, kModeMax = 2, kModeFallback = 3 };

// Error flags raised by device code (bit set in *err).
enum : int { kErrNonFiniteScore = 1, kErrNonFiniteLogJoint = 2 };

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Row p of entry e of a strict upper triangle stored row-major (H' columns):
// start(p) = p(2H'−p−1)/2 ≤ e < start(p+1); closed form, corrected by one step.
__device__ __forceinline__ int pair_row(int e, int hp) {
  const float b = 2.0f * hp - 1.0f;
  int p = static_cast<int>((b - sqrtf(fmaxf(b * b - 8.0f * e, 0.0f))) * 0.5f);
  p = max(0, min(p, hp - 2));
  if (p * (2 * hp - p - 1) / 2 > e)
    --p;
  else if ((p + 1) * (2 * hp - p - 2) / 2 <= e)
    ++p;
  return p;
}

// One row of `cnt16` 16-byte chunks global → shared by the warp (cp.async, L2 only).
__device__ __forceinline__ void cp_async_row(double* dst, const double* src, int cnt16, int lane) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  for (int c = lane; c < cnt16; c += 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + c * 16), "l"(src + 2 * c) : "memory");
}

// Σ⟨ssᵀ⟩ candidate pairs in fixed point: each contribution v ∈ [0, 1] is added
// as the integer rint(v·2^k) to the 64-bit image of its (strict upper) entry,
// with 2^k chosen per E-step so that N·2^k < 2⁶³ (BscEngine::fx_scale). Integer
// addition is associative, so the sum, unlike fp64 atomics, is the same bits
// whatever order the points land in; the rounding (≤ 2^-(k+1) per term, 2.8e-14
// at c2) is the order of one fp64 add into a running sum of 100-1000.
// finalize_stats_kernel converts the triangle back to fp64 and mirrors it.
__device__ __forceinline__ void pair_fx_add(double* entry, double v, double fx_scale) {
  atomicAdd(reinterpret_cast<unsigned long long*>(entry), __double2ull_rn(v * fx_scale));
}

// (value desc, index asc): true when (v1,i1) ranks before (v2,i2).
__device__ __forceinline__ bool ranks_before(double v1, int i1, double v2, int i2) {
  return v1 > v2 || (v1 == v2 && i1 < i2);
}

// ---------------------------------------------------------------------------
// K0: the Gram diagonal G_hh = Σ_d W_dh² in the oracle's order (acc = 0;
// acc += w·w over d, separately rounded) — the selection scores use it, so it
// must match bit for bit — plus column norms for the selection error bound.
// The off-diagonal Gram (pairwise log-joint terms, t3) comes from the DMMA GEMM.
static __global__ void gram_diag_exact_kernel(const double* __restrict__ W, int D, int H, int ldw,
                                       double* __restrict__ G, int ldg, double* __restrict__ wnorm,
                                       double* __restrict__ gdiag) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  // loads batched 16 ahead (the adds stay strictly sequential)
  double acc = 0.0;
  int d = 0;
  for (; d + 16 <= D; d += 16) {
    double a[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) a[u] = W[(long long)(d + u) * ldw + h];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, __dmul_rn(a[u], a[u]));
  }
  for (; d < D; ++d) {
    const double a = W[(long long)d * ldw + h];
    acc = __dadd_rn(acc, __dmul_rn(a, a));
  }
  G[(long long)h * ldg + h] = acc;
  wnorm[h] = sqrt(acc);
  gdiag[h] = acc;
}

// e^x for x < −32 (only ever added to sums whose largest term is 1): fp32
// ex2 — its 2⁻²² relative error is < 2⁻⁶⁸ of the sum. Underflow flushes to 0.
__device__ __forceinline__ double small_exp(double x) {
  float r;
  const float t = static_cast<float>(fmax(x, -300.0) * 1.4426950408889634);
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
  return static_cast<double>(r);
}

// e^x for x ≤ 0 (and, exactly as well, for 0 < x ≤ 709) in fp64 (the
// posterior weights exp(lj − max) and the guarded factors e^u, e^P): Cody–Waite
// reduction x = k·ln2 + r, |r| ≤ ln2/2, Taylor polynomial of degree 13
// (truncation < 5e-18 relative), and 2^k applied as two exact power-of-two
// factors so gradual underflow rounds once (x < −745.2 gives 0). About 1 ulp;
// ~20 instructions against ~45 for the general-range exp().
__device__ __forceinline__ double exp_nonpos(double x) {
  x = fmax(x, -746.0);
  const double k = rint(x * 1.4426950408889634);
  double r = fma(k, -6.93147180559945286227e-01, x);
  r = fma(k, -2.319046813846299558e-17, r);
  // Estrin evaluation (dependency depth 6 instead of Horner's 14): the
  // kernel's exp loops are latency-bound.
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double q0 = fma(r, 1.0, 1.0);
  const double q1 = fma(r, 1.66666666666666657e-01, 0.5);                    // 1/2!, 1/3!
  const double q2 = fma(r, 8.33333333333333322e-03, 4.16666666666666644e-02);  // 1/4!, 1/5!
  const double q3 = fma(r, 1.98412698412698413e-04, 1.38888888888888894e-03);  // 1/6!, 1/7!
  const double q4 = fma(r, 2.75573192239858883e-06, 2.48015873015873016e-05);  // 1/8!, 1/9!
  const double q5 = fma(r, 2.50521083854417188e-08, 2.75573192239858907e-07);  // 1/10!, 1/11!
  const double q6 = fma(r, 1.6059043836821613e-10, 2.08767569878680990e-09);   // 1/12!, 1/13!
  const double v0 = fma(r2, q1, q0), v1 = fma(r2, q3, q2), v2 = fma(r2, q5, q4);
  const double w0 = fma(r4, v1, v0), w1 = fma(r4, q6, v2);
  const double p = fma(r8, w1, w0);
  const int ki = static_cast<int>(k);
  const int k1 = ki >> 1, k2 = ki - k1;
  const double s1 = __longlong_as_double(static_cast<long long>(k1 + 1023) << 52);
  const double s2 = __longlong_as_double(static_cast<long long>(k2 + 1023) << 52);
  return (p * s1) * s2;
}

// exp_nonpos for bulk use (the H singleton weights per point): the same
// reduction and Taylor polynomial (evaluated as two Horner chains instead of
// Estrin's scheme), with round(x·log2e) taken from the low word of
// x·log2e + 1.5·2⁵² and the power of two applied by one integer add to the
// exponent field. Results below 2⁻¹⁰²¹ (x < −707) are returned as 0 instead of
// as subnormals: they are weights of at most 1e-307 relative to Z.
// Taylor coefficients 1/k!, k = 0..13, in constant memory: an FMA takes one of them straight from the
// constant bank, where an immediate costs two moves per use (a quarter of the loop's instructions).
static __constant__ double kExpTaylor[14] = {
    1.0, 1.0, 0.5, 1.66666666666666657e-01, 4.16666666666666644e-02, 8.33333333333333322e-03,
    1.38888888888888894e-03, 1.98412698412698413e-04, 2.48015873015873016e-05, 2.75573192239858907e-06,
    2.75573192239858883e-07, 2.50521083854417188e-08, 2.08767569878680990e-09, 1.6059043836821613e-10};
__device__ __forceinline__ double exp_nonpos_ftz(double x) {
  const double kd = fma(x, 1.4426950408889634, 6755399441055744.0);
  const int ki = __double2loint(kd);
  const double k = kd - 6755399441055744.0;
  double r = fma(k, -6.93147180559945286227e-01, x);
  r = fma(k, -2.319046813846299558e-17, r);
  // even and odd parts by Horner in r² (two independent chains, one constant operand per FMA)
  const double r2 = r * r;
  double e = kExpTaylor[12], o = kExpTaylor[13];
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    e = fma(e, r2, kExpTaylor[2 * i]);
    o = fma(o, r2, kExpTaylor[2 * i + 1]);
  }
  const double p = fma(o, r, e);
  const double y = __hiloint2double(__double2hiint(p) + (ki << 20), __double2loint(p));
  return x < -707.0 ? 0.0 : y;
}

// ‖y_n‖² per data point (linear_discrete.cpp:242), once per resident dataset:
// one warp per row.
static __global__ void row_sqnorm_kernel(const double* __restrict__ Y, long long N, int D, int ldy,
                                  double* __restrict__ y2) {
  const long long n = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  double s = 0.0;
  for (int d = lane; d < D; d += 32) s = fma(Y[n * ldy + d], Y[n * ldy + d], s);
  s = warp_sum(s);
  if (lane == 0) y2[n] = s;
}

// ---------------------------------------------------------------------------
// K2+K3: per data point (one warp each, grid-stride): selection scores from
// the DMMA product row B[n,:], deterministic top-H' (value desc, lowest index
// wins ties, bit-exact against the oracle through the exact re-rank of the
// near-tie band), log-joints of all truncated states, warp log-sum-exp,
// posterior q, ⟨s_n⟩ and the candidate-pair block of ⟨s sᵀ⟩.
//
// State table (host-built, shared by all points). Candidate subsets of size
// 1..γ in level-lexicographic order: entries [0, H') are the level-1 nodes
// {p}; the multi-active states (levels 2..γ, truncation.cpp:116-147) follow.
// For S = A ∪ {z} (z = max S, parent A, x = max A, sibling A\{x} ∪ {z}):
//   coup(S) = Σ_{p∈A} P[p][z] = coup(sibling) + P[x][z]
//   rel(S)  = rel(A) + u[z] + coup(S)
// so every log-joint costs O(1) whatever |S|. Posterior moments use subtree
// sums of the prefix tree (children of A are contiguous in the next level):
//   sub(A) = q(A) + Σ_children sub(child)
//   ⟨s_p⟩  = Σ_{A: max A = p} sub(A),  ⟨s_p s_q⟩ = Σ_{A: max A = q, p ∈ A} sub(A).
//
// Sums over node lists (children of a node, nodes feeding an output) run as a
// balanced per-lane schedule: the host concatenates the lists in output order
// and cuts the sequence into 32 equal runs; lane l walks run l, accumulating,
// and at the end of each list segment stores the partial into a slot; a
// second pass adds each output's (1–2) slots and writes the result.
// Entry encoding (int2 {src, dst}): src = byte offset of the value to add;
// dst = −1 continue, ≥ 0 segment complete in this lane: store acc·scale at
// byte offset dst, ≤ −2 segment split across lanes: store acc in slot −dst−2.
// Split outputs (at most one per lane boundary) are finished after a
// __syncwarp from their slot ranges.
struct SchedDesc {
  int iters;      // entries per lane
  int row_base;   // first row (of 32 int2) in sched_ent
  int n_split;    // outputs split across lanes (≤ 31)
  int split_base; // sched_split[split_base + l] = {target byte offset, first slot, end slot}
};

// Packed entry (uint32): low 16 bits = source offset / 8; high 16 bits =
// 0xffff continue, else segment end: bit 15 clear → store acc·scale at
// offset (bits 0-14)·8 (an output), set → store acc unscaled (a split slot).
// ACC: outputs accumulate (the moment gather of a chunked table) instead of
// being overwritten; split slots are always overwritten.
template <bool ACC = false>
__device__ __forceinline__ void seg_flush(uint32_t v, double& acc, uint32_t sbase, double scale) {
  const uint32_t hi = v >> 16;
  double val = (hi & 0x8000u) ? acc : acc * scale;
  const uint32_t addr = sbase + (hi & 0x7fffu) * 8;
  if (ACC && hi < 0x8000u) {
    double old;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(old) : "r"(addr) : "memory");
    val += old;
  }
  // predicated store (no branch): taken only at a segment end
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 65535;\n\t@p st.shared.f64 [%1], %2;\n\t}" ::"r"(hi),
      "r"(addr), "d"(val)
      : "memory");
  acc = hi != 0xffffu ? 0.0 : acc;
}
__device__ __forceinline__ double ent_src(const char* smb, uint32_t v) {
  return *reinterpret_cast<const double*>(smb + (v & 0xffffu) * 8);
}

// 64 runs: lane l walks runs l and l+32 interleaved — two independent
// accumulation chains per lane, ≤ 63 outputs split across runs.
constexpr int kSchedRuns = 64;

// Software-pipelined: the next entry pair and its values are loaded before
// this iteration's stores. Safe because a store only ever targets the node
// (or slot) of a segment that has just ended in this lane, and no later entry
// of the same schedule reads it.
template <bool ACC = false>
__device__ __forceinline__ void run_schedule(const SchedDesc& sd, const uint32_t* ent,
                                             const int4* __restrict__ split, char* smb, double* spart, double scale,
                                             int lane) {
  const int n = sd.iters;
  const uint32_t* e = ent + (long long)sd.row_base * kSchedRuns + lane;
  // split descriptors (≤ 63) fetched up front: they land during the main loop
  const int4 sp0 = lane < sd.n_split ? __ldg(split + sd.split_base + lane) : int4{0, 0, 0, 0};
  const int4 sp1 = lane + 32 < sd.n_split ? __ldg(split + sd.split_base + lane + 32) : int4{0, 0, 0, 0};
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smb));
  if (n > 0) {
    double a0 = 0.0, a1 = 0.0;
    uint32_t v0 = e[0], v1 = e[32];
    double x0 = ent_src(smb, v0), x1 = ent_src(smb, v1);
    for (int it = 0; it < n; ++it) {
      const uint32_t* r = e + (it + 1 < n ? it + 1 : it) * kSchedRuns;
      const uint32_t w0 = r[0], w1 = r[32];
      const double y0 = ent_src(smb, w0), y1 = ent_src(smb, w1);
      a0 += x0;
      a1 += x1;
      seg_flush<ACC>(v0, a0, sbase, scale);
      seg_flush<ACC>(v1, a1, sbase, scale);
      v0 = w0;
      v1 = w1;
      x0 = y0;
      x1 = y1;
    }
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int4 sp = u ? sp1 : sp0;
    if (lane + 32 * u < sd.n_split) {
      double s = 0.0;
      for (int j = sp.y; j < sp.z; ++j) s += spart[j];
      double* t = reinterpret_cast<double*>(smb + sp.x);
      *t = ACC ? *t + s * scale : s * scale;
    }
  }
  __syncwarp();
}

struct EnumArgs {
  int N, D, H, Dp, Hp, hprime, gamma;
  const double* Y;
  const double* W;
  const double* B;
  const double* G;        // H × Hp
  const double* wnorm;
  const double* gdiag;    // diag(G), contiguous
  const double* y2;       // N: ‖y_n‖², computed once per dataset
  double* ES;             // N × Hp
  double* ssT;            // H × H, off-diagonal candidate pairs via RED (upper triangle)
  double* warp_scalars;   // [nctas][2] Σ lse_n, Σ ‖y_n‖²
  uint32_t* cand_out;     // N × hprime or null
  double* map_mass;       // inference outputs or null
  int* map_state;         // N: index of the MAP state in reference order
  int* err;               // [0] error flags, [1] points marked kModeFallback (lane path)
  unsigned long long* prof;  // [8] cycles per phase (profiling mode) or null
  // [n_tab] offsets/8 (u16) {rel(parent), coup(sibling) | P[x][z], u[z]}; < hprime unused
  const uint2* sdesc;
  // shared-memory staging of sdesc / sched_ent per CTA (bytes, 0 = read global)
  int stage_desc_bytes, stage_ent_bytes;
  // The state table is cut into chunks of consecutive roots (the smallest
  // member of a state): parents and siblings never cross a chunk, so a point's
  // chunks run one after the other through the same per-warp table region.
  // chunk[c] = {first row of the chunk in sdesc/dfs, rows, level-1 rows (= its
  // roots), first root}.
  const int4* chunk;
  int n_chunks;
  const int* dfs;         // [rows] index of the state in the reference (DFS) order
  const int* level_off;   // [c][gamma + 1]: level k of chunk c is [level_off[k-1], level_off[k]) (chunk rows)
  int n_multi, n_tab, n_coup;  // n_tab / n_coup: the largest chunk's rows / rows of levels 2..γ-1
  // schedules: sched[c][0 .. γ−2] the subtree levels γ−1 … 1 of chunk c,
  // sched[c][γ−1] its part of the moment gather, accumulated into souts
  // (n_out = hprime + hprime·(hprime−1)/2 outputs)
  const SchedDesc* sched;
  const uint32_t* sched_ent;  // packed entries [rows][kSchedRuns]
  const int4* sched_split;
  int n_slots, n_out;
  int weight_mode;  // 0 auto, 1 multiplicative after the exact maximum, 2 exp per state
  // lane path (lane_kernels.cuh): deferred-point records and per-point modes
  double* rec;
  int* pmode;
  double* pscale;  // optional per-point ⟨s⟩-row scale for the slicer (unused: null)
  double log_pi, dlp, inv2s, base0, inv_T;  // base0 = zero_prior + norm_const
  double eps_dot;                           // 2·(D+2)·2⁻⁵³: |b_fast − b_exact| ≤ eps_dot·‖W_h‖·‖y‖
  double fx_scale;                          // 2^k of the fixed-point Σ⟨ssᵀ⟩ pairs (pair_fx_add)
};

constexpr int kPoolCap = 64;

struct EnumSmem {
  // offsets (in doubles) of the per-warp region. n_tab / n_coup are the
  // largest chunk's (see EnumArgs::chunk); the moment outputs persist across
  // the chunks of a point and get their own region.
  int u, P, tab, coup, part, outs, qs, pool_v, pool_i, cand, total;
  __host__ __device__ static EnumSmem make(int hprime, int n_tab, int n_coup, int n_items, int n_out, int h) {
    EnumSmem s;
    s.u = 0;
    s.P = s.u + hprime;                           // strict upper triangle, row-major
    s.qs = s.P + hprime * (hprime - 1) / 2 + 1;   // level-1 weights of all candidates
    s.cand = s.qs + hprime;                       // uint32 candidates packed 2 per double
    s.tab = s.cand + (hprime + 1) / 2 + 1;
    // the selection pool (values + indices) is dead before the table is filled
    s.pool_v = s.tab;
    s.pool_i = s.pool_v + kPoolCap + 2;          // ints packed 2 per double
    int tab_end = s.tab + n_tab + 1;              // tab[n_tab] = 0: padding slot of the lists
    if (tab_end < s.pool_i + kPoolCap / 2 + 1) tab_end = s.pool_i + kPoolCap / 2 + 1;
    s.coup = tab_end;
    // coup (weight pass), the exp compaction queue (n_tab ints) and the schedule
    // slots (moment pass) are live one after the other within a chunk: they overlay
    s.part = s.coup;
    int region = n_coup;
    if (region < n_tab / 2 + 1) region = n_tab / 2 + 1;
    if (region < n_items) region = n_items;
    s.outs = s.coup + region;
    s.total = s.outs + n_out;
    if (s.total < h + 2) s.total = h + 2;  // end-of-kernel CTA reduction reuses the regions
    s.total = (s.total + 1) & ~1;
    return s;
  }
};

// One round of the warp arg-max over register-resident keys (lane owns units
// lane + 32·j): best by (key desc, index asc) among units not yet removed.
template <int MAXJ>
__device__ __forceinline__ void select_round(const double (&key)[MAXJ], uint32_t rem, int lane, double& wv,
                                             int& wi) {
  double bv = -INFINITY;
  int bi = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < MAXJ; ++j) {
    const int h = lane + 32 * j;
    if (!((rem >> j) & 1u) && ranks_before(key[j], h, bv, bi)) {
      bv = key[j];
      bi = h;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ranks_before(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  wv = bv;
  wi = bi;
}

// Top-k (k = H' picks written to cand[0..k) in rank order) over register keys,
// plus the (k+1)-th key. Pool method: the (k+1)-th best of the 32 lane bests
// bounds the top k+1 from below, the pool of units ranking at or above it is
// ranked exactly. Falls back to k+1 arg-max rounds when k ≥ 31 or the pool
// overflows. `valid` marks lanes' real units (h < H).
template <int MAXJ>
__device__ __forceinline__ void top_k(const double (&f)[MAXJ], uint32_t removed, int k, int H, int lane,
                                      double* pool_v, int* pool_i, uint32_t* cand, double& t_k, double& t_next) {
  bool done = false;
  if (k < 31) {
    double lv = -INFINITY;
    int li = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (!((removed >> j) & 1u) && ranks_before(f[j], h, lv, li)) {
        lv = f[j];
        li = h;
      }
    }
    int rk = 0;
#pragma unroll 8
    for (int s = 0; s < 32; ++s) {
      const double ov = __shfl_sync(0xffffffffu, lv, s);
      const int oi = __shfl_sync(0xffffffffu, li, s);
      rk += ranks_before(ov, oi, lv, li);
    }
    // τ = lane best of rank k (the (k+1)-th of the lane bests)
    const unsigned who = __ballot_sync(0xffffffffu, rk == k);
    const int src = __ffs(who) - 1;
    const double tv = __shfl_sync(0xffffffffu, lv, src);
    const int ti = __shfl_sync(0xffffffffu, li, src);
    int base = 0;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      const bool in = h < H && !ranks_before(tv, ti, f[j], h);  // (f,h) ⪯ τ
      const unsigned b = __ballot_sync(0xffffffffu, in);
      if (in) {
        const int pos = base + __popc(b & ((1u << lane) - 1u));
        if (pos < kPoolCap) {
          pool_v[pos] = f[j];
          pool_i[pos] = h;
        }
      }
      base += __popc(b);
    }
    __syncwarp();
    if (base <= kPoolCap) {
      for (int e = lane; e < base; e += 32) {
        const double v = pool_v[e];
        const int i = pool_i[e];
        int r = 0;
        for (int o = 0; o < base; ++o) r += ranks_before(pool_v[o], pool_i[o], v, i);
        if (r < k) cand[r] = static_cast<uint32_t>(i);
        if (r == k - 1) pool_v[kPoolCap] = v;
        if (r == k) pool_v[kPoolCap + 1] = v;
      }
      __syncwarp();
      t_k = pool_v[kPoolCap];
      t_next = pool_v[kPoolCap + 1];
      done = true;
    }
    __syncwarp();
  }
  if (!done) {
    uint32_t rem = removed;
    for (int r = 0; r <= k; ++r) {
      double wv;
      int wi;
      select_round<MAXJ>(f, rem, lane, wv, wi);
      if ((wi & 31) == lane) rem |= 1u << (wi >> 5);
      if (r < k) {
        if (lane == 0) cand[r] = static_cast<uint32_t>(wi);
        t_k = wv;
      } else {
        t_next = wv;
      }
    }
    __syncwarp();
  }
}

// Launch roles of enumerate_kernel: the whole per-point pass (inference, T ≠ 1, shapes outside the
// lane path), or the same pass over only the points the lane path's selection pass
// (select_kernels.cuh) marked for the fallback: near-ties, terms outside the range guard.
enum : int { kPassFull = 0, kPassFallback = 2 };

// STAGED: the state descriptors and schedule entries are staged in shared
// memory (compile-time, so every table access is an LDS, not a generic load)
template <int MAXJ, bool STAGED, int PASS = kPassFull>
__global__ void __launch_bounds__(256, 2) enumerate_kernel(EnumArgs a) {
  extern __shared__ __align__(16) double esm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + wib;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  if constexpr (PASS == kPassFallback) {
    // the selection pass counts the points it leaves to this launch (err[1], zeroed with the
    // error flag per E-step): none, the common case, and the CTA is gone before it stages a table
    if (a.err[1] == 0) return;
  }
  const EnumSmem L = EnumSmem::make(a.hprime, a.n_tab, a.n_coup, a.n_slots, a.n_out, a.H);
  // The state descriptors and schedule entries are the same for every point:
  // staged once per CTA in shared memory when they fit (else read from L1/L2).
  const uint2* sdesc = a.sdesc;
  const uint32_t* sent = a.sched_ent;
  const int stage_bytes = STAGED ? a.stage_desc_bytes + a.stage_ent_bytes : 0;
  if (STAGED) {
    char* cta = reinterpret_cast<char*>(esm);
    const int4* src0 = reinterpret_cast<const int4*>(a.sdesc);
    const int4* src1 = reinterpret_cast<const int4*>(a.sched_ent);
    int4* dst0 = reinterpret_cast<int4*>(cta);
    int4* dst1 = reinterpret_cast<int4*>(cta + a.stage_desc_bytes);
    for (int i = threadIdx.x; i < a.stage_desc_bytes / 16; i += blockDim.x) dst0[i] = __ldg(src0 + i);
    for (int i = threadIdx.x; i < a.stage_ent_bytes / 16; i += blockDim.x) dst1[i] = __ldg(src1 + i);
    __syncthreads();
    sdesc = reinterpret_cast<const uint2*>(cta);
    sent = reinterpret_cast<const uint32_t*>(cta + a.stage_desc_bytes);
  }
  const double* gdiag = a.gdiag;
  double* sm = reinterpret_cast<double*>(reinterpret_cast<char*>(esm) + stage_bytes) + (long long)wib * L.total;
  double* su = sm + L.u;
  double* sP = sm + L.P;
  double* tab = sm + L.tab;
  double* coup = sm + L.coup;
  double* spart = sm + L.part;
  double* souts = sm + L.outs;
  double* sqs = sm + L.qs;
  double* pool_v = sm + L.pool_v;
  int* pool_i = reinterpret_cast<int*>(sm + L.pool_i);
  uint32_t* scand = reinterpret_cast<uint32_t*>(sm + L.cand);

  const int H = a.H, HP = a.hprime, GM = a.gamma;
  double lse_acc = 0.0, y2_acc = 0.0;
  double bound = 0.0;  // max_h ‖W_h‖ (per iteration)
  for (int h = lane; h < H; h += 32) bound = fmax(bound, a.wnorm[h]);
  bound = warp_max(bound);
  const int row_lines = (a.Hp * 8 + 127) / 128;
  // optional per-phase cycle accounting (engine profiling mode only)
  long long t_last = a.prof ? clock64() : 0;
#define ENUM_PHASE(k)                                                                   \
  if (a.prof) {                                                                         \
    const long long t_ = clock64();                                                     \
    if (lane == 0) atomicAdd(a.prof + (k), static_cast<unsigned long long>(t_ - t_last)); \
    t_last = t_;                                                                        \
  }

  int it = 0;
  for (int n = gwarp; n < a.N; n += nwarps, ++it) {
    if constexpr (PASS == kPassFallback) {
      if (a.pmode[n] != kModeFallback) continue;
    }
    ENUM_PHASE(7);
    const double* y = a.Y + (long long)n * a.Dp;
    const double* brow = a.B + (long long)n * a.Hp;
    {  // pull the B row two points ahead into L2 while this point is processed
      const long long nn = n + 2LL * nwarps;
      if (nn < a.N)
        for (int l = lane; l < row_lines; l += 32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.B + nn * a.Hp + l * 16));
      // and the next point's row into L1
      const long long n1 = n + nwarps;
      if (n1 < a.N)
        for (int l = lane; l < row_lines; l += 32)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.B + n1 * a.Hp + l * 16));
    }
    // ‖y‖² (precomputed once per dataset; any order: only the base term and
    // the error bound use it)
    const double y2 = a.y2[n];

    // ---- selection scores (linear_discrete.cpp:244-252), non-fused as the oracle
    double f[MAXJ];
    uint32_t removed = 0;
    double mag = 0.0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) {
        const double b = brow[h], g = gdiag[h];
        f[j] = __dadd_rn(a.log_pi, __dmul_rn(__dsub_rn(__dmul_rn(2.0, b), g), a.inv2s));
        bad |= !isfinite(f[j]);
        mag = fmax(mag, fabs(f[j]) + a.inv2s * (2.0 * fabs(b) + g));
      } else {
        f[j] = -INFINITY;
        removed |= 1u << j;
      }
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(a.err, kErrNonFiniteScore);
      continue;
    }
    // |f_fast − f_exact| ≤ eps: b error (any summation order, γ_D bound)
    // propagated through ×2, −G, ×inv2s, +log π, plus the rounding of those ops.
    mag = warp_max(mag) + fabs(a.log_pi);
    const double eps = 2.5 * a.inv2s * a.eps_dot * bound * sqrt(y2) * 1.0001 + 0x1.0p-46 * mag;

    ENUM_PHASE(0);
    // ---- top-H' by (score desc, index asc), truncation.cpp:38-57
    if (HP < H) {
      double t, nv;
      top_k<MAXJ>(f, removed, HP, H, lane, pool_v, pool_i, scand, t, nv);
      if (!(t - nv > 2.0 * eps)) {
        // Near-tie band: rank the band by exact scores (the oracle's
        // left-to-right b = Wᵀy), everything above it is in, below it out.
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
            double acc = 0.0;
            for (int d = 0; d < a.D; ++d)
              acc = __dadd_rn(acc, __dmul_rn(a.W[(long long)d * a.Hp + h], y[d]));
            f[j] = __dadd_rn(a.log_pi, __dmul_rn(__dsub_rn(__dmul_rn(2.0, acc), a.gdiag[h]), a.inv2s));
          }
        }
        for (int r = 0; r < HP; ++r) {
          double wv;
          int wi;
          select_round<MAXJ>(f, rem2, lane, wv, wi);
          if ((wi & 31) == lane) rem2 |= 1u << (wi >> 5);
          if (lane == 0) scand[r] = static_cast<uint32_t>(wi);
        }
      }
    } else {
      for (int p = lane; p < HP; p += 32) scand[p] = static_cast<uint32_t>(p);
    }
    __syncwarp();
    // candidates ascending (truncation.cpp:55): rank by count of smaller picks
    {
      uint32_t mine[2] = {0xffffffffu, 0xffffffffu};
      int pos[2] = {-1, -1};
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int p = lane + 32 * s;
        if (p < HP) {
          mine[s] = scand[p];
          int rk = 0;
          for (int q = 0; q < HP; ++q) rk += scand[q] < mine[s];
          pos[s] = rk;
        }
      }
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 2; ++s)
        if (pos[s] >= 0) scand[pos[s]] = mine[s];
      __syncwarp();
    }
    if (a.cand_out)
      for (int p = lane; p < HP; p += 32) a.cand_out[(long long)n * HP + p] = scand[p];

    ENUM_PHASE(1);
    // ---- unary / pairwise log-joint terms relative to the zero state:
    // lj(S) − base = Σ_a [dlp + inv2s(2b_a − G_aa)] + Σ_{a<c} (−2 inv2s G_ac)
    for (int p = lane; p < HP; p += 32) {
      const uint32_t c = scand[p];
      const double v = a.dlp + a.inv2s * (2.0 * brow[c] - gdiag[c]);
      su[p] = v;
    }
    // pairwise terms (strict upper triangle, row-major): the Gram gathers are
    // issued first and land while the singleton terms are computed
    const int npairs = HP * (HP - 1) / 2;
    double gp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = lane + 32 * u;
      gp[u] = 0.0;
      if (e < npairs) {
        const int p = pair_row(e, HP), q = e - p * (2 * HP - p - 1) / 2 + p + 1;
        gp[u] = a.G[(long long)scand[p] * a.Hp + scand[q]];
      }
    }
    for (int e = lane + 128; e < npairs; e += 32) {  // H' > 16
      const int p = pair_row(e, HP), q = e - p * (2 * HP - p - 1) / 2 + p + 1;
      sP[e] = -2.0 * a.inv2s * a.G[(long long)scand[p] * a.Hp + scand[q]];
    }
    // zero slot (the selection pool overlays the table)
    if (lane == 0) tab[a.n_tab] = 0.0;

    ENUM_PHASE(2);
    // singletons over all H units and the zero state (rel = 0)
    double(&rel1)[MAXJ] = f;  // scores are no longer needed: reuse the registers
    double mx = 0.0;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      rel1[j] = h < H ? a.dlp + a.inv2s * (2.0 * brow[h] - gdiag[h]) : -INFINITY;
      mx = fmax(mx, rel1[j]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (lane + 32 * u < npairs) sP[lane + 32 * u] = -2.0 * a.inv2s * gp[u];
    __syncwarp();
    // finiteness of every log-joint term (a non-finite log-joint is an error,
    // core.cpp:36-45) and the range guard of the multiplicative weight pass
    double umax = -INFINITY, uabs = 0.0, pmax = -INFINITY, pabs = 0.0;
    bool fin = true;
    for (int p = lane; p < HP; p += 32) {
      const double v = su[p];
      fin = fin && isfinite(v);
      umax = fmax(umax, v);
      uabs = fmax(uabs, fabs(v));
    }
    for (int e = lane; e < npairs; e += 32) {
      const double v = sP[e];
      fin = fin && isfinite(v);
      pmax = fmax(pmax, v);
      pabs = fmax(pabs, fabs(v));
    }
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) fin = fin && (lane + 32 * j >= H || isfinite(rel1[j]));
    if (!__all_sync(0xffffffffu, fin)) {
      if (lane == 0) atomicOr(a.err, kErrNonFiniteLogJoint);
      continue;
    }
    mx = warp_max(mx);
    umax = warp_max(umax);
    uabs = warp_max(uabs);
    pmax = warp_max(pmax);
    pabs = warp_max(pabs);
    const bool t1 = a.inv_T == 1.0;
    // q(S) = q(A)·e^{u_z}·e^{coup(S)} keeps every factor and partial product in
    // fp64 range when |u| ≤ 300 and (γ−1)|P| ≤ 300 (phase 3)
    const bool mult_ok = t1 && a.weight_mode != 2 && uabs <= 300.0 && (GM - 1) * pabs <= 300.0;
    // the multiplicative pass needs no maximum: any shift ≥ max rel works, and
    // an upper bound within e^300 of the true maximum loses nothing to underflow
    const double ub = GM * fmax(umax, 0.0) + 0.5 * GM * (GM - 1) * fmax(pmax, 0.0);
    const bool skip_rel = mult_ok && a.weight_mode == 0 && ub - mx <= 300.0;
    // singleton weights, summed relative to the singleton maximum; rel1 dies
    // here (the MAP and moment passes recompute single_q from B) so the state
    // passes below run with MAXJ more registers of ILP
    const double mxs = mx;
    double* esrow = a.ES + (long long)n * a.Hp;
    double zs1 = lane == 0 ? exp_nonpos(-mxs) : 0.0;
    double zsT = lane == 0 && !t1 ? exp_nonpos(-mxs * a.inv_T) : 0.0;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const double x = rel1[j] - mxs;  // −inf beyond H: exp_nonpos gives 0
      zs1 += exp_nonpos(x);
      if (!t1) zsT += exp_nonpos(x * a.inv_T);
    }
    if (t1) zsT = zs1;
    char* smb = reinterpret_cast<char*>(sm);
    const uint32_t zero_w = static_cast<uint32_t>(L.tab + a.n_tab);  // the zero slot, / 8

    // log-joints relative to the zero state of chunk c's multi-active states,
    // level by level (table entries hold byte offsets into this warp's region):
    //   coup(S) = coup(sibling) + P[x][z],  rel(S) = rel(parent) + u[z] + coup(S).
    // Four states per lane per iteration, all loads before any store (a level
    // only reads earlier levels): four independent chains.
    auto rel_chunk = [&](int c) -> double {
      const int4 ci = a.chunk[c];
      const uint2* cdesc = sdesc + ci.x;
      const int* lo = a.level_off + c * (GM + 1);
      const int nl1 = ci.z;
      for (int l = lane; l < nl1; l += 32) tab[l] = su[ci.w + l];  // level-1 nodes {r}
      __syncwarp();
      double m = -INFINITY;
      for (int k = 2; k <= GM; ++k) {
        const int e = lo[k];
        const bool keep = k < GM;
        for (int i0 = lo[k - 1] + lane; i0 < e; i0 += 128) {
          uint2 d[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + 32 * u;
            d[u] = i < e ? cdesc[i] : make_uint2(zero_w | (zero_w << 16), zero_w | (zero_w << 16));
          }
          double cc[4], r[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // {parent rel | sibling coup, P[x][z] | u[z]} as offsets / 8
            cc[u] = *reinterpret_cast<const double*>(smb + (d[u].x >> 16) * 8) +
                    *reinterpret_cast<const double*>(smb + (d[u].y & 0xffffu) * 8);
            r[u] = *reinterpret_cast<const double*>(smb + (d[u].x & 0xffffu) * 8) +
                   *reinterpret_cast<const double*>(smb + (d[u].y >> 16) * 8) + cc[u];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + 32 * u;
            if (i < e) {
              tab[i] = r[u];
              if (keep) coup[i - nl1] = cc[u];
              m = fmax(m, r[u]);
            }
          }
        }
        __syncwarp();
      }
      return m;
    };

    if (skip_rel) {
      mx = fmax(mx, ub);
    } else {
      for (int c = 0; c < a.n_chunks; ++c) mx = fmax(mx, rel_chunk(c));
      mx = warp_max(mx);
      if (!isfinite(mx)) {
        if (lane == 0) atomicOr(a.err, kErrNonFiniteLogJoint);
        continue;
      }
    }

    ENUM_PHASE(3);
    // log-sum-exp at T = 1 (core.cpp:36-45) and q at temperature T (:272-286);
    // the moment outputs accumulate over the chunks, unnormalised
    double z1 = zs1 * exp_nonpos(mxs - mx), zt = t1 ? 0.0 : zsT * exp_nonpos((mxs - mx) * a.inv_T);
    for (int o = lane; o < a.n_out; o += 32) souts[o] = 0.0;  // outputs without states stay 0
    if (mult_ok) {
      // Multiplicative posterior weights: with |u| ≤ 300 and (γ−1)·|P| ≤ 300
      // every factor and partial product stays inside fp64 range, and
      //   q(S) = q(A) · e^{u_z} · e^{coup(S)},  e^{coup(S)} = e^{coup(sib)} · e^{P_xz},
      // so a multi-active state costs three multiplications instead of an
      // exp (a state whose parent underflowed is below e^-145 of the sum).
      for (int p = lane; p < HP; p += 32) {
        sqs[p] = exp_nonpos(su[p] - mx);  // level-1 nodes {p}
        su[p] = exp_nonpos(su[p]);        // |u| ≤ 300: the reduction + two scale factors are exact here too
      }
      for (int e = lane; e < npairs; e += 32) sP[e] = exp_nonpos(sP[e]);
      __syncwarp();
    }
    double bv = -1.0;  // running MAP candidate over the chunks (value, reference index)
    int bi = 0x7fffffff;
    for (int c = 0; c < a.n_chunks; ++c) {
      const int4 ci = a.chunk[c];
      const uint2* cdesc = sdesc + ci.x;
      const int* lo = a.level_off + c * (GM + 1);
      const int nl1 = ci.z, ntab = ci.y;
      if (mult_ok) {
        for (int l = lane; l < nl1; l += 32) tab[l] = sqs[ci.w + l];
        __syncwarp();
        for (int k = 2; k <= GM; ++k) {
          const int e = lo[k];
          const bool keep = k < GM, first = k == 2;
          for (int i0 = lo[k - 1] + lane; i0 < e; i0 += 128) {
            uint2 d[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + 32 * u;
              d[u] = i < e ? cdesc[i] : make_uint2(zero_w | (zero_w << 16), zero_w | (zero_w << 16));
            }
            double cc[4], q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double es = first ? 1.0 : *reinterpret_cast<const double*>(smb + (d[u].x >> 16) * 8);
              cc[u] = es * *reinterpret_cast<const double*>(smb + (d[u].y & 0xffffu) * 8);
              q[u] = *reinterpret_cast<const double*>(smb + (d[u].x & 0xffffu) * 8) *
                     *reinterpret_cast<const double*>(smb + (d[u].y >> 16) * 8) * cc[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + 32 * u;
              if (i < e) {
                tab[i] = q[u];
                if (keep) coup[i - nl1] = cc[u];
                z1 += q[u];
              }
            }
          }
          __syncwarp();
        }
      } else {
        if (a.n_chunks > 1) rel_chunk(c);  // one chunk: still in place from the max pass
        if (t1) {
          // q = exp_nonpos(rel − max). Terms below e^-32 of the largest state change no
          // fp64 sum they enter (< 2^-46 relative each) and are evaluated in fp32
          // (MUFU.EX2); the others — typically a few dozen — in fp64, compacted.
          int* queue = reinterpret_cast<int*>(coup);  // coup/part are free here
          int nq = 0;
          for (int b0 = 0; b0 < ntab; b0 += 128) {
            double x[4];
            bool big[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = b0 + 32 * u + lane;
              x[u] = i < ntab ? tab[i] - mx : -INFINITY;
              big[u] = x[u] >= -32.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = b0 + 32 * u + lane;
              if (i < ntab) tab[i] = big[u] ? x[u] : small_exp(x[u]);
              const unsigned bm = __ballot_sync(0xffffffffu, big[u]);
              if (big[u]) queue[nq + __popc(bm & ((1u << lane) - 1u))] = i;
              nq += __popc(bm);
            }
          }
          __syncwarp();
          for (int e0 = lane; e0 < nq; e0 += 128) {  // fp64 for the compacted terms, 4 chains
            int idx[4];
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int e = e0 + 32 * u;
              idx[u] = e < nq ? queue[e] : -1;
              x[u] = idx[u] >= 0 ? tab[idx[u]] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = exp_nonpos(x[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (idx[u] >= 0) tab[idx[u]] = x[u];
          }
          __syncwarp();
          for (int i = nl1 + lane; i < ntab; i += 32) z1 += tab[i];
        } else {
          for (int i = lane; i < ntab; i += 32) {
            const double r = tab[i] - mx;
            const double et = exp_nonpos(r * a.inv_T);
            tab[i] = et;
            if (i >= nl1) {
              z1 += exp_nonpos(r);
              zt += et;
            }
          }
        }
        __syncwarp();
      }
      if (a.map_state)  // MAP candidates among this chunk's multi-active states (DFS order index)
        for (int i = nl1 + lane; i < ntab; i += 32) {
          const int ri = 1 + H + a.dfs[ci.x + i];
          if (ranks_before(tab[i], ri, bv, bi)) {
            bv = tab[i];
            bi = ri;
          }
        }
      // subtree sums, bottom-up (level γ nodes are leaves): sub(A) = q(A) + Σ
      // children, one balanced schedule per level; then this chunk's share of
      // ⟨s_p⟩ and ⟨s_p s_q⟩ as sums of subtree values, accumulated into souts
      const SchedDesc* sc = a.sched + c * GM;
      for (int k = 0; k < GM - 1; ++k) run_schedule(sc[k], sent, a.sched_split, smb, spart, 1.0, lane);
      if (a.n_chunks == 1)  // a single table writes the outputs once
        run_schedule<false>(sc[GM - 1], sent, a.sched_split, smb, spart, 1.0, lane);
      else
        run_schedule<true>(sc[GM - 1], sent, a.sched_split, smb, spart, 1.0, lane);
    }
    z1 = warp_sum(z1);
    zt = t1 ? z1 : warp_sum(zt);
    const double lse_rel = mx + log(z1);
    const double base = a.base0 - y2 * a.inv2s;
    const double inv_z = 1.0 / zt;
    if (lane == 0) {
      lse_acc += base + lse_rel;
      if (PASS == kPassFull) y2_acc += y2;  // the fallback's points: counted by the front pass
    }
    __syncwarp();

    // B row and Gram diagonal for the singleton weights of phases 4/6: held in
    // registers when they are few (MAXJ ≤ 12), else re-read where used
    constexpr bool kHold = MAXJ <= 12;
    constexpr int NB = kHold ? MAXJ : 1;
    double bb[NB], gg[NB];
    if (kHold) {
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int h = lane + 32 * j;
        bb[j] = h < H ? brow[h] : 0.0;
        gg[j] = h < H ? a.gdiag[h] : 0.0;
      }
    }
    auto single_qj = [&](int j) {
      const int h = lane + 32 * j;
      const double b = kHold ? bb[kHold ? j : 0] : (h < H ? brow[h] : 0.0);
      const double g = kHold ? gg[kHold ? j : 0] : (h < H ? a.gdiag[h] : 0.0);
      return exp_nonpos((a.dlp + a.inv2s * (2.0 * b - g) - mx) * a.inv_T);
    };

    ENUM_PHASE(4);
    if (a.map_state) {
      // MAP state (linear_discrete.cpp:314-316: first maximum in reference
      // order: zero, singletons 0..H−1, then multi-active in DFS order)
      if (lane == 0 && ranks_before(exp(-mx * a.inv_T), 0, bv, bi)) {
        bv = exp(-mx * a.inv_T);
        bi = 0;
      }
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) {
        const int h = lane + 32 * j;
        const double q = single_qj(j);
        if (h < H && ranks_before(q, 1 + h, bv, bi)) {
          bv = q;
          bi = 1 + h;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ranks_before(ov, oi, bv, bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        a.map_state[n] = bi;
        a.map_mass[n] = bv * inv_z;
      }
    }

    ENUM_PHASE(6);
    // ---- ⟨s_n⟩ row: singleton mass for every unit; candidates then take their
    // full marginal (linear_discrete.cpp:288-304). Σ_n ⟨s_n⟩ is summed by the
    // Yᵀ⟨S⟩ GEMM from these rows.
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) esrow[h] = single_qj(j) * inv_z;
    }
    __syncwarp();
    for (int p = lane; p < HP; p += 32) esrow[scand[p]] = souts[p] * inv_z;
    // candidate pairs (upper triangle: scand ascending ⇒ c_p < c_q)
    for (int o = HP + lane; o < a.n_out; o += 32) {
      // o − HP enumerates (p, q), p < q, row-major
      int idx = o - HP, p = 0;
      while (idx >= HP - 1 - p) {
        idx -= HP - 1 - p;
        ++p;
      }
      const int q = p + 1 + idx;
      pair_fx_add(a.ssT + (long long)scand[p] * H + scand[q], souts[o] * inv_z, a.fx_scale);
    }
    __syncwarp();
  }

  // per-CTA partial sums of Σ log Z_n and Σ ‖y_n‖² in fixed warp order
  __syncthreads();
  double* red = esm;
  const int nw = blockDim.x >> 5;
  if (lane == 0) {
    red[2 * wib] = lse_acc;
    red[2 * wib + 1] = y2_acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0, q = 0.0;
    for (int w = 0; w < nw; ++w) {
      l += red[2 * w];
      q += red[2 * w + 1];
    }
    a.warp_scalars[2 * blockIdx.x] = l;
    a.warp_scalars[2 * blockIdx.x + 1] = q;
  }
}

// Split-K partial reduction (fixed order ⇒ deterministic) into the packed
// statistics [ysT D·H | s H | ssT H·H | counts | y2 | logZ | points]:
// Σ y⟨s⟩ᵀ from the GEMM partials, Σ⟨s⟩ (= diag Σ⟨ssᵀ⟩, v = 1) from its
// fused column sums.
static __global__ void reduce_ysT_kernel(const double* __restrict__ part, const double* __restrict__ colsum, int splits,
                                  int colsum_rows, long long split_stride, int D, int H, int ldp,
                                  double* __restrict__ stats, long long off_s, long long off_ssT) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long DH = (long long)D * H;
  if (idx < DH) {
    const int d = static_cast<int>(idx / H), h = static_cast<int>(idx % H);
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * split_stride + (long long)d * ldp + h];
    stats[idx] = s;
  } else if (idx < DH + H && colsum_rows > 0) {  // (0: the column sums are reduced elsewhere)
    const int h = static_cast<int>(idx - DH);
    double s = 0.0;
    for (int z = 0; z < colsum_rows; ++z) s += colsum[(long long)z * ldp + h];
    stats[off_s + h] = s;
    if (off_ssT >= 0) stats[off_ssT + (long long)h * H + h] = s;  // BSC: ⟨s_h²⟩ = ⟨s_h⟩
  }
}

// Σ⟨ssᵀ⟩ off-diagonals: the fixed-point upper triangle (pair_fx_add) back to
// fp64 (one rounding), mirrored; and the scalars.
static __global__ void finalize_stats_kernel(int nctas, const double* __restrict__ cta_scalars, int H, long long npoints,
                                      double* __restrict__ stats, long long off_ssT, long long off_tail,
                                      double fx_inv) {
  double* ssT = stats + off_ssT;
  const long long HH = (long long)H * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < HH; e += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(e / H), j = static_cast<int>(e % H);
    if (i < j) {
      const double v =
          __ull2double_rn(static_cast<unsigned long long>(__double_as_longlong(ssT[e]))) * fx_inv;
      ssT[e] = v;
      ssT[(long long)j * H + i] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double l = 0.0, y2 = 0.0;
    for (int w = threadIdx.x; w < nctas; w += 32) {
      l += cta_scalars[2 * w];
      y2 += cta_scalars[2 * w + 1];
    }
    l = warp_sum(l);
    y2 = warp_sum(y2);
    if (threadIdx.x == 0) {
      stats[off_tail + 1] = y2;
      stats[off_tail + 2] = l;
      stats[off_tail + 3] = static_cast<double>(npoints);
    }
  }
}

// Start of an E-step: the accumulators every launch adds into, cleared in one launch
// (Σ⟨ssᵀ⟩ fixed-point triangle, error flags, split-K column sums, per-CTA scalars).
static __global__ void estep_clear_kernel(double* __restrict__ ssT, long long n_ssT, int* __restrict__ err,
                                          double* __restrict__ colsums, long long n_colsums,
                                          double* __restrict__ cta_scalars, long long n_scalars) {
  const long long stride = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long e = t0; e < n_ssT; e += stride) ssT[e] = 0.0;
  for (long long e = t0; e < n_colsums; e += stride) colsums[e] = 0.0;
  for (long long e = t0; e < n_scalars; e += stride) cta_scalars[e] = 0.0;
  if (t0 < 2) err[t0] = 0;
}

// value_counts = Σ_h Σ⟨s⟩_h (every active unit carries value 1)
static __global__ void counts_kernel(double* stats, long long off_s, int H, long long off_tail) {
  double acc = 0.0;
  for (int h = threadIdx.x; h < H; h += 32) acc += stats[off_s + h];
  acc = warp_sum(acc);
  if (threadIdx.x == 0) stats[off_tail] = acc;
}

}  // namespace bscgpu
