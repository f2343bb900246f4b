// Max-causes log-joint on sm_100a.
//
// Reference: MaxCausesModel (max_causes.cpp): binary latents; the data mean
// at dimension d is W(d, winner), the winner being the active unit with the
// largest W (mca) or |W| (mmca), ties to the lowest unit (winner_at, :27-41).
// The log-joint is not Gram-expressible, so every multi-active state costs a
// D-loop: one warp per data point, lanes over the dimensions, the states
// visited depth-first in the reference pattern order (truncation.cpp:116-147)
// with a stack of per-depth running maxima:  M_k = max(M_{k−1}, W_{c_z})
// (value and winner per dimension), so a state costs one pass over D whatever
// its size. Singletons use resid_h = ‖y‖² − 2 b_h + ‖W_h‖² from the DMMA
// product B = Y·W; the zero state resid = ‖y‖².
//
// Pass E (estep_impl, :180-281): log Z, the singleton posteriors as an N×H
// row block (their winner statistics come from one DMMA GEMM Yᵀ·Q_s and its
// column sums), and per point the multi-state winner masses den_pt[d][p]
// (soft winner shares when ρ > 0), flushed with fp64 RED into winner_num /
// winner_den. Pass R (residual_impl, :283-350): the posterior at the incoming
// parameters against the residuals under the updated dictionary.
#pragma once
#include "bsc_kernels.cuh"
#include "warp_select.cuh"

namespace bscgpu {

struct McaArgs {
  int N, D, H, Dp, Hp, hprime, gamma, mode, n_multi, pass;  // pass 0 = E, 1 = R
  const double* Y;
  const double* W;      // Dp × Hp (exact band re-rank of the selection)
  const double* WT;     // H × Dp, incoming dictionary
  const double* WTn;    // H × Dp, updated dictionary (pass R)
  const double* B;      // N × Hp, Y·W
  const double* Bn;     // N × Hp, Y·W' (pass R)
  const double* gdiag;  // ‖W_h‖², oracle order
  const double* gdiagn; // ‖W'_h‖² (pass R)
  const double* wnorm;
  const double* y2;
  const uint32_t* pdesc;  // per pattern (reference DFS order): depth | last position << 8 | first position << 16
  double* Qs;             // N × Hp singleton posteriors (pass E)
  double* num;            // D × H winner_num (RED, pass E)
  double* den;            // D × H winner_den (RED, pass E)
  double* cta_part;       // [nctas][4]: Σ lse, Σ activity, Σ residual, -
  uint32_t* cand_out;
  double* ES;             // inference ⟨s_n⟩ rows (N × Hp) or null
  double* map_mass;
  int* map_state;
  int* err;
  double lp1, lp0, norm_const, inv2s, inv_T, rho, eps_dot;
};

struct McaSmem {
  // offsets (in doubles) of the per-warp region
  int y, M, win, Mn, lj, rn, denpt, espt, path, cand, flags, pool_v, pool_i, total;
  __host__ __device__ static McaSmem make(int Dp, int gamma, int n_multi, int hprime, int h) {
    McaSmem s;
    s.y = 0;
    s.M = s.y + Dp;
    s.win = s.M + gamma * Dp;             // uint8 winners, 8 per double
    s.Mn = s.win + (gamma * Dp + 7) / 8;
    s.lj = s.Mn + gamma * Dp;
    s.rn = s.lj + n_multi + 1;
    s.denpt = s.rn + n_multi + 1;         // Dp × H′ winner masses of this point
    s.espt = s.denpt + Dp * hprime;
    s.path = s.espt + hprime;             // int path of candidate positions (≤ γ)
    s.cand = s.path + (gamma + 1) / 2 + 1;
    s.flags = s.cand + (hprime + 1) / 2 + 1;
    s.pool_v = s.flags + (h + 63) / 64 + 1;
    s.pool_i = s.pool_v + kPoolCap + 2;
    s.total = s.pool_i + kPoolCap / 2 + 1;
    s.total = (s.total + 1) & ~1;
    return s;
  }
};

// W (Dp × Hp) → Wᵀ (H × Dp).
static __global__ void transpose_w_kernel(const double* __restrict__ W, int D, int H, int ldw, double* __restrict__ WT,
                                          int ldt) {
  __shared__ double tile[32][33];
  const int h0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int d = d0 + r, h = h0 + threadIdx.x;
    tile[r][threadIdx.x] = (d < D && h < H) ? W[(long long)d * ldw + h] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int h = h0 + r, d = d0 + threadIdx.x;
    if (h < H && d < ldt) WT[(long long)h * ldt + d] = d < D ? tile[threadIdx.x][r] : 0.0;
  }
}

template <int MAXJ>
__global__ void __launch_bounds__(256) mca_enumerate_kernel(McaArgs a) {
  extern __shared__ __align__(16) double esm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int gwarp = blockIdx.x * nw + wib;
  const int nwarps = gridDim.x * nw;
  const int H = a.H, HP = a.hprime, GM = a.gamma, D = a.D, Dp = a.Dp;
  const McaSmem L = McaSmem::make(Dp, GM, a.n_multi, HP, H);
  double* sm = esm + (long long)wib * L.total;
  double* sy = sm + L.y;
  double* sM = sm + L.M;
  uint8_t* swin = reinterpret_cast<uint8_t*>(sm + L.win);
  double* sMn = sm + L.Mn;
  double* slj = sm + L.lj;
  double* srn = sm + L.rn;
  double* denpt = sm + L.denpt;
  double* espt = sm + L.espt;
  int* path = reinterpret_cast<int*>(sm + L.path);
  uint32_t* scand = reinterpret_cast<uint32_t*>(sm + L.cand);
  uint32_t* cflag = reinterpret_cast<uint32_t*>(sm + L.flags);
  double* pool_v = sm + L.pool_v;
  int* pool_i = reinterpret_cast<int*>(sm + L.pool_i);
  const bool passR = a.pass == 1;
  const bool absmax = a.mode == 1;
  for (int e = lane; e < Dp * HP; e += 32) denpt[e] = 0.0;

  double bound = 0.0;
  for (int h = lane; h < H; h += 32) bound = fmax(bound, a.wnorm[h]);
  bound = warp_max(bound);
  double lse_acc = 0.0, act_acc = 0.0, res_acc = 0.0;
  const double kfull = static_cast<double>(H);

  for (int n = gwarp; n < a.N; n += nwarps) {
    const double* y = a.Y + (long long)n * Dp;
    const double* brow = a.B + (long long)n * a.Hp;
    const double y2 = a.y2[n];
    for (int t = lane; t < Dp; t += 32) sy[t] = y[t];

    // ---- selection scores (max_causes.cpp:174-176), non-fused as the oracle
    double f[MAXJ];
    uint32_t removed = 0;
    double mag = 0.0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) {
        const double b = brow[h], g = a.gdiag[h];
        f[j] = __dmul_rn(__dsub_rn(__dmul_rn(2.0, b), g), a.inv2s);
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
    mag = warp_max(mag);
    const double eps = 2.5 * a.inv2s * a.eps_dot * bound * sqrt(y2) * 1.0001 + 0x1.0p-46 * mag;
    warp_select<MAXJ>(f, removed, eps, H, HP, lane, pool_v, pool_i, scand, [&](int h) {
      double acc = 0.0;
      for (int d = 0; d < D; ++d) acc = __dadd_rn(acc, __dmul_rn(a.W[(long long)d * a.Hp + h], y[d]));
      return __dmul_rn(__dsub_rn(__dmul_rn(2.0, acc), a.gdiag[h]), a.inv2s);
    });
    if (a.cand_out && !passR)
      for (int p = lane; p < HP; p += 32) a.cand_out[(long long)n * HP + p] = scand[p];
    for (int w = lane; w < (H + 31) / 32; w += 32) cflag[w] = 0u;
    __syncwarp();
    for (int p = lane; p < HP; p += 32) atomicOr(cflag + (scand[p] >> 5), 1u << (scand[p] & 31));

    // ---- log-joints: k·log π + (H − k)·log(1−π) + norm − resid·inv2s (:213-216)
    const double lj0 = kfull * a.lp0 + a.norm_const - y2 * a.inv2s;
    const double lj1 = a.lp1 + (kfull - 1.0) * a.lp0 + a.norm_const;  // + (−resid_h·inv2s)
    double mx = lj0;
    bool fin = isfinite(lj0);
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) {
        const double r = lj1 - (y2 - 2.0 * brow[h] + a.gdiag[h]) * a.inv2s;
        fin = fin && isfinite(r);
        mx = fmax(mx, r);
      }
    }
    // multi-active states, depth first (reference pattern order)
    int cur_p1 = -1;
    for (int i = 0; i < a.n_multi; ++i) {
      const uint32_t pd = a.pdesc[i];
      const int k = pd & 0xff, z = (pd >> 8) & 0xff, p1 = pd >> 16;
      if (k == 2 && p1 != cur_p1) {  // depth-1 base: the first unit's column
        const double* w1 = a.WT + (long long)scand[p1] * Dp;
        const double* w1n = passR ? a.WTn + (long long)scand[p1] * Dp : nullptr;
        for (int t = lane; t < D; t += 32) {
          sM[t] = w1[t];
          swin[t] = static_cast<uint8_t>(p1);
          if (passR) sMn[t] = w1n[t];
        }
        cur_p1 = p1;
        if (lane == 0) path[0] = p1;
      }
      if (lane == 0) path[k - 1] = z;
      const double* wz = a.WT + (long long)scand[z] * Dp;
      const double* wzn = passR ? a.WTn + (long long)scand[z] * Dp : nullptr;
      const double* Mp = sM + (k - 2) * Dp;
      double* Mc = sM + (k - 1) * Dp;
      const uint8_t* wp = swin + (k - 2) * Dp;
      uint8_t* wc = swin + (k - 1) * Dp;
      double ro = 0.0, rn = 0.0;
      for (int t = lane; t < D; t += 32) {
        const double mp = Mp[t], wv = wz[t];
        const bool better = absmax ? fabs(wv) > fabs(mp) : wv > mp;
        const double m = better ? wv : mp;
        Mc[t] = m;
        wc[t] = better ? static_cast<uint8_t>(z) : wp[t];
        const double r = sy[t] - m;
        ro = fma(r, r, ro);
        if (passR) {
          const double mpn = sMn[(k - 2) * Dp + t], wvn = wzn[t];
          const double mn = (absmax ? fabs(wvn) > fabs(mpn) : wvn > mpn) ? wvn : mpn;
          sMn[(k - 1) * Dp + t] = mn;
          const double r2 = sy[t] - mn;
          rn = fma(r2, r2, rn);
        }
      }
      ro = warp_sum(ro);
      const double l = static_cast<double>(k) * a.lp1 + (kfull - static_cast<double>(k)) * a.lp0 + a.norm_const -
                       ro * a.inv2s;
      if (passR) rn = warp_sum(rn);
      if (lane == 0) {
        slj[i] = l;
        if (passR) srn[i] = rn;
      }
      fin = fin && isfinite(l);
      mx = fmax(mx, l);
      __syncwarp();
    }
    if (!__all_sync(0xffffffffu, fin)) {
      if (lane == 0) atomicOr(a.err, kErrNonFiniteLogJoint);
      continue;
    }
    mx = warp_max(mx);

    // ---- normalisers: z1 at T = 1 (log Z), zt at T
    double z1 = 0.0, zt = 0.0, rq = 0.0;
    const double* bnrow = passR ? a.Bn + (long long)n * a.Hp : nullptr;
    if (lane == 0) {
      z1 = exp(lj0 - mx);
      zt = exp((lj0 - mx) * a.inv_T);
      if (passR) rq = zt * y2;
    }
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) {
        const double r = lj1 - (y2 - 2.0 * brow[h] + a.gdiag[h]) * a.inv2s - mx;
        z1 += exp(r);
        const double et = exp(r * a.inv_T);
        zt += et;
        if (passR) rq += et * (y2 - 2.0 * bnrow[h] + a.gdiagn[h]);
      }
    }
    for (int i = lane; i < a.n_multi; i += 32) {
      const double r = slj[i] - mx;
      z1 += exp(r);
      const double et = exp(r * a.inv_T);
      zt += et;
      if (passR) rq += et * srn[i];
    }
    z1 = warp_sum(z1);
    zt = warp_sum(zt);
    if (passR) {
      rq = warp_sum(rq);
      if (lane == 0) res_acc += rq / zt;  // residual_impl :341-347
      __syncwarp();
      continue;
    }
    const double inv_z = 1.0 / zt;
    if (lane == 0) lse_acc += mx + log(z1);

    // ---- pass E: singleton posteriors (row for Yᵀ·Q_s), activity, MAP, ⟨s⟩
    double act = 0.0;
    double bv = lane == 0 ? exp((lj0 - mx) * a.inv_T) : -1.0;
    int bi = lane == 0 ? 0 : 0x7fffffff;
    double* qrow = a.Qs + (long long)n * a.Hp;
    for (int h = lane; h < H; h += 32) {
      const double q = exp((lj1 - (y2 - 2.0 * brow[h] + a.gdiag[h]) * a.inv2s - mx) * a.inv_T);
      qrow[h] = q * inv_z;
      act += q * inv_z;
      if (a.map_state && ranks_before(q, 1 + h, bv, bi)) {
        bv = q;
        bi = 1 + h;
      }
      if (a.ES && !((cflag[h >> 5] >> (h & 31)) & 1u)) a.ES[(long long)n * a.Hp + h] = q * inv_z;
    }
    for (int p = lane; p < HP; p += 32) espt[p] = 0.0;
    __syncwarp();
    // multi-active states again: winner masses per (dimension, candidate)
    cur_p1 = -1;
    for (int i = 0; i < a.n_multi; ++i) {
      const uint32_t pd = a.pdesc[i];
      const int k = pd & 0xff, z = (pd >> 8) & 0xff, p1 = pd >> 16;
      if (k == 2 && p1 != cur_p1) {
        const double* w1 = a.WT + (long long)scand[p1] * Dp;
        for (int t = lane; t < D; t += 32) {
          sM[t] = w1[t];
          swin[t] = static_cast<uint8_t>(p1);
        }
        cur_p1 = p1;
        if (lane == 0) path[0] = p1;
      }
      if (lane == 0) path[k - 1] = z;
      __syncwarp();
      const double qt = exp((slj[i] - mx) * a.inv_T);
      const double q = qt * inv_z;
      if (lane == 0) act += q * k;
      if (a.map_state && lane == (i & 31) && ranks_before(qt, 1 + H + i, bv, bi)) {
        bv = qt;
        bi = 1 + H + i;
      }
      if (a.ES && lane < k) espt[path[lane]] += q;
      const double* wz = a.WT + (long long)scand[z] * Dp;
      const double* Mp = sM + (k - 2) * Dp;
      double* Mc = sM + (k - 1) * Dp;
      const uint8_t* wp = swin + (k - 2) * Dp;
      uint8_t* wc = swin + (k - 1) * Dp;
      for (int t = lane; t < D; t += 32) {
        const double mp = Mp[t], wv = wz[t];
        const bool better = absmax ? fabs(wv) > fabs(mp) : wv > mp;
        const double m = better ? wv : mp;
        Mc[t] = m;
        const uint8_t wi = better ? static_cast<uint8_t>(z) : wp[t];
        wc[t] = wi;
        if (a.rho > 0.0) {  // soft credit assignment (:236-251), max mode: m = max_a W_da
          double tot = 0.0;
          for (int u = 0; u < k; ++u) tot += pow(a.WT[(long long)scand[path[u]] * Dp + t] / m, a.rho);
          for (int u = 0; u < k; ++u)
            denpt[t * HP + path[u]] += q * (pow(a.WT[(long long)scand[path[u]] * Dp + t] / m, a.rho) / tot);
        } else {
          denpt[t * HP + wi] += q;
        }
      }
      __syncwarp();
    }
    act = warp_sum(act);
    if (lane == 0) act_acc += act;
    // flush the winner masses: winner_den += m, winner_num += y_d·m (:252-257)
    for (int t = lane; t < D; t += 32)
      for (int p = 0; p < HP; ++p) {
        const double m = denpt[t * HP + p];
        if (m != 0.0) {
          atomicAdd(a.den + (long long)t * H + scand[p], m);
          atomicAdd(a.num + (long long)t * H + scand[p], sy[t] * m);
          denpt[t * HP + p] = 0.0;
        }
      }
    if (a.map_state) {
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
    __syncwarp();
    if (a.ES)
      for (int p = lane; p < HP; p += 32) a.ES[(long long)n * a.Hp + scand[p]] = qrow[scand[p]] + espt[p];
    __syncwarp();
  }

  // ---- per-CTA partials, fixed order
  __shared__ double wsc[32][3];
  if (lane == 0) {
    wsc[wib][0] = lse_acc;
    wsc[wib][1] = act_acc;
    wsc[wib][2] = res_acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double l = 0.0, s = 0.0, r = 0.0;
    for (int w = 0; w < nw; ++w) {
      l += wsc[w][0];
      s += wsc[w][1];
      r += wsc[w][2];
    }
    a.cta_part[4 * blockIdx.x] = l;
    a.cta_part[4 * blockIdx.x + 1] = s;
    a.cta_part[4 * blockIdx.x + 2] = r;
  }
}

// winner_num += Σ split-K partials of Yᵀ·Q_s; winner_den(d,h) += Σ_n Q_s(n,h);
// scalars {sum_act, log_partition, points} from the per-CTA partials.
static __global__ void mca_finalize_kernel(const double* __restrict__ part, long long split_stride, int splits,
                                           const double* __restrict__ colsum, int colsum_rows, int D, int H, int ldp,
                                           const double* __restrict__ cta_part, int nctas, long long npoints,
                                           double* __restrict__ stats) {
  const long long DH = (long long)D * H;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx < DH) {
    const int d = static_cast<int>(idx / H), h = static_cast<int>(idx % H);
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * split_stride + (long long)d * ldp + h];
    stats[idx] += s;
    double c = 0.0;
    for (int z = 0; z < colsum_rows; ++z) c += colsum[(long long)z * ldp + h];
    stats[DH + idx] += c;
  } else if (idx == DH) {
    double l = 0.0, act = 0.0;
    for (int c = 0; c < nctas; ++c) {
      l += cta_part[4 * c];
      act += cta_part[4 * c + 1];
    }
    stats[2 * DH] = act;
    stats[2 * DH + 1] = l;
    stats[2 * DH + 2] = static_cast<double>(npoints);
  }
}

struct McaScalars {
  double pi, sigma2, residual;
};

// mstep_fixedpoint (:393-414): W' = num/den where den ≥ 1e-9 (max(·, 1e-8) in
// mca mode), else the previous entry; π' = clip(sum_act/(N·H), 1e-6, 1−1e-6).
static __global__ void mca_mstep_kernel(const double* __restrict__ stats, const double* __restrict__ W, int D, int H,
                                        int ldw, int mode, double* __restrict__ Wn, McaScalars* sc) {
  const long long DH = (long long)D * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < DH; e += (long long)gridDim.x * blockDim.x) {
    const int d = static_cast<int>(e / H), h = static_cast<int>(e % H);
    const double num = stats[e], den = stats[DH + e];
    double v = W[(long long)d * ldw + h];
    if (den >= 1e-9) {
      v = num / den;
      if (mode == 0) v = v < 1e-8 ? 1e-8 : v;
    }
    Wn[(long long)d * ldw + h] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double nh = stats[2 * DH + 2] * static_cast<double>(H);
    double p = stats[2 * DH] / nh;
    p = p < 1e-6 ? 1e-6 : p;
    p = (1.0 - 1e-6) < p ? (1.0 - 1e-6) : p;
    sc->pi = p;
  }
}

// σ²' = max(Σ_n residual / (N·D), 1e-12) (step, :431-436).
static __global__ void mca_sigma_kernel(const double* __restrict__ cta_part, int nctas, long long npoints, int D,
                                        McaScalars* sc) {
  if (threadIdx.x != 0) return;
  double r = 0.0;
  for (int c = 0; c < nctas; ++c) r += cta_part[4 * c + 2];
  sc->residual = r;
  const double s2 = r / (static_cast<double>(npoints) * static_cast<double>(D));
  sc->sigma2 = s2 < 1e-12 ? 1e-12 : s2;
}

}  // namespace bscgpu
