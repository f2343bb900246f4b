// Multi-valued linear discrete families (TSC: {−1,+1}; DSC: an alphabet with
// 0) through the same truncated E-step as BSC.
//
// Reference: LinearDiscreteModel::value_table (linear_discrete.cpp:71-97),
// estep_impl (:202-325) and the value odometer of the state template
// (truncation.cpp:116-147). Per data point (one warp, grid-stride):
//   scores   s_h = max_v [log p_v + (2 v b_h − v² G_hh)·inv2s]   (non-fused, oracle order)
//   selection top-H′ exactly as the BSC kernel (pool + exact near-tie re-rank)
//   states   zero, (h, v) for all H units and values, and the multi-active
//            patterns: candidate supports of size 2..γ with every value
//            assignment. Table order is level-lexicographic over the
//            interleaved tuple (p₁,v₁,p₂,v₂,…) so the children of a node are
//            contiguous; a state S = A ∪ {(z,v_z)} costs O(1):
//              coup(S) = coup(sibling) + v_x v_z P[x][z],  P = −2·inv2s·G
//              rel(S)  = rel(A) + u[z][v_z] + coup(S),     u = dlp_v + inv2s(2 v b − v² G_zz)
//   moments  subtree sums as in BSC; outputs split by value:
//              M1[p][v]         = Σ_{max A = (p,v)} sub(A)
//              M2[p,v_p,q,v_q]  = Σ_{max A = (q,v_q), (p,v_p) ∈ A} sub(A)
//            then ⟨s_p⟩ = Σ_v v·M1, ⟨s_p²⟩ = Σ_v v²·M1, counts[v] += Σ_p M1[p][v],
//            ⟨s_p s_q⟩ = Σ v_p v_q M2.
// Σ⟨s_h²⟩ (the diagonal of Σ⟨ssᵀ⟩) and the value counts are accumulated per
// warp in shared memory and reduced per CTA in fixed order.
#pragma once
#include "bsc_kernels.cuh"
#include "warp_select.cuh"

namespace bscgpu {

constexpr int kMaxValues = 8;

struct LdvArgs {
  EnumArgs e;  // common fields (e.log_pi / e.dlp / e.weight_mode unused)
  int V;
  double values[kMaxValues];  // non-zero alphabet, ascending
  double logp[kMaxValues];    // log p_v (selection scores)
  double dlpv[kMaxValues];    // log p_v − log p_0 (log-joint terms)
  double vmax;                // max |v|
  double* cta_part;           // [nctas][part_stride]: Σ⟨s_h²⟩ (H), counts (V), Σ lse, Σ ‖y‖²
  int part_stride;
};

struct LdvSmem {
  // offsets (in doubles) of the per-warp region
  int u, P, cand, flags, acc2, cntl, tab, pool_v, pool_i, coup, part, outs, total;
  __host__ __device__ static LdvSmem make(int hprime, int V, int n_tab, int n_coup, int n_items, int n_out,
                                           int h) {
    LdvSmem s;
    const int npairs = hprime * (hprime - 1) / 2;
    s.u = 0;
    s.P = s.u + hprime * V;
    s.cand = s.P + npairs * V * V + 1;
    s.flags = s.cand + (hprime + 1) / 2 + 1;  // candidate bitmask, uint32 words
    s.acc2 = s.flags + (h + 63) / 64 + 1;     // Σ over this warp's points of ⟨s_h²⟩
    s.cntl = s.acc2 + h;                      // per-lane value counts [32][V]
    s.tab = s.cntl + 32 * V;
    s.pool_v = s.tab;
    s.pool_i = s.pool_v + kPoolCap + 2;
    int tab_end = s.tab + n_tab + 1;  // tab[n_tab] = 0: the zero slot
    if (tab_end < s.pool_i + kPoolCap / 2 + 1) tab_end = s.pool_i + kPoolCap / 2 + 1;
    s.coup = tab_end;
    s.part = s.coup;
    s.outs = s.part + n_items;
    s.total = s.outs + n_out;
    if (s.total < s.coup + n_coup) s.total = s.coup + n_coup;
    s.total = (s.total + 1) & ~1;
    return s;
  }
};

template <int MAXJ, bool STAGED>
__global__ void __launch_bounds__(256, 2) ldv_enumerate_kernel(LdvArgs la) {
  const EnumArgs& a = la.e;
  extern __shared__ __align__(16) double esm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int gwarp = blockIdx.x * nw + wib;
  const int nwarps = gridDim.x * nw;
  const int V = la.V;
  const int H = a.H, HP = a.hprime, GM = a.gamma;
  const int HV = HP * V;
  const LdvSmem L = LdvSmem::make(HP, V, a.n_tab, a.n_coup, a.n_slots, a.n_out, H);
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
    sdesc = reinterpret_cast<const uint2*>(cta);
    sent = reinterpret_cast<const uint32_t*>(cta + a.stage_desc_bytes);
  }
  double* sm = reinterpret_cast<double*>(reinterpret_cast<char*>(esm) + stage_bytes) + (long long)wib * L.total;
  double* su = sm + L.u;
  double* sP = sm + L.P;
  double* tab = sm + L.tab;
  double* coup = sm + L.coup;
  double* spart = sm + L.part;
  double* souts = sm + L.outs;
  double* acc2 = sm + L.acc2;
  double* cntl = sm + L.cntl;
  double* pool_v = sm + L.pool_v;
  int* pool_i = reinterpret_cast<int*>(sm + L.pool_i);
  uint32_t* scand = reinterpret_cast<uint32_t*>(sm + L.cand);
  uint32_t* cflag = reinterpret_cast<uint32_t*>(sm + L.flags);
  for (int h = lane; h < H; h += 32) acc2[h] = 0.0;
  for (int k = 0; k < V; ++k) cntl[lane * V + k] = 0.0;
  __syncthreads();

  double lse_acc = 0.0, y2_acc = 0.0;
  double bound = 0.0;
  for (int h = lane; h < H; h += 32) bound = fmax(bound, a.wnorm[h]);
  bound = warp_max(bound);
  double lpmax = 0.0;
  for (int k = 0; k < V; ++k) lpmax = fmax(lpmax, fabs(la.logp[k]));
  const int npairs = HP * (HP - 1) / 2;
  char* smb = reinterpret_cast<char*>(sm);
  const uint32_t zero_w = static_cast<uint32_t>(L.tab + a.n_tab);
  const bool t1 = a.inv_T == 1.0;

  for (int n = gwarp; n < a.N; n += nwarps) {
    const double* y = a.Y + (long long)n * a.Dp;
    const double* brow = a.B + (long long)n * a.Hp;
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
        const double b = brow[h], g = a.gdiag[h];
        double best = -INFINITY;
        for (int k = 0; k < V; ++k) {
          const double v = la.values[k];
          const double sc =
              __dadd_rn(la.logp[k], __dmul_rn(__dsub_rn(__dmul_rn(2.0 * v, b), __dmul_rn(__dmul_rn(v, v), g)), a.inv2s));
          best = best < sc ? sc : best;  // std::max
          mag = fmax(mag, fabs(sc) + a.inv2s * (2.0 * fabs(v * b) + v * v * g));
        }
        f[j] = best;
        bad |= !isfinite(best);
      } else {
        f[j] = -INFINITY;
        removed |= 1u << j;
      }
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(a.err, kErrNonFiniteScore);
      continue;
    }
    mag = warp_max(mag) + lpmax;
    const double eps = 2.5 * a.inv2s * la.vmax * a.eps_dot * bound * sqrt(y2) * 1.0001 + 0x1.0p-46 * mag;

    // ---- top-H' (truncation.cpp:38-57), exact re-rank of the near-tie band
    warp_select<MAXJ>(f, removed, eps, H, HP, lane, pool_v, pool_i, scand, [&](int h) {
      double acc = 0.0;
      for (int d = 0; d < a.D; ++d) acc = __dadd_rn(acc, __dmul_rn(a.W[(long long)d * a.Hp + h], y[d]));
      const double g = a.gdiag[h];
      double best = -INFINITY;
      for (int k = 0; k < V; ++k) {
        const double v = la.values[k];
        const double sc =
            __dadd_rn(la.logp[k], __dmul_rn(__dsub_rn(__dmul_rn(2.0 * v, acc), __dmul_rn(__dmul_rn(v, v), g)), a.inv2s));
        best = best < sc ? sc : best;
      }
      return best;
    });
    if (a.cand_out)
      for (int p = lane; p < HP; p += 32) a.cand_out[(long long)n * HP + p] = scand[p];

    // ---- unary u[p][v] and pairwise v_p v_q P[p][q] log-joint terms
    for (int w = lane; w < (H + 31) / 32; w += 32) cflag[w] = 0u;
    for (int idx = lane; idx < HV; idx += 32) {
      const int p = idx / V, k = idx - p * V;
      const uint32_t c = scand[p];
      const double v = la.values[k];
      const double val = la.dlpv[k] + a.inv2s * (2.0 * v * brow[c] - v * v * a.gdiag[c]);
      su[idx] = val;
      tab[idx] = val;  // level-1 node (p, v)
    }
    for (int e2 = lane; e2 < npairs * V * V; e2 += 32) {
      const int e = e2 / (V * V), r = e2 - e * V * V, kp = r / V, kq = r - kp * V;
      int idx = e, p = 0;
      while (idx >= HP - 1 - p) {
        idx -= HP - 1 - p;
        ++p;
      }
      const int q = p + 1 + idx;
      sP[e2] = -2.0 * a.inv2s * la.values[kp] * la.values[kq] * a.G[(long long)scand[p] * a.Hp + scand[q]];
    }
    if (lane == 0) tab[a.n_tab] = 0.0;
    __syncwarp();
    for (int p = lane; p < HP; p += 32) atomicOr(cflag + (scand[p] >> 5), 1u << (scand[p] & 31));

    // ---- singletons (h, v) over all H (rel = dlp_v + inv2s(2 v b − v² G)), zero state rel 0
    double mx = 0.0;
    bool fin = true;
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) {
        const double b = brow[h], g = a.gdiag[h];
        for (int k = 0; k < V; ++k) {
          const double v = la.values[k];
          const double r = la.dlpv[k] + a.inv2s * (2.0 * v * b - v * v * g);
          fin = fin && isfinite(r);
          mx = fmax(mx, r);
        }
      }
    }
    // multi-active states, level by level (four independent chains per lane)
    for (int k = 2; k <= GM; ++k) {
      const int e = a.level_off[k];
      const bool keep = k < GM;
      for (int i0 = a.level_off[k - 1] + lane; i0 < e; i0 += 128) {
        uint2 d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + 32 * u;
          d[u] = i < e ? sdesc[i] : make_uint2(zero_w | (zero_w << 16), zero_w | (zero_w << 16));
        }
        double c[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          c[u] = *reinterpret_cast<const double*>(smb + (d[u].x >> 16) * 8) +
                 *reinterpret_cast<const double*>(smb + (d[u].y & 0xffffu) * 8);
          r[u] = *reinterpret_cast<const double*>(smb + (d[u].x & 0xffffu) * 8) +
                 *reinterpret_cast<const double*>(smb + (d[u].y >> 16) * 8) + c[u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + 32 * u;
          if (i < e) {
            tab[i] = r[u];
            if (keep) coup[i - HV] = c[u];
            mx = fmax(mx, r[u]);
            fin = fin && isfinite(r[u]);
          }
        }
      }
      __syncwarp();
    }
    for (int i = lane; i < HV; i += 32) fin = fin && isfinite(tab[i]);
    if (!__all_sync(0xffffffffu, fin)) {
      if (lane == 0) atomicOr(a.err, kErrNonFiniteLogJoint);
      continue;
    }
    mx = warp_max(mx);

    // ---- log Z at T = 1 (core.cpp:36-45) and q at temperature T (:272-286)
    double z1 = 0.0, zt = 0.0;
    if (lane == 0) {
      z1 = exp_nonpos(-mx);
      zt = t1 ? z1 : exp_nonpos(-mx * a.inv_T);
    }
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int h = lane + 32 * j;
      if (h < H) {
        const double b = brow[h], g = a.gdiag[h];
        for (int k = 0; k < V; ++k) {
          const double v = la.values[k];
          const double r = la.dlpv[k] + a.inv2s * (2.0 * v * b - v * v * g) - mx;
          const double e1 = exp_nonpos(r);
          z1 += e1;
          zt += t1 ? e1 : exp_nonpos(r * a.inv_T);
        }
      }
    }
    for (int i0 = lane; i0 < a.n_tab; i0 += 128) {
      double r[4], q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u;
        r[u] = i < a.n_tab ? tab[i] - mx : -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = exp_nonpos(r[u] * a.inv_T);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u;
        if (i < a.n_tab) {
          tab[i] = q[u];
          if (i >= HV) {
            z1 += t1 ? q[u] : exp_nonpos(r[u]);
            zt += q[u];
          }
        }
      }
    }
    z1 = warp_sum(z1);
    zt = warp_sum(zt);
    const double inv_z = 1.0 / zt;
    if (lane == 0) {
      lse_acc += a.base0 - y2 * a.inv2s + mx + log(z1);
      y2_acc += y2;
    }
    __syncwarp();

    if (a.map_state) {
      // MAP state (linear_discrete.cpp:314-316): first maximum in reference order
      // (zero, singletons h-major / value-minor, then patterns in DFS order)
      double bv = lane == 0 ? exp(-mx * a.inv_T) : -1.0;
      int bi = lane == 0 ? 0 : 0x7fffffff;
      for (int h = lane; h < H; h += 32) {
        const double b = brow[h], g = a.gdiag[h];
        for (int k = 0; k < V; ++k) {
          const double v = la.values[k];
          const double q = exp_nonpos((la.dlpv[k] + a.inv2s * (2.0 * v * b - v * v * g) - mx) * a.inv_T);
          const int ri = 1 + h * V + k;
          if (ranks_before(q, ri, bv, bi)) {
            bv = q;
            bi = ri;
          }
        }
      }
      for (int i = HV + lane; i < a.n_tab; i += 32) {
        const int ri = 1 + H * V + a.dfs[i];
        if (ranks_before(tab[i], ri, bv, bi)) {
          bv = tab[i];
          bi = ri;
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

    // ---- subtree sums and the value-split moment gather (scaled by 1/Z)
    for (int k = 0; k < GM - 1; ++k) run_schedule(a.sched[k], sent, a.sched_split, smb, spart, 1.0, lane);
    run_schedule(a.sched[GM - 1], sent, a.sched_split, smb, spart, inv_z, lane);

    // ---- ⟨s_n⟩ row, Σ⟨s_h²⟩, value counts, candidate pairs
    double* esrow = a.ES + (long long)n * a.Hp;
    double* cl = cntl + lane * V;
    for (int h = lane; h < H; h += 32) {
      if ((cflag[h >> 5] >> (h & 31)) & 1u) continue;  // candidates take their full marginal below
      const double b = brow[h], g = a.gdiag[h];
      double s1 = 0.0, s2 = 0.0;
      for (int k = 0; k < V; ++k) {
        const double v = la.values[k];
        const double q = exp_nonpos((la.dlpv[k] + a.inv2s * (2.0 * v * b - v * v * g) - mx) * a.inv_T) * inv_z;
        s1 += v * q;
        s2 += v * v * q;
        cl[k] += q;
      }
      esrow[h] = s1;
      acc2[h] += s2;
    }
    for (int p = lane; p < HP; p += 32) {
      const uint32_t c = scand[p];
      double s1 = 0.0, s2 = 0.0;
      for (int k = 0; k < V; ++k) {
        const double v = la.values[k], m = souts[p * V + k];
        s1 += v * m;
        s2 += v * v * m;
        cl[k] += m;
      }
      esrow[c] = s1;
      acc2[c] += s2;
    }
    for (int e = lane; e < npairs; e += 32) {
      int idx = e, p = 0;
      while (idx >= HP - 1 - p) {
        idx -= HP - 1 - p;
        ++p;
      }
      const int q = p + 1 + idx;
      double s = 0.0;
      for (int kp = 0; kp < V; ++kp)
        for (int kq = 0; kq < V; ++kq)
          s += la.values[kp] * la.values[kq] * souts[HV + (e * V + kp) * V + kq];
      atomicAdd(a.ssT + (long long)scand[p] * H + scand[q], s);
    }
    __syncwarp();
  }

  // ---- per-CTA partials in fixed order: Σ⟨s_h²⟩, counts, Σ lse, Σ ‖y‖²
  __shared__ double wsc[32][2];
  if (lane == 0) {
    wsc[wib][0] = lse_acc;
    wsc[wib][1] = y2_acc;
  }
  __syncthreads();
  double* out = la.cta_part + (long long)blockIdx.x * la.part_stride;
  const double* base = reinterpret_cast<double*>(reinterpret_cast<char*>(esm) + stage_bytes);
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += base[(long long)w * L.total + L.acc2 + h];
    out[h] = s;
  }
  for (int k = threadIdx.x; k < V; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w)
      for (int l = 0; l < 32; ++l) s += base[(long long)w * L.total + L.cntl + l * V + k];
    out[H + k] = s;
  }
  if (threadIdx.x == 0) {
    double l = 0.0, s = 0.0;
    for (int w = 0; w < nw; ++w) {
      l += wsc[w][0];
      s += wsc[w][1];
    }
    out[H + V] = l;
    out[H + V + 1] = s;
  }
}

// Mirror of the upper triangle of Σ⟨ssᵀ⟩; its diagonal, the value counts and
// the scalars from the per-CTA partials (fixed order).
__global__ void finalize_v_kernel(int nparts, const double* __restrict__ part, int stride, int H, int V,
                                  long long npoints, double* __restrict__ stats, long long off_ssT,
                                  long long off_tail) {
  double* ssT = stats + off_ssT;
  const long long HH = (long long)H * H;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < HH; e += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(e / H), j = static_cast<int>(e % H);
    if (i > j) ssT[e] = ssT[(long long)j * H + i];
  }
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < H + V + 2) {
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += part[(long long)c * stride + t];
    if (t < H)
      ssT[(long long)t * H + t] = s;
    else if (t < H + V)
      stats[off_tail + (t - H)] = s;
    else if (t == H + V)
      stats[off_tail + V + 1] = s;  // Σ log Z
    else
      stats[off_tail + V] = s;      // Σ ‖y‖²
  }
  if (t == 0) stats[off_tail + V + 2] = static_cast<double>(npoints);
}

}  // namespace bscgpu
