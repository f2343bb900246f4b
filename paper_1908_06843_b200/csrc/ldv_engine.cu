// BscEngine, multi-valued families (tsc / dsc): state template with the value
// odometer, the enumerator launch and the statistics finalisation.
// Reference: LinearDiscreteModel (linear_discrete.cpp:71-97, :202-408) and
// StateTemplate (truncation.cpp:95-169).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "bsc_engine.hpp"
#include "engine_util.hpp"
#include "ldv_kernels.cuh"
#include "sched_builder.hpp"

namespace bscgpu {

using namespace util;

namespace {

template <bool STAGED>
const void* ldv_fn_t(int maxj) {
  switch (maxj) {
    case 1: return (const void*)ldv_enumerate_kernel<1, STAGED>;
    case 2: return (const void*)ldv_enumerate_kernel<2, STAGED>;
    case 4: return (const void*)ldv_enumerate_kernel<4, STAGED>;
    case 6: return (const void*)ldv_enumerate_kernel<6, STAGED>;
    case 8: return (const void*)ldv_enumerate_kernel<8, STAGED>;
    case 10: return (const void*)ldv_enumerate_kernel<10, STAGED>;
    case 12: return (const void*)ldv_enumerate_kernel<12, STAGED>;
    case 16: return (const void*)ldv_enumerate_kernel<16, STAGED>;
    case 24: return (const void*)ldv_enumerate_kernel<24, STAGED>;
    default: return (const void*)ldv_enumerate_kernel<32, STAGED>;
  }
}

using Node = std::vector<std::pair<int, int>>;  // (candidate position, value index), positions ascending

}  // namespace

const void* ldv_kernel_fn(int maxj, bool staged) { return staged ? ldv_fn_t<true>(maxj) : ldv_fn_t<false>(maxj); }

int BscEngine::ldv_per_warp_bytes() const {
  return 8 * LdvSmem::make(hprime_, static_cast<int>(values_.size()), n_tab_, n_coup_, n_slots_, n_out_,
                           static_cast<int>(H_))
                 .total;
}

// StateTemplate with V values (truncation.cpp:95-151): patterns in reference
// order = supports depth-first (prefixes first), the value odometer (last
// slot fastest) inside each support. The GPU table orders nodes level by level,
// lexicographically in the interleaved tuple (p1,v1,p2,v2,…), so the children
// (A + (z, v_z), z > max A) of a node are contiguous.
void BscEngine::build_template_v() {
  const int V = static_cast<int>(values_.size());
  const int hp = static_cast<int>(hprime_);
  auto sat_add = [](uint64_t a, uint64_t b) { return UINT64_MAX - a < b ? UINT64_MAX : a + b; };
  auto sat_mul = [](uint64_t a, uint64_t b) { return (a != 0 && b > UINT64_MAX / a) ? UINT64_MAX : a * b; };
  auto binom = [&](uint64_t n, uint64_t k) -> uint64_t {
    if (k > n) return 0;
    k = std::min(k, n - k);
    uint64_t r = 1;
    for (uint64_t i = 1; i <= k; ++i) r = sat_mul(r, n - k + i) / i;
    return r;
  };
  // truncated_state_count (truncation.cpp:83-93)
  uint64_t total = sat_add(1, sat_mul(H_, V));
  uint64_t vpow = V;
  for (uint32_t k = 2; k <= gamma_; ++k) {
    vpow = sat_mul(vpow, V);
    total = sat_add(total, sat_mul(binom(hprime_, k), vpow));
  }
  if (total > cap_)
    throw Error(kConfig, "state explosion: " + std::to_string(total) + " states per data point exceeds cap of " +
                             std::to_string(cap_));
  if (total > 2000000) throw Error(kConfig, "gpu: state template too large for the enumerator");

  // reference DFS order of the multi-active patterns
  std::map<Node, int> dfs_of;
  dfs_patterns_.clear();
  {
    std::vector<int> support;
    auto emit = [&]() {
      const size_t k = support.size();
      std::vector<int> vi(k, 0);
      for (;;) {
        Node nd;
        std::vector<std::pair<uint8_t, uint8_t>> pat;
        for (size_t i = 0; i < k; ++i) {
          nd.emplace_back(support[i], vi[i]);
          pat.emplace_back(static_cast<uint8_t>(support[i]), static_cast<uint8_t>(vi[i]));
        }
        dfs_of[nd] = static_cast<int>(dfs_patterns_.size());
        dfs_patterns_.push_back(pat);
        size_t i = k;
        bool done = false;
        for (;;) {
          if (i == 0) {
            done = true;
            break;
          }
          --i;
          if (++vi[i] < V) break;
          vi[i] = 0;
          if (i == 0) {
            done = true;
            break;
          }
        }
        if (done) return;
      }
    };
    auto dfs = [&](auto&& self, int next) -> void {
      if (support.size() >= 2) emit();
      if (support.size() == gamma_) return;
      for (int p = next; p < hp; ++p) {
        support.push_back(p);
        self(self, p + 1);
        support.pop_back();
      }
    };
    if (gamma_ >= 2) dfs(dfs, 0);
  }
  n_multi_ = static_cast<int>(dfs_patterns_.size());

  // level-lexicographic table
  std::vector<Node> nodes;
  std::vector<int> level_off{0};
  for (int p = 0; p < hp; ++p)
    for (int k = 0; k < V; ++k) nodes.push_back(Node{{p, k}});
  level_off.push_back(static_cast<int>(nodes.size()));
  for (uint32_t lvl = 2; lvl <= gamma_; ++lvl) {
    const int b = level_off[lvl - 2], e = level_off[lvl - 1];
    for (int i = b; i < e; ++i) {
      const Node A = nodes[i];
      for (int z = A.back().first + 1; z < hp; ++z)
        for (int k = 0; k < V; ++k) {
          Node S = A;
          S.emplace_back(z, k);
          nodes.push_back(S);
        }
    }
    level_off.push_back(static_cast<int>(nodes.size()));
  }
  const int n_tab = static_cast<int>(nodes.size());
  const int HV = hp * V;
  if (n_tab != HV + n_multi_) throw Error(kInternal, "state template size mismatch");
  std::map<Node, int> index_of;
  for (int i = 0; i < n_tab; ++i) index_of[nodes[i]] = i;
  const int n_coup = gamma_ >= 3 ? level_off[gamma_ - 1] - HV : 0;
  n_out_ = HV + hp * (hp - 1) / 2 * V * V;
  const LdvSmem L0 = LdvSmem::make(hp, V, n_tab, n_coup, kSlots, n_out_, static_cast<int>(H_));
  auto tab_off = [&](int i) { return (L0.tab + i) * 8; };
  auto pair_of = [hp](int p, int q) { return p * (2 * hp - p - 1) / 2 + (q - p - 1); };  // p < q, row-major

  std::vector<uint2> desc(n_tab, uint2{0, 0});
  std::vector<int> dfs_idx(n_tab, -1);
  for (int i = HV; i < n_tab; ++i) {
    const Node& S = nodes[i];
    const auto zk = S.back();
    Node A(S.begin(), S.end() - 1);
    const auto xk = A.back();
    Node sib(A.begin(), A.end() - 1);
    sib.push_back(zk);
    const int si = index_of.at(sib);
    const int par_off = tab_off(index_of.at(A));
    const int sib_off = si < HV ? tab_off(n_tab) : (L0.coup + si - HV) * 8;
    const int p_off = (L0.P + (pair_of(xk.first, zk.first) * V + xk.second) * V + zk.second) * 8;
    const int u_off = (L0.u + zk.first * V + zk.second) * 8;
    desc[i] = uint2{ScheduleBuilder::w16(par_off) | (ScheduleBuilder::w16(sib_off) << 16),
                    ScheduleBuilder::w16(p_off) | (ScheduleBuilder::w16(u_off) << 16)};
    dfs_idx[i] = dfs_of.at(S);
  }
  n_tab_ = n_tab;
  n_coup_ = n_coup;

  ScheduleBuilder sb;
  sb.zero_off = tab_off(n_tab);
  sb.part_base = L0.part;
  // subtree sums, levels γ−1 … 1: sub(A) = q(A) + Σ children (contiguous)
  for (int lvl = static_cast<int>(gamma_) - 1; lvl >= 1; --lvl) {
    std::vector<std::vector<int>> ls;
    std::vector<int> tg;
    for (int i = level_off[lvl - 1]; i < level_off[lvl]; ++i) {
      std::vector<int> l{tab_off(i)};
      const Node& A = nodes[i];
      const int nc = (hp - 1 - A.back().first) * V;
      if (nc > 0) {
        Node c0 = A;
        c0.emplace_back(A.back().first + 1, 0);
        const int fc = index_of.at(c0);
        for (int c = 0; c < nc; ++c) l.push_back(tab_off(fc + c));
      }
      ls.push_back(l);
      tg.push_back(tab_off(i));
    }
    sb.add(ls, tg);
  }
  {  // value-split moments: M1[(p,v)] and M2[(p,vp),(q,vq)]
    std::vector<std::vector<int>> ls(n_out_);
    std::vector<int> tg(n_out_);
    for (int i = 0; i < n_tab; ++i) {
      const Node& S = nodes[i];
      const auto qk = S.back();
      ls[qk.first * V + qk.second].push_back(tab_off(i));
      for (size_t a = 0; a + 1 < S.size(); ++a)
        ls[HV + (pair_of(S[a].first, qk.first) * V + S[a].second) * V + qk.second].push_back(tab_off(i));
    }
    for (int o = 0; o < n_out_; ++o) tg[o] = (L0.outs + o) * 8;
    sb.add(ls, tg);
  }
  n_slots_ = kSlots;

  auto& ent = sb.ent;
  while ((desc.size() * sizeof(uint2)) % 16) desc.push_back(uint2{0, 0});
  while ((ent.size() * sizeof(uint32_t)) % 16) ent.push_back(0);
  desc_bytes_ = static_cast<int>(desc.size() * sizeof(uint2));
  ent_bytes_ = static_cast<int>(ent.size() * sizeof(uint32_t));
  d_desc_ = dalloc<uint2>(desc.size(), "desc");
  d_dfs_ = dalloc<int>(dfs_idx.size(), "dfs");
  d_level_off_ = dalloc<int>(level_off.size(), "level_off");
  d_sched_ = dalloc<SchedDesc>(sb.sched.size(), "schedules");
  d_sched_ent_ = dalloc<uint32_t>(ent.size(), "schedule entries");
  d_sched_split_ = dalloc<int4>(sb.splits.size(), "schedule splits");
  ck(cudaMemcpy(d_desc_, desc.data(), desc_bytes_, cudaMemcpyHostToDevice), "desc");
  ck(cudaMemcpy(d_dfs_, dfs_idx.data(), dfs_idx.size() * 4, cudaMemcpyHostToDevice), "dfs");
  ck(cudaMemcpy(d_level_off_, level_off.data(), level_off.size() * 4, cudaMemcpyHostToDevice), "level_off");
  ck(cudaMemcpy(d_sched_, sb.sched.data(), sb.sched.size() * sizeof(SchedDesc), cudaMemcpyHostToDevice), "sched");
  if (!ent.empty()) ck(cudaMemcpy(d_sched_ent_, ent.data(), ent_bytes_, cudaMemcpyHostToDevice), "ent");
  if (!sb.splits.empty())
    ck(cudaMemcpy(d_sched_split_, sb.splits.data(), sb.splits.size() * sizeof(int4), cudaMemcpyHostToDevice),
       "splits");
}

// value_table (linear_discrete.cpp:71-97): tsc log(π/2) for ±1; dsc log p_v
// over the non-zero alphabet, log p_0 from the zero entry.
void BscEngine::launch_enumerate_v(double temperature, bool cands, bool infer, uint64_t off, uint64_t rows,
                                   int chunk) {
  auto s = static_cast<cudaStream_t>(stream_);
  const int V = static_cast<int>(values_.size());
  LdvArgs la{};
  double log_p0 = 0.0;
  if (family_ == kTsc) {
    log_p0 = std::log(1.0 - pi_);
    for (int k = 0; k < V; ++k) la.logp[k] = std::log(pi_ / 2.0);
  } else {
    int k = 0;
    for (size_t i = 0; i < alphabet_.size(); ++i) {
      if (alphabet_[i] == 0.0)
        log_p0 = std::log(probs_[i]);
      else
        la.logp[k++] = std::log(probs_[i]);
    }
  }
  la.V = V;
  la.vmax = 0.0;
  for (int k = 0; k < V; ++k) {
    la.values[k] = values_[k];
    la.dlpv[k] = la.logp[k] - log_p0;
    la.vmax = std::max(la.vmax, std::abs(values_[k]));
  }
  fill_enum_args(&la.e, temperature, cands, infer, off, rows, chunk, log_p0);
  la.cta_part = d_vpart_ + (size_t)chunk * enum_ctas_ * vpart_stride_;
  la.part_stride = vpart_stride_;
  void* args[] = {&la};
  ck(cudaLaunchKernel(ldv_kernel_fn(maxj_for(H_), stage_tables_), dim3(enum_ctas_), dim3(enum_block_), args,
                      enum_smem_, s),
     "enumerate launch");
  ck(cudaGetLastError(), "enumerate");
  ++launches_;
}

void BscEngine::finalize_v(int nparts, uint64_t n) {
  auto s = static_cast<cudaStream_t>(stream_);
  const int V = static_cast<int>(values_.size());
  const unsigned blocks = std::max<unsigned>((H_ * H_ + 255) / 256, (H_ + V + 2 + 255) / 256);
  finalize_v_kernel<<<std::min(blocks, 1024u), 256, 0, s>>>(nparts, d_vpart_, vpart_stride_, H_, V,
                                                           static_cast<long long>(n), d_stats_, lay_.off_ssT(),
                                                           lay_.off_tail());
  ck(cudaGetLastError(), "finalize");
}

}  // namespace bscgpu
