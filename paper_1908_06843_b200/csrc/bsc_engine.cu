// BscEngine implementation: buffers, state template, kernel orchestration.
// See bsc_engine.hpp; the reference path is LinearDiscreteModel::step
// (/root/reference/proj/src/linear_discrete.cpp:410-427).
#include "bsc_engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

#include "bsc_kernels.cuh"
#include "lane_kernels.cuh"
#include "finish_slice_kernels.cuh"
#include "dgemm.cuh"
#include "ozaki_gemm.cuh"
#include "mstep_kernels.cuh"
#include "engine_util.hpp"
#include "sched_builder.hpp"

namespace bscgpu {

namespace {

using namespace util;

template <bool STAGED>
const void* enum_fn_t(int maxj) {
  switch (maxj) {
    case 1: return (const void*)enumerate_kernel<1, STAGED>;
    case 2: return (const void*)enumerate_kernel<2, STAGED>;
    case 4: return (const void*)enumerate_kernel<4, STAGED>;
    case 6: return (const void*)enumerate_kernel<6, STAGED>;
    case 8: return (const void*)enumerate_kernel<8, STAGED>;
    case 10: return (const void*)enumerate_kernel<10, STAGED>;
    case 12: return (const void*)enumerate_kernel<12, STAGED>;
    case 16: return (const void*)enumerate_kernel<16, STAGED>;
    case 24: return (const void*)enumerate_kernel<24, STAGED>;
    default: return (const void*)enumerate_kernel<32, STAGED>;
  }
}
const void* enum_fn(int maxj, bool staged) { return staged ? enum_fn_t<true>(maxj) : enum_fn_t<false>(maxj); }

// the lane path's launches of enumerate_kernel: front half (unstaged, no state
// tables) and the fallback over the points the front half marked
template <int PASS, bool STAGED>
const void* enum_pass_fn_t(int maxj) {
  switch (maxj) {
    case 1: return (const void*)enumerate_kernel<1, STAGED, PASS>;
    case 2: return (const void*)enumerate_kernel<2, STAGED, PASS>;
    case 4: return (const void*)enumerate_kernel<4, STAGED, PASS>;
    case 6: return (const void*)enumerate_kernel<6, STAGED, PASS>;
    case 8: return (const void*)enumerate_kernel<8, STAGED, PASS>;
    case 10: return (const void*)enumerate_kernel<10, STAGED, PASS>;
    case 12: return (const void*)enumerate_kernel<12, STAGED, PASS>;
    case 16: return (const void*)enumerate_kernel<16, STAGED, PASS>;
    case 24: return (const void*)enumerate_kernel<24, STAGED, PASS>;
    default: return (const void*)enumerate_kernel<32, STAGED, PASS>;
  }
}
const void* fallback_fn(int maxj, bool staged) {
  return staged ? enum_pass_fn_t<kPassFallback, true>(maxj) : enum_pass_fn_t<kPassFallback, false>(maxj);
}

using SolveFn = void (*)(const double*, int, int, double*, int, int, int);
template <bool FWD>
SolveFn solve_rows_t(int s) {
  switch (s) {
    case 1: return solve_rows_kernel<1, FWD>;
    case 2: return solve_rows_kernel<2, FWD>;
    case 4: return solve_rows_kernel<4, FWD>;
    case 6: return solve_rows_kernel<6, FWD>;
    case 8: return solve_rows_kernel<8, FWD>;
    case 10: return solve_rows_kernel<10, FWD>;
    case 12: return solve_rows_kernel<12, FWD>;
    case 16: return solve_rows_kernel<16, FWD>;
    case 24: return solve_rows_kernel<24, FWD>;
    default: return solve_rows_kernel<32, FWD>;
  }
}
SolveFn solve_rows_fn(int s, bool fwd) { return fwd ? solve_rows_t<true>(s) : solve_rows_t<false>(s); }

// Tile configurations (see dgemm.cuh).
// GEMM1  B = Y·W:     M = points, N = Hp, K = Dp.
// (tools/gemm_bench.cu sweep at c2 shapes: 64×32 warp tiles, 2 stages, 4 warps is the fastest)
#define GEMM1_CFG 128, 64, 16, 64, 32, true, true, 2
// GEMM2  Yᵀ·⟨S⟩:      M = Dp, N = Hp, K = points (split-K).
// (64×16 warp tiles: 1.09 ms against 1.13 ms for 32×32 in the sweep)
#define GEMM2_CFG 128, 64, 16, 64, 16, false, true, 3
// (64-row tiles when Dp is not a multiple of 128: no half-empty last row tile)
#define GEMM2_CFG64 64, 64, 16, 32, 32, false, true, 4
// M-step products (C −= A·Bᵀ and C −= A·B).
// (32×32 tiles: these products are skinny — N = 64 — so small tiles give the CTAs)
#define SYRK_CFG 32, 32, 16, 16, 16, true, false, 3
#define SOLVE_CFG 32, 32, 16, 16, 16, true, true, 3
// Gram WᵀW: M = N = H, K = Dp.
#define GRAM_CFG 64, 64, 16, 32, 32, false, true, 3

int oz_sms(int device) {
  static int cache[64] = {};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[device] = v;
  }
  return cache[device];
}

}  // namespace

BscEngine::BscEngine(uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma, uint64_t state_cap,
                     int device)
    : alphabet_{0.0, 1.0}, values_{1.0}, D_(dim), H_(latents), hprime_(hprime), gamma_(gamma), cap_(state_cap),
      device_(device) {
  init(device);
}

// LinearDiscreteModel ctor (linear_discrete.cpp:32-61) and value_table
// (:71-97): bsc {1}, tsc {−1, +1}, dsc the sorted alphabet without 0.
BscEngine::BscEngine(int family, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma,
                     uint64_t state_cap, const double* alphabet, uint32_t n_alpha, int device)
    : family_(family), D_(dim), H_(latents), hprime_(hprime), gamma_(gamma), cap_(state_cap), device_(device) {
  switch (family) {
    case kBsc:
      alphabet_ = {0.0, 1.0};
      break;
    case kTsc:
      alphabet_ = {-1.0, 0.0, 1.0};
      break;
    case kDsc: {
      if (!alphabet || n_alpha < 2) throw Error(kConfig, "dsc: alphabet needs at least two values");
      alphabet_.assign(alphabet, alphabet + n_alpha);
      for (double v : alphabet_)
        if (!std::isfinite(v)) throw Error(kConfig, "dsc: alphabet values must be finite");
      std::sort(alphabet_.begin(), alphabet_.end());
      if (std::adjacent_find(alphabet_.begin(), alphabet_.end()) != alphabet_.end())
        throw Error(kConfig, "dsc: alphabet values must be distinct");
      if (std::find(alphabet_.begin(), alphabet_.end(), 0.0) == alphabet_.end())
        throw Error(kConfig, "dsc: alphabet must contain 0");
      break;
    }
    default:
      throw Error(kConfig, "linear model: unknown family");
  }
  for (double v : alphabet_)
    if (v != 0.0) values_.push_back(v);
  if (values_.size() > 8) throw Error(kConfig, "gpu: more than 8 non-zero latent values are not supported");
  if (family_ == kDsc) probs_.assign(alphabet_.size(), 1.0 / alphabet_.size());
  init(device);
}

namespace {
__global__ void guard_probe_kernel(const unsigned char* p, long long i, unsigned char* out) { *out = p[i]; }
}  // namespace

// Test hook of the guarded allocations: one device read at byte `index` of a fresh `bytes`-byte
// buffer (past its end under BSC_GUARD=2 that is a device fault, which leaves the context unusable:
// call it from a process of its own).
void guard_probe(long long bytes, long long index) {
  auto* p = util::dalloc<unsigned char>(static_cast<size_t>(bytes), "guard probe");
  auto* out = util::dalloc<unsigned char>(1, "guard probe out");
  guard_probe_kernel<<<1, 1>>>(p, index, out);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) throw Error(kInternal, std::string("guard probe: ") + cudaGetErrorString(e));
  util::dfree(p);
  util::dfree(out);
}

void check_device_guards() {
  const std::string bad = util::check_guards();
  if (!bad.empty()) throw Error(kInternal, "guard: " + bad);
}

void BscEngine::init(int device) {
  if (D_ == 0 || H_ == 0) throw Error(kConfig, "linear model: dim and latents must be >= 1");
  // TruncationConfig::validate, truncation.cpp:23-30
  if (hprime_ == 0 || hprime_ > H_) throw Error(kConfig, "truncation: hprime must satisfy 1 <= hprime <= latents");
  if (gamma_ == 0 || gamma_ > hprime_) throw Error(kConfig, "truncation: gamma must satisfy 1 <= gamma <= hprime");
  if (cap_ == 0) throw Error(kConfig, "truncation: state cap must be >= 1");
  if (hprime_ > static_cast<uint32_t>(kMaxHprime))
    throw Error(kConfig, "gpu: hprime > 64 is not supported by the sm_100a enumerator");
  if (H_ > 1024) throw Error(kConfig, "gpu: latents > 1024 is not supported by the sm_100a enumerator");
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "device count");
  if (device_ < 0 || device_ >= ndev) throw Error(kConfig, "gpu: device index out of range");
  ck(cudaSetDevice(device_), "set device");
  cudaStream_t s;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  stream_ = s;
  own_stream_ = true;
  Dp_ = round_up(static_cast<int>(D_), 8);
  Hp_ = round_up(static_cast<int>(H_), 8);
  lay_ = StatsLayout{static_cast<long long>(D_), static_cast<long long>(H_), static_cast<long long>(values_.size())};
  if (vpath())
    build_template_v();
  else
    build_template();
  if (const char* e = std::getenv("BSC_ENUM_PROFILE")) prof_on_ = e[0] == '1';
  // posterior-weight path (tests and A/B runs): 0 auto, 1 multiplicative after the
  // exact maximum, 2 exp per state
  if (const char* e = std::getenv("BSC_WEIGHT_MODE")) weight_mode_ = std::atoi(e);
  // lane-per-point state pass (lane_kernels.cuh) for the shapes it is built for
  lane_ok_ = !vpath() && gamma_ >= 2 && gamma_ <= 6 && hprime_ >= 2 && hprime_ <= 16;
  if (const char* e = std::getenv("BSC_LANE")) lane_ok_ = lane_ok_ && e[0] != '0';

  // Y·W and Yᵀ⟨S⟩ on the integer tensor cores (ozaki_gemm.cuh) for the binary
  // family (⟨s⟩ ∈ [0, 1] gives ⟨S⟩ a fixed slice scale); BSC_GEMM=dmma keeps them on DMMA
  Kp_ = round_up(Dp_, 16);
  oz_ = !vpath() && Kp_ <= oz::MAX_KROW;
  if (const char* e = std::getenv("BSC_GEMM")) oz_ = oz_ && std::strcmp(e, "dmma") != 0;
  if (oz_) {
    d_ws_ = dalloc<int8_t>((size_t)oz::S * Hp_ * round_up(Dp_, oz::BK), "W slices");
    d_wsb_ = dalloc<double>(Hp_, "W slice scales");
    d_two_ = dalloc<double>(Hp_, "ES slice scale");
    d_ytsa_ = dalloc<double>((size_t)kMaxChunks * Dp_, "Yt slice scales");
    d_ozmax_ = dalloc<unsigned long long>(Dp_ + Hp_, "column maxima");
    std::vector<double> two(Hp_, 2.0);  // ⟨s⟩ ≤ 1 < 2
    ck(cudaMemcpy(d_two_, two.data(), Hp_ * 8, cudaMemcpyHostToDevice), "ES scale");
  }
  d_w_ = dalloc<double>((size_t)Dp_ * Hp_, "W");
  d_g_ = dalloc<double>((size_t)H_ * Hp_, "G");
  d_trace_part_ = dalloc<double>(2 * kTraceCtas, "trace partials");
  d_wnorm_ = dalloc<double>(H_, "wnorm");
  d_gdiag_ = dalloc<double>(H_, "gdiag");
  d_stats_ = dalloc<double>(lay_.count(), "stats");
  d_smulti_ = dalloc<double>(H_, "s_multi");
  d_err_ = dalloc<int>(2, "err");  // error flags, fallback-point count
  d_bm_ = dalloc<double>((size_t)H_ * Hp_, "Bm");
  d_u_ = dalloc<double>((size_t)H_ * Hp_, "U");
  d_x_ = dalloc<double>((size_t)Dp_ * Hp_, "X");
  d_msc_ = dalloc<MstepScalars>(1, "mstep scalars");
  // one pinned, device-mapped block: the last M-step kernel writes the iteration's result into it
  ck(cudaHostAlloc(&h_result_, kHostResultTail + (values_.size() + 3) * sizeof(double), cudaHostAllocMapped),
     "pinned");
  ck(cudaHostGetDevicePointer(&d_result_, h_result_, 0), "mapped pointer");
  h_msc_ = h_result_;
  h_err_ = static_cast<char*>(h_result_) + kHostResultErr;
  h_tail_ = static_cast<char*>(h_result_) + kHostResultTail;
  cudaStream_t cs;
  ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream");
  copy_stream_ = cs;
  ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "side stream");
  side_stream_ = cs;
  for (void** e : {&ev_fork_, &ev_join_, &ev_branch_[0], &ev_branch_[1]}) {
    cudaEvent_t ev;
    ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    *e = ev;
  }
  if (const char* v = std::getenv("BSC_MSTEP_OVERLAP")) overlap_enabled_ = std::atoi(v) != 0;
  for (auto& e : chunk_ev_) {
    cudaEvent_t ev;
    ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    e = ev;
  }
  for (auto& e : ev_) {
    cudaEvent_t ev;
    ck(cudaEventCreate(&ev), "event");
    e = ev;
  }
}

BscEngine::~BscEngine() {
  cudaSetDevice(device_);
  for (void* p : {(void*)d_desc_, (void*)d_dfs_, (void*)d_level_off_, d_sched_, (void*)d_sched_ent_,
                  d_sched_split_, (void*)d_y_, (void*)d_y2_,
                  (void*)d_w_, (void*)d_g_, (void*)d_wnorm_, (void*)d_gdiag_, (void*)d_b_, (void*)d_es_, (void*)d_stats_,
                  (void*)d_smulti_, (void*)d_warp_es_, (void*)d_warp_sc_, (void*)d_part_, (void*)d_cand_,
                  (void*)d_map_state_, (void*)d_map_mass_, (void*)d_err_, (void*)d_bm_, (void*)d_x_, (void*)d_trace_part_, d_msc_,
                  (void*)d_vpart_, (void*)d_u_, d_chunk_, (void*)d_rec_, (void*)d_lout_, (void*)d_pmode_,
                  (void*)d_ys_, (void*)d_yts_, (void*)d_ws_, (void*)d_ess_, (void*)d_ysa_, (void*)d_ytsa_,
                  (void*)d_wsb_, (void*)d_two_, (void*)d_ozpart_, (void*)d_ozcs_, (void*)d_ozmax_, (void*)d_pscale_})
    dfree(p);
  if (h_result_) cudaFreeHost(h_result_);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (GraphPart* g : {&factor_part_, &update_part_})
    if (g->exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g->exec));
  for (void* e : {ev_fork_, ev_join_, ev_branch_[0], ev_branch_[1]})
    if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  if (side_stream_) cudaStreamDestroy(static_cast<cudaStream_t>(side_stream_));
  for (auto& e : chunk_ev_)
    if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  if (copy_stream_) cudaStreamDestroy(static_cast<cudaStream_t>(copy_stream_));
  if (own_stream_ && stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

void BscEngine::set_stream(void* stream) {
  if (own_stream_ && stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
  stream_ = stream;
  own_stream_ = false;
}

void BscEngine::sync() { ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)), "sync"); }

void BscEngine::enum_phase_cycles(unsigned long long* out8) {
  std::memset(out8, 0, 8 * sizeof(unsigned long long));
  if (!d_prof_) return;
  ck(cudaMemcpyAsync(out8, d_prof_, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     static_cast<cudaStream_t>(stream_)),
     "profile D2H");
  sync();
}

// StateTemplate (truncation.cpp:95-151): multi-active supports of size
// 2..γ over candidate positions, depth-first, prefixes first. The gather
// tables invert it: for every candidate position p and pair (p<q) the list of
// states containing it, cut into work items of similar length.
void BscEngine::build_template() {
  // truncated_state_count (truncation.cpp:83-93), saturating, V = 1
  auto sat_add = [](uint64_t a, uint64_t b) { return UINT64_MAX - a < b ? UINT64_MAX : a + b; };
  auto binom = [](uint64_t n, uint64_t k) -> uint64_t {
    if (k > n) return 0;
    k = std::min(k, n - k);
    unsigned __int128 r = 1;
    for (uint64_t i = 1; i <= k; ++i) {
      r = r * (n - k + i) / i;
      if (r > UINT64_MAX) return UINT64_MAX;
    }
    return static_cast<uint64_t>(r);
  };
  uint64_t total = sat_add(1, H_);
  for (uint32_t k = 2; k <= gamma_; ++k) total = sat_add(total, binom(hprime_, k));
  if (total > cap_)
    throw Error(kConfig, "state explosion: " + std::to_string(total) + " states per data point exceeds cap of " +
                             std::to_string(cap_));

  // reference DFS order (truncation.cpp:116-147) → dfs index of each support
  std::vector<uint64_t> masks;
  masks.reserve(total - 1 - H_);
  std::vector<int> support;
  auto dfs = [&](auto&& self, uint32_t next) -> void {
    if (support.size() >= 2) {
      uint64_t m = 0;
      for (int p : support) m |= 1ull << p;
      masks.push_back(m);
    }
    if (support.size() == gamma_) return;
    for (uint32_t p = next; p < hprime_; ++p) {
      support.push_back(static_cast<int>(p));
      self(self, p + 1);
      support.pop_back();
    }
  };
  if (gamma_ >= 2) dfs(dfs, 0);
  n_multi_ = static_cast<int>(masks.size());
  dfs_masks_ = masks;

  // level-lexicographic table: level 1 = {p}, then combinations of size k
  const int hp = static_cast<int>(hprime_);
  std::vector<std::vector<int>> sets;  // sorted member lists
  for (int p = 0; p < hp; ++p) sets.push_back({p});
  std::vector<int> comb;
  for (uint32_t k = 2; k <= gamma_; ++k) {
    comb.assign(k, 0);
    for (uint32_t i = 0; i < k; ++i) comb[i] = static_cast<int>(i);
    for (;;) {
      sets.push_back(comb);
      int i = static_cast<int>(k) - 1;
      while (i >= 0 && comb[i] == hp - static_cast<int>(k) + i) --i;
      if (i < 0) break;
      ++comb[i];
      for (uint32_t j = i + 1; j < k; ++j) comb[j] = comb[j - 1] + 1;
    }
  }
  if (static_cast<int>(sets.size()) != hp + n_multi_) throw Error(kInternal, "state template size mismatch");
  auto key = [](const std::vector<int>& v) {
    uint64_t m = 0;
    for (int p : v) m |= 1ull << p;
    return m;
  };
  std::unordered_map<uint64_t, int> dfs_of;
  for (int i = 0; i < n_multi_; ++i) dfs_of[masks[i]] = i;

  // Chunks of consecutive roots (root = smallest member): a state's parent and
  // sibling share its root, so chunks are independent tables run one after the
  // other per point through one per-warp region. One chunk when the whole
  // table leaves room for 16 warps per SM, else groups no larger than needed
  // (never below the largest root's subtree).
  std::vector<int> root_size(hp, 0), root_coup(hp, 0);
  for (const auto& S : sets) {
    ++root_size[S[0]];
    if (S.size() >= 2 && S.size() + 1 <= gamma_) ++root_coup[S[0]];  // levels 2..γ−1
  }
  const int total_rows = static_cast<int>(sets.size());
  auto make_groups = [&](int cap) {
    std::vector<std::pair<int, int>> g;  // [first root, end root)
    for (int r = 0; r < hp;) {
      int e = r, rows = 0;
      while (e < hp && (e == r || rows + root_size[e] <= cap)) rows += root_size[e++];
      g.emplace_back(r, e);
      r = e;
    }
    return g;
  };
  auto per_warp_bytes = [&](const std::vector<std::pair<int, int>>& g) {
    int rows = 0, coup = 0;
    for (const auto& [r0, r1] : g) {
      int a = 0, b = 0;
      for (int r = r0; r < r1; ++r) {
        a += root_size[r];
        b += root_coup[r];
      }
      rows = std::max(rows, a);
      coup = std::max(coup, b);
    }
    return 8 * EnumSmem::make(hp, rows, coup, kSlots, hp + hp * (hp - 1) / 2, static_cast<int>(H_)).total;
  };
  const int budget = (228 * 1024 - 2 * 1024) / 16;  // per warp at 16 warps/SM
  int cap_rows = total_rows;
  const int min_cap = *std::max_element(root_size.begin(), root_size.end());
  while (cap_rows > min_cap && per_warp_bytes(make_groups(cap_rows)) > budget)
    cap_rows = std::max(min_cap, cap_rows * 7 / 8);
  const auto groups = make_groups(cap_rows);

  // per-chunk tables: rows in level-lexicographic order restricted to the chunk
  std::vector<uint2> desc;
  std::vector<int> dfs_idx, level_off_all;
  std::vector<int4> chunk_info;
  struct ChunkRows {
    std::vector<int> rows;  // global set indices, chunk order
    std::vector<int> lo;    // level offsets (γ+1)
    int n_coup;
  };
  std::vector<ChunkRows> chunks;
  int max_rows = 0, max_coup = 0;
  for (const auto& [r0, r1] : groups) {
    ChunkRows cr;
    cr.lo.assign(gamma_ + 1, 0);
    for (uint32_t k = 1; k <= gamma_; ++k) {
      for (int i = 0; i < total_rows; ++i)
        if (sets[i].size() == k && sets[i][0] >= r0 && sets[i][0] < r1) cr.rows.push_back(i);
      cr.lo[k] = static_cast<int>(cr.rows.size());
    }
    cr.n_coup = gamma_ >= 3 ? cr.lo[gamma_ - 1] - cr.lo[1] : 0;
    max_rows = std::max(max_rows, static_cast<int>(cr.rows.size()));
    max_coup = std::max(max_coup, cr.n_coup);
    chunks.push_back(std::move(cr));
  }
  n_tab_ = max_rows;
  n_coup_ = max_coup;
  n_chunks_ = static_cast<int>(chunks.size());
  n_out_ = hp + hp * (hp - 1) / 2;
  const EnumSmem L1 = EnumSmem::make(hp, n_tab_, n_coup_, kSlots, n_out_, 0);
  auto tab_off = [&](int i) { return (L1.tab + i) * 8; };
  auto w16 = [](int byte_off) { return ScheduleBuilder::w16(byte_off); };
  auto pair_index = [hp](int p, int q) {  // row-major p < q
    return hp + p * (2 * hp - p - 1) / 2 + (q - p - 1);
  };
  ScheduleBuilder sb;
  sb.zero_off = tab_off(n_tab_);
  sb.part_base = L1.part;
  for (size_t c = 0; c < chunks.size(); ++c) {
    const auto& cr = chunks[c];
    const int base = static_cast<int>(desc.size());
    const int nl1 = cr.lo[1], nrows = static_cast<int>(cr.rows.size());
    chunk_info.push_back(int4{base, nrows, nl1, groups[c].first});
    level_off_all.insert(level_off_all.end(), cr.lo.begin(), cr.lo.end());
    std::unordered_map<uint64_t, int> local;
    for (int i = 0; i < nrows; ++i) local[key(sets[cr.rows[i]])] = i;
    for (int i = 0; i < nrows; ++i) {
      const auto& S = sets[cr.rows[i]];
      if (S.size() == 1) {
        desc.push_back(uint2{0, 0});
        dfs_idx.push_back(-1);
        continue;
      }
      const int z = S.back();
      std::vector<int> A(S.begin(), S.end() - 1);
      const int x = A.back();
      std::vector<int> sib(A.begin(), A.end() - 1);
      sib.push_back(z);
      const int par_off = tab_off(local.at(key(A)));
      const int sib_off = sib.size() == 1 ? tab_off(n_tab_) : (L1.coup + local.at(key(sib)) - nl1) * 8;
      const int p_off = (L1.P + x * (2 * hp - x - 1) / 2 + (z - x - 1)) * 8;  // strict upper triangle
      const int u_off = (L1.u + z) * 8;
      desc.push_back(uint2{w16(par_off) | (w16(sib_off) << 16), w16(p_off) | (w16(u_off) << 16)});
      dfs_idx.push_back(dfs_of.at(key(S)));
    }
    // subtree sums, level γ−1 down to 1: sub(A) = q(A) + Σ_{children} sub(c);
    // children are contiguous in the next level of the chunk
    for (int k = static_cast<int>(gamma_) - 1; k >= 1; --k) {
      std::vector<std::vector<int>> ls;
      std::vector<int> tg;
      for (int i = cr.lo[k - 1]; i < cr.lo[k]; ++i) {
        const auto& A = sets[cr.rows[i]];
        std::vector<int> l{tab_off(i)};
        for (int z = A.back() + 1; z < hp; ++z) {
          std::vector<int> ch = A;
          ch.push_back(z);
          const int li = local.at(key(ch));
          if (l.size() > 1 && li != l.back() / 8 - L1.tab + 1)
            throw Error(kInternal, "state template: children not contiguous");
          l.push_back(tab_off(li));
        }
        ls.push_back(l);
        tg.push_back(tab_off(i));
      }
      sb.add(ls, tg);
    }
    {  // this chunk's share of the moments: ⟨s_p⟩ ← nodes with max p; ⟨s_p s_q⟩ ← max q, p ∈ S
      std::vector<std::vector<int>> ls(n_out_);
      std::vector<int> tg(n_out_);
      for (int i = 0; i < nrows; ++i) {
        const auto& S = sets[cr.rows[i]];
        const int q = S.back();
        ls[q].push_back(tab_off(i));
        for (size_t m = 0; m + 1 < S.size(); ++m) ls[pair_index(S[m], q)].push_back(tab_off(i));
      }
      for (int o = 0; o < n_out_; ++o) tg[o] = (L1.outs + o) * 8;
      // outputs with no state in this chunk stay out of its schedule
      std::vector<std::vector<int>> ls2;
      std::vector<int> tg2;
      for (int o = 0; o < n_out_; ++o)
        if (!ls[o].empty()) {
          ls2.push_back(ls[o]);
          tg2.push_back(tg[o]);
        }
      sb.add(ls2, tg2);
    }
  }
  n_slots_ = kSlots;
  auto& sched = sb.sched;
  auto& ent = sb.ent;
  auto& splits = sb.splits;

  // 16-byte multiples: the kernel stages both tables into shared memory as int4
  while ((desc.size() * sizeof(uint2)) % 16) desc.push_back(uint2{0, 0});
  while ((ent.size() * sizeof(uint32_t)) % 16) ent.push_back(0);
  desc_bytes_ = static_cast<int>(desc.size() * sizeof(uint2));
  ent_bytes_ = static_cast<int>(ent.size() * sizeof(uint32_t));
  d_desc_ = dalloc<uint2>(desc.size(), "desc");
  d_dfs_ = dalloc<int>(dfs_idx.size(), "dfs");
  ck(cudaMemcpy(d_dfs_, dfs_idx.data(), dfs_idx.size() * 4, cudaMemcpyHostToDevice), "dfs");
  d_level_off_ = dalloc<int>(level_off_all.size(), "level_off");
  d_chunk_ = dalloc<int4>(chunk_info.size(), "chunks");
  d_sched_ = dalloc<SchedDesc>(sched.size(), "schedules");
  d_sched_ent_ = dalloc<uint32_t>(ent.size(), "schedule entries");
  d_sched_split_ = dalloc<int4>(splits.size(), "schedule splits");
  ck(cudaMemcpy(d_desc_, desc.data(), desc_bytes_, cudaMemcpyHostToDevice), "desc");
  ck(cudaMemcpy(d_level_off_, level_off_all.data(), level_off_all.size() * 4, cudaMemcpyHostToDevice), "level_off");
  ck(cudaMemcpy(d_chunk_, chunk_info.data(), chunk_info.size() * sizeof(int4), cudaMemcpyHostToDevice), "chunks");
  ck(cudaMemcpy(d_sched_, sched.data(), sched.size() * sizeof(SchedDesc), cudaMemcpyHostToDevice), "sched");
  if (!ent.empty()) ck(cudaMemcpy(d_sched_ent_, ent.data(), ent_bytes_, cudaMemcpyHostToDevice), "ent");
  if (!splits.empty())
    ck(cudaMemcpy(d_sched_split_, splits.data(), splits.size() * sizeof(int4), cudaMemcpyHostToDevice), "splits");
}

void BscEngine::ensure_work(uint64_t n) {
  if (n <= cap_n_ && d_y_) return;
  for (void* p : {(void*)d_y_, (void*)d_y2_, (void*)d_b_, (void*)d_es_, (void*)d_cand_, (void*)d_map_state_,
                  (void*)d_map_mass_, (void*)d_part_, (void*)d_warp_es_, (void*)d_warp_sc_, (void*)d_rec_,
                  (void*)d_lout_, (void*)d_pmode_, (void*)d_ys_, (void*)d_ysa_, (void*)d_yts_, (void*)d_ozcs_, (void*)d_pscale_})
    dfree(p);
  const uint64_t rows = (n + 1) & ~1ull;  // even: GEMM2 reads K in pairs
  if (oz_) {
    oz_np_ = (static_cast<long long>(rows) + 127) / 128 * 128;
    d_ys_ = dalloc<int8_t>((size_t)oz::S * rows * Kp_, "Y slices");
    d_ysa_ = dalloc<double>(rows, "Y slice scales");
    d_yts_ = dalloc<int8_t>((size_t)oz::S * Dp_ * oz_np_, "Yt slices");
    d_ozcs_ = dalloc<double>((size_t)(oz_np_ / 128) * Hp_, "ES column sums");
    d_pscale_ = dalloc<double>(rows, "ES row scales");
  }
  d_y_ = dalloc<double>(rows * Dp_, "Y");
  d_y2_ = dalloc<double>(rows, "y2");
  d_b_ = dalloc<double>(rows * Hp_, "B");
  d_es_ = dalloc<double>(rows * Hp_, "ES");
  d_cand_ = dalloc<uint32_t>(rows * hprime_, "cand");
  d_map_state_ = dalloc<int>(rows, "map_state");
  d_map_mass_ = dalloc<double>(rows, "map_mass");
  cap_n_ = n;

  // split-K for Yᵀ⟨S⟩: ≈4 waves of 148 SMs over the output tiles
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, device_), "props");
  // split-K for Yᵀ⟨S⟩: whole waves (2 resident CTAs per SM), never a ragged tail
  const int bm = Dp_ % 128 == 0 ? 128 : 64;  // GEMM2 row tile (GEMM2_CFG / GEMM2_CFG64)
  const int tiles = ((Dp_ + bm - 1) / bm) * ((Hp_ + 63) / 64);
  const int slots = 2 * prop.multiProcessorCount;
  int waves = 1;
  while (waves < 8 && (waves * slots) / tiles < 8) ++waves;  // ≥ 8 splits when the output is small
  splits_ = std::max(1, std::min<int>((waves * slots) / tiles, static_cast<int>(std::max<uint64_t>(1, rows / 512))));
  part_stride_ = (long long)Dp_ * Hp_;
  d_part_ = dalloc<double>((size_t)splits_ * part_stride_, "splitK partials");

  // enumerator launch shape: per-warp shared region, as many warps as fit
  const int V = static_cast<int>(values_.size());
  const int per_warp =
      vpath() ? ldv_per_warp_bytes()
              : 8 * EnumSmem::make(hprime_, n_tab_, n_coup_, n_slots_, n_out_, static_cast<int>(H_)).total;
  if (per_warp > 200 * 1024)
    throw Error(kConfig, "gpu: state template too large for shared memory (" + std::to_string(n_multi_) + " states)");
  // Pick (warps per CTA, staged tables) maximising resident warps per SM
  // (registers cap it at 16 warps: 128 regs/thread), staged first on ties.
  const int smem_cap = 227 * 1024 - 1024;
  const int table_bytes = desc_bytes_ + ent_bytes_;
  int best_w = 1, best_total = 0;
  bool best_stage = false;
  for (int stage = 1; stage >= 0; --stage)
    for (int w : {8, 4, 2, 1}) {
      const int cta_bytes = w * per_warp + (stage ? table_bytes : 0);
      if (cta_bytes > smem_cap) continue;
      const int ctas = std::min(smem_cap / cta_bytes, 16 / w);
      if (ctas * w > best_total) {
        best_total = ctas * w;
        best_w = w;
        best_stage = stage != 0;
      }
    }
  const int warps = best_w;
  stage_tables_ = best_stage;
  enum_block_ = warps * 32;
  enum_smem_ = warps * per_warp + (stage_tables_ ? table_bytes : 0);
  const int maxj = maxj_for(H_);
  const void* fn = vpath() ? ldv_kernel_fn(maxj, stage_tables_) : enum_fn(maxj, stage_tables_);
  ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, enum_smem_), "enum smem attr");
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, enum_block_, enum_smem_), "occupancy");
  per_sm = std::max(per_sm, 1);
  enum_ctas_ = per_sm * prop.multiProcessorCount;
  const uint64_t need = (n + warps - 1) / warps;
  enum_ctas_ = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(enum_ctas_, need)));
  enum_warps_total_ = enum_ctas_ * warps;
  sc_ctas_ = enum_ctas_;
  if (lane_ok_) {
    // selection pass: thread per point, persistent over CTA tiles of 128 points
    front_smem_ = select_smem(static_cast<int>(H_));
    const void* sf = select_fn(static_cast<int>(hprime_));
    ck(cudaFuncSetAttribute(sf, cudaFuncAttributeMaxDynamicSharedMemorySize, front_smem_), "select smem attr");
    int fs = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fs, sf, 128, front_smem_), "occupancy");
    front_ctas_ = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)std::max(fs, 1) * prop.multiProcessorCount, (n + 127) / 128)));
    const void* fb = fallback_fn(maxj, stage_tables_);
    ck(cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, enum_smem_), "fallback smem attr");
    lane_smem_ = lane_smem(static_cast<int>(gamma_), static_cast<int>(hprime_));
    ck(cudaFuncSetAttribute(lane_fn(gamma_, hprime_), cudaFuncAttributeMaxDynamicSharedMemorySize, lane_smem_),
       "lane smem attr");
    // shared-memory carveout of the lane state pass (percent of the SM's maximum; A/B runs:
    // with e^P read through L1 the carveout trades resident warps against L1 hits)
    if (const char* e = std::getenv("BSC_LANE_CARVEOUT"))
      ck(cudaFuncSetAttribute(lane_fn(gamma_, hprime_), cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e)),
         "lane carveout");
    int fz = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fz, finish_fn(maxj), 256, 0), "occupancy");
    fin_ctas_ = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)std::max(fz, 1) * prop.multiProcessorCount, (n + 7) / 8)));
    // finish fused with the ⟨S⟩ᵀ slicer (sliced path): 32-point sub-tiles while two CTAs fit an
    // SM's shared memory beside each other or one does, else 16-point sub-tiles
    fs_ctas_ = 0;
    const char* fse = std::getenv("BSC_FUSED_FINISH");
    if (oz_ && !(fse && fse[0] == '0')) {
      fs_pt_ = finish_slice_smem(32, static_cast<int>(H_), Hp_, static_cast<int>(hprime_)) <= 200 * 1024 ? 32 : 16;
      fs_smem_ = finish_slice_smem(fs_pt_, static_cast<int>(H_), Hp_, static_cast<int>(hprime_));
      ck(cudaFuncSetAttribute(finish_slice_fn(fs_pt_), cudaFuncAttributeMaxDynamicSharedMemorySize, fs_smem_),
         "finish+slice smem attr");
      int fo = 0;
      ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fo, finish_slice_fn(fs_pt_), fs_threads(fs_pt_), fs_smem_),
         "occupancy");
      fs_ctas_ = std::max(fo, 1) * prop.multiProcessorCount;
    }
    sc_ctas_ = std::max({enum_ctas_, front_ctas_, fin_ctas_, fs_ctas_});
    const uint64_t tiles = (n + 31) / 32;
    d_rec_ = dalloc<double>(tiles * 32 * lane_rec_fields(static_cast<int>(hprime_)), "lane records");
    d_lout_ = dalloc<double>(tiles * 32 * lane_out_fields(static_cast<int>(hprime_)), "lane moments");
    d_pmode_ = dalloc<int>(tiles * 32, "point modes");
  }
  d_warp_es_ = dalloc<double>((size_t)splits_ * Hp_, "split-K column sums");
  d_warp_sc_ = dalloc<double>((size_t)3 * sc_ctas_ * 2, "cta_scalars");
  colsum_chunks_ = 1;
  if (vpath()) {
    dfree(d_vpart_);
    vpart_stride_ = (static_cast<int>(H_) + V + 2 + 1) & ~1;
    d_vpart_ = dalloc<double>((size_t)enum_ctas_ * vpart_stride_, "cta partials");
    vpart_chunks_ = 1;
  }
}

void BscEngine::load_data(const double* y, uint64_t n, bool device_ptr) {
  if (n == 0) throw Error(kData, "run: empty dataset");
  ck(cudaSetDevice(device_), "set device");
  const uint64_t prev_cap = cap_n_;
  ensure_work(n);
  auto s = static_cast<cudaStream_t>(stream_);
  if (n < prev_cap && n_ > n) {
    // shrinking inside an existing allocation: clear stale rows past n
    ck(cudaMemsetAsync(d_y_ + n * Dp_, 0, (cap_n_ - n) * Dp_ * sizeof(double), s), "clear Y");
  }
  ck(cudaMemcpy2DAsync(d_y_, (size_t)Dp_ * 8, y, (size_t)D_ * 8, (size_t)D_ * 8, n,
                       device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s),
     "upload Y");
  row_sqnorm_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(d_y_, static_cast<long long>(n), D_, Dp_,
                                                                       d_y2_);
  ck(cudaGetLastError(), "y2");
  n_ = n;
  if (oz_) slice_y(0, n, 0, s);
  yts_whole_ = true;
}

// int8 slices of the resident Y for the two tensor-core products: rows with
// per-point scales (A of Y·W) and columns with per-dimension scales over the
// chunk (A of Yᵀ⟨S⟩, k = point index contiguous; scale vector `chunk`).
void BscEngine::slice_y(uint64_t off, uint64_t rows, int chunk, void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  const long long cap_rows = static_cast<long long>((cap_n_ + 1) & ~1ull);
  const double* y = d_y_ + off * Dp_;
  ck(oz::slice_rows(y, Dp_, static_cast<int>(rows), Dp_, Kp_, d_ys_ + off * Kp_, cap_rows * Kp_, d_ysa_ + off, s),
     "slice Y rows");
  ck(cudaMemsetAsync(d_ozmax_ + Hp_, 0, (size_t)Dp_ * 8, s), "zero maxima");
  const unsigned gy = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(256, rows / 512)));
  oz::oz_colmax_kernel<<<dim3((Dp_ + 31) / 32, gy), 256, 0, s>>>(y, Dp_, static_cast<long long>(rows),
                                                                 static_cast<int>(D_), d_ozmax_ + Hp_);
  double* sc = d_ytsa_ + (size_t)chunk * Dp_;
  oz::oz_scale_from_max_kernel<<<(Dp_ + 255) / 256, 256, 0, s>>>(d_ozmax_ + Hp_, static_cast<int>(D_), Dp_, 0.0, sc);
  oz::oz_slice_cols_kernel<<<dim3((Dp_ + 31) / 32, static_cast<unsigned>((rows + 127) / 128)), 256, 0, s>>>(
      y, Dp_, static_cast<long long>(rows), static_cast<int>(D_), Dp_, (static_cast<long long>(rows) + 127) / 128 * 128,
      sc, d_yts_ + (off / oz::BK) * Dp_ * oz::BK, static_cast<long long>(Dp_) * oz_np_, nullptr);
  ck(cudaGetLastError(), "slice Y");
  launches_ += 4;
}

// int8 slices of Wᵀ (rows h, k = d contiguous) with per-column scales.
void BscEngine::slice_w(void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  ck(cudaMemsetAsync(d_ozmax_, 0, (size_t)Hp_ * 8, s), "zero maxima");
  oz::oz_colmax_kernel<<<dim3((Hp_ + 31) / 32, 4), 256, 0, s>>>(d_w_, Hp_, static_cast<long long>(D_),
                                                                static_cast<int>(H_), d_ozmax_);
  oz::oz_scale_from_max_kernel<<<(Hp_ + 255) / 256, 256, 0, s>>>(d_ozmax_, static_cast<int>(H_), Hp_, 0.0, d_wsb_);
  const int kpw = round_up(Dp_, oz::BK);
  oz::oz_slice_cols_kernel<<<dim3((Hp_ + 31) / 32, (kpw + 127) / 128), 256, 0, s>>>(
      d_w_, Hp_, static_cast<long long>(D_), static_cast<int>(H_), Hp_, kpw, d_wsb_, d_ws_,
      static_cast<long long>(Hp_) * kpw, nullptr);
  ck(cudaGetLastError(), "slice W");
  launches_ += 3;
}

// Model::step with a host DataSet (the call em.cpp:39 makes): the data are
// copied in chunks on the copy stream, each chunk's E-step starting as soon
// as it lands, then the M-step. Returns F.
double BscEngine::step_streamed(const double* y_host, uint64_t n, double temperature, uint64_t chunk) {
  if (n == 0) throw Error(kData, "run: empty dataset");
  if (!have_params_) throw Error(kConfig, "bsc: parameters not set");
  if (!(temperature >= 1.0) || !std::isfinite(temperature))
    throw Error(kConfig, "temperature must be finite and >= 1");
  ck(cudaSetDevice(device_), "set device");
  const uint64_t prev_cap = cap_n_;
  ensure_work(n);
  if (n < prev_cap && n_ > n)
    ck(cudaMemsetAsync(d_y_ + n * Dp_, 0, (cap_n_ - n) * Dp_ * sizeof(double), static_cast<cudaStream_t>(stream_)),
       "clear Y");
  n_ = n;
  overlap_factor_ = overlap_enabled_;
  try {
    estep_chunked(temperature, false, y_host, chunk);
  } catch (...) {
    overlap_factor_ = factored_ = false;
    throw;
  }
  overlap_factor_ = false;
  mstep();
  return last_F_;
}

void BscEngine::set_params(const double* w, double pi, double sigma2) {
  if (family_ == kDsc) throw Error(kConfig, "dsc: parameters need the value probabilities (set_params_ex)");
  set_params_ex(w, pi, sigma2, nullptr, 0);
}

// LinearDiscreteModel::validate, linear_discrete.cpp:99-127.
void BscEngine::set_params_ex(const double* w, double pi, double sigma2, const double* probs, uint32_t n_probs) {
  const char* nm = family_ == kBsc ? "bsc" : family_ == kTsc ? "tsc" : "dsc";
  for (size_t i = 0; i < (size_t)D_ * H_; ++i)
    if (!std::isfinite(w[i])) throw Error(kNumeric, std::string(nm) + ": non-finite dictionary");
  if (!(sigma2 > 0.0) || !std::isfinite(sigma2)) throw Error(kConfig, std::string(nm) + ": sigma2 must be positive");
  if (family_ == kDsc) {
    if (!probs || n_probs != alphabet_.size()) throw Error(kConfig, "dsc: values/probs size mismatch");
    double total = 0.0;
    for (uint32_t i = 0; i < n_probs; ++i) {
      if (!(probs[i] > 0.0)) throw Error(kConfig, "dsc: probabilities must be positive");
      total += probs[i];
    }
    if (std::abs(total - 1.0) > 1e-6) throw Error(kConfig, "dsc: probabilities must sum to 1");
    probs_.assign(probs, probs + n_probs);
  } else if (!(pi > 0.0 && pi < 1.0)) {
    throw Error(kConfig, std::string(nm) + ": pi must lie in (0,1)");
  }
  ck(cudaSetDevice(device_), "set device");
  ck(cudaMemcpy2DAsync(d_w_, (size_t)Hp_ * 8, w, (size_t)H_ * 8, (size_t)H_ * 8, D_, cudaMemcpyHostToDevice,
                       static_cast<cudaStream_t>(stream_)),
     "upload W");
  pi_ = pi;
  sigma2_ = sigma2;
  have_params_ = true;
  gram_fresh_ = false;
}

void BscEngine::get_params_ex(double* w, double* pi, double* sigma2, double* probs) {
  get_params(w, pi, sigma2);
  if (probs && family_ == kDsc) std::memcpy(probs, probs_.data(), probs_.size() * 8);
}

void BscEngine::get_params(double* w, double* pi, double* sigma2) {
  if (w)
    ck(cudaMemcpy2DAsync(w, (size_t)H_ * 8, d_w_, (size_t)Hp_ * 8, (size_t)H_ * 8, D_, cudaMemcpyDeviceToHost,
                         static_cast<cudaStream_t>(stream_)),
       "download W");
  sync();
  if (pi) *pi = pi_;
  if (sigma2) *sigma2 = sigma2_;
}

void BscEngine::refresh_gram() {
  enqueue_gram(stream_);
  gram_fresh_ = true;
}

// G = WᵀW on the DMMA GEMM, then the diagonal (selection scores) recomputed in
// the oracle's left-to-right order.
void BscEngine::enqueue_gram(void* stream, bool with_slices) {
  auto s = static_cast<cudaStream_t>(stream);
  const int H = static_cast<int>(H_);
  GemmArgs g{H, H, Dp_, d_w_, Hp_, d_w_, Hp_, d_g_, Hp_, 1.0, 0.0, Dp_, 0};
  ck(launch_dgemm<GRAM_CFG>(g, 1, s), "gram gemm");
  gram_diag_exact_kernel<<<(H_ + 31) / 32, 32, 0, s>>>(d_w_, D_, H_, Hp_, d_g_, Hp_, d_wnorm_, d_gdiag_);
  ck(cudaGetLastError(), "gram");
  launches_ += 2;
  if (oz_ && with_slices) slice_w(stream);
}

// The fields both enumerators share (EnumArgs, bsc_kernels.cuh): shapes, the
// resident buffers of this chunk, the state tables and the per-shard
// constants of linear_discrete.cpp:219-227 (host libm, as the reference).
void BscEngine::fill_enum_args(void* out, double temperature, bool cands, bool infer, uint64_t off, uint64_t rows,
                               int chunk, double log_p0) {
  (void)chunk;
  auto s = static_cast<cudaStream_t>(stream_);
  EnumArgs& a = *static_cast<EnumArgs*>(out);
  const double inv2s = 1.0 / (2.0 * sigma2_);
  const double norm_const = -0.5 * static_cast<double>(D_) * (kLog2Pi + std::log(sigma2_));
  const double zero_prior = static_cast<double>(H_) * log_p0;
  a.N = static_cast<int>(rows);
  a.D = D_;
  a.H = H_;
  a.Dp = Dp_;
  a.Hp = Hp_;
  a.hprime = hprime_;
  a.gamma = gamma_;
  a.Y = d_y_ + off * Dp_;
  a.W = d_w_;
  a.B = d_b_ + off * Hp_;
  a.G = d_g_;
  a.wnorm = d_wnorm_;
  a.gdiag = d_gdiag_;
  a.y2 = d_y2_ + off;
  a.ES = d_es_ + off * Hp_;
  a.ssT = d_stats_ + lay_.off_ssT();
  a.cand_out = cands ? d_cand_ + off * hprime_ : nullptr;
  a.map_mass = infer ? d_map_mass_ + off : nullptr;
  a.map_state = infer ? d_map_state_ + off : nullptr;
  a.err = d_err_;
  if (prof_on_) {
    if (!d_prof_) d_prof_ = dalloc<unsigned long long>(8, "enumerate phase profile");
    ck(cudaMemsetAsync(d_prof_, 0, 8 * sizeof(unsigned long long), s), "zero profile");
  }
  a.prof = prof_on_ ? static_cast<unsigned long long*>(d_prof_) : nullptr;
  a.sdesc = static_cast<const uint2*>(d_desc_);
  a.stage_desc_bytes = stage_tables_ ? desc_bytes_ : 0;
  a.stage_ent_bytes = stage_tables_ ? ent_bytes_ : 0;
  a.dfs = d_dfs_;
  a.level_off = d_level_off_;
  a.chunk = static_cast<const int4*>(d_chunk_);
  a.n_chunks = n_chunks_;
  a.n_multi = n_multi_;
  a.n_tab = n_tab_;
  a.n_coup = n_coup_;
  a.sched = static_cast<const SchedDesc*>(d_sched_);
  a.sched_ent = static_cast<const uint32_t*>(d_sched_ent_);
  a.sched_split = static_cast<const int4*>(d_sched_split_);
  a.n_slots = n_slots_;
  a.n_out = n_out_;
  a.inv2s = inv2s;
  a.base0 = zero_prior + norm_const;
  a.inv_T = 1.0 / temperature;
  a.weight_mode = weight_mode_;
  // |b_fast − b_oracle| ≤ eps_dot·‖W_h‖·‖y‖: DMMA (any order) and the oracle's
  // left-to-right sum each within γ_D; the int8-sliced product within
  // D·11·2⁻⁵⁶·s_y·s_h ≤ 5.5·D·2⁻⁵³‖y‖‖W_h‖ plus its fp64 group combine (ozaki_gemm.cuh)
  // fixed-point Σ⟨ssᵀ⟩ pairs: N contributions ≤ 1 per entry below 2^62
  int kfx = 62;
  for (uint64_t m = 1; m < std::max<uint64_t>(n_, 1) && kfx > 0; m <<= 1) --kfx;
  fx_scale_ = std::ldexp(1.0, kfx);
  a.fx_scale = fx_scale_;
  a.eps_dot = (oz_ && !infer) ? (7.0 * static_cast<double>(Dp_) + 16.0) * 0x1.0p-53
                              : 2.0 * (static_cast<double>(D_) + 2.0) * 0x1.0p-53;
}

void BscEngine::launch_enumerate(double temperature, bool cands, bool infer, uint64_t off, uint64_t rows,
                                 int chunk) {
  if (vpath()) {
    launch_enumerate_v(temperature, cands, infer, off, rows, chunk);
    return;
  }
  auto s = static_cast<cudaStream_t>(stream_);
  // value_table (:71-97, BSC :75-79) and the per-shard constants (:219-227),
  // computed on the host with the same libm as the reference.
  const double log_p1 = std::log(pi_), log_p0 = std::log(1.0 - pi_);
  EnumArgs a{};
  fill_enum_args(&a, temperature, cands, infer, off, rows, chunk, log_p0);
  a.log_pi = log_p1;
  a.dlp = log_p1 - log_p0;
  // scalar partial regions of this chunk (see estep_chunked)
  double* sc_front = d_warp_sc_ + ((size_t)0 * sc_chunks_ + chunk) * sc_ctas_ * 2;
  double* sc_fin = d_warp_sc_ + ((size_t)1 * sc_chunks_ + chunk) * sc_ctas_ * 2;
  double* sc_fb = d_warp_sc_ + ((size_t)2 * sc_chunks_ + chunk) * sc_ctas_ * 2;
  a.warp_scalars = sc_front;
  const int maxj = maxj_for(H_);
  void* args[] = {&a};
  const bool lane = lane_ok_ && !infer && temperature == 1.0 && weight_mode_ != 2;
  pscale_used_ = false;
  a.pscale = nullptr;
  if (!lane) {
    ck(cudaLaunchKernel(enum_fn(maxj, stage_tables_), dim3(enum_ctas_), dim3(enum_block_), args, enum_smem_, s),
       "enumerate launch");
    ck(cudaGetLastError(), "enumerate");
    ++launches_;
    return;
  }
  // lane path: selection (thread per point) → lane-per-point states → fallback points → finish
  a.rec = d_rec_;
  a.pmode = d_pmode_;
  a.cand_out = d_cand_ + off * hprime_;
  a.pscale = nullptr;
  pscale_used_ = false;
  const bool tm = timing_ && chunk == 0;
  lane_timed_ = tm;
  ck(cudaLaunchKernel(select_fn(static_cast<int>(hprime_)), dim3(front_ctas_), dim3(128), args, front_smem_, s),
     "select launch");
  if (tm) ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_[8]), s), "event");
  LaneArgs la{static_cast<int>(rows), static_cast<int>(hprime_), d_rec_, d_lout_, d_pmode_};
  void* largs[] = {&la};
  const unsigned wpc = static_cast<unsigned>(lane_wpc(gamma_, hprime_));
  ck(cudaLaunchKernel(lane_fn(gamma_, hprime_), dim3(static_cast<unsigned>(((rows + 31) / 32 + wpc - 1) / wpc)),
                      dim3(32 * wpc), largs, lane_smem_, s),
     "lane states launch");
  if (tm) ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_[9]), s), "event");
  a.warp_scalars = sc_fb;
  ck(cudaLaunchKernel(fallback_fn(maxj, stage_tables_), dim3(enum_ctas_), dim3(enum_block_), args, enum_smem_, s),
     "fallback launch");
  if (tm) ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_[10]), s), "event");
  FinishArgs fa{};
  fa.N = static_cast<int>(rows);
  fa.H = H_;
  fa.Hp = Hp_;
  fa.hp = hprime_;
  fa.out = d_lout_;
  fa.pmode = d_pmode_;
  fa.cand = d_cand_ + off * hprime_;
  fa.y2 = d_y2_ + off;
  fa.B = d_b_ + off * Hp_;
  fa.gdiag = d_gdiag_;
  fa.ES = d_es_ + off * Hp_;
  fa.ssT = d_stats_ + lay_.off_ssT();
  fa.cta_scalars = sc_fin;
  fa.base0 = a.base0;
  fa.inv2s = a.inv2s;
  fa.dlp = a.dlp;
  fa.fx_scale = a.fx_scale;
  es_sliced_ = false;
  if (oz_ && fs_ctas_ > 0) {
    // sliced path: the ⟨s⟩ rows go straight to the int8 operand of Yᵀ⟨S⟩ (finish_slice_kernels.cuh)
    FinishSliceArgs fsa{};
    fsa.f = fa;
    fsa.ess = d_ess_;
    fsa.slice_stride = static_cast<long long>(Hp_) * oz_npc_;
    fsa.colsum = d_ozcs_ + (off / 128) * Hp_;
    fsa.inv56 = 0x1.0p55;  // 2^56 / the ⟨S⟩ slice scale 2 (d_two_)
    void* fsargs[] = {&fsa};
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(fs_ctas_, (rows + 127) / 128));
    ck(cudaLaunchKernel(finish_slice_fn(fs_pt_), dim3(grid), dim3(fs_threads(fs_pt_)), fsargs, fs_smem_, s),
       "finish+slice launch");
    es_sliced_ = true;
  } else {
    void* fargs[] = {&fa};
    ck(cudaLaunchKernel(finish_fn(maxj), dim3(fin_ctas_), dim3(256), fargs, 0, s), "finish launch");
  }
  ck(cudaGetLastError(), "lane path");
  launches_ += 4;
}

void BscEngine::estep(double temperature, bool want_candidates) {
  if (!have_params_) throw Error(kConfig, "bsc: parameters not set");
  if (n_ == 0) throw Error(kData, "run: empty dataset");
  if (!(temperature >= 1.0) || !std::isfinite(temperature))
    throw Error(kConfig, "temperature must be finite and >= 1");
  ck(cudaSetDevice(device_), "set device");
  auto s = static_cast<cudaStream_t>(stream_);
  auto ev = [&](int i) {
    if (timing_) ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_[i]), s), "event");
  };
  estep_chunked(temperature, want_candidates, nullptr, n_);
}

// The E-step runs over row chunks: K1 (Y·W), the enumerator and K4 (Yᵀ⟨S⟩,
// accumulated into the same split-K partials, chunk after chunk) per chunk.
// With `host_y`, chunk c+1 is copied host→device on the copy stream while
// chunk c computes (the reference-facing step that takes host data).
void BscEngine::estep_chunked(double temperature, bool want_candidates, const double* host_y, uint64_t chunk) {
  auto s = static_cast<cudaStream_t>(stream_);
  auto ev = [&](int i) {
    if (timing_) ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_[i]), s), "event");
  };
  const uint64_t n = n_;
  chunk = std::max<uint64_t>(2, std::min<uint64_t>(n, chunk));
  chunk = (chunk + 1) & ~1ull;  // even row offsets (K4 reads K in pairs)
  if (oz_ && chunk < n) chunk = std::min<uint64_t>(n, (chunk + 127) & ~127ull);  // 16-byte Yᵀ slice offsets
  const int nchunks = static_cast<int>((n + chunk - 1) / chunk);
  if (nchunks > kMaxChunks) throw Error(kConfig, "gpu: too many E-step chunks");
  if (nchunks > colsum_chunks_) {
    dfree(d_warp_es_);
    dfree(d_warp_sc_);
    d_warp_es_ = dalloc<double>((size_t)nchunks * splits_ * Hp_, "split-K column sums");
    d_warp_sc_ = dalloc<double>((size_t)3 * nchunks * sc_ctas_ * 2, "cta scalars");
    colsum_chunks_ = nchunks;
  }
  if (vpath() && nchunks > vpart_chunks_) {
    dfree(d_vpart_);
    d_vpart_ = dalloc<double>((size_t)nchunks * enum_ctas_ * vpart_stride_, "cta partials");
    vpart_chunks_ = nchunks;
  }
  launches_ = 0;
  factored_ = false;
  NvtxRange nv_estep("bsc.estep");
  ev(0);
  if (!gram_fresh_) {
    NvtxRange nv("bsc.gram");
    refresh_gram();
  }
  ev(1);
  // per-CTA scalar partials: [role: whole/front pass, lane finish, fallback][chunk][sc_ctas_]
  estep_clear_kernel<<<64, 256, 0, s>>>(d_stats_ + lay_.off_ssT(), (long long)H_ * H_, d_err_, d_warp_es_,
                                        (long long)nchunks * splits_ * Hp_, d_warp_sc_,
                                        (long long)3 * nchunks * sc_ctas_ * 2);
  ck(cudaGetLastError(), "clear accumulators");
  ++launches_;
  sc_chunks_ = nchunks;
  // Yᵀ⟨S⟩ on the integer tensor cores: k-splits sized on the first (largest) chunk
  int oz_kchunk = 0, oz_splits0 = 0;
  if (oz_) {
    const long long npc = (static_cast<long long>(chunk) + 127) / 128 * 128;
    if (npc * Hp_ * oz::S > oz_ess_bytes_) {
      dfree(d_ess_);
      d_ess_ = dalloc<int8_t>((size_t)npc * Hp_ * oz::S, "ES slices");
      oz_ess_bytes_ = npc * Hp_ * oz::S;
    }
    oz_npc_ = npc;
    int sms = 148;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "sms");
    const int tiles = ((static_cast<int>(D_) + oz::BM - 1) / oz::BM) * ((static_cast<int>(H_) + oz::BN - 1) / oz::BN);
    const long long want = std::max(1, sms / tiles);
    const long long per = (static_cast<long long>(chunk) + want - 1) / want;
    oz_kchunk = static_cast<int>(std::min<long long>(oz::MAX_KJOB, (per + oz::BK - 1) / oz::BK * oz::BK));
    oz_splits0 = static_cast<int>((static_cast<long long>(chunk) + oz_kchunk - 1) / oz_kchunk);
    if (oz_splits0 > oz_part_slots_) {
      dfree(d_ozpart_);
      d_ozpart_ = dalloc<double>((size_t)oz_splits0 * part_stride_, "Yt<S> partials");
      oz_part_slots_ = oz_splits0;
    }
  }
  auto cs = static_cast<cudaStream_t>(copy_stream_);
  if (host_y) {
    ck(cudaEventRecord(static_cast<cudaEvent_t>(chunk_ev_[kMaxChunks]), s), "event");
    ck(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(chunk_ev_[kMaxChunks]), 0), "wait");
    for (int c = 0; c < nchunks; ++c) {  // all copies queued up front; compute waits per chunk
      const uint64_t off = c * chunk, rows = std::min<uint64_t>(chunk, n - off);
      if (static_cast<int>(D_) == Dp_)  // unpadded rows: one contiguous copy
        ck(cudaMemcpyAsync(d_y_ + off * Dp_, host_y + off * D_, rows * D_ * 8, cudaMemcpyHostToDevice, cs),
           "upload Y chunk");
      else
        ck(cudaMemcpy2DAsync(d_y_ + off * Dp_, (size_t)Dp_ * 8, host_y + off * D_, (size_t)D_ * 8, (size_t)D_ * 8, rows,
                             cudaMemcpyHostToDevice, cs),
           "upload Y chunk");
      ck(cudaEventRecord(static_cast<cudaEvent_t>(chunk_ev_[c]), cs), "event");
    }
  }
  for (int c = 0; c < nchunks; ++c) {
    const uint64_t off = c * chunk, rows = std::min<uint64_t>(chunk, n - off);
    if (host_y) {
      ck(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(chunk_ev_[c]), 0), "wait chunk");
      row_sqnorm_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(
          d_y_ + off * Dp_, static_cast<long long>(rows), D_, Dp_, d_y2_ + off);
      ++launches_;
    }
    if (oz_ && (host_y || nchunks > 1)) slice_y(off, rows, c, s);
    if (oz_ && c == 0 && !host_y && nchunks == 1 && !yts_whole_) slice_y(0, n, 0, s);  // after step_host
    nvtxRangePushA("bsc.gemm_yw");
    if (oz_) {  // K1: B = Y·W, int8 slices on tcgen05
      const long long cap_rows = static_cast<long long>((cap_n_ + 1) & ~1ull);
      oz::Args g{};
      g.sa = d_ysa_ + off;
      g.sb = d_wsb_;
      g.C = d_b_ + off * Hp_;
      g.ldc = Hp_;
      const oz::Operand A{d_ys_ + off * Kp_, cap_rows * Kp_, Kp_, static_cast<int>(rows), 0};
      const oz::Operand B{d_ws_, static_cast<long long>(Hp_) * round_up(Dp_, oz::BK), Hp_, Hp_, 1};
      ck(oz::launch_gemm(A, B, static_cast<int>(rows), Hp_, Kp_, g, oz_sms(device_), s), "oz gemm Y·W");
      ++launches_;
    } else {  // K1: B = Y·W
      GemmArgs g{static_cast<int>(rows), Hp_, Dp_, d_y_ + off * Dp_, Dp_, d_w_, Hp_, d_b_ + off * Hp_, Hp_,
                 1.0, 0.0, Dp_, 0};
      ck(launch_dgemm<GEMM1_CFG>(g, 1, s), "gemm Y·W");
      ++launches_;
    }
    nvtxRangePop();
    if (c == 0) ev(2);
    {
      NvtxRange nv("bsc.enumerate");
      launch_enumerate(temperature, want_candidates, false, off, rows, c);
    }
    if (c == 0) ev(3);
    NvtxRange nv_k4("bsc.gemm_ytes");
    if (oz_) {  // K4: Σ y⟨s⟩ᵀ += Yᵀ·ES — ⟨S⟩ᵀ slices (+ column sums = Σ⟨s⟩ partials), then tcgen05
      if (!es_sliced_) {  // (the lane path's finish pass has written the slices already)
        const unsigned kb = static_cast<unsigned>((rows + 127) / 128);
        oz::oz_slice_cols_kernel<<<dim3((Hp_ + 31) / 32, kb), 256, 0, s>>>(
            d_es_ + off * Hp_, Hp_, static_cast<long long>(rows), static_cast<int>(H_), Hp_,
            (static_cast<long long>(rows) + 127) / 128 * 128, d_two_, d_ess_, static_cast<long long>(Hp_) * oz_npc_,
            d_ozcs_ + (off / 128) * Hp_, pscale_used_ ? d_pscale_ + off : nullptr);
        ck(cudaGetLastError(), "slice ES");
        ++launches_;
      }
      es_sliced_ = false;
      if (c == nchunks - 1 && overlap_factor_ && !vpath()) fork_factor(nchunks, n);
      oz::Args g{};
      g.sa = d_ytsa_ + (size_t)((host_y || nchunks > 1) ? c : 0) * Dp_;
      g.sb = d_two_;
      g.C = d_ozpart_;
      g.ldc = Hp_;
      g.kchunk = oz_kchunk;
      g.c_split_stride = part_stride_;
      g.accumulate = c > 0;
      const oz::Operand A{d_yts_ + (off / oz::BK) * Dp_ * oz::BK, static_cast<long long>(Dp_) * oz_np_, Dp_, Dp_, 1};
      const oz::Operand B{d_ess_, static_cast<long long>(Hp_) * oz_npc_, Hp_, Hp_, 1};
      ck(oz::launch_gemm(A, B, static_cast<int>(D_), static_cast<int>(H_), static_cast<int>(rows), g, oz_sms(device_),
                         s),
         "oz gemm Yt·ES");
      ++launches_;
    } else {  // K4: Σ y⟨s⟩ᵀ += Yᵀ·ES over this chunk (+ fused Σ⟨s⟩), split-K over its rows
      const int krows = static_cast<int>((rows + 1) & ~1ull);
      int kchunk = (krows + splits_ - 1) / splits_;
      kchunk = (kchunk + 1) & ~1;
      const int splits = (krows + kchunk - 1) / kchunk;
      // the first chunk overwrites its partial slots (β = 0; the largest chunk, so
      // later chunks accumulate into slots it wrote); slots it leaves unused are cleared
      if (c == 0 && splits < splits_)
        ck(cudaMemsetAsync(d_part_ + (size_t)splits * part_stride_, 0,
                           (size_t)(splits_ - splits) * part_stride_ * 8, s),
           "zero partials");
      GemmArgs g{Dp_, Hp_, krows, d_y_ + off * Dp_, Dp_, d_es_ + off * Hp_, Hp_, d_part_, Hp_, 1.0,
                 c == 0 ? 0.0 : 1.0, kchunk, part_stride_, d_warp_es_ + (size_t)c * splits_ * Hp_};
      ck(Dp_ % 128 == 0 ? launch_dgemm<GEMM2_CFG>(g, splits, s) : launch_dgemm<GEMM2_CFG64>(g, splits, s),
         "gemm Yᵀ·ES");
      ++launches_;
    }
    if (c == 0) ev(4);
  }
  // the Yᵀ slices now carry one column scale per chunk (d_ytsa_[c]) unless one chunk ran
  if (oz_) yts_whole_ = nchunks == 1;
  NvtxRange nv_fin("bsc.finalize_stats");
  const long long DH = (long long)D_ * H_;
  if (oz_)  // Σ⟨s⟩ and the Σ⟨ssᵀ⟩ diagonal come from the slicer's column sums (finalize_moments)
    reduce_ysT_kernel<<<(DH + 255) / 256, 256, 0, s>>>(d_ozpart_, d_ozcs_, oz_splits0, 0, part_stride_, D_, H_, Hp_,
                                                        d_stats_, lay_.off_s(), lay_.off_ssT());
  else
    reduce_ysT_kernel<<<(DH + H_ + 255) / 256, 256, 0, s>>>(d_part_, d_warp_es_, splits_, nchunks * splits_,
                                                             part_stride_, D_, H_, Hp_, d_stats_, lay_.off_s(),
                                                             vpath() ? -1 : lay_.off_ssT());
  ++launches_;
  if (vpath()) {
    finalize_v(nchunks * enum_ctas_, n);
    ++launches_;
  } else if (factored_) {  // the side stream has finalised the moments and factored Σ⟨ssᵀ⟩
    ck(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_join_), 0), "join wait");
  } else if (oz_) {
    finalize_moments(s, nchunks, n);
  } else {
    finalize_stats_kernel<<<std::max(1u, std::min(1024u, (H_ * H_ + 255) / 256)), 256, 0, s>>>(
        3 * nchunks * sc_ctas_, d_warp_sc_, H_, static_cast<long long>(n), d_stats_, lay_.off_ssT(), lay_.off_tail(),
        1.0 / fx_scale_);
    counts_kernel<<<1, 32, 0, s>>>(d_stats_, lay_.off_s(), H_, lay_.off_tail());
    launches_ += 2;
  }
  ck(cudaGetLastError(), "finalize");
  ev(5);
}

void BscEngine::check_err() {
  int err = 0;
  ck(cudaMemcpyAsync(&err, d_err_, sizeof(int), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)),
     "err");
  sync();
  if (err & kErrNonFiniteScore) throw Error(kConfig, "select_candidates: scores must be finite");
  if (err & kErrNonFiniteLogJoint) throw Error(kNumeric, "log_sum_exp: empty support");
}

// The M-step is a fixed sequence of ~40 small launches for a given (D, H), in two
// parts: each runs eagerly once, is then captured into a CUDA graph and replayed.
void BscEngine::run_part(GraphPart& part, void (BscEngine::*enqueue)(void*), void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  if (!part.exec) {
    const int before = launches_;
    if (part.calls++ == 0) {
      (this->*enqueue)(s);
      part.nodes = launches_ - before;
      return;
    }
    cudaStream_t cap;
    ck(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
    ck(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
    (this->*enqueue)(cap);
    cudaGraph_t graph;
    ck(cudaStreamEndCapture(cap, &graph), "end capture");
    cudaGraphExec_t exec;
    ck(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    part.exec = exec;
    part.nodes = launches_ - before;
    launches_ = before;
  }
  ck(cudaGraphLaunch(static_cast<cudaGraphExec_t>(part.exec), s), "mstep graph");
  launches_ += part.nodes;
}

void BscEngine::mstep() {
  NvtxRange nv("bsc.mstep");
  ck(cudaSetDevice(device_), "set device");
  if (!factored_) run_part(factor_part_, &BscEngine::enqueue_factor, stream_);
  factored_ = false;
  run_part(update_part_, &BscEngine::enqueue_update, stream_);
  finish_mstep();
}

// Inside a step(), before the last chunk's Yᵀ⟨S⟩ product: every moment sum the factor needs
// is complete (pair sums, ⟨S⟩ column sums, per-CTA scalars), so the statistics' Σ⟨s⟩ / Σ⟨ssᵀ⟩ /
// scalar entries are finalised and Σ⟨ssᵀ⟩ + ridge·I factored on the side stream while the
// product runs. The same kernels in the same order as the serial path: identical bits.
void BscEngine::fork_factor(int nchunks, uint64_t n) {
  auto s = static_cast<cudaStream_t>(stream_);
  auto side = static_cast<cudaStream_t>(side_stream_);
  ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_fork_), s), "fork");
  ck(cudaStreamWaitEvent(side, static_cast<cudaEvent_t>(ev_fork_), 0), "fork wait");
  finalize_moments(side, nchunks, n);
  run_part(factor_part_, &BscEngine::enqueue_factor, side);
  ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_join_), side), "join");
  factored_ = true;
}

// Σ⟨s⟩ and the Σ⟨ssᵀ⟩ diagonal from the ⟨S⟩ column sums, the off-diagonals from the
// fixed-point pair sums, the scalars (BSC on the tensor-core product path).
void BscEngine::finalize_moments(void* stream, int nchunks, uint64_t n) {
  auto s = static_cast<cudaStream_t>(stream);
  oz::oz_colsum_reduce_kernel<<<(H_ + 7) / 8, 256, 0, s>>>(d_ozcs_, static_cast<int>((n + 127) / 128), Hp_,
                                                           static_cast<int>(H_), d_stats_ + lay_.off_s(),
                                                           d_stats_ + lay_.off_ssT(), static_cast<int>(H_));
  finalize_stats_kernel<<<std::max(1u, std::min(1024u, (H_ * H_ + 255) / 256)), 256, 0, s>>>(
      3 * nchunks * sc_ctas_, d_warp_sc_, H_, static_cast<long long>(n), d_stats_, lay_.off_ssT(), lay_.off_tail(),
      1.0 / fx_scale_);
  counts_kernel<<<1, 32, 0, s>>>(d_stats_, lay_.off_s(), H_, lay_.off_tail());
  ck(cudaGetLastError(), "finalize");
  launches_ += 3;
}

void BscEngine::enqueue_factor(void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  auto* sc = static_cast<MstepScalars*>(d_msc_);
  const int H = static_cast<int>(H_), D = static_cast<int>(D_);
  mstep_prepare_kernel<<<64, 256, 0, s>>>(d_stats_, lay_.off_ssT(), D, H, Hp_, d_bm_, d_x_, Hp_, sc, kPrepareFactor);
  ck(cudaGetLastError(), "mstep prepare");
  ++launches_;
  // blocked right-looking Cholesky, lower: L overwrites Bm
  for (int k0 = 0; k0 < H; k0 += kCholNb) {
    const int kb = std::min(kCholNb, H - k0), k1 = k0 + kb;
    potrf_diag_kernel<<<1, 256, 0, s>>>(d_bm_, Hp_, k0, kb, sc);
    ++launches_;
    if (k1 < H) {
      const int rows = H - k1;
      trsm_panel_warp_kernel<<<(rows + 7) / 8, 256, 0, s>>>(d_bm_, Hp_, k0, kb, k1, rows);
      GemmArgs g{rows, rows, kb, d_bm_ + (long long)k1 * Hp_ + k0, Hp_, d_bm_ + (long long)k1 * Hp_ + k0, Hp_,
                 d_bm_ + (long long)k1 * Hp_ + k1, Hp_, -1.0, 1.0, kb, 0};
      ck(launch_dgemm<SYRK_CFG>(g, 1, s), "syrk");
      launches_ += 2;
    }
  }
  // U = Lᵀ for the forward solve
  transpose_lower_kernel<<<dim3((H + 31) / 32, (Hp_ + 31) / 32), dim3(32, 8), 0, s>>>(d_bm_, Hp_, H, d_u_);
  ck(cudaGetLastError(), "cholesky");
  ++launches_;
}

void BscEngine::enqueue_update(void* stream) {
  auto s = static_cast<cudaStream_t>(stream);
  auto* sc = static_cast<MstepScalars*>(d_msc_);
  const int H = static_cast<int>(H_), D = static_cast<int>(D_);
  mstep_prepare_kernel<<<64, 256, 0, s>>>(d_stats_, lay_.off_ssT(), D, H, Hp_, d_bm_, d_x_, Hp_, sc, kPrepareRhs);
  ++launches_;
  // X·L·Lᵀ = Σy⟨s⟩ᵀ: forward (Z·Lᵀ = R, against U = Lᵀ) then backward (X·L = Z),
  // one warp per row of X over the full width
  {
    // 4 rows per CTA; pivot rows staged in blocks of rb (double-buffered)
    const unsigned blocks = static_cast<unsigned>((D + 3) / 4);
    const int rb = std::max(1, std::min(32, (160 * 1024) / (2 * Hp_ * 8)));
    const size_t smem = (static_cast<size_t>((H + 1) & ~1) + 2ull * rb * Hp_) * sizeof(double);
    for (bool fwd : {true, false}) {
      auto fn = solve_rows_fn(maxj_for(H_), fwd);
      ck(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem)),
         "solve smem");
      fn<<<blocks, 128, smem, s>>>(fwd ? d_u_ : d_bm_, Hp_, H, d_x_, Hp_, D, rb);
    }
  }
  launches_ += 2;
  ck(cudaGetLastError(), "solve");
  commit_w_kernel<<<64, 256, 0, s>>>(d_x_, Hp_, d_w_, Hp_, D, H, sc);
  // two branches from W': the next E-step's int8 operand slices on the side stream, and the
  // Gram (the next E-step's G; exact diagonal) that also feeds t3, σ² and π here
  auto side = static_cast<cudaStream_t>(side_stream_);
  const bool branch = oz_ && overlap_enabled_ && s != side;
  if (branch) {
    ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_branch_[0]), s), "branch");
    ck(cudaStreamWaitEvent(side, static_cast<cudaEvent_t>(ev_branch_[0]), 0), "branch wait");
    slice_w(side);
    ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_branch_[1]), side), "branch join");
  }
  enqueue_gram(s, !branch);
  mstep_traces_kernel<<<kTraceCtas, 256, 0, s>>>(d_w_, Hp_, d_g_, Hp_, d_stats_, lay_.off_ssT(), D, H,
                                                  d_trace_part_);
  mstep_scalars_kernel<<<1, 1, 0, s>>>(d_stats_, lay_.off_tail(), D, H, static_cast<int>(values_.size()),
                                       d_trace_part_, sc, d_err_, static_cast<char*>(d_result_));
  if (branch) ck(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_branch_[1]), 0), "branch join wait");
  ck(cudaGetLastError(), "mstep scalars");
  launches_ += 3;
}

void BscEngine::finish_mstep() {
  auto s = static_cast<cudaStream_t>(stream_);
  gram_fresh_ = true;
  if (timing_) ck(cudaEventRecord(static_cast<cudaEvent_t>(ev_[6]), s), "event");
  // one synchronisation per iteration: new π, σ², the (all-reduced) F and the E-step error
  // flag are in the mapped host block when the last M-step kernel (mstep_scalars_kernel) ends
  const size_t V = values_.size();
  sync();
  const int err = *static_cast<int*>(h_err_);
  if (err & kErrNonFiniteScore) throw Error(kConfig, "select_candidates: scores must be finite");
  if (err & kErrNonFiniteLogJoint) throw Error(kNumeric, "log_sum_exp: empty support");
  const auto* h = static_cast<const MstepScalars*>(h_msc_);
  const double* tail = static_cast<const double*>(h_tail_);
  sigma2_ = h->sigma2;
  last_F_ = tail[V + 1];
  if (family_ == kDsc) {
    // linear_discrete.cpp:382-404: probs of the non-zero values from the
    // counts, the rest on 0, floored at 1e-9 (model.hpp:34) and renormalised
    const double nh = tail[V + 2] * static_cast<double>(H_);
    double nonzero = 0.0;
    size_t k = 0;
    for (size_t i = 0; i < alphabet_.size(); ++i) {
      if (alphabet_[i] == 0.0) continue;
      probs_[i] = tail[k++] / nh;
      nonzero += probs_[i];
    }
    for (size_t i = 0; i < alphabet_.size(); ++i)
      if (alphabet_[i] == 0.0) probs_[i] = 1.0 - nonzero;
    bool floored = false;
    for (double& q : probs_)
      if (q < 1e-9) {
        q = 1e-9;
        floored = true;
      }
    if (floored) {
      double tot = 0.0;
      for (double q : probs_) tot += q;
      for (double& q : probs_) q /= tot;
    }
  } else {
    pi_ = h->pi;
  }
  if (timing_) {
    auto el = [&](int a, int b) {
      float ms = 0;
      cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(ev_[a]), static_cast<cudaEvent_t>(ev_[b]));
      return ms;
    };
    t_.gram_ms = el(0, 1);
    t_.gemm1_ms = el(1, 2);
    t_.enum_ms = el(2, 3);
    t_.gemm2_ms = el(3, 4);
    t_.finalize_ms = el(4, 5);
    t_.mstep_ms = el(5, 6);
    if (lane_timed_) {
      t_.front_ms = el(2, 8);
      t_.states_ms = el(8, 9);
      t_.fallback_ms = el(9, 10);
      t_.finish_ms = el(10, 3);
    } else {
      t_.front_ms = t_.states_ms = t_.fallback_ms = t_.finish_ms = 0.f;
    }
  }
}

double BscEngine::step(double temperature) {
  overlap_factor_ = overlap_enabled_;
  try {
    estep(temperature);
  } catch (...) {
    overlap_factor_ = factored_ = false;
    throw;
  }
  overlap_factor_ = false;
  mstep();
  return last_F_;
}

void BscEngine::get_stats(double* sum_s, double* sum_ssT, double* sum_y_sT, double* value_counts, double* scalars) {
  std::vector<double> h(lay_.count());
  ck(cudaMemcpyAsync(h.data(), d_stats_, h.size() * 8, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)),
     "stats D2H");
  sync();
  if (sum_y_sT) std::memcpy(sum_y_sT, h.data() + lay_.off_ysT(), (size_t)D_ * H_ * 8);
  if (sum_s) std::memcpy(sum_s, h.data() + lay_.off_s(), (size_t)H_ * 8);
  if (sum_ssT) std::memcpy(sum_ssT, h.data() + lay_.off_ssT(), (size_t)H_ * H_ * 8);
  const double* t = h.data() + lay_.off_tail();
  const size_t V = values_.size();
  if (value_counts) std::memcpy(value_counts, t, V * 8);
  if (scalars) {
    scalars[0] = t[V];
    scalars[1] = t[V + 1];
    scalars[2] = t[V + 2];
  }
}

void BscEngine::set_stats(const double* sum_s, const double* sum_ssT, const double* sum_y_sT,
                          const double* value_counts, const double* scalars) {
  std::vector<double> h(lay_.count(), 0.0);
  std::memcpy(h.data() + lay_.off_ysT(), sum_y_sT, (size_t)D_ * H_ * 8);
  std::memcpy(h.data() + lay_.off_s(), sum_s, (size_t)H_ * 8);
  std::memcpy(h.data() + lay_.off_ssT(), sum_ssT, (size_t)H_ * H_ * 8);
  double* t = h.data() + lay_.off_tail();
  const size_t V = values_.size();
  std::memcpy(t, value_counts, V * 8);
  t[V] = scalars[0];
  t[V + 1] = scalars[1];
  t[V + 2] = scalars[2];
  if (!(t[V + 2] >= 1.0)) throw Error(kConfig, "linear model: mstep without data");
  ck(cudaMemcpyAsync(d_stats_, h.data(), h.size() * 8, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream_)),
     "stats H2D");
  sync();
}

void BscEngine::get_candidates(uint32_t* out) {
  ck(cudaMemcpyAsync(out, d_cand_, n_ * hprime_ * 4, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)),
     "cand D2H");
  sync();
}

// LinearDiscreteModel::inference (linear_discrete.cpp:429-450): T = 1, MAP
// state (first maximum in reference order), its mass, and ⟨s_n⟩.
void BscEngine::inference(double* map_states, double* map_mass, double* expected) {
  if (!have_params_) throw Error(kConfig, "bsc: parameters not set");
  ck(cudaSetDevice(device_), "set device");
  auto s = static_cast<cudaStream_t>(stream_);
  if (!gram_fresh_) refresh_gram();
  GemmArgs g{static_cast<int>(n_), Hp_, Dp_, d_y_, Dp_, d_w_, Hp_, d_b_, Hp_, 1.0, 0.0, Dp_, 0};
  ck(launch_dgemm<GEMM1_CFG>(g, 1, s), "gemm Y·W");
  ck(cudaMemsetAsync(d_stats_ + lay_.off_ssT(), 0, (size_t)H_ * H_ * 8, s), "zero ssT");
  ck(cudaMemsetAsync(d_err_, 0, 2 * sizeof(int), s), "zero err");
  launch_enumerate(1.0, true, true, 0, n_, 0);
  std::vector<int> st(n_);
  std::vector<uint32_t> cand(n_ * hprime_);
  ck(cudaMemcpyAsync(st.data(), d_map_state_, n_ * 4, cudaMemcpyDeviceToHost, s), "map D2H");
  ck(cudaMemcpyAsync(cand.data(), d_cand_, cand.size() * 4, cudaMemcpyDeviceToHost, s), "cand D2H");
  ck(cudaMemcpyAsync(map_mass, d_map_mass_, n_ * 8, cudaMemcpyDeviceToHost, s), "mass D2H");
  ck(cudaMemcpy2DAsync(expected, (size_t)H_ * 8, d_es_, (size_t)Hp_ * 8, (size_t)H_ * 8, n_, cudaMemcpyDeviceToHost,
                       s),
     "ES D2H");
  check_err();
  const std::vector<uint64_t>& masks = dfs_masks_;
  std::memset(map_states, 0, n_ * H_ * 8);
  if (vpath()) {  // index → (unit, value) lists: zero, (h, v) h-major, then DFS patterns
    const uint64_t V = values_.size();
    for (uint64_t n = 0; n < n_; ++n) {
      const uint64_t i = static_cast<uint64_t>(st[n]);
      double* row = map_states + n * H_;
      if (i == 0) continue;
      if (i <= H_ * V) {
        row[(i - 1) / V] = values_[(i - 1) % V];
        continue;
      }
      for (const auto& pv : dfs_patterns_[i - 1 - H_ * V]) row[cand[n * hprime_ + pv.first]] = values_[pv.second];
    }
    return;
  }
  for (uint64_t n = 0; n < n_; ++n) {
    const int i = st[n];
    double* row = map_states + n * H_;
    if (i == 0) continue;
    if (i <= static_cast<int>(H_)) {
      row[i - 1] = 1.0;
      continue;
    }
    const uint64_t m = masks[i - 1 - H_];
    for (uint32_t p = 0; p < hprime_; ++p)
      if ((m >> p) & 1) row[cand[n * hprime_ + p]] = 1.0;
  }
}

}  // namespace bscgpu
