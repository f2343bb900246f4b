// McaEngine implementation (see mca_engine.hpp). Reference:
// MaxCausesModel::step / estep_impl / residual_impl / mstep_fixedpoint
// (/root/reference/proj/src/max_causes.cpp:180-446).
#include "mca_engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "dgemm.cuh"
#include "engine_util.hpp"
#include "mca_kernels.cuh"

namespace bscgpu {

using namespace util;

namespace {

#define MCA_GEMM1_CFG 128, 64, 16, 32, 32, true, true, 3
#define MCA_GEMM2_CFG 128, 64, 16, 32, 32, false, true, 3

const void* mca_fn(int maxj) {
  switch (maxj) {
    case 1: return (const void*)mca_enumerate_kernel<1>;
    case 2: return (const void*)mca_enumerate_kernel<2>;
    case 4: return (const void*)mca_enumerate_kernel<4>;
    case 6: return (const void*)mca_enumerate_kernel<6>;
    case 8: return (const void*)mca_enumerate_kernel<8>;
    case 10: return (const void*)mca_enumerate_kernel<10>;
    case 12: return (const void*)mca_enumerate_kernel<12>;
    case 16: return (const void*)mca_enumerate_kernel<16>;
    case 24: return (const void*)mca_enumerate_kernel<24>;
    default: return (const void*)mca_enumerate_kernel<32>;
  }
}

}  // namespace

McaEngine::McaEngine(int mode, double rho, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma,
                     uint64_t state_cap, int device)
    : mode_(mode), rho_(rho), D_(dim), H_(latents), hprime_(hprime), gamma_(gamma), cap_(state_cap),
      device_(device) {
  const std::string nm = mode == 0 ? "mca" : "mmca";
  if (mode != 0 && mode != 1) throw Error(kConfig, "max causes: unknown mode");
  // MaxCausesModel ctor (:83-99) and TruncationConfig::validate (truncation.cpp:23-30)
  if (D_ == 0 || H_ == 0) throw Error(kConfig, nm + ": dim and latents must be >= 1");
  if (hprime_ == 0 || hprime_ > H_) throw Error(kConfig, "truncation: hprime must satisfy 1 <= hprime <= latents");
  if (gamma_ == 0 || gamma_ > hprime_) throw Error(kConfig, "truncation: gamma must satisfy 1 <= gamma <= hprime");
  if (cap_ == 0) throw Error(kConfig, "truncation: state cap must be >= 1");
  if (rho_ < 0.0) throw Error(kConfig, nm + ": soft winner exponent must be >= 0");
  if (rho_ > 0.0 && mode_ != 0) throw Error(kConfig, "soft winners require the non-negative max mode");
  if (hprime_ > 64) throw Error(kConfig, "gpu: hprime > 64 is not supported by the sm_100a enumerator");
  if (H_ > 1024) throw Error(kConfig, "gpu: latents > 1024 is not supported by the sm_100a enumerator");
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "device count");
  if (device_ < 0 || device_ >= ndev) throw Error(kConfig, "gpu: device index out of range");
  ck(cudaSetDevice(device_), "set device");
  cudaStream_t s;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  stream_ = s;
  Dp_ = round_up(static_cast<int>(D_), 8);
  Hp_ = round_up(static_cast<int>(H_), 8);

  // reference pattern order (truncation.cpp:116-147, V = 1): depth | last << 8 | first << 16
  std::vector<uint32_t> pdesc;
  std::vector<int> support;
  auto dfs = [&](auto&& self, uint32_t next) -> void {
    if (support.size() >= 2)
      pdesc.push_back(static_cast<uint32_t>(support.size()) | (static_cast<uint32_t>(support.back()) << 8) |
                      (static_cast<uint32_t>(support[0]) << 16));
    if (support.size() == gamma_) return;
    for (uint32_t p = next; p < hprime_; ++p) {
      support.push_back(static_cast<int>(p));
      self(self, p + 1);
      support.pop_back();
    }
  };
  uint64_t total = 1 + H_;
  {
    // truncated_state_count (truncation.cpp:83-93), saturating
    auto binom = [](uint64_t n, uint64_t k) -> long double {
      long double r = 1;
      for (uint64_t i = 1; i <= k; ++i) r = r * (n - k + i) / i;
      return r;
    };
    long double t = 1.0L + H_;
    for (uint32_t k = 2; k <= gamma_; ++k) t += binom(hprime_, k);
    if (t > static_cast<long double>(cap_))
      throw Error(kConfig, "state explosion: " + std::to_string(static_cast<unsigned long long>(t)) +
                               " states per data point exceeds cap of " + std::to_string(cap_));
    total = static_cast<uint64_t>(t);
  }
  if (total > 200000) throw Error(kConfig, "gpu: state template too large for the max-causes enumerator");
  if (gamma_ >= 2) dfs(dfs, 0);
  n_multi_ = static_cast<int>(pdesc.size());
  d_pdesc_ = dalloc<uint32_t>(pdesc.size(), "patterns");
  if (!pdesc.empty())
    ck(cudaMemcpy(d_pdesc_, pdesc.data(), pdesc.size() * 4, cudaMemcpyHostToDevice), "patterns");

  d_w_ = dalloc<double>((size_t)Dp_ * Hp_, "W");
  d_wn_ = dalloc<double>((size_t)Dp_ * Hp_, "W'");
  d_wt_ = dalloc<double>((size_t)H_ * Dp_, "Wt");
  d_wtn_ = dalloc<double>((size_t)H_ * Dp_, "W't");
  d_g_ = dalloc<double>((size_t)H_ * Hp_, "gram scratch");
  d_gdiag_ = dalloc<double>(H_, "gdiag");
  d_gdiagn_ = dalloc<double>(H_, "gdiag'");
  d_wnorm_ = dalloc<double>(H_, "wnorm");
  d_wnormn_ = dalloc<double>(H_, "wnorm'");
  d_stats_ = dalloc<double>(stats_count(), "stats");
  d_err_ = dalloc<int>(1, "err");
  d_sc_ = dalloc<McaScalars>(1, "scalars");
  const int per_warp = McaSmem::make(Dp_, static_cast<int>(gamma_), n_multi_, static_cast<int>(hprime_),
                                     static_cast<int>(H_))
                           .total *
                       8;
  const int cap = 227 * 1024 - 1024 - 1024;
  if (per_warp > cap) throw Error(kConfig, "gpu: max-causes working set too large for shared memory");
  int warps = std::min(8, cap / per_warp);
  block_ = warps * 32;
  smem_ = warps * per_warp;
  const void* fn = mca_fn(maxj_for(H_));
  ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_), "mca smem attr");
}

McaEngine::~McaEngine() {
  cudaSetDevice(device_);
  for (void* p : {(void*)d_y_, (void*)d_y2_, (void*)d_w_, (void*)d_wn_, (void*)d_wt_, (void*)d_wtn_, (void*)d_g_,
                  (void*)d_gdiag_, (void*)d_gdiagn_, (void*)d_wnorm_, (void*)d_wnormn_, (void*)d_b_, (void*)d_bn_,
                  (void*)d_qs_, (void*)d_es_, (void*)d_stats_, (void*)d_part_, (void*)d_colsum_, (void*)d_cta_,
                  (void*)d_pdesc_, (void*)d_cand_, (void*)d_map_state_, (void*)d_map_mass_, (void*)d_err_, d_sc_})
    dfree(p);
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

void McaEngine::sync() { ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)), "sync"); }

void McaEngine::ensure_work(uint64_t n) {
  if (n <= cap_n_ && d_y_) return;
  for (void* p : {(void*)d_y_, (void*)d_y2_, (void*)d_b_, (void*)d_bn_, (void*)d_qs_, (void*)d_es_, (void*)d_part_,
                  (void*)d_colsum_, (void*)d_cta_, (void*)d_cand_, (void*)d_map_state_, (void*)d_map_mass_})
    dfree(p);
  const uint64_t rows = (n + 1) & ~1ull;
  d_y_ = dalloc<double>(rows * Dp_, "Y");
  d_y2_ = dalloc<double>(rows, "y2");
  d_b_ = dalloc<double>(rows * Hp_, "B");
  d_bn_ = dalloc<double>(rows * Hp_, "B'");
  d_qs_ = dalloc<double>(rows * Hp_, "Qs");
  d_es_ = dalloc<double>(rows * Hp_, "ES");
  d_cand_ = dalloc<uint32_t>(rows * hprime_, "cand");
  d_map_state_ = dalloc<int>(rows, "map state");
  d_map_mass_ = dalloc<double>(rows, "map mass");
  cap_n_ = n;
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, device_), "props");
  const int tiles = ((Dp_ + 127) / 128) * ((Hp_ + 63) / 64);
  splits_ = std::max(1, std::min<int>((2 * prop.multiProcessorCount) / tiles, static_cast<int>(rows / 512)));
  splits_ = std::max(1, splits_);
  part_stride_ = (long long)Dp_ * Hp_;
  d_part_ = dalloc<double>((size_t)splits_ * part_stride_, "splitK partials");
  d_colsum_ = dalloc<double>((size_t)splits_ * Hp_, "colsums");
  const int warps = block_ / 32;
  int per_sm = 0;
  ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mca_fn(maxj_for(H_)), block_, smem_), "occupancy");
  ctas_ = std::max(1, per_sm) * prop.multiProcessorCount;
  ctas_ = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ctas_, (n + warps - 1) / warps)));
  d_cta_ = dalloc<double>((size_t)ctas_ * 4, "cta partials");
}

void McaEngine::load_data(const double* y, uint64_t n) {
  if (n == 0) throw Error(kData, "run: empty dataset");
  ck(cudaSetDevice(device_), "set device");
  ensure_work(n);
  auto s = static_cast<cudaStream_t>(stream_);
  ck(cudaMemsetAsync(d_y_, 0, cap_n_ * Dp_ * 8, s), "clear Y");
  ck(cudaMemcpy2DAsync(d_y_, (size_t)Dp_ * 8, y, (size_t)D_ * 8, (size_t)D_ * 8, n, cudaMemcpyHostToDevice, s),
     "upload Y");
  row_sqnorm_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(d_y_, static_cast<long long>(n), D_, Dp_,
                                                                       d_y2_);
  ck(cudaGetLastError(), "y2");
  n_ = n;
  sync();
}

// MaxCausesModel::validate (:101-117).
void McaEngine::set_params(const double* w, double pi, double sigma2) {
  const std::string nm = mode_ == 0 ? "mca" : "mmca";
  for (size_t i = 0; i < (size_t)D_ * H_; ++i)
    if (!std::isfinite(w[i])) throw Error(kNumeric, nm + ": non-finite dictionary");
  if (mode_ == 0)
    for (size_t i = 0; i < (size_t)D_ * H_; ++i)
      if (w[i] < 1e-8) throw Error(kConfig, "mca: dictionary entries must be >= the weight floor");
  if (!(pi > 0.0 && pi < 1.0)) throw Error(kConfig, nm + ": pi must lie in (0,1)");
  if (!(sigma2 > 0.0)) throw Error(kConfig, nm + ": sigma2 must be positive");
  ck(cudaSetDevice(device_), "set device");
  ck(cudaMemcpy2DAsync(d_w_, (size_t)Hp_ * 8, w, (size_t)H_ * 8, (size_t)H_ * 8, D_, cudaMemcpyHostToDevice,
                       static_cast<cudaStream_t>(stream_)),
     "upload W");
  pi_ = pi;
  sigma2_ = sigma2;
  have_params_ = true;
  have_update_ = false;
  sync();
}

void McaEngine::get_params(double* w, double* pi, double* sigma2) {
  if (w)
    ck(cudaMemcpy2DAsync(w, (size_t)H_ * 8, d_w_, (size_t)Hp_ * 8, (size_t)H_ * 8, D_, cudaMemcpyDeviceToHost,
                         static_cast<cudaStream_t>(stream_)),
       "download W");
  sync();
  if (pi) *pi = pi_;
  if (sigma2) *sigma2 = sigma2_;
}

// Wᵀ, ‖W_h‖² (oracle order, as w.col(h).squaredNorm()) and B = Y·W.
void McaEngine::refresh(const double* w, double* wt, double* gdiag, double* wnorm, double* b) {
  auto s = static_cast<cudaStream_t>(stream_);
  transpose_w_kernel<<<dim3((H_ + 31) / 32, (Dp_ + 31) / 32), dim3(32, 8), 0, s>>>(w, D_, H_, Hp_, wt, Dp_);
  gram_diag_exact_kernel<<<(H_ + 31) / 32, 32, 0, s>>>(w, D_, H_, Hp_, d_g_, Hp_, wnorm, gdiag);
  GemmArgs g{static_cast<int>(n_), Hp_, Dp_, d_y_, Dp_, w, Hp_, b, Hp_, 1.0, 0.0, Dp_, 0};
  ck(launch_dgemm<MCA_GEMM1_CFG>(g, 1, s), "gemm Y·W");
}

void McaEngine::launch(int pass, double temperature, bool cands, bool infer) {
  auto s = static_cast<cudaStream_t>(stream_);
  const double pi = pi_, s2 = sigma2_;
  McaArgs a{};
  a.N = static_cast<int>(n_);
  a.D = D_;
  a.H = H_;
  a.Dp = Dp_;
  a.Hp = Hp_;
  a.hprime = hprime_;
  a.gamma = gamma_;
  a.mode = mode_;
  a.n_multi = n_multi_;
  a.pass = pass;
  a.Y = d_y_;
  a.W = d_w_;
  a.WT = d_wt_;
  a.WTn = d_wtn_;
  a.B = d_b_;
  a.Bn = d_bn_;
  a.gdiag = d_gdiag_;
  a.gdiagn = d_gdiagn_;
  a.wnorm = d_wnorm_;
  a.y2 = d_y2_;
  a.pdesc = d_pdesc_;
  a.Qs = d_qs_;
  a.num = d_stats_;
  a.den = d_stats_ + (size_t)D_ * H_;
  a.cta_part = d_cta_;
  a.cand_out = cands ? d_cand_ : nullptr;
  a.ES = infer ? d_es_ : nullptr;
  a.map_mass = infer ? d_map_mass_ : nullptr;
  a.map_state = infer ? d_map_state_ : nullptr;
  a.err = d_err_;
  // constants of estep_impl (:199-203), host libm as the reference
  a.lp1 = std::log(pi);
  a.lp0 = std::log(1.0 - pi);
  a.norm_const = -0.5 * static_cast<double>(D_) * (kLog2Pi + std::log(s2));
  a.inv2s = 1.0 / (2.0 * s2);
  a.inv_T = 1.0 / temperature;
  a.rho = rho_;
  a.eps_dot = 2.0 * (static_cast<double>(D_) + 2.0) * 0x1.0p-53;
  void* args[] = {&a};
  ck(cudaLaunchKernel(mca_fn(maxj_for(H_)), dim3(ctas_), dim3(block_), args, smem_, s), "mca launch");
  ck(cudaGetLastError(), "mca enumerate");
}

void McaEngine::estep(double temperature) {
  if (!have_params_) throw Error(kConfig, "max causes: parameters not set");
  if (n_ == 0) throw Error(kData, "run: empty dataset");
  if (!(temperature >= 1.0) || !std::isfinite(temperature))
    throw Error(kConfig, "temperature must be finite and >= 1");
  ck(cudaSetDevice(device_), "set device");
  auto s = static_cast<cudaStream_t>(stream_);
  refresh(d_w_, d_wt_, d_gdiag_, d_wnorm_, d_b_);
  ck(cudaMemsetAsync(d_stats_, 0, stats_count() * 8, s), "zero stats");
  ck(cudaMemsetAsync(d_err_, 0, sizeof(int), s), "zero err");
  ck(cudaMemsetAsync(d_part_, 0, (size_t)splits_ * part_stride_ * 8, s), "zero partials");
  ck(cudaMemsetAsync(d_colsum_, 0, (size_t)splits_ * Hp_ * 8, s), "zero colsums");
  launch(0, temperature, true, false);
  {  // singleton winner statistics: Σ_n y_n Q_s(n,:)ᵀ (+ column sums) on DMMA
    const int krows = static_cast<int>((n_ + 1) & ~1ull);
    int kchunk = (krows + splits_ - 1) / splits_;
    kchunk = (kchunk + 1) & ~1;
    const int splits = (krows + kchunk - 1) / kchunk;
    GemmArgs g{Dp_, Hp_, krows, d_y_, Dp_, d_qs_, Hp_, d_part_, Hp_, 1.0, 1.0, kchunk, part_stride_, d_colsum_};
    ck(launch_dgemm<MCA_GEMM2_CFG>(g, splits, s), "gemm Yᵀ·Qs");
  }
  const long long DH = (long long)D_ * H_;
  mca_finalize_kernel<<<static_cast<unsigned>((DH + 1 + 255) / 256), 256, 0, s>>>(
      d_part_, part_stride_, splits_, d_colsum_, splits_, D_, H_, Hp_, d_cta_, ctas_, static_cast<long long>(n_),
      d_stats_);
  ck(cudaGetLastError(), "mca finalize");
  int err = 0;
  ck(cudaMemcpyAsync(&err, d_err_, sizeof(int), cudaMemcpyDeviceToHost, s), "err");
  double tail[3];
  ck(cudaMemcpyAsync(tail, d_stats_ + 2 * DH, sizeof tail, cudaMemcpyDeviceToHost, s), "tail");
  sync();
  if (err & kErrNonFiniteScore) throw Error(kConfig, "select_candidates: scores must be finite");
  if (err & kErrNonFiniteLogJoint) throw Error(kNumeric, "log_sum_exp: empty support");
  last_F_ = tail[1];
}

void McaEngine::get_stats(double* num, double* den, double* scalars) {
  const size_t DH = (size_t)D_ * H_;
  std::vector<double> h(stats_count());
  ck(cudaMemcpyAsync(h.data(), d_stats_, h.size() * 8, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)),
     "stats D2H");
  sync();
  if (num) std::memcpy(num, h.data(), DH * 8);
  if (den) std::memcpy(den, h.data() + DH, DH * 8);
  if (scalars) std::memcpy(scalars, h.data() + 2 * DH, 3 * 8);
}

void McaEngine::set_stats(const double* num, const double* den, const double* scalars) {
  const size_t DH = (size_t)D_ * H_;
  std::vector<double> h(stats_count());
  std::memcpy(h.data(), num, DH * 8);
  std::memcpy(h.data() + DH, den, DH * 8);
  std::memcpy(h.data() + 2 * DH, scalars, 3 * 8);
  if (!(scalars[2] >= 1.0)) throw Error(kConfig, std::string(mode_ == 0 ? "mca" : "mmca") + ": mstep without data");
  ck(cudaMemcpyAsync(d_stats_, h.data(), h.size() * 8, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream_)),
     "stats H2D");
  sync();
}

void McaEngine::mstep_fixedpoint() {
  auto s = static_cast<cudaStream_t>(stream_);
  const long long DH = (long long)D_ * H_;
  double pts = 0.0;
  ck(cudaMemcpyAsync(&pts, d_stats_ + 2 * DH + 2, 8, cudaMemcpyDeviceToHost, s), "points");
  sync();
  if (!(pts >= 1.0)) throw Error(kConfig, std::string(mode_ == 0 ? "mca" : "mmca") + ": mstep without data");
  ck(cudaMemcpyAsync(d_wn_, d_w_, (size_t)Dp_ * Hp_ * 8, cudaMemcpyDeviceToDevice, s), "W' init");
  mca_mstep_kernel<<<static_cast<unsigned>(std::min<long long>((DH + 255) / 256, 1024)), 256, 0, s>>>(
      d_stats_, d_w_, D_, H_, Hp_, mode_, d_wn_, static_cast<McaScalars*>(d_sc_));
  ck(cudaGetLastError(), "mca mstep");
  McaScalars sc{};
  ck(cudaMemcpyAsync(&sc, d_sc_, sizeof sc, cudaMemcpyDeviceToHost, s), "scalars");
  sync();
  pi_new_ = sc.pi;
  have_update_ = true;
}

void McaEngine::get_updated(double* w, double* pi) {
  if (!have_update_) throw Error(kConfig, "max causes: no M-step update");
  if (w)
    ck(cudaMemcpy2DAsync(w, (size_t)H_ * 8, d_wn_, (size_t)Hp_ * 8, (size_t)H_ * 8, D_, cudaMemcpyDeviceToHost,
                         static_cast<cudaStream_t>(stream_)),
       "download W'");
  sync();
  if (pi) *pi = pi_new_;
}

void McaEngine::residual_and_commit(double temperature) {
  if (!have_update_) throw Error(kConfig, "max causes: no M-step update");
  auto s = static_cast<cudaStream_t>(stream_);
  refresh(d_wn_, d_wtn_, d_gdiagn_, d_wnormn_, d_bn_);
  launch(1, temperature, false, false);
  mca_sigma_kernel<<<1, 32, 0, s>>>(d_cta_, ctas_, static_cast<long long>(n_), D_, static_cast<McaScalars*>(d_sc_));
  ck(cudaGetLastError(), "mca sigma");
  McaScalars sc{};
  ck(cudaMemcpyAsync(&sc, d_sc_, sizeof sc, cudaMemcpyDeviceToHost, s), "scalars");
  ck(cudaMemcpyAsync(d_w_, d_wn_, (size_t)Dp_ * Hp_ * 8, cudaMemcpyDeviceToDevice, s), "commit W");
  sync();
  sigma2_ = sc.sigma2;
  pi_ = pi_new_;
  have_update_ = false;
}

double McaEngine::residual_device_sum() {
  McaScalars sc{};
  ck(cudaMemcpyAsync(&sc, d_sc_, sizeof sc, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)), "scalars");
  sync();
  return sc.residual;
}

double McaEngine::step(double temperature) {
  estep(temperature);
  const double f = last_F_;
  mstep_fixedpoint();
  residual_and_commit(temperature);
  return f;
}

void McaEngine::candidates(uint32_t* out) {
  estep(1.0);
  ck(cudaMemcpyAsync(out, d_cand_, n_ * hprime_ * 4, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream_)),
     "cand D2H");
  sync();
}

// MaxCausesModel::inference (:448-468): T = 1, MAP (first maximum in
// reference order), its mass and ⟨s_n⟩.
void McaEngine::inference(double* map_states, double* map_mass, double* expected) {
  if (!have_params_) throw Error(kConfig, "max causes: parameters not set");
  auto s = static_cast<cudaStream_t>(stream_);
  refresh(d_w_, d_wt_, d_gdiag_, d_wnorm_, d_b_);
  ck(cudaMemsetAsync(d_stats_, 0, stats_count() * 8, s), "zero stats");
  ck(cudaMemsetAsync(d_err_, 0, sizeof(int), s), "zero err");
  launch(0, 1.0, true, true);
  std::vector<int> st(n_);
  std::vector<uint32_t> cand(n_ * hprime_);
  int err = 0;
  ck(cudaMemcpyAsync(st.data(), d_map_state_, n_ * 4, cudaMemcpyDeviceToHost, s), "map D2H");
  ck(cudaMemcpyAsync(cand.data(), d_cand_, cand.size() * 4, cudaMemcpyDeviceToHost, s), "cand D2H");
  ck(cudaMemcpyAsync(map_mass, d_map_mass_, n_ * 8, cudaMemcpyDeviceToHost, s), "mass D2H");
  ck(cudaMemcpy2DAsync(expected, (size_t)H_ * 8, d_es_, (size_t)Hp_ * 8, (size_t)H_ * 8, n_, cudaMemcpyDeviceToHost,
                       s),
     "ES D2H");
  ck(cudaMemcpyAsync(&err, d_err_, sizeof(int), cudaMemcpyDeviceToHost, s), "err");
  sync();
  if (err & kErrNonFiniteScore) throw Error(kConfig, "select_candidates: scores must be finite");
  if (err & kErrNonFiniteLogJoint) throw Error(kNumeric, "log_sum_exp: empty support");
  // pattern list (reference order) for decoding multi-active MAP states
  std::vector<std::vector<int>> pats;
  std::vector<int> support;
  auto dfs = [&](auto&& self, uint32_t next) -> void {
    if (support.size() >= 2) pats.push_back(support);
    if (support.size() == gamma_) return;
    for (uint32_t p = next; p < hprime_; ++p) {
      support.push_back(static_cast<int>(p));
      self(self, p + 1);
      support.pop_back();
    }
  };
  if (gamma_ >= 2) dfs(dfs, 0);
  std::memset(map_states, 0, n_ * H_ * 8);
  for (uint64_t n = 0; n < n_; ++n) {
    const int i = st[n];
    double* row = map_states + n * H_;
    if (i == 0) continue;
    if (i <= static_cast<int>(H_)) {
      row[i - 1] = 1.0;
      continue;
    }
    for (int p : pats[i - 1 - H_]) row[cand[n * hprime_ + p]] = 1.0;
  }
}

}  // namespace bscgpu
