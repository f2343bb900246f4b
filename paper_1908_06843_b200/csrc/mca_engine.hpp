// McaEngine: one device's share of the max-causes truncated-EM step
// (MaxCausesModel, /root/reference/proj/src/max_causes.cpp) on sm_100a.
//
// Step = E pass (log Z, winner statistics) → fixed-point M-step (W', π') →
// residual pass under W' with the incoming posterior (σ²'), as
// MaxCausesModel::step (:416-446). Kernels: mca_kernels.cuh, DMMA GEMMs from
// dgemm.cuh. One host thread per engine; not re-entrant.
#pragma once
#include <cstdint>
#include <vector>

#include "bsc_engine.hpp"

namespace bscgpu {

class McaEngine {
 public:
  // mode 0 = mca (max), 1 = mmca (absmax); rho = soft winner exponent (mca only)
  McaEngine(int mode, double rho, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma,
            uint64_t state_cap, int device);
  ~McaEngine();
  McaEngine(const McaEngine&) = delete;
  McaEngine& operator=(const McaEngine&) = delete;

  void load_data(const double* y, uint64_t n);
  void set_params(const double* w, double pi, double sigma2);
  void get_params(double* w, double* pi, double* sigma2);
  // E pass → device stats [winner_num D·H | winner_den D·H | sum_act | log_partition | points]
  void estep(double temperature);
  void get_stats(double* winner_num, double* winner_den, double* scalars);
  void set_stats(const double* winner_num, const double* winner_den, const double* scalars);
  // fixed-point M-step from the device stats: W' and π' (kept beside W until commit)
  void mstep_fixedpoint();
  void get_updated(double* w, double* pi);
  // residual pass (posterior at the current params, residual under W'), then W ← W', π, σ²
  void residual_and_commit(double temperature);
  double step(double temperature);  // returns F = Σ log Z at the incoming params
  void set_sigma2(double s2) {
    if (!(s2 > 0.0)) throw Error(kConfig, "max causes: sigma2 must be positive");
    sigma2_ = s2;
  }
  void candidates(uint32_t* out);
  void inference(double* map_states, double* map_mass, double* expected);
  double* stats_device() { return d_stats_; }
  uint64_t stats_count() const { return 2ull * D_ * H_ + 3; }
  double residual_device_sum();  // Σ_n residual of the last residual pass (for cross-rank sums)
  uint64_t states_per_point() const { return 1 + H_ + n_multi_; }
  double last_free_energy() const { return last_F_; }
  void sync();

 private:
  void refresh(const double* w_dev, double* wt, double* gdiag, double* wnorm, double* b_out);
  void launch(int pass, double temperature, bool cands, bool infer);
  void ensure_work(uint64_t n);

  int mode_;
  double rho_;
  uint32_t D_, H_, hprime_, gamma_;
  uint64_t cap_;
  int device_;
  int Dp_, Hp_;
  void* stream_ = nullptr;
  double pi_ = 0.1, sigma2_ = 1.0, pi_new_ = 0.1;
  bool have_params_ = false, have_update_ = false;
  int n_multi_ = 0;
  uint64_t n_ = 0, cap_n_ = 0;
  double *d_y_ = nullptr, *d_y2_ = nullptr;
  double *d_w_ = nullptr, *d_wn_ = nullptr, *d_wt_ = nullptr, *d_wtn_ = nullptr;
  double *d_gdiag_ = nullptr, *d_gdiagn_ = nullptr, *d_wnorm_ = nullptr, *d_wnormn_ = nullptr, *d_g_ = nullptr;
  double *d_b_ = nullptr, *d_bn_ = nullptr, *d_qs_ = nullptr, *d_es_ = nullptr;
  double *d_stats_ = nullptr, *d_part_ = nullptr, *d_colsum_ = nullptr, *d_cta_ = nullptr;
  uint32_t* d_pdesc_ = nullptr;
  uint32_t* d_cand_ = nullptr;
  int* d_map_state_ = nullptr;
  double* d_map_mass_ = nullptr;
  int* d_err_ = nullptr;
  void* d_sc_ = nullptr;
  int splits_ = 1;
  long long part_stride_ = 0;
  int ctas_ = 0, block_ = 256, smem_ = 0;
  double last_F_ = 0.0;
};

}  // namespace bscgpu
