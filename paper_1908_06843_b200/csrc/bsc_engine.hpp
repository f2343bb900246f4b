// BscEngine: one device's share of the BSC truncated-EM step.
//
// Owns the resident data shard, the dictionary and the device statistics,
// and launches the sm_100a kernels of bsc_kernels.cuh / mstep_kernels.cuh /
// dgemm.cuh. One host thread per engine; not re-entrant.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace bscgpu {

// Error taxonomy mirroring prsp (core.hpp:32-43); codes are prsp_status.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline constexpr int kConfig = 2, kData = 3, kNumeric = 4, kInternal = 5;

// Packed statistics buffer (the all-reduce payload): [Σy⟨s⟩ᵀ D·H | Σ⟨s⟩ H |
// Σ⟨ssᵀ⟩ H·H | value_counts V | Σ‖y‖² | Σ log Z | N] (SuffStats fields,
// linear_discrete.cpp:211-217; V = number of non-zero values).
struct StatsLayout {
  long long D, H, V = 1;
  long long off_ysT() const { return 0; }
  long long off_s() const { return D * H; }
  long long off_ssT() const { return D * H + H; }
  long long off_tail() const { return D * H + H + H * H; }  // counts[V], y2, logZ, points
  long long count() const { return off_tail() + V + 3; }
};

// Linear discrete families (LinearDiscreteModel, linear_discrete.hpp:31-87).
enum Family : int { kBsc = 0, kTsc = 1, kDsc = 2 };

// The lane-per-point state pass for (γ, H') (lane_engine.cu).
// BSC_GUARD=1: throws Error(kInternal) naming the first device buffer with a damaged guard region
void check_device_guards();
void guard_probe(long long bytes, long long index);
const void* lane_fn(int gamma, int hprime);
int lane_smem(int gamma, int hprime);  // its dynamic shared memory per CTA (bytes)
int lane_wpc(int gamma, int hprime);   // its warps (32-point tiles) per CTA
const void* select_fn(int hprime);     // thread-per-point selection pass (select_kernels.cuh)
int select_smem(int latents);          // its dynamic shared memory per CTA (bytes)
const void* finish_fn(int maxj);       // lane_finish_kernel<MAXJ>
const void* finish_slice_fn(int pt);   // lane_finish_slice_kernel<PT> (finish_slice_kernels.cuh)
int finish_slice_smem(int pt, int latents, int hp_padded, int hprime);

// The multi-valued enumerator instantiation for (MAXJ, staged) (ldv_engine.cu).
const void* ldv_kernel_fn(int maxj, bool staged);

struct EngineTimings {
  float gram_ms, gemm1_ms, enum_ms, gemm2_ms, finalize_ms, mstep_ms;
  // the enumerator's lane path, split (0 when the single-kernel pass ran)
  float front_ms, states_ms, fallback_ms, finish_ms;
};

class BscEngine {
 public:
  BscEngine(uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma, uint64_t state_cap, int device);
  // family kTsc / kDsc (dsc: `alphabet` of n_alpha distinct values containing 0)
  BscEngine(int family, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma, uint64_t state_cap,
            const double* alphabet, uint32_t n_alpha, int device);
  ~BscEngine();
  BscEngine(const BscEngine&) = delete;
  BscEngine& operator=(const BscEngine&) = delete;

  void set_stream(void* stream);
  int device() const { return device_; }
  void* stream() const { return stream_; }

  // Data shard (row-major N×D, host or device pointer); stays resident.
  void load_data(const double* y, uint64_t n, bool device_ptr);
  uint64_t points() const { return n_; }

  void set_params(const double* w_host, double pi, double sigma2);
  void get_params(double* w_host, double* pi, double* sigma2);
  // dsc: probabilities aligned with the sorted alphabet (pi unused)
  void set_params_ex(const double* w_host, double pi, double sigma2, const double* probs, uint32_t n_probs);
  void get_params_ex(double* w_host, double* pi, double* sigma2, double* probs);
  int family() const { return family_; }
  uint32_t num_values() const { return static_cast<uint32_t>(values_.size()); }  // non-zero values
  uint32_t alphabet_size() const { return static_cast<uint32_t>(alphabet_.size()); }
  const std::vector<double>& alphabet() const { return alphabet_; }

  // E-step over the resident shard at temperature T → device stats buffer.
  void estep(double temperature, bool want_candidates = false);
  // M-step from the device stats buffer → device params (W, π, σ²).
  void mstep();
  // estep + mstep; returns F = Σ_n log Z_n at the incoming params.
  double step(double temperature);
  // The same step over host data (copied per call, chunk by chunk, the copies
  // overlapping the E-step of earlier chunks).
  double step_streamed(const double* y_host, uint64_t n, double temperature, uint64_t chunk);

  double* stats_device() { return d_stats_; }
  double last_free_energy() const { return last_F_; }
  const StatsLayout& layout() const { return lay_; }
  void get_stats(double* sum_s, double* sum_ssT, double* sum_y_sT, double* value_counts, double* scalars);
  void set_stats(const double* sum_s, const double* sum_ssT, const double* sum_y_sT, const double* value_counts,
                 const double* scalars);
  void get_candidates(uint32_t* out);  // N×H' from the last estep(…, true)
  void inference(double* map_states, double* map_mass, double* expected);

  uint32_t dim() const { return D_; }
  uint32_t latents() const { return H_; }
  uint32_t hprime() const { return hprime_; }
  uint32_t gamma() const { return gamma_; }
  uint64_t states_per_point() const { return 1 + (uint64_t)H_ * values_.size() + n_multi_; }
  int enum_launch_ctas() const { return enum_ctas_; }
  int enum_warps() const { return enum_warps_total_; }
  const EngineTimings& timings() const { return t_; }
  void set_timing(bool on) { timing_ = on; }
  // per-phase cycle accounting inside the enumerator (profiling builds of a
  // run: BSC_ENUM_PROFILE=1); summed over warps, last E-step
  void enum_phase_cycles(unsigned long long* out8);
  int kernel_launches_last_step() const { return launches_; }
  void sync();

 private:
  void init(int device);
  void build_template();
  void build_template_v();  // multi-valued families (ldv_engine.cu)
  void launch_enumerate_v(double temperature, bool cands, bool infer, uint64_t off, uint64_t rows, int chunk);
  void fill_enum_args(void* enum_args, double temperature, bool cands, bool infer, uint64_t off, uint64_t rows,
                      int chunk, double log_p0);
  bool vpath() const { return family_ != kBsc; }
  int ldv_per_warp_bytes() const;
  void finalize_v(int nparts, uint64_t n);
  void ensure_work(uint64_t n);
  void refresh_gram();
  void launch_enumerate(double temperature, bool cands, bool infer, uint64_t off, uint64_t rows, int chunk);
  void estep_chunked(double temperature, bool want_candidates, const double* host_y, uint64_t chunk);
  void check_err();
  // The M-step in two graph-captured parts: the factor (Bm, Cholesky, Lᵀ) needs only the
  // E-step's moment sums; the update (right-hand side, solves, W', Gram, σ²/π) needs Yᵀ⟨S⟩.
  struct GraphPart {
    void* exec = nullptr;  // cudaGraphExec_t
    int calls = 0, nodes = 0;
  };
  void run_part(GraphPart& part, void (BscEngine::*enqueue)(void*), void* stream);
  void enqueue_factor(void* stream);
  void enqueue_update(void* stream);
  void fork_factor(int nchunks, uint64_t n);
  void finalize_moments(void* stream, int nchunks, uint64_t n);
  void enqueue_gram(void* stream, bool with_slices = true);
  void finish_mstep();

  int family_ = kBsc;
  std::vector<double> alphabet_;  // dsc: sorted alphabet with 0; bsc {0,1}; tsc {-1,0,1}
  std::vector<double> values_;    // the non-zero values, ascending
  std::vector<double> probs_;     // dsc probabilities (aligned with alphabet_)
  uint32_t D_, H_, hprime_, gamma_;
  uint64_t cap_;
  int device_;
  int Dp_, Hp_;
  void* stream_ = nullptr;
  bool own_stream_ = false;
  StatsLayout lay_{};

  // params (host mirror of the scalars; W lives on the device)
  double pi_ = 0.5, sigma2_ = 1.0;
  bool have_params_ = false, gram_fresh_ = false;

  // template tables
  int n_multi_ = 0, n_tab_ = 0, n_coup_ = 0, n_slots_ = 0, n_out_ = 0;
  int n_chunks_ = 1;          // BSC table chunks (consecutive roots); n_tab_ / n_coup_ are per chunk maxima
  void* d_chunk_ = nullptr;   // int4 per chunk {row base, rows, level-1 rows, first root}
  int desc_bytes_ = 0, ent_bytes_ = 0;  // table sizes (16-byte multiples)
  bool stage_tables_ = false;           // staged into shared memory per CTA
  std::vector<uint64_t> dfs_masks_;  // multi-active supports in reference order
  std::vector<std::vector<std::pair<uint8_t, uint8_t>>> dfs_patterns_;  // V path: (position, value index)
  double* d_vpart_ = nullptr;        // V path: per-CTA partials [chunks][ctas][vpart_stride_]
  int vpart_stride_ = 0, vpart_chunks_ = 0;
  void* d_desc_ = nullptr;
  int* d_dfs_ = nullptr;
  int* d_level_off_ = nullptr;
  void* d_sched_ = nullptr;  // SchedDesc[γ]: subtree levels γ−1 … 1, then the moment gather
  void* d_sched_ent_ = nullptr;  // int2 entries, [rows][32]
  void* d_sched_split_ = nullptr;  // int4 {target, first slot, end slot, -} per split output

  uint64_t n_ = 0, cap_n_ = 0;
  double *d_y_ = nullptr, *d_w_ = nullptr, *d_g_ = nullptr, *d_wnorm_ = nullptr, *d_gdiag_ = nullptr;
  double* d_y2_ = nullptr;  // ‖y_n‖² per resident point
  double *d_b_ = nullptr, *d_es_ = nullptr;
  double *d_stats_ = nullptr, *d_smulti_ = nullptr;
  double *d_warp_es_ = nullptr, *d_warp_sc_ = nullptr;
  double* d_part_ = nullptr;  // split-K partials
  int splits_ = 1;
  long long part_stride_ = 0;
  uint32_t* d_cand_ = nullptr;
  int* d_map_state_ = nullptr;
  double* d_map_mass_ = nullptr;
  int* d_err_ = nullptr;
  // M-step workspace
  double *d_bm_ = nullptr, *d_x_ = nullptr, *d_trace_part_ = nullptr, *d_u_ = nullptr;
  void* d_msc_ = nullptr;
  void *h_result_ = nullptr, *d_result_ = nullptr;                // pinned + mapped: the iteration's result
  void *h_msc_ = nullptr, *h_tail_ = nullptr, *h_err_ = nullptr;  // views into h_result_
  double last_F_ = 0.0;
  GraphPart factor_part_, update_part_;
  // step(): the factor runs on a side stream beside the Yᵀ⟨S⟩ product, which leaves SMs idle
  // (its grid is a multiple of the output tiles: 144 of 148 CTAs at c2, 120 at c3)
  void* side_stream_ = nullptr;
  void *ev_fork_ = nullptr, *ev_join_ = nullptr, *ev_branch_[2] = {};
  bool overlap_enabled_ = true;  // BSC_MSTEP_OVERLAP=0 turns it off
  bool overlap_factor_ = false;  // this E-step belongs to a step(): fork the factor
  bool factored_ = false;        // the factor of the current statistics is in Bm / U

  int enum_ctas_ = 0, enum_warps_total_ = 0, enum_block_ = 256, enum_smem_ = 0;
  // host-streamed E-step: copy stream + per-chunk events
  static constexpr int kMaxChunks = 256;
  void* copy_stream_ = nullptr;
  void* chunk_ev_[kMaxChunks + 1] = {};
  int colsum_chunks_ = 0;
  bool timing_ = false;
  bool prof_on_ = false;
  int weight_mode_ = 0;
  // lane-per-point state pass (lane_kernels.cuh)
  bool lane_ok_ = false;
  int front_ctas_ = 0, front_smem_ = 0, fin_ctas_ = 0, lane_smem_ = 0;
  int fs_ctas_ = 0, fs_pt_ = 32, fs_smem_ = 0;  // finish fused with the ⟨S⟩ᵀ slicer
  bool es_sliced_ = false;                      // the finish pass of this chunk wrote the ⟨S⟩ᵀ slices
  int sc_ctas_ = 0, sc_chunks_ = 1;  // per-CTA scalar partial regions
  double *d_rec_ = nullptr, *d_lout_ = nullptr;
  int* d_pmode_ = nullptr;
  void* d_prof_ = nullptr;
  EngineTimings t_{};
  int launches_ = 0;
  // int8-sliced tcgen05 GEMMs (ozaki_gemm.cuh) for the binary family's Y·W and Yᵀ⟨S⟩
  bool oz_ = false;
  int Kp_ = 0;                          // Y / W slice row length (Dp_ rounded to 16)
  long long oz_np_ = 0;                 // Yᵀ slice row length (resident rows rounded to 128)
  long long oz_npc_ = 0;                // ⟨S⟩ᵀ slice row length (chunk rows rounded to 128)
  int8_t *d_ys_ = nullptr, *d_yts_ = nullptr, *d_ws_ = nullptr, *d_ess_ = nullptr;
  double *d_ysa_ = nullptr, *d_ytsa_ = nullptr, *d_wsb_ = nullptr, *d_two_ = nullptr;
  double *d_ozpart_ = nullptr, *d_ozcs_ = nullptr;
  double* d_pscale_ = nullptr;  // per-point ⟨s⟩-row scales deferred to the ⟨S⟩ slicer (lane path)
  bool pscale_used_ = false;
  bool yts_whole_ = true;
  double fx_scale_ = 1.0;  // 2^k of the fixed-point Σ⟨ssᵀ⟩ pair accumulation (this E-step)  // Yᵀ slices scaled over the whole resident shard (false after a chunked step_host)
  unsigned long long* d_ozmax_ = nullptr;
  int oz_part_slots_ = 0, oz_ytsa_chunks_ = 0;
  long long oz_ess_bytes_ = 0;
  void slice_y(uint64_t off, uint64_t rows, int chunk, void* stream);
  void slice_w(void* stream);
  void* ev_[12] = {};
  bool lane_timed_ = false;
};

}  // namespace bscgpu
