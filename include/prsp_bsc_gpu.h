/* prsp_bsc_gpu — B200 (sm_100a) drop-in for the BSC truncated-EM step of prsp.
 *
 * C ABI over the CUDA engine (paper_1908_06843_b200/csrc). Plain pointers
 * and sizes only. Conventions follow the reference C API
 * (/root/reference/proj/include/prsp.h:23-26, :39-45):
 *   - functions return PRSP_OK (0) or a prsp_status code
 *     (2 config, 3 data, 4 numeric, 5 internal);
 *   - the message of the last failure on this thread is prsp_bsc_gpu_last_error();
 *   - outputs are written only on success; the caller owns host buffers,
 *     the context owns all device memory;
 *   - one host thread per context (not re-entrant).
 * Matrices are row-major fp64: Y is N×D (one data point per row), W is D×H.
 * "scalars" arrays are {sum_y2, log_partition, points}.
 *
 * Reference interfaces replaced (paths under /root/reference/proj/src):
 *   prsp_bsc_gpu_create        LinearDiscreteModel ctor (linear_discrete.cpp:32-62)
 *                              + TruncationConfig::validate (truncation.cpp:23-30)
 *   prsp_bsc_gpu_step          LinearDiscreteModel::step (linear_discrete.cpp:410-427)
 *   prsp_bsc_gpu_estep         LinearDiscreteModel::estep_stats (:327-334) over the resident shard
 *   prsp_bsc_gpu_mstep         LinearDiscreteModel::mstep (:336-408)
 *   prsp_bsc_gpu_inference     LinearDiscreteModel::inference (:429-450)
 *   prsp_bsc_gpu_candidates    select_candidates per point as in estep_impl (:240-253)
 *   prsp_bsc_gpu_step_host     Model::step with host DataSet + params in, params + F out
 *                              (the call em.cpp:39 makes every iteration)
 *   prsp_bsc_generate          LinearDiscreteModel::generate (:452-479)
 *   prsp_bsc_bars_generate     make_bars (bars.cpp:33-65) / prsp_bars_generate (prsp.h:76-80)
 *   prsp_bsc_standard_init     LinearDiscreteModel::standard_init (:129-148)
 *   prsp_bsc_gpu_create_model  LinearDiscreteModel(DiscreteFamily, …, dsc_values) (:32-61) for
 *                              "bsc" / "tsc" / "dsc"; prsp_session_set_model / _set_values
 *                              (prsp.h:95-101) name the family and the dsc alphabet the same way
 *   prsp_bsc_gpu_set_params_ex LinearDiscreteParams{w, sigma2, pi, values, probs} (model.hpp:41-47)
 *                              + LinearDiscreteModel::validate (:99-127)
 *
 * Families other than bsc: value_counts (get/set_stats and the statistics
 * buffer) has one entry per non-zero latent value (SuffStats "value_counts"
 * 1×V, linear_discrete.cpp:214), tail = [value_counts V | sum_y2 | log_partition | points].
 */
#ifndef PRSP_BSC_GPU_H
#define PRSP_BSC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes: the values of prsp_status (prsp.h:39-45), under names that do not
 * clash with prsp.h when both are included. */
enum {
  PRSP_BSC_GPU_OK = 0,
  PRSP_BSC_GPU_ERR_CONFIG = 2,
  PRSP_BSC_GPU_ERR_DATA = 3,
  PRSP_BSC_GPU_ERR_NUMERIC = 4,
  PRSP_BSC_GPU_ERR_INTERNAL = 5
};

typedef struct prsp_bsc_gpu prsp_bsc_gpu; /* one device's engine + resident shard */

const char* prsp_bsc_gpu_version(void);
const char* prsp_bsc_gpu_last_error(void);
int prsp_bsc_gpu_device_count(void);

/* ---- context ----------------------------------------------------------- */
int prsp_bsc_gpu_create(uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma, uint64_t state_cap,
                        int device, prsp_bsc_gpu** out);
/* model: "bsc", "tsc" or "dsc"; dsc takes its latent alphabet (`values`, n_values ≥ 2
 * distinct values containing 0, any order: sorted like the reference ctor);
 * values/n_values are ignored for bsc and tsc. */
int prsp_bsc_gpu_create_model(const char* model, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma,
                              uint64_t state_cap, const double* values, uint32_t n_values, int device,
                              prsp_bsc_gpu** out);
/* family: 0 bsc, 1 tsc, 2 dsc; n_values: non-zero values (the value_counts length);
 * alphabet_out (nullable) receives the sorted alphabet including 0 (alphabet_size entries). */
int prsp_bsc_gpu_model_info(const prsp_bsc_gpu* ctx, int* family, uint32_t* n_values, uint32_t* alphabet_size,
                            double* alphabet_out);
void prsp_bsc_gpu_free(prsp_bsc_gpu* ctx);
/* Run on an existing cudaStream_t (e.g. torch's current stream); NULL = own stream. */
int prsp_bsc_gpu_set_stream(prsp_bsc_gpu* ctx, void* cuda_stream);
int prsp_bsc_gpu_sync(prsp_bsc_gpu* ctx);
int prsp_bsc_gpu_states_per_point(const prsp_bsc_gpu* ctx, uint64_t* out);

/* ---- resident data shard and parameters -------------------------------- */
int prsp_bsc_gpu_load_data(prsp_bsc_gpu* ctx, const double* y_host, uint64_t n);
int prsp_bsc_gpu_load_data_device(prsp_bsc_gpu* ctx, const double* y_device, uint64_t n);
int prsp_bsc_gpu_set_params(prsp_bsc_gpu* ctx, const double* w, double pi, double sigma2);
int prsp_bsc_gpu_get_params(prsp_bsc_gpu* ctx, double* w, double* pi, double* sigma2);
/* Any family: pi for bsc/tsc; probs (alphabet_size entries, aligned with the
 * sorted alphabet, summing to 1) for dsc. get_params_ex writes probs for dsc only. */
int prsp_bsc_gpu_set_params_ex(prsp_bsc_gpu* ctx, const double* w, double pi, double sigma2, const double* probs,
                               uint32_t n_probs);
int prsp_bsc_gpu_get_params_ex(prsp_bsc_gpu* ctx, double* w, double* pi, double* sigma2, double* probs);

/* ---- the hot path ------------------------------------------------------- */
/* E-step over the resident shard into the device statistics buffer. */
int prsp_bsc_gpu_estep(prsp_bsc_gpu* ctx, double temperature);
/* Device statistics buffer (fp64, packed [sum_y_sT D·H | sum_s H | sum_ssT H·H |
 * value_counts | sum_y2 | log_partition | points]) for an in-place all-reduce
 * across ranks between estep and mstep. */
int prsp_bsc_gpu_stats_buffer(prsp_bsc_gpu* ctx, double** device_ptr, uint64_t* count);
int prsp_bsc_gpu_get_stats(prsp_bsc_gpu* ctx, double* sum_s, double* sum_ssT, double* sum_y_sT,
                           double* value_counts, double* scalars);
int prsp_bsc_gpu_set_stats(prsp_bsc_gpu* ctx, const double* sum_s, const double* sum_ssT, const double* sum_y_sT,
                           const double* value_counts, const double* scalars);
/* M-step from the device statistics buffer; the new params stay resident. */
int prsp_bsc_gpu_mstep(prsp_bsc_gpu* ctx);
/* estep + mstep on the resident shard; *free_energy = Σ_n log Z_n at the incoming params. */
int prsp_bsc_gpu_step(prsp_bsc_gpu* ctx, double temperature, double* free_energy);
/* ---- multi-GPU: one process per GPU, each holding its row
 * shard (ShardPlan::with_shards, parallel.cpp:27-43); the only exchange is the
 * sum of the packed statistics, replacing map_reduce's ordered fold
 * (parallel.cpp:109-158). NCCL is resolved at run time (dlopen libnccl.so.2).
 *   prsp_bsc_gpu_nccl_unique_id   ncclGetUniqueId (root rank; send the 128 bytes to the others)
 *   prsp_bsc_gpu_nccl_init        ncclCommInitRank on the context's device (owned by ctx)
 *   prsp_bsc_gpu_nccl_attach      use a communicator the host owns (ncclComm_t, borrowed)
 *   prsp_bsc_gpu_step_allreduce   LinearDiscreteModel::step over the job: local E-step,
 *                                 ncclAllReduce(sum) of the statistics on the engine stream,
 *                                 replicated M-step; F = the job's Σ log Z. */
int prsp_bsc_gpu_nccl_unique_id(char* id128);
int prsp_bsc_gpu_nccl_init(prsp_bsc_gpu* ctx, const char* id128, int nranks, int rank);
int prsp_bsc_gpu_nccl_attach(prsp_bsc_gpu* ctx, void* nccl_comm);
int prsp_bsc_gpu_step_allreduce(prsp_bsc_gpu* ctx, double temperature, double* free_energy);
/* F = Σ_n log Z_n (all ranks, once the statistics were all-reduced) of the last M-step's input. */
int prsp_bsc_gpu_free_energy(prsp_bsc_gpu* ctx, double* out);
/* Reference-facing step: host Y and params in, host params and F out
 * (copies inside; Y may be pinned for full PCIe rate). */
int prsp_bsc_gpu_step_host(prsp_bsc_gpu* ctx, const double* y_host, uint64_t n, const double* w, double pi,
                           double sigma2, double temperature, double* w_out, double* pi_out, double* sigma2_out,
                           double* free_energy);

/* ---- parity hooks and inference ----------------------------------------- */
/* Candidate sets (N×H', ascending) of the resident shard at the current params. */
int prsp_bsc_gpu_candidates(prsp_bsc_gpu* ctx, uint32_t* out);
/* map_states N×H (0/1), map_mass N, expected N×H (⟨s_n⟩). */
int prsp_bsc_gpu_inference(prsp_bsc_gpu* ctx, double* map_states, double* map_mass, double* expected);
/* Device timings of the last step (ms): gram, gemm Y·W, enumerate, gemm Yᵀ⟨S⟩, finalize, mstep. */
int prsp_bsc_gpu_set_timing(prsp_bsc_gpu* ctx, int on);
int prsp_bsc_gpu_timings(prsp_bsc_gpu* ctx, float* out6);
/* The same six, then the enumerator's lane-path launches (front pass, lane-per-point states,
   fallback, finish; zeros when the single-kernel pass ran): the first min(n, 10) values. */
int prsp_bsc_gpu_timings_ex(prsp_bsc_gpu* ctx, float* out, int n);
int prsp_bsc_gpu_launches(prsp_bsc_gpu* ctx, int* out);
/* Test hook (compute-sanitizer's memcheck is not available on every pool): with BSC_GUARD=1 in the
 * environment every device buffer of the library carries 256 guard bytes on both sides;
 * this call synchronises the device and returns PRSP_BSC_GPU_ERR_INTERNAL, naming the buffer in
 * last_error, if a kernel has written into any guard. Without BSC_GUARD it returns OK. */
int prsp_bsc_gpu_check_guards(void);
/* BSC_GUARD=2 maps every device buffer so that it ends (to 16 bytes) at the end of its mapping with an
 * unmapped page behind it: a device load or store past the end of a buffer is an immediate fault
 * (overruns by reads included, which guard bytes cannot see). This probe reads byte `index` of a
 * fresh `bytes`-byte buffer on the device; past the end it returns PRSP_BSC_GPU_ERR_INTERNAL and
 * leaves the CUDA context unusable, so tests call it from a process of their own. */
int prsp_bsc_gpu_guard_probe(int64_t bytes, int64_t index);
/* Enumerator cycles per phase (summed over warps) of the last E-step when the
 * process runs with BSC_ENUM_PROFILE=1, else zeros: scores, selection, log-joint
 * terms, state log-joints, exp, MAP, subtree + moment sums, output + loop. */
int prsp_bsc_gpu_enum_phase_cycles(prsp_bsc_gpu* ctx, uint64_t* out8);

/* ---- fixtures (CPU; the reference's generators, same draw order) -------- */
int prsp_bsc_bars_generate(uint32_t size, uint64_t n, double prob, double amplitude, double noise, int max_mode,
                           uint64_t seed, double* y_out, double* truth_out);
int prsp_bsc_generate(uint32_t dim, uint32_t latents, const double* w, double pi, double sigma2, uint64_t n,
                      uint64_t seed, double* y_out);
/* Unit-norm columns × scale, N(0,1) from RngStream::derived(seed, "wtru"). */
int prsp_bsc_random_dictionary(uint32_t dim, uint32_t latents, uint64_t seed, double scale, double* w_out);
/* BASELINE.json init: W = mean_d + 0.25·std_d·z, π = 1/H, σ² = mean data variance. */
int prsp_bsc_baseline_init(uint32_t dim, uint32_t latents, const double* y, uint64_t n, uint64_t seed,
                           double* w_out, double* pi_out, double* sigma2_out);
int prsp_bsc_standard_init(uint32_t dim, uint32_t latents, uint32_t hprime, const double* y, uint64_t n,
                           uint64_t seed, double* w_out, double* pi_out, double* sigma2_out);

/* ---- max causes ----------------------------------
 * MaxCausesModel (max_causes.cpp): mca (max) / mmca (absmax) superposition.
 *   prsp_mca_gpu_create      MaxCausesModel ctor (max_causes.cpp:83-99); model "mca" | "mmca",
 *                            soft_winner_rho >= 0 (mca only)
 *   prsp_mca_gpu_step        MaxCausesModel::step (:416-446): E pass, fixed-point M-step,
 *                            residual pass for sigma2; *free_energy at the incoming params
 *   prsp_mca_gpu_estep       MaxCausesModel::estep_stats (:384-391) over the resident shard;
 *                            stats [winner_num D·H | winner_den D·H | sum_act | log_partition | points]
 *   prsp_mca_gpu_mstep_fixedpoint  MaxCausesModel::mstep_fixedpoint (:393-414) from the device stats
 *   prsp_mca_gpu_residual_commit   the residual pass of step (:423-436) and the update of W, pi, sigma2
 *   prsp_mca_gpu_inference / _candidates   inference (:448-468) / selection as estep_impl (:205-207)
 */
typedef struct prsp_mca_gpu prsp_mca_gpu;
int prsp_mca_gpu_create(const char* model, double soft_winner_rho, uint32_t dim, uint32_t latents, uint32_t hprime,
                        uint32_t gamma, uint64_t state_cap, int device, prsp_mca_gpu** out);
void prsp_mca_gpu_free(prsp_mca_gpu* ctx);
int prsp_mca_gpu_states_per_point(const prsp_mca_gpu* ctx, uint64_t* out);
int prsp_mca_gpu_load_data(prsp_mca_gpu* ctx, const double* y_host, uint64_t n);
int prsp_mca_gpu_set_params(prsp_mca_gpu* ctx, const double* w, double pi, double sigma2);
int prsp_mca_gpu_get_params(prsp_mca_gpu* ctx, double* w, double* pi, double* sigma2);
int prsp_mca_gpu_step(prsp_mca_gpu* ctx, double temperature, double* free_energy);
int prsp_mca_gpu_estep(prsp_mca_gpu* ctx, double temperature);
int prsp_mca_gpu_stats_buffer(prsp_mca_gpu* ctx, double** device_ptr, uint64_t* count);
int prsp_mca_gpu_get_stats(prsp_mca_gpu* ctx, double* winner_num, double* winner_den, double* scalars);
int prsp_mca_gpu_set_stats(prsp_mca_gpu* ctx, const double* winner_num, const double* winner_den,
                           const double* scalars);
int prsp_mca_gpu_mstep_fixedpoint(prsp_mca_gpu* ctx, double* w_out, double* pi_out);
int prsp_mca_gpu_residual_commit(prsp_mca_gpu* ctx, double temperature, double* residual_out);
/* Multi-rank σ²: after summing residual_out across ranks, σ² = max(Σ/(N·D), 1e-12) (:431-436). */
int prsp_mca_gpu_set_sigma2(prsp_mca_gpu* ctx, double sigma2);
int prsp_mca_gpu_candidates(prsp_mca_gpu* ctx, uint32_t* out);
int prsp_mca_gpu_inference(prsp_mca_gpu* ctx, double* map_states, double* map_mass, double* expected);

/* ---- run I/O and the training driver ----------------
 *   prsp_gpu_array_save / _load   save_array / load_array, PRSPAR01 (array_io.cpp:53-95);
 *                                 prsp_matrix_save / prsp_matrix_load (prsp.h:71-72)
 *   prsp_gpu_dataset_load         load_dataset: PRSPAR01 by magic, else headerless CSV
 *                                 (array_io.cpp:97-153); prsp_dataset_load (prsp.h:60)
 *   prsp_gpu_sha256[_file]        sha256_hex / sha256_hex_file (sha256.hpp), the manifest data hash
 *   prsp_gpu_format_double        format_double (array_io.cpp:159-164)
 *   prsp_gpu_train                train_run (run_io.cpp:196-230) + run (em.cpp:27-77) with every EM
 *                                 step on the GPU; out_dir (nullable) receives free_energy.csv,
 *                                 checkpoint_*.prsp (cadence of run_io.cpp:150-151), final_*.prsp and
 *                                 manifest.json (prsp-manifest-1); prsp_train (prsp.h:117-118)
 *   prsp_gpu_result_*             prsp_result_iterations / _trace / _param (prsp.h:120-127)
 *   prsp_gpu_run_open / _infer    load_run (run_io.cpp:165-194) / prsp_infer (capi.cpp:389-407)
 * Array loads are two-call: with out == NULL only the shape is returned.
 * Schedules are piecewise linear over the fraction of the iteration budget
 * (annealing.cpp); NULL / 0 anchors mean constant T = 1 and no weight noise. */
typedef struct {
  const char* model; /* "bsc" | "tsc" | "dsc" | "mca" | "mmca" */
  uint32_t latents, hprime, gamma; /* hprime 0 → latents, gamma 0 → hprime */
  const double* values; /* dsc alphabet */
  uint32_t n_values;
  uint64_t iterations, seed;
  uint32_t workers, shards; /* recorded in the manifest */
  int has_tolerance;
  double tolerance;
  const double* temperature_pos;
  const double* temperature_val;
  uint32_t n_temperature;
  const double* w_noise_pos;
  const double* w_noise_val;
  uint32_t n_w_noise;
  double soft_winner_rho; /* mca */
  int device;
} prsp_gpu_train_config;
typedef struct prsp_gpu_result prsp_gpu_result;
typedef struct prsp_gpu_run prsp_gpu_run;

int prsp_gpu_array_save(const char* path, const double* data, uint64_t rows, uint64_t cols);
int prsp_gpu_array_load(const char* path, uint64_t* rows, uint64_t* cols, double* out);
int prsp_gpu_dataset_load(const char* path, uint64_t* rows, uint64_t* cols, double* out);
int prsp_gpu_sha256(const void* data, uint64_t bytes, char* hex65);
int prsp_gpu_sha256_file(const char* path, char* hex65);
int prsp_gpu_format_double(double v, char* out, uint32_t capacity);
int prsp_gpu_train(const prsp_gpu_train_config* config, const double* y, uint64_t n, uint64_t d,
                   const char* data_file, const char* out_dir, prsp_gpu_result** out);
int prsp_gpu_result_iterations(const prsp_gpu_result* r, uint64_t* out);
int prsp_gpu_result_trace(const prsp_gpu_result* r, double* free_energy);
int prsp_gpu_result_param(const prsp_gpu_result* r, const char* name, uint64_t* rows, uint64_t* cols, double* out);
void prsp_gpu_result_free(prsp_gpu_result* r);
int prsp_gpu_run_open(const char* dir, prsp_gpu_run** out);
int prsp_gpu_run_info(const prsp_gpu_run* run, char* model, uint32_t capacity, uint32_t* dim, uint32_t* latents);
int prsp_gpu_run_param(const prsp_gpu_run* run, const char* name, uint64_t* rows, uint64_t* cols, double* out);
int prsp_gpu_run_infer(const prsp_gpu_run* run, const double* y, uint64_t n, uint64_t d, int device,
                       double* map_states, double* map_mass, double* expected);
void prsp_gpu_run_free(prsp_gpu_run* run);

#ifdef __cplusplus
}
#endif

#endif /* PRSP_BSC_GPU_H */
