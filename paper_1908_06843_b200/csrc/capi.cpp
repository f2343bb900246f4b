// C ABI (include/prsp_bsc_gpu.h) over BscEngine and the fixtures. Exceptions
// map to prsp_status codes as the reference's `guarded` does
// (/root/reference/proj/src/capi.cpp:63-82); outputs are written only on success.
#include "prsp_bsc_gpu.h"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "bsc_engine.hpp"
#include "fixtures.hpp"
#include "mca_engine.hpp"
#include "nccl_link.hpp"
#include "run_io.hpp"

struct prsp_bsc_gpu {
  bscgpu::BscEngine engine;
  bscgpu::nccl::Comm comm = nullptr;  // the statistics all-reduce across ranks
  bool own_comm = false;
  ~prsp_bsc_gpu() {
    if (comm && own_comm) bscgpu::nccl::api().comm_destroy(comm);
  }
  prsp_bsc_gpu(uint32_t d, uint32_t h, uint32_t hp, uint32_t g, uint64_t cap, int dev) : engine(d, h, hp, g, cap, dev) {}
  prsp_bsc_gpu(int fam, uint32_t d, uint32_t h, uint32_t hp, uint32_t g, uint64_t cap, const double* vals, uint32_t nv,
               int dev)
      : engine(fam, d, h, hp, g, cap, vals, nv, dev) {}
};

struct prsp_mca_gpu {
  bscgpu::McaEngine engine;
  prsp_mca_gpu(int mode, double rho, uint32_t d, uint32_t h, uint32_t hp, uint32_t g, uint64_t cap, int dev)
      : engine(mode, rho, d, h, hp, g, cap, dev) {}
};

struct prsp_gpu_result {
  bscgpu::TrainResult r;
};
struct prsp_gpu_run {
  bscgpu::TrainedRun run;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const bscgpu::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return bscgpu::kInternal;
  } catch (const std::exception& e) {
    g_err = e.what();
    return bscgpu::kInternal;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw bscgpu::Error(bscgpu::kConfig, std::string("null argument: ") + what);
}

}  // namespace

extern "C" {

const char* prsp_bsc_gpu_version(void) { return "0.1.0-b200"; }
const char* prsp_bsc_gpu_last_error(void) { return g_err.c_str(); }

int prsp_bsc_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int prsp_bsc_gpu_create(uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma, uint64_t state_cap,
                        int device, prsp_bsc_gpu** out) {
  return guarded([&] {
    need(out, "out");
    *out = new prsp_bsc_gpu(dim, latents, hprime, gamma, state_cap, device);
  });
}

int prsp_bsc_gpu_create_model(const char* model, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma,
                              uint64_t state_cap, const double* values, uint32_t n_values, int device,
                              prsp_bsc_gpu** out) {
  return guarded([&] {
    need(out, "out");
    need(model, "model");
    const std::string m(model);
    int fam = -1;
    if (m == "bsc") fam = bscgpu::kBsc;
    if (m == "tsc") fam = bscgpu::kTsc;
    if (m == "dsc") fam = bscgpu::kDsc;
    if (fam < 0) throw bscgpu::Error(bscgpu::kConfig, "unknown model '" + m + "' (gpu: bsc, tsc, dsc)");
    *out = new prsp_bsc_gpu(fam, dim, latents, hprime, gamma, state_cap, values, n_values, device);
  });
}

int prsp_bsc_gpu_model_info(const prsp_bsc_gpu* ctx, int* family, uint32_t* n_values, uint32_t* alphabet_size,
                            double* alphabet_out) {
  return guarded([&] {
    need(ctx, "ctx");
    const auto& e = ctx->engine;
    if (family) *family = e.family();
    if (n_values) *n_values = e.num_values();
    if (alphabet_size) *alphabet_size = e.alphabet_size();
    if (alphabet_out) std::memcpy(alphabet_out, e.alphabet().data(), e.alphabet().size() * sizeof(double));
  });
}

void prsp_bsc_gpu_free(prsp_bsc_gpu* ctx) { delete ctx; }

int prsp_bsc_gpu_set_stream(prsp_bsc_gpu* ctx, void* stream) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.set_stream(stream);
  });
}

int prsp_bsc_gpu_sync(prsp_bsc_gpu* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.sync();
  });
}

int prsp_bsc_gpu_states_per_point(const prsp_bsc_gpu* ctx, uint64_t* out) {
  return guarded([&] {
    need(ctx, "ctx");
    *out = ctx->engine.states_per_point();
  });
}

int prsp_bsc_gpu_load_data(prsp_bsc_gpu* ctx, const double* y, uint64_t n) {
  return guarded([&] {
    need(ctx, "ctx");
    need(y, "y");
    ctx->engine.load_data(y, n, false);
    ctx->engine.sync();
  });
}

int prsp_bsc_gpu_load_data_device(prsp_bsc_gpu* ctx, const double* y, uint64_t n) {
  return guarded([&] {
    need(ctx, "ctx");
    need(y, "y");
    ctx->engine.load_data(y, n, true);
  });
}

int prsp_bsc_gpu_set_params(prsp_bsc_gpu* ctx, const double* w, double pi, double sigma2) {
  return guarded([&] {
    need(ctx, "ctx");
    need(w, "w");
    ctx->engine.set_params(w, pi, sigma2);
    ctx->engine.sync();
  });
}

int prsp_bsc_gpu_set_params_ex(prsp_bsc_gpu* ctx, const double* w, double pi, double sigma2, const double* probs,
                               uint32_t n_probs) {
  return guarded([&] {
    need(ctx, "ctx");
    need(w, "w");
    ctx->engine.set_params_ex(w, pi, sigma2, probs, n_probs);
    ctx->engine.sync();
  });
}

int prsp_bsc_gpu_get_params_ex(prsp_bsc_gpu* ctx, double* w, double* pi, double* sigma2, double* probs) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.get_params_ex(w, pi, sigma2, probs);
  });
}

int prsp_bsc_gpu_get_params(prsp_bsc_gpu* ctx, double* w, double* pi, double* sigma2) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.get_params(w, pi, sigma2);
  });
}

int prsp_bsc_gpu_estep(prsp_bsc_gpu* ctx, double temperature) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.estep(temperature);
  });
}

int prsp_bsc_gpu_stats_buffer(prsp_bsc_gpu* ctx, double** ptr, uint64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    *ptr = ctx->engine.stats_device();
    *count = static_cast<uint64_t>(ctx->engine.layout().count());
  });
}

int prsp_bsc_gpu_get_stats(prsp_bsc_gpu* ctx, double* sum_s, double* sum_ssT, double* sum_y_sT,
                           double* value_counts, double* scalars) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.get_stats(sum_s, sum_ssT, sum_y_sT, value_counts, scalars);
  });
}

int prsp_bsc_gpu_set_stats(prsp_bsc_gpu* ctx, const double* sum_s, const double* sum_ssT, const double* sum_y_sT,
                           const double* value_counts, const double* scalars) {
  return guarded([&] {
    need(ctx, "ctx");
    need(sum_s, "sum_s");
    need(sum_ssT, "sum_ssT");
    need(sum_y_sT, "sum_y_sT");
    need(value_counts, "value_counts");
    need(scalars, "scalars");
    ctx->engine.set_stats(sum_s, sum_ssT, sum_y_sT, value_counts, scalars);
  });
}

int prsp_bsc_gpu_mstep(prsp_bsc_gpu* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.mstep();
  });
}

int prsp_bsc_gpu_step(prsp_bsc_gpu* ctx, double temperature, double* free_energy) {
  return guarded([&] {
    need(ctx, "ctx");
    const double f = ctx->engine.step(temperature);
    if (free_energy) *free_energy = f;
  });
}

int prsp_bsc_gpu_nccl_unique_id(char* id128) {
  return guarded([&] {
    need(id128, "id");
    bscgpu::nccl::UniqueId id;
    bscgpu::nccl::check(bscgpu::nccl::need().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id128, id.internal, sizeof id.internal);
  });
}

int prsp_bsc_gpu_nccl_init(prsp_bsc_gpu* ctx, const char* id128, int nranks, int rank) {
  return guarded([&] {
    need(ctx, "ctx");
    need(id128, "id");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw bscgpu::Error(bscgpu::kConfig, "nccl: bad rank / nranks");
    const auto& api = bscgpu::nccl::need();
    bscgpu::nccl::UniqueId id;
    std::memcpy(id.internal, id128, sizeof id.internal);
    if (cudaSetDevice(ctx->engine.device()) != cudaSuccess) throw bscgpu::Error(bscgpu::kInternal, "cuda: set device");
    bscgpu::nccl::Comm comm = nullptr;
    bscgpu::nccl::check(api.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
    if (ctx->comm && ctx->own_comm) api.comm_destroy(ctx->comm);
    ctx->comm = comm;
    ctx->own_comm = true;
  });
}

int prsp_bsc_gpu_nccl_attach(prsp_bsc_gpu* ctx, void* nccl_comm) {
  return guarded([&] {
    need(ctx, "ctx");
    need(nccl_comm, "comm");
    bscgpu::nccl::need();
    if (ctx->comm && ctx->own_comm) bscgpu::nccl::api().comm_destroy(ctx->comm);
    ctx->comm = nccl_comm;
    ctx->own_comm = false;
  });
}

int prsp_bsc_gpu_step_allreduce(prsp_bsc_gpu* ctx, double temperature, double* free_energy) {
  return guarded([&] {
    need(ctx, "ctx");
    if (!ctx->comm) throw bscgpu::Error(bscgpu::kConfig, "nccl: no communicator (prsp_bsc_gpu_nccl_init / _attach)");
    auto& e = ctx->engine;
    e.estep(temperature);
    // the packed statistics, summed in place over the ranks on the engine's stream:
    // the M-step (replicated, deterministic) then reads the global sums
    bscgpu::nccl::check(bscgpu::nccl::need().all_reduce(e.stats_device(), e.stats_device(), e.layout().count(),
                                                        bscgpu::nccl::kFloat64, bscgpu::nccl::kSum, ctx->comm,
                                                        static_cast<cudaStream_t>(e.stream())),
                        "ncclAllReduce");
    e.mstep();
    if (free_energy) *free_energy = e.last_free_energy();
  });
}

int prsp_bsc_gpu_free_energy(prsp_bsc_gpu* ctx, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    *out = ctx->engine.last_free_energy();
  });
}

int prsp_bsc_gpu_step_host(prsp_bsc_gpu* ctx, const double* y, uint64_t n, const double* w, double pi,
                           double sigma2, double temperature, double* w_out, double* pi_out, double* sigma2_out,
                           double* free_energy) {
  return guarded([&] {
    need(ctx, "ctx");
    need(y, "y");
    need(w, "w");
    auto& e = ctx->engine;
    e.set_params(w, pi, sigma2);
    // ~8 chunks of ≥ 16k points: the H2D copy of chunk c+1 overlaps chunk c
    // (BSC_HOST_CHUNK overrides the chunk size in points, for tuning)
    uint64_t chunk = std::max<uint64_t>(16384, (n + 7) / 8);
    if (const char* v = std::getenv("BSC_HOST_CHUNK")) chunk = std::max<uint64_t>(128, std::strtoull(v, nullptr, 10));
    const double f = e.step_streamed(y, n, temperature, chunk);
    double p = 0, s2 = 0;
    e.get_params(w_out, &p, &s2);
    if (pi_out) *pi_out = p;
    if (sigma2_out) *sigma2_out = s2;
    if (free_energy) *free_energy = f;
  });
}

int prsp_bsc_gpu_candidates(prsp_bsc_gpu* ctx, uint32_t* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    ctx->engine.estep(1.0, true);
    ctx->engine.sync();
    ctx->engine.get_candidates(out);
  });
}

int prsp_bsc_gpu_inference(prsp_bsc_gpu* ctx, double* map_states, double* map_mass, double* expected) {
  return guarded([&] {
    need(ctx, "ctx");
    need(map_states, "map_states");
    need(map_mass, "map_mass");
    need(expected, "expected");
    ctx->engine.inference(map_states, map_mass, expected);
  });
}

int prsp_bsc_gpu_set_timing(prsp_bsc_gpu* ctx, int on) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.set_timing(on != 0);
  });
}

int prsp_bsc_gpu_timings(prsp_bsc_gpu* ctx, float* out6) {
  return guarded([&] {
    need(ctx, "ctx");
    const auto& t = ctx->engine.timings();
    const float v[6] = {t.gram_ms, t.gemm1_ms, t.enum_ms, t.gemm2_ms, t.finalize_ms, t.mstep_ms};
    std::memcpy(out6, v, sizeof v);
  });
}

int prsp_bsc_gpu_timings_ex(prsp_bsc_gpu* ctx, float* out, int n) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    const auto& t = ctx->engine.timings();
    const float v[10] = {t.gram_ms,  t.gemm1_ms,  t.enum_ms,     t.gemm2_ms,   t.finalize_ms,
                         t.mstep_ms, t.front_ms,  t.states_ms,   t.fallback_ms, t.finish_ms};
    std::memcpy(out, v, sizeof(float) * static_cast<size_t>(std::max(0, std::min(n, 10))));
  });
}

int prsp_bsc_gpu_launches(prsp_bsc_gpu* ctx, int* out) {
  return guarded([&] {
    need(ctx, "ctx");
    *out = ctx->engine.kernel_launches_last_step();
  });
}

int prsp_bsc_gpu_guard_probe(int64_t bytes, int64_t index) {
  return guarded([&] { bscgpu::guard_probe(bytes, index); });
}

int prsp_bsc_gpu_check_guards(void) {
  return guarded([&] { bscgpu::check_device_guards(); });
}

int prsp_bsc_gpu_enum_phase_cycles(prsp_bsc_gpu* ctx, uint64_t* out8) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out8, "out8");
    unsigned long long v[8];
    ctx->engine.enum_phase_cycles(v);
    for (int i = 0; i < 8; ++i) out8[i] = v[i];
  });
}

int prsp_bsc_bars_generate(uint32_t size, uint64_t n, double prob, double amplitude, double noise, int max_mode,
                           uint64_t seed, double* y_out, double* truth_out) {
  return guarded([&] {
    need(y_out, "y_out");
    bscgpu::bars_generate(size, n, prob, amplitude, noise, max_mode != 0, seed, y_out, truth_out);
  });
}

int prsp_bsc_generate(uint32_t dim, uint32_t latents, const double* w, double pi, double sigma2, uint64_t n,
                      uint64_t seed, double* y_out) {
  return guarded([&] {
    need(w, "w");
    need(y_out, "y_out");
    bscgpu::generate(dim, latents, w, pi, sigma2, n, seed, y_out);
  });
}

int prsp_bsc_random_dictionary(uint32_t dim, uint32_t latents, uint64_t seed, double scale, double* w_out) {
  return guarded([&] {
    need(w_out, "w_out");
    bscgpu::random_dictionary(dim, latents, seed, scale, w_out);
  });
}

int prsp_bsc_baseline_init(uint32_t dim, uint32_t latents, const double* y, uint64_t n, uint64_t seed,
                           double* w_out, double* pi_out, double* sigma2_out) {
  return guarded([&] {
    need(y, "y");
    bscgpu::baseline_init(dim, latents, y, n, seed, w_out, pi_out, sigma2_out);
  });
}

int prsp_bsc_standard_init(uint32_t dim, uint32_t latents, uint32_t hprime, const double* y, uint64_t n,
                           uint64_t seed, double* w_out, double* pi_out, double* sigma2_out) {
  return guarded([&] {
    need(y, "y");
    bscgpu::standard_init(dim, latents, hprime, y, n, seed, w_out, pi_out, sigma2_out);
  });
}

int prsp_mca_gpu_create(const char* model, double rho, uint32_t dim, uint32_t latents, uint32_t hprime, uint32_t gamma,
                        uint64_t state_cap, int device, prsp_mca_gpu** out) {
  return guarded([&] {
    need(out, "out");
    need(model, "model");
    const std::string m(model);
    if (m != "mca" && m != "mmca") throw bscgpu::Error(bscgpu::kConfig, "unknown model '" + m + "' (mca, mmca)");
    *out = new prsp_mca_gpu(m == "mca" ? 0 : 1, rho, dim, latents, hprime, gamma, state_cap, device);
  });
}

void prsp_mca_gpu_free(prsp_mca_gpu* ctx) { delete ctx; }

int prsp_mca_gpu_states_per_point(const prsp_mca_gpu* ctx, uint64_t* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    *out = ctx->engine.states_per_point();
  });
}

int prsp_mca_gpu_load_data(prsp_mca_gpu* ctx, const double* y, uint64_t n) {
  return guarded([&] {
    need(ctx, "ctx");
    need(y, "y");
    ctx->engine.load_data(y, n);
  });
}

int prsp_mca_gpu_set_params(prsp_mca_gpu* ctx, const double* w, double pi, double sigma2) {
  return guarded([&] {
    need(ctx, "ctx");
    need(w, "w");
    ctx->engine.set_params(w, pi, sigma2);
  });
}

int prsp_mca_gpu_get_params(prsp_mca_gpu* ctx, double* w, double* pi, double* sigma2) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.get_params(w, pi, sigma2);
  });
}

int prsp_mca_gpu_step(prsp_mca_gpu* ctx, double temperature, double* free_energy) {
  return guarded([&] {
    need(ctx, "ctx");
    const double f = ctx->engine.step(temperature);
    if (free_energy) *free_energy = f;
  });
}

int prsp_mca_gpu_estep(prsp_mca_gpu* ctx, double temperature) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.estep(temperature);
  });
}

int prsp_mca_gpu_stats_buffer(prsp_mca_gpu* ctx, double** ptr, uint64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    *ptr = ctx->engine.stats_device();
    *count = ctx->engine.stats_count();
  });
}

int prsp_mca_gpu_get_stats(prsp_mca_gpu* ctx, double* num, double* den, double* scalars) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.get_stats(num, den, scalars);
  });
}

int prsp_mca_gpu_set_stats(prsp_mca_gpu* ctx, const double* num, const double* den, const double* scalars) {
  return guarded([&] {
    need(ctx, "ctx");
    need(num, "winner_num");
    need(den, "winner_den");
    need(scalars, "scalars");
    ctx->engine.set_stats(num, den, scalars);
  });
}

int prsp_mca_gpu_mstep_fixedpoint(prsp_mca_gpu* ctx, double* w_out, double* pi_out) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.mstep_fixedpoint();
    ctx->engine.get_updated(w_out, pi_out);
  });
}

int prsp_mca_gpu_residual_commit(prsp_mca_gpu* ctx, double temperature, double* residual_out) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.residual_and_commit(temperature);
    if (residual_out) *residual_out = ctx->engine.residual_device_sum();
  });
}

int prsp_mca_gpu_set_sigma2(prsp_mca_gpu* ctx, double sigma2) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->engine.set_sigma2(sigma2);
  });
}

int prsp_mca_gpu_candidates(prsp_mca_gpu* ctx, uint32_t* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    ctx->engine.candidates(out);
  });
}

int prsp_mca_gpu_inference(prsp_mca_gpu* ctx, double* map_states, double* map_mass, double* expected) {
  return guarded([&] {
    need(ctx, "ctx");
    need(map_states, "map_states");
    need(map_mass, "map_mass");
    need(expected, "expected");
    ctx->engine.inference(map_states, map_mass, expected);
  });
}

int prsp_gpu_array_save(const char* path, const double* data, uint64_t rows, uint64_t cols) {
  return guarded([&] {
    need(path, "path");
    if (rows * cols) need(data, "data");
    bscgpu::save_array(path, data, rows, cols);
  });
}

static int load_into(const bscgpu::Array& a, uint64_t* rows, uint64_t* cols, double* out) {
  if (rows) *rows = a.rows;
  if (cols) *cols = a.cols;
  if (out && !a.data.empty()) std::memcpy(out, a.data.data(), a.data.size() * sizeof(double));
  return 0;
}

int prsp_gpu_array_load(const char* path, uint64_t* rows, uint64_t* cols, double* out) {
  return guarded([&] {
    need(path, "path");
    load_into(bscgpu::load_array(path), rows, cols, out);
  });
}

int prsp_gpu_dataset_load(const char* path, uint64_t* rows, uint64_t* cols, double* out) {
  return guarded([&] {
    need(path, "path");
    load_into(bscgpu::load_dataset(path), rows, cols, out);
  });
}

int prsp_gpu_sha256(const void* data, uint64_t bytes, char* hex65) {
  return guarded([&] {
    need(hex65, "hex65");
    if (bytes) need(data, "data");
    std::memcpy(hex65, bscgpu::sha256_hex(data, bytes).c_str(), 65);
  });
}

int prsp_gpu_sha256_file(const char* path, char* hex65) {
  return guarded([&] {
    need(path, "path");
    need(hex65, "hex65");
    std::memcpy(hex65, bscgpu::sha256_hex_file(path).c_str(), 65);
  });
}

int prsp_gpu_format_double(double v, char* out, uint32_t capacity) {
  return guarded([&] {
    need(out, "out");
    const std::string s = bscgpu::format_double(v);
    if (s.size() + 1 > capacity) throw bscgpu::Error(bscgpu::kConfig, "format_double: buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

int prsp_gpu_train(const prsp_gpu_train_config* c, const double* y, uint64_t n, uint64_t d, const char* data_file,
                   const char* out_dir, prsp_gpu_result** out) {
  return guarded([&] {
    need(c, "config");
    need(c->model, "model");
    need(y, "y");
    need(out, "out");
    bscgpu::RunConfig rc;
    rc.model = c->model;
    rc.latents = c->latents;
    rc.hprime = c->hprime;
    rc.gamma = c->gamma;
    if (c->values && c->n_values) rc.values.assign(c->values, c->values + c->n_values);
    rc.iterations = c->iterations;
    rc.seed = c->seed;
    rc.workers = c->workers;
    rc.shards = c->shards;
    if (c->has_tolerance) rc.tolerance = c->tolerance;
    auto sched = [](const double* pos, const double* val, uint32_t k, double dflt) {
      bscgpu::Schedule s;
      if (!pos || !val || k == 0) {
        s.anchors = {{0.0, dflt}};
      } else {
        for (uint32_t i = 0; i < k; ++i) s.anchors.emplace_back(pos[i], val[i]);
      }
      return s;
    };
    rc.temperature = sched(c->temperature_pos, c->temperature_val, c->n_temperature, 1.0);
    rc.w_noise = sched(c->w_noise_pos, c->w_noise_val, c->n_w_noise, 0.0);
    rc.soft_winner_rho = c->soft_winner_rho;
    rc.device = c->device;
    auto* r = new prsp_gpu_result{bscgpu::train_run(rc, y, n, d, data_file ? data_file : "", out_dir ? out_dir : "")};
    *out = r;
  });
}

int prsp_gpu_result_iterations(const prsp_gpu_result* r, uint64_t* out) {
  return guarded([&] {
    need(r, "result");
    need(out, "out");
    *out = r->r.trace.size();
  });
}

int prsp_gpu_result_trace(const prsp_gpu_result* r, double* f) {
  return guarded([&] {
    need(r, "result");
    need(f, "free_energy");
    std::memcpy(f, r->r.trace.data(), r->r.trace.size() * sizeof(double));
  });
}

static const bscgpu::Array& named(const std::vector<bscgpu::NamedArray>& v, const char* name) {
  for (const auto& p : v)
    if (p.name == name) return p.a;
  throw bscgpu::Error(bscgpu::kConfig, std::string("no parameter array named ") + name);
}

int prsp_gpu_result_param(const prsp_gpu_result* r, const char* name, uint64_t* rows, uint64_t* cols, double* out) {
  return guarded([&] {
    need(r, "result");
    need(name, "name");
    load_into(named(r->r.params, name), rows, cols, out);
  });
}

void prsp_gpu_result_free(prsp_gpu_result* r) { delete r; }

int prsp_gpu_run_open(const char* dir, prsp_gpu_run** out) {
  return guarded([&] {
    need(dir, "dir");
    need(out, "out");
    *out = new prsp_gpu_run{bscgpu::load_run(dir)};
  });
}

int prsp_gpu_run_info(const prsp_gpu_run* run, char* model, uint32_t capacity, uint32_t* dim, uint32_t* latents) {
  return guarded([&] {
    need(run, "run");
    const auto& c = run->run.config;
    if (model) {
      if (c.model.size() + 1 > capacity) throw bscgpu::Error(bscgpu::kConfig, "run_info: buffer too small");
      std::memcpy(model, c.model.c_str(), c.model.size() + 1);
    }
    if (dim) *dim = c.dim;
    if (latents) *latents = c.latents;
  });
}

int prsp_gpu_run_param(const prsp_gpu_run* run, const char* name, uint64_t* rows, uint64_t* cols, double* out) {
  return guarded([&] {
    need(run, "run");
    need(name, "name");
    load_into(named(run->run.params, name), rows, cols, out);
  });
}

int prsp_gpu_run_infer(const prsp_gpu_run* run, const double* y, uint64_t n, uint64_t d, int device,
                       double* map_states, double* map_mass, double* expected) {
  return guarded([&] {
    need(run, "run");
    need(y, "y");
    need(map_states, "map_states");
    need(map_mass, "map_mass");
    bscgpu::infer_run(run->run, y, n, d, map_states, map_mass, expected, device);
  });
}

void prsp_gpu_run_free(prsp_gpu_run* run) { delete run; }

}  // extern "C"
