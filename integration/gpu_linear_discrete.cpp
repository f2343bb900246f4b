// The drop-in, compiled: a prsp::Model whose step() runs on the B200 engine
// through the C ABI (include/prsp_bsc_gpu.h), built against the reference's
// unmodified headers (/root/reference/proj/src) and driven by the reference's
// own EM loop prsp::run (em.cpp:22-70). This is the binding INTEGRATION.md §1
// shows a maintainer adding inside LinearDiscreteModel; as LinearDiscreteModel
// is `final`, the adapter here wraps one and forwards everything but step().
//
// TEST INFRASTRUCTURE: built by integration/Makefile into _build/libprsp_dropin.so
// (linked with the oracle/_ref build of the reference sources and the engine
// library) and called from tests/test_gpu_dropin.py.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "em.hpp"
#include "linear_discrete.hpp"
#include "prsp_bsc_gpu.h"

namespace {

using namespace prsp;

// prsp_status → the reference's exception taxonomy (core.hpp:32-43)
void ok(int rc) {
  if (rc == PRSP_BSC_GPU_OK) return;
  const std::string m = prsp_bsc_gpu_last_error();
  if (rc == PRSP_BSC_GPU_ERR_CONFIG) throw ConfigError(m);
  if (rc == PRSP_BSC_GPU_ERR_DATA) throw DataError(m);
  if (rc == PRSP_BSC_GPU_ERR_NUMERIC) throw NumericError(m);
  throw Error(m);
}

class GpuLinearDiscreteModel final : public Model {
 public:
  GpuLinearDiscreteModel(DiscreteFamily family, std::uint32_t dim, std::uint32_t latents, TruncationConfig trunc,
                         std::vector<double> dsc_values = {})
      : cpu_(family, dim, latents, trunc, dsc_values), trunc_(trunc), values_(std::move(dsc_values)) {}
  ~GpuLinearDiscreteModel() override {
    if (gpu_) prsp_bsc_gpu_free(gpu_);
  }

  const std::string& name() const override { return cpu_.name(); }
  std::uint32_t dim() const override { return cpu_.dim(); }
  std::uint32_t latents() const override { return cpu_.latents(); }
  void validate(const ModelParams& p, const DataSet* d) const override { cpu_.validate(p, d); }
  ModelParams standard_init(const DataSet& d, RngStream& rng) const override { return cpu_.standard_init(d, rng); }
  InferenceResult inference(const ModelParams& p, const DataSet& d, const ShardPlan& plan) const override {
    return cpu_.inference(p, d, plan);
  }
  DataSet generate(const ModelParams& p, std::size_t n, RngStream& rng) const override {
    return cpu_.generate(p, n, rng);
  }
  double exact_log_likelihood(const ModelParams& p, const DataSet& d) const override {
    return cpu_.exact_log_likelihood(p, d);
  }
  void perturb_weights(ModelParams& p, double noise_std, RngStream& rng) const override {
    cpu_.perturb_weights(p, noise_std, rng);
  }

  // LinearDiscreteModel::step (linear_discrete.cpp:410-427) on the GPU: the data
  // are uploaded once and stay resident across EM iterations.
  StepResult step(const ModelParams& params, const AnnealState& anneal, const DataSet& data,
                  const ShardPlan& plan) const override {
    validate(params, &data);
    plan.validate(data.size());
    const auto& p = std::get<LinearDiscreteParams>(params);
    if (!gpu_) {
      const char* fam = cpu_.family() == DiscreteFamily::kBsc ? "bsc" : cpu_.family() == DiscreteFamily::kTsc ? "tsc" : "dsc";
      ok(prsp_bsc_gpu_create_model(fam, dim(), latents(), trunc_.hprime, trunc_.gamma, trunc_.state_cap,
                                   values_.empty() ? nullptr : values_.data(),
                                   static_cast<uint32_t>(values_.size()), /*device=*/0, &gpu_));
    }
    if (resident_ != data.y.data()) {
      ok(prsp_bsc_gpu_load_data(gpu_, data.y.data(), data.size()));
      resident_ = data.y.data();
    }
    ok(prsp_bsc_gpu_set_params_ex(gpu_, p.w.data(), p.pi, p.sigma2, p.probs.empty() ? nullptr : p.probs.data(),
                                  static_cast<uint32_t>(p.probs.size())));
    double f = 0.0;
    ok(prsp_bsc_gpu_step(gpu_, anneal.temperature, &f));
    LinearDiscreteParams out = p;
    ok(prsp_bsc_gpu_get_params_ex(gpu_, out.w.data(), &out.pi, &out.sigma2, out.probs.empty() ? nullptr : out.probs.data()));
    return StepResult{out, f};
  }

 private:
  LinearDiscreteModel cpu_;
  TruncationConfig trunc_;
  std::vector<double> values_;
  mutable prsp_bsc_gpu* gpu_ = nullptr;
  mutable const double* resident_ = nullptr;
};

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* dropin_last_error() { return g_err.c_str(); }

// prsp::run over a BSC model — the GPU adapter (gpu != 0) or the reference's own
// LinearDiscreteModel — from the given parameters, `iterations` EM steps at
// T = 1 (optionally annealed from t0 down to 1 by the reference's schedule),
// all shards on `shards` workers. Writes the free-energy trace and the final
// parameters.
int dropin_run_bsc(int gpu, const double* y, uint64_t n, uint32_t d, uint32_t h, uint32_t hprime, uint32_t gamma,
                   const double* w0, double pi0, double sigma2_0, uint32_t iterations, double t0, uint32_t shards,
                   double* trace, double* w_out, double* pi_out, double* sigma2_out) {
  try {
    const TruncationConfig tc{h, hprime, gamma, 1000000};
    std::unique_ptr<Model> model;
    if (gpu)
      model = std::make_unique<GpuLinearDiscreteModel>(DiscreteFamily::kBsc, d, h, tc);
    else
      model = std::make_unique<LinearDiscreteModel>(DiscreteFamily::kBsc, d, h, tc);
    DataSet data = DataSet::wrap(DenseMatrix(n, d, std::vector<double>(y, y + n * d)));
    LinearDiscreteParams p;
    p.w = DenseMatrix(d, h, std::vector<double>(w0, w0 + std::size_t(d) * h));
    p.pi = pi0;
    p.sigma2 = sigma2_0;
    LinearAnnealing anneal(iterations, t0 > 1.0 ? Schedule({{0.0, t0}, {0.5, 1.0}}) : Schedule::constant(1.0));
    const ShardPlan plan = ShardPlan::with_shards(n, shards, shards);
    TrainResult r = run(*model, ModelParams{p}, data, anneal, plan);
    std::memcpy(trace, r.free_energy_trace.data(), r.free_energy_trace.size() * sizeof(double));
    const auto& q = std::get<LinearDiscreteParams>(r.final_params);
    std::memcpy(w_out, q.w.data(), std::size_t(d) * h * sizeof(double));
    *pi_out = q.pi;
    *sigma2_out = q.sigma2;
    g_err.clear();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // extern "C"
