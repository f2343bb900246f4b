// TEST INFRASTRUCTURE ONLY (oracle/): the parity oracle, never the product.
//
// extern "C" entry points over the *unmodified* reference C++ classes
// (/root/reference/proj/src, compiled by oracle/Makefile against the
// clean-room Eigen subset in oracle/eigen_shim). Output: oracle/_ref/libprsp_ref.so.
// Used by tests/ to pin oracle/bsc_oracle.c and by bench.py's reference arm
// (cpu_baseline.kind = "reference").
//
// Status codes follow prsp_status (/root/reference/proj/include/prsp.h:39-45).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "array_io.hpp"
#include "bars.hpp"
#include "em.hpp"
#include "annealing.hpp"
#include "sha256.hpp"
#include "core.hpp"
#include "linear_discrete.hpp"
#include "max_causes.hpp"
#include "model.hpp"
#include "parallel.hpp"
#include "truncation.hpp"

using namespace prsp;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

DataSet wrap_data(const double* y, std::uint64_t n, std::uint32_t d) {
  return DataSet::wrap(DenseMatrix(n, d, std::vector<double>(y, y + n * d)));
}

LinearDiscreteParams bsc_params(std::uint32_t d, std::uint32_t h,
                                const double* w, double pi, double sigma2) {
  LinearDiscreteParams p;
  p.w = DenseMatrix(d, h, std::vector<double>(w, w + std::size_t(d) * h));
  p.pi = pi;
  p.sigma2 = sigma2;
  return p;
}

LinearDiscreteModel bsc_model(std::uint32_t d, std::uint32_t h,
                              std::uint32_t hprime, std::uint32_t gamma) {
  return LinearDiscreteModel(DiscreteFamily::kBsc, d, h,
                             TruncationConfig{h, hprime, gamma, 1000000});
}

DiscreteFamily fam_of(std::uint32_t f) {
  return f == 0 ? DiscreteFamily::kBsc : f == 1 ? DiscreteFamily::kTsc : DiscreteFamily::kDsc;
}

LinearDiscreteModel ld_model(std::uint32_t family, std::uint32_t d, std::uint32_t h,
                             std::uint32_t hprime, std::uint32_t gamma, const double* alpha,
                             std::uint32_t nalpha) {
  std::vector<double> vals;
  if (family == 2) vals.assign(alpha, alpha + nalpha);
  return LinearDiscreteModel(fam_of(family), d, h, TruncationConfig{h, hprime, gamma, 1000000},
                             vals);
}

LinearDiscreteParams ld_params(std::uint32_t family, std::uint32_t d, std::uint32_t h,
                               const double* w, double sigma2, double pi, const double* alpha,
                               const double* probs, std::uint32_t nalpha) {
  LinearDiscreteParams p = bsc_params(d, h, w, pi, sigma2);
  if (family == 2) {
    p.values.assign(alpha, alpha + nalpha);
    p.probs.assign(probs, probs + nalpha);
  }
  return p;
}

MaxCausesModel mca_model(std::uint32_t mode, std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                         std::uint32_t gamma, double rho) {
  return MaxCausesModel(mode == 0 ? MaxMode::kMax : MaxMode::kAbsMax, d, h,
                        TruncationConfig{h, hprime, gamma, 1000000}, rho);
}

McaParams mca_params(std::uint32_t d, std::uint32_t h, const double* w, double pi, double sigma2) {
  McaParams p;
  p.w = DenseMatrix(d, h, std::vector<double>(w, w + std::size_t(d) * h));
  p.pi = pi;
  p.sigma2 = sigma2;
  return p;
}

void copy_stats(const SuffStats& s, double* sum_s, double* sum_ssT,
                double* sum_y_sT, double* value_counts, double* scalars) {
  const auto put = [](const DenseMatrix& m, double* out) {
    if (out) std::memcpy(out, m.data(), m.size() * sizeof(double));
  };
  put(s.at("sum_s"), sum_s);
  put(s.at("sum_ssT"), sum_ssT);
  put(s.at("sum_y_sT"), sum_y_sT);
  put(s.at("value_counts"), value_counts);  // one entry per non-zero value
  if (scalars) {
    scalars[0] = s.scalar("sum_y2");
    scalars[1] = s.scalar("log_partition");
    scalars[2] = static_cast<double>(s.points);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_rng_normals(std::uint64_t base_seed, std::uint64_t index, int derived,
                    std::uint64_t n, double* out) {
  return guarded([&] {
    RngStream rng = derived ? RngStream::derived(base_seed, index)
                            : RngStream(base_seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.normal();
  });
}

int ref_make_bars(std::uint32_t size, std::uint64_t n, double prob,
                  double amplitude, double noise, int max_mode,
                  std::uint64_t seed, double* y_out, double* truth_out) {
  return guarded([&] {
    BarsSpec spec;
    spec.size = size;
    spec.n = n;
    spec.prob = prob;
    spec.amplitude = amplitude;
    spec.noise = noise;
    spec.max_mode = max_mode != 0;
    spec.seed = seed;
    BarsData b = make_bars(spec);
    std::memcpy(y_out, b.data.y.data(), b.data.y.size() * sizeof(double));
    if (truth_out)
      std::memcpy(truth_out, b.truth.data(), b.truth.size() * sizeof(double));
  });
}

int ref_generate(std::uint32_t d, std::uint32_t h, const double* w, double pi,
                 double sigma2, std::uint64_t n, std::uint64_t seed,
                 double* y_out) {
  return guarded([&] {
    auto m = bsc_model(d, h, h, 1);
    RngStream rng(seed);
    DataSet ds = m.generate(bsc_params(d, h, w, pi, sigma2), n, rng);
    std::memcpy(y_out, ds.y.data(), ds.y.size() * sizeof(double));
  });
}

int ref_select_candidates(const double* scores, std::uint32_t h,
                          std::uint32_t hprime, std::uint32_t* out) {
  return guarded([&] {
    auto c = select_candidates(std::span<const double>(scores, h), hprime);
    std::memcpy(out, c.data(), c.size() * sizeof(std::uint32_t));
  });
}

int ref_state_count(std::uint32_t h, std::uint32_t hprime, std::uint32_t gamma,
                    std::uint64_t* out) {
  return guarded([&] {
    TruncationConfig cfg{h, hprime, gamma, 1000000};
    cfg.validate();
    *out = truncated_state_count(cfg, 1);
  });
}

// Dense 0/1 state rows (count × h) in the reference enumeration order.
int ref_enumerate_binary(const std::uint32_t* cand, std::uint32_t hprime,
                         std::uint32_t h, std::uint32_t gamma, double* out,
                         std::uint64_t* count) {
  return guarded([&] {
    StateSet s = enumerate_binary_states(
        std::vector<std::uint32_t>(cand, cand + hprime), h, gamma);
    *count = s.states.size();
    if (out)
      for (std::size_t i = 0; i < s.states.size(); ++i) {
        auto dense = s.states[i].to_dense(h);
        std::memcpy(out + i * h, dense.data(), h * sizeof(double));
      }
  });
}

int ref_log_sum_exp(const double* v, std::uint64_t n, double* out) {
  return guarded([&] { *out = log_sum_exp(std::span<const double>(v, n)); });
}

int ref_log_joint(std::uint32_t d, std::uint32_t h, const double* w, double pi,
                  double sigma2, const double* y, const double* s, double* out) {
  return guarded([&] {
    auto m = bsc_model(d, h, h, 1);
    *out = m.log_joint(bsc_params(d, h, w, pi, sigma2),
                       std::span<const double>(y, d),
                       std::span<const double>(s, h));
  });
}

int ref_estep_stats(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                    std::uint32_t gamma, const double* w, double pi,
                    double sigma2, double temperature, const double* y,
                    std::uint64_t n, std::uint64_t row_begin,
                    std::uint64_t row_end, double* sum_s, double* sum_ssT,
                    double* sum_y_sT, double* value_counts, double* scalars) {
  return guarded([&] {
    auto m = bsc_model(d, h, hprime, gamma);
    DataSet ds = wrap_data(y, n, d);
    SuffStats s = m.estep_stats(bsc_params(d, h, w, pi, sigma2), ds,
                                RowRange{row_begin, row_end}, temperature);
    copy_stats(s, sum_s, sum_ssT, sum_y_sT, value_counts, scalars);
  });
}

// scalars = {sum_y2, log_partition, points}.
int ref_mstep(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
              std::uint32_t gamma, const double* w_prev, double pi_prev,
              double sigma2_prev, const double* sum_s, const double* sum_ssT,
              const double* sum_y_sT, const double* value_counts,
              const double* scalars, double* w_out, double* pi_out,
              double* sigma2_out) {
  return guarded([&] {
    auto m = bsc_model(d, h, hprime, gamma);
    SuffStats s;
    const auto fill = [&](const char* name, std::size_t r, std::size_t c,
                          const double* src) {
      DenseMatrix& f = s.field(name, r, c);
      std::memcpy(f.data(), src, r * c * sizeof(double));
    };
    fill("sum_s", 1, h, sum_s);
    fill("sum_ssT", h, h, sum_ssT);
    fill("sum_y_sT", d, h, sum_y_sT);
    fill("value_counts", 1, 1, value_counts);
    s.scalar("sum_y2") = scalars[0];
    s.scalar("log_partition") = scalars[1];
    s.points = static_cast<std::uint64_t>(scalars[2]);
    ModelParams out = m.mstep(s, bsc_params(d, h, w_prev, pi_prev, sigma2_prev));
    const auto& p = std::get<LinearDiscreteParams>(out);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    *pi_out = p.pi;
    *sigma2_out = p.sigma2;
  });
}

// One LinearDiscreteModel::step with ShardPlan::with_shards(n, shards, workers).
int ref_step(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
             std::uint32_t gamma, const double* w, double pi, double sigma2,
             double temperature, const double* y, std::uint64_t n,
             std::uint32_t shards, std::uint32_t workers, double* w_out,
             double* pi_out, double* sigma2_out, double* free_energy) {
  return guarded([&] {
    auto m = bsc_model(d, h, hprime, gamma);
    DataSet ds = wrap_data(y, n, d);
    ShardPlan plan = ShardPlan::with_shards(n, shards, workers);
    AnnealState st;
    st.temperature = temperature;
    StepResult r = m.step(bsc_params(d, h, w, pi, sigma2), st, ds, plan);
    const auto& p = std::get<LinearDiscreteParams>(r.params);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    *pi_out = p.pi;
    *sigma2_out = p.sigma2;
    *free_energy = r.free_energy;
  });
}

// A persistent dataset + model for timing many steps without re-copying Y.
struct RefSession {
  LinearDiscreteModel model;
  DataSet data;
};

int ref_session_create(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                       std::uint32_t gamma, const double* y, std::uint64_t n,
                       void** out) {
  return guarded([&] {
    *out = new RefSession{bsc_model(d, h, hprime, gamma), wrap_data(y, n, d)};
  });
}

void ref_session_free(void* s) { delete static_cast<RefSession*>(s); }

int ref_session_step(void* sp, const double* w, double pi, double sigma2,
                     std::uint32_t shards, std::uint32_t workers,
                     double* w_out, double* pi_out, double* sigma2_out,
                     double* free_energy) {
  return guarded([&] {
    auto* s = static_cast<RefSession*>(sp);
    const std::uint32_t d = s->model.dim(), h = s->model.latents();
    ShardPlan plan = ShardPlan::with_shards(s->data.size(), shards, workers);
    AnnealState st;
    StepResult r = s->model.step(bsc_params(d, h, w, pi, sigma2), st, s->data, plan);
    const auto& p = std::get<LinearDiscreteParams>(r.params);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    *pi_out = p.pi;
    *sigma2_out = p.sigma2;
    *free_energy = r.free_energy;
  });
}

// Per-point candidate sets, recomputed exactly as estep_impl does
// (linear_discrete.cpp:219-253: gram = W^T W, b = W^T y, score of :248-249,
// select_candidates). estep_impl is private, so the harness restates the
// selection with the same Eigen-shim operations.
int ref_candidates(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                   const double* w, double pi, double sigma2, const double* y,
                   std::uint64_t n, std::uint32_t* out) {
  return guarded([&] {
    const ConstMatView wv(w, d, h);
    const Eigen::MatrixXd gram = wv.transpose() * wv;
    const double inv2s = 1.0 / (2.0 * sigma2);
    const double lp = std::log(pi);
    std::vector<double> scores(h);
    Eigen::VectorXd b(h);
    for (std::uint64_t i = 0; i < n; ++i) {
      ConstVecView yv(y + i * d, d);
      b.noalias() = wv.transpose() * yv;
      for (std::uint32_t u = 0; u < h; ++u) {
        double best = -std::numeric_limits<double>::infinity();
        best = std::max(best, lp + (2.0 * 1.0 * b[u] - 1.0 * 1.0 * gram(u, u)) * inv2s);
        scores[u] = best;
      }
      auto c = select_candidates(scores, hprime);
      std::memcpy(out + i * hprime, c.data(), hprime * sizeof(std::uint32_t));
    }
  });
}

int ref_inference(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                  std::uint32_t gamma, const double* w, double pi, double sigma2,
                  const double* y, std::uint64_t n, std::uint32_t shards,
                  double* map_states, double* map_mass, double* expected) {
  return guarded([&] {
    auto m = bsc_model(d, h, hprime, gamma);
    DataSet ds = wrap_data(y, n, d);
    InferenceResult r = m.inference(bsc_params(d, h, w, pi, sigma2), ds,
                                    ShardPlan::with_shards(n, shards, shards));
    std::memcpy(map_states, r.map_states.data(), r.map_states.size() * sizeof(double));
    std::memcpy(map_mass, r.map_mass.data(), r.map_mass.size() * sizeof(double));
    std::memcpy(expected, r.expected_states.data(),
                r.expected_states.size() * sizeof(double));
  });
}

int ref_exact_log_likelihood(std::uint32_t d, std::uint32_t h, const double* w,
                             double pi, double sigma2, const double* y,
                             std::uint64_t n, double* out) {
  return guarded([&] {
    auto m = bsc_model(d, h, h, h);
    *out = m.exact_log_likelihood(bsc_params(d, h, w, pi, sigma2),
                                  wrap_data(y, n, d));
  });
}

int ref_standard_init(std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                      std::uint32_t gamma, const double* y, std::uint64_t n,
                      std::uint64_t seed, double* w_out, double* pi_out,
                      double* sigma2_out) {
  return guarded([&] {
    auto m = bsc_model(d, h, hprime, gamma);
    RngStream rng(seed);
    ModelParams p = m.standard_init(wrap_data(y, n, d), rng);
    const auto& lp = std::get<LinearDiscreteParams>(p);
    std::memcpy(w_out, lp.w.data(), lp.w.size() * sizeof(double));
    *pi_out = lp.pi;
    *sigma2_out = lp.sigma2;
  });
}

int ref_data_mean_variance(const double* y, std::uint64_t n, std::uint32_t d,
                           double* out) {
  return guarded([&] { *out = detail::data_mean_variance(wrap_data(y, n, d)); });
}

// ---- linear discrete families (bsc 0 / tsc 1 / dsc 2); the dsc alphabet
// (ascending, with 0) and probabilities are passed as alpha/probs/nalpha.
int ref_ld_estep_stats(std::uint32_t family, const double* alpha, const double* probs,
                       std::uint32_t nalpha, double pi, std::uint32_t d, std::uint32_t h,
                       std::uint32_t hprime, std::uint32_t gamma, const double* w, double sigma2,
                       double temperature, const double* y, std::uint64_t n,
                       std::uint64_t row_begin, std::uint64_t row_end, double* sum_s,
                       double* sum_ssT, double* sum_y_sT, double* value_counts, double* scalars) {
  return guarded([&] {
    auto m = ld_model(family, d, h, hprime, gamma, alpha, nalpha);
    DataSet ds = wrap_data(y, n, d);
    SuffStats s = m.estep_stats(ld_params(family, d, h, w, sigma2, pi, alpha, probs, nalpha), ds,
                                RowRange{row_begin, row_end}, temperature);
    copy_stats(s, sum_s, sum_ssT, sum_y_sT, value_counts, scalars);
  });
}

int ref_ld_mstep(std::uint32_t family, const double* alpha, const double* probs_prev,
                 std::uint32_t nalpha, double pi_prev, std::uint32_t d, std::uint32_t h,
                 std::uint32_t nv, const double* w_prev, double sigma2_prev, const double* sum_s,
                 const double* sum_ssT, const double* sum_y_sT, const double* value_counts,
                 const double* scalars, double* w_out, double* pi_out, double* probs_out,
                 double* sigma2_out) {
  return guarded([&] {
    auto m = ld_model(family, d, h, h, 1, alpha, nalpha);
    SuffStats s;
    const auto fill = [&](const char* name, std::size_t r, std::size_t c, const double* src) {
      DenseMatrix& f = s.field(name, r, c);
      std::memcpy(f.data(), src, r * c * sizeof(double));
    };
    fill("sum_s", 1, h, sum_s);
    fill("sum_ssT", h, h, sum_ssT);
    fill("sum_y_sT", d, h, sum_y_sT);
    fill("value_counts", 1, nv, value_counts);
    s.scalar("sum_y2") = scalars[0];
    s.scalar("log_partition") = scalars[1];
    s.points = static_cast<std::uint64_t>(scalars[2]);
    ModelParams out = m.mstep(
        s, ld_params(family, d, h, w_prev, sigma2_prev, pi_prev, alpha, probs_prev, nalpha));
    const auto& p = std::get<LinearDiscreteParams>(out);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    if (pi_out) *pi_out = p.pi;
    if (probs_out && family == 2) std::memcpy(probs_out, p.probs.data(), nalpha * sizeof(double));
    *sigma2_out = p.sigma2;
  });
}

int ref_ld_step(std::uint32_t family, const double* alpha, const double* probs,
                std::uint32_t nalpha, double pi, std::uint32_t d, std::uint32_t h,
                std::uint32_t hprime, std::uint32_t gamma, const double* w, double sigma2,
                double temperature, const double* y, std::uint64_t n, std::uint32_t shards,
                std::uint32_t workers, double* w_out, double* pi_out, double* probs_out,
                double* sigma2_out, double* free_energy) {
  return guarded([&] {
    auto m = ld_model(family, d, h, hprime, gamma, alpha, nalpha);
    DataSet ds = wrap_data(y, n, d);
    ShardPlan plan = ShardPlan::with_shards(n, shards, workers);
    AnnealState st;
    st.temperature = temperature;
    StepResult r =
        m.step(ld_params(family, d, h, w, sigma2, pi, alpha, probs, nalpha), st, ds, plan);
    const auto& p = std::get<LinearDiscreteParams>(r.params);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    if (pi_out) *pi_out = p.pi;
    if (probs_out && family == 2) std::memcpy(probs_out, p.probs.data(), nalpha * sizeof(double));
    *sigma2_out = p.sigma2;
    *free_energy = r.free_energy;
  });
}

int ref_ld_inference(std::uint32_t family, const double* alpha, const double* probs,
                     std::uint32_t nalpha, double pi, std::uint32_t d, std::uint32_t h,
                     std::uint32_t hprime, std::uint32_t gamma, const double* w, double sigma2,
                     const double* y, std::uint64_t n, std::uint32_t shards, double* map_states,
                     double* map_mass, double* expected) {
  return guarded([&] {
    auto m = ld_model(family, d, h, hprime, gamma, alpha, nalpha);
    DataSet ds = wrap_data(y, n, d);
    InferenceResult r = m.inference(ld_params(family, d, h, w, sigma2, pi, alpha, probs, nalpha),
                                    ds, ShardPlan::with_shards(n, shards, shards));
    std::memcpy(map_states, r.map_states.data(), r.map_states.size() * sizeof(double));
    std::memcpy(map_mass, r.map_mass.data(), r.map_mass.size() * sizeof(double));
    std::memcpy(expected, r.expected_states.data(), r.expected_states.size() * sizeof(double));
  });
}

// Candidates as estep_impl selects them (:240-253) with the family's value
// table (:71-97, restated: value_table is private).
int ref_ld_candidates(std::uint32_t family, const double* alpha, const double* probs,
                      std::uint32_t nalpha, double pi, std::uint32_t d, std::uint32_t h,
                      std::uint32_t hprime, const double* w, double sigma2, const double* y,
                      std::uint64_t n, std::uint32_t* out) {
  return guarded([&] {
    std::vector<double> values, log_probs;
    if (family == 0) {
      values = {1.0};
      log_probs = {std::log(pi)};
    } else if (family == 1) {
      values = {-1.0, 1.0};
      log_probs = {std::log(pi / 2.0), std::log(pi / 2.0)};
    } else {
      for (std::uint32_t k = 0; k < nalpha; ++k)
        if (alpha[k] != 0.0) {
          values.push_back(alpha[k]);
          log_probs.push_back(std::log(probs[k]));
        }
    }
    const ConstMatView wv(w, d, h);
    const Eigen::MatrixXd gram = wv.transpose() * wv;
    const double inv2s = 1.0 / (2.0 * sigma2);
    std::vector<double> scores(h);
    Eigen::VectorXd b(h);
    for (std::uint64_t i = 0; i < n; ++i) {
      ConstVecView yv(y + i * d, d);
      b.noalias() = wv.transpose() * yv;
      for (std::uint32_t u = 0; u < h; ++u) {
        double best = -std::numeric_limits<double>::infinity();
        for (std::size_t k = 0; k < values.size(); ++k) {
          const double v = values[k];
          best = std::max(best, log_probs[k] + (2.0 * v * b[u] - v * v * gram(u, u)) * inv2s);
        }
        scores[u] = best;
      }
      auto c = select_candidates(scores, hprime);
      std::memcpy(out + i * hprime, c.data(), hprime * sizeof(std::uint32_t));
    }
  });
}

int ref_ld_generate(std::uint32_t family, const double* alpha, const double* probs,
                    std::uint32_t nalpha, double pi, std::uint32_t d, std::uint32_t h,
                    const double* w, double sigma2, std::uint64_t n, std::uint64_t seed,
                    double* y_out) {
  return guarded([&] {
    auto m = ld_model(family, d, h, h, 1, alpha, nalpha);
    RngStream rng(seed);
    DataSet ds = m.generate(ld_params(family, d, h, w, sigma2, pi, alpha, probs, nalpha), n, rng);
    std::memcpy(y_out, ds.y.data(), ds.y.size() * sizeof(double));
  });
}

int ref_ld_exact_log_likelihood(std::uint32_t family, const double* alpha, const double* probs,
                                std::uint32_t nalpha, double pi, std::uint32_t d,
                                std::uint32_t h, const double* w, double sigma2, const double* y,
                                std::uint64_t n, double* out) {
  return guarded([&] {
    auto m = ld_model(family, d, h, h, h, alpha, nalpha);
    *out = m.exact_log_likelihood(ld_params(family, d, h, w, sigma2, pi, alpha, probs, nalpha),
                                  wrap_data(y, n, d));
  });
}

int ref_ld_state_count(std::uint32_t h, std::uint32_t hprime, std::uint32_t gamma,
                       std::uint32_t nv, std::uint64_t* out) {
  return guarded([&] {
    TruncationConfig cfg{h, hprime, gamma, 1000000};
    cfg.validate();
    *out = truncated_state_count(cfg, nv);
  });
}

// ---- max causes (mode 0 mca, 1 mmca; rho = soft winner exponent)
int ref_mca_estep_stats(std::uint32_t mode, double rho, std::uint32_t d, std::uint32_t h,
                        std::uint32_t hprime, std::uint32_t gamma, const double* w, double pi,
                        double sigma2, double temperature, const double* y, std::uint64_t n,
                        std::uint64_t row_begin, std::uint64_t row_end, double* winner_num,
                        double* winner_den, double* scalars) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, hprime, gamma, rho);
    SuffStats s = m.estep_stats(mca_params(d, h, w, pi, sigma2), wrap_data(y, n, d),
                                RowRange{row_begin, row_end}, temperature);
    std::memcpy(winner_num, s.at("winner_num").data(), std::size_t(d) * h * sizeof(double));
    std::memcpy(winner_den, s.at("winner_den").data(), std::size_t(d) * h * sizeof(double));
    scalars[0] = s.scalar("sum_act");
    scalars[1] = s.scalar("log_partition");
    scalars[2] = static_cast<double>(s.points);
  });
}

int ref_mca_mstep_fixedpoint(std::uint32_t mode, std::uint32_t d, std::uint32_t h,
                             const double* w_prev, double pi_prev, double sigma2_prev,
                             const double* winner_num, const double* winner_den,
                             const double* scalars, double* w_out, double* pi_out) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, h, 1, 0.0);
    SuffStats s;
    std::memcpy(s.field("winner_num", d, h).data(), winner_num, std::size_t(d) * h * sizeof(double));
    std::memcpy(s.field("winner_den", d, h).data(), winner_den, std::size_t(d) * h * sizeof(double));
    s.scalar("sum_act") = scalars[0];
    s.scalar("log_partition") = scalars[1];
    s.points = static_cast<std::uint64_t>(scalars[2]);
    ModelParams out = m.mstep_fixedpoint(s, mca_params(d, h, w_prev, pi_prev, sigma2_prev));
    const auto& p = std::get<McaParams>(out);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    *pi_out = p.pi;
  });
}

int ref_mca_step(std::uint32_t mode, double rho, std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                 std::uint32_t gamma, const double* w, double pi, double sigma2, double temperature,
                 const double* y, std::uint64_t n, std::uint32_t shards, std::uint32_t workers,
                 double* w_out, double* pi_out, double* sigma2_out, double* free_energy) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, hprime, gamma, rho);
    AnnealState st;
    st.temperature = temperature;
    StepResult r = m.step(mca_params(d, h, w, pi, sigma2), st, wrap_data(y, n, d),
                          ShardPlan::with_shards(n, shards, workers));
    const auto& p = std::get<McaParams>(r.params);
    std::memcpy(w_out, p.w.data(), p.w.size() * sizeof(double));
    *pi_out = p.pi;
    *sigma2_out = p.sigma2;
    *free_energy = r.free_energy;
  });
}

int ref_mca_candidates(std::uint32_t mode, std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                       const double* w, double pi, double sigma2, const double* y, std::uint64_t n,
                       std::uint32_t* out) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, hprime, 1, 0.0);
    const McaParams p = mca_params(d, h, w, pi, sigma2);
    for (std::uint64_t i = 0; i < n; ++i) {
      auto c = select_candidates(m.selection_scores(p, std::span<const double>(y + i * d, d)), hprime);
      std::memcpy(out + i * hprime, c.data(), hprime * sizeof(std::uint32_t));
    }
  });
}

int ref_mca_inference(std::uint32_t mode, std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                      std::uint32_t gamma, const double* w, double pi, double sigma2, const double* y,
                      std::uint64_t n, std::uint32_t shards, double* map_states, double* map_mass,
                      double* expected) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, hprime, gamma, 0.0);
    InferenceResult r = m.inference(mca_params(d, h, w, pi, sigma2), wrap_data(y, n, d),
                                    ShardPlan::with_shards(n, shards, shards));
    std::memcpy(map_states, r.map_states.data(), r.map_states.size() * sizeof(double));
    std::memcpy(map_mass, r.map_mass.data(), r.map_mass.size() * sizeof(double));
    std::memcpy(expected, r.expected_states.data(), r.expected_states.size() * sizeof(double));
  });
}

int ref_mca_log_joint(std::uint32_t mode, std::uint32_t d, std::uint32_t h, const double* w, double pi,
                      double sigma2, const double* y, const double* s, double* out) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, h, 1, 0.0);
    *out = m.log_joint(mca_params(d, h, w, pi, sigma2), std::span<const double>(y, d),
                       std::span<const double>(s, h));
  });
}

int ref_mca_exact_log_likelihood(std::uint32_t mode, std::uint32_t d, std::uint32_t h, const double* w,
                                 double pi, double sigma2, const double* y, std::uint64_t n, double* out) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, h, h, 0.0);
    *out = m.exact_log_likelihood(mca_params(d, h, w, pi, sigma2), wrap_data(y, n, d));
  });
}

int ref_mca_generate(std::uint32_t mode, std::uint32_t d, std::uint32_t h, const double* w, double pi,
                     double sigma2, std::uint64_t n, std::uint64_t seed, double* y_out) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, h, 1, 0.0);
    RngStream rng(seed);
    DataSet ds = m.generate(mca_params(d, h, w, pi, sigma2), n, rng);
    std::memcpy(y_out, ds.y.data(), ds.y.size() * sizeof(double));
  });
}

int ref_mca_standard_init(std::uint32_t mode, std::uint32_t d, std::uint32_t h, std::uint32_t hprime,
                          const double* y, std::uint64_t n, std::uint64_t seed, double* w_out,
                          double* pi_out, double* sigma2_out) {
  return guarded([&] {
    auto m = mca_model(mode, d, h, hprime, 1, 0.0);
    RngStream rng(seed);
    ModelParams p = m.standard_init(wrap_data(y, n, d), rng);
    const auto& mp = std::get<McaParams>(p);
    std::memcpy(w_out, mp.w.data(), mp.w.size() * sizeof(double));
    *pi_out = mp.pi;
    *sigma2_out = mp.sigma2;
  });
}

// ---- run I/O and the EM driver (array_io.cpp, sha256.cpp, em.cpp, annealing.cpp)
int ref_save_array(const char* path, const double* data, std::uint64_t rows, std::uint64_t cols) {
  return guarded([&] { save_array(path, DenseMatrix(rows, cols, std::vector<double>(data, data + rows * cols))); });
}

int ref_load_dataset(const char* path, std::uint64_t* rows, std::uint64_t* cols, double* out) {
  return guarded([&] {
    DataSet ds = load_dataset(path);
    *rows = ds.size();
    *cols = ds.dim();
    if (out) std::memcpy(out, ds.y.data(), ds.y.size() * sizeof(double));
  });
}

int ref_sha256(const void* data, std::uint64_t bytes, char* hex65) {
  return guarded([&] {
    const std::string h = sha256_hex({static_cast<const std::uint8_t*>(data), static_cast<std::size_t>(bytes)});
    std::memcpy(hex65, h.c_str(), 65);
  });
}

int ref_sha256_file(const char* path, char* hex65) {
  return guarded([&] { std::memcpy(hex65, sha256_hex_file(path).c_str(), 65); });
}

int ref_format_double(double v, char* out, std::uint32_t cap) {
  return guarded([&] {
    const std::string s = format_double(v);
    if (s.size() + 1 > cap) throw ConfigError("buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

// train_run's model setup and EM loop (run_io.cpp:196-230, em.cpp:27-77)
// without the directory logger: standard_init from RngStream::derived(seed,
// "init"), LinearAnnealing over the schedules, TrainOptions{tol, seed}.
int ref_train(const char* model, const double* values, std::uint32_t n_values, std::uint32_t d,
              std::uint32_t h, std::uint32_t hprime, std::uint32_t gamma, std::uint64_t iterations,
              std::uint64_t seed, std::uint32_t shards, std::uint32_t workers, int has_tol, double tol,
              const double* tpos, const double* tval, std::uint32_t nt, const double* npos,
              const double* nval, std::uint32_t nn, const double* y, std::uint64_t n, double* trace,
              std::uint64_t* iters, double* w_out, double* pi_out, double* sigma2_out, double* probs_out) {
  return guarded([&] {
    std::vector<double> vals(values, values + n_values);
    auto m = make_model(model, d, h, TruncationConfig{h, hprime, gamma}, vals);
    DataSet ds = wrap_data(y, n, d);
    RngStream init_rng = RngStream::derived(seed, 0x696e6974);
    ModelParams params = m->standard_init(ds, init_rng);
    auto sched = [](const double* p, const double* v, std::uint32_t k, double dflt) {
      if (!p || k == 0) return Schedule::constant(dflt);
      std::vector<std::pair<double, double>> a;
      for (std::uint32_t i = 0; i < k; ++i) a.emplace_back(p[i], v[i]);
      return Schedule(a);
    };
    LinearAnnealing ann(iterations, sched(tpos, tval, nt, 1.0), sched(npos, nval, nn, 0.0));
    TrainOptions opt;
    if (has_tol) opt.tol = tol;
    opt.noise_seed = seed;
    TrainResult r = run(*m, std::move(params), ds, ann, ShardPlan::with_shards(n, shards, workers), nullptr, opt);
    *iters = r.free_energy_trace.size();
    std::memcpy(trace, r.free_energy_trace.data(), r.free_energy_trace.size() * sizeof(double));
    if (const auto* p = std::get_if<LinearDiscreteParams>(&r.final_params)) {
      std::memcpy(w_out, p->w.data(), p->w.size() * sizeof(double));
      *pi_out = p->pi;
      *sigma2_out = p->sigma2;
      if (probs_out && !p->probs.empty()) std::memcpy(probs_out, p->probs.data(), p->probs.size() * sizeof(double));
    } else {
      const auto& q = std::get<McaParams>(r.final_params);
      std::memcpy(w_out, q.w.data(), q.w.size() * sizeof(double));
      *pi_out = q.pi;
      *sigma2_out = q.sigma2;
    }
  });
}

}  // extern "C"
