// CPU data fixtures of the reference (not the hot path): the seeded stream,
// the bars generator, the BSC sampler and the two initialisations. They follow
// the reference draw order so the bench's synthetic inputs are the same bytes
// the parity oracle sees.
#include "fixtures.hpp"

#include <algorithm>
#include <cmath>
#include <random>

#include "bsc_engine.hpp"
#include "rng_stream.hpp"

namespace bscgpu {

namespace {

void column_means(const double* y, uint64_t n, uint32_t d, std::vector<double>& m) {
  m.assign(d, 0.0);
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) m[j] += y[i * d + j];
  for (auto& v : m) v /= static_cast<double>(n);
}

double mean_variance(const double* y, uint64_t n, uint32_t d, const std::vector<double>& m) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) {
      const double c = y[i * d + j] - m[j];
      acc += c * c;
    }
  return acc / static_cast<double>(n * d);
}

}  // namespace

void bars_generate(uint32_t size, uint64_t n, double prob, double amplitude, double noise, bool max_mode,
                   uint64_t seed, double* y, double* truth) {
  if (size == 0) throw Error(kConfig, "bars: size must be >= 1");
  if (n == 0) throw Error(kConfig, "bars: need at least one data point");
  if (amplitude <= 0.0) throw Error(kConfig, "bars: amplitude must be > 0");
  if (noise < 0.0) throw Error(kConfig, "bars: noise must be >= 0");
  const uint32_t nb = 2 * size;
  const double p = prob > 0.0 ? prob : 2.0 / static_cast<double>(nb);
  if (p >= 1.0) throw Error(kConfig, "bars: prob must lie in (0,1)");
  const size_t d = static_cast<size_t>(size) * size;
  std::vector<double> w(d * nb, 0.0);
  for (uint32_t k = 0; k < size; ++k)
    for (uint32_t j = 0; j < size; ++j) {
      w[(static_cast<size_t>(k) * size + j) * nb + k] = amplitude;
      w[(static_cast<size_t>(j) * size + k) * nb + size + k] = amplitude;
    }
  Stream rng(seed);
  std::vector<uint32_t> act;
  for (uint64_t i = 0; i < n; ++i) {
    act.clear();
    for (uint32_t b = 0; b < nb; ++b)
      if (rng.bernoulli(p)) act.push_back(b);
    for (size_t px = 0; px < d; ++px) {
      double v = 0.0;
      for (uint32_t b : act) v = max_mode ? std::max(v, w[px * nb + b]) : v + w[px * nb + b];
      y[i * d + px] = v + noise * rng.normal();
    }
  }
  if (truth) std::copy(w.begin(), w.end(), truth);
}

void generate(uint32_t d, uint32_t h, const double* w, double pi, double sigma2, uint64_t n, uint64_t seed,
              double* y) {
  for (size_t i = 0; i < static_cast<size_t>(d) * h; ++i)
    if (!std::isfinite(w[i])) throw Error(kNumeric, "bsc: non-finite dictionary");
  if (!(sigma2 > 0.0)) throw Error(kConfig, "bsc: sigma2 must be positive");
  if (!(pi > 0.0 && pi < 1.0)) throw Error(kConfig, "bsc: pi must lie in (0,1)");
  const double sd = std::sqrt(sigma2);
  Stream rng(seed);
  std::vector<uint32_t> act;
  for (uint64_t i = 0; i < n; ++i) {
    act.clear();
    for (uint32_t j = 0; j < h; ++j)
      if (rng.bernoulli(pi)) act.push_back(j);
    for (uint32_t r = 0; r < d; ++r) {
      // mean = W s, left to right; zero terms add exact zeros, unit terms add W
      double acc = 0.0;
      for (uint32_t j : act) acc += w[static_cast<size_t>(r) * h + j];
      y[i * d + r] = acc + sd * rng.normal();
    }
  }
}

void random_dictionary(uint32_t d, uint32_t h, uint64_t seed, double scale, double* w) {
  Stream rng = Stream::derived(seed, 0x77747275ULL);
  for (size_t i = 0; i < static_cast<size_t>(d) * h; ++i) w[i] = rng.normal();
  for (uint32_t j = 0; j < h; ++j) {
    double acc = 0.0;
    for (uint32_t i = 0; i < d; ++i) acc += w[static_cast<size_t>(i) * h + j] * w[static_cast<size_t>(i) * h + j];
    const double nrm = std::sqrt(acc);
    for (uint32_t i = 0; i < d; ++i) w[static_cast<size_t>(i) * h + j] = w[static_cast<size_t>(i) * h + j] / nrm * scale;
  }
}

void baseline_init(uint32_t d, uint32_t h, const double* y, uint64_t n, uint64_t seed, double* w, double* pi,
                   double* sigma2) {
  if (n < 2) throw Error(kData, "init requires at least two data points");
  std::vector<double> m, sd(d, 0.0);
  column_means(y, n, d, m);
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) {
      const double c = y[i * d + j] - m[j];
      sd[j] += c * c;
    }
  for (auto& v : sd) v = std::sqrt(v / static_cast<double>(n));
  Stream rng = Stream::derived(seed, 0x696e6974ULL);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) w[static_cast<size_t>(i) * h + j] = m[i] + 0.25 * sd[i] * rng.normal();
  *pi = 1.0 / static_cast<double>(h);
  *sigma2 = std::max(mean_variance(y, n, d, m), 1e-12);
}

// LinearDiscreteModel::standard_init (linear_discrete.cpp:129-148) with
// detail::init_weights (model.cpp:201-220).
void standard_init(uint32_t d, uint32_t h, uint32_t hprime, const double* y, uint64_t n, uint64_t seed, double* w,
                   double* pi, double* sigma2) {
  if (n < 2) throw Error(kData, "standard_init requires at least two data points");
  std::vector<double> m;
  column_means(y, n, d, m);
  const double var = mean_variance(y, n, d, m);
  const double sd = var > 0.0 ? std::sqrt(var / h) : 0.0;
  Stream rng(seed);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) w[static_cast<size_t>(i) * h + j] = m[i] + sd * rng.normal();
  *sigma2 = std::max(var, 1e-12);
  *pi = static_cast<double>(std::min(hprime, h)) / (2.0 * static_cast<double>(h));
}

}  // namespace bscgpu
