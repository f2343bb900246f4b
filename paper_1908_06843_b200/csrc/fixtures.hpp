// CPU fixtures of the reference (bars, sampler, initialisations); see fixtures.cpp.
#pragma once
#include <cstdint>

namespace bscgpu {

void bars_generate(uint32_t size, uint64_t n, double prob, double amplitude, double noise, bool max_mode,
                   uint64_t seed, double* y, double* truth);
void generate(uint32_t d, uint32_t h, const double* w, double pi, double sigma2, uint64_t n, uint64_t seed,
              double* y);
void random_dictionary(uint32_t d, uint32_t h, uint64_t seed, double scale, double* w);
void baseline_init(uint32_t d, uint32_t h, const double* y, uint64_t n, uint64_t seed, double* w, double* pi,
                   double* sigma2);
void standard_init(uint32_t d, uint32_t h, uint32_t hprime, const double* y, uint64_t n, uint64_t seed, double* w,
                   double* pi, double* sigma2);

}  // namespace bscgpu
