// RngStream of the reference (core.hpp:129-150, core.cpp:50-91), host side:
// mt19937_64 engine, 53-bit uniforms, Box-Muller normals, splitmix64-derived
// sub-streams. Shared by the fixtures and the run driver (run_io.cpp).
#pragma once
#include <cmath>
#include <cstdint>
#include <random>

namespace bscgpu {

// splitmix64 (core.cpp:50-57)
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

class Stream {
 public:
  explicit Stream(uint64_t seed) : eng_(seed) {}
  static Stream derived(uint64_t base, uint64_t index) { return Stream(mix64(mix64(base) ^ mix64(index + 1))); }
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double normal() {
    double u1 = uniform01();
    while (u1 <= 0.0) u1 = uniform01();
    const double u2 = uniform01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
  bool bernoulli(double p) { return uniform01() < p; }

 private:
  std::mt19937_64 eng_;
};

}  // namespace bscgpu
