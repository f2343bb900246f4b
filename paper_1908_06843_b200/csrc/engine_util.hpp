// Small host helpers shared by the engine translation units.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <string>

#include "bsc_engine.hpp"

namespace bscgpu {
namespace util {

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(kInternal, std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t count, const char* what) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), what);
  ck(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T)), what);
  return static_cast<T*>(p);
}

// NVTX range over the host-side enqueue of one phase (header-only NVTX 3: a no-op
// unless a tool injects itself; SURVEY.md §5 tracing).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

inline void dfree(void* p) {
  if (p) cudaFree(p);
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Register-resident unit slots per lane (H ≤ 32·MAXJ).
inline int maxj_for(uint32_t h) {
  const int need = static_cast<int>((h + 31) / 32);
  for (int m : {1, 2, 4, 6, 8, 10, 12, 16, 24, 32})
    if (need <= m) return m;
  return 32;
}

constexpr double kLog2Pi = 1.8378770664093454836;  // linear_discrete.cpp:24

}  // namespace util
}  // namespace bscgpu
