// Small host helpers shared by the engine translation units.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "bsc_engine.hpp"

namespace bscgpu {
namespace util {

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(kInternal, std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

// Guarded allocations (BSC_GUARD=1; the pool's compute-sanitizer is closed): every device buffer
// gets 256 bytes of 0xA5 in front and behind, and check_guards() — prsp_bsc_gpu_check_guards in the
// C ABI — reports the first buffer whose guards a kernel has written. Off by default.
struct GuardRegistry {
  struct Entry {
    size_t bytes;
    std::string what;
  };
  std::mutex m;
  std::unordered_map<void*, Entry> live;
  bool on = false;
};
inline GuardRegistry& guard_registry() {
  static GuardRegistry g;
  static const bool init = [] {
    const char* e = std::getenv("BSC_GUARD");
    g.on = e && e[0] == '1';
    return true;
  }();
  (void)init;
  return g;
}
constexpr size_t kGuardBytes = 256;

inline void* dalloc_bytes(size_t bytes, const char* what) {
  GuardRegistry& g = guard_registry();
  bytes = std::max<size_t>(bytes, 1);
  void* p = nullptr;
  if (!g.on) {
    ck(cudaMalloc(&p, bytes), what);
    ck(cudaMemset(p, 0, bytes), what);
    return p;
  }
  ck(cudaMalloc(&p, bytes + 2 * kGuardBytes), what);
  char* base = static_cast<char*>(p);
  ck(cudaMemset(base, 0xA5, kGuardBytes), what);
  ck(cudaMemset(base + kGuardBytes, 0, bytes), what);
  ck(cudaMemset(base + kGuardBytes + bytes, 0xA5, kGuardBytes), what);
  std::lock_guard<std::mutex> lock(g.m);
  g.live[base + kGuardBytes] = GuardRegistry::Entry{bytes, what};
  return base + kGuardBytes;
}

template <class T>
T* dalloc(size_t count, const char* what) {
  return static_cast<T*>(dalloc_bytes(std::max<size_t>(count, 1) * sizeof(T), what));
}

// Empty when every live buffer's guards are intact (or guarding is off), else a description.
inline std::string check_guards() {
  GuardRegistry& g = guard_registry();
  if (!g.on) return "";
  ck(cudaDeviceSynchronize(), "guard check");
  std::lock_guard<std::mutex> lock(g.m);
  std::vector<unsigned char> h(2 * kGuardBytes);
  for (const auto& kv : g.live) {
    const char* user = static_cast<const char*>(kv.first);
    ck(cudaMemcpy(h.data(), user - kGuardBytes, kGuardBytes, cudaMemcpyDeviceToHost), "guard D2H");
    ck(cudaMemcpy(h.data() + kGuardBytes, user + kv.second.bytes, kGuardBytes, cudaMemcpyDeviceToHost), "guard D2H");
    for (size_t i = 0; i < 2 * kGuardBytes; ++i)
      if (h[i] != 0xA5)
        return "buffer '" + kv.second.what + "' (" + std::to_string(kv.second.bytes) + " bytes): write " +
               (i < kGuardBytes ? std::to_string(kGuardBytes - i) + " bytes before its start"
                                : std::to_string(i - kGuardBytes) + " bytes past its end");
  }
  return "";
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
  if (!p) return;
  GuardRegistry& g = guard_registry();
  if (g.on) {
    std::lock_guard<std::mutex> lock(g.m);
    auto it = g.live.find(p);
    if (it != g.live.end()) {
      g.live.erase(it);
      cudaFree(static_cast<char*>(p) - kGuardBytes);
      return;
    }
  }
  cudaFree(p);
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
