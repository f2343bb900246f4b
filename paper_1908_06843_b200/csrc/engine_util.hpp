// Small host helpers shared by the engine translation units.
#pragma once
#include <cuda.h>
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
//
// BSC_GUARD=2 catches overruns by READS as well: every buffer is mapped through the driver's
// virtual-memory API so that it ENDS (to 16 bytes) at the end of its mapping, followed by an unmapped
// page of address space — a load or store past the end of a buffer is an immediate device fault.
// BSC_GUARD=3 is the mirror image for underruns (the buffer starts its mapping, unmapped page in front).
struct GuardRegistry {
  struct Entry {
    size_t bytes;
    std::string what;
  };
  struct Mapping {
    CUdeviceptr va;
    size_t reserved, mapped;
    CUmemGenericAllocationHandle handle;
  };
  std::mutex m;
  std::unordered_map<void*, Entry> live;
  std::unordered_map<void*, Mapping> mappings;
  bool on = false;   // BSC_GUARD=1: guard bytes
  bool vmm = false;  // BSC_GUARD=2: end-aligned mappings with an unmapped page behind
  bool vmm_front = false;  // BSC_GUARD=3: mappings that START at the buffer, with an unmapped page in front (underruns)
};
inline GuardRegistry& guard_registry() {
  static GuardRegistry g;
  static const bool init = [] {
    const char* e = std::getenv("BSC_GUARD");
    g.on = e && e[0] == '1';
    g.vmm = e && (e[0] == '2' || e[0] == '3');
    g.vmm_front = e && e[0] == '3';
    return true;
  }();
  (void)init;
  return g;
}

// driver entry points of the virtual-memory API (the library links cudart statically, not libcuda)
struct VmmApi {
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*address_free)(CUdeviceptr, size_t) = nullptr;
  bool ok = false;
};
inline VmmApi& vmm_api() {
  static VmmApi a = [] {
    VmmApi v;
    auto get = [](const char* name) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
      return p;
    };
    v.granularity = reinterpret_cast<decltype(v.granularity)>(get("cuMemGetAllocationGranularity"));
    v.reserve = reinterpret_cast<decltype(v.reserve)>(get("cuMemAddressReserve"));
    v.create = reinterpret_cast<decltype(v.create)>(get("cuMemCreate"));
    v.map = reinterpret_cast<decltype(v.map)>(get("cuMemMap"));
    v.set_access = reinterpret_cast<decltype(v.set_access)>(get("cuMemSetAccess"));
    v.unmap = reinterpret_cast<decltype(v.unmap)>(get("cuMemUnmap"));
    v.release = reinterpret_cast<decltype(v.release)>(get("cuMemRelease"));
    v.address_free = reinterpret_cast<decltype(v.address_free)>(get("cuMemAddressFree"));
    v.ok = v.granularity && v.reserve && v.create && v.map && v.set_access && v.unmap && v.release && v.address_free;
    return v;
  }();
  return a;
}

inline void* vmm_alloc(size_t bytes, const char* what) {
  VmmApi& v = vmm_api();
  if (!v.ok) throw Error(kInternal, std::string("guard: virtual-memory API unavailable (") + what + ")");
  auto cu = [&](CUresult r, const char* step) {
    if (r != CUDA_SUCCESS) throw Error(kInternal, std::string("guard: ") + step + " failed for " + what);
  };
  int dev = 0;
  ck(cudaGetDevice(&dev), what);
  ck(cudaFree(nullptr), what);  // (a context on this device)
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  size_t gran = 0;
  cu(v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "granularity");
  const size_t user = (bytes + 15) & ~size_t(15);
  GuardRegistry::Mapping m{};
  m.mapped = (user + gran - 1) / gran * gran;
  m.reserved = m.mapped + gran;  // one granule of unmapped address space behind (or in front of) the mapping
  const bool front = guard_registry().vmm_front;
  CUdeviceptr base = 0;
  cu(v.reserve(&base, m.reserved, gran, 0, 0), "address reserve");
  m.va = front ? base + gran : base;  // (Mapping::va is the mapped range; the reservation starts at va or va − gran)
  cu(v.create(&m.handle, m.mapped, &prop, 0), "create");
  cu(v.map(m.va, m.mapped, 0, m.handle, 0), "map");
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu(v.set_access(m.va, m.mapped, &acc, 1), "set access");
  // the buffer ends where the mapping ends (overruns fault), or starts where it starts (underruns fault)
  void* p = reinterpret_cast<void*>(front ? m.va : m.va + m.mapped - user);
  ck(cudaMemset(reinterpret_cast<void*>(m.va), 0, m.mapped), what);
  GuardRegistry& g = guard_registry();
  std::lock_guard<std::mutex> lock(g.m);
  g.mappings[p] = m;
  return p;
}
inline bool vmm_free(void* p) {
  GuardRegistry& g = guard_registry();
  GuardRegistry::Mapping m{};
  {
    std::lock_guard<std::mutex> lock(g.m);
    auto it = g.mappings.find(p);
    if (it == g.mappings.end()) return false;
    m = it->second;
    g.mappings.erase(it);
  }
  cudaDeviceSynchronize();
  VmmApi& v = vmm_api();
  v.unmap(m.va, m.mapped);
  v.release(m.handle);
  v.address_free(guard_registry().vmm_front ? m.va - (m.reserved - m.mapped) : m.va, m.reserved);
  return true;
}
constexpr size_t kGuardBytes = 256;

inline void* dalloc_bytes(size_t bytes, const char* what) {
  GuardRegistry& g = guard_registry();
  bytes = std::max<size_t>(bytes, 1);
  if (g.vmm) return vmm_alloc(bytes, what);
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
  if (g.vmm && vmm_free(p)) return;
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
