// NCCL, resolved at run time (one all-reduce of the packed
// sufficient statistics per EM iteration over NVLink/NVSwitch).
//
// The engine library does not link NCCL: the first use dlopen()s
// "libnccl.so.2" — the copy already mapped by the host process (torch's, for
// instance) when there is one, else the system library — and looks up the five
// entry points it calls. A host program that owns its communicator hands it
// over as an opaque pointer; one that does not builds one from a unique id.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "bsc_engine.hpp"

namespace bscgpu {
namespace nccl {

// the fixed NCCL ABI pieces used here (nccl.h: ncclUniqueId, ncclFloat64, ncclSum)
struct UniqueId {
  char internal[128];
};
using Comm = void*;
enum : int { kSuccess = 0, kFloat64 = 8, kSum = 0 };

struct Api {
  int (*get_unique_id)(UniqueId*) = nullptr;
  int (*comm_init_rank)(Comm*, int, UniqueId, int) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*comm_destroy)(Comm) = nullptr;
  const char* (*error_string)(int) = nullptr;
  int (*comm_count)(Comm, int*) = nullptr;
  std::string why;  // empty when loaded
};

inline const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("nccl: cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp && a.why.empty()) a.why = std::string("nccl: missing symbol ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.error_string, "ncclGetErrorString");
    sym(a.comm_count, "ncclCommCount");
  });
  return a;
}

inline const Api& need() {
  const Api& a = api();
  if (!a.why.empty()) throw Error(kInternal, a.why);
  return a;
}

inline void check(int rc, const char* what) {
  if (rc != kSuccess) {
    const Api& a = api();
    throw Error(kInternal, std::string("nccl: ") + what + ": " + (a.error_string ? a.error_string(rc) : "error"));
  }
}

}  // namespace nccl
}  // namespace bscgpu
