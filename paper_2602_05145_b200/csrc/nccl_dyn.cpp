#include "nccl_dyn.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.h"

namespace specsim {
namespace nccl {

const Api& api() {
  static Api a{};
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    // an explicit SPECSIM_NCCL_LIB wins (deployment pinning, or the tests'
    // in-process stand-in); then a copy the host framework already loaded;
    // then the loader search path
    void* h = nullptr;
    if (const char* p = std::getenv("SPECSIM_NCCL_LIB")) {
      h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
      if (!h) {
        err = std::string("cannot load SPECSIM_NCCL_LIB=") + p + ": " + dlerror();
        return;
      }
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.ReduceScatter =
        reinterpret_cast<decltype(a.ReduceScatter)>(dlsym(h, "ncclReduceScatter"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString =
        reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.ReduceScatter ||
        !a.AllGather || !a.CommDestroy || !a.GetErrorString)
      err = "libnccl.so.2 lacks a required symbol";
  });
  if (!err.empty()) throw NcclError(err);
  return a;
}

}  // namespace nccl
}  // namespace specsim
