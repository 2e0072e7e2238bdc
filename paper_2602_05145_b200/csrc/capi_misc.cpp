// C-ABI plumbing: last-error slot and version string.
#include <string>

#include "common.h"

namespace specsim {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
std::atomic<unsigned long long> g_kernel_launches{0};
}  // namespace specsim

extern "C" const char* specsim_last_error(void) { return specsim::g_last_error.c_str(); }

extern "C" const char* specsim_version(void) { return "specsim-draft-b200 0.1 (sm_100a)"; }

extern "C" int specsim_kernel_launches(uint64_t* out) {
  if (!out) return SPECSIM_EDOMAIN;
  *out = specsim::g_kernel_launches.load();
  return SPECSIM_OK;
}
