// C-ABI plumbing: last-error slot and version string.
#include <string>

#include "common.h"

namespace specsim {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace specsim

extern "C" const char* specsim_last_error(void) { return specsim::g_last_error.c_str(); }

extern "C" const char* specsim_version(void) { return "specsim-draft-b200 0.1 (sm_100a)"; }
