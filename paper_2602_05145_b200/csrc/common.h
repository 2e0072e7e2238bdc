// Error taxonomy and C-ABI guard.
//
// Mirrors the reference's split (proj/include/specsim/errors.hpp:8-13):
// std::invalid_argument = domain error (CLI exit 1), specsim::ConfigError =
// configuration error (CLI exit 2).  Device failures get their own codes.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "specsim_draft_trainer.h"
#include "specsim/draft_trainer.hpp"  // ConfigError / CudaError / NcclError (public)

namespace specsim {

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                  std::to_string(line) + ")");
}

#define SPECSIM_CUDA(call)                                                 \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) ::specsim::throw_cuda(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define SPECSIM_CHECK_LAUNCH() SPECSIM_CUDA(cudaGetLastError())

// Collect-all-problems validation, like LatencyProfile's constructor
// (perf_model.cpp:57-82): gather every problem, throw once.
class Problems {
 public:
  explicit Problems(std::string what) : what_(std::move(what)) {}
  void check(bool ok, const std::string& msg) {
    if (!ok) items_.push_back(msg);
  }
  template <class E = std::invalid_argument>
  void throw_if_any() const {
    if (items_.empty()) return;
    std::string m = what_ + ":";
    for (const auto& p : items_) m += "\n  - " + p;
    throw E(m);
  }

 private:
  std::string what_;
  std::vector<std::string> items_;
};

void set_last_error(const std::string& msg);

// Number of device kernels this library has launched (all streams); read by
// the benchmark as its gpu_launches evidence.
extern std::atomic<unsigned long long> g_kernel_launches;
inline void count_launches(unsigned n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }

// Runs f, mapping exceptions onto specsim_status codes.
template <class F>
int guard(F&& f) {
  try {
    f();
    set_last_error("");
    return SPECSIM_OK;
  } catch (const ConfigError& e) {
    set_last_error(e.what());
    return SPECSIM_ECONFIG;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return SPECSIM_ECUDA;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return SPECSIM_ENCCL;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return SPECSIM_EDOMAIN;
  } catch (const std::out_of_range& e) {
    set_last_error(e.what());
    return SPECSIM_EDOMAIN;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SPECSIM_ECUDA;
  }
}

}  // namespace specsim
