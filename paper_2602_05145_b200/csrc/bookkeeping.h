// Internal bit-exact restatement of the reference's bookkeeping: the seeded
// Rng (rng.hpp:13-39) and the accept-length model (perf_model.cpp:159-177,
// 213-224), plus the analytic current_alpha law (workload.cpp:41-47).
//
// Deliberately NOT in the public C++ header and NOT exported (the library is
// built with -fvisibility=hidden): a reference translation unit that
// includes rng.hpp / perf_model.hpp and links perf_model.cpp next to this
// library must see exactly one definition of those names.  Callers outside
// the library reach these through the C ABI (specsim_rng_*,
// specsim_*accept_length, specsim_current_alpha).
#pragma once

#include <cstdint>
#include <random>

namespace specsim {
namespace bk {

// mt19937_64 with the reference's hand-rolled conversions.
class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  uint64_t next_u64() { return eng_(); }
  double uniform();                       // [0, 1), 53 bits
  double normal(double mean, double sd);  // Box-Muller, cosine branch
  long long geometric(double mean);       // {1, 2, ...}

 private:
  std::mt19937_64 eng_;
};

double expected_accept_length(double alpha, int gamma);
int sample_accept_length(Rng& rng, double alpha, int gamma);
double alpha_from_accept_length(double ell, int gamma);
// alpha(n) = ceiling - (ceiling - start) exp(-n / tau), clamped to [0, 1]
double current_alpha(double alpha_start, double alpha_ceiling, double tau_samples,
                     double trained_samples);

}  // namespace bk
}  // namespace specsim
