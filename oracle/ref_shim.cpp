// C shim over the UNMODIFIED reference sources (compiled in place from
// /root/reference/proj by build_ref.sh).  Test infrastructure only: it lets
// the tests and tests/golden/make_golden.py call the reference's own
// Rng / perf_model / workload code through ctypes.
#include <cstdint>
#include <exception>

#include "specsim/perf_model.hpp"
#include "specsim/rng.hpp"
#include "specsim/workload.hpp"

extern "C" {

void* ref_rng_create(uint64_t seed) { return new specsim::Rng(seed); }
void ref_rng_destroy(void* r) { delete static_cast<specsim::Rng*>(r); }
double ref_rng_uniform(void* r) { return static_cast<specsim::Rng*>(r)->uniform(); }
double ref_rng_normal(void* r, double mean, double sd) {
  return static_cast<specsim::Rng*>(r)->normal(mean, sd);
}
long long ref_rng_geometric(void* r, double mean) {
  return static_cast<specsim::Rng*>(r)->geometric(mean);
}

int ref_expected_accept_length(double alpha, int gamma, double* out) {
  try { *out = specsim::expected_accept_length(alpha, gamma); return 0; }
  catch (const std::invalid_argument&) { return 1; }
}
int ref_sample_accept_length(void* r, double alpha, int gamma, int* out) {
  try { *out = specsim::sample_accept_length(*static_cast<specsim::Rng*>(r), alpha, gamma); return 0; }
  catch (const std::invalid_argument&) { return 1; }
}
int ref_alpha_from_accept_length(double ell, int gamma, double* out) {
  try { *out = specsim::alpha_from_accept_length(ell, gamma); return 0; }
  catch (const std::invalid_argument&) { return 1; }
}
double ref_current_alpha(double a0, double astar, double tau, double n) {
  specsim::PhaseSpec p;
  p.name = "p";
  p.alpha_start = a0;
  p.alpha_ceiling = astar;
  p.tau_samples = tau;
  return specsim::current_alpha(p, n);
}
// Workload script of one phase: returns total tokens, first request length.
long long ref_workload_tokens(int n, int mean_tokens, double noise_sd, uint64_t seed,
                              long long* first_len) {
  specsim::PhaseSpec p;
  p.name = "p";
  p.num_requests = n;
  p.concurrency = 1;
  p.mean_output_tokens = mean_tokens;
  p.alpha_start = 0.3;
  p.alpha_ceiling = 0.6;
  p.tau_samples = 100;
  p.alpha_noise_sd = noise_sd;
  specsim::WorkloadScript w({p}, seed);
  *first_len = w.request(0).output_tokens_remaining;
  return w.total_output_tokens();
}
}
