// Host bookkeeping of the hot path: seeded Rng, accept-length draws, alpha
// inverse, chronological split, signal geometry, synthetic captures.
// Semantics follow the reference (rng.hpp:13-39, perf_model.cpp:30-41,
// perf_model.cpp:159-177, perf_model.cpp:213-224, SPEC.md:237-241,
// SPEC.md:294) and are checked bit-exact against the compiled
// reference by tests/test_capi_cpu.py (golden vectors from oracle/_ref).  Compiled without FP
// contraction (see Makefile) so every double rounds like the reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>
#include <thread>
#include <vector>

#include "bookkeeping.h"
#include "common.h"
#include "specsim/draft_trainer.hpp"

namespace specsim {
namespace bk {

double Rng::uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }

double Rng::normal(double mean, double sd) {
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * std::numbers::pi * u2;
  return mean + sd * radius * std::cos(angle);
}

long long Rng::geometric(double mean) {
  if (mean <= 1.0) return 1;
  const double q = std::log1p(-1.0 / mean);
  const double k = std::floor(std::log1p(-uniform()) / q);
  return k > 0.0 ? 1 + static_cast<long long>(k) : 1;
}

namespace {
void require_alpha_gamma(double alpha, int gamma) {
  Problems p("accept-length model");
  p.check(alpha >= 0.0 && alpha <= 1.0, "alpha must be in [0,1], got " + std::to_string(alpha));
  p.check(gamma >= 1, "gamma must be >= 1, got " + std::to_string(gamma));
  p.throw_if_any();
}
}  // namespace

double expected_accept_length(double alpha, int gamma) {
  require_alpha_gamma(alpha, gamma);
  // power sum 1 + a + ... + a^gamma (exact at alpha = 1)
  double power = 1.0, total = 1.0;
  for (int i = 0; i < gamma; ++i) {
    power *= alpha;
    total += power;
  }
  return total;
}

int sample_accept_length(Rng& rng, double alpha, int gamma) {
  require_alpha_gamma(alpha, gamma);
  int k = 1;
  while (k <= gamma && rng.uniform() < alpha) ++k;
  return k;
}

// workload.cpp:41-47 (+ the PhaseSpec checks of workload.cpp:25-36, as a
// ConfigError): the analytic draft-quality law the reference's train() uses
// for alpha_eval; kept so simulator-mode callers have it next to the real
// trainer that replaces it.
double current_alpha(double alpha_start, double alpha_ceiling, double tau_samples,
                     double trained_samples) {
  Problems p("invalid phase");
  p.check(alpha_start >= 0.0 && alpha_start <= 1.0, "alpha_start outside [0,1]");
  p.check(alpha_ceiling >= 0.0 && alpha_ceiling <= 1.0, "alpha_ceiling outside [0,1]");
  p.check(alpha_start <= alpha_ceiling, "alpha_start > alpha_ceiling");
  p.check(tau_samples > 0.0, "tau_samples <= 0");
  p.throw_if_any<ConfigError>();
  const double n = std::max(0.0, trained_samples);
  const double alpha =
      alpha_ceiling - (alpha_ceiling - alpha_start) * std::exp(-n / tau_samples);
  return std::clamp(alpha, 0.0, 1.0);
}

double alpha_from_accept_length(double ell, int gamma) {
  if (gamma < 1) throw std::invalid_argument("gamma must be >= 1");
  if (!(ell >= 1.0 && ell <= gamma + 1.0))
    throw std::invalid_argument("accept length must be in [1, gamma+1], got " +
                                std::to_string(ell));
  if (ell <= 1.0) return 0.0;
  if (ell >= gamma + 1.0) return 1.0;
  // bisection on the monotone E[l](alpha) to 1e-6, returning the midpoint
  double lo = 0.0, hi = 1.0;
  while (hi - lo > 1e-6) {
    const double mid = 0.5 * (lo + hi);
    (expected_accept_length(mid, gamma) < ell ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}

}  // namespace bk

void split_train_eval(int64_t n, int64_t* n_train, int64_t* n_eval) {
  if (n < 0) throw std::invalid_argument("sample count must be >= 0");
  *n_train = (9 * n) / 10;
  *n_eval = n - *n_train;
}

int64_t SignalGeometry::bytes_per_token() const {
  return static_cast<int64_t>(layers_tapped) * hidden_dim * bytes_per_element;
}

void SignalGeometry::validate() const {
  Problems p("invalid signal geometry");
  p.check(hidden_dim > 0, "hidden_dim must be > 0");
  p.check(layers_tapped > 0 && layers_tapped <= 8, "layers_tapped must be in [1, 8]");
  p.check(bytes_per_element > 0, "bytes_per_element must be > 0");
  p.throw_if_any();
}

static inline uint16_t bf16_rne(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

void synth_capture(uint64_t seed, int64_t index, int length, int vocab, int hidden, int layers,
                   double alpha, int gamma, int32_t* ids, uint16_t* features,
                   int32_t* accept_lengths, int32_t* n_steps, double* alpha_s) {
  Problems p("synth_capture");
  p.check(length >= 1, "length must be >= 1");
  p.check(vocab >= 1, "vocab must be >= 1");
  p.check(hidden >= 1 && layers >= 1, "hidden and layers must be >= 1");
  p.throw_if_any();
  bk::Rng rng(seed + static_cast<uint64_t>(index));
  int total = 0, steps = 0;
  while (total < length) {
    int k = bk::sample_accept_length(rng, alpha, gamma);
    k = std::min(k, length - total);  // request completes mid-step
    if (accept_lengths) accept_lengths[steps] = k;
    total += k;
    ++steps;
  }
  if (n_steps) *n_steps = steps;
  if (alpha_s)
    *alpha_s = bk::alpha_from_accept_length(static_cast<double>(length) / steps, gamma);
  for (int i = 0; i < length; ++i) {
    const auto id = static_cast<int32_t>(std::floor(rng.uniform() * vocab));
    if (ids) ids[i] = id;
  }
  if (features) {
    const int64_t n = static_cast<int64_t>(length) * layers * hidden;
    for (int64_t i = 0; i < n; ++i)
      features[i] = bf16_rne(static_cast<float>(rng.normal(0.0, 1.0)));
  }
}

}  // namespace specsim

// ================================================================== C ABI
using namespace specsim;

struct specsim_rng {
  bk::Rng r;
};

extern "C" {

int specsim_rng_create(uint64_t seed, specsim_rng** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is null");
    *out = new specsim_rng{bk::Rng(seed)};
  });
}
int specsim_rng_destroy(specsim_rng* r) {
  return guard([&] { delete r; });
}
int specsim_rng_uniform(specsim_rng* r, double* out) {
  return guard([&] { *out = r->r.uniform(); });
}
int specsim_rng_normal(specsim_rng* r, double mean, double sd, double* out) {
  return guard([&] { *out = r->r.normal(mean, sd); });
}
int specsim_rng_geometric(specsim_rng* r, double mean, int64_t* out) {
  return guard([&] { *out = r->r.geometric(mean); });
}
int specsim_rng_next_u64(specsim_rng* r, uint64_t* out) {
  return guard([&] { *out = r->r.next_u64(); });
}
int specsim_expected_accept_length(double alpha, int32_t gamma, double* out) {
  return guard([&] { *out = bk::expected_accept_length(alpha, gamma); });
}
int specsim_sample_accept_length(specsim_rng* r, double alpha, int32_t gamma, int32_t* out) {
  return guard([&] { *out = bk::sample_accept_length(r->r, alpha, gamma); });
}
int specsim_alpha_from_accept_length(double ell, int32_t gamma, double* out) {
  return guard([&] { *out = bk::alpha_from_accept_length(ell, gamma); });
}
int specsim_current_alpha(double alpha_start, double alpha_ceiling, double tau_samples,
                          double trained_samples, double* out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output");
    *out = bk::current_alpha(alpha_start, alpha_ceiling, tau_samples, trained_samples);
  });
}
int specsim_split_train_eval(int64_t n, int64_t* n_train, int64_t* n_eval) {
  return guard([&] { split_train_eval(n, n_train, n_eval); });
}
int specsim_bytes_per_token(const specsim_signal_geometry* g, int64_t* out) {
  return guard([&] {
    SignalGeometry geo{g->hidden_dim, g->layers_tapped, g->bytes_per_element};
    geo.validate();
    *out = geo.bytes_per_token();
  });
}
int specsim_dp_shard(int64_t n_items, int32_t per_rank, int32_t world, int32_t rank,
                     int64_t step, int64_t* out_idx, int32_t* out_n) {
  return guard([&] {
    Problems p("dp_shard");
    p.check(n_items >= 0, "n_items must be >= 0");
    p.check(per_rank >= 1, "per_rank must be >= 1");
    p.check(world >= 1 && rank >= 0 && rank < world, "rank must be in [0, world)");
    p.check(step >= 0, "step must be >= 0");
    p.check(out_n != nullptr, "out_n is null");
    p.throw_if_any();
    // step k covers items [k*per_rank*world, (k+1)*per_rank*world); item i of
    // that slice goes to rank i mod world
    const int64_t s0 = step * per_rank * static_cast<int64_t>(world);
    int32_t n = 0;
    for (int64_t i = s0 + rank; i < std::min<int64_t>(n_items, s0 + per_rank * static_cast<int64_t>(world));
         i += world) {
      if (out_idx) out_idx[n] = i;
      ++n;
    }
    *out_n = n;
  });
}

int specsim_synth_capture(uint64_t seed, int64_t index, int32_t length, int32_t vocab,
                          int32_t hidden, int32_t layers, double alpha, int32_t gamma,
                          int32_t* ids, uint16_t* features, int32_t* accept_lengths,
                          int32_t* n_steps, double* alpha_s) {
  return guard([&] {
    synth_capture(seed, index, length, vocab, hidden, layers, alpha, gamma, ids, features,
                  accept_lengths, n_steps, alpha_s);
  });
}

}  // extern "C"
