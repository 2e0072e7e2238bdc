// tide_loop: Algorithm 1 of TIDE (SPEC.md adapt_control)
// run end to end on one B200 with the real draft trainer behind train(job)
// (SURVEY §8(f) row 4): measured training durations and a measured serving
// acceptance rate instead of the reference's analytic samples_per_hour and
// current_alpha law (workload.cpp:41-47).
//
// Synthetic serving world (host code, C++ like the reference simulator):
//   * a "domain" is a token process over an active vocabulary subset: the
//     next token follows a fixed random successor map with probability
//     1 - noise, else a random active token;
//   * the serving draft's per-token acceptance alpha is MEASURED: top-1
//     accuracy of the deployed draft on a held-out probe set of the current
//     domain (DraftTrainer::eval), re-measured after every deployment and at
//     the domain shift;
//   * each request's verify steps draw accept lengths k with
//     sample_accept_length(alpha, gamma) (perf_model.cpp:171-177, bit-exact
//     Rng) until the request's tokens are covered; its label is
//     alpha_from_accept_length(mean k);
//   * the controller observes every label, stores captured requests while
//     collection is on (extract_signals into the HBM ring), and triggers
//     train(job) at n_threshold; the deploy gate compares alpha_eval (top-1
//     on D_eval) with the mean label of D_train.
//
// Phases: pre-train the initial draft on domain A, serve domain A, shift to
// domain B (the drift that makes the short EMA fall below the long one and
// switches collection on), keep serving.  One JSON line per event on stdout,
// a summary line last.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "specsim/draft_trainer.hpp"
#include "specsim_draft_trainer.h"

using namespace specsim;

namespace {
// The reference's Rng / accept-length model (rng.hpp:13-39,
// perf_model.cpp:171-177, 213-224) through the library's C ABI: the C++
// header does not redeclare those reference names.
void ok(int status) {
  if (status != SPECSIM_OK) throw std::runtime_error(specsim_last_error());
}
class Rng {
 public:
  explicit Rng(uint64_t seed) { ok(specsim_rng_create(seed, &r_)); }
  ~Rng() { specsim_rng_destroy(r_); }
  Rng(const Rng&) = delete;
  Rng& operator=(const Rng&) = delete;
  double uniform() {
    double u = 0;
    ok(specsim_rng_uniform(r_, &u));
    return u;
  }
  double normal(double mean, double sd) {
    double v = 0;
    ok(specsim_rng_normal(r_, mean, sd, &v));
    return v;
  }
  specsim_rng* get() { return r_; }

 private:
  specsim_rng* r_ = nullptr;
};
int sample_accept_length(Rng& rng, double alpha, int gamma) {
  int32_t k = 0;
  ok(specsim_sample_accept_length(rng.get(), alpha, gamma, &k));
  return k;
}
double alpha_from_accept_length(double ell, int gamma) {
  double a = 0;
  ok(specsim_alpha_from_accept_length(ell, gamma, &a));
  return a;
}
}  // namespace

namespace {

struct Args {
  int requests = 1500;   // per phase
  int threshold = 256;   // n_threshold
  int epochs = 4;
  int pretrain = 300;    // optimiser steps of the initial draft on domain A
  int active = 512;      // active vocabulary per domain
  double noise = 0.05;
  int gamma = 3;
  uint64_t seed = 20260217;
  int device = 0;
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const char* v = argv[i + 1];
    if (k == "--requests") a.requests = std::atoi(v);
    else if (k == "--threshold") a.threshold = std::atoi(v);
    else if (k == "--epochs") a.epochs = std::atoi(v);
    else if (k == "--pretrain") a.pretrain = std::atoi(v);
    else if (k == "--active") a.active = std::atoi(v);
    else if (k == "--noise") a.noise = std::atof(v);
    else if (k == "--seed") a.seed = std::strtoull(v, nullptr, 10);
    else if (k == "--device") a.device = std::atoi(v);
    else throw std::invalid_argument("unknown option " + k);
  }
  return a;
}

uint16_t bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// A token process: active ids and a successor map.
struct Domain {
  std::vector<int32_t> ids;
  std::vector<int32_t> next;  // indexed by vocabulary id (-1 outside the domain)
  double noise;
  Domain(Rng& rng, int vocab, int active, double noise_) : next(vocab, -1), noise(noise_) {
    std::vector<int32_t> all(vocab);
    for (int i = 0; i < vocab; ++i) all[i] = i;
    for (int i = vocab - 1; i > 0; --i)
      std::swap(all[i], all[static_cast<int>(rng.uniform() * (i + 1))]);
    ids.assign(all.begin(), all.begin() + active);
    std::vector<int32_t> perm = ids;
    for (int i = active - 1; i > 0; --i)
      std::swap(perm[i], perm[static_cast<int>(rng.uniform() * (i + 1))]);
    for (int i = 0; i < active; ++i) next[ids[i]] = perm[i];
  }
  int32_t any(Rng& rng) const { return ids[static_cast<int>(rng.uniform() * ids.size())]; }
  void tokens(Rng& rng, int L, int32_t* out) const {
    out[0] = any(rng);
    for (int i = 1; i < L; ++i) out[i] = rng.uniform() < noise ? any(rng) : next[out[i - 1]];
  }
};

struct World {
  Args a;
  DraftShape shape;
  int L;  // tokens per request
  Rng rng;
  HiddenStateBuffer buf;
  DraftTrainer trainer;
  AdaptiveController ctrl;
  int64_t next_id = 0;
  std::vector<int32_t> ids;
  std::vector<uint16_t> feats;
  std::vector<int64_t> probe;  // held-out probe samples of the current domain
  double alpha_serving = 0;
  double t0;

  static DraftShape c1() {
    DraftShape s;  // BASELINE config C1 (tiny draft head)
    s.hidden = 256;
    s.vocab = 4096;
    s.seq_len = 128;
    s.n_heads = 4;
    s.n_kv_heads = 2;
    s.head_dim = 64;
    s.ffn = 1024;
    s.micro_batch = 8;
    return s;
  }
  static AdamWConfig opt() {
    AdamWConfig o;
    o.lr = 3e-3f;
    return o;
  }
  explicit World(const Args& args)
      : a(args),
        shape(c1()),
        L(shape.seq_len + 2),
        rng(args.seed),
        buf(SignalGeometry{shape.hidden, 3, 2},
            int64_t(args.threshold + 320) * 4 * (c1().seq_len + 2),
            0, args.device),
        trainer(shape, opt(), args.seed, 0, 1, nullptr, args.device),
        ctrl(ControllerConfig{0.9, 0.99, 0.05, 32, args.threshold}),
        ids(L),
        feats(static_cast<size_t>(L) * 3 * shape.hidden) {
    t0 = now();
  }
  static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  }

  // one captured request of the domain, appended to the ring as sample `id`
  void capture(const Domain& d, int64_t id, double alpha) {
    d.tokens(rng, L, ids.data());
    for (auto& f : feats) f = bf16(static_cast<float>(rng.normal(0.0, 1.0)));
    buf.append_packed(id, alpha, feats.data(), ids.data(), L, 0);
  }

  double measure_alpha() {
    double correct = 0, valid = 0;
    for (size_t i = 0; i < probe.size(); i += shape.micro_batch) {
      const int n = static_cast<int>(std::min<size_t>(shape.micro_batch, probe.size() - i));
      const StepResult r = trainer.eval(buf, probe.data() + i, n);
      correct += static_cast<double>(r.top1_correct);
      valid += static_cast<double>(r.valid_tokens);
    }
    return valid > 0 ? correct / valid : 0.0;
  }

  void new_probe(const Domain& d) {
    probe.clear();
    for (int i = 0; i < 2 * shape.micro_batch; ++i) {
      const int64_t id = next_id++;
      capture(d, id, 0.0);
      probe.push_back(id);
    }
  }

  void event(const char* kind, const std::string& extra) {
    std::printf("{\"event\": \"%s\", \"t_s\": %.3f, \"observation\": %lld, \"alpha_serving\": %.4f%s}\n",
                kind, now() - t0, static_cast<long long>(ctrl.observations()), alpha_serving,
                extra.c_str());
    std::fflush(stdout);
  }

  void pretrain(const Domain& d) {
    std::vector<int64_t> pool;
    for (int i = 0; i < 32 * shape.micro_batch; ++i) {  // 256 captured requests
      const int64_t id = next_id++;
      capture(d, id, 0.0);
      pool.push_back(id);
    }
    TrainJob job;
    for (int s = 0; s < a.pretrain; ++s)
      for (int b = 0; b < shape.micro_batch; ++b)
        job.train_ids.push_back(pool[(s * shape.micro_batch + b) % pool.size()]);
    const TrainingOutcome o = trainer.train(buf, job);
    alpha_serving = measure_alpha();
    char x[160];
    std::snprintf(x, sizeof x, ", \"steps\": %lld, \"duration_s\": %.3f, \"mean_loss\": %.4f",
                  static_cast<long long>(o.steps), o.duration_hours * 3600.0, o.mean_loss);
    event("pretrain", x);
  }

  // one request: verify steps with accept lengths drawn at the serving alpha
  void serve(const Domain& d, int phase) {
    int covered = 0, steps = 0;
    while (covered < L) {
      covered += sample_accept_length(rng, alpha_serving, a.gamma);
      ++steps;
    }
    const double mean_k = static_cast<double>(L) / steps;  // last step truncated
    const double label = alpha_from_accept_length(std::min(mean_k, a.gamma + 1.0), a.gamma);
    const bool was_on = ctrl.collection_enabled();
    ctrl.observe(label);
    if (!was_on && ctrl.collection_enabled()) event("collect_on", "");
    const int64_t id = next_id++;
    if (ctrl.record_sample(id, label)) capture(d, id, label);
    const TriggerDecision dec = ctrl.maybe_trigger_training(trainer, buf, a.epochs);
    if (!dec.triggered) return;
    const double before = alpha_serving;
    if (dec.action == 1) alpha_serving = measure_alpha();
    char x[320];
    std::snprintf(x, sizeof x,
                  ", \"phase\": %d, \"n_train\": %lld, \"n_eval\": %lld, \"alpha_train\": %.4f, "
                  "\"alpha_eval\": %.4f, \"duration_s\": %.3f, \"steps\": %lld, "
                  "\"mean_loss\": %.4f, \"action\": \"%s\", \"draft_version\": %lld, "
                  "\"alpha_serving_before\": %.4f",
                  phase, static_cast<long long>(dec.n_train), static_cast<long long>(dec.n_eval),
                  dec.alpha_train, dec.outcome.alpha_eval, dec.outcome.duration_hours * 3600.0,
                  static_cast<long long>(dec.outcome.steps), dec.outcome.mean_loss,
                  dec.action == 1 ? "deploy" : (dec.action == 0 ? "tie" : "reject"),
                  static_cast<long long>(ctrl.draft_version()), before);
    event("train", x);
  }
};

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    World w(a);
    Rng dom_rng(a.seed + 7);
    const Domain A(dom_rng, w.shape.vocab, a.active, a.noise);
    const Domain B(dom_rng, w.shape.vocab, a.active, a.noise);
    w.new_probe(A);
    w.pretrain(A);
    for (int i = 0; i < a.requests; ++i) w.serve(A, 0);
    // distribution shift: the deployed draft now serves domain B
    w.new_probe(B);
    w.alpha_serving = w.measure_alpha();
    w.event("domain_shift", "");
    for (int i = 0; i < a.requests; ++i) w.serve(B, 1);
    std::printf(
        "{\"summary\": true, \"observations\": %lld, \"draft_version\": %lld, "
        "\"alpha_serving\": %.4f, \"collection_enabled\": %s, \"events\": %zu}\n",
        static_cast<long long>(w.ctrl.observations()), static_cast<long long>(w.ctrl.draft_version()),
        w.alpha_serving, w.ctrl.collection_enabled() ? "true" : "false", w.ctrl.events().size());
    return 0;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "runtime error: %s\n", e.what());
    return 3;
  }
}
