// sim_serving: the SPEC's discrete-event serving engine (SPEC.md sim_serving,
// step / adaptive_drafter_decide / extract_signals / run) --
// specified by the reference but not shipped -- built ON the reference's own
// simulator code and driving this repo's real trainer behind train(job)
// (SURVEY §8(f) row 4):
//
//   reference, compiled in place from /root/reference/proj (never copied):
//     LatencyProfile (T(n), D0), SpeculationConfig, practical_speedup,
//     sample_accept_length, alpha_from_accept_length, Rng      (perf_model.cpp)
//     PhaseSpec, WorkloadScript, ScriptCursor, refill_batch     (workload.cpp)
//   this repo (libspecsim_draft.so, proj/include/specsim/draft_trainer.hpp):
//     HiddenStateBuffer (extract_signals into the HBM ring), DraftTrainer
//     (train(job) on the B200), AdaptiveController (Algorithm 1)
//
// The simulated clock advances by the profile's iteration latency (SPEC step:
// speculation on -> gamma D0 + T(b (gamma + 1)), off -> T(b)); the trainer is
// the second actor of SPEC.md:436: a training job triggered at clock t
// deploys at t + its MEASURED duration (a timestamped deploy event), and the
// serving acceptance after a deploy is MEASURED (top-1 of the deployed draft
// on a held-out probe of each phase's token domain), replacing the analytic
// current_alpha law (workload.cpp:41-47).  Requests of phase p draw their
// tokens from synthetic domain p (phase 1 is the drift that switches
// collection on).
//
// Modes (SPEC run): tide_adaptive | tide_default | speculation_off |
// speculation_on_no_training.  Output: --emit-iterations writes the RunMetrics
// CSV (SPEC External Interfaces, columns in the SPEC's order) to stdout
// before one JSON summary line.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "specsim/errors.hpp"
#include "specsim/perf_model.hpp"
#include "specsim/rng.hpp"
#include "specsim/workload.hpp"
#include "specsim/draft_trainer.hpp"

using namespace specsim;

namespace {

struct Args {
  std::string mode = "tide_adaptive";
  std::string profile;  // CSV in the reference's format (LatencyProfile::from_csv)
  int requests = 400;   // per phase
  int concurrency = 8;
  int mean_tokens = 130;
  double jitter_sd = 0.02;
  int threshold = 128;
  int epochs = 4;
  int pretrain = 200;
  int active = 512;
  double noise = 0.05;
  int collect = 1;  // speculation_on_no_training: capture signals (never train)
  int emit = 0;
  uint64_t seed = 20260217;
  int device = 0;
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const char* v = argv[i + 1];
    if (k == "--mode") a.mode = v;
    else if (k == "--profile") a.profile = v;
    else if (k == "--requests") a.requests = std::atoi(v);
    else if (k == "--concurrency") a.concurrency = std::atoi(v);
    else if (k == "--mean-tokens") a.mean_tokens = std::atoi(v);
    else if (k == "--jitter") a.jitter_sd = std::atof(v);
    else if (k == "--threshold") a.threshold = std::atoi(v);
    else if (k == "--epochs") a.epochs = std::atoi(v);
    else if (k == "--pretrain") a.pretrain = std::atoi(v);
    else if (k == "--collect") a.collect = std::atoi(v);
    else if (k == "--emit-iterations") a.emit = std::atoi(v);
    else if (k == "--seed") a.seed = std::strtoull(v, nullptr, 10);
    else if (k == "--device") a.device = std::atoi(v);
    else throw ConfigError("unknown option " + k);
  }
  if (a.mode != "tide_adaptive" && a.mode != "tide_default" && a.mode != "speculation_off" &&
      a.mode != "speculation_on_no_training")
    throw ConfigError("unknown mode " + a.mode);
  if (a.profile.empty()) throw ConfigError("--profile is required");
  return a;
}

uint16_t bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// A token process: active ids and a fixed successor map, followed with
// probability 1 - noise (the draft can learn it from the embeddings).
struct Domain {
  std::vector<int32_t> ids, next;
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

DraftShape c1() {  // BASELINE config C1 (tiny draft head)
  DraftShape s;
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

struct Engine {
  Args a;
  LatencyProfile profile;
  SpeculationConfig spec;
  DraftShape shape = c1();
  bool train_mode, spec_always, spec_never;
  Rng rng;        // accept-length draws (the reference's Rng)
  Rng data_rng;   // synthetic token streams / features
  HiddenStateBuffer buf;        // serving captures (D_train / D_eval)
  HiddenStateBuffer probe_buf;  // held-out probes + the initial draft's pre-training pool
  DraftTrainer trainer;
  AdaptiveController ctrl;
  std::vector<Domain> domains;
  std::vector<std::vector<int64_t>> probes;  // held-out probe samples per domain
  std::vector<double> alpha_dom;             // serving acceptance per domain (measured)
  std::vector<double> pending_alpha;         // measured for the next deploy event
  double deploy_at = -1;                     // simulated time of the pending deploy
  int64_t next_id = 1000000;
  // per live request: emitted tokens of its speculative steps (the last one
  // truncated at the request's end)
  std::unordered_map<int, std::vector<int>> accepts;
  // EngineState / RunMetrics
  double clock = 0;
  bool speculation_enabled;
  int64_t tokens = 0, iterations = 0, spec_iterations = 0, collect_iterations = 0;
  int64_t trainings = 0, deploys = 0, rejects = 0;
  double train_ms_total = 0;
  std::vector<double> phase_tokens, phase_ms;
  std::string train_log;  // JSON objects of the training jobs
  double wall0;

  Engine(const Args& args, const WorkloadScript& script)
      : a(args),
        profile(LatencyProfile::from_csv(args.profile)),
        train_mode(args.mode == "tide_adaptive" || args.mode == "tide_default"),
        spec_always(args.mode == "tide_default" || args.mode == "speculation_on_no_training"),
        spec_never(args.mode == "speculation_off"),
        rng(args.seed),
        data_rng(args.seed + 11),
        buf(SignalGeometry{c1().hidden, 3, 2},
            int64_t(args.threshold) * 3 * 8 * std::max(args.mean_tokens, 16), 0, args.device),
        probe_buf(SignalGeometry{c1().hidden, 3, 2}, int64_t(64 * 8 + 64) * (c1().seq_len + 2),
                  0, args.device),
        trainer(c1(), opt(), args.seed, 0, 1, nullptr, args.device),
        ctrl(ControllerConfig{0.9, 0.99, 0.05, 32, args.threshold}) {
    spec.validate();
    speculation_enabled = spec.initial_on;
    const int phases = static_cast<int>(script.phases().size());
    Rng dom_rng(args.seed + 7);
    for (int p = 0; p < phases; ++p) domains.emplace_back(dom_rng, shape.vocab, a.active, a.noise);
    probes.resize(phases);
    alpha_dom.assign(phases, 0.0);
    phase_tokens.assign(phases, 0.0);
    phase_ms.assign(phases, 0.0);
    wall0 = now();
  }
  static AdamWConfig opt() {
    AdamWConfig o;
    o.lr = 3e-3f;
    return o;
  }
  static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  }

  // captured hidden states of one request of domain d (synthetic features,
  // the domain's tokens), appended as sample `id`: extract_signals +
  // record_sample of SPEC.md:267-275 / 341-344 into the device ring
  void capture(HiddenStateBuffer& into, int d, int64_t id, int L, double alpha) {
    std::vector<int32_t> ids(L);
    domains[d].tokens(data_rng, L, ids.data());
    std::vector<uint16_t> f(static_cast<size_t>(L) * 3 * shape.hidden);
    for (auto& x : f) x = bf16(static_cast<float>(data_rng.normal(0.0, 1.0)));
    into.append_packed(id, alpha, f.data(), ids.data(), L, 0);
  }

  double measure(int d) {
    double correct = 0, valid = 0;
    const auto& p = probes[d];
    for (size_t i = 0; i < p.size(); i += shape.micro_batch) {
      const int n = static_cast<int>(std::min<size_t>(shape.micro_batch, p.size() - i));
      const StepResult r = trainer.eval(probe_buf, p.data() + i, n);
      correct += static_cast<double>(r.top1_correct);
      valid += static_cast<double>(r.valid_tokens);
    }
    return valid > 0 ? correct / valid : 0.0;
  }
  std::vector<double> measure_all() {
    std::vector<double> r(domains.size());
    for (size_t d = 0; d < domains.size(); ++d) r[d] = measure(static_cast<int>(d));
    return r;
  }

  void setup() {
    const int L = shape.seq_len + 2;
    for (size_t d = 0; d < domains.size(); ++d)
      for (int i = 0; i < 2 * shape.micro_batch; ++i) {
        const int64_t id = next_id++;
        capture(probe_buf, static_cast<int>(d), id, L, 0.0);
        probes[d].push_back(id);
      }
    if (a.pretrain > 0 && !spec_never) {  // the initial draft: trained on phase 0's domain
      std::vector<int64_t> pool;
      for (int i = 0; i < 32 * shape.micro_batch; ++i) {
        const int64_t id = next_id++;
        capture(probe_buf, 0, id, L, 0.0);
        pool.push_back(id);
      }
      TrainJob job;
      for (int s = 0; s < a.pretrain; ++s)
        for (int b = 0; b < shape.micro_batch; ++b)
          job.train_ids.push_back(pool[(s * shape.micro_batch + b) % pool.size()]);
      trainer.train(probe_buf, job);
    }
    alpha_dom = measure_all();
  }

  // SPEC adaptive_drafter_decide: practical_speedup at the monitored alpha
  // (the controller's short-term EMA) and batch b against 1 + margin
  bool decide(int b) const {
    if (spec_never) return false;
    if (spec_always) return true;
    if (!ctrl.initialized()) return spec.initial_on;
    return practical_speedup(profile, ctrl.ema_short(), spec.gamma, b) >
           1.0 + spec.hysteresis_margin;
  }

  // one finished request: its acceptance label feeds Algorithm 1
  void finish(const Request& r) {
    auto it = accepts.find(r.id);
    if (it == accepts.end()) return;  // never speculated: no acceptance signal
    const auto& ks = it->second;
    long long sum = 0;
    for (int k : ks) sum += k;
    const double mean_k = static_cast<double>(sum) / static_cast<double>(ks.size());
    const double label = alpha_from_accept_length(std::min(mean_k, spec.gamma + 1.0), spec.gamma);
    accepts.erase(it);
    ctrl.observe(label);
    const bool collect = train_mode || a.collect;
    if (!collect) return;
    const int64_t id = next_id++;
    // extract_signals: every token the request emitted while speculating
    // (the trainer cuts samples longer than S + 2 in its gather)
    if (ctrl.record_sample(id, label)) capture(buf, r.phase_index, id, static_cast<int>(sum), label);
    if (!train_mode || deploy_at >= 0) return;  // one job in flight
    const TriggerDecision dec = ctrl.maybe_trigger_training(trainer, buf, a.epochs);
    if (!dec.triggered) return;
    ++trainings;
    const double dur_ms = dec.outcome.duration_hours * 3.6e6;
    train_ms_total += dur_ms;
    if (dec.action == 1) {
      ++deploys;
      pending_alpha = measure_all();  // the deployed draft, served from clock + duration
      deploy_at = clock + dur_ms;
    } else if (dec.action == -1) {
      ++rejects;
    }
    char x[400];
    std::snprintf(x, sizeof x,
                  "%s{\"clock_ms\": %.3f, \"phase\": %d, \"n_train\": %lld, \"alpha_train\": "
                  "%.4f, \"alpha_eval\": %.4f, \"duration_ms\": %.3f, \"action\": %d, "
                  "\"alpha_deployed\": [%.4f, %.4f]}",
                  train_log.empty() ? "" : ", ", clock, r.phase_index,
                  static_cast<long long>(dec.n_train), dec.alpha_train, dec.outcome.alpha_eval,
                  dur_ms, dec.action, dec.action == 1 ? pending_alpha[0] : -1.0,
                  dec.action == 1 && pending_alpha.size() > 1 ? pending_alpha[1] : -1.0);
    train_log += x;
  }

  // SPEC step: one decode iteration of the whole batch
  void step(std::vector<Request>& batch, const WorkloadScript& script, FILE* csv) {
    if (deploy_at >= 0 && clock >= deploy_at) {  // timestamped deploy event
      alpha_dom = pending_alpha;
      deploy_at = -1;
    }
    const int b = static_cast<int>(batch.size());
    speculation_enabled = decide(b);
    const double lat = speculation_enabled
                           ? spec.gamma * profile.d0_ms() + profile.latency_ms(b * (spec.gamma + 1.0))
                           : profile.latency_ms(b);
    int64_t emitted = 0;
    double accepted_sum = 0;
    for (Request& r : batch) {
      int k = 1;
      if (speculation_enabled) {
        const double alpha = std::clamp(alpha_dom[r.phase_index] + r.alpha_jitter, 0.0, 1.0);
        k = sample_accept_length(rng, alpha, spec.gamma);
        accepted_sum += k;
      }
      const long long take = std::min<long long>(k, r.output_tokens_remaining);
      if (speculation_enabled) accepts[r.id].push_back(static_cast<int>(take));
      r.output_tokens_remaining -= take;
      emitted += take;
    }
    clock += lat;
    tokens += emitted;
    ++iterations;
    spec_iterations += speculation_enabled ? 1 : 0;
    collect_iterations += ctrl.collection_enabled() ? 1 : 0;
    const int ph = batch.front().phase_index;
    phase_tokens[ph] += static_cast<double>(emitted);
    phase_ms[ph] += lat;
    for (const Request& r : batch)
      if (r.output_tokens_remaining <= 0) finish(r);
    if (csv) {
      const auto st = buf.stats();
      std::fprintf(csv, "%.6f,%d,%d,%.6f,%lld,%.6f,%d,%lld,%lld,%lld\n", clock, b,
                   speculation_enabled ? 1 : 0,
                   speculation_enabled ? accepted_sum / b : 1.0, static_cast<long long>(emitted),
                   1e3 * static_cast<double>(emitted) / lat, ctrl.collection_enabled() ? 1 : 0,
                   static_cast<long long>(st.bytes), static_cast<long long>(st.cumulative_bytes),
                   static_cast<long long>(ctrl.draft_version()));
    }
    (void)script;
  }
};

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    // SPEC run: a two-phase closed-loop script (domain A, then the drift to B)
    std::vector<PhaseSpec> phases(2);
    for (int p = 0; p < 2; ++p) {
      phases[p].name = p == 0 ? "domain_a" : "domain_b";
      phases[p].num_requests = a.requests;
      phases[p].concurrency = a.concurrency;
      phases[p].mean_output_tokens = a.mean_tokens;
      phases[p].alpha_start = 0.0;  // measured, not the analytic law
      phases[p].alpha_ceiling = 1.0;
      phases[p].tau_samples = 1.0;
      phases[p].alpha_noise_sd = a.jitter_sd;
    }
    const WorkloadScript script(phases, a.seed);
    Engine e(a, script);  // configuration errors before the clock starts
    e.setup();
    ScriptCursor cursor(script);
    std::vector<Request> batch;
    refill_batch(cursor, batch);
    FILE* csv = a.emit ? stdout : nullptr;
    if (csv)
      std::fprintf(csv,
                   "clock_ms,batch_size,speculation_on,mean_accept_length,tokens_emitted,"
                   "throughput_tokens_per_s,collection_on,buffer_bytes,cumulative_storage_bytes,"
                   "draft_version\n");
    double last = -1;
    while (!batch.empty()) {
      e.step(batch, script, csv);
      if (e.clock < last) throw std::logic_error("clock went backwards");
      last = e.clock;
      refill_batch(cursor, batch);
    }
    const auto st = e.buf.stats();
    std::printf(
        "{\"summary\": true, \"mode\": \"%s\", \"clock_ms\": %.6f, \"tokens\": %lld, "
        "\"script_tokens\": %lld, \"iterations\": %lld, \"throughput_tokens_per_s\": %.3f, "
        "\"phase_throughput\": [%.3f, %.3f], \"speculation_duty\": %.4f, "
        "\"collection_duty\": %.4f, \"flushes\": %lld, \"cumulative_storage_bytes\": %lld, "
        "\"buffer_bytes\": %lld, \"signal_records\": %lld, \"trainings\": %lld, \"deploys\": %lld, \"rejects\": %lld, "
        "\"train_ms\": %.3f, \"draft_version\": %lld, \"alpha_domain\": [%.4f, %.4f], "
        "\"wall_s\": %.3f, \"jobs\": [%s]}\n",
        a.mode.c_str(), e.clock, static_cast<long long>(e.tokens),
        static_cast<long long>(script.total_output_tokens()), static_cast<long long>(e.iterations),
        1e3 * static_cast<double>(e.tokens) / e.clock,
        e.phase_ms[0] > 0 ? 1e3 * e.phase_tokens[0] / e.phase_ms[0] : 0.0,
        e.phase_ms[1] > 0 ? 1e3 * e.phase_tokens[1] / e.phase_ms[1] : 0.0,
        static_cast<double>(e.spec_iterations) / e.iterations,
        static_cast<double>(e.collect_iterations) / e.iterations,
        static_cast<long long>(st.flushes), static_cast<long long>(st.cumulative_bytes),
        static_cast<long long>(st.bytes), static_cast<long long>(st.records),
        static_cast<long long>(e.trainings),
        static_cast<long long>(e.deploys), static_cast<long long>(e.rejects), e.train_ms_total,
        static_cast<long long>(e.ctrl.draft_version()), e.alpha_dom[0], e.alpha_dom[1],
        Engine::now() - e.wall0, e.train_log.c_str());
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
