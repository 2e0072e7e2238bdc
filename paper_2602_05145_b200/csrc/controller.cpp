// Algorithm 1 of TIDE as specified by SPEC.md's
// adapt_control module: the dual-EMA collection gate (Eq. 6), the sample
// store, and maybe_trigger_training -- the caller of train(job) -- with the
// deploy-if-improved gate.  Host-only double-precision logic, compiled with
// -ffp-contract=off so the recurrences round exactly like the SPEC's
// restatement in oracle/controller.py.
#include <cmath>
#include <stdexcept>

#include "common.h"
#include "handles.h"
#include "specsim/draft_trainer.hpp"

namespace specsim {

void ControllerConfig::validate() const {
  Problems p("invalid controller config");
  p.check(lambda_short > 0 && lambda_short < 1, "lambda_short must be in (0, 1)");
  p.check(lambda_long > 0 && lambda_long < 1, "lambda_long must be in (0, 1)");
  // SPEC adapt_control ControllerState invariant: the long average decays slower
  p.check(lambda_long > lambda_short, "lambda_long must be > lambda_short");
  p.check(epsilon > 0 && std::isfinite(epsilon), "epsilon must be > 0");
  p.check(n_init > 0, "n_init must be > 0");
  // the 9:1 split must leave D_train non-empty (floor(9n/10) >= 1)
  p.check(n_threshold >= 2, "n_threshold must be >= 2");
  p.throw_if_any<ConfigError>();
}

AdaptiveController::AdaptiveController(const ControllerConfig& cfg) : cfg_(cfg) {
  cfg_.validate();
}

namespace {
void check_alpha(double a) {
  if (!(a >= 0.0 && a <= 1.0)) throw std::invalid_argument("alpha must be in [0, 1]");
}
}  // namespace

void AdaptiveController::observe(double alpha) {
  check_alpha(alpha);
  observations_ += 1;
  if (!initialized_) {
    // init_from_warmup: both EMAs = arithmetic mean of the first n_init
    // observations (summed in arrival order); collection starts disabled
    warmup_.push_back(alpha);
    if (static_cast<int64_t>(warmup_.size()) == cfg_.n_init) {
      double s = 0.0;
      for (double a : warmup_) s += a;
      ema_short_ = ema_long_ = s / static_cast<double>(cfg_.n_init);
      initialized_ = true;
      warmup_.clear();
    }
    return;
  }
  // Eq. 6 (Algorithm 1): a <- lambda a + (1 - lambda) alpha, both averages,
  // evaluated as a + (1 - lambda)(alpha - a) so a constant stream leaves the
  // averages exactly unchanged (SPEC adapt_control observe example 1)
  ema_short_ = ema_short_ + (1.0 - cfg_.lambda_short) * (alpha - ema_short_);
  ema_long_ = ema_long_ + (1.0 - cfg_.lambda_long) * (alpha - ema_long_);
  // epsilon gap: never set False here (SPEC adapt_control observe post)
  if (!collection_enabled_ && ema_short_ < ema_long_ - cfg_.epsilon) {
    collection_enabled_ = true;
    events_.push_back({ControllerEventKind::COLLECT_ON, observations_});
  }
}

bool AdaptiveController::record_sample(int64_t sample_id, double alpha) {
  if (!collection_enabled_) return false;  // no-op, not an error
  check_alpha(alpha);
  pending_ids_.push_back(sample_id);
  pending_alpha_.push_back(alpha);
  return true;
}

TriggerDecision AdaptiveController::maybe_trigger_training(DraftTrainer& trainer,
                                                           HiddenStateBuffer& buf, int epochs) {
  TriggerDecision d;
  if (stored_samples() < cfg_.n_threshold) return d;
  // Samples the ring has evicted since they were recorded can never be
  // trained on: drop them (keeping order) instead of failing every later
  // trigger on the same ids; collection continues until the threshold is
  // met with resident samples.
  {
    size_t w = 0;
    for (size_t i = 0; i < pending_ids_.size(); ++i) {
      bool resident = true;
      try {
        buf.sample(pending_ids_[i]);
      } catch (const std::out_of_range&) {
        resident = false;
      }
      if (!resident) continue;
      pending_ids_[w] = pending_ids_[i];
      pending_alpha_[w] = pending_alpha_[i];
      ++w;
    }
    pending_ids_.resize(w);
    pending_alpha_.resize(w);
  }
  const int64_t n = stored_samples();
  if (n < cfg_.n_threshold) return d;
  // chronological 9:1 split: oldest 90% train
  split_train_eval(n, &d.n_train, &d.n_eval);
  TrainJob job;
  job.epochs = epochs;
  job.train_ids.assign(pending_ids_.begin(), pending_ids_.begin() + d.n_train);
  job.eval_ids.assign(pending_ids_.begin() + d.n_train, pending_ids_.end());
  double s = 0.0;
  for (int64_t i = 0; i < d.n_train; ++i) s += pending_alpha_[static_cast<size_t>(i)];
  d.alpha_train = d.n_train > 0 ? s / static_cast<double>(d.n_train) : 0.0;

  // M_new <- train(M_draft, D_train) on a copy: the trainer trains in place,
  // so the deployed model is snapshotted first and restored unless deployed
  trainer.snapshot();
  try {
    d.outcome = trainer.train(buf, job);
  } catch (...) {
    // trainer failure: controller state, pending set and model unchanged
    try {
      trainer.restore();
    } catch (...) {
    }
    throw;
  }
  d.triggered = true;
  events_.push_back({ControllerEventKind::TRAIN_TRIGGER, observations_});
  if (d.outcome.alpha_eval > d.alpha_train) {
    draft_version_ += 1;
    d.action = 1;
    events_.push_back({ControllerEventKind::DEPLOY, observations_});
  } else {
    trainer.restore();
    if (d.outcome.alpha_eval < d.alpha_train) {
      d.action = -1;
      events_.push_back({ControllerEventKind::REJECT, observations_});
      if (collection_enabled_) {
        collection_enabled_ = false;
        events_.push_back({ControllerEventKind::COLLECT_OFF, observations_});
      }
    } else {
      d.action = 0;  // tie: keep collecting, do not deploy (SPEC design decision)
    }
  }
  pending_ids_.clear();
  pending_alpha_.clear();
  return d;
}

}  // namespace specsim

// ================================================================== C ABI
using namespace specsim;

struct specsim_controller {
  AdaptiveController* c;
};

extern "C" {

int specsim_controller_create(const specsim_controller_config* cfg, specsim_controller** out) {
  return guard([&] {
    if (!cfg || !out) throw std::invalid_argument("null argument");
    ControllerConfig c{cfg->lambda_short, cfg->lambda_long, cfg->epsilon, cfg->n_init,
                       cfg->n_threshold};
    *out = new specsim_controller{new AdaptiveController(c)};
  });
}

void specsim_controller_destroy(specsim_controller* c) {
  if (!c) return;
  delete c->c;
  delete c;
}

int specsim_controller_observe(specsim_controller* c, double alpha) {
  return guard([&] { c->c->observe(alpha); });
}

int specsim_controller_record_sample(specsim_controller* c, int64_t sample_id, double alpha,
                                     int32_t* stored) {
  return guard([&] {
    const bool s = c->c->record_sample(sample_id, alpha);
    if (stored) *stored = s ? 1 : 0;
  });
}

int specsim_controller_maybe_trigger_training(specsim_controller* c, specsim_trainer* t,
                                              specsim_hsbuf* buf, int32_t epochs,
                                              specsim_trigger_decision* out) {
  return guard([&] {
    if (!t || !buf || !out) throw std::invalid_argument("null argument");
    const TriggerDecision d = c->c->maybe_trigger_training(*t->t, *buf->b, epochs);
    out->triggered = d.triggered ? 1 : 0;
    out->action = d.action;
    out->alpha_train = d.alpha_train;
    out->n_train = d.n_train;
    out->n_eval = d.n_eval;
    out->outcome = specsim_training_outcome{d.outcome.duration_hours, d.outcome.alpha_eval,
                                            d.outcome.new_version, d.outcome.mean_loss,
                                            d.outcome.steps};
  });
}

int specsim_controller_state_get(const specsim_controller* c, specsim_controller_state* out) {
  return guard([&] {
    const AdaptiveController& a = *c->c;
    *out = specsim_controller_state{a.initialized() ? 1 : 0,
                                    a.collection_enabled() ? 1 : 0,
                                    a.ema_short(),
                                    a.ema_long(),
                                    a.stored_samples(),
                                    a.draft_version(),
                                    a.observations(),
                                    static_cast<int64_t>(a.events().size())};
  });
}

int specsim_controller_events(const specsim_controller* c, int32_t* kinds, int64_t* at,
                              int64_t cap, int64_t* n) {
  return guard([&] {
    const auto& ev = c->c->events();
    const int64_t m = static_cast<int64_t>(ev.size());
    for (int64_t i = 0; i < m && i < cap; ++i) {
      if (kinds) kinds[i] = static_cast<int32_t>(ev[static_cast<size_t>(i)].kind);
      if (at) at[i] = ev[static_cast<size_t>(i)].observation;
    }
    if (n) *n = m;
  });
}

}  // extern "C"
