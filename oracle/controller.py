"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Pure-Python restatement of Algorithm 1 as SPEC.md's
adapt_control module specifies it, used to check the library's
AdaptiveController bit-for-bit (same double-precision operation order):

* init_from_warmup -- SPEC.md:316-323: both EMAs = mean of the first N_init
  observations (summed in arrival order); collection starts disabled.
* observe -- SPEC.md:324-331 (Eq. 6): ema <- lambda ema + (1 - lambda) alpha for
  both averages (evaluated as ema + (1 - lambda)(alpha - ema)); collection_enabled := True when ema_short < ema_long - epsilon
  (never set False here).
* record_sample -- SPEC.md:332-336: store (handle, alpha) when enabled, else no-op.
* maybe_trigger_training -- SPEC.md:337-344: at >= N_threshold stored samples,
  chronological 9:1 split (oldest floor(9n/10) train), alpha_train =
  mean alpha of D_train, train; deploy iff alpha_eval > alpha_train, disable
  collection iff <, neither on a tie; pending cleared; a failing
  trainer leaves everything unchanged.
The reference ships no code for this module: parity rests on
the SPEC's examples (closed-form step-drop recurrence) and this
restatement.
"""
from __future__ import annotations


class Controller:
    def __init__(self, lambda_short=0.9, lambda_long=0.99, epsilon=0.05, n_init=32,
                 n_threshold=2048):
        self.ls, self.ll, self.eps = lambda_short, lambda_long, epsilon
        self.n_init, self.n_threshold = n_init, n_threshold
        self.initialized = False
        self.warmup = []
        self.ema_short = self.ema_long = 0.0
        self.collection_enabled = False
        self.pending = []  # (id, alpha)
        self.draft_version = 0
        self.observations = 0
        self.events = []

    def observe(self, alpha):
        if not (0.0 <= alpha <= 1.0):
            raise ValueError("alpha must be in [0, 1]")
        self.observations += 1
        if not self.initialized:
            self.warmup.append(alpha)
            if len(self.warmup) == self.n_init:
                s = 0.0
                for a in self.warmup:
                    s += a
                self.ema_short = self.ema_long = s / self.n_init
                self.initialized = True
                self.warmup = []
            return
        # lambda a + (1 - lambda) alpha, as a + (1 - lambda)(alpha - a): exact on constants
        self.ema_short = self.ema_short + (1.0 - self.ls) * (alpha - self.ema_short)
        self.ema_long = self.ema_long + (1.0 - self.ll) * (alpha - self.ema_long)
        if not self.collection_enabled and self.ema_short < self.ema_long - self.eps:
            self.collection_enabled = True
            self.events.append(("COLLECT_ON", self.observations))

    def record_sample(self, sid, alpha):
        if not self.collection_enabled:
            return False
        self.pending.append((sid, alpha))
        return True

    def maybe_trigger_training(self, train_fn):
        """train_fn(train_ids, eval_ids) -> alpha_eval (may raise)."""
        n = len(self.pending)
        if n < self.n_threshold:
            return None
        n_train = (9 * n) // 10
        s = 0.0
        for _, a in self.pending[:n_train]:
            s += a
        alpha_train = s / n_train if n_train > 0 else 0.0
        alpha_eval = train_fn([i for i, _ in self.pending[:n_train]],
                              [i for i, _ in self.pending[n_train:]])
        self.events.append(("TRAIN_TRIGGER", self.observations))
        if alpha_eval > alpha_train:
            self.draft_version += 1
            action = 1
            self.events.append(("DEPLOY", self.observations))
        elif alpha_eval < alpha_train:
            action = -1
            self.events.append(("REJECT", self.observations))
            if self.collection_enabled:
                self.collection_enabled = False
                self.events.append(("COLLECT_OFF", self.observations))
        else:
            action = 0
        self.pending = []
        return dict(action=action, alpha_train=alpha_train, n_train=n_train, n_eval=n - n_train)
