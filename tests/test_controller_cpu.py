"""Algorithm 1 controller (SPEC.md adapt_control) through the C ABI, checked
against the SPEC's examples and bit-for-bit against oracle/controller.py on
seeded streams.  No GPU: the trigger path is covered in test_controller_gpu.py."""
import random

import pytest

from oracle.controller import Controller
from paper_2602_05145_b200 import _lib, api


def state(c):
    return c.state()


def test_warmup_mean_initialises_both_emas():
    c = api.AdaptiveController(n_init=2)
    c.observe(0.6)
    assert state(c)["initialized"] == 0
    c.observe(0.8)
    s = state(c)
    assert s["initialized"] == 1 and s["ema_short"] == s["ema_long"] == (0.6 + 0.8) / 2
    assert s["collection_enabled"] == 0
    c2 = api.AdaptiveController(n_init=4)
    for _ in range(4):
        c2.observe(0.8)
    assert state(c2)["ema_short"] == state(c2)["ema_long"] == 0.8


def test_step_drop_enables_collection_at_k2():
    # EMAs at 0.8, alpha drops to 0.5, lambda 0.9 / 0.99, eps 0.05:
    # ema_short(k) = 0.5 + 0.3 * 0.9^k, ema_long(k) = 0.5 + 0.3 * 0.99^k; first true at k=2
    c = api.AdaptiveController(0.9, 0.99, 0.05, n_init=1)
    c.observe(0.8)
    c.observe(0.5)
    s = state(c)
    assert s["collection_enabled"] == 0
    assert abs(s["ema_short"] - (0.5 + 0.3 * 0.9)) < 1e-15
    c.observe(0.5)
    s = state(c)
    assert s["collection_enabled"] == 1
    assert abs(s["ema_short"] - (0.5 + 0.3 * 0.9 ** 2)) < 1e-15
    assert abs(s["ema_long"] - (0.5 + 0.3 * 0.99 ** 2)) < 1e-15
    assert c.events() == [("COLLECT_ON", 3)]


def test_constant_stream_and_eps_one_never_enable():
    c = api.AdaptiveController(n_init=3)
    for _ in range(3):
        c.observe(0.7)
    init = state(c)["ema_short"]  # mean of the warm-up (0.7 up to rounding)
    for _ in range(500):
        c.observe(init)
    s = state(c)
    assert s["collection_enabled"] == 0 and s["ema_short"] == s["ema_long"] == init
    c = api.AdaptiveController(epsilon=1.0, n_init=1)
    c.observe(1.0)
    for _ in range(300):
        c.observe(0.0)
    assert state(c)["collection_enabled"] == 0


def test_record_sample_is_noop_when_collection_off():
    c = api.AdaptiveController(n_init=1)
    assert c.record_sample(1, 0.5) is False
    assert state(c)["stored_samples"] == 0
    c.observe(0.9)
    for _ in range(10):
        c.observe(0.1)
    assert state(c)["collection_enabled"] == 1
    assert c.record_sample(2, 0.5) is True and state(c)["stored_samples"] == 1


def test_validation():
    with pytest.raises(_lib.ConfigError):
        api.AdaptiveController(lambda_short=0.99, lambda_long=0.9)
    with pytest.raises(_lib.ConfigError):
        api.AdaptiveController(lambda_short=0.9, lambda_long=0.9)  # long must decay slower
    with pytest.raises(_lib.ConfigError):
        api.AdaptiveController(n_init=0, n_threshold=0, epsilon=0.0)
    with pytest.raises(_lib.ConfigError):  # floor(9 * 1 / 10) = 0: empty D_train
        api.AdaptiveController(n_threshold=1)
    api.AdaptiveController(n_threshold=2)
    c = api.AdaptiveController(n_init=1)
    for bad in (-0.1, 1.5, float("nan")):
        with pytest.raises(_lib.DomainError):
            c.observe(bad)
    assert state(c)["observations"] == 0
    # the trigger needs a trainer and a buffer
    with pytest.raises(_lib.DomainError):
        c.maybe_trigger_training(type("T", (), {"h": None})(), type("B", (), {"h": None})())


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_emas_bit_exact_against_oracle(seed):
    rnd = random.Random(seed)
    kw = dict(lambda_short=0.9, lambda_long=0.99, epsilon=0.03, n_init=8, n_threshold=10 ** 9)
    c, o = api.AdaptiveController(**kw), Controller(**kw)
    level = 0.8
    seen = []
    for i in range(3000):
        if i % 700 == 0:
            level = rnd.uniform(0.2, 0.9)  # distribution shifts (SPEC langshift scenarios)
        a = min(1.0, max(0.0, rnd.gauss(level, 0.1)))
        c.observe(a)
        o.observe(a)
        if o.collection_enabled:
            assert c.record_sample(i, a) == o.record_sample(i, a)
        s = state(c)
        assert s["ema_short"] == o.ema_short and s["ema_long"] == o.ema_long, i
        seen.append(a)
        lo, hi = min(seen), max(seen)  # EMA boundedness (SPEC adapt_control invariants)
        if s["initialized"]:
            assert lo <= s["ema_short"] <= hi and lo <= s["ema_long"] <= hi
        assert bool(s["collection_enabled"]) == o.collection_enabled
    assert state(c)["stored_samples"] == len(o.pending)
    assert c.events() == o.events
