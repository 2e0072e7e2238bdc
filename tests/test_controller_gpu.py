"""maybe_trigger_training driving the real trainer: the 9:1
chronological split, alpha_train, deploy / reject gate with the model
restored unless deployed, and failure atomicity -- checked against the
oracle/controller.py restatement fed the trainer's own alpha_eval."""
import numpy as np
import pytest

import oracle
from oracle.controller import Controller
from paper_2602_05145_b200 import _lib, api

pytestmark = pytest.mark.gpu
SEED = 4242
C1 = api.CONFIGS["C1"]


def make_buffer(n, constant_tokens):
    buf = api.HiddenStateBuffer(api.SignalGeometry(C1["hidden"]), 1 << 16)
    for i in range(n):
        cap = oracle.synth_capture(SEED, i, C1["seq_len"] + 2, C1["vocab"], C1["hidden"])
        ids = cap["ids"]
        if constant_tokens:
            ids = np.full_like(ids, 7)  # learnable: every target is token 7
        buf.append_packed(i, cap["alpha_s"], cap["features"], ids)
    return buf


def enable_collection(ctrl, ref):
    for a in [0.8, 0.8] + [0.3] * 6:
        ctrl.observe(a)
        ref.observe(a)
    assert ctrl.state()["collection_enabled"] == 1 and ref.collection_enabled


def params(tr):
    return {n: tr.get_param(n).copy() for n, *_ in tr.params()[0]}


def run(constant_tokens, label_alpha, n=20, epochs=3):
    tr = api.DraftTrainer(C1, lr=3e-3, seed=SEED)
    buf = make_buffer(n, constant_tokens)
    kw = dict(n_init=2, n_threshold=n)
    ctrl, ref = api.AdaptiveController(**kw), Controller(**kw)
    enable_collection(ctrl, ref)
    for i in range(n):
        assert ctrl.record_sample(i, label_alpha[i]) and ref.record_sample(i, label_alpha[i])
        if i < n - 1:  # below threshold: nothing happens
            assert not ctrl.maybe_trigger_training(tr, buf).triggered
    before = params(tr)
    d = ctrl.maybe_trigger_training(tr, buf, epochs=epochs)
    r = ref.maybe_trigger_training(lambda t, e: d.outcome.alpha_eval)
    assert d.triggered and (d.n_train, d.n_eval) == (r["n_train"], r["n_eval"]) == (18, 2)
    assert d.alpha_train == r["alpha_train"] and d.action == r["action"]
    s = ctrl.state()
    assert s["stored_samples"] == 0 and s["draft_version"] == ref.draft_version
    assert bool(s["collection_enabled"]) == ref.collection_enabled
    assert ctrl.events() == ref.events
    return tr, buf, d, before


def test_deploy_keeps_the_trained_model():
    tr, buf, d, before = run(True, [0.5] * 20)
    assert d.outcome.alpha_eval > 0.5 and d.action == 1
    after = params(tr)
    assert any(not np.array_equal(before[k], after[k]) for k in before)
    tr.close()
    buf.close()


def test_reject_restores_the_model_and_stops_collection():
    tr, buf, d, before = run(False, [0.95] * 20, epochs=1)
    assert d.outcome.alpha_eval < 0.95 and d.action == -1
    after = params(tr)
    for k in before:
        assert np.array_equal(before[k], after[k]), k  # M_draft kept, bit-exact
    # the restored model trains on exactly as the untouched one would
    tr2 = api.DraftTrainer(C1, lr=3e-3, seed=SEED)
    for _ in range(2):  # 2nd step depends on the restored AdamW state and step count
        r1, r2 = tr.step(buf, [0, 1]), tr2.step(buf, [0, 1])
        assert r1["loss"] == r2["loss"]
    tr.close()
    tr2.close()
    buf.close()


def test_trainer_failure_leaves_everything_unchanged():
    """A trainer that throws (here: the buffer's signal geometry does not
    match the draft shape) leaves controller state, pending set, events and
    the model unchanged."""
    tr = api.DraftTrainer(C1, lr=3e-3, seed=SEED)
    buf = api.HiddenStateBuffer(api.SignalGeometry(2 * C1["hidden"]), 1 << 14)
    for i in range(2):
        cap = oracle.synth_capture(SEED, i, 40, C1["vocab"], 2 * C1["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
    ctrl = api.AdaptiveController(n_init=2, n_threshold=2)
    enable_collection(ctrl, Controller(n_init=2, n_threshold=2))
    assert ctrl.record_sample(0, 0.5) and ctrl.record_sample(1, 0.5)
    s0, e0, p0 = ctrl.state(), ctrl.events(), params(tr)
    with pytest.raises(_lib.DomainError):
        ctrl.maybe_trigger_training(tr, buf)
    assert ctrl.state() == s0 and ctrl.events() == e0
    p1 = params(tr)
    assert all(np.array_equal(p0[k], p1[k]) for k in p0)
    tr.close()
    buf.close()


def test_evicted_pending_samples_are_dropped():
    """Pending samples the ring evicted are dropped at the trigger (they can
    never be trained on) instead of failing every later trigger; training
    starts once n_threshold resident samples are pending."""
    tr = api.DraftTrainer(C1, lr=3e-3, seed=SEED)
    L = C1["seq_len"] + 2
    buf = api.HiddenStateBuffer(api.SignalGeometry(C1["hidden"]), 5 * L)  # holds 5 samples
    ctrl = api.AdaptiveController(n_init=2, n_threshold=4)
    enable_collection(ctrl, Controller(n_init=2, n_threshold=4))
    for i in range(4):
        cap = oracle.synth_capture(SEED, i, L, C1["vocab"], C1["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
        if i < 2:
            assert ctrl.record_sample(i, 0.5)  # 0, 1 pending
    for i in range(4, 7):  # 0 and 1 are evicted by 5 and 6; 4, 5, 6 pending
        cap = oracle.synth_capture(SEED, i, L, C1["vocab"], C1["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
        assert ctrl.record_sample(i, 0.5)
    assert ctrl.state()["stored_samples"] == 5
    d = ctrl.maybe_trigger_training(tr, buf)
    assert not d.triggered and ctrl.state()["stored_samples"] == 3  # 0, 1 dropped
    assert ctrl.record_sample(3, 0.5)  # resident: the threshold is met again
    d = ctrl.maybe_trigger_training(tr, buf)
    assert d.triggered and (d.n_train, d.n_eval) == (3, 1)
    tr.close()
    buf.close()


def test_train_with_missing_sample_changes_nothing():
    """train(job) checks every sample before the first launch: a missing id
    fails the whole job with the model untouched (not after earlier steps
    have updated it); the outcome's version follows snapshot / restore."""
    tr = api.DraftTrainer(C1, lr=3e-3, seed=SEED)
    buf = make_buffer(10, False)
    p0 = params(tr)
    with pytest.raises(_lib.DomainError):
        tr.train(buf, list(range(9)) + [999], [9], epochs=2)  # 999: last step's sample
    p1 = params(tr)
    assert all(np.array_equal(p0[k], p1[k]) for k in p0)
    tr.snapshot()
    o1 = tr.train(buf, [0, 1], [2])
    assert o1.new_version == 1
    tr.restore()  # not deployed: the model (and its version) is the snapshot's
    o2 = tr.train(buf, [0, 1], [2])
    assert o2.new_version == 1
    o3 = tr.train(buf, [0, 1], [2])  # deployed o2 in place, trained again
    assert o3.new_version == 2
    tr.close()
    buf.close()


def test_restore_without_snapshot_is_a_domain_error():
    tr = api.DraftTrainer(C1, seed=SEED)
    with pytest.raises(_lib.DomainError):
        tr.restore()
    tr.snapshot()
    tr.restore()
    tr.close()
