"""SPEC sim_serving (step / run) on the reference's own
simulator code (perf_model.cpp, workload.cpp compiled in place by
integration/sim_serving/Makefile) driving the real B200 trainer behind
train(job).  Checks the SPEC's invariants and examples:
the per-iteration latency model, token conservation, the zero-overhead signal
model, extract_signals byte accounting, and Algorithm 1 deploying a draft
after the domain shift with measured durations."""
import json
import pathlib
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]
EXE = ROOT / "integration" / "sim_serving" / "_build" / "sim_serving"
PROFILE = ROOT / "integration" / "sim_serving" / "gpt-oss-120b.csv"
T = {1: 3.416, 2: 3.844, 4: 4.341, 8: 5.236, 16: 6.123, 32: 7.637, 64: 9.345, 128: 11.79,
     256: 15.50, 512: 21.50}
D0, GAMMA = 0.393, 3


def lat(n):
    """T(n): exact at profiled points, linear between (perf_model.hpp:34-36)."""
    xs = sorted(T)
    return float(np.interp(n, xs, [T[x] for x in xs]))


def run(mode, **kw):
    if not EXE.exists():
        pytest.skip("integration/sim_serving not built (needs the reference sources)")
    args = [str(EXE), "--mode", mode, "--profile", str(PROFILE)]
    for k, v in kw.items():
        args += ["--" + k.replace("_", "-"), str(v)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    summary = json.loads(lines[-1])
    rows = None
    if kw.get("emit_iterations"):
        hdr = lines[0].split(",")
        assert hdr == ["clock_ms", "batch_size", "speculation_on", "mean_accept_length",
                       "tokens_emitted", "throughput_tokens_per_s", "collection_on",
                       "buffer_bytes", "cumulative_storage_bytes", "draft_version"]
        rows = np.array([[float(x) for x in ln.split(",")] for ln in lines[1:-1]])
    return summary, rows


def test_speculation_off_latency_model_and_conservation():
    s, rows = run("speculation_off", requests=40, concurrency=4, mean_tokens=20,
                  emit_iterations=1)
    assert s["tokens"] == s["script_tokens"]  # token conservation
    clock = np.concatenate([[0.0], rows[:, 0]])
    dt = np.diff(clock)
    assert (dt > 0).all()  # clock non-decreasing
    b = rows[:, 1]
    assert (rows[:, 2] == 0).all() and (rows[:, 4] == b).all()
    # throughput for batch b is b / T(b) exactly (SPEC invariant)
    np.testing.assert_allclose(dt, [lat(x) for x in b], rtol=1e-12)
    # SPEC example: speculation off, b = 1 -> clock += 3.416 ms, 1 token
    _, one = run("speculation_off", requests=3, concurrency=1, mean_tokens=5, emit_iterations=1)
    assert abs(one[0, 0] - 3.416) < 1e-12 and one[0, 4] == 1


def test_speculation_on_iteration_latency_example():
    s, rows = run("speculation_on_no_training", requests=5, concurrency=1, mean_tokens=8,
                  emit_iterations=1, collect=0, pretrain=20)
    # SPEC example: on, b = 1, gamma 3 -> 3 * 0.393 + T(4) = 5.520 ms
    assert abs(rows[0, 0] - (GAMMA * D0 + 4.341)) < 1e-9
    dt = np.diff(np.concatenate([[0.0], rows[:, 0]]))
    np.testing.assert_allclose(dt, [GAMMA * D0 + lat(x * (GAMMA + 1)) for x in rows[:, 1]],
                               rtol=1e-12)
    assert ((rows[:, 4] >= rows[:, 1]) & (rows[:, 4] <= rows[:, 1] * (GAMMA + 1))).all()
    assert s["tokens"] == s["script_tokens"]


def test_zero_overhead_signal_model_and_accounting():
    """Collecting signals (extract_signals into the HBM ring) changes no clock
    or throughput value; the buffer accounting is records x bytes/token."""
    kw = dict(requests=150, concurrency=8, mean_tokens=60, pretrain=200)
    off, _ = run("speculation_on_no_training", collect=0, **kw)
    on, _ = run("speculation_on_no_training", collect=1, **kw)
    assert on["clock_ms"] == off["clock_ms"] and on["tokens"] == off["tokens"]
    assert off["signal_records"] == 0
    assert on["signal_records"] > 0  # the drift switched collection on
    assert on["buffer_bytes"] + on["cumulative_storage_bytes"] == on["signal_records"] * 3 * 256 * 2


def test_tide_trains_and_deploys_after_the_drift():
    """tide_default (speculation always on): the drift to domain B drops the
    acceptance, collection switches on, train(job) runs on the B200 with its
    measured duration, and the deployed draft (served from trigger time +
    duration) raises domain B's measured acceptance."""
    s, rows = run("tide_default", requests=500, concurrency=8, mean_tokens=130, threshold=128,
                  emit_iterations=1)
    print(s)
    assert s["tokens"] == s["script_tokens"] and s["speculation_duty"] == 1.0
    assert s["trainings"] >= 1 and s["deploys"] >= 1 and s["draft_version"] == s["deploys"]
    assert s["train_ms"] > 0
    deployed = [j for j in s["jobs"] if j["action"] == 1]
    assert max(j["alpha_deployed"][1] for j in deployed) > 0.3  # the draft learned domain B
    dv = rows[:, 9]
    assert (np.diff(dv) >= 0).all() and dv[-1] == s["draft_version"]


def test_tide_adaptive_run_invariants():
    """tide_adaptive: the drafter switches speculation by practical_speedup at
    the monitored alpha; tokens are conserved and the clock is monotone."""
    s, rows = run("tide_adaptive", requests=300, concurrency=8, mean_tokens=100, threshold=128,
                  emit_iterations=1)
    print(s)
    assert s["tokens"] == s["script_tokens"]
    assert (np.diff(rows[:, 0]) > 0).all()
    assert 0 < s["speculation_duty"] <= 1
