"""bench.py host logic on CPU: the reference arm's JSON line (the driver runs it
on the GPU box's host cores) and the weak / strong scaling workload split."""
import json
import pathlib
import subprocess
import sys
import types

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2602_05145_b200 import api  # noqa: E402


def _args(**kw):
    base = dict(config="C2", ttt=1, global_batch=0, gpus=1)
    base.update(kw)
    return types.SimpleNamespace(**base)


def test_weak_scaling_keeps_the_per_rank_micro_batch(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "8")
    cfg = bench.workload_cfg(_args(gpus=8), api)
    assert cfg["micro_batch"] == api.CONFIGS["C2"]["micro_batch"]
    assert bench.scaling_of(_args()) == "weak"


def test_strong_scaling_splits_the_global_batch(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "8")
    a = _args(config="C5", global_batch=16, gpus=8)
    cfg = bench.workload_cfg(a, api)
    assert cfg["micro_batch"] == 2
    assert bench.scaling_of(a) == "strong"
    assert bench.config_block(a, cfg)["global_batch"] == 16
    monkeypatch.setenv("WORLD_SIZE", "3")
    with pytest.raises(SystemExit):
        bench.workload_cfg(_args(global_batch=16, gpus=3), api)


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "0",
                          "--cpu-sample-seq", "64"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "draft-train tokens/sec"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["higher_is_better"] is True and d["scaling"] == "weak"
    # the line states what was actually timed: 1 sequence x 64 positions
    c = d["config"]
    assert c["micro_batch"] == 1 and c["seq_len"] == 64 and c["tokens_per_rank_step"] == 64
    assert c["workload_seq_len"] == api.CONFIGS["C1"]["seq_len"]
    assert "model" in d["host_cpu"]


def test_multi_gpu_request_spawns_ranks(monkeypatch):
    """--gpus N without a torchrun environment re-executes under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous); a WORLD_SIZE
    that disagrees with --gpus is an error, not a silent 1-rank run."""
    seen = {}

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd
        return types.SimpleNamespace(returncode=0)

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.main()


def test_config_block_reports_the_launched_world(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "8")
    a = _args(gpus=8)
    blk = bench.config_block(a, bench.workload_cfg(a, api))
    assert blk["parallelism"] == "dp8" and blk["global_batch"] == 8 * api.CONFIGS["C2"]["micro_batch"]


@pytest.mark.gpu
def test_bench_line_contract_gpu():
    """The driver parses one JSON line from `bench.py`: every contract key with
    sane values, on the tiny config so it runs in seconds."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "C1", "--steps", "4",
                          "--warmup", "3", "--cpu-sample-seq", "32"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 4 and d["warmup"] == 3 and d["n_gpus"] == 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["ingest"]["h2d_GBps"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor"
    assert 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"], abs=1e-4)  # 4 decimals
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["gpu_launches"] >= 4 * 20  # every step is tens of our own kernels
    assert d["clocks"]["sm_max_mhz"] > 0
    assert d["config"]["workload"].startswith("C1")
