"""Algorithm 1 end to end on the B200: the C++ tool
paper_2602_05145_b200/tide_loop drives the AdaptiveController with the real
DraftTrainer behind train(job) -- measured training durations, serving
acceptance measured as the deployed draft's top-1 on the current domain.
A domain shift must switch collection on, trigger training at n_threshold,
and the retrained draft must pass the deploy gate and raise the serving
acceptance on the new domain."""
import json
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu
TOOL = pathlib.Path(__file__).resolve().parents[1] / "paper_2602_05145_b200" / "tide_loop"


def test_tide_loop_adapts_after_domain_shift():
    assert TOOL.exists(), "build with make -C paper_2602_05145_b200/csrc"
    out = subprocess.run([str(TOOL), "--requests", "600", "--threshold", "256"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    print("\n".join(json.dumps(l) for l in lines))
    pre = next(l for l in lines if l.get("event") == "pretrain")
    shift = next(l for l in lines if l.get("event") == "domain_shift")
    summary = lines[-1]
    assert summary["summary"]
    # the pre-trained draft has learned domain A; it is useless on domain B
    assert pre["alpha_serving"] > 0.5
    assert shift["alpha_serving"] < 0.2
    after = [l for l in lines if l.get("observation", 0) >= shift["observation"]]
    assert any(l.get("event") == "collect_on" for l in after)
    trains = [l for l in after if l.get("event") == "train"]
    assert trains, "no training triggered after the shift"
    t = trains[0]
    assert t["n_train"] + t["n_eval"] == 256 and t["n_train"] == 230  # 9:1 split
    assert t["duration_s"] > 0 and t["steps"] > 0  # measured, not samples_per_hour
    assert t["action"] == "deploy" and t["alpha_eval"] > t["alpha_train"]
    assert summary["draft_version"] >= 1
    assert summary["alpha_serving"] > shift["alpha_serving"] + 0.3
