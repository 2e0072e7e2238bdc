"""CPU-only checks of the C ABI: the library loads without a GPU, exports every
entry point include/specsim_draft_trainer.h declares, and its host-side
bookkeeping is bit-exact with the reference (golden vectors) and the oracle."""
import json
import pathlib
import re

import numpy as np
import pytest

import oracle
from paper_2602_05145_b200 import _lib, api

ROOT = pathlib.Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "bookkeeping.json").read_text())


def declared_functions():
    text = (ROOT / "include" / "specsim_draft_trainer.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(specsim_\w+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 35
    L = _lib.lib()
    missing = [n for n in names if getattr(L, n, None) is None]
    assert not missing, missing
    # and the ctypes signature table covers them all
    assert not [n for n in names if n not in _lib.SIGNATURES]


def test_version_and_last_error():
    assert b"sm_100a" in _lib.lib().specsim_version()


@pytest.mark.parametrize("seed", list(GOLD["rng"].keys()))
def test_rng_bit_exact_with_reference(seed):
    g = GOLD["rng"][seed]
    r = api.Rng(int(seed))
    assert [r.uniform().hex() for _ in range(32)] == g["uniform"]
    assert [r.normal(0.0, 1.0).hex() for _ in range(16)] == g["normal"]
    assert [r.normal(3.0, 2.0).hex() for _ in range(8)] == g["normal_3_2"]
    for m, seq in g["geometric"].items():
        assert [r.geometric(float(m)) for _ in range(16)] == seq


def test_accept_length_bookkeeping_bit_exact():
    for a, gm, hx in GOLD["expected_accept_length"]:
        assert api.expected_accept_length(a, gm).hex() == hx
    for case in GOLD["sample_accept_length"]:
        r = api.Rng(case["seed"])
        assert [r.sample_accept_length(case["alpha"], case["gamma"]) for _ in range(64)] == case["seq"]
    for ell, gm, hx in GOLD["alpha_from_accept_length"]:
        assert api.alpha_from_accept_length(ell, gm).hex() == hx


def test_domain_errors_map_to_status_1():
    with pytest.raises(_lib.DomainError):
        api.expected_accept_length(1.5, 3)
    with pytest.raises(_lib.DomainError):
        api.alpha_from_accept_length(0.5, 3)
    with pytest.raises(_lib.DomainError):
        api.Rng(1).sample_accept_length(0.5, 0)


def test_split_and_geometry():
    for n in (0, 1, 9, 10, 11, 2048, 12345):
        assert api.split_train_eval(n) == oracle.split_train_eval(n)
    assert api.SignalGeometry(4096).bytes_per_token() * 100 == GOLD["spec_bytes_100tok_h4096_3layers_bf16"]
    with pytest.raises(_lib.DomainError):
        api.SignalGeometry(0).bytes_per_token()


@pytest.mark.parametrize("idx,length,alpha", [(0, 50, 0.6), (3, 131, 0.0), (7, 7, 1.0), (11, 300, 0.36)])
def test_synth_capture_matches_oracle(idx, length, alpha):
    a = api.synth_capture(20260217, idx, length, 512, 64, alpha=alpha)
    b = oracle.synth_capture(20260217, idx, length, 512, 64, alpha=alpha)
    assert np.array_equal(a["ids"], b["ids"])
    assert np.array_equal(a["features"], b["features"])
    assert np.array_equal(a["accept_lengths"], b["accept_lengths"])
    assert a["alpha_s"].hex() == b["alpha_s"].hex()
    assert a["accept_lengths"].sum() == length  # truncated last step


def test_shape_validation_collects_all_problems():
    bad = dict(api.CONFIGS["C1"], hidden=100, head_dim=96, seq_len=100)
    with pytest.raises(_lib.DomainError) as e:
        api.DraftTrainer(bad)
    msg = str(e.value)
    assert "hidden" in msg and "head_dim" in msg and "seq_len" in msg


def test_gpu_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.SpecsimError) as e:
        api.HiddenStateBuffer(api.SignalGeometry(64), 1024)
    assert e.value.status == _lib.ECUDA


def test_flop_convention_matches_survey():
    f = api.gemm_flops_per_token(api.CONFIGS["C2"])
    assert abs(f["total"] / 1e9 - 4.8633) < 1e-3
    assert abs(api.gemm_flops_per_token(api.CONFIGS["C1"])["total"] / 1e9 - 0.01398) < 1e-4
    assert abs(api.gemm_flops_per_token(api.CONFIGS["C5"])["total"] / 1e9 - 12.9479) < 1e-3


def test_shape_validation_precedes_device_checks():
    """Invalid draft shapes (incl. the training-time-test fields) are domain
    errors reported with every problem at once, before any device access;
    a valid shape on a GPU-less host fails with SPECSIM_ECUDA (no fallback)."""
    bad = dict(api.CONFIGS["C1"], ttt_steps=17, seq_len=192, head_dim=96)
    with pytest.raises(_lib.DomainError) as e:
        api.DraftTrainer(bad)
    msg = str(e.value)
    assert "ttt_steps" in msg and "head_dim" in msg and "seq_len" in msg
    with pytest.raises(_lib.DomainError, match="ttt_decay"):
        api.DraftTrainer(dict(api.CONFIGS["C1"], ttt_steps=2, ttt_decay=1.5))
    import torch
    if torch.cuda.is_available():
        return
    with pytest.raises(_lib.SpecsimError) as e:
        api.DraftTrainer(dict(api.CONFIGS["C1"], ttt_steps=3))
    assert e.value.status == _lib.ECUDA


def test_current_alpha_bit_exact_with_reference():
    """workload.cpp:41-47 through the C ABI vs the compiled reference's own
    outputs (golden vectors); phase checks are configuration errors."""
    for a0, astar, tau, n, hx in GOLD["current_alpha"]:
        assert api.current_alpha(a0, astar, tau, n).hex() == hx, (a0, astar, tau, n)
    assert api.current_alpha(0.3, 0.6, 100.0, -5.0) == 0.3  # n clamped at 0
    with pytest.raises(_lib.ConfigError):
        api.current_alpha(0.7, 0.6, 100.0, 1.0)
    with pytest.raises(_lib.ConfigError):
        api.current_alpha(0.3, 0.6, 0.0, 1.0)
