"""Parity at the driver-benchmarked configuration and at the large configs
(SURVEY §8(d) tolerances, tests/_parity.py):

* C2 at its full sequence length (S 2048: 16 attention key blocks, the shape
  `bench.py` times), one full sample and one short one;
* C4 model dimensions (H 5120, Q 8192 != H, GQA 64:8, V 151936, FFN 25600,
  eps 1e-6, theta 1e6) and C5 model dimensions (H 8192, FFN 28672) on short
  batches the CPU oracle finishes in seconds;
* the target gather bit-exact across a ring wrap with every training-time-test
  slice, and exact top-1 on a learned (decided) batch.

The oracle starts from the trainer's weights (initialisation is bit-exact,
tests/test_trainer_gpu.py::test_init_is_bit_exact).
"""
import numpy as np
import pytest

import oracle
from paper_2602_05145_b200 import api
from _parity import (LARGE_LOGIT_TOL, check_gather, oracle_state, sample_rows,
                     step_and_compare)

pytestmark = pytest.mark.gpu
SEED = 20260217
# lr 1e-4 (the library default): at these widths one lr-1e-3 Adam step moves
# the logits of the batch's targets so far that the second step's loss is
# ~1e-4 and its relative error meaningless
HP = [1e-4, 0.9, 0.95, 1e-8, 0.0]


def oshape(c):
    return oracle.make_shape(c["hidden"], c["vocab"], c["seq_len"], c["n_heads"], c["n_kv_heads"],
                             c["head_dim"], c["ffn"], c["micro_batch"], eps=c["rms_eps"],
                             theta=c["rope_theta"], ttt=c.get("ttt_steps", 1),
                             ttt_decay=c.get("ttt_decay", 0.8))


def run_parity(c, lens, steps=1, check_update=True):
    shp = oshape(c)
    tr = api.DraftTrainer(c, lr=HP[0], betas=(HP[1], HP[2]), eps=HP[3], weight_decay=HP[4],
                          seed=SEED)
    tr.keep_grads(True)
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), sum(lens) + 1024)
    samples = []
    for i, L in enumerate(lens):
        cap = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
        samples.append((cap["ids"], cap["features"]))
    _, P, E = oracle_state(tr, shp)
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    reports, well = [], {}
    for k in range(1, steps + 1):
        rep = step_and_compare(tr, buf, list(range(len(lens))), shp, samples, P, Mst, Vst, E, k,
                               HP, check_update=check_update, sync_weights=k < steps,
                               logit_tol=LARGE_LOGIT_TOL, well=well)
        print(k, rep)
        reports.append(rep)
    tr.close()
    buf.close()
    return reports


def test_c2_full_sequence_step():
    """The benchmarked shape: C2 at S 2048 (B 2: one sample longer than S + 2,
    one ending mid-sequence in the 9th key block)."""
    c = dict(api.CONFIGS["C2"], micro_batch=2)
    run_parity(c, [c["seq_len"] + 40, 1100], steps=2)


def test_c4_model_dims_step():
    c = dict(api.CONFIGS["C4"], seq_len=256, micro_batch=2)
    run_parity(c, [c["seq_len"] + 2, 141])


def test_c5_model_dims_step():
    c = dict(api.CONFIGS["C5"], seq_len=256, micro_batch=2)
    run_parity(c, [c["seq_len"] + 2, 197])


def test_c2_full_sequence_ttt2_step():
    """Training-time test (K 2) at the bench shape's full sequence length."""
    c = dict(api.CONFIGS["C2"], micro_batch=1, ttt_steps=2)
    run_parity(c, [c["seq_len"] + 5])


def test_gather_bit_exact_across_ring_wrap_ttt():
    """Samples straddling the ring's end (capacity 480 tokens; rows are
    assigned in append order, the oldest sample is evicted), a sample too
    short for the later unroll slices, padding rows: the device u / y / m of
    all K = 3 slices and the F rows equal oracle.gather_batch bit for bit,
    for a training step and for an eval (slice 0)."""
    c = dict(api.CONFIGS["C1"], micro_batch=4, ttt_steps=3)
    S = c["seq_len"]
    lens = [130, 130, 131, 132, 70]  # 0 evicted by 3; 3 straddles row 480 -> 0; 4 after it
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 480)
    caps = {}
    for i, L in enumerate(lens):
        caps[i] = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
        buf.append_packed(i, caps[i]["alpha_s"], caps[i]["features"], caps[i]["ids"])
    with pytest.raises(Exception):
        buf.sample_info(0)
    assert [buf.sample_info(i)[0] for i in (1, 2, 3, 4)] == lens[1:]
    tr = api.DraftTrainer(c, seed=SEED)
    shp = oshape(c)
    for ids in ([3, 4, 1], [2, 3, 4, 1], [4]):
        samples = [(caps[i]["ids"], caps[i]["features"]) for i in ids]
        F, u, y, m = oracle.gather_batch(shp, samples)
        inside = sample_rows(shp, samples)
        tr.step(buf, ids)
        check_gather(tr, F, u, y, m, inside=inside)
        tr.eval(buf, ids)
        check_gather(tr, F, u, y, m, rows=c["micro_batch"] * S, inside=inside)
    tr.close()
    buf.close()


def test_top1_exact_on_decided_batch():
    """After a few steps on a learnable batch (85% of the tokens the same id)
    the draft is confident: every valid row's top-1 / top-2 margin exceeds
    1e-2, so the eval's top-1 count and per-row argmax must equal the oracle
    forward's on the GPU-trained weights exactly."""
    c = dict(api.CONFIGS["C1"], micro_batch=4)
    S = c["seq_len"]
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 1 << 12)
    samples = []
    rng = np.random.default_rng(5)
    for i, L in enumerate([S + 2, S + 2, 90, S + 9]):
        cap = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
        # mostly one token, 15% random ones: learnable but never all right
        ids = np.where(rng.random(L) < 0.15, cap["ids"], 7).astype(np.int32)
        buf.append_packed(i, cap["alpha_s"], cap["features"], ids)
        samples.append((ids, cap["features"]))
    tr = api.DraftTrainer(c, lr=3e-3, seed=SEED)
    for _ in range(25):
        tr.step(buf, [0, 1, 2, 3])
    shp = oshape(c)
    _, P, E = oracle_state(tr, shp)
    F, u, y, m = oracle.gather_batch(shp, samples)
    out, lse, am, margin = oracle.forward(shp, P, E, F, u, y, m, round_bf16=True, margin=True)
    r = tr.eval(buf, [0, 1, 2, 3])
    valid = m == 1
    assert (margin[valid] > 1e-2).all(), float(margin[valid].min())
    assert r["valid_tokens"] == out.valid
    assert r["top1_correct"] == out.top1, (r["top1_correct"], out.top1)
    assert 0 < out.top1 < out.valid  # neither trivially all-right nor all-wrong
    am_g = tr.read_rows("argmax")[:len(am)]
    assert np.array_equal(am_g[valid], am[valid])
    np.testing.assert_allclose(tr.read_rows("lse")[:len(lse)][valid], lse[valid], atol=5e-3)
    tr.close()
    buf.close()
