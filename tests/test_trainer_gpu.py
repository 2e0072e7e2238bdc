"""Draft-training step on the B200 vs the CPU oracle at BASELINE config C1
(and a GQA variant with head_dim 128): identical seeded synthetic captures and
weights (initialisation is bit-exact), then loss, every parameter gradient,
the AdamW update, eval top-1 and train(job) outcome.

Tolerances (fp32 accumulation-order + bf16 rounding-point noise; the oracle
rounds at the same points, oracle.h) are tests/_parity.py's: loss rel <= 2e-3;
grads rel-Frobenius <= 1e-2; post-AdamW |dp_gpu - dp_cpu| <= 0.05 lr on >=
99.9% of elements whose oracle gradient is well determined; token gather
(u / y / m / F rows) bit-exact; top-1 exact on rows with logit margin > 1e-2.
"""
import numpy as np
import pytest

import oracle
from paper_2602_05145_b200 import _lib, api
from _parity import LARGE_LOGIT_TOL, oracle_state, step_and_compare

pytestmark = pytest.mark.gpu
SEED = 20260217
HP = [1e-3, 0.9, 0.95, 1e-8, 0.0]

SHAPES = {
    "C1": api.CONFIGS["C1"],
    "gqa128": dict(hidden=256, vocab=2048, seq_len=128, n_heads=4, n_kv_heads=1, head_dim=128,
                   ffn=512, micro_batch=3, rms_eps=1e-6, rope_theta=500000.0),
    # vocabulary > one 32k backward chunk and not a multiple of the 256-wide N tile
    # (exercises the chunk loop, the fp32-accumulate dX epilogue and N tails, as C2/C4 do)
    "bigvocab": dict(hidden=256, vocab=40000, seq_len=128, n_heads=4, n_kv_heads=2, head_dim=64,
                     ffn=512, micro_batch=4, rms_eps=1e-5, rope_theta=10000.0),
    # several 128-query / 128-key attention blocks per sample (causal tiling, lazy
    # rescale and the tcgen05 backward's multi-block loops inside the full step)
    "s384": dict(hidden=256, vocab=2048, seq_len=384, n_heads=4, n_kv_heads=2, head_dim=128,
                 ffn=512, micro_batch=2, rms_eps=1e-5, rope_theta=10000.0),
    # seq_len not a multiple of 128: mma.sync attention fallback, whose backward
    # leaves the inverse RoPE to the standalone kernel (the tcgen05 one fuses it)
    "s192": dict(hidden=256, vocab=2048, seq_len=192, n_heads=4, n_kv_heads=2, head_dim=64,
                ffn=512, micro_batch=3, rms_eps=1e-5, rope_theta=10000.0),
}


def oshape(c):
    return oracle.make_shape(c["hidden"], c["vocab"], c["seq_len"], c["n_heads"], c["n_kv_heads"],
                             c["head_dim"], c["ffn"], c["micro_batch"], eps=c["rms_eps"],
                             theta=c["rope_theta"])


def setup(name, lens, n_present=None):
    c = SHAPES[name]
    shp = oshape(c)
    tr = api.DraftTrainer(c, lr=HP[0], betas=(HP[1], HP[2]), eps=HP[3], weight_decay=HP[4],
                          seed=SEED)
    tr.keep_grads(True)
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 1 << 16)
    samples = []
    for i, L in enumerate(lens):
        cap = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
        buf.append_packed(100 + i, cap["alpha_s"], cap["features"], cap["ids"])
        samples.append((cap["ids"], cap["features"]))
    n = len(lens) if n_present is None else n_present
    F, u, y, m = oracle.gather_batch(shp, samples[:n])
    return c, shp, tr, buf, [100 + i for i in range(n)], (F, u, y, m)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("name", list(SHAPES))
def test_init_is_bit_exact(name):
    c = SHAPES[name]
    shp = oshape(c)
    tr = api.DraftTrainer(c, seed=SEED)
    P = oracle.init_params(shp, SEED)
    layout, total = oracle.param_layout(shp)
    params, t2 = tr.params()
    assert t2 == total and [p[0] for p in params] == [l[0] for l in layout]
    for nm, r, cc, off in layout:
        assert np.array_equal(tr.get_param(nm).reshape(-1), P[off:off + r * cc]), nm
    assert np.array_equal(tr.get_embedding(), oracle.init_embedding(shp, SEED))
    tr.close()


@pytest.mark.parametrize("name", list(SHAPES))
def test_step_matches_oracle(name):
    c = SHAPES[name]
    S, B = c["seq_len"], c["micro_batch"]
    lens = [S + 2] * (B - 2) + [S // 2 + 3, S + 40]
    c, shp, tr, buf, ids, _ = setup(name, lens, n_present=B - 1 if B > 2 else None)
    caps = [oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
            for i, L in enumerate(lens[:len(ids)])]
    samples = [(cp["ids"], cp["features"]) for cp in caps]
    P = oracle.init_params(shp, SEED)
    E = oracle.init_embedding(shp, SEED)
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    well = {}
    for k in (1, 2):
        rep = step_and_compare(tr, buf, ids, shp, samples, P, Mst, Vst, E, k, HP, well=well)
        print(name, k, rep)
    tr.close()
    buf.close()


def test_eval_and_forward_stats():
    c, shp, tr, buf, ids, (F, u, y, m) = setup("C1", [130] * 8)
    P = oracle.init_params(shp, SEED)
    E = oracle.init_embedding(shp, SEED)
    out, lse, am = oracle.forward(shp, P, E, F, u, y, m, round_bf16=True)
    r = tr.eval(buf, ids)
    assert r["valid_tokens"] == out.valid
    assert abs(r["loss"] - out.loss) <= 2e-3 * out.loss
    assert abs(r["loss"] - np.log(c["vocab"])) < 0.5  # near-uniform logits at init
    tr.close()
    buf.close()


def test_train_job_outcome_and_learning():
    c = SHAPES["C1"]
    tr = api.DraftTrainer(c, lr=3e-3, seed=SEED)
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 1 << 16)
    n = 20
    for i in range(n):
        cap = oracle.synth_capture(SEED, i, c["seq_len"] + 2, c["vocab"], c["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
    n_train, n_eval = api.split_train_eval(n)
    before = tr.eval(buf, list(range(8)))
    out = tr.train(buf, list(range(n_train)), list(range(n_train, n)), epochs=3)
    after = tr.eval(buf, list(range(8)))
    assert out.new_version == 1 and out.steps == 3 * ((n_train + 7) // 8)
    assert 0.0 <= out.alpha_eval <= 1.0 and out.duration_hours > 0
    assert after["loss"] < before["loss"]  # memorises the training samples
    out2 = tr.train(buf, [0, 1], [2], epochs=1)
    assert out2.new_version == 2
    with pytest.raises(_lib.DomainError):
        tr.train(buf, [], [1])
    with pytest.raises(_lib.DomainError):
        tr.step(buf, [12345])  # not resident
    tr.close()
    buf.close()


def test_step_is_deterministic():
    c, shp, tr, buf, ids, _ = setup("C1", [130] * 8)
    tr2 = api.DraftTrainer(c, lr=HP[0], betas=(HP[1], HP[2]), seed=SEED)
    tr2.keep_grads(True)
    r1 = tr.step(buf, ids)
    r2 = tr2.step(buf, ids)
    assert r1["loss"] == r2["loss"]
    for nm in ("lm_head", "qkv", "fc", "w_in"):
        assert np.array_equal(tr.get_grad(nm), tr2.get_grad(nm)), nm
    tr.close()
    tr2.close()
    buf.close()


@pytest.mark.parametrize("mode", ["zero", "allreduce"])
def test_fused_adamw_equals_separate_path(monkeypatch, mode):
    """Single replica: AdamW fused into the weight-gradient GEMM epilogue.  The
    data-parallel path is forced with a 1-rank communicator, in both modes:
    ZeRO-1 (per bucket on the comm stream: in-place reduce-scatter, AdamW on
    the rank's shard, in-place all-gather of the bf16 weights) and all-reduce
    (bucketed NCCL all-reduce, standalone AdamW after the join).  All must give
    the same losses and weights over three steps."""
    c = SHAPES["C1"]
    monkeypatch.setenv("SPECSIM_DP_MODE", mode)
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 1 << 16)
    for i in range(8):
        cap = oracle.synth_capture(SEED, i, 130, c["vocab"], c["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
    fused = api.DraftTrainer(c, lr=1e-3, seed=SEED)
    monkeypatch.setenv("SPECSIM_FORCE_NCCL", "1")
    dp = api.DraftTrainer(c, lr=1e-3, seed=SEED)
    monkeypatch.delenv("SPECSIM_FORCE_NCCL")
    for k in range(3):
        ids = [(k * 3 + j) % 8 for j in range(8)]
        r1 = fused.step(buf, ids)
        r2 = dp.step(buf, ids)
        assert abs(r1["loss"] - r2["loss"]) <= 1e-4 * abs(r2["loss"]), (k, r1, r2)
        if k == 0:  # identical inputs: the two AdamW placements agree to fp32 rounding
            for nm in ("fc", "qkv", "o", "gate_up", "down", "lm_head", "w_in", "w_fin"):
                a, b = fused.get_param(nm), dp.get_param(nm)
                assert np.abs(a - b).max() <= 1e-6 * np.abs(b).max() + 1e-9, nm
    with pytest.raises(_lib.DomainError):  # fused path does not keep GEMM-weight grads
        fused.get_grad("lm_head")
    fused.get_grad("w_fin")  # norm-weight grads always exist
    dp.get_grad("lm_head")   # data-parallel path always materialises them
    fused.close(); dp.close(); buf.close()


def test_cuda_graph_replay_equals_eager(monkeypatch):
    """The step is captured once into a CUDA graph and replayed; per-step inputs
    (batch spec, global count, AdamW constants) flow through captured copies
    from pinned staging.  Replays with changing batches must equal eager runs."""
    c = SHAPES["C1"]
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 1 << 16)
    for i in range(12):
        cap = oracle.synth_capture(SEED, i, 60 + 10 * i, c["vocab"], c["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
    g = api.DraftTrainer(c, lr=1e-3, seed=SEED)
    monkeypatch.setenv("SPECSIM_NO_GRAPH", "1")
    e = api.DraftTrainer(c, lr=1e-3, seed=SEED)
    monkeypatch.delenv("SPECSIM_NO_GRAPH")
    batches = [list(range(0, 8)), list(range(4, 12)), [11, 3, 5], list(range(2, 10))]
    for k, ids in enumerate(batches):
        gv = 0 if k != 2 else 777  # caller-provided global count on one step
        r1, r2 = g.step(buf, ids, global_valid=gv), e.step(buf, ids, global_valid=gv)
        assert r1["loss"] == r2["loss"] and r1["valid_tokens"] == r2["valid_tokens"], (k, r1, r2)
        v1, v2 = g.eval(buf, ids[:4]), e.eval(buf, ids[:4])
        assert v1["loss"] == v2["loss"] and v1["top1_correct"] == v2["top1_correct"]
    for nm in ("lm_head", "fc", "w_fin"):
        assert np.array_equal(g.get_param(nm), e.get_param(nm)), nm
    g.set_timing(True)  # a timing graph is captured separately
    r = g.step(buf, batches[0])
    ph = g.phase_times()
    assert ph["gemm"]["ms"] > 0 and ph["lm_head_ce"]["launches"] >= 3
    g.close(); e.close(); buf.close()


def test_all_masked_batch_is_finite():
    """Samples too short to have a target (L <= 2) contribute no valid tokens:
    loss 0, zero gradients, finite parameters afterwards."""
    c = SHAPES["C1"]
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 4096)
    for i, L in enumerate([1, 2]):
        cap = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
        buf.append_packed(i, 0.5, cap["features"], cap["ids"])
    tr = api.DraftTrainer(c, seed=SEED)
    tr.keep_grads(True)
    before = tr.get_param("lm_head")
    r = tr.step(buf, [0, 1])
    assert r["valid_tokens"] == 0 and r["loss"] == 0.0 and r["top1_correct"] == 0
    for nm in ("lm_head", "qkv", "fc", "w_fin"):
        g = tr.get_grad(nm)
        assert np.isfinite(g).all() and np.abs(g).max() == 0.0, nm
    after = tr.get_param("lm_head")
    assert np.isfinite(after).all() and np.array_equal(before, after)
    ev = tr.eval(buf, [0])
    assert ev["valid_tokens"] == 0 and np.isfinite(ev["loss"])
    tr.close(); buf.close()


def test_partial_batch_matches_oracle():
    """n < micro_batch: missing samples are padding rows (zero features, no
    targets); the step equals the oracle's on the same padded batch."""
    c = SHAPES["C1"]
    c, shp, tr, buf, ids, (F, u, y, m) = setup("C1", [130, 90, 130], n_present=3)
    P = oracle.init_params(shp, SEED)
    E = oracle.init_embedding(shp, SEED)
    z = np.zeros_like(P)
    out, grads = oracle.train_step(shp, HP, 1, P, z, z.copy(), E, F, u, y, m, update=False)
    r = tr.step(buf, ids)
    assert r["valid_tokens"] == out.valid == int(m.sum())
    assert abs(r["loss"] - out.loss) <= 2e-3 * out.loss
    layout, _ = oracle.param_layout(shp)
    off = {n: (o, rr * cc) for n, rr, cc, o in layout}
    for nm in ("lm_head", "fc"):
        o, n = off[nm]
        assert rel(tr.get_grad(nm).reshape(-1), grads[o:o + n]) < 1e-2, nm
    tr.close(); buf.close()


@pytest.mark.parametrize("name", ["bigvocab", "gqa128"])
def test_stored_logits_equal_recompute(name, monkeypatch):
    """The default backward reads the logits the forward GEMM stored (fp16
    offsets from each 128-column half tile's row max); the SPECSIM_CE_RECOMPUTE
    path recomputes them chunk by chunk (EPI_CE_BWD) in fp32.  The loss comes
    from the forward's statistics in both (fp32 noise); the gradients differ
    only where the fp16 offset flips a bf16 rounding of the softmax gradient
    (|offset error| <= 2^-11 |l - max|), measured <= 1.3e-3 rel."""
    c = SHAPES[name]
    S, B = c["seq_len"], c["micro_batch"]
    lens = [S + 2] * (B - 1) + [S // 2 + 5]
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("SPECSIM_CE_RECOMPUTE", mode)
        c, shp, tr, buf, ids, _ = setup(name, lens)
        r = tr.step(buf, ids)
        out[mode] = (r["loss"], {nm: tr.get_grad(nm).copy() for nm in ("lm_head", "fc", "qkv")})
        tr.close()
        buf.close()
    (l0, g0), (l1, g1) = out["0"], out["1"]
    assert abs(l0 - l1) <= 1e-6 * abs(l1)
    for nm in g0:
        assert rel(g0[nm], g1[nm]) <= 3e-3, (nm, rel(g0[nm], g1[nm]))
    print(name, {nm: rel(g0[nm], g1[nm]) for nm in g0})


def test_step_matches_oracle_at_bench_model_dims():
    """Parity at the bench workload's model dimensions (C2: H 4096, 3H concat,
    V 128256 = 4 vocabulary chunks with a ragged last one, 32 q / 8 kv heads of
    128, FFN 14336; 818.9 M parameters) on a short batch (S 128, B 2: one full
    sample and one masked tail) so the CPU oracle finishes in seconds.  The
    oracle starts from the trainer's own weights (init is bit-exact, tested
    above at small shapes).  The full-length (S 2048) step is in
    tests/test_parity_large_gpu.py."""
    c = dict(api.CONFIGS["C2"], seq_len=128, micro_batch=2)
    shp = oshape(c)
    tr = api.DraftTrainer(c, lr=HP[0], betas=(HP[1], HP[2]), eps=HP[3], weight_decay=HP[4],
                          seed=SEED)
    tr.keep_grads(True)
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 1 << 12)
    samples = []
    for i, L in enumerate([c["seq_len"] + 2, 77]):
        cap = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
        samples.append((cap["ids"], cap["features"]))
    _, P, E = oracle_state(tr, shp)
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    rep = step_and_compare(tr, buf, [0, 1], shp, samples, P, Mst, Vst, E, 1, HP,
                           sync_weights=False, logit_tol=LARGE_LOGIT_TOL)
    print("C2-dims:", rep)
    tr.close()
    buf.close()


def test_swiglu_backward_epilogue_equals_unfused(monkeypatch):
    """The SwiGLU backward fused into the d act GEMM epilogue (reads gate | up,
    writes d gate | d up) equals the separate kernel over the stored bf16 d act:
    same rounding point, same formula (FMA contraction may differ: 1e-5)."""
    c = SHAPES["C1"]
    lens = [c["seq_len"] + 2] * c["micro_batch"]
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("SPECSIM_SWIGLU_UNFUSED", mode)
        c, shp, tr, buf, ids, _ = setup("C1", lens)
        r = tr.step(buf, ids)
        out[mode] = (r["loss"], {nm: tr.get_grad(nm).copy() for nm in ("gate_up", "qkv", "fc")})
        tr.close()
        buf.close()
    (l0, g0), (l1, g1) = out["0"], out["1"]
    assert l0 == l1
    for nm in g0:
        assert rel(g0[nm], g1[nm]) <= 1e-5, (nm, rel(g0[nm], g1[nm]))


def test_max_batch_rows_split_additivity():
    """Maximum micro-batch (kMaxBatch = 64 sequences, T = 65,536 rows: more rows
    than a CUDA grid's y extent) vs the same rows in four 16-sequence steps
    normalised by the full batch's valid count (`global_valid`): the loss and
    every gradient are additive over rows, so the four parts must sum to the
    full step.  lr = 1e-30 keeps the weights fixed between the steps.  Bound:
    fp32 accumulation order over different row tilings, rel-Frobenius <= 2e-3."""
    c = dict(hidden=256, vocab=4096, seq_len=1024, n_heads=4, n_kv_heads=2, head_dim=64,
             ffn=512, micro_batch=64, rms_eps=1e-5, rope_theta=10000.0)
    L = c["seq_len"] + 2
    buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 64 * L + 1024)
    for i in range(64):
        # ragged tail: a few short samples (masked positions, padding rows)
        n = L if i % 9 else L - 300 - i
        cap = oracle.synth_capture(SEED, i, n, c["vocab"], c["hidden"])
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
    tr = api.DraftTrainer(c, lr=1e-30, seed=SEED)
    tr.keep_grads(True)
    names = ("fc", "qkv", "o", "gate_up", "down", "lm_head", "w_in", "w_hid", "w_post", "w_fin")
    full = tr.step(buf, list(range(64)))
    g_full = {nm: tr.get_grad(nm).astype(np.float64) for nm in names}
    n_valid = full["valid_tokens"]
    assert full["positions"] == 64 * c["seq_len"]
    loss, g_sum, valid = 0.0, {nm: 0.0 for nm in names}, 0
    for q in range(4):
        r = tr.step(buf, list(range(16 * q, 16 * q + 16)), global_valid=n_valid)
        loss += r["loss"]
        valid += r["valid_tokens"]
        for nm in names:
            g_sum[nm] = g_sum[nm] + tr.get_grad(nm).astype(np.float64)
    assert valid == n_valid
    assert abs(loss - full["loss"]) <= 1e-4 * abs(full["loss"]), (loss, full["loss"])
    for nm in names:
        rel = np.linalg.norm(g_sum[nm] - g_full[nm]) / np.linalg.norm(g_full[nm])
        assert rel <= 2e-3, (nm, rel)
    tr.close(); buf.close()


def test_ring_direct_fc_equals_gathered_copy(monkeypatch):
    """The fc GEMMs read the micro-batch's feature rows straight from the
    signal ring (64-row block table + mirrored ring rows); SPECSIM_F_GATHER=1
    copies them into a [T, 3H] buffer first.  Rows past a sample's end hold
    other ring rows on the direct path (zeros on the copy path) but every
    gradient they receive is exactly zero, so the two paths agree bit for bit
    -- here with samples straddling the ring's end, short samples and a
    padding row, over two steps and the training-time-test unroll."""
    for ttt in (1, 2):
        c = dict(SHAPES["s384"], micro_batch=3, ttt_steps=ttt)
        S = c["seq_len"]
        lens = [S + 4, S // 2 + 9, S + 3, 77, S + 10]
        buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 2 * S + 200)
        for i, L in enumerate(lens):  # 0, 1 evicted; 2 straddles the end
            cap = oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"])
            buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
        out = {}
        for mode in ("0", "1"):
            monkeypatch.setenv("SPECSIM_F_GATHER", mode)
            tr = api.DraftTrainer(c, lr=1e-3, seed=SEED)
            tr.keep_grads(True)
            res = []
            for ids in ([2, 3, 4], [3, 4]):
                r = tr.step(buf, ids)
                res.append((r["loss"], {nm: tr.get_grad(nm).copy() for nm, *_ in tr.params()[0]}))
            out[mode] = res
            tr.close()
        for (l0, g0), (l1, g1) in zip(out["0"], out["1"]):
            assert l0 == l1, (ttt, l0, l1)
            for nm in g0:
                assert np.array_equal(g0[nm], g1[nm]), (ttt, nm)
        buf.close()
