"""Hidden-state buffer: per-verify-step extract_signals appends (host and
device layer tensors), packing bit-exact, byte accounting vs the oracle's
restatement of SPEC.md:267-275, eviction and ring wrap."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2602_05145_b200 import _lib, api

pytestmark = pytest.mark.gpu
H = 64


def verify_steps(seed, index, length, gamma=3):
    """Simulate capture: per verify step gamma+1 candidate rows per layer,
    the first k (sampled accept length) accepted."""
    cap = oracle.synth_capture(seed, index, length, 1000, H)
    rng = np.random.default_rng(index)
    steps = []
    pos = 0
    for k in cap["accept_lengths"]:
        rows = gamma + 1
        layers = [rng.integers(0, 1 << 16, (rows, H), dtype=np.uint16) for _ in range(3)]
        # place the sample's packed features into the accepted rows (in a permuted order)
        perm = rng.permutation(rows)[:k]
        for i in range(k):
            f = cap["features"][pos + i]
            for l in range(3):
                layers[l][perm[i]] = f[l * H:(l + 1) * H]
        steps.append((layers, cap["ids"][pos:pos + k], perm.astype(np.int32)))
        pos += k
    return cap, steps


@pytest.mark.parametrize("on_device", [False, True])
def test_extract_signals_pack_bit_exact(on_device):
    buf = api.HiddenStateBuffer(api.SignalGeometry(H), 4096, flush_threshold=1 << 14)
    st = np.zeros(4, np.int64)
    bpt = 3 * H * 2
    keep = []
    for sid in range(5):
        cap, steps = verify_steps(7, sid, 37 + 13 * sid)
        for layers, ids, idx in steps:
            if on_device:
                import torch
                tl = [torch.from_numpy(l.view(np.int16)).cuda() for l in layers]
                keep.append(tl)
                arr = (C.c_void_p * 3)(*[t.data_ptr() for t in tl])
                idn = np.ascontiguousarray(ids, np.int32)
                _lib.call("specsim_hsbuf_append", buf.h, sid, cap["alpha_s"],
                          C.cast(arr, C.POINTER(C.c_void_p)), layers[0].shape[0], H,
                          _lib.ptr(idn), _lib.ptr(idx), len(idn), 1)
            else:
                buf.extract_signals(sid, cap["alpha_s"], layers, ids, accepted_idx=idx)
            oracle.lib().orc_extract_signals(C.c_void_p(st.ctypes.data), len(ids), bpt, 1 << 14)
        f, ids = buf.read_sample(sid)
        assert np.array_equal(f, cap["features"]), sid
        assert np.array_equal(ids, cap["ids"])
        n, a = buf.sample_info(sid)
        assert n == len(cap["ids"]) and a == cap["alpha_s"]
    s = buf.stats()
    assert [s["records"], s["bytes"], s["flushes"], s["cumulative_bytes"]] == list(st)
    assert s["samples"] == 5
    assert s["bytes"] + s["cumulative_bytes"] == s["records"] * bpt
    buf.close()


def test_ring_wrap_and_eviction():
    buf = api.HiddenStateBuffer(api.SignalGeometry(H), 300)
    caps = []
    for sid in range(8):
        cap = oracle.synth_capture(3, sid, 70 + sid, 1000, H)
        buf.append_packed(sid, 0.5, cap["features"], cap["ids"])
        caps.append(cap)
    # capacity 300 tokens: only the newest samples survive, possibly wrapped
    st = buf.stats()
    assert st["resident_tokens"] <= 300
    with pytest.raises(_lib.DomainError):
        buf.sample_info(0)
    for sid in (6, 7):
        f, ids = buf.read_sample(sid)
        assert np.array_equal(f, caps[sid]["features"])
        assert np.array_equal(ids, caps[sid]["ids"])
    with pytest.raises(_lib.DomainError):  # closed samples cannot be reopened
        buf.append_packed(6, 0.5, caps[6]["features"][:1], caps[6]["ids"][:1])
    with pytest.raises(_lib.DomainError):
        buf.append_packed(99, 0.5, np.zeros((301, 3 * H), np.uint16), np.zeros(301, np.int32))
    buf.close()


def test_validation_errors():
    with pytest.raises(_lib.DomainError):
        api.HiddenStateBuffer(api.SignalGeometry(60), 100)  # not a multiple of 8
    buf = api.HiddenStateBuffer(api.SignalGeometry(H), 100)
    with pytest.raises(_lib.DomainError):
        buf.extract_signals(1, 1.5, [np.zeros((4, H), np.uint16)] * 3, [1, 2])
    with pytest.raises(_lib.DomainError):
        buf.extract_signals(1, 0.5, [np.zeros((4, H), np.uint16)] * 3, [1, 2], accepted_idx=[0, 9])
    buf.close()


def test_async_pinned_append_feeds_the_step():
    """mode 2 (pinned host, asynchronous DMA) must be ordered before the step
    that consumes it: a step on asynchronously appended samples equals a step on
    synchronously appended copies."""
    import torch
    cfg = dict(api.CONFIGS["C1"], micro_batch=2)
    buf = api.HiddenStateBuffer(api.SignalGeometry(cfg["hidden"]), 8192)
    pins = []
    for i in range(2):
        cap = oracle.synth_capture(11, i, cfg["seq_len"] + 2, cfg["vocab"], cfg["hidden"])
        buf.append_packed(i, 0.5, cap["features"], cap["ids"])  # mode 0
        f = torch.from_numpy(cap["features"].view(np.int16)).pin_memory()
        ids = torch.from_numpy(cap["ids"]).pin_memory()
        pins.append((f, ids))
        _lib.call("specsim_hsbuf_append_packed", buf.h, 10 + i, 0.5, f.data_ptr(), ids.data_ptr(),
                  len(cap["ids"]), 2)
    t1 = api.DraftTrainer(cfg, seed=1)
    t2 = api.DraftTrainer(cfg, seed=1)
    t1.keep_grads(True)
    t2.keep_grads(True)
    r1 = t1.step(buf, [0, 1])
    r2 = t2.step(buf, [10, 11])
    assert r1["loss"] == r2["loss"]
    assert np.array_equal(t1.get_grad("fc"), t2.get_grad("fc"))
    f, ids = buf.read_sample(11)
    assert np.array_equal(f.view(np.int16), pins[1][0].numpy())
    with pytest.raises(_lib.DomainError):  # pageable memory is rejected for mode 2
        z = np.zeros((4, 3 * cfg["hidden"]), np.uint16)
        zi = np.zeros(4, np.int32)
        _lib.call("specsim_hsbuf_append_packed", buf.h, 99, 0.5, z.ctypes.data, zi.ctypes.data, 4, 2)
    t1.close(); t2.close(); buf.close()
