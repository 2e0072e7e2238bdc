"""Causal GQA attention kernels (forward + backward) vs a float64 numpy
statement of the same maths on identical bf16 inputs."""
import numpy as np
import pytest

from paper_2602_05145_b200 import _lib
from _util import rand_bf16, bf16_bits_to_f32

pytestmark = pytest.mark.gpu


def ref(qkv, dO, B, S, nh, nkv, hd):
    Q, KV = nh * hd, nkv * hd
    x = qkv.astype(np.float64).reshape(B, S, -1)
    q = x[..., :Q].reshape(B, S, nh, hd).transpose(0, 2, 1, 3)
    k = x[..., Q:Q + KV].reshape(B, S, nkv, hd).transpose(0, 2, 1, 3)
    v = x[..., Q + KV:].reshape(B, S, nkv, hd).transpose(0, 2, 1, 3)
    rep = nh // nkv
    k = np.repeat(k, rep, axis=1)
    v = np.repeat(v, rep, axis=1)
    sc = q @ k.transpose(0, 1, 3, 2) / np.sqrt(hd)
    mask = np.triu(np.ones((S, S), bool), 1)
    sc = np.where(mask, -np.inf, sc)
    mx = sc.max(-1, keepdims=True)
    e = np.exp(sc - mx)
    l = e.sum(-1, keepdims=True)
    p = e / l
    o = p @ v
    lse = (mx + np.log(l))[..., 0]  # [B, nh, S]
    do = dO.astype(np.float64).reshape(B, S, nh, hd).transpose(0, 2, 1, 3)
    dp = do @ v.transpose(0, 1, 3, 2)
    D = (do * o).sum(-1, keepdims=True)
    ds = p * (dp - D) / np.sqrt(hd)
    dq = ds @ k
    dk = (ds.transpose(0, 1, 3, 2) @ q).reshape(B, nkv, rep, S, hd).sum(2)
    dv = (p.transpose(0, 1, 3, 2) @ do).reshape(B, nkv, rep, S, hd).sum(2)
    O = o.transpose(0, 2, 1, 3).reshape(B * S, Q)
    dQ = dq.transpose(0, 2, 1, 3).reshape(B * S, Q)
    dK = dk.transpose(0, 2, 1, 3).reshape(B * S, KV)
    dV = dv.transpose(0, 2, 1, 3).reshape(B * S, KV)
    LSE = lse.transpose(1, 0, 2).reshape(nh, B * S)
    return O, LSE, np.concatenate([dQ, dK, dV], axis=1)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


# S % 128 == 0 runs the tcgen05 forward (attention_tc.cu); other lengths the
# mma.sync fallback.  S = 1024 exercises many KV blocks and the lazy rescale.
@pytest.mark.parametrize("B,S,nh,nkv,hd", [(2, 128, 4, 2, 64), (1, 256, 8, 2, 128), (2, 192, 4, 4, 128),
                                           (1, 64, 2, 1, 64), (1, 1024, 4, 1, 128), (2, 512, 4, 2, 64)])
def test_attention_fwd_bwd(B, S, nh, nkv, hd):
    rng = np.random.default_rng(B * 1000 + S + nh)
    NQ = (nh + 2 * nkv) * hd
    qkv_bits, qkv = rand_bf16(rng, (B * S, NQ))
    do_bits, do = rand_bf16(rng, (B * S, nh * hd))
    o = np.zeros((B * S, nh * hd), np.uint16)
    lse = np.zeros((nh, B * S), np.float32)
    dqkv = np.zeros((B * S, NQ), np.uint16)
    _lib.call("specsim_debug_attention", B, S, nh, nkv, hd, _lib.ptr(qkv_bits), _lib.ptr(do_bits),
              _lib.ptr(o), _lib.ptr(lse), _lib.ptr(dqkv))
    O, LSE, dQKV = ref(qkv, do, B, S, nh, nkv, hd)
    assert rel(bf16_bits_to_f32(o), O) < 1e-2
    np.testing.assert_allclose(lse, LSE, rtol=1e-4, atol=1e-3)
    g = bf16_bits_to_f32(dqkv)
    Q, KV = nh * hd, nkv * hd
    assert rel(g[:, :Q], dQKV[:, :Q]) < 2e-2
    assert rel(g[:, Q:Q + KV], dQKV[:, Q:Q + KV]) < 2e-2
    assert rel(g[:, Q + KV:], dQKV[:, Q + KV:]) < 2e-2


def ref_by_head(qkv, dO, S, nh, nkv, hd):
    """float64 reference one head at a time (B = 1): S x S score matrices only,
    so S = 4096 with 64 heads fits in host memory."""
    Q, KV, rep = nh * hd, nkv * hd, nh // nkv
    x = qkv.astype(np.float64)
    do_all = dO.astype(np.float64)
    O = np.zeros((S, Q))
    LSE = np.zeros((nh, S))
    dQKV = np.zeros((S, Q + 2 * KV))
    mask = np.triu(np.ones((S, S), bool), 1)
    for h in range(nh):
        kv = h // rep
        q = x[:, h * hd:(h + 1) * hd]
        k = x[:, Q + kv * hd:Q + (kv + 1) * hd]
        v = x[:, Q + KV + kv * hd:Q + KV + (kv + 1) * hd]
        sc = np.where(mask, -np.inf, q @ k.T / np.sqrt(hd))
        mx = sc.max(-1, keepdims=True)
        p = np.exp(sc - mx)
        l = p.sum(-1, keepdims=True)
        p /= l
        o = p @ v
        O[:, h * hd:(h + 1) * hd] = o
        LSE[h] = (mx + np.log(l))[:, 0]
        do = do_all[:, h * hd:(h + 1) * hd]
        ds = p * (do @ v.T - (do * o).sum(-1, keepdims=True)) / np.sqrt(hd)
        dQKV[:, h * hd:(h + 1) * hd] = ds @ k
        dQKV[:, Q + kv * hd:Q + (kv + 1) * hd] += ds.T @ q
        dQKV[:, Q + KV + kv * hd:Q + KV + (kv + 1) * hd] += p.T @ do
    return O, LSE, dQKV


# The large configurations' head geometry at their full sequence lengths: C2
# (S 2048, 32 q / 8 kv heads, GQA group 4: 16 key blocks per query block) and
# C4 / C5 (S 4096, 64 q / 8 kv heads, GQA group 8: 32 key blocks).
@pytest.mark.parametrize("S,nh,nkv", [(2048, 32, 8), (4096, 64, 8)])
def test_attention_large_configs(S, nh, nkv):
    hd = 128
    rng = np.random.default_rng(S + nh)
    NQ = (nh + 2 * nkv) * hd
    qkv_bits, qkv = rand_bf16(rng, (S, NQ))
    do_bits, do = rand_bf16(rng, (S, nh * hd))
    o = np.zeros((S, nh * hd), np.uint16)
    lse = np.zeros((nh, S), np.float32)
    dqkv = np.zeros((S, NQ), np.uint16)
    _lib.call("specsim_debug_attention", 1, S, nh, nkv, hd, _lib.ptr(qkv_bits), _lib.ptr(do_bits),
              _lib.ptr(o), _lib.ptr(lse), _lib.ptr(dqkv))
    O, LSE, dQKV = ref_by_head(qkv, do, S, nh, nkv, hd)
    assert rel(bf16_bits_to_f32(o), O) < 1e-2
    np.testing.assert_allclose(lse, LSE, rtol=1e-4, atol=1e-3)
    g = bf16_bits_to_f32(dqkv)
    Q, KV = nh * hd, nkv * hd
    errs = [rel(g[:, :Q], dQKV[:, :Q]), rel(g[:, Q:Q + KV], dQKV[:, Q:Q + KV]),
            rel(g[:, Q + KV:], dQKV[:, Q + KV:])]
    print(S, nh, nkv, "dq/dk/dv rel", errs)
    assert max(errs) < 2e-2


def test_attention_rejects_bad_shapes():
    z = np.zeros(16, np.uint16)
    f = np.zeros(16, np.float32)
    with pytest.raises(_lib.DomainError):
        _lib.call("specsim_debug_attention", 1, 100, 2, 1, 64, _lib.ptr(z), None, _lib.ptr(z),
                  _lib.ptr(f), None)


def test_large_logit_range_rescale():
    """Scores that grow along the sequence force the lazy O rescale path."""
    B, S, nh, nkv, hd = 1, 512, 2, 1, 128
    rng = np.random.default_rng(7)
    NQ = (nh + 2 * nkv) * hd
    x = rng.standard_normal((B * S, NQ)).astype(np.float32)
    ramp = np.linspace(0.5, 6.0, S, dtype=np.float32)[:, None]
    x[:, nh * hd:(nh + nkv) * hd] *= ramp  # keys get larger later -> row max keeps growing
    x[:, :nh * hd] *= 2.0
    from _util import f32_to_bf16_bits
    bits = f32_to_bf16_bits(x)
    q = bf16_bits_to_f32(bits)
    do_bits, do = rand_bf16(rng, (B * S, nh * hd))
    o = np.zeros((B * S, nh * hd), np.uint16)
    lse = np.zeros((nh, B * S), np.float32)
    _lib.call("specsim_debug_attention", B, S, nh, nkv, hd, _lib.ptr(bits), None,
              _lib.ptr(o), _lib.ptr(lse), None)
    O, LSE, _ = ref(q, do, B, S, nh, nkv, hd)
    assert rel(bf16_bits_to_f32(o), O) < 1e-2
    np.testing.assert_allclose(lse, LSE, rtol=1e-4, atol=2e-3)


_TWO_TILE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
from paper_2602_05145_b200 import _lib
from _util import rand_bf16
B, S, nh, nkv, hd = (int(x) for x in sys.argv[3:8])
rng = np.random.default_rng(11)
NQ = (nh + 2 * nkv) * hd
qkv_bits, _ = rand_bf16(rng, (B * S, NQ))
do_bits, _ = rand_bf16(rng, (B * S, nh * hd))
o = np.zeros((B * S, nh * hd), np.uint16)
lse = np.zeros((nh, B * S), np.float32)
dqkv = np.zeros((B * S, NQ), np.uint16)
_lib.call("specsim_debug_attention", B, S, nh, nkv, hd, _lib.ptr(qkv_bits), _lib.ptr(do_bits),
          _lib.ptr(o), _lib.ptr(lse), _lib.ptr(dqkv))
np.savez(sys.argv[2], o=o, lse=lse)
"""


@pytest.mark.parametrize("B,S,nh,nkv,hd", [(2, 512, 8, 2, 128), (1, 1024, 4, 2, 64),
                                           (1, 2048, 32, 8, 128)])
def test_two_tile_forward_bit_identical_to_one_tile(tmp_path, B, S, nh, nkv, hd):
    """The default forward (attn_fwd2_tc_kernel: a head pair per CTA, P in TMEM)
    runs the same per-row arithmetic in the same order as the one-tile kernel
    (SPECSIM_ATTN_FWD1=1), so O and lse must match bit for bit."""
    import os
    import pathlib
    import subprocess
    import sys
    root = pathlib.Path(__file__).resolve().parents[1]
    script = tmp_path / "fwd.py"
    script.write_text(_TWO_TILE_SCRIPT)
    outs = {}
    for one in ("0", "1"):
        out = tmp_path / f"fwd{one}.npz"
        env = dict(os.environ, SPECSIM_ATTN_FWD1=one)
        r = subprocess.run([sys.executable, str(script), str(root), str(out), str(B), str(S),
                            str(nh), str(nkv), str(hd)], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[one] = np.load(out)
    assert np.array_equal(outs["0"]["o"], outs["1"]["o"])
    assert np.array_equal(outs["0"]["lse"], outs["1"]["lse"])
