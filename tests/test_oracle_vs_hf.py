"""The C oracle's draft-head step (fp32) vs the same EAGLE-3 head composed from
HuggingFace transformers' Llama building blocks -- LlamaRMSNorm,
LlamaRotaryEmbedding + apply_rotary_pos_emb (rotate-half RoPE), repeat_kv +
eager_attention_forward (GQA), LlamaMLP (SwiGLU) -- the modules SpecForge's
EAGLE-3 draft model is built from.  Pins the layer conventions the oracle
restates (RMSNorm, RoPE pairing and angles, GQA head grouping, SwiGLU order)
to that public implementation, independently of tests/torch_ref.py."""
import types

import numpy as np
import pytest
import torch

import oracle

transformers = pytest.importorskip("transformers")
from transformers.models.llama import modeling_llama as ml  # noqa: E402

SHAPES = [
    dict(H=64, V=512, S=32, nh=4, nkv=2, hd=16, I=128, B=2),
    dict(H=64, V=256, S=16, nh=8, nkv=2, hd=8, I=96, B=2),
]


def hf_head(shp, P, E):
    layout, _ = oracle.param_layout(shp)
    W = {}
    for name, r, c, off in layout:
        t = torch.from_numpy(P[off:off + r * c].reshape(r, c).copy())
        W[name] = (t.reshape(c) if name.startswith("w_") else t).requires_grad_(True)
    H, nh, nkv, hd, I = shp.H, shp.nh, shp.nkv, shp.hd, shp.I
    Q, KV = nh * hd, nkv * hd
    cfg = ml.LlamaConfig(hidden_size=H, intermediate_size=I, num_attention_heads=nh,
                         num_key_value_heads=nkv, head_dim=hd, rms_norm_eps=shp.eps,
                         rope_theta=shp.theta, max_position_embeddings=4 * shp.S,
                         attention_bias=False, mlp_bias=False, hidden_act="silu",
                         vocab_size=shp.V)
    rotary = ml.LlamaRotaryEmbedding(cfg)
    norms = {n: ml.LlamaRMSNorm(H, eps=shp.eps) for n in ("w_in", "w_hid", "w_post", "w_fin")}
    mlp = ml.LlamaMLP(cfg)
    attn_mod = types.SimpleNamespace(num_key_value_groups=nh // nkv, training=False)
    Et = torch.from_numpy(oracle.bf16_to_f32(E).reshape(shp.V, H))

    def rms(name, x):
        # LlamaRMSNorm with a unit weight (its own normalisation code), scaled
        # by our leaf so the weight gradient lands on it
        n = norms[name]
        with torch.no_grad():
            n.weight.fill_(1.0)
        return W[name] * n(x)

    def forward(F, u, y, m):
        B, S = shp.B, shp.S
        g = F @ W["fc"].T
        e = Et[u]
        U = torch.cat([rms("w_in", e), rms("w_hid", g)], -1)
        q = (U @ W["qkv"][:Q].T).view(B, S, nh, hd).transpose(1, 2)
        k = (U @ W["qkv"][Q:Q + KV].T).view(B, S, nkv, hd).transpose(1, 2)
        v = (U @ W["qkv"][Q + KV:].T).view(B, S, nkv, hd).transpose(1, 2)
        pos = torch.arange(S)[None].expand(B, S)
        cos, sin = rotary(v, pos)
        q, k = ml.apply_rotary_pos_emb(q, k, cos, sin)
        mask = torch.full((S, S), float("-inf")).triu(1)[None, None]
        o, _ = ml.eager_attention_forward(attn_mod, q, k, v, mask, scaling=hd ** -0.5)
        o = o.reshape(B * S, Q)
        r = g + o @ W["o"].T
        mlp.gate_proj.weight = torch.nn.Parameter(W["gate_up"][:I], requires_grad=False)
        mlp.up_proj.weight = torch.nn.Parameter(W["gate_up"][I:], requires_grad=False)
        mlp.down_proj.weight = torch.nn.Parameter(W["down"], requires_grad=False)
        z = rms("w_post", r)
        # LlamaMLP(z) = down(silu(gate(z)) * up(z)), evaluated with our leaves
        act = mlp.act_fn(z @ W["gate_up"][:I].T) * (z @ W["gate_up"][I:].T)
        assert torch.allclose(mlp(z), act @ W["down"].T, rtol=1e-5, atol=1e-6)
        h = r + act @ W["down"].T
        logits = rms("w_fin", h) @ W["lm_head"].T
        lse = torch.logsumexp(logits, -1)
        tl = logits.gather(1, y[:, None].long())[:, 0]
        mf = m.float()
        return ((lse - tl) * mf).sum() / max(1.0, float(mf.sum()))

    return W, layout, forward


@pytest.mark.parametrize("sh", SHAPES)
def test_oracle_matches_hf_llama_modules(sh):
    shp = oracle.make_shape(**sh, theta=500000.0)
    P = oracle.init_params(shp, 17)
    E = oracle.init_embedding(shp, 17)
    samples = []
    for b, L in enumerate([sh["S"] + 2, sh["S"] // 2]):
        c = oracle.synth_capture(17, b, L, shp.V, shp.H)
        samples.append((c["ids"], c["features"]))
    F, u, y, m = oracle.gather_batch(shp, samples)
    z = np.zeros_like(P)
    out, grads = oracle.train_step(shp, [1e-3, 0.9, 0.95, 1e-8, 0.0], 1, P.copy(), z.copy(),
                                   z.copy(), E, F, u, y, m, round_bf16=False, update=False)
    W, layout, fwd = hf_head(shp, P, E)
    loss = fwd(torch.from_numpy(oracle.bf16_to_f32(F).reshape(F.shape)),
               torch.from_numpy(u).long(), torch.from_numpy(y), torch.from_numpy(m))
    loss.backward()
    assert abs(out.loss - loss.item()) <= 1e-5 * abs(loss.item()), (out.loss, loss.item())
    for name, r, c, off in layout:
        gt = W[name].grad.numpy().reshape(-1)
        go = grads[off:off + r * c]
        rel = np.linalg.norm(go - gt) / max(np.linalg.norm(gt), 1e-30)
        assert rel < 2e-4, (name, rel)
