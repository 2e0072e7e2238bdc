"""The C oracle's draft-head step (round_bf16 = 0, pure fp32) vs an independent
torch autograd statement: loss, every parameter gradient, and the AdamW update
(torch.optim.AdamW).  Pins the oracle's maths (the reference has none)."""
import numpy as np
import pytest
import torch

import oracle
from torch_ref import forward_loss

SHAPES = [
    dict(H=64, V=512, S=32, nh=4, nkv=2, hd=16, I=128, B=2),
    dict(H=32, V=128, S=16, nh=2, nkv=1, hd=16, I=64, B=3),
]


def build(sh, seed, lens):
    shp = oracle.make_shape(**sh)
    P = oracle.init_params(shp, seed)
    E = oracle.init_embedding(shp, seed)
    samples = []
    for b, L in enumerate(lens):
        c = oracle.synth_capture(seed, b, L, shp.V, shp.H)
        samples.append((c["ids"], c["features"]))
    F, u, y, m = oracle.gather_batch(shp, samples)
    return shp, P, E, F, u, y, m


def torch_params(shp, P):
    layout, _ = oracle.param_layout(shp)
    W = {}
    for name, r, c, off in layout:
        t = torch.from_numpy(P[off:off + r * c].reshape(r, c).copy())
        if name.startswith("w_"):
            t = t.reshape(c)
        W[name] = t.requires_grad_(True)
    return W, layout


@pytest.mark.parametrize("sh", SHAPES)
def test_step_matches_torch(sh):
    lens = [sh["S"] + 2] * (sh["B"] - 1) + [sh["S"] // 2]  # one short (masked tail) sample
    shp, P, E, F, u, y, m = build(sh, 11, lens)
    hp = [1e-3, 0.9, 0.95, 1e-8, 0.01]
    Pc = P.copy()
    mst = np.zeros_like(P)
    vst = np.zeros_like(P)
    out, grads = oracle.train_step(shp, hp, 1, Pc, mst, vst, E, F, u, y, m, round_bf16=False)

    W, layout = torch_params(shp, P)
    Et = torch.from_numpy(oracle.bf16_to_f32(E).reshape(shp.V, shp.H))
    Ft = torch.from_numpy(oracle.bf16_to_f32(F).reshape(F.shape))
    loss, _ = forward_loss(shp, W, Et, Ft, torch.from_numpy(u).long(), torch.from_numpy(y),
                           torch.from_numpy(m), 0)
    loss.backward()
    assert out.valid == int(m.sum())
    assert abs(out.loss - loss.item()) <= 1e-5 * abs(loss.item())
    for name, r, c, off in layout:
        gt = W[name].grad.numpy().reshape(-1)
        go = grads[off:off + r * c]
        rel = np.linalg.norm(go - gt) / max(np.linalg.norm(gt), 1e-30)
        assert rel < 2e-4, (name, rel)

    opt = torch.optim.AdamW(list(W.values()), lr=hp[0], betas=(hp[1], hp[2]), eps=hp[3],
                            weight_decay=hp[4])
    opt.step()
    for name, r, c, off in layout:
        pt = W[name].detach().numpy().reshape(-1)
        po = Pc[off:off + r * c]
        # update ~ lr * sign(g): compare updates relative to lr where grads are well determined
        gt = W[name].grad.numpy().reshape(-1)
        ok = np.abs(gt) > 1e-3 * np.abs(gt).max()
        d = np.abs((po - P[off:off + r * c]) - (pt - P[off:off + r * c]))
        assert (d[ok] <= 1e-2 * hp[0]).mean() >= 0.999, name


def test_forward_stats_match_torch():
    sh = SHAPES[0]
    shp, P, E, F, u, y, m = build(sh, 5, [sh["S"] + 2, 10])
    out, lse, am = oracle.forward(shp, P, E, F, u, y, m, round_bf16=False)
    W, _ = torch_params(shp, P)
    Et = torch.from_numpy(oracle.bf16_to_f32(E).reshape(shp.V, shp.H))
    Ft = torch.from_numpy(oracle.bf16_to_f32(F).reshape(F.shape))
    loss, logits = forward_loss(shp, W, Et, Ft, torch.from_numpy(u).long(), torch.from_numpy(y),
                                torch.from_numpy(m), 0)
    np.testing.assert_allclose(lse, torch.logsumexp(logits, -1).detach().numpy(), rtol=1e-5, atol=1e-5)
    srt = torch.sort(logits, -1, descending=True).values.detach().numpy()
    clear = (srt[:, 0] - srt[:, 1]) > 1e-4
    assert (am[clear] == logits.argmax(-1).numpy()[clear]).all()
    assert abs(out.loss - loss.item()) < 1e-5 * abs(loss.item())


def test_bf16_rounding_mode_is_close():
    sh = SHAPES[0]
    shp, P, E, F, u, y, m = build(sh, 9, [sh["S"] + 2] * sh["B"])
    hp = [1e-3, 0.9, 0.95, 1e-8, 0.0]
    z = np.zeros_like(P)
    o32, g32 = oracle.train_step(shp, hp, 1, P.copy(), z.copy(), z.copy(), E, F, u, y, m,
                                 round_bf16=False, update=False)
    o16, g16 = oracle.train_step(shp, hp, 1, P.copy(), z.copy(), z.copy(), E, F, u, y, m,
                                 round_bf16=True, update=False)
    assert abs(o16.loss - o32.loss) < 2e-3 * o32.loss
    assert np.linalg.norm(g16 - g32) / np.linalg.norm(g32) < 3e-2


@pytest.mark.parametrize("sh,K", [(SHAPES[0], 3), (SHAPES[1], 2)])
def test_ttt_step_matches_torch(sh, K):
    """Training-time-test unroll (K steps): C oracle (fp32) vs torch autograd of
    the SpecForge-layout restatement (tests/torch_ref.forward_loss_ttt)."""
    from torch_ref import forward_loss_ttt
    sh = dict(sh, ttt=K)
    # one full-length sample, one whose shifted masks run out at different steps
    lens = [sh["S"] + 2 + K] * (sh["B"] - 1) + [sh["S"] // 2 + 1]
    shp, P, E, F, u, y, m = build(sh, 13, lens)
    assert u.size == K * sh["B"] * sh["S"]
    hp = [1e-3, 0.9, 0.95, 1e-8, 0.01]
    z = np.zeros_like(P)
    out, grads = oracle.train_step(shp, hp, 1, P.copy(), z.copy(), z.copy(), E, F, u, y, m,
                                   round_bf16=False, update=False)
    W, layout = torch_params(shp, P)
    Et = torch.from_numpy(oracle.bf16_to_f32(E).reshape(shp.V, shp.H))
    Ft = torch.from_numpy(oracle.bf16_to_f32(F).reshape(F.shape))
    loss, logits = forward_loss_ttt(shp, W, Et, Ft, torch.from_numpy(u).long(),
                                    torch.from_numpy(y), torch.from_numpy(m), 0, K)
    loss.backward()
    T = sh["B"] * sh["S"]
    assert out.valid == int(m[:T].sum())
    assert abs(out.loss - loss.item()) <= 1e-5 * abs(loss.item()), (out.loss, loss.item())
    for name, r, c, off in layout:
        gt = W[name].grad.numpy().reshape(-1)
        go = grads[off:off + r * c]
        rel = np.linalg.norm(go - gt) / max(np.linalg.norm(gt), 1e-30)
        assert rel < 2e-4, (name, rel)
    o2, lse, am = oracle.forward(shp, P, E, F, u, y, m, round_bf16=False)
    np.testing.assert_allclose(lse, torch.logsumexp(logits, -1).detach().numpy(), rtol=1e-5,
                               atol=1e-5)
    assert abs(o2.loss - out.loss) <= 1e-9 * abs(out.loss)


def test_ttt_gather_shifts():
    """Slice j of u / y / m is the step-0 rule shifted by j tokens (bit-exact)."""
    sh = dict(SHAPES[1], ttt=3)
    shp = oracle.make_shape(**sh)
    L = [sh["S"] + 4, 7, 0]
    samples = [(np.arange(100, 100 + n, dtype=np.int32), np.zeros((n, 3 * sh["H"]), np.uint16))
               for n in L]
    F, u, y, m = oracle.gather_batch(shp, samples)
    S, T = sh["S"], sh["B"] * sh["S"]
    for j in range(3):
        for b, n in enumerate(L):
            for t in range(S):
                r = j * T + b * S + t
                assert m[r] == (t + 2 + j < n)
                assert y[r] == (100 + t + 2 + j if t + 2 + j < n else 0)
                assert u[r] == (100 + t + 1 + j if t + 1 + j < n else 0)
