"""Independent fp32 torch-autograd statement of the draft-head step
 used to cross-check the C oracle.  CPU only."""
import math

import numpy as np
import torch


def rope_tables(S, hd, theta):
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    inv = np.power(theta, -2.0 * i / hd)
    ang = np.arange(S, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


def rot(x, cos, sin):
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def forward_loss(shp, W, E, F, u, y, m, global_valid):
    H, V, S, nh, nkv, hd, I, B = shp.H, shp.V, shp.S, shp.nh, shp.nkv, shp.hd, shp.I, shp.B
    Q, KV = nh * hd, nkv * hd
    T = B * S
    eps = shp.eps

    def rms(x, w):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w

    g = F @ W["fc"].T
    e = E[u]
    U = torch.cat([rms(e, W["w_in"]), rms(g, W["w_hid"])], dim=-1)
    qkv = U @ W["qkv"].T
    cos, sin = rope_tables(S, hd, shp.theta)
    q = qkv[:, :Q].view(B, S, nh, hd)
    k = qkv[:, Q:Q + KV].view(B, S, nkv, hd)
    v = qkv[:, Q + KV:].view(B, S, nkv, hd)
    q = rot(q, cos[None, :, None, :], sin[None, :, None, :]).permute(0, 2, 1, 3)
    k = rot(k, cos[None, :, None, :], sin[None, :, None, :]).permute(0, 2, 1, 3)
    v = v.permute(0, 2, 1, 3)
    rep = nh // nkv
    k = k.repeat_interleave(rep, dim=1)
    v = v.repeat_interleave(rep, dim=1)
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool), 1)
    sc = sc.masked_fill(mask, float("-inf"))
    o = (torch.softmax(sc, dim=-1) @ v).permute(0, 2, 1, 3).reshape(T, Q)
    r = g + o @ W["o"].T
    z = rms(r, W["w_post"])
    gu = z @ W["gate_up"].T
    act = torch.nn.functional.silu(gu[:, :I]) * gu[:, I:]
    h = r + act @ W["down"].T
    n = rms(h, W["w_fin"])
    logits = n @ W["lm_head"].T
    lse = torch.logsumexp(logits, dim=-1)
    tl = logits.gather(1, y[:, None].long())[:, 0]
    mf = m.float()
    denom = float(global_valid) if global_valid > 0 else max(1.0, float(mf.sum()))
    loss = ((lse - tl) * mf).sum() / denom
    return loss, logits


def forward_loss_ttt(shp, W, E, F, u, y, m, global_valid, K, decay=0.8):
    """Training-time-test unroll in the layout of SpecForge's EAGLE-3 trainer
    (independent restatement, [EXT]): per unroll step the layer appends its
    k / v to a cache; attention scores are the causal scores against cache[0]
    concatenated with one diagonal score per later cache entry, softmaxed
    together; RoPE positions are offset by the cache length; the next step's
    hidden input is this step's layer output.  u / y / m: [K * T] (slice j
    shifted by j tokens).  loss = sum_j decay^j * CE_j / N (N = valid count of
    step 0)."""
    H, V, S, nh, nkv, hd, I, B = shp.H, shp.V, shp.S, shp.nh, shp.nkv, shp.hd, shp.I, shp.B
    Q, KV = nh * hd, nkv * hd
    T = B * S
    eps = shp.eps
    rep = nh // nkv

    def rms(x, w):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w

    cos, sin = rope_tables(S + K - 1, hd, shp.theta)
    hidden = F @ W["fc"].T
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool), 1)
    cache_k, cache_v = [], []
    m0 = m[:T].float()
    denom = float(global_valid) if global_valid > 0 else max(1.0, float(m0.sum()))
    total = 0.0
    logits_all = []
    for j in range(K):
        uj, yj, mj = u[j * T:(j + 1) * T], y[j * T:(j + 1) * T], m[j * T:(j + 1) * T]
        e = E[uj]
        Uc = torch.cat([rms(e, W["w_in"]), rms(hidden, W["w_hid"])], dim=-1)
        qkv = Uc @ W["qkv"].T
        c = cos[j:j + S][None, :, None, :]
        s_ = sin[j:j + S][None, :, None, :]
        q = rot(qkv[:, :Q].view(B, S, nh, hd), c, s_).permute(0, 2, 1, 3)
        k = rot(qkv[:, Q:Q + KV].view(B, S, nkv, hd), c, s_).permute(0, 2, 1, 3)
        v = qkv[:, Q + KV:].view(B, S, nkv, hd).permute(0, 2, 1, 3)
        cache_k.append(k.repeat_interleave(rep, dim=1))
        cache_v.append(v.repeat_interleave(rep, dim=1))
        w0 = (q @ cache_k[0].transpose(-1, -2)) / math.sqrt(hd)
        w0 = w0.masked_fill(mask, float("-inf"))
        cols = [w0] + [((q * cache_k[i]).sum(-1) / math.sqrt(hd))[..., None]
                       for i in range(1, len(cache_k))]
        p = torch.softmax(torch.cat(cols, dim=-1), dim=-1)
        o = p[..., :S] @ cache_v[0]
        for i in range(1, len(cache_k)):
            o = o + p[..., S + i - 1:S + i] * cache_v[i]
        o = o.permute(0, 2, 1, 3).reshape(T, Q)
        r = hidden + o @ W["o"].T
        z = rms(r, W["w_post"])
        gu = z @ W["gate_up"].T
        act = torch.nn.functional.silu(gu[:, :I]) * gu[:, I:]
        h = r + act @ W["down"].T
        logits = rms(h, W["w_fin"]) @ W["lm_head"].T
        lse = torch.logsumexp(logits, dim=-1)
        tl = logits.gather(1, yj[:, None].long())[:, 0]
        wj = float(np.float32(decay ** j))
        total = total + wj * (((lse - tl) * mj.float()).sum() / denom)
        logits_all.append(logits)
        hidden = h
    return total, torch.cat(logits_all, 0)
