"""Shared GPU-vs-oracle step comparison (SURVEY §8(d) tolerances).

One optimiser step on both sides from identical weights and identical seeded
captures, then:

* target gather: the device u / y / m (all unroll slices) and the fc input
  rows F equal `oracle.gather_batch` bit for bit;
* top-1: on every row the token the device picked has an oracle logit within
  `logit_tol` of the oracle's maximum, hence the argmax is exact on every row
  whose top-1 / top-2 margin exceeds logit_tol, and the step's top-1 count
  differs from the oracle's by at most the number of valid rows below that
  margin (0 when every valid row is decided).  logit_tol = 1e-2 (SURVEY
  §8(d)) for the small heads; at H >= 4096 the two pipelines' logits differ by
  sigma ~ 1e-2 (both round the same activations to bf16, but fp32 summation
  order flips some roundings and the flips propagate through the layer:
  measured argmax flips at margins up to 0.031 over 4096-row batches at
  C2 / C4 / C5 dims), so those tests use logit_tol = 0.1 (~10 sigma);
* loss rel <= 2e-3, per-row lse within 5e-3;
* every parameter gradient rel-Frobenius <= 1e-2 (x sqrt(H / 4096) above
  H 4096: the bf16-flip noise above grows with the summation lengths --
  measured 0.5-0.7% at C2 dims, 1.1% for fc at C5 dims, i.e. the sqrt(2)
  of H 8192 vs 4096);
* post-AdamW update |dp_gpu - dp_cpu| <= 0.05 lr on >= 99.9% of the elements
  whose oracle gradient is well determined (|g| > 0.05 std: below that the
  sign of g, hence the sign of the first Adam update, is fp32 noise) after
  step 1.  Later steps use the elements well determined at
  every step so far and >= 99% (UPDATE_FRAC_LATER): the update m^/sqrt(v^)
  then divides gradients the two sides computed with independent noise, and
  where successive gradients nearly cancel in m the ratio amplifies that
  noise (measured 99.3-99.5% at the C2 full-sequence step 2, >= 99.98% on
  the small heads).
"""
from __future__ import annotations

import numpy as np

import oracle

MARGIN = 1e-2
LARGE_LOGIT_TOL = 0.1  # H >= 4096 (see above)
UPDATE_FRAC = 0.999
UPDATE_FRAC_LATER = 0.99


def grad_tol_for(hidden):
    return 1e-2 * max(1.0, (hidden / 4096.0) ** 0.5)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def oracle_state(tr, shp):
    """Flat fp32 master vector and bf16 embedding read from the trainer."""
    layout, total = oracle.param_layout(shp)
    P = np.zeros(total, np.float32)
    for nm, rr, cc, off in layout:
        P[off:off + rr * cc] = tr.get_param(nm).reshape(-1)
    return layout, P, tr.get_embedding()


def sample_rows(shp, samples):
    """[B*S] mask of the rows inside a sample (t < L).  The fc GEMMs read the
    features straight from the signal ring, so rows past a sample's end hold
    other ring rows instead of the oracle's zeros; their targets are masked
    (t + 2 >= L), every gradient they receive is exactly zero, and nothing a
    row inside a sample computes depends on them (causal attention): lse /
    argmax / F are compared on these rows."""
    S = shp.S
    ok = np.zeros(shp.B * S, bool)
    for b, (ids, _) in enumerate(samples):
        ok[b * S:b * S + min(S, len(ids))] = True
    return ok


def check_gather(tr, F, u, y, m, rows=None, inside=None):
    """Device gather vs oracle, bit-exact: u / y / m over the first `rows`
    rows (default all unroll slices; an eval fills slice 0 only), the fc
    input rows F on the rows inside a sample (`inside`, default all)."""
    n = len(u) if rows is None else rows
    for nm, ref in (("u", u), ("y", y), ("m", m)):
        got = tr.read_rows(nm)[:n]
        assert np.array_equal(got, ref[:n]), (nm, np.flatnonzero(got != ref[:n])[:8])
    Fg = tr.read_rows("F")
    sel = np.ones(len(F), bool) if inside is None else inside
    assert np.array_equal(Fg[sel], F[sel]), "F rows differ"


def check_top1(tr, r, out, am_o, margin, gap, m, T, logit_tol, rows_ok):
    """gap[row] = oracle max logit - oracle logit at the device's argmax, on
    the rows inside a sample (rows_ok, all unroll slices).  Returns (decided
    rows, ambiguous valid rows, rows whose argmax differs, max gap)."""
    am_g = tr.read_rows("argmax")[:len(am_o)]
    am_g, am_o, margin, gap = am_g[rows_ok], am_o[rows_ok], margin[rows_ok], gap[rows_ok]
    far = np.flatnonzero(~(gap <= logit_tol))
    assert far.size == 0, ("device argmax not a near-maximum", far[:8], gap[far[:8]])
    sure = margin > logit_tol
    assert np.array_equal(am_g[sure], am_o[sure])
    valid0 = (m[:T] == 1)[rows_ok[:T]]
    ambiguous = int((valid0 & ~sure[:len(valid0)]).sum())
    assert abs(r["top1_correct"] - out.top1) <= ambiguous, (r["top1_correct"], out.top1, ambiguous)
    if ambiguous == 0:
        assert r["top1_correct"] == out.top1
    return int(sure.sum()), ambiguous, int((am_g != am_o).sum()), float(np.nanmax(gap))


def step_and_compare(tr, buf, ids, shp, samples, P, Mst, Vst, E, k, hp, *, grad_tol=None,
                     check_update=True, sync_weights=True, logit_tol=MARGIN, well=None):
    """One step on the trainer and the oracle (in place on P / Mst / Vst).
    `well` (dict, kept by the caller across steps) accumulates the
    well-determined element masks.  Returns a report dict."""
    layout, _ = oracle.param_layout(shp)
    if grad_tol is None:
        grad_tol = grad_tol_for(shp.H)
    F, u, y, m = oracle.gather_batch(shp, samples)
    T = shp.B * shp.S
    r = tr.step(buf, ids)
    am_g = tr.read_rows("argmax")
    lse_g = tr.read_rows("lse")
    # oracle forward on the pre-step weights, probing the device's argmax
    _, lse_o, am_o, margin, gap = oracle.forward(shp, P, E, F, u, y, m, round_bf16=True,
                                                margin=True, probe=am_g)
    P0 = P.copy()
    out, grads = oracle.train_step(shp, hp, k, P, Mst, Vst, E, F, u, y, m, round_bf16=True,
                                   update=check_update)
    inside = sample_rows(shp, samples)
    rows_ok = np.tile(inside, len(am_o) // T)  # every unroll slice
    check_gather(tr, F, u, y, m, inside=inside)
    assert r["valid_tokens"] == int(m[:T].sum()) == out.valid
    assert r["positions"] == T
    assert abs(r["loss"] - out.loss) <= 2e-3 * max(abs(out.loss), 1e-30), (r["loss"], out.loss)
    lse_err = float(np.abs(lse_g[:len(lse_o)] - lse_o)[rows_ok].max())
    assert lse_err <= 5e-3 * max(1.0, logit_tol / MARGIN), lse_err
    decided, ambiguous, differ, max_gap = check_top1(tr, r, out, am_o, margin, gap, m, T,
                                                     logit_tol, rows_ok)
    report = dict(loss_gpu=r["loss"], loss_cpu=out.loss, lse_err=lse_err, decided_rows=decided,
                  ambiguous_valid_rows=ambiguous, argmax_differs=differ, max_gap=max_gap,
                  top1=(r["top1_correct"], out.top1), grads={}, update_frac={})
    if well is None:
        well = {}
    bad = []
    for nm, rr, cc, off in layout:
        g_cpu = grads[off:off + rr * cc]
        e = rel(tr.get_grad(nm).reshape(-1), g_cpu)
        report["grads"][nm] = round(e, 6)
        if e > grad_tol:
            bad.append((k, nm, e))
        if check_update:
            d_gpu = tr.get_param(nm).reshape(-1) - P0[off:off + rr * cc]
            d_cpu = P[off:off + rr * cc] - P0[off:off + rr * cc]
            w = np.abs(g_cpu) > 0.05 * np.abs(g_cpu).std() + 1e-12
            well[nm] = w if nm not in well else (well[nm] & w)
            w = well[nm]
            if w.sum() > 0:
                frac = float((np.abs(d_gpu - d_cpu)[w] <= 0.05 * hp[0]).mean())
                report["update_frac"][nm] = round(frac, 6)
                if frac < (UPDATE_FRAC if k == 1 else UPDATE_FRAC_LATER):
                    bad.append((k, nm, "update", frac))
            if sync_weights:  # identical weights for the next step
                tr.set_param(nm, P[off:off + rr * cc].reshape(rr, cc))
    assert not bad, (bad, report)
    return report
