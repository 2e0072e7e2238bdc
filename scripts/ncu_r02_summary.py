"""Summarise the round-2 ncu metric captures of one draft-training step
(scripts/ncu_r02.sh) into profiles/r02_*.{json,txt}.

* HBM-bound kernels (gather, norms, SwiGLU, CE reduce / gradient, attention
  D, standalone AdamW): per launch DRAM bytes read + written (ncu), duration,
  achieved GB/s against MEASURED_PEAKS.json hbm_gbs, and the algorithmic
  bytes per launch (DESIGN.md §3 per-token figures x tokens) with the
  measured / algorithmic ratio.
* GEMMs: per launch FLOPs, duration, SM clock, FLOP-derived tensor
  utilisation (FLOPs / (148 SMs x 8192 FLOP/clk x clock x time), the dense
  bf16 tcgen05 rate per SM) next to the candidate ncu tensor-pipe counters, so
  the counter that measures the tcgen05 pipe is the one that agrees.

Usage: python scripts/ncu_r02_summary.py <step.csv> <adamw.csv> <config> <out_prefix>
(the CSVs are `ncu --csv --page raw` logs of scripts/step_probe.py).
"""
import csv
import io
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1,
         "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
         "Kcycle/second": 1e3, "Mcycle/second": 1e6, "Gcycle/second": 1e9, "%": 1, "cycle": 1,
         "inst": 1, "": 1}
PIPE = ["sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed"]


def load(path):
    """Rows of an `ncu --csv --page raw` log (one row per kernel launch)."""
    text = pathlib.Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"name": r[hdr.index("Kernel Name")]}
        for i, h in enumerate(hdr):
            if "__" not in h:
                continue
            try:
                d[h] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
            except ValueError:
                pass
        out.append(d)
    return out


def short(name):
    """kernel name without namespaces / parameters, template arguments kept"""
    n = name.split("(")[0].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    n = n.replace("void ", "").strip()
    head, _, tmpl = n.partition("<")
    return head.split("::")[-1] + (("<" + tmpl) if tmpl else "")


def last_step(rows):
    """Launches of the last complete step: from the last gather kernel to
    the end (the step's trailing store_mapped included)."""
    idx = [i for i, r in enumerate(rows)
           if "gather_batch_kernel" in r["name"] or "gather_tokens_kernel" in r["name"]]
    if not idx:
        raise SystemExit("no gather kernel launch in the capture")
    return rows[idx[-1]:]


def algorithmic(cfg, T):
    """Per-call algorithmic bytes of the step's HBM-bound kernels, in call
    order (trainer.cu forward / backward, single pass), DESIGN.md §3."""
    H, V, I = cfg["hidden"], cfg["vocab"], cfg["ffn"]
    Q = cfg["n_heads"] * cfg["head_dim"]
    nh = cfg["n_heads"]
    W3 = 3 * H
    Vc = min(32768, V)
    nb = (V + 255) // 256
    nbT = (T + 15) // 16  # rmsnorm_bwd weight-gradient partial rows
    norm_fwd = 4 * H * T + 4 * T
    a = {
        "gather_batch_kernel": [("ring -> F rows + u/y/m", 2 * W3 * 2 * T + 8 * T + 12 * T)],
        # u / y / m of one pass + the ids they read + the 64-row block table
        "gather_tokens_kernel": [("ring ids -> u/y/m + block table", 24 * T + 4 * (T // 64))],
        "rmsnorm_fwd_kernel": [("a = RMSNorm(E[u])", norm_fwd), ("b = RMSNorm(g)", norm_fwd),
                               ("z = RMSNorm(r)", norm_fwd), ("n = RMSNorm(h)", norm_fwd)],
        "swiglu_fwd_kernel": [("act = silu(g) u", 6 * I * T)],
        "ce_reduce_kernel": [("partials -> lse/loss/argmax", 2 * nb * T * 16 + 8 * T + 12 * T)],
        "attn_bwd_dot_kernel": [("D = rowsum(dO o)", 4 * Q * T + 4 * nh * T)],
        "rmsnorm_bwd_kernel": [
            ("w_fin: dn, h -> dh, dh_b", 12 * H * T + 4 * nbT * H),
            ("w_post: dz, r, +dh -> dr, dr_b", 16 * H * T + 4 * nbT * H),
            ("w_in: dU, E[u] (dw only)", 6 * H * T + 4 * nbT * H),
            ("w_hid: dU, g, +dr -> dg_b", 12 * H * T + 4 * nbT * H)],
        "colsum_kernel": [("norm dw partials", 4 * nbT * H + 4 * H)] * 4,
    }
    ce = []
    for v0 in range(0, V, Vc):
        vn = min(Vc, V - v0)
        ce.append((f"chunk {v0 // Vc}: fp16 logits -> bf16 dlogits",
                   2 * vn * T + (vn // 128) * T * 16 + 12 * T + 2 * vn * T))
    a["ce_grad_kernel"] = ce
    return a


def gemm_list(cfg, T):
    H, V, I = cfg["hidden"], cfg["vocab"], cfg["ffn"]
    Q = cfg["n_heads"] * cfg["head_dim"]
    KV = cfg["n_kv_heads"] * cfg["head_dim"]
    Vc = min(32768, V)
    L = [("fc fwd", T, H, 3 * H), ("qkv fwd + RoPE", T, Q + 2 * KV, 2 * H),
         ("o fwd + residual", T, H, Q), ("gate_up fwd", T, 2 * I, H),
         ("down fwd + residual", T, H, I), ("LM head CE fwd (stats + fp16 logits)", T, V, H)]
    for c in range(0, V, Vc):
        vn = min(Vc, V - c)
        L += [(f"LM head dX chunk {c // Vc}", T, H, vn),
              (f"LM head dW chunk {c // Vc} + AdamW", vn, H, T)]
    L += [("dact (down dX) + SwiGLU bwd", T, I, H), ("down dW + AdamW", H, I, T),
          ("dz (gate_up dX)", T, H, 2 * I), ("gate_up dW + AdamW", 2 * I, H, T),
          ("dO (o dX)", T, Q, H), ("o dW + AdamW", H, Q, T),
          ("dU (qkv dX)", T, 2 * H, Q + 2 * KV), ("qkv dW + AdamW", Q + 2 * KV, 2 * H, T),
          ("fc dW + AdamW", H, 3 * H, T)]
    return L


def gemm_alg_bytes(label, M, N, K, cfg):
    """Operands once (bf16) + the epilogue's own traffic per output element."""
    ab = 2.0 * (M * K + N * K)
    if "AdamW" in label:
        per = 26  # p, m, v read; p, m, v, bf16 p written (fp32 except p16)
    elif "CE fwd" in label:
        per = 2  # fp16 logits (+ per-tile partials below)
        ab += 2 * ((N + 255) // 256) * M * 16
    elif "SwiGLU" in label:
        per = 8  # gate | up read, d gate | d up written (bf16, two per output)
    elif "residual" in label:
        per = 4  # residual read + bf16 out
    elif "dX chunk" in label:
        per = 4 if label.endswith("0") else 8  # fp32 store; later chunks accumulate (read + write)
    elif label.startswith(("dz", "dU")):
        per = 4  # fp32 out
    else:
        per = 2  # bf16 out
    return ab + per * M * N


def main(step_csv, adamw_csv, config, prefix):
    from paper_2602_05145_b200 import api
    cfg = api.CONFIGS[config]
    T = cfg["micro_batch"] * cfg["seq_len"]
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    hbm = peaks["hbm_gbs"]
    rows = last_step(load(step_csv))
    alg = algorithmic(cfg, T)
    seen = {}
    hbm_rows, gemm_rows = [], []
    gl = iter(gemm_list(cfg, T))
    for r in rows:
        nm = short(r["name"])
        base = nm.split("<")[0]
        t = r.get("gpu__time_duration.sum", 0.0)
        rd, wr = r.get("dram__bytes_read.sum", 0.0), r.get("dram__bytes_write.sum", 0.0)
        clk = r.get("sm__cycles_elapsed.avg.per_second", 0.0)
        if base == "gemm_kernel":
            label, M, N, K = next(gl)
            fl = 2.0 * M * N * K
            ab = gemm_alg_bytes(label, M, N, K, cfg)
            util = fl / (t * 148 * 8192 * clk) if t and clk else None
            gemm_rows.append(dict(launch=label, kernel=nm, M=M, N=N, K=K, ms=round(t * 1e3, 4),
                                  tflops=round(fl / t / 1e12, 1), sm_ghz=round(clk / 1e9, 3),
                                  flop_util_pct=round(100 * util, 1) if util else None,
                                  dram_gb=round((rd + wr) / 1e9, 3),
                                  algorithmic_gb=round(ab / 1e9, 3),
                                  dram_over_algorithmic=round((rd + wr) / ab, 2),
                                  **{p.split(".")[0]: r.get(p) for p in PIPE}))
            continue
        k = seen.get(base, 0)
        seen[base] = k + 1
        if base not in alg:
            continue
        lst = alg[base]
        what, ab = lst[k] if k < len(lst) else (f"call {k}", None)
        hbm_rows.append(dict(kernel=nm, call=what, us=round(t * 1e6, 2),
                             dram_read_mb=round(rd / 1e6, 2), dram_write_mb=round(wr / 1e6, 2),
                             achieved_gbs=round((rd + wr) / t / 1e9, 1) if t else None,
                             frac_of_hbm_peak=round((rd + wr) / t / 1e9 / hbm, 3) if t else None,
                             algorithmic_mb=round(ab / 1e6, 2) if ab else None,
                             dram_over_algorithmic=round((rd + wr) / ab, 3) if ab else None,
                             sm_ghz=round(clk / 1e9, 3)))
    if adamw_csv and pathlib.Path(adamw_csv).exists():
        ad = [r for r in load(adamw_csv) if "adamw_kernel" in r["name"]]
        if ad:
            r = ad[-1]
            n = sum(rr * cc for rr, cc in api_param_shapes(cfg))
            t = r["gpu__time_duration.sum"]
            rd, wr = r.get("dram__bytes_read.sum", 0.0), r.get("dram__bytes_write.sum", 0.0)
            ab = 30 * n
            hbm_rows.append(dict(kernel=short(r["name"]),
                                 call=f"standalone AdamW over all {n / 1e6:.1f} M params "
                                      "(SPECSIM_NO_FUSED_ADAMW=1; the default fuses it into the "
                                      "dW GEMM epilogues)",
                                 us=round(t * 1e6, 2), dram_read_mb=round(rd / 1e6, 2),
                                 dram_write_mb=round(wr / 1e6, 2),
                                 achieved_gbs=round((rd + wr) / t / 1e9, 1),
                                 frac_of_hbm_peak=round((rd + wr) / t / 1e9 / hbm, 3),
                                 algorithmic_mb=round(ab / 1e6, 2),
                                 dram_over_algorithmic=round((rd + wr) / ab, 3),
                                 sm_ghz=round(r.get("sm__cycles_elapsed.avg.per_second", 0) / 1e9, 3)))
    note = (f"ncu --clock-control none metric capture of one {config} step (the second of "
            "scripts/step_probe.py); kernels serialised and replayed per metric pass, cold L2: "
            "absolute times are not step times, bytes and rates are the signal. "
            f"HBM peak {hbm} GB/s = MEASURED_PEAKS.json hbm_gbs (copy bandwidth).")
    out = dict(note=note, config=config, tokens=T, hbm_peak_gbs=hbm, hbm_kernels=hbm_rows,
               gemms=gemm_rows)
    pathlib.Path(prefix + ".json").write_text(json.dumps(out, indent=1))
    lines = [note, "", f"{'kernel / call':58s} {'us':>8s} {'GB/s':>7s} {'%pk':>5s} "
             f"{'DRAM MB':>9s} {'alg MB':>9s} {'ratio':>6s}"]
    for h in hbm_rows:
        lines.append(f"{(h['kernel'][:22] + ' ' + h['call'])[:58]:58s} {h['us']:8.1f} "
                     f"{h['achieved_gbs'] or 0:7.0f} {100 * (h['frac_of_hbm_peak'] or 0):5.1f} "
                     f"{h['dram_read_mb'] + h['dram_write_mb']:9.1f} "
                     f"{h['algorithmic_mb'] or 0:9.1f} {h['dram_over_algorithmic'] or 0:6.2f}")
    lines += ["", f"{'GEMM':40s} {'ms':>7s} {'TF/s':>7s} {'GHz':>5s} {'flop%':>6s} "
              f"{'DRAM GB':>8s} {'alg GB':>7s} {'ratio':>5s} "
              + " ".join(f"{p.split('.')[0].replace('sm__', '')[:22]:>22s}" for p in PIPE)]
    for g in gemm_rows:
        lines.append(f"{g['launch'][:40]:40s} {g['ms']:7.3f} {g['tflops']:7.1f} {g['sm_ghz']:5.2f} "
                     f"{g['flop_util_pct'] or 0:6.1f} {g['dram_gb']:8.2f} {g['algorithmic_gb']:7.2f} "
                     f"{g['dram_over_algorithmic']:5.2f} "
                     + " ".join(f"{(g[p.split('.')[0]] or 0):22.1f}" for p in PIPE))
    pathlib.Path(prefix + ".txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def api_param_shapes(cfg):
    H, V, I = cfg["hidden"], cfg["vocab"], cfg["ffn"]
    Q = cfg["n_heads"] * cfg["head_dim"]
    KV = cfg["n_kv_heads"] * cfg["head_dim"]
    return [(H, 3 * H), (1, H), (1, H), (Q + 2 * KV, 2 * H), (H, Q), (1, H), (2 * I, H), (H, I),
            (1, H), (V, H)]


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", sys.argv[3] if len(sys.argv) > 3
         else "C2", sys.argv[4] if len(sys.argv) > 4 else "profiles/r02_step_ncu")
