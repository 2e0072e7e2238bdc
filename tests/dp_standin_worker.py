"""World-2 data-parallel step on ONE GPU through the in-process NCCL stand-in
(tests/nccl_standin): two DraftTrainers (rank 0 and rank 1) on two host
threads, each with its own signal buffer, exchange gradients through the
library's real data-parallel code path (trainer.cu bucket_ready /
sync_master: ZeRO-1 reduce-scatter -> shard AdamW -> all-gather, or bucketed
all-reduce + AdamW).  Run as a subprocess by tests/test_dp_standin_gpu.py
(SPECSIM_NCCL_LIB must be set before the library first resolves NCCL, and
SPECSIM_NO_GRAPH=1 because the stand-in cannot be captured).

Prints one JSON line: per step, both ranks' loss / valid counts and the max
difference between the ranks' weights, and the oracle comparison of rank 0's
weights against the single-process step on the whole global batch.
"""
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_2602_05145_b200 import api  # noqa: E402

SEED = 20260217
HP = [1e-3, 0.9, 0.95, 1e-8, 0.0]
WORLD = 2


def main():
    ttt = int(os.environ.get("STANDIN_TTT", "1"))
    steps = int(os.environ.get("STANDIN_STEPS", "2"))
    c = dict(api.CONFIGS["C1"], micro_batch=3, ttt_steps=ttt)
    S, B = c["seq_len"], c["micro_batch"]
    n_samples = WORLD * B * steps - 1  # last global step is partial (rank 1 gets a short slice)
    lens = [(S + 2 + ttt) if i % 4 else (S // 2 + 7) for i in range(n_samples)]
    caps = [oracle.synth_capture(SEED, i, L, c["vocab"], c["hidden"]) for i, L in enumerate(lens)]
    nid = api.DraftTrainer.nccl_unique_id()
    trainers, bufs, errs = [None] * WORLD, [None] * WORLD, []
    step_res = [[None] * WORLD for _ in range(steps)]
    params = [[None] * WORLD for _ in range(steps)]
    names = ("fc", "w_in", "w_hid", "qkv", "o", "w_post", "gate_up", "down", "w_fin", "lm_head")
    barrier = threading.Barrier(WORLD)

    def rank_main(r):
        try:
            buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), sum(lens) + 1024)
            for i, cp in enumerate(caps):
                buf.append_packed(i, cp["alpha_s"], cp["features"], cp["ids"])
            bufs[r] = buf
            tr = api.DraftTrainer(c, lr=HP[0], betas=(HP[1], HP[2]), eps=HP[3],
                                  weight_decay=HP[4], seed=SEED, rank=r, world=WORLD,
                                  nccl_id=nid)
            trainers[r] = tr
            for k in range(steps):
                mine = api.dp_shard(n_samples, B, WORLD, r, k)
                step_res[k][r] = dict(tr.step(buf, mine), mine=mine)
                barrier.wait()
                # get_param all-gathers the ZeRO-1 fp32 master shards: collective,
                # every rank calls it in the same order
                params[k][r] = {nm: tr.get_param(nm) for nm in names}
        except Exception as e:  # surfaced in the JSON line
            errs.append(f"rank {r}: {type(e).__name__}: {e}")
            try:
                barrier.abort()
            except Exception:
                pass

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(WORLD)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        print(json.dumps({"error": errs}))
        return
    # oracle: single process, whole global batch per step (B_global = WORLD * B)
    shp = oracle.make_shape(c["hidden"], c["vocab"], S, c["n_heads"], c["n_kv_heads"],
                            c["head_dim"], c["ffn"], WORLD * B, eps=c["rms_eps"],
                            theta=c["rope_theta"], ttt=ttt)
    P = oracle.init_params(shp, SEED)
    E = oracle.init_embedding(shp, SEED)
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    layout, _ = oracle.param_layout(shp)
    out_steps, well = [], {}
    for k in range(steps):
        ids = sorted(step_res[k][0]["mine"] + step_res[k][1]["mine"])
        F, u, y, m = oracle.gather_batch(shp, [(caps[i]["ids"], caps[i]["features"]) for i in ids])
        P0 = P.copy()
        o, grads = oracle.train_step(shp, HP, k + 1, P, Mst, Vst, E, F, u, y, m)
        rec = dict(loss=[step_res[k][r]["loss"] for r in range(WORLD)],
                   valid=[step_res[k][r]["valid_tokens"] for r in range(WORLD)],
                   mine=[step_res[k][r]["mine"] for r in range(WORLD)],
                   oracle_loss=o.loss, oracle_valid=o.valid, rank_param_maxdiff=0.0,
                   update_frac={}, master_rel={})
        for nm, rr, cc, off in layout:
            a0, a1 = params[k][0][nm].reshape(-1), params[k][1][nm].reshape(-1)
            rec["rank_param_maxdiff"] = max(rec["rank_param_maxdiff"], float(np.abs(a0 - a1).max()))
            g = grads[off:off + rr * cc]
            w = np.abs(g) > 0.05 * np.abs(g).std() + 1e-12
            well[nm] = w if nm not in well else (well[nm] & w)
            d_gpu = a0 - P0[off:off + rr * cc]
            d_cpu = P[off:off + rr * cc] - P0[off:off + rr * cc]
            if well[nm].sum():
                rec["update_frac"][nm] = float(
                    (np.abs(d_gpu - d_cpu)[well[nm]] <= 0.05 * HP[0]).mean())
            rec["master_rel"][nm] = float(np.linalg.norm(a0 - P[off:off + rr * cc]) /
                                          np.linalg.norm(P[off:off + rr * cc]))
        out_steps.append(rec)
        # identical weights on both sides for the next step
        for nm, rr, cc, off in layout:
            P[off:off + rr * cc] = params[k][0][nm].reshape(-1)
    for t in trainers:
        t.close()
    for b in bufs:
        b.close()
    print(json.dumps({"steps": out_steps}))


if __name__ == "__main__":
    main()
