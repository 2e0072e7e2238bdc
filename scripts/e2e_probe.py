"""Where the e2e leg's extra time goes (C2, 20 steps, jobs of 5 steps as in
bench.py): (a) bench's e2e leg (pinned-host appends of job i+1 issued before
job i trains); (b) the same jobs on samples already resident (no DMA, same
host / job structure); (c) one 20-step job on resident samples (the value
leg).  Device time of the region on the trainer stream, ms per step."""
import json
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib, api  # noqa: E402

cfg = api.CONFIGS["C2"]
B, S, H, V = cfg["micro_batch"], cfg["seq_len"], cfg["hidden"], cfg["vocab"]
L, W = S + 2, 3 * H
STEPS, JOB = 20, 5
tr = api.DraftTrainer(cfg, seed=1)
pool_n = 2 * B
buf = api.HiddenStateBuffer(api.SignalGeometry(H), capacity_tokens=(pool_n + (2 * JOB + 1) * B) * L)
caps = [api.synth_capture(1, i, L, V, H) for i in range(pool_n)]
pinned = []
for c in caps:
    t = torch.empty((L, W), dtype=torch.int16, pin_memory=True)
    t.numpy()[:] = c["features"].view(np.int16)
    ids = torch.empty(L, dtype=torch.int32, pin_memory=True)
    ids.numpy()[:] = c["ids"]
    pinned.append((t, ids))
nid = [0]


def append_job(n, mode):
    base = nid[0]
    for k in range(n * B):
        t, ids = pinned[k % pool_n]
        _lib.call("specsim_hsbuf_append_packed", buf.h, base + k, 0.5, t.data_ptr(),
                  ids.data_ptr(), L, mode)
    nid[0] += n * B
    return list(range(base, base + n * B))


def region(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.region_begin()
    fn()
    ms = tr.region_end()
    return ms / STEPS, 1e3 * (time.perf_counter() - t0) / STEPS


def leg_e2e():
    pend = append_job(JOB, 2)
    for i in range(STEPS // JOB):
        nxt = append_job(JOB, 2) if i + 1 < STEPS // JOB else None
        tr.train(buf, pend, [], epochs=1)
        pend = nxt


def leg_jobs_resident():
    ids = append_job(JOB, 0)  # resident before the region
    torch.cuda.synchronize()
    return ids


out = {}
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for _ in range(3):
        tr.train(buf, append_job(JOB, 0), [], epochs=1)  # warm-up
    out[f"a_e2e_{rep}"] = region(leg_e2e)
    ids = leg_jobs_resident()
    out[f"b_jobs_resident_{rep}"] = region(
        lambda: [tr.train(buf, ids, [], epochs=1) for _ in range(STEPS // JOB)])
    out[f"c_one_job_resident_{rep}"] = region(
        lambda: tr.train(buf, ids * (STEPS // JOB), [], epochs=1))
print(json.dumps({k: dict(device_ms_per_step=round(v[0], 3), wall_ms_per_step=round(v[1], 3))
                  for k, v in out.items()}, indent=1))
