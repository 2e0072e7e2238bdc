"""Where the end-to-end leg of bench.py spends its time at 10 steps: host time
issuing the asynchronous pinned appends, then train(job) wall time, vs the
same job on resident samples."""
import json
import sys
import pathlib
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib, api  # noqa: E402

cfg = api.CONFIGS["C2"]
B, S, H, V = cfg["micro_batch"], cfg["seq_len"], cfg["hidden"], cfg["vocab"]
L, W, K = S + 2, 3 * H, 10
tr = api.DraftTrainer(cfg, seed=1)
pool = 2 * B
buf = api.HiddenStateBuffer(api.SignalGeometry(H), capacity_tokens=(pool + 7 * K * B) * L)
caps = [api.synth_capture(1, i, L, V, H) for i in range(pool)]
pinned = []
for c in caps:
    t = torch.empty((L, W), dtype=torch.int16, pin_memory=True)
    t.numpy()[:] = c["features"].view(np.int16)
    ids = torch.empty(L, dtype=torch.int32, pin_memory=True)
    ids.numpy()[:] = c["ids"]
    pinned.append((t, ids))
for i, (t, ids) in enumerate(pinned):
    _lib.call("specsim_hsbuf_append_packed", buf.h, i, 0.5, t.data_ptr(), ids.data_ptr(), L, 0)
nid = [1000]


def appends(n):
    out = []
    for k in range(n * B):
        t, ids = pinned[k % pool]
        _lib.call("specsim_hsbuf_append_packed", buf.h, nid[0], 0.5, t.data_ptr(), ids.data_ptr(),
                  L, 2)
        out.append(nid[0])
        nid[0] += 1
    return out


res = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.train(buf, [k % pool for k in range(K * B)], [], epochs=1)
    t1 = time.perf_counter()
    res["resident_ms"] = round(1e3 * (t1 - t0), 2)
    t0 = time.perf_counter()
    ids = appends(K)
    t1 = time.perf_counter()
    tr.train(buf, ids, [], epochs=1)
    t2 = time.perf_counter()
    res["append_issue_ms"] = round(1e3 * (t1 - t0), 2)
    res["train_after_appends_ms"] = round(1e3 * (t2 - t1), 2)
    res["e2e_ms"] = round(1e3 * (t2 - t0), 2)
# copy engine alone: the K steps' appends with nothing else running
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    appends(K)
    torch.cuda.synchronize()
    res["dma_only_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
res["h2d_GBps"] = round(K * B * L * (2 * W + 4) / res["dma_only_ms"] / 1e6, 1)
# resident job while the DMA of a later job streams in (no dependency)
torch.cuda.synchronize()
t0 = time.perf_counter()
appends(K)
tr.train(buf, [k % pool for k in range(K * B)], [], epochs=1)
res["resident_with_concurrent_dma_ms"] = round(1e3 * (time.perf_counter() - t0), 2)
print(json.dumps(res))
