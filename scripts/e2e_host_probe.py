"""Host-side cost at a train(job) boundary of the bench's e2e leg (C2): the
20 pinned-host appends of a 5-step job (append_packed mode 2) and the
train(job) call itself vs its device time."""
import json, pathlib, sys, time
import numpy as np
import torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib, api  # noqa: E402

cfg = api.CONFIGS["C2"]
B, S, H, V = cfg["micro_batch"], cfg["seq_len"], cfg["hidden"], cfg["vocab"]
L, W, JOB = S + 2, 3 * H, 5
tr = api.DraftTrainer(cfg, seed=1)
buf = api.HiddenStateBuffer(api.SignalGeometry(H), capacity_tokens=(3 * JOB + 2) * B * L)
caps = [api.synth_capture(1, i, L, V, H) for i in range(2 * B)]
pinned = []
for c in caps:
    t = torch.empty((L, W), dtype=torch.int16, pin_memory=True)
    t.numpy()[:] = c["features"].view(np.int16)
    ids = torch.empty(L, dtype=torch.int32, pin_memory=True)
    ids.numpy()[:] = c["ids"]
    pinned.append((t, ids))
nid = [0]
def append_job(n):
    base = nid[0]
    for k in range(n * B):
        t, ids = pinned[k % len(pinned)]
        _lib.call("specsim_hsbuf_append_packed", buf.h, base + k, 0.5, t.data_ptr(), ids.data_ptr(), L, 2)
    nid[0] += n * B
    return list(range(base, base + n * B))
out = {}
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ids = append_job(JOB); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    tr.region_begin(); t3 = time.perf_counter(); o = tr.train(buf, ids, [], epochs=1); t4 = time.perf_counter()
    dev = tr.region_end()
    out[rep] = dict(append_host_ms=round(1e3 * (t1 - t0), 2), append_dma_ms=round(1e3 * (t2 - t0), 2),
                    train_host_ms=round(1e3 * (t4 - t3), 2), train_device_ms=round(dev, 2))
print(json.dumps(out, indent=1))
