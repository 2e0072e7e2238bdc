"""Where does the e2e (host-ingest) leg lose time relative to the resident leg?"""
import ctypes as C, json, sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2602_05145_b200 import _lib, api

cfg = api.CONFIGS["C2"]; B, S, H, V = cfg["micro_batch"], cfg["seq_len"], cfg["hidden"], cfg["vocab"]
L, W, K = S + 2, 3 * H, 16
tr = api.DraftTrainer(cfg, seed=1)
buf = api.HiddenStateBuffer(api.SignalGeometry(H), capacity_tokens=(8 + 3 * K * B) * L)
caps = [api.synth_capture(1, i, L, V, H) for i in range(8)]
pinned = [(torch.from_numpy(c["features"].view(np.int16)).pin_memory(), torch.from_numpy(c["ids"]).pin_memory()) for c in caps]
dev = [(f.cuda(), i.cuda()) for f, i in pinned]
for i, (f, ids) in enumerate(pinned):
    _lib.call("specsim_hsbuf_append_packed", buf.h, i, 0.5, f.data_ptr(), ids.data_ptr(), L, 2)
nid = [100]
def app(mode, n):
    out = []
    for k in range(n):
        f, ids = (dev if mode == 1 else pinned)[k % 8]
        _lib.call("specsim_hsbuf_append_packed", buf.h, nid[0], 0.5, f.data_ptr(), ids.data_ptr(), L, mode)
        out.append(nid[0]); nid[0] += 1
    return out
res = {}
for name in ["resident", "dma_train_on_new", "d2d_train_on_new", "dma_unused", "resident2"]:
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if name.startswith("resident"):
            ids = [k % 8 for k in range(K * B)]
        elif name == "dma_train_on_new":
            ids = app(2, K * B)
        elif name == "d2d_train_on_new":
            ids = app(1, K * B)
        else:
            app(2, K * B); ids = [k % 8 for k in range(K * B)]
        tr.train(buf, ids, [], epochs=1)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    res[name] = round(1e3 * dt / K, 2)
    print(name, res[name], "ms/step", flush=True)
