"""Where does the value leg lose time vs single steps?  Times the same C2
workload as (a) K step() calls, (b) one train(job) of K steps, (c) K timed
single steps (phase events), alternating, on one trainer."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_05145_b200 import _lib, api  # noqa: E402

cfg = api.CONFIGS[os.environ.get("CFG", "C2")]
B, S, H, V = cfg["micro_batch"], cfg["seq_len"], cfg["hidden"], cfg["vocab"]
tr = api.DraftTrainer(cfg, seed=1)
L = S + 2
buf = api.HiddenStateBuffer(api.SignalGeometry(H), capacity_tokens=4 * B * L)
for i in range(2 * B):
    c = api.synth_capture(1, i, L, V, H)
    buf.append_packed(i, c["alpha_s"], c["features"], c["ids"])
K = int(os.environ.get("K", "20"))


def batch(k):
    return [(k * B + j) % (2 * B) for j in range(B)]


for k in range(10):
    tr.step(buf, batch(k))
torch.cuda.synchronize()
for rep in range(2):
    tr.region_begin()
    for k in range(K):
        tr.step(buf, batch(k))
    a = tr.region_end() / K
    job = api.global_job(K, B, 1, lambda r, k, j: (k * B + j) % (2 * B))
    tr.region_begin()
    tr.train(buf, job, [], epochs=1)
    b = tr.region_end() / K
    tr.set_timing(True)
    ms = [tr.step(buf, batch(k))["ms"] for k in range(K)]
    tr.set_timing(False)
    time.sleep(float(os.environ.get("SLEEP", "0")))
    print(f"rep {rep}: step() loop {a:.3f} ms/step | train(job) {b:.3f} | timed steps "
          f"{np.mean(ms):.3f} (first {ms[0]:.3f} last {ms[-1]:.3f})", flush=True)
