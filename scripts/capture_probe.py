"""Capture-side overhead probe (PAPER.md:130 claims the
D2H of accepted-token states overlaps the next verification step).

A stand-in verification step (bf16 GEMMs of a C2-sized batch on one stream)
runs N iterations with and without SignalCapture appending every request's
accepted rows of three tapped layers (hidden 4096).  Prints one JSON line:
iteration ms with / without capture, captured GB/s, shards written."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_05145_b200 import api  # noqa: E402

H, BATCH, GAMMA, ITERS = 4096, int(os.environ.get("BATCH", "64")), 3, 200
WT = int(os.environ.get("WIDTH", "8192"))      # target model width (taps are its first H columns)
NL = int(os.environ.get("LAYERS", "32"))       # target layers per verification step
dev = torch.device("cuda")
s = torch.cuda.Stream()
x = torch.randn(BATCH * (GAMMA + 1), WT, device=dev, dtype=torch.bfloat16) * 0.01
w = [torch.randn(WT, WT, device=dev, dtype=torch.bfloat16) * 0.01 for _ in range(NL)]
TAPS = (1, NL // 2, NL - 2)
rng = np.random.default_rng(0)
acc = [rng.integers(1, GAMMA + 2, BATCH) for _ in range(ITERS)]


def verify(layers):
    h = x
    for i, wi in enumerate(w):  # the target's layers; low / mid / high taps
        h = torch.relu(h @ wi)
        if i in TAPS:
            layers.append(h)
    return h


def run(capture):
    cap = api.SignalCapture(api.SignalGeometry(H), tmp, 0) if capture else None
    rows = GAMMA + 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        e0.record(s)
        for it in range(ITERS):
            layers = []
            verify(layers)
            if cap:
                k = acc[it]
                rows_acc = np.concatenate([r * rows + np.arange(k[r]) for r in range(BATCH)])
                sids = np.arange(BATCH) + 1000 * (it // 50)  # requests live 50 iterations
                cap.append_batch(sids, k, rows_acc, [l.data_ptr() for l in layers],
                                 BATCH * rows, WT, np.zeros(len(rows_acc), np.int32),
                                 stream=s.cuda_stream)
                if it % 50 == 49:
                    for sid in sids:
                        cap.end_sample(int(sid), 0.5)
        e1.record(s)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st = cap.stats() if cap else None
    files = cap.close() if cap else []
    return e0.elapsed_time(e1) / ITERS, wall, st, files


root = "/dev/shm" if os.path.isdir("/dev/shm") else None
with tempfile.TemporaryDirectory(dir=root) as tmp:
    run(False)
    base, wall0, _, _ = run(False)
    with_cap, wall1, st, files = run(True)
    toks = int(sum(a.sum() for a in acc))
    print(json.dumps(dict(
        probe="capture overhead", batch=BATCH, iters=ITERS, tokens=toks, target_width=WT,
        target_layers=NL, storage=root or "tmp",
        bytes=toks * 3 * H * 2, ms_per_iter_no_capture=round(base, 4),
        ms_per_iter_capture=round(with_cap, 4), overhead_pct=round(100 * (with_cap / base - 1), 2),
        host_wall_s_no_capture=round(wall0, 3), host_wall_s_capture=round(wall1, 3),
        capture_gbps_of_wall=round(toks * 3 * H * 2 / wall1 / 1e9, 2),
        shards=len(files), spec_flushes=st["flushes"])))
