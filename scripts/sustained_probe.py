"""Sustained (4 s back to back) bf16 GEMM throughput at 8192^3: this repo's
tcgen05 kernel through the debug hook vs torch.matmul (cuBLAS), same box,
same process -- separates kernel efficiency from the step's power budget."""
import ctypes as C
import json
import sys
import pathlib
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib  # noqa: E402

n = 8192
flops = 2.0 * n ** 3
res = {}
a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
for _ in range(20):
    torch.matmul(a, b)
torch.cuda.synchronize()
for tag, iters in (("burst", 10), ("sustained", 5600)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    res[f"cublas_{tag}_tflops"] = round(flops * iters / (e0.elapsed_time(e1) * 1e-3) / 1e12, 1)
A = (np.random.default_rng(0).integers(0, 1 << 16, (n, n), dtype=np.uint32) & 0x3FFF | 0x3C00).astype(np.uint16)
Cb = np.zeros((n, n), np.float32)
for tag, iters in (("burst", 10), ("sustained", 5600)):
    ms = C.c_float(0)
    _lib.call("specsim_debug_gemm", 0, 0, 1 | (2 << 8), n, n, n, _lib.ptr(A), n, _lib.ptr(A), n,
              _lib.ptr(Cb), n, None, 0, iters, C.byref(ms))
    res[f"ours_{tag}_tflops"] = round(flops / (ms.value * 1e-3) / 1e12, 1)
print(json.dumps(res))
