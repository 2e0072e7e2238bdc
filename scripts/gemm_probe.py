"""Throughput probe of the tcgen05 GEMM at the C2 (Llama-3.1-8B-shape) step shapes."""
import ctypes as C
import json
import sys
import pathlib

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib  # noqa: E402

T = 8192
SHAPES = [  # name, a_mn, b_mn, M, N, K
    ("fc_fwd", 0, 0, T, 4096, 12288),
    ("qkv_fwd", 0, 0, T, 6144, 8192),
    ("gate_up_fwd", 0, 0, T, 28672, 4096),
    ("down_fwd", 0, 0, T, 4096, 14336),
    ("lm_chunk_fwd", 0, 0, T, 32768, 4096),
    ("down_dX", 0, 1, T, 14336, 4096),
    ("lm_chunk_dX", 0, 1, T, 4096, 32768),
    ("gate_up_dW", 1, 1, 28672, 4096, T),
    ("lm_chunk_dW", 1, 1, 32768, 4096, T),
    ("sq8192", 0, 0, 8192, 8192, 8192),
]
out = []
rng = np.random.default_rng(0)
for (name, a_mn, b_mn, M, N, K), cg in [(s, c) for s in SHAPES for c in (1, 2)]:
    # random bf16 operands (power draw of real data); checked on a few entries
    A = (rng.integers(0, 1 << 16, ((K if a_mn else M), (M if a_mn else K)), dtype=np.uint32) & 0x3FFF | 0x3C00).astype(np.uint16)
    B = (rng.integers(0, 1 << 16, ((K if b_mn else N), (N if b_mn else K)), dtype=np.uint32) & 0x3FFF | 0x3C00).astype(np.uint16)
    Cb = np.zeros((M, N), np.float32)
    ms = C.c_float(0)
    _lib.call("specsim_debug_gemm", a_mn, b_mn, 1 | (cg << 8), M, N, K, _lib.ptr(A), A.shape[1], _lib.ptr(B),
              B.shape[1], _lib.ptr(Cb), N, None, 0, 10, C.byref(ms))
    tf = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
    def f32(b):
        return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    ok = True
    for (i, j) in [(0, 0), (M - 1, N - 1), (M // 3, N // 2)]:
        a = f32(A[:, i] if a_mn else A[i, :])
        b = f32(B[:, j] if b_mn else B[j, :])
        ref = float(a @ b)
        ok &= abs(Cb[i, j] - ref) <= 1e-3 * abs(ref) + 1e-2
    rec = dict(name=name, cg=cg, M=M, N=N, K=K, ms=round(ms.value, 4), tflops=round(tf, 1), check=bool(ok))
    print(json.dumps(rec), flush=True)
    out.append(rec)
pathlib.Path("gpurun_out").mkdir(exist_ok=True)
pathlib.Path("gpurun_out/gemm_probe.json").write_text(json.dumps(out, indent=1))
