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
for name, a_mn, b_mn, M, N, K in SHAPES:
    A = np.zeros(((K if a_mn else M), (M if a_mn else K)), np.uint16)
    A[:] = 0x3F80  # 1.0
    B = np.zeros(((K if b_mn else N), (N if b_mn else K)), np.uint16)
    B[:] = 0x3C00
    Cb = np.zeros((M, N), np.float32)
    ms = C.c_float(0)
    _lib.call("specsim_debug_gemm", a_mn, b_mn, 1, M, N, K, _lib.ptr(A), A.shape[1], _lib.ptr(B),
              B.shape[1], _lib.ptr(Cb), N, None, 0, 10, C.byref(ms))
    tf = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
    expect = 1.0 * (1.0 / 128) * K
    ok = bool(abs(Cb[0, 0] - expect) < 1e-3 * expect and abs(Cb[-1, -1] - expect) < 1e-3 * expect)
    rec = dict(name=name, M=M, N=N, K=K, ms=round(ms.value, 4), tflops=round(tf, 1), check=ok)
    print(json.dumps(rec), flush=True)
    out.append(rec)
pathlib.Path("gpurun_out").mkdir(exist_ok=True)
pathlib.Path("gpurun_out/gemm_probe.json").write_text(json.dumps(out, indent=1))
