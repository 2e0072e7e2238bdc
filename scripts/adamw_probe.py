"""Fused-AdamW weight-gradient GEMM probe: the same C2 dW shapes through the
debug GEMM hook with a plain fp32 epilogue (epi 1) and with the AdamW epilogue
(epi 6), for whichever build SPECSIM_LIB points at (scripts/adamw_probe.sh
builds the SPECSIM_ADAMW_VARIANT probe libraries)."""
import ctypes as C
import json
import os
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib  # noqa: E402

T = 8192
SHAPES = [("lm_chunk_dW", 1, 1, 32768, 4096, T), ("gate_up_dW", 1, 1, 28672, 4096, T),
          ("lm_chunk_dX", 0, 1, T, 4096, 32768)]
rng = np.random.default_rng(0)
tag = os.environ.get("TAG", "base")
for name, a_mn, b_mn, M, N, K in SHAPES:
    A = (rng.integers(0, 1 << 16, ((K if a_mn else M), (M if a_mn else K)), dtype=np.uint32) & 0x3FFF | 0x3C00).astype(np.uint16)
    B = (rng.integers(0, 1 << 16, ((K if b_mn else N), (N if b_mn else K)), dtype=np.uint32) & 0x3FFF | 0x3C00).astype(np.uint16)
    for epi in ((1, 6) if a_mn else (1,)):
        Cb = np.full((M, N), 0.01, np.float32)
        ms = C.c_float(0)
        _lib.call("specsim_debug_gemm", a_mn, b_mn, epi | (2 << 8), M, N, K, _lib.ptr(A), A.shape[1],
                  _lib.ptr(B), B.shape[1], _lib.ptr(Cb), N, None, 0, int(os.environ.get("ITERS", 20)),
                  C.byref(ms))
        print(json.dumps(dict(tag=tag, name=name, epi=epi, ms=round(ms.value, 4),
                              tflops=round(2.0 * M * N * K / (ms.value * 1e-3) / 1e12, 1))), flush=True)
