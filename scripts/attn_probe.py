"""Attention kernels at C2 head geometry with different sequence lengths (same
positions per call): separates the per-CTA fixed cost (S = 128: one key block
per CTA) from the per-block cost.  Run under ncu for kernel times."""
import sys
import pathlib

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2602_05145_b200 import _lib  # noqa: E402

nh, nkv, hd = 32, 8, 128
for B, S in [(64, 128), (16, 512), (4, 2048)]:
    T = B * S
    NQ = (nh + 2 * nkv) * hd
    rng = np.random.default_rng(0)
    qkv = (rng.standard_normal((T, NQ), np.float32) * 0.5).astype(np.float32)
    qkv16 = (qkv.view(np.uint32) >> 16).astype(np.uint16)
    dout = (rng.standard_normal((T, nh * hd), np.float32).view(np.uint32) >> 16).astype(np.uint16)
    o = np.zeros((T, nh * hd), np.uint16)
    lse = np.zeros((nh, T), np.float32)
    dq = np.zeros((T, NQ), np.uint16)
    _lib.call("specsim_debug_attention", B, S, nh, nkv, hd, _lib.ptr(qkv16), _lib.ptr(dout),
              _lib.ptr(o), _lib.ptr(lse), _lib.ptr(dq))
    print(B, S, "done", flush=True)
