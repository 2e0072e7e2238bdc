"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/liboracle.so (plain C restatement, see oracle.h) and
of oracle/_ref/libspecsim_ref.so (the reference's own perf_model / Rng /
workload code compiled in place by build_ref.sh).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this package, and only as the checker or the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libspecsim_ref.so"


class RngState(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class Shape(C.Structure):
    _fields_ = [("H", C.c_int), ("V", C.c_int), ("S", C.c_int), ("nh", C.c_int),
                ("nkv", C.c_int), ("hd", C.c_int), ("I", C.c_int), ("layers", C.c_int),
                ("B", C.c_int), ("eps", C.c_float), ("theta", C.c_double), ("ttt", C.c_int),
                ("ttt_decay", C.c_float)]


class StepOut(C.Structure):
    _fields_ = [("loss", C.c_double), ("valid", C.c_int64), ("top1", C.c_int64)]


_lib = None
_ref = None
P = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} not built (make -C oracle)")
        L = C.CDLL(str(LIB))
        L.orc_rng_seed.argtypes = [C.POINTER(RngState), C.c_uint64]
        L.orc_rng_next.argtypes = [C.POINTER(RngState)]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_uniform.argtypes = [C.POINTER(RngState)]
        L.orc_uniform.restype = C.c_double
        L.orc_normal.argtypes = [C.POINTER(RngState), C.c_double, C.c_double]
        L.orc_normal.restype = C.c_double
        L.orc_geometric.argtypes = [C.POINTER(RngState), C.c_double]
        L.orc_geometric.restype = C.c_int64
        L.orc_expected_accept_length.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.orc_sample_accept_length.argtypes = [C.POINTER(RngState), C.c_double, C.c_int,
                                               C.POINTER(C.c_int)]
        L.orc_alpha_from_accept_length.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.orc_split_train_eval.argtypes = [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_bytes_per_token.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_bytes_per_token.restype = C.c_int64
        L.orc_extract_signals.argtypes = [P, C.c_int64, C.c_int64, C.c_int64]
        L.orc_f32_to_bf16.argtypes = [C.c_float]
        L.orc_f32_to_bf16.restype = C.c_uint16
        L.orc_synth_capture.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_int, P, P, P, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_double)]
        L.orc_init_normal_block.argtypes = [C.c_uint64, C.c_int, C.c_int64, P]
        L.orc_param_layout.argtypes = [C.POINTER(Shape), P, P, P, P]
        L.orc_param_layout.restype = C.c_int64
        L.orc_gather_batch.argtypes = [C.POINTER(Shape), C.c_int, P, P, P, P, P, P, P]
        L.orc_train_step.argtypes = [C.POINTER(Shape), P, C.c_int64, P, P, P, P, P, P, P, P, P,
                                     C.c_int64, C.c_int, C.c_int, C.POINTER(StepOut)]
        L.orc_forward.argtypes = [C.POINTER(Shape), P, P, P, P, P, P, C.c_int64, C.c_int,
                                  C.POINTER(StepOut), P, P]
        L.orc_forward_ex.argtypes = [C.POINTER(Shape), P, P, P, P, P, P, C.c_int64, C.c_int,
                                     C.POINTER(StepOut), P, P, P, P, P]
        L.orc_adamw.argtypes = [C.c_int64, P, P, P, P, P, C.c_int64]
        L.orc_num_threads.restype = C.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_LIB.exists()


def ref():
    """The compiled reference (bookkeeping only)."""
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} not built (oracle/build_ref.sh needs /root/reference)")
        R = C.CDLL(str(REF_LIB))
        R.ref_rng_create.argtypes = [C.c_uint64]
        R.ref_rng_create.restype = P
        R.ref_rng_destroy.argtypes = [P]
        R.ref_rng_uniform.argtypes = [P]
        R.ref_rng_uniform.restype = C.c_double
        R.ref_rng_normal.argtypes = [P, C.c_double, C.c_double]
        R.ref_rng_normal.restype = C.c_double
        R.ref_rng_geometric.argtypes = [P, C.c_double]
        R.ref_rng_geometric.restype = C.c_longlong
        R.ref_expected_accept_length.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double)]
        R.ref_sample_accept_length.argtypes = [P, C.c_double, C.c_int, C.POINTER(C.c_int)]
        R.ref_alpha_from_accept_length.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double)]
        R.ref_current_alpha.argtypes = [C.c_double] * 4
        R.ref_current_alpha.restype = C.c_double
        R.ref_workload_tokens.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64,
                                          C.POINTER(C.c_longlong)]
        R.ref_workload_tokens.restype = C.c_longlong
        _ref = R
    return _ref


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


# ------------------------------------------------------------------ helpers
class Rng:
    """Oracle restatement of specsim::Rng (rng.hpp:13-39)."""

    def __init__(self, seed: int):
        self.st = RngState()
        lib().orc_rng_seed(C.byref(self.st), seed)

    def next_u64(self):
        return lib().orc_rng_next(C.byref(self.st))

    def uniform(self):
        return lib().orc_uniform(C.byref(self.st))

    def normal(self, mean, sd):
        return lib().orc_normal(C.byref(self.st), mean, sd)

    def geometric(self, mean):
        return lib().orc_geometric(C.byref(self.st), mean)

    def sample_accept_length(self, alpha, gamma):
        k = C.c_int()
        if lib().orc_sample_accept_length(C.byref(self.st), alpha, gamma, C.byref(k)):
            raise ValueError("domain error")
        return k.value


def expected_accept_length(alpha, gamma):
    o = C.c_double()
    if lib().orc_expected_accept_length(alpha, gamma, C.byref(o)):
        raise ValueError("domain error")
    return o.value


def alpha_from_accept_length(ell, gamma):
    o = C.c_double()
    if lib().orc_alpha_from_accept_length(ell, gamma, C.byref(o)):
        raise ValueError("domain error")
    return o.value


def split_train_eval(n):
    a, b = C.c_int64(), C.c_int64()
    lib().orc_split_train_eval(n, C.byref(a), C.byref(b))
    return a.value, b.value


def synth_capture(seed, index, length, vocab, hidden, layers=3, alpha=0.6, gamma=3,
                  features=True):
    ids = np.zeros(length, np.int32)
    feats = np.zeros((length, layers * hidden), np.uint16) if features else None
    acc = np.zeros(length, np.int32)
    n = C.c_int32()
    a_s = C.c_double()
    rc = lib().orc_synth_capture(seed, index, length, vocab, hidden, layers, alpha, gamma,
                                 _p(ids), _p(feats), _p(acc), C.byref(n), C.byref(a_s))
    if rc:
        raise ValueError("domain error")
    return dict(ids=ids, features=feats, accept_lengths=acc[: n.value].copy(),
                alpha_s=a_s.value)


def make_shape(H, V, S, nh, nkv, hd, I, B, layers=3, eps=1e-5, theta=10000.0, ttt=1,
               ttt_decay=0.8):
    return Shape(H, V, S, nh, nkv, hd, I, layers, B, eps, theta, ttt, ttt_decay)


def ttt_of(shape):
    return max(1, shape.ttt)


def param_layout(shape):
    names = (C.c_char_p * 10)()
    rows = np.zeros(10, np.int64)
    cols = np.zeros(10, np.int64)
    offs = np.zeros(10, np.int64)
    total = lib().orc_param_layout(C.byref(shape), C.cast(names, C.c_void_p), _p(rows), _p(cols),
                                   _p(offs))
    return [(names[i].decode(), int(rows[i]), int(cols[i]), int(offs[i])) for i in range(10)], total


NORM_PARAMS = ("w_in", "w_hid", "w_post", "w_fin")


def init_params(shape, seed):
    """Flat fp32 master vector, same init as the library (bit-exact)."""
    layout, total = param_layout(shape)
    P_ = np.zeros(total, np.float32)
    for p, (name, r, c, off) in enumerate(layout):
        if name in NORM_PARAMS:
            P_[off:off + r * c] = 1.0
        else:
            blk = np.zeros(r * c, np.float32)
            lib().orc_init_normal_block(seed + 1, p, r * c, _p(blk))
            P_[off:off + r * c] = blk
    return P_


def init_embedding(shape, seed):
    e = np.zeros(shape.V * shape.H, np.float32)
    lib().orc_init_normal_block(seed + 2, 15, e.size, _p(e))
    return f32_to_bf16(e).reshape(shape.V, shape.H)


def f32_to_bf16(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def bf16_to_f32(b):
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def gather_batch(shape, samples):
    """samples: list of (ids int32[L], feats uint16[L, 3H]); len <= B.
    u / y / m hold ttt slices of B*S rows (slice j shifted by j tokens)."""
    T = shape.B * shape.S * ttt_of(shape)
    W = shape.layers * shape.H
    F = np.zeros((shape.B * shape.S, W), np.uint16)
    u = np.zeros(T, np.int32)
    y = np.zeros(T, np.int32)
    m = np.zeros(T, np.int32)
    keep = [(np.ascontiguousarray(i, np.int32), np.ascontiguousarray(f, np.uint16))
            for i, f in samples]
    ids_arr = (C.c_void_p * max(1, len(keep)))(*[i.ctypes.data for i, _ in keep])
    f_arr = (C.c_void_p * max(1, len(keep)))(*[f.ctypes.data for _, f in keep])
    lens = np.array([len(i) for i, _ in keep] or [0], np.int32)
    lib().orc_gather_batch(C.byref(shape), len(keep), C.cast(ids_arr, C.c_void_p),
                           C.cast(f_arr, C.c_void_p), _p(lens), _p(F), _p(u), _p(y), _p(m))
    return F, u, y, m


def train_step(shape, adamw, step_k, params, mst, vst, E, F, u, y, m, global_valid=0,
               round_bf16=True, update=True):
    """In-place on params/mst/vst; returns (StepOut, grads)."""
    grads = np.zeros_like(params)
    out = StepOut()
    hp = np.asarray(adamw, np.float32)
    rc = lib().orc_train_step(C.byref(shape), _p(hp), step_k, _p(params), _p(mst), _p(vst),
                              _p(grads), _p(E), _p(F), _p(u), _p(y), _p(m), global_valid,
                              1 if round_bf16 else 0, 1 if update else 0, C.byref(out))
    if rc:
        raise ValueError("bad shape")
    return out, grads


def forward(shape, params, E, F, u, y, m, global_valid=0, round_bf16=True, margin=False,
            probe=None):
    """(StepOut, lse, argmax[, margin][, probe_gap]) over the K*B*S rows;
    margin = top-1 minus top-2 logit per row (0 on ties); probe_gap[r] = the
    oracle's max logit minus its logit at vocabulary index probe[r]."""
    out = StepOut()
    T = shape.B * shape.S * ttt_of(shape)
    lse = np.zeros(T, np.float32)
    am = np.zeros(T, np.int32)
    mg = np.zeros(T, np.float32) if margin else None
    pr = None if probe is None else np.ascontiguousarray(probe[:T], np.int32)
    pl = None if probe is None else np.zeros(T, np.float32)
    if lib().orc_forward_ex(C.byref(shape), _p(params), _p(E), _p(F), _p(u), _p(y), _p(m),
                            global_valid, 1 if round_bf16 else 0, C.byref(out), _p(lse), _p(am),
                            _p(mg), _p(pr), _p(pl)):
        raise ValueError("bad shape")
    res = (out, lse, am) + ((mg,) if margin else ()) + ((pl,) if probe is not None else ())
    return res


def adamw(p, m, v, g, hp, step_k):
    hp = np.asarray(hp, np.float32)
    lib().orc_adamw(p.size, _p(p), _p(m), _p(v), _p(g), _p(hp), step_k)


def num_threads():
    return lib().orc_num_threads()
