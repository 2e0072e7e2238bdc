"""Python mirror of the reference-facing interface (thin ctypes wrappers).

Names follow the reference's domain: SignalGeometry,
extract_signals / record_sample, train(job) ->
TrainingOutcome, the perf_model bookkeeping
(perf_model.hpp:52-80) and the seeded Rng (rng.hpp:13-39).  Every call goes
through the C ABI of libspecsim_draft.so; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import call, ptr

# ------------------------------------------------------------- configs
CONFIGS = {
    # BASELINE.json configs; head / FFN dims from SURVEY §8 (public HF configs)
    "C1": dict(hidden=256, vocab=4096, seq_len=128, n_heads=4, n_kv_heads=2, head_dim=64,
               ffn=1024, micro_batch=8, rms_eps=1e-5, rope_theta=10000.0),
    "C2": dict(hidden=4096, vocab=128256, seq_len=2048, n_heads=32, n_kv_heads=8, head_dim=128,
               ffn=14336, micro_batch=4, rms_eps=1e-5, rope_theta=500000.0),
    "C4": dict(hidden=5120, vocab=151936, seq_len=2048, n_heads=64, n_kv_heads=8, head_dim=128,
               ffn=25600, micro_batch=4, rms_eps=1e-6, rope_theta=1000000.0),
    "C5": dict(hidden=8192, vocab=128256, seq_len=4096, n_heads=64, n_kv_heads=8, head_dim=128,
               ffn=28672, micro_batch=2, rms_eps=1e-5, rope_theta=500000.0),
}


def gemm_flops_per_token(c: dict) -> dict:
    """Algorithmic FLOPs per processed token (SURVEY §8(d) convention).  With a
    training-time-test unroll of K passes the decoder layer and the LM head
    run K times (fc once) and pass j's attention adds 4Q FLOPs per cache
    entry (j of them) to the forward."""
    H, V, S = c["hidden"], c["vocab"], c["seq_len"]
    Q = c["n_heads"] * c["head_dim"]
    KV = c["n_kv_heads"] * c["head_dim"]
    I = c["ffn"]
    L = c.get("layers_tapped", 3)
    K = c.get("ttt_steps", 1)
    fc = 2 * L * H * H
    per_pass = 2 * (2 * H * (Q + 2 * KV) + Q * H + 3 * H * I + H * V)
    gemm_fwd = fc + K * per_pass
    attn_fwd = K * 2 * Q * (S + 1) + sum(4 * Q * j for j in range(K))
    fwd = gemm_fwd + attn_fwd
    bwd = 2 * gemm_fwd - fc + 2 * attn_fwd
    lm = K * 2 * H * V
    return dict(total=fwd + bwd, gemm=3 * gemm_fwd - fc, attn=3 * attn_fwd,
                lm=3 * lm, decoder_gemm=3 * gemm_fwd - fc - 3 * lm)


# ------------------------------------------------------------ bookkeeping
class Rng:
    """The library's seeded Rng (bit-compatible with the reference)."""

    def __init__(self, seed: int):
        self.h = C.c_void_p()
        call("specsim_rng_create", seed, C.byref(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.specsim_rng_destroy(self.h)
        self.h = None

    def uniform(self) -> float:
        o = C.c_double()
        call("specsim_rng_uniform", self.h, C.byref(o))
        return o.value

    def normal(self, mean: float, sd: float) -> float:
        o = C.c_double()
        call("specsim_rng_normal", self.h, mean, sd, C.byref(o))
        return o.value

    def geometric(self, mean: float) -> int:
        o = C.c_int64()
        call("specsim_rng_geometric", self.h, mean, C.byref(o))
        return o.value

    def next_u64(self) -> int:
        o = C.c_uint64()
        call("specsim_rng_next_u64", self.h, C.byref(o))
        return o.value

    def sample_accept_length(self, alpha: float, gamma: int) -> int:
        o = C.c_int32()
        call("specsim_sample_accept_length", self.h, alpha, gamma, C.byref(o))
        return o.value


def expected_accept_length(alpha: float, gamma: int) -> float:
    o = C.c_double()
    call("specsim_expected_accept_length", alpha, gamma, C.byref(o))
    return o.value


def alpha_from_accept_length(ell: float, gamma: int) -> float:
    o = C.c_double()
    call("specsim_alpha_from_accept_length", ell, gamma, C.byref(o))
    return o.value


def split_train_eval(n: int):
    a, b = C.c_int64(), C.c_int64()
    call("specsim_split_train_eval", n, C.byref(a), C.byref(b))
    return a.value, b.value


def current_alpha(alpha_start, alpha_ceiling, tau_samples, trained_samples):
    """workload.cpp:41-47 (the reference's analytic alpha law)."""
    o = C.c_double()
    call("specsim_current_alpha", alpha_start, alpha_ceiling, tau_samples, trained_samples,
         C.byref(o))
    return o.value


def dp_shard(n_items: int, per_rank: int, world: int, rank: int, step: int):
    idx = np.zeros(max(1, per_rank), np.int64)
    n = C.c_int32()
    call("specsim_dp_shard", n_items, per_rank, world, rank, step, ptr(idx), C.byref(n))
    return idx[: n.value].tolist()


def draft_shape(shape: dict):
    """ctypes specsim_draft_shape from a config dict (api.CONFIGS entry)."""
    return _lib.DraftShape(shape["hidden"], shape["vocab"], shape["seq_len"], shape["n_heads"],
                           shape["n_kv_heads"], shape["head_dim"], shape["ffn"],
                           shape.get("layers_tapped", 3), shape.get("micro_batch", 1),
                           shape.get("rms_eps", 1e-5), shape.get("rope_theta", 10000.0),
                           shape.get("ttt_steps", 1), shape.get("ttt_decay", 0.8))


def dp_buckets(shape: dict, world: int):
    """(buckets [(off, n)], zero_ok) of the data-parallel gradient exchange."""
    s = draft_shape(shape)
    cnt, ok = C.c_int32(), C.c_int32()
    call("specsim_dp_buckets", C.byref(s), world, None, None, 0, C.byref(cnt), C.byref(ok))
    off = np.zeros(cnt.value, np.int64)
    n = np.zeros(cnt.value, np.int64)
    call("specsim_dp_buckets", C.byref(s), world, ptr(off), ptr(n), cnt.value, C.byref(cnt),
         C.byref(ok))
    return list(zip(off.tolist(), n.tolist())), bool(ok.value)


def zero_shard(bucket, world: int, rank: int):
    """Range [lo, hi) of a bucket owned by `rank` under ZeRO-1."""
    off, n = bucket
    c = n // world
    return off + rank * c, off + (rank + 1) * c


def global_job(steps: int, per_rank: int, world: int, id_of):
    """Global train(job) list for data parallelism: slot j of step k belongs to
    rank j % world (the specsim_dp_shard rule) and holds id_of(rank, k, j // world),
    i.e. that rank's (j // world)-th sample of step k.  Every rank passes the
    same list; each trains only its own ids."""
    return [id_of(j % world, k, j // world) for k in range(steps) for j in range(per_rank * world)]


@dataclass
class SignalGeometry:
    hidden_dim: int
    layers_tapped: int = 3
    bytes_per_element: int = 2

    def c(self):
        return _lib.SignalGeometry(self.hidden_dim, self.layers_tapped, self.bytes_per_element)

    def bytes_per_token(self) -> int:
        o = C.c_int64()
        g = self.c()
        call("specsim_bytes_per_token", C.byref(g), C.byref(o))
        return o.value


def synth_capture(seed, index, length, vocab, hidden, layers=3, alpha=0.6, gamma=3,
                  features=True):
    ids = np.zeros(length, np.int32)
    feats = np.zeros((length, layers * hidden), np.uint16) if features else None
    acc = np.zeros(length, np.int32)
    n = C.c_int32()
    a_s = C.c_double()
    call("specsim_synth_capture", seed, index, length, vocab, hidden, layers, alpha, gamma,
         ptr(ids), ptr(feats), ptr(acc), C.byref(n), C.byref(a_s))
    return dict(ids=ids, features=feats, accept_lengths=acc[: n.value].copy(), alpha_s=a_s.value)


# --------------------------------------------------------- signal buffer
class HiddenStateBuffer:
    def __init__(self, geometry: SignalGeometry, capacity_tokens: int, flush_threshold: int = 0,
                 device: int = 0):
        self.geometry = geometry
        self.h = C.c_void_p()
        g = geometry.c()
        call("specsim_hsbuf_create", C.byref(g), capacity_tokens, flush_threshold, device,
             C.byref(self.h))

    def close(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.specsim_hsbuf_destroy(self.h)
        self.h = None

    __del__ = close

    def extract_signals(self, sample_id, alpha, layers, token_ids, accepted_idx=None,
                        on_device=False):
        """One verify step: layers = list of [rows, H] uint16 (bf16) arrays."""
        layers = [np.ascontiguousarray(l) for l in layers]
        rows, ld = layers[0].shape
        arr = (C.c_void_p * len(layers))(*[l.ctypes.data for l in layers])
        ids = np.ascontiguousarray(token_ids, np.int32)
        idx = None if accepted_idx is None else np.ascontiguousarray(accepted_idx, np.int32)
        n = len(ids)
        call("specsim_hsbuf_append", self.h, sample_id, alpha, C.cast(arr, C.POINTER(C.c_void_p)),
             rows, ld, ptr(ids), ptr(idx), n, 1 if on_device else 0)

    def append_packed(self, sample_id, alpha, features, token_ids):
        f = np.ascontiguousarray(features, np.uint16)
        ids = np.ascontiguousarray(token_ids, np.int32)
        call("specsim_hsbuf_append_packed", self.h, sample_id, alpha, ptr(f), ptr(ids), len(ids), 0)

    def load_shards(self, paths) -> int:
        """Append the samples of TIDESIG1 shard files (SignalCapture output)."""
        arr = (C.c_char_p * max(1, len(paths)))(*[str(p).encode() for p in paths])
        n = C.c_int64()
        call("specsim_hsbuf_load_shards", self.h, arr, len(paths), C.byref(n))
        return n.value

    def stats(self) -> dict:
        s = _lib.HsbufStats()
        call("specsim_hsbuf_stats_get", self.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def sample_info(self, sample_id):
        n = C.c_int32()
        a = C.c_double()
        call("specsim_hsbuf_sample_info", self.h, sample_id, C.byref(n), C.byref(a))
        return n.value, a.value

    def read_sample(self, sample_id):
        n, _ = self.sample_info(sample_id)
        W = self.geometry.hidden_dim * self.geometry.layers_tapped
        f = np.zeros((n, W), np.uint16)
        ids = np.zeros(n, np.int32)
        call("specsim_hsbuf_read_sample", self.h, sample_id, ptr(f), ptr(ids))
        return f, ids


class SignalCapture:
    """Serving-side capture: pack on the serving stream,
    D2H into pinned segments on a side stream, TIDESIG1 shards at the flush
    threshold.  Layer arguments are device pointers (ints) valid on `stream`
    (a cudaStream_t as int; 0 = legacy default stream)."""

    def __init__(self, geometry: SignalGeometry, directory, flush_threshold: int = 0,
                 device: int = 0):
        self.geometry = geometry
        self.h = C.c_void_p()
        g = geometry.c()
        call("specsim_capture_create", C.byref(g), str(directory).encode(), flush_threshold,
             device, C.byref(self.h))

    def append(self, sample_id, layer_ptrs, rows, ld, token_ids, accepted_idx=None, stream=0):
        arr = (C.c_void_p * len(layer_ptrs))(*layer_ptrs)
        ids = np.ascontiguousarray(token_ids, np.int32)
        idx = None if accepted_idx is None else np.ascontiguousarray(accepted_idx, np.int32)
        call("specsim_capture_append", self.h, sample_id, C.cast(arr, C.POINTER(C.c_void_p)),
             rows, ld, ptr(ids), ptr(idx), len(ids), stream)

    def append_batch(self, sample_ids, counts, accepted_rows, layer_ptrs, rows, ld, token_ids,
                     stream=0):
        """One serving iteration: request r's accepted rows are the next counts[r]
        entries of accepted_rows (rows of the [rows, ld] layer matrices)."""
        sid = np.ascontiguousarray(sample_ids, np.int64)
        off = np.zeros(len(sid) + 1, np.int32)
        off[1:] = np.cumsum(np.asarray(counts, np.int64))
        acc = np.ascontiguousarray(accepted_rows, np.int32)
        ids = np.ascontiguousarray(token_ids, np.int32)
        arr = (C.c_void_p * len(layer_ptrs))(*layer_ptrs)
        call("specsim_capture_append_batch", self.h, ptr(sid), len(sid), ptr(off), ptr(acc),
             C.cast(arr, C.POINTER(C.c_void_p)), rows, ld, ptr(ids), stream)

    def end_sample(self, sample_id, alpha):
        call("specsim_capture_end_sample", self.h, sample_id, alpha)

    def flush(self):
        call("specsim_capture_flush", self.h)

    def stats(self) -> dict:
        s = _lib.CaptureStats()
        call("specsim_capture_stats_get", self.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def files(self):
        out = []
        b = C.create_string_buffer(4096)
        for i in range(self.stats()["files"]):
            call("specsim_capture_file", self.h, i, b, 4096)
            out.append(b.value.decode())
        return out

    def close(self):
        """Flush, join the writer; returns the shard paths."""
        if getattr(self, "h", None) is None:
            return []
        call("specsim_capture_close", self.h)
        files = self.files()
        if _lib is not None and _lib._lib is not None:
            _lib._lib.specsim_capture_destroy(self.h)
        self.h = None
        return files

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.specsim_capture_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------- trainer
@dataclass
class TrainingOutcome:
    duration_hours: float
    alpha_eval: float
    new_version: int
    mean_loss: float
    steps: int


class DraftTrainer:
    PHASES = ("ingest", "gemm", "attention", "elementwise", "lm_head_ce", "adamw", "allreduce")

    def __init__(self, shape: dict, lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0,
                 seed=20260217, rank=0, world=1, nccl_id: bytes | None = None, device=0):
        self.shape = dict(shape)
        s = draft_shape(shape)
        a = _lib.AdamW(lr, betas[0], betas[1], eps, weight_decay)
        self.h = C.c_void_p()
        nid = None
        if nccl_id is not None:
            nid = C.create_string_buffer(bytes(nccl_id), 128)
        call("specsim_trainer_create", C.byref(s), C.byref(a), seed, rank, world,
             C.cast(nid, C.c_void_p) if nid is not None else None, device, C.byref(self.h))

    def close(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.specsim_trainer_destroy(self.h)
        self.h = None

    __del__ = close

    @staticmethod
    def nccl_unique_id() -> bytes:
        b = C.create_string_buffer(128)
        call("specsim_nccl_unique_id", C.cast(b, C.c_void_p))
        return b.raw

    @staticmethod
    def _res(r):
        return dict(loss=r.loss, valid_tokens=r.valid_tokens, top1_correct=r.top1_correct,
                    positions=r.positions, ms=r.ms)

    def step(self, buf: HiddenStateBuffer, sample_ids, global_valid=0):
        ids = np.ascontiguousarray(sample_ids, np.int64)
        r = _lib.StepResult()
        call("specsim_trainer_step", self.h, buf.h, ids.ctypes.data_as(_lib.PI64), len(ids),
             global_valid, C.byref(r))
        return self._res(r)

    def eval(self, buf: HiddenStateBuffer, sample_ids):
        ids = np.ascontiguousarray(sample_ids, np.int64)
        r = _lib.StepResult()
        call("specsim_trainer_eval", self.h, buf.h, ids.ctypes.data_as(_lib.PI64), len(ids),
             C.byref(r))
        return self._res(r)

    def train(self, buf, train_ids, eval_ids, epochs=1) -> TrainingOutcome:
        t = np.ascontiguousarray(train_ids, np.int64)
        e = np.ascontiguousarray(eval_ids, np.int64)
        o = _lib.TrainingOutcome()
        call("specsim_trainer_train", self.h, buf.h, t.ctypes.data_as(_lib.PI64), len(t),
             e.ctypes.data_as(_lib.PI64), len(e), epochs, C.byref(o))
        return TrainingOutcome(o.duration_hours, o.alpha_eval, o.new_version, o.mean_loss, o.steps)

    def params(self):
        n = C.c_int32()
        tot = C.c_int64()
        call("specsim_trainer_num_params", self.h, C.byref(n), C.byref(tot))
        out = []
        for i in range(n.value):
            nm = C.c_char_p()
            r, c = C.c_int64(), C.c_int64()
            call("specsim_trainer_param_info", self.h, i, C.byref(nm), C.byref(r), C.byref(c))
            out.append((nm.value.decode(), r.value, c.value))
        return out, tot.value

    def get_param(self, name):
        shp = {n: (r, c) for n, r, c in self.params()[0]}[name]
        a = np.zeros(shp, np.float32)
        call("specsim_trainer_get_param", self.h, name.encode(), ptr(a))
        return a

    def set_param(self, name, value):
        a = np.ascontiguousarray(value, np.float32)
        call("specsim_trainer_set_param", self.h, name.encode(), ptr(a))

    def get_grad(self, name):
        shp = {n: (r, c) for n, r, c in self.params()[0]}[name]
        a = np.zeros(shp, np.float32)
        call("specsim_trainer_get_grad", self.h, name.encode(), ptr(a))
        return a

    def keep_grads(self, on: bool = True):
        call("specsim_trainer_keep_grads", self.h, 1 if on else 0)

    _ROW_DTYPES = {"u": np.int32, "y": np.int32, "m": np.int32, "argmax": np.int32,
                   "lse": np.float32, "F": np.uint16}

    def read_rows(self, name):
        """Device per-row state of the last step / eval (u, y, m, argmax, lse
        over K*B*S rows; F as [B*S, layers*hidden] bf16 bits)."""
        n = C.c_int64()
        call("specsim_trainer_read_rows", self.h, name.encode(), None, 0, C.byref(n))
        a = np.zeros(n.value, self._ROW_DTYPES[name])
        call("specsim_trainer_read_rows", self.h, name.encode(), ptr(a), n.value, C.byref(n))
        if name == "F":
            a = a.reshape(self.shape["micro_batch"] * self.shape["seq_len"], -1)
        return a

    def set_embedding(self, e_bf16):
        a = np.ascontiguousarray(e_bf16, np.uint16)
        call("specsim_trainer_set_embedding", self.h, ptr(a))

    def get_embedding(self):
        a = np.zeros((self.shape["vocab"], self.shape["hidden"]), np.uint16)
        call("specsim_trainer_get_embedding", self.h, ptr(a))
        return a

    def set_step_count(self, k):
        call("specsim_trainer_set_step_count", self.h, k)

    def snapshot(self):
        """Device copy of the model (deploy gate)."""
        call("specsim_trainer_snapshot", self.h)

    def restore(self):
        call("specsim_trainer_restore", self.h)

    def region_begin(self):
        call("specsim_trainer_region", self.h, 0, None)

    def region_end(self) -> float:
        ms = C.c_double()
        call("specsim_trainer_region", self.h, 1, C.byref(ms))
        return ms.value

    def set_timing(self, on: bool):
        call("specsim_trainer_set_timing", self.h, 1 if on else 0)

    def last_step_ms(self):
        v = C.c_double(0)
        call("specsim_trainer_last_step_ms", self.h, C.byref(v))
        return v.value

    def phase_times(self):
        ms = (C.c_double * 7)()
        fl = (C.c_double * 7)()
        ln = (C.c_int32 * 7)()
        call("specsim_trainer_phase_times", self.h, ms, fl, ln)
        return {p: dict(ms=ms[i], flops=fl[i], launches=ln[i]) for i, p in enumerate(self.PHASES)}


# ---------------------------------------------------------------- controller
EVENT_NAMES = ("COLLECT_ON", "COLLECT_OFF", "TRAIN_TRIGGER", "DEPLOY", "REJECT")


@dataclass
class TriggerDecision:
    triggered: bool
    action: int  # 1 deploy, 0 tie, -1 reject / not triggered
    alpha_train: float
    n_train: int
    n_eval: int
    outcome: TrainingOutcome | None


class AdaptiveController:
    """Algorithm 1 (SPEC.md adapt_control) over the C ABI:
    observe() / record_sample() / maybe_trigger_training(trainer, buf)."""

    def __init__(self, lambda_short=0.9, lambda_long=0.99, epsilon=0.05, n_init=32,
                 n_threshold=2048):
        cfg = _lib.ControllerConfig(lambda_short, lambda_long, epsilon, n_init, n_threshold)
        self.h = C.c_void_p()
        call("specsim_controller_create", C.byref(cfg), C.byref(self.h))

    def close(self):
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.specsim_controller_destroy(self.h)
        self.h = None

    __del__ = close

    def observe(self, alpha: float):
        call("specsim_controller_observe", self.h, alpha)

    def record_sample(self, sample_id: int, alpha: float) -> bool:
        s = C.c_int32()
        call("specsim_controller_record_sample", self.h, sample_id, alpha, C.byref(s))
        return bool(s.value)

    def maybe_trigger_training(self, trainer: "DraftTrainer", buf: HiddenStateBuffer,
                               epochs: int = 1) -> TriggerDecision:
        d = _lib.TriggerDecision()
        call("specsim_controller_maybe_trigger_training", self.h, trainer.h, buf.h, epochs,
             C.byref(d))
        o = d.outcome
        out = TrainingOutcome(o.duration_hours, o.alpha_eval, o.new_version, o.mean_loss,
                              o.steps) if d.triggered else None
        return TriggerDecision(bool(d.triggered), d.action, d.alpha_train, d.n_train, d.n_eval,
                               out)

    def state(self) -> dict:
        s = _lib.ControllerState()
        call("specsim_controller_state_get", self.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def events(self):
        n = C.c_int64()
        call("specsim_controller_events", self.h, None, None, 0, C.byref(n))
        k = (C.c_int32 * max(1, n.value))()
        t = (C.c_int64 * max(1, n.value))()
        call("specsim_controller_events", self.h, k, t, n.value, C.byref(n))
        return [(EVENT_NAMES[k[i]], t[i]) for i in range(n.value)]
