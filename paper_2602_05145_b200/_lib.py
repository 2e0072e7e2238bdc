"""ctypes binding of the C ABI declared in include/specsim_draft_trainer.h.

This is the reference-side binding a Python caller would add (the same
entry points a cgo / JNI stub would bind).  It loads the in-tree
``libspecsim_draft.so`` and fails loudly if it is missing: there is no CPU
fallback for the trainer.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
# SPECSIM_LIB selects another build of the same library (A/B experiments)
LIB_PATH = pathlib.Path(os.environ.get("SPECSIM_LIB", str(_HERE / "libspecsim_draft.so")))

OK, EDOMAIN, ECONFIG, ECUDA, ENCCL = 0, 1, 2, 3, 4


class SpecsimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class DomainError(SpecsimError, ValueError):
    """std::invalid_argument in the reference (CLI exit 1)."""


class ConfigError(SpecsimError):
    """specsim::ConfigError in the reference (errors.hpp:10-13, CLI exit 2)."""


class SignalGeometry(C.Structure):
    _fields_ = [("hidden_dim", C.c_int32), ("layers_tapped", C.c_int32),
                ("bytes_per_element", C.c_int32)]


class HsbufStats(C.Structure):
    _fields_ = [("records", C.c_int64), ("bytes", C.c_int64), ("flushes", C.c_int64),
                ("cumulative_bytes", C.c_int64), ("samples", C.c_int64),
                ("resident_tokens", C.c_int64)]


class DraftShape(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("vocab", C.c_int32), ("seq_len", C.c_int32),
                ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("ffn", C.c_int32), ("layers_tapped", C.c_int32), ("micro_batch", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_double), ("ttt_steps", C.c_int32),
                ("ttt_decay", C.c_float)]


class AdamW(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float)]


class StepResult(C.Structure):
    _fields_ = [("loss", C.c_double), ("valid_tokens", C.c_int64),
                ("top1_correct", C.c_int64), ("positions", C.c_int64), ("ms", C.c_double)]


class TrainingOutcome(C.Structure):
    _fields_ = [("duration_hours", C.c_double), ("alpha_eval", C.c_double),
                ("new_version", C.c_int64), ("mean_loss", C.c_double), ("steps", C.c_int64)]


class CaptureStats(C.Structure):
    _fields_ = [("records", C.c_int64), ("bytes", C.c_int64), ("flushes", C.c_int64),
                ("cumulative_bytes", C.c_int64), ("samples", C.c_int64), ("files", C.c_int64),
                ("file_bytes", C.c_int64)]


class ControllerConfig(C.Structure):
    _fields_ = [("lambda_short", C.c_double), ("lambda_long", C.c_double),
                ("epsilon", C.c_double), ("n_init", C.c_int32), ("n_threshold", C.c_int64)]


class ControllerState(C.Structure):
    _fields_ = [("initialized", C.c_int32), ("collection_enabled", C.c_int32),
                ("ema_short", C.c_double), ("ema_long", C.c_double),
                ("stored_samples", C.c_int64), ("draft_version", C.c_int64),
                ("observations", C.c_int64), ("n_events", C.c_int64)]


class TriggerDecision(C.Structure):
    _fields_ = [("triggered", C.c_int32), ("action", C.c_int32), ("alpha_train", C.c_double),
                ("n_train", C.c_int64), ("n_eval", C.c_int64), ("outcome", TrainingOutcome)]


P = C.c_void_p
I32, I64, U64, F32, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
PI32, PI64, PU64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
PF32, PF64, PU16 = C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_uint16)

# name -> argtypes (all return int status unless listed in _RESTYPE)
SIGNATURES = {
    "specsim_last_error": [],
    "specsim_version": [],
    "specsim_kernel_launches": [PU64],
    "specsim_rng_create": [U64, C.POINTER(P)],
    "specsim_rng_destroy": [P],
    "specsim_rng_uniform": [P, PF64],
    "specsim_rng_normal": [P, F64, F64, PF64],
    "specsim_rng_geometric": [P, F64, PI64],
    "specsim_rng_next_u64": [P, PU64],
    "specsim_expected_accept_length": [F64, I32, PF64],
    "specsim_sample_accept_length": [P, F64, I32, PI32],
    "specsim_alpha_from_accept_length": [F64, I32, PF64],
    "specsim_split_train_eval": [I64, PI64, PI64],
    "specsim_current_alpha": [F64, F64, F64, F64, PF64],
    "specsim_dp_shard": [I64, I32, I32, I32, I64, P, PI32],
    "specsim_dp_buckets": [C.POINTER(DraftShape), I32, P, P, I32, PI32, PI32],
    "specsim_bytes_per_token": [C.POINTER(SignalGeometry), PI64],
    "specsim_synth_capture": [U64, I64, I32, I32, I32, I32, F64, I32, P, P, P, PI32, PF64],
    "specsim_hsbuf_create": [C.POINTER(SignalGeometry), I64, I64, C.c_int, C.POINTER(P)],
    "specsim_hsbuf_destroy": [P],
    "specsim_hsbuf_append": [P, I64, F64, C.POINTER(P), I64, I64, P, P, I32, C.c_int],
    "specsim_hsbuf_append_packed": [P, I64, F64, P, P, I32, C.c_int],
    "specsim_hsbuf_sync": [P],
    "specsim_hsbuf_stats_get": [P, C.POINTER(HsbufStats)],
    "specsim_hsbuf_sample_info": [P, I64, PI32, PF64],
    "specsim_hsbuf_read_sample": [P, I64, P, P],
    "specsim_nccl_unique_id": [P],
    "specsim_trainer_create": [C.POINTER(DraftShape), C.POINTER(AdamW), U64, C.c_int, C.c_int,
                               P, C.c_int, C.POINTER(P)],
    "specsim_trainer_destroy": [P],
    "specsim_trainer_step": [P, P, PI64, I32, I64, C.POINTER(StepResult)],
    "specsim_trainer_eval": [P, P, PI64, I32, C.POINTER(StepResult)],
    "specsim_trainer_train": [P, P, PI64, I64, PI64, I64, I32, C.POINTER(TrainingOutcome)],
    "specsim_trainer_num_params": [P, PI32, PI64],
    "specsim_trainer_param_info": [P, I32, C.POINTER(C.c_char_p), PI64, PI64],
    "specsim_trainer_get_param": [P, C.c_char_p, P],
    "specsim_trainer_set_param": [P, C.c_char_p, P],
    "specsim_trainer_get_grad": [P, C.c_char_p, P],
    "specsim_trainer_keep_grads": [P, C.c_int],
    "specsim_trainer_set_embedding": [P, P],
    "specsim_trainer_get_embedding": [P, P],
    "specsim_trainer_set_step_count": [P, I64],
    "specsim_trainer_set_timing": [P, C.c_int],
    "specsim_trainer_region": [P, C.c_int, PF64],
    "specsim_trainer_phase_times": [P, PF64, PF64, PI32],
    "specsim_trainer_last_step_ms": [P, PF64],
    "specsim_trainer_read_rows": [P, C.c_char_p, P, I64, PI64],
    "specsim_capture_create": [C.POINTER(SignalGeometry), C.c_char_p, I64, C.c_int, C.POINTER(P)],
    "specsim_capture_destroy": [P],
    "specsim_capture_append": [P, I64, C.POINTER(P), I64, I64, P, P, I32, P],
    "specsim_capture_append_batch": [P, P, I32, P, P, C.POINTER(P), I64, I64, P, P],
    "specsim_capture_end_sample": [P, I64, F64],
    "specsim_capture_flush": [P],
    "specsim_capture_close": [P],
    "specsim_capture_stats_get": [P, C.POINTER(CaptureStats)],
    "specsim_capture_file": [P, I64, C.c_char_p, I64],
    "specsim_hsbuf_load_shards": [P, C.POINTER(C.c_char_p), I32, PI64],
    "specsim_trainer_snapshot": [P],
    "specsim_trainer_restore": [P],
    "specsim_controller_create": [C.POINTER(ControllerConfig), C.POINTER(P)],
    "specsim_controller_destroy": [P],
    "specsim_controller_observe": [P, F64],
    "specsim_controller_record_sample": [P, I64, F64, PI32],
    "specsim_controller_maybe_trigger_training": [P, P, P, I32, C.POINTER(TriggerDecision)],
    "specsim_controller_state_get": [P, C.POINTER(ControllerState)],
    "specsim_controller_events": [P, PI32, PI64, I64, PI64],
    "specsim_debug_gemm": [C.c_int, C.c_int, C.c_int, I32, I32, I32, P, I64, P, I64, P, I64, P,
                           I64, I32, PF32],
    "specsim_debug_attention": [I32, I32, I32, I32, I32, P, P, P, P, P],
}
_RESTYPE = {"specsim_last_error": C.c_char_p, "specsim_version": C.c_char_p}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def kernel_launches() -> int:
    o = C.c_uint64()
    check(lib().specsim_kernel_launches(C.byref(o)))
    return o.value


def exported_symbols() -> list[str]:
    L = lib()
    return [n for n in SIGNATURES if getattr(L, n, None) is not None]


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().specsim_last_error().decode(errors="replace")
    if status == EDOMAIN:
        raise DomainError(status, msg)
    if status == ECONFIG:
        raise ConfigError(status, msg)
    raise SpecsimError(status, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(a) -> C.c_void_p:
    """Raw data pointer of a numpy array (must stay alive during the call)."""
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


if os.environ.get("SPECSIM_EAGER_LOAD"):
    lib()
