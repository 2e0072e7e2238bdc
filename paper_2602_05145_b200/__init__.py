"""B200-native TIDE draft-training hot path (arxiv 2602.05145).

The product is the native library ``libspecsim_draft.so`` (C ABI in
``include/specsim_draft_trainer.h``; C++ API in ``include/specsim/``).  This
package holds its sources (``csrc/``) and a thin ctypes mirror of the
reference-facing interface (``api``) used by tests and the benchmark.
"""
from ._lib import LIB_PATH, SpecsimError, DomainError, ConfigError, lib  # noqa: F401

__all__ = ["LIB_PATH", "SpecsimError", "DomainError", "ConfigError", "lib"]
