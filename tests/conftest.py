import os
import sys
import pathlib

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

# torch first: it links its own (newer) libnccl.so.2.  The library dlopens
# NCCL lazily and reuses an already loaded copy; if it loaded the system
# libnccl.so.2 first (a forced-NCCL test before any test imported torch), a
# later `import torch` would bind to that older copy and fail on a missing
# symbol.  Importing torch here fixes the order for the whole session.
try:
    import torch  # noqa: F401
except ImportError:  # the oracle / host tests do not need it
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")
