"""One training step (optionally TTT) + eval at a small shape, for
compute-sanitizer runs: SPECSIM_NO_GRAPH=1 compute-sanitizer python scripts/sanitize_step.py"""
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402  (synthetic captures only)
from paper_2602_05145_b200 import api  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = dict(api.CONFIGS["C1"], micro_batch=3, ttt_steps=K)
tr = api.DraftTrainer(c, seed=3)
buf = api.HiddenStateBuffer(api.SignalGeometry(c["hidden"]), 4096)
for i, L in enumerate([c["seq_len"] + 2 + K, 70, 130]):
    cap = oracle.synth_capture(3, i, L, c["vocab"], c["hidden"])
    buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
# one sample through extract_signals (host layers -> staging -> TMA bulk-copy pack kernel)
import numpy as np  # noqa: E402
rng = np.random.default_rng(0)
rows = 40
layers = [rng.integers(0, 1 << 15, (rows, c["hidden"]), dtype=np.uint16) & 0x3FFF for _ in range(3)]
acc = np.arange(0, rows, 2, dtype=np.int32)
buf.extract_signals(9, 0.5, layers, rng.integers(0, c["vocab"], len(acc)), accepted_idx=acc)
r = tr.step(buf, [0, 1, 9])
e = tr.eval(buf, [0, 1])
print("K", K, "loss", r["loss"], "eval", e["loss"])
tr.close()
buf.close()
