"""Driver for the ncu captures of one draft-training step (scripts/ncu_r02.sh):
a C2 trainer (or --config), one resident micro-batch, `--steps` optimiser
steps through the C ABI (the first is the warm-up the summaries skip).
Nothing is timed here: the numbers come from ncu."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_05145_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    c = dict(api.CONFIGS[a.config])
    B, S, H, V = c["micro_batch"], c["seq_len"], c["hidden"], c["vocab"]
    buf = api.HiddenStateBuffer(api.SignalGeometry(H), B * (S + 2) + 64)
    for i in range(B):
        cap = api.synth_capture(20260217, i, S + 2, V, H)
        buf.append_packed(i, cap["alpha_s"], cap["features"], cap["ids"])
    tr = api.DraftTrainer(c, seed=20260217)
    for _ in range(a.steps):
        r = tr.step(buf, list(range(B)))
    print(f"{a.config}: {a.steps} steps, last loss {r['loss']:.4f}", file=sys.stderr)
    tr.close()
    buf.close()


if __name__ == "__main__":
    main()
