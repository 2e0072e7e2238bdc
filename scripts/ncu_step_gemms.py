"""Summarise an `ncu --set full` capture of one C2 step's 23 GEMM launches
(scripts/ncu_step.sh) into profiles/<name>.json: per launch time, DRAM bytes,
tensor-pipe activity and SM clock, with the algorithmic bytes / FLOPs of the
launch (SURVEY §8(d) convention)."""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1, "ms": 1,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1,
         "Kcycle/second": 1e3, "Mcycle/second": 1e6, "Gcycle/second": 1e9, "%": 1}


def gemm_list(T=8192, H=4096, V=128256, Q=4096, KV=1024, I=14336, Vc=32768):
    L = [("fc fwd", T, H, 3 * H), ("qkv fwd + RoPE", T, Q + 2 * KV, 2 * H),
         ("o fwd + residual", T, H, Q), ("gate_up fwd", T, 2 * I, H),
         ("down fwd + residual", T, H, I), ("LM head CE fwd (stats + fp16 logits)", T, V, H)]
    for c in range(0, V, Vc):
        vn = min(Vc, V - c)
        L += [(f"LM head dX chunk {c // Vc}", T, H, vn),
              (f"LM head dW chunk {c // Vc} + AdamW", vn, H, T)]
    L += [("dact (down dX)", T, I, H), ("down dW + AdamW", H, I, T), ("dz (gate_up dX)", T, H, 2 * I),
          ("gate_up dW + AdamW", 2 * I, H, T), ("dO (o dX)", T, Q, H), ("o dW + AdamW", H, Q, T),
          ("dU (qkv dX)", T, 2 * H, Q + 2 * KV), ("qkv dW + AdamW", Q + 2 * KV, 2 * H, T),
          ("fc dW + AdamW", H, 3 * H, T)]
    return L


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]

    def get(r, key):
        i = hdr.index(key)
        v = r[i].replace(",", "")
        try:
            return float(v) * SCALE.get(units[i], 1)
        except ValueError:
            return None

    gl = gemm_list()
    launches = []
    for r, (label, M, N, K) in zip(data, gl):
        ms = get(r, "gpu__time_duration.sum")
        rd = get(r, "dram__bytes_read.sum")
        wr = get(r, "dram__bytes_write.sum")
        out_b = 4 if ("dX chunk" in label or "dz" in label or "dU" in label) else 2
        alg = 2 * (M * K + N * K) + out_b * M * N
        if "AdamW" in label:
            alg = 2 * (M * K + N * K) + 26 * M * N  # p m v read, p m v p16 written
        if "CE fwd" in label:  # fp16 logit offsets + one 16-byte partial per 128-column half tile
            alg = 2 * (M * K + N * K) + 2 * M * N + 2 * ((N + 255) // 256) * M * 16
        launches.append(dict(
            launch=label, kernel=r[hdr.index("Kernel Name")][:60], M=M, N=N, K=K, ms=ms,
            tflops=round(2 * M * N * K / (ms * 1e-3) / 1e12, 1), dram_read=rd, dram_write=wr,
            algorithmic_bytes=alg,
            # the tcgen05 pipe: this counter equals FLOPs / (148 x 8192 x clock x
            # time) launch for launch (profiles/r02_step_ncu_C2.txt); the
            # TriageCompute realtime counter used in round 1 does not
            tensor_active_pct=get(r, "sm__pipe_tensor_subpipe_hmma_cycles_active"
                                     ".avg.pct_of_peak_sustained_elapsed"),
            sm_ghz=round(get(r, "sm__cycles_elapsed.avg.per_second") / 1e9, 3)))
    ce = [l for l in launches if l["launch"].startswith("LM head CE fwd")]
    summary = dict(
        source=rep, note="ncu --set full --clock-control none, one C2 step (second step of "
        "`bench.py --steps 1 --warmup 1`); kernels serialised and replayed, so absolute "
        "times are cold-cache / unthrottled -- shares, bytes and pipe activity are the signal",
        kernel="gemm_kernel<0,0,EPI_CE_FWD,2> (LM head + CE forward, C2; logits stored as fp16)",
        dram_bytes_per_launch=(ce[0]["dram_read"] + ce[0]["dram_write"]) if ce else None,
        algorithmic_bytes=ce[0]["algorithmic_bytes"] if ce else None,
        total_ms=round(sum(l["ms"] for l in launches), 3), launches=launches)
    json.dump(summary, open(out, "w"), indent=1)
    for l in launches:
        print(f"{l['launch']:40s} {l['ms']:7.3f} ms {l['tflops']:7.1f} TF/s  dram "
              f"{(l['dram_read'] + l['dram_write']) / 1e9:6.2f} GB (alg {l['algorithmic_bytes'] / 1e9:5.2f})"
              f"  tensor {l['tensor_active_pct']:5.1f}%  {l['sm_ghz']} GHz")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
