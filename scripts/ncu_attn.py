"""Summarise an `ncu --set full` capture of one C2 step's attention launches
(forward, bwd_dot, dQ, dK/dV) into JSON + a text table: time, tensor FLOP/s
(causal FLOPs, SURVEY §8(d) convention), tensor-pipe activity, MUFU / FMA pipe
activity, DRAM bytes and SM clock.

    ncu --set full --clock-control none -k regex:attn -c 4 -o rep python bench.py \
        --steps 1 --warmup 0 --no-e2e --no-cpu-baseline
    python scripts/ncu_attn.py rep.ncu-rep out.json
"""
import csv
import io
import json
import subprocess
import sys

from ncu_step_gemms import SCALE

# C2: B 4, S 2048, 32 query heads of 128; causal matmul = B*nh*S*(S+1)/2*hd*2 FLOP
B, S, NH, HD = 4, 2048, 32, 128
MM = B * NH * S * (S + 1) / 2 * HD * 2
FLOPS = {"attn_fwd": 2 * MM, "attn_bwd_q": 3 * MM, "attn_bwd_kv": 4 * MM}
PIPES = {
    "tensor_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime"
                  ".avg.pct_of_peak_sustained_elapsed",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]

    def get(r, key):
        if key not in hdr:
            return None
        i = hdr.index(key)
        try:
            return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        except ValueError:
            return None

    res = []
    for r in data:
        name = r[hdr.index("Kernel Name")]
        ms = get(r, "gpu__time_duration.sum")
        fl = next((v for k, v in FLOPS.items() if k in name), None)
        d = dict(kernel=name[:60], ms=ms, tflops=round(fl / (ms * 1e-3) / 1e12, 1) if fl else None,
                 dram_gb=round(((get(r, "dram__bytes_read.sum") or 0) +
                                (get(r, "dram__bytes_write.sum") or 0)) / 1e9, 3),
                 sm_ghz=round((get(r, "sm__cycles_elapsed.avg.per_second") or 0) / 1e9, 3))
        for k, m in PIPES.items():
            v = get(r, m)
            d[k] = round(v, 1) if v is not None else None
        res.append(d)
    json.dump(dict(source=rep, note="ncu --set full --clock-control none, C2 dims, one step; "
                   "serialised replays: compare pipe activity and shares, not absolutes",
                   launches=res), open(out, "w"), indent=1)
    for d in res:
        print(f"{d['kernel'][:44]:44s} {d['ms']:7.3f} ms  {d['tflops'] or 0:7.1f} TF/s  "
              f"tensor {d['tensor_pct']}%  xu {d['xu_pct']}%  fma {d['fma_pct']}%  "
              f"issue {d['issue_pct']}%  dram {d['dram_gb']} GB  {d['sm_ghz']} GHz")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
