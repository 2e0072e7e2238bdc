#!/usr/bin/env bash
# GEMM rasterisation A/B by DRAM bytes and duration per launch (ncu metric
# pass over one C2 step per variant; VAR=value pairs per variant).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 900 ncu --metrics $M --clock-control none --csv --page raw -k regex:gemm_kernel \
    --log-file gpurun_out/l2ab_$i.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
  echo "== $cfg"
  python - "$i" <<'PY'
import sys
sys.path.insert(0, "scripts")
import ncu_r02_summary as m
rows = m.load(f"gpurun_out/l2ab_{sys.argv[1]}.csv")
rows = rows[len(rows) // 2:]  # second step
gl = m.gemm_list(__import__("paper_2602_05145_b200.api", fromlist=["api"]).CONFIGS["C2"], 8192)
for (label, M_, N, K), r in zip(gl, rows):
    t = r["gpu__time_duration.sum"]; d = r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"]
    print(f"{label:36s} {t*1e3:7.3f} ms  dram {d/1e9:6.2f} GB  util {r.get('sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed',0):5.1f}%  {r['sm__cycles_elapsed.avg.per_second']/1e9:.2f} GHz")
PY
done
