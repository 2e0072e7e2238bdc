#!/usr/bin/env bash
# Round-2 ncu evidence (run on a B200 via gpurun; outputs in gpurun_out/):
#  1. one metric pass over every kernel of two C2 steps (scripts/step_probe.py):
#     duration, DRAM bytes, SM clock and the candidate tensor-pipe counters;
#  2. the standalone AdamW kernel over all parameters (SPECSIM_NO_FUSED_ADAMW=1);
#  3. the summary (scripts/ncu_r02_summary.py) -> gpurun_out/r02_step_ncu.{json,txt}.
set -u
CFG=${1:-C2}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
M=$M,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
M=$M,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --metrics $M --clock-control none --csv --page raw \
  --log-file gpurun_out/r02_step_${CFG}.csv python scripts/step_probe.py --config $CFG --steps 2 \
  > gpurun_out/r02_step_${CFG}.log 2>&1
echo "step capture rc=$?"
SPECSIM_NO_FUSED_ADAMW=1 timeout 600 ncu --metrics $M --clock-control none --csv --page raw \
  -k regex:adamw_kernel --log-file gpurun_out/r02_adamw_${CFG}.csv \
  python scripts/step_probe.py --config $CFG --steps 2 > gpurun_out/r02_adamw_${CFG}.log 2>&1
echo "adamw capture rc=$?"
python scripts/ncu_r02_summary.py gpurun_out/r02_step_${CFG}.csv gpurun_out/r02_adamw_${CFG}.csv \
  $CFG gpurun_out/r02_step_ncu_${CFG}
