#!/usr/bin/env bash
# ncu --set full over the 23 GEMM launches of one C2 step (the second step the
# bench runs), plus the launch list of two steps.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel \
  -s 23 -c 23 -o gpurun_out/step_gemms -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_step.txt 2>&1
echo "full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e \
  --no-cpu-baseline > /dev/null 2>&1
echo "launches rc=$?"
