#!/usr/bin/env bash
# Back-to-back steady-state A/B runs on one box: VAR=value pairs per run.
mkdir -p gpurun_out
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 600 python bench.py --steps ${STEPS:-40} --warmup ${WARM:-20} --no-e2e --no-cpu-baseline > gpurun_out/ab_$i.json 2>gpurun_out/ab_$i.err
  python -c "
import json,sys; b=json.load(open('gpurun_out/ab_$i.json'))
print('$cfg', round(b['value']), 'ms', b['ms_per_step'], 'clk', b['clocks']['sm_mhz'], {k: v['ms_per_step'] for k, v in b['phases'].items() if v['ms_per_step'] > 0.05})"
done
