#!/usr/bin/env bash
# Same-box A/B of the round-1 final build (_ab_r01/, a copy of commit fdf805c built
# in place; git-ignored) against HEAD: alternating default-config bench runs.
mkdir -p gpurun_out
for i in 1 2; do
  (cd _ab_r01 && timeout 600 python bench.py --steps 30 --warmup 10 --no-e2e --no-cpu-baseline) > gpurun_out/abr01_r01_$i.json 2>/dev/null
  timeout 600 python bench.py --steps 30 --warmup 10 --no-e2e --no-cpu-baseline --no-ce-probe > gpurun_out/abr01_head_$i.json 2>/dev/null
done
for f in gpurun_out/abr01_*.json; do python -c "
import json,sys; b=json.load(open('$f'))
print('$f', round(b['value']), 'ms', b['ms_per_step'], 'clk', b['clocks']['sm_mhz'], {k: v['ms_per_step'] for k, v in b['phases'].items() if v['ms_per_step'] > 0.05})"; done
