#!/usr/bin/env bash
# Same-box A/B, alternating runs: the round-1 final build (_ab_r01/, a copy of
# commit fdf805c built in place; git-ignored) against HEAD under env variants.
# usage: scripts/ab_r01.sh REPS "ENV=1 ..." ...   (config "r01" = the round-1 tree)
mkdir -p gpurun_out
reps=$1; shift
for i in $(seq 1 $reps); do
  j=0
  for cfg in "$@"; do
    j=$((j+1))
    if [ "$cfg" = "r01" ]; then
      (cd _ab_r01 && timeout 600 python bench.py --steps ${STEPS:-40} --warmup ${WARM:-10} --no-e2e --no-cpu-baseline) > gpurun_out/ab_${j}_$i.json 2>/dev/null
    else
      env $cfg timeout 600 python bench.py --steps ${STEPS:-40} --warmup ${WARM:-10} --no-e2e --no-cpu-baseline --no-ce-probe > gpurun_out/ab_${j}_$i.json 2>/dev/null
    fi
    python -c "
import json,sys; b=json.load(open('gpurun_out/ab_${j}_$i.json'))
print('[$cfg]', round(b['value']), 'ms', b['ms_per_step'], 'clk', b['clocks']['sm_mhz'], {k: v['ms_per_step'] for k, v in b['phases'].items() if v['ms_per_step'] > 0.05})"
  done
done
