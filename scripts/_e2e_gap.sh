set -u
mkdir -p gpurun_out
for rep in 1 2; do
for m in dma resident; do
  SPECSIM_BENCH_E2E_PROBE=$m timeout 600 python bench.py --steps 30 --warmup 10 --no-cpu-baseline --no-ce-probe > gpurun_out/gap_$m.json 2>/dev/null
  python -c "
import json; b=json.load(open('gpurun_out/gap_$m.json')); e=b['e2e']
print('$m value', round(b['value']), 'e2e', round(e['value']), 'ratio', round(e['value']/b['value'],4), 'clk', b['clocks']['sm_mhz'])"
done
done
