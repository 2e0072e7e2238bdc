set -u
mkdir -p gpurun_out
for rep in 1 2; do
for j in 5 2 8 1; do
  SPECSIM_BENCH_E2E_JOB=$j timeout 600 python bench.py --steps 30 --warmup 10 --no-cpu-baseline --no-ce-probe > gpurun_out/e2ejob_$j.json 2>/dev/null
  python -c "
import json; b=json.load(open('gpurun_out/e2ejob_$j.json'))
print('job $j value', round(b['value']), b['ms_per_step'], 'e2e', round(b['e2e']['value']), b['e2e']['ms_per_step'], 'clk', b['clocks']['sm_mhz'])"
done
done
