#!/usr/bin/env bash
# Round-2 measurement artefacts in one GPU session (outputs in gpurun_out/):
# bench lines C2 (x2), C4, C5, C2-TTT7, C5 strong scaling at global batch 16,
# the launch list of one C2 step, the metric capture of one C2 step
# (scripts/ncu_r02.sh: HBM kernels + GEMM tcgen05 counter), and the SPEC
# sim_serving runs.
set -u
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name"; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv) > gpurun_out/r02_host.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_C2_a.json 2> gpurun_out/r02_bench_C2_a.err
timeout 900 python bench.py --steps 30 --warmup 10 --no-cpu-baseline --no-ce-probe > gpurun_out/r02_bench_C2_b.json 2> gpurun_out/r02_bench_C2_b.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 6 --no-cpu-baseline > gpurun_out/r02_bench_C4.json 2> gpurun_out/r02_bench_C4.err
timeout 900 python bench.py --config C5 --steps 20 --warmup 6 --no-cpu-baseline > gpurun_out/r02_bench_C5.json 2> gpurun_out/r02_bench_C5.err
timeout 900 python bench.py --ttt 7 --steps 12 --warmup 4 --no-cpu-baseline --no-ce-probe > gpurun_out/r02_bench_C2_ttt7.json 2> gpurun_out/r02_bench_C2_ttt7.err
timeout 900 python bench.py --config C5 --global-batch 16 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-ce-probe > gpurun_out/r02_bench_C5_gb16.json 2> gpurun_out/r02_bench_C5_gb16.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/r02_launches_C2.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
echo "launches rc=$?"
python scripts/launch_table.py gpurun_out/r02_launches_C2.csv > gpurun_out/r02_launches_C2.txt 2>&1
bash scripts/ncu_r02.sh C2 > gpurun_out/r02_ncu_C2.log 2>&1
for m in tide_default tide_adaptive speculation_on_no_training speculation_off; do
  integration/sim_serving/_build/sim_serving --mode $m --profile integration/sim_serving/gpt-oss-120b.csv \
    --requests 500 --concurrency 8 --mean-tokens 130 --threshold 128 >> gpurun_out/r02_sim_serving.jsonl 2>&1
done
for f in gpurun_out/r02_bench_*.json; do echo "$f: $(head -c 200 $f)"; done
