#!/usr/bin/env bash
# One GPU session: parity tests, smoke, bench, ncu launch list + one full GEMM capture.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
(nproc; lscpu | grep -E "Model name|Socket|Thread") > gpurun_out/host.txt
timeout 900 python -m pytest tests/ -m gpu -x -q -p no:cacheprovider -s 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_run.txt 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-gemm_kernel} -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-3} \
     -o gpurun_out/prof -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_run.txt 2>&1
fi
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt | tail -2; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
