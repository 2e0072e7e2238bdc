#!/usr/bin/env bash
# One GPU session that regenerates the round's measurement artefacts:
# default bench line (C2, e2e + CPU baseline), C4 / C5 / C2-TTT7 lines, the
# ncu launch list of one C2 step, and the ncu --set full capture of its 23
# GEMM launches.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name") > gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 900 python bench.py --config C4 --steps 20 --warmup 6 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 900 python bench.py --config C5 --steps 20 --warmup 6 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 python bench.py --ttt 7 --steps 12 --warmup 4 --no-cpu-baseline > gpurun_out/bench_C2_ttt7.json 2> gpurun_out/bench_C2_ttt7.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e \
  --no-cpu-baseline > /dev/null 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel \
  -s 23 -c 23 -o gpurun_out/step_gemms -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_step.txt 2>&1
echo "full rc=$?"
# summarise on the box: gpurun copies back <= 64 MiB
python scripts/ncu_step_gemms.py gpurun_out/step_gemms.ncu-rep gpurun_out/gemm_ncu.json > gpurun_out/gemm_ncu.txt 2>&1
python scripts/launch_table.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
rm -f gpurun_out/step_gemms.ncu-rep
for f in gpurun_out/bench_*.json; do echo "$f: $(head -c 300 $f)"; done
