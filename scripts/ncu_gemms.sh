#!/usr/bin/env bash
# Full ncu captures of selected GEMM template instances in the C2 step.
mkdir -p gpurun_out
i=0
for k in "$@"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${k}" -s ${NCU_SKIP:-2} -c 1 -o gpurun_out/g$i -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_g$i.txt 2>&1
  echo "$k -> g$i rc=$?"
done
