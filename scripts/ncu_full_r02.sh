#!/usr/bin/env bash
# ncu --set full (source-correlated) of: the LM-head dX and dW+AdamW chunk-0
# GEMMs and the four attention kernels of the second C2 step.  Reports and
# their details / source pages land in gpurun_out/.
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 29 -c 2 \
  -o gpurun_out/r02_lmhead -f python scripts/step_probe.py --steps 2 > gpurun_out/r02_lmhead.log 2>&1
echo "lmhead rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_ -s 4 -c 4 \
  -o gpurun_out/r02_attn -f python scripts/step_probe.py --steps 2 > gpurun_out/r02_attn.log 2>&1
echo "attn rc=$?"
for r in r02_lmhead r02_attn; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out/r02_lmhead* gpurun_out/r02_attn*
