#!/usr/bin/env bash
# ncu --set full of the step's GEMMs with the lowest tensor-pipe activity in
# profiles/r02_step_ncu_C2.txt: d act (SwiGLU-backward epilogue), o / qkv / fc dW
# (+AdamW), second C2 step of scripts/step_probe.py.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 37 -c 1 \
  -o gpurun_out/r02_dact -f python scripts/step_probe.py --steps 2 > gpurun_out/r02_dact.log 2>&1
echo "dact rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 42 -c 4 \
  -o gpurun_out/r02_smalldw -f python scripts/step_probe.py --steps 2 > gpurun_out/r02_smalldw.log 2>&1
echo "dw rc=$?"
for r in r02_dact r02_smalldw; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv > gpurun_out/${r}_source.csv 2>/dev/null
done
ls -la gpurun_out/r02_dact* gpurun_out/r02_smalldw*
