STEPS=60 WARM=10 bash scripts/ab_r01.sh 3 r01 "SPECSIM_X=0" "SPECSIM_F_GATHER=1"
(cd _ab_r01 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ../gpurun_out/launch_r01.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline >/dev/null 2>&1)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launch_head.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ce-probe >/dev/null 2>&1
ls -la gpurun_out/
