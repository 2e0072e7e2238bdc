set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_trainer_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/sw_new.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
SPECSIM_LIB=$PWD/probe/libv11.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/sw_base.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
for t in base new; do echo "$t: $(grep 'gemm_kernel<0, 1, 8' gpurun_out/sw_$t.csv | awk -F'","' '{print $(NF)}' | tr '\n' ' ')"; done
STEPS=40 WARM=10 bash scripts/ab_r01.sh 2 "SPECSIM_LIB=$PWD/probe/libv11.so" "SPECSIM_X=0"
