set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_trainer_gpu.py tests/test_ttt_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/kt_new.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
SPECSIM_LIB=$PWD/probe/libbase.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_kernel --csv --log-file gpurun_out/kt_base.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
for t in base new; do echo "$t: $(grep 'gemm_kernel' gpurun_out/kt_$t.csv | awk -F'","' '{print $(NF)}' | tr -d '"' | tail -23 | tr '\n' ' ')"; done
STEPS=40 WARM=10 bash scripts/ab_r01.sh 2 "SPECSIM_LIB=$PWD/probe/libbase.so" "SPECSIM_X=0"
