set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_trainer_gpu.py tests/test_parity_large_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in 1 0; do
  SPECSIM_CE_GRAD_TMA=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ce_grad --csv --log-file gpurun_out/ce_$v.csv python scripts/step_probe.py --steps 2 > /dev/null 2>&1
  echo "TMA=$v: $(grep duration gpurun_out/ce_$v.csv | awk -F'","' '{print $(NF)}' | tr -d '"' | tr '\n' ' ')"
done
STEPS=40 WARM=10 bash scripts/ab_r01.sh 2 "SPECSIM_CE_GRAD_TMA=0" "SPECSIM_CE_GRAD_TMA=1"
