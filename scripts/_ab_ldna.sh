set -u
mkdir -p gpurun_out
for v in 0 9 0 9; do
  lib=$PWD/probe/libv$v.so; [ $v = 0 ] && lib=$PWD/paper_2602_05145_b200/libspecsim_draft.so
  TAG=v$v SPECSIM_LIB=$lib timeout 300 python scripts/adamw_probe.py
done
STEPS=40 WARM=10 bash scripts/ab_r01.sh 2 "SPECSIM_X=0" "SPECSIM_LIB=$PWD/probe/libv9.so"
