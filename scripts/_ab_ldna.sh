set -u
mkdir -p gpurun_out
STEPS=40 WARM=10 bash scripts/ab_r01.sh 3 "SPECSIM_X=0" "SPECSIM_LIB=$PWD/probe/libv9.so" "SPECSIM_LIB=$PWD/probe/libv10.so"
