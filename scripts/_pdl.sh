set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_trainer_gpu.py tests/test_ttt_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
STEPS=40 WARM=10 bash scripts/ab_r01.sh 3 "SPECSIM_GEMM_PDL=0" "SPECSIM_GEMM_PDL=1"
