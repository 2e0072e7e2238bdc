set -u
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:attn_fwd --csv --log-file gpurun_out/attn_fwd_$tag.csv python scripts/attn_probe.py > /dev/null 2>&1
  echo "== $tag"; grep -E "attn_fwd" gpurun_out/attn_fwd_$tag.csv | grep duration | awk -F'","' '{print $(NF)}' | tr '\n' ' '; echo
}
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
run fwd1 SPECSIM_ATTN_FWD1=1
run head SPECSIM_X=1
for t in poly1; do run $t SPECSIM_LIB=$PWD/_ab_r01/libspecsim_$t.so; done
timeout 900 python -m pytest tests/test_ttt_gpu.py tests/test_trainer_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
