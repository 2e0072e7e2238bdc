set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q -p no:cacheprovider -k "large_configs or fwd_bwd" 2>&1 | tail -3
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_fwd --csv --log-file gpurun_out/attn_$tag.csv python scripts/attn_probe.py > /dev/null 2>&1
  echo "== $tag"; grep -E "attn_" gpurun_out/attn_$tag.csv | grep duration | awk -F'","' '{split($5,a,"("); print a[1], $(NF)}' | sed 's/void specsim::attn::<unnamed>:://' | tr '\n' ';'; echo
}
run pair SPECSIM_X=1
run fwd2 SPECSIM_ATTN_FWD_PAIR=0
