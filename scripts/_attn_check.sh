set -u
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:attn_fwd --csv --log-file gpurun_out/attn_fwd_$tag.csv python scripts/attn_probe.py > /dev/null 2>&1
  echo "== $tag"; grep -E "attn_fwd" gpurun_out/attn_fwd_$tag.csv | grep duration | awk -F'","' '{print $(NF)}' | tr '\n' ' '; echo
}
run fwd1 SPECSIM_ATTN_FWD1=1
run poly0 SPECSIM_X=1
run poly1 SPECSIM_LIB=$PWD/_ab_r01/libspecsim_poly1.so
run poly2 SPECSIM_LIB=$PWD/_ab_r01/libspecsim_poly2.so
SPECSIM_LIB=$PWD/_ab_r01/libspecsim_poly1.so timeout 900 python -m pytest tests/test_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
