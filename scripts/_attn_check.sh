set -u
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ --csv --log-file gpurun_out/attn_$tag.csv python scripts/attn_probe.py > /dev/null 2>&1
  echo "== $tag"; grep -E "attn_" gpurun_out/attn_$tag.csv | grep duration | awk -F'","' '{split($5,a,"("); print a[1], $(NF)}' | sed 's/void specsim::attn::<unnamed>:://' | tail -4 | tr '\n' ';'; echo
}
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
run base SPECSIM_LIB=$PWD/probe/libbase.so
run head SPECSIM_X=1
timeout 900 python -m pytest tests/test_ttt_gpu.py tests/test_trainer_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2

