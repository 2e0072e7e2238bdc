set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for K in 1 3; do
  SPECSIM_NO_GRAPH=1 timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 1000000 python scripts/sanitize_step.py $K > /tmp/rc_$K.txt 2>&1
  echo "== racecheck K=$K rc=$? $(grep -E 'RACECHECK SUMMARY' /tmp/rc_$K.txt)"
  echo "reports: $(grep -c 'hazard detected' /tmp/rc_$K.txt)"
  echo "read sites:"; grep -E "Read Thread" /tmp/rc_$K.txt | sed -E 's/.* at //; s/\+0x[0-9a-f]+//' | sort | uniq -c
  echo "write sites:"; grep -E "Write Thread" /tmp/rc_$K.txt | sed -E 's/.* at //; s/\(CUtensor.*//; s/\+0x[0-9a-f]+//' | sort | uniq -c
  echo "addresses:"; grep -E "hazard detected" /tmp/rc_$K.txt | sed -E 's/.*__shared__ (0x[0-9a-f]+).*/\1/' | sort | uniq -c | sort -rn | head -20
done > gpurun_out/r02_racecheck_summary.txt 2>&1
cat gpurun_out/r02_racecheck_summary.txt | head -60
