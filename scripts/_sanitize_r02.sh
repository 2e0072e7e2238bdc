set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for t in "memcheck 1" "memcheck 3" "synccheck 1" "racecheck 1"; do
  set -- $t
  extra=""; [ $1 = racecheck ] && extra="--racecheck-report hazard"
  SPECSIM_NO_GRAPH=1 timeout 1200 $CS --tool $1 $extra python scripts/sanitize_step.py $2 > gpurun_out/san_$1_$2.txt 2>&1
  echo "$1 K=$2 rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_$1_$2.txt | tail -2 | tr '\n' ' ')"
done
