SPECSIM_NO_GRAPH=1 timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python scripts/sanitize_step.py 1 > /tmp/rc_1.txt 2>&1
grep -n "attention_tc.cu:116" /tmp/rc_1.txt | head -3
L=$(grep -n "attention_tc.cu:1168" /tmp/rc_1.txt | head -1 | cut -d: -f1)
sed -n "$((L-3)),$((L+4))p" /tmp/rc_1.txt
grep -B2 "attention_tc.cu:1168" /tmp/rc_1.txt | grep "hazard detected" | sed -E 's/.*__shared__ (0x[0-9a-f]+) in block \(([0-9]+),.*/\1 \2/' | sort | uniq -c | sort -rn | head -12
grep -B1 "attention_tc.cu:1168" /tmp/rc_1.txt | grep "Write Thread" | sed -E 's/ at .*//' | sort | uniq -c | head
