set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd2 -s 2 -c 1 -o gpurun_out/attn_fwd2 -f python scripts/attn_probe.py > gpurun_out/attn_ncu_run.txt 2>&1
ncu -i gpurun_out/attn_fwd2.ncu-rep --page source --csv > gpurun_out/attn_fwd2_source.csv 2>/dev/null
ncu -i gpurun_out/attn_fwd2.ncu-rep --page details --csv > gpurun_out/attn_fwd2_details.csv 2>/dev/null
ncu -i gpurun_out/attn_fwd2.ncu-rep --page raw --csv > gpurun_out/attn_fwd2_raw.csv 2>/dev/null
ls -la gpurun_out/
