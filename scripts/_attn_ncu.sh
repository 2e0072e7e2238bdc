set -u
mkdir -p gpurun_out
K=${1:-attn_bwd_kv}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o gpurun_out/$K -f python scripts/attn_probe.py > gpurun_out/${K}_run.txt 2>&1
ncu -i gpurun_out/$K.ncu-rep --page source --csv > gpurun_out/${K}_source.csv 2>/dev/null
ncu -i gpurun_out/$K.ncu-rep --page details --csv > gpurun_out/${K}_details.csv 2>/dev/null
ncu -i gpurun_out/$K.ncu-rep --page raw --csv > gpurun_out/${K}_raw.csv 2>/dev/null
ls -la gpurun_out/$K*
