#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list of the bench command + one full
# capture of the step GEMMs, then summarise into profiles/. Usage: tools/profile_round.sh r1 [skip count]
set -u
R=${1:-r1}
SKIP=${2:-12}
COUNT=${3:-3}
mkdir -p gpurun_out profiles
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$R.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rtp_gemm -s $SKIP -c $COUNT \
    -o gpurun_out/full_$R python bench.py --steps 3 --warmup 3 --no-cpu-baseline --eager > gpurun_out/ncu_full_$R.log 2>&1
ncu -i gpurun_out/full_$R.ncu-rep --page raw --csv > gpurun_out/full_raw_$R.csv 2>/dev/null
ncu -i gpurun_out/full_$R.ncu-rep --page source --csv --print-source sass > gpurun_out/full_src_$R.csv 2>/dev/null
python tools/summarize_ncu.py $R
