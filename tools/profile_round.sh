#!/bin/bash
# Run on the GPU box (gpurun): ncu launch list of the bench command + one full
# capture of the step GEMMs, then summarise into profiles/.
# Usage: tools/profile_round.sh <round tag> [skip] [count]   (BENCH_ARGS: extra bench.py args, e.g. "--config b")
set -u
R=${1:-r2}
SKIP=${2:-12}
COUNT=${3:-3}
ARGS=${BENCH_ARGS:-}
mkdir -p gpurun_out profiles
ncu --metrics gpu__time_duration.sum --clock-control none -c ${LAUNCH_CAP:-2500} --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-profile $ARGS > gpurun_out/ncu_launch_$R.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:rtp_gemm -s $SKIP -c $COUNT \
    -o gpurun_out/full_$R python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile --eager $ARGS \
    > gpurun_out/ncu_full_$R.log 2>&1
ncu -i gpurun_out/full_$R.ncu-rep --page raw --csv > gpurun_out/full_raw_$R.csv 2>/dev/null
ncu -i gpurun_out/full_$R.ncu-rep --page source --csv --print-source sass > gpurun_out/full_src_$R.csv 2>/dev/null
python tools/summarize_ncu.py $R
