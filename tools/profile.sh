#!/usr/bin/env bash
# GPU-box profiling recipe (B200_PROFILING.md): launch list of bench.py + one
# full ncu capture of the two aggregation kernels.  Usage: tools/profile.sh TAG
set -uo pipefail
TAG="${1:-r1}"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 70 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 12 --warmup 8 \
    > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sd_|prep|xpass|ypass|post" -s 10 -c 5 \
    -o gpurun_out/prof_${TAG} -f python tools/quick_timing.py > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
echo done
