#!/usr/bin/env bash
# GPU-box profiling recipe (B200_PROFILING.md), as used for profiles/r02_*:
# the launch list of bench.py, one ncu --set full capture per kernel at one
# frame per launch and at bench.py's two frames per launch (QT_BATCH=2; the
# capture profiles/ncu_traffic.json is written from, stamped with the source
# digest bench.py checks).  Usage: tools/profile.sh TAG ; then, here:
#   QT_BATCH=2 python tools/ncu_traffic.py gpurun_out/prof_TAG_b2_raw.csv TAG
#   python tools/ncu_summary.py gpurun_out/prof_TAG_raw.csv > profiles/TAG_ncu_full_summary.txt
#   python tools/launch_summary.py gpurun_out/launches_TAG.csv > profiles/TAG_launches_summary.txt
set -uo pipefail
TAG="${1:-r2}"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 70 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 12 --warmup 8 \
    > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sd_|prep|xpass|ypass|post" -s 10 -c 5 \
    -o gpurun_out/prof_${TAG} -f python tools/quick_timing.py > gpurun_out/ncu_full_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_raw.csv 2>/dev/null
QT_BATCH=2 ncu --set full --clock-control none --import-source on -k regex:"sd_|prep|xpass|ypass|post" -s 10 -c 5 \
    -o gpurun_out/prof_${TAG}_b2 -f python tools/quick_timing.py > gpurun_out/ncu_full_${TAG}_b2.log 2>&1
ncu -i gpurun_out/prof_${TAG}_b2.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_b2_raw.csv 2>/dev/null
echo done
