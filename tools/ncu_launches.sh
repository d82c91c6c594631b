#!/bin/bash
# Per-kernel device times + DRAM bytes of steady-state C3 frames (run under gpurun):
#   bash tools/ncu_launches.sh <out.csv> [frames]
# Only the profiled region of tools/prof_frame.py is captured.
OUT=${1:-gpurun_out/launches.csv}
FR=${2:-4}
shift 2 2>/dev/null
EXTRA="$@"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file $OUT python tools/prof_frame.py --frames $FR $EXTRA \
    > gpurun_out/ncu_launches.log 2>&1
