#!/bin/bash
# Per-kernel device times of steady-state C3 frames (run under gpurun):
#   bash tools/ncu_launches.sh <out.csv> [frames]
OUT=${1:-gpurun_out/launches.csv}
FR=${2:-4}
CMD="python tools/prof_frame.py --frames $FR"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
PER=$(python -c "import re;print(re.search(r'launches/frame (\d+)', open('gpurun_out/prof_plain.log').read()).group(1))")
SKIP=$((2003 * PER))
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^(fft_|inject|advect|smooth|compose|splat|normals)" -s $SKIP -c $((FR * PER)) --csv --log-file $OUT $CMD > gpurun_out/ncu_launches.log 2>&1
