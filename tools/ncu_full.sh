#!/bin/bash
# One `ncu --set full` capture per matched kernel of steady-state C3 frames
# (run under gpurun, one GPU):  bash tools/ncu_full.sh <out-basename> <regex> <count>
# Only the profiled region of tools/prof_frame.py (cudaProfilerStart/Stop
# around the last frames) is captured.
OUT=${1:-gpurun_out/full}
RE=${2:-"^(compose|advect|smooth|inject|append)"}
CNT=${3:-8}
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$RE" -c $CNT \
    -o $OUT -f python tools/prof_frame.py --frames 3 > ${OUT}.log 2>&1
