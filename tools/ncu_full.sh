#!/bin/bash
# One `ncu --set full` capture per matched kernel of a steady-state C3 frame
# (run under gpurun, one GPU):  bash tools/ncu_full.sh <out-basename> <regex> <matches-per-frame>
OUT=${1:-gpurun_out/full}
RE=${2:-"^(compose|advect_scatter|smooth|inject)"}
PER=${3:-4}
SKIP=$((2003 * PER))
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $PER \
    -o $OUT -f python tools/prof_frame.py --frames 2 > ${OUT}.log 2>&1
