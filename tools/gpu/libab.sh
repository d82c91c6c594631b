#!/bin/bash
# A/B of library builds on the C3 frame (mean of 300 L2-flushed frames per run, alternating):
# bash tools/gpu/libab.sh <scene> <libA> <libB> ... ; "-" = the product library
scene=$1; shift
for r in 1 2 3; do
  for L in "$@"; do
    if [ "$L" = "-" ]; then unset HS_LIB; else export HS_LIB=$L; fi
    echo "== $L"; SKIP_SETS="" timeout 300 python tools/skip_frame.py $scene 2>&1 | tail -1
  done
done
unset HS_LIB
for L in "$@"; do
  if [ "$L" = "-" ]; then unset HS_LIB; else export HS_LIB=$L; fi
  echo "== kernels $L"; timeout 300 python tools/bench_kernels.py --stages compose 2>&1 | tail -2
done
