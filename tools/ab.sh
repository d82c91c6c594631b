#!/bin/bash
# A/B of two library builds on the C3 bench (under gpurun): bash tools/ab.sh <libA> <libB> [rounds]
A=$1; B=$2; R=${3:-3}
for i in $(seq 1 $R); do
  for L in $A $B; do
    HS_LIB=$L timeout 500 python bench.py --steps 1000 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step']*1e3,2), round(d['step_ms_percentiles']['p50']*1e3,2), {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})"
  done
done
