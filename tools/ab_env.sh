#!/bin/bash
# A/B of an environment toggle on the C3 bench (under gpurun):
#   bash tools/ab_env.sh "<envA>" "<envB>" [rounds]     e.g. "HS_ADVECT_STATIC=1" ""
A=$1; B=$2; R=${3:-3}
for i in $(seq 1 $R); do
  for E in "$A" "$B"; do
    env $E timeout 500 python bench.py --steps 1000 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$E]', round(d['ms_per_step']*1e3,2), round(d['step_ms_percentiles']['p50']*1e3,2), {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})"
  done
done
