#!/bin/bash
# In-frame A/B/C... of environment settings on the bench (under gpurun):
#   bash tools/ab_multi.sh <rounds> "<envA>" "<envB>" ...    (BENCH_ARGS for extra bench flags)
R=$1; shift
for i in $(seq 1 $R); do
  for E in "$@"; do
    env $E timeout 500 python bench.py --steps 1000 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$E]', round(d['ms_per_step']*1e3,2), round(d['step_ms_percentiles']['p50']*1e3,2), {k: round(v*1e3,1) for k,v in d['stages_ms'].items() if k in ('advect','fft','frame')})"
  done
done
