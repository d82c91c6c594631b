# bench lines of the other BASELINE scenes (one GPU)
mkdir -p gpurun_out
TAG=${1:-r02}
for c in PR1 C2 C4; do
  timeout 900 python bench.py --config $c --steps 500 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config C5 --patches 8 --steps 300 --no-cpu-baseline > gpurun_out/${TAG}_bench_C5_8.json 2> gpurun_out/${TAG}_bench_C5_8.err; echo "C5_8 rc=$?"
timeout 900 python bench.py --deterministic --steps 500 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3_det.json 2> gpurun_out/${TAG}_bench_c3_det.err; echo "det rc=$?"
timeout 900 python bench.py --exchange --steps 500 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3_exch.json 2> gpurun_out/${TAG}_bench_c3_exch.err; echo "exch rc=$?"
for f in gpurun_out/${TAG}_bench_*.json; do python -c "
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d['config'].get('workload'), d['config'].get('live_particles'), round(d['ms_per_step']*1e3,2), '%.3g'%d['value'], '%.3g'%d['e2e']['value'])
except Exception as e: print(sys.argv[1], 'ERR', e)
" $f; done
