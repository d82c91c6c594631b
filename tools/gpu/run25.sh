mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r25.log 2>&1; echo "gpu rc=$?"; tail -4 gpurun_out/r25.log
for rep in 1 2; do for v in 0 1; do echo "== stream=$v"; HS_ADVECT_STREAM=$v timeout 300 python tools/bench_kernels.py --stages advect 2>&1 | tail -1; done; done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r25_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r25_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('stages_ms'))"
