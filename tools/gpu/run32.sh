mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r32.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r32.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r32_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r32_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
