mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r23_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r23_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('stages_ms')); print(json.dumps(d['roofline'])[:1500])"
