mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r28.log 2>&1; echo "gpu rc=$?"; tail -4 gpurun_out/r28.log
timeout 300 python tools/bench_kernels.py --stages compose,smooth 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r28_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r28_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d.get('stages_ms'))"
