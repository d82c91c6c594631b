timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r48.log 2>&1; echo "gpu rc=$?"; tail -2 gpurun_out/r48.log
timeout 300 python tools/bench_kernels.py --stages compose,interior 2>&1 | tail -2
bash tools/gpu/ab.sh "compose_split=True|compose_split=False"
