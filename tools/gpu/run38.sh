for k in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q -x -k "scene or parity or exchange or cascade or output" > gpurun_out/r38.log 2>&1; echo "gpu rc=$?"; tail -1 gpurun_out/r38.log; done
timeout 300 python tools/bench_kernels.py --stages compose 2>&1 | tail -1
