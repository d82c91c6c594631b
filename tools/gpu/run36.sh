timeout 900 python -m pytest tests -m gpu -q -x -k "scene or parity or exchange or cascade or output" > gpurun_out/r36.log 2>&1; echo "gpu rc=$?"; tail -2 gpurun_out/r36.log
timeout 300 python tools/bench_kernels.py --stages compose 2>&1 | tail -1
SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
