timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r66.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r66.log
timeout 300 python tools/bench_kernels.py --stages compose,smooth 2>&1 | tail -2
for rep in 1 2 3; do SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done
