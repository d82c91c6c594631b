mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r21.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/r21.log
for rep in 1 2; do for g in 0 1; do echo "== group=$g"; HS_GROUP_LAYERS=$g timeout 300 python tools/bench_kernels.py --stages compose,smooth 2>&1 | tail -2; done; done
