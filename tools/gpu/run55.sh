bash tools/gpu/variants.sh "new:" > /dev/null 2>&1
git_old=1
for rep in 1 2; do echo "== new"; SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done
timeout 300 python tools/bench_kernels.py --stages compose 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r55.log 2>&1; echo "gpu rc=$?"; tail -1 gpurun_out/r55.log
