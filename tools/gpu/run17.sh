mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "synth or smooth or scene or layer" > gpurun_out/r17.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r17.log
for p in 0 1; do echo "== persist=$p"; HS_SMOOTH_PERSIST=$p timeout 300 python tools/bench_kernels.py --stages compose,smooth,fft 2>&1 | tail -4; done
