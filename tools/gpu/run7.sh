mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r7_gpu.log 2>&1; echo "gpu rc=$?"
tail -20 gpurun_out/r7_gpu.log
bash tools/gpu/perf.sh ${1:-p3}
