mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r27.log 2>&1; echo "gpu rc=$?"; tail -4 gpurun_out/r27.log
bash tools/gpu/itrace.sh
bash tools/gpu/skip.sh 2>&1 | head -12
