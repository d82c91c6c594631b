mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r16.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r16.log
bash tools/gpu/variants.sh "cur:"
