mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "fft or scene or cascade" > gpurun_out/r15.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r15.log
bash tools/gpu/variants.sh "cur:"
