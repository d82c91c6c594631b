mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r12_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/r12_gpu.log
timeout 900 python tools/ref_suite.py > gpurun_out/ref_suite.log 2>&1; echo rc=$?; tail -3 gpurun_out/ref_suite.log
