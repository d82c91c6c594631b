mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_api.py -q -x > gpurun_out/r13_api.log 2>&1; echo "api rc=$?"; tail -30 gpurun_out/r13_api.log
timeout 900 python tools/ref_suite.py > gpurun_out/ref_suite.log 2>&1; echo rc=$?; tail -2 gpurun_out/ref_suite.log
