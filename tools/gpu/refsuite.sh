mkdir -p gpurun_out
timeout 900 python tools/ref_suite.py > gpurun_out/ref_suite.log 2>&1; echo rc=$?; tail -3 gpurun_out/ref_suite.log
