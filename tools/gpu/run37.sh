timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x > gpurun_out/r37.log 2>&1; echo "cur rc=$?"; tail -2 gpurun_out/r37.log
grep -n "Error" gpurun_out/r37.log | head -5
