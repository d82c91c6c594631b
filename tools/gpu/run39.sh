timeout 900 python -m pytest tests -m gpu -q -x -v -k "scene or parity or exchange or cascade or output" > gpurun_out/r39a.log 2>&1; echo "subset rc=$?"; grep -E "PASSED|FAILED" gpurun_out/r39a.log | head
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r39b.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/r39b.log
