timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r53.log 2>&1; echo "gpu rc=$?"; tail -1 gpurun_out/r53.log
bash tools/gpu/ab.sh "compose_writes_background=True|compose_writes_background=False"
