timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r47.log 2>&1; echo "gpu rc=$?"; tail -2 gpurun_out/r47.log
bash tools/gpu/ab.sh "compose_split=True|compose_split=False"
