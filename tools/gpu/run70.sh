timeout 600 python -m pytest tests -m gpu -q -x -k "parity or scene or api or output" > gpurun_out/r70.log 2>&1; echo "gpu rc=$?"; tail -1 gpurun_out/r70.log
bash tools/gpu/ab.sh "compose_param_layers=True|compose_param_layers=False"
