mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r14_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/r14_gpu.log
bash tools/gpu/variants.sh "b9:" "b10:-DHS_COMPOSE_MINB=10" "b8:-DHS_COMPOSE_MINB=8"
