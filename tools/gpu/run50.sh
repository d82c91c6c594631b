timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r50.log 2>&1; echo "gpu rc=$?"; tail -2 gpurun_out/r50.log
bash tools/gpu/ab.sh "band_warps=0|band_warps=4|band_warps=8|band_warps=16"
