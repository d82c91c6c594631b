set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_scenes.py -x -q -s > gpurun_out/r1_scenes.log 2>&1; echo "scenes rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_scenes.py > gpurun_out/r1_gpu.log 2>&1; echo "gpu rc=$?"
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/r1_scenes.log gpurun_out/r1_gpu.log; tail -c 3000 gpurun_out/r1_bench.log
