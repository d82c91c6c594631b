mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r10_gpu.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/r10_gpu.log
timeout 600 python bench.py --steps 300 --warmup 5 > gpurun_out/r10_bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/r10_bench.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/r10_ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/r10_ref.log
timeout 600 python bench.py --config C4 --exchange --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/r10_c4x.log 2>&1; echo "c4x rc=$?"; tail -c 600 gpurun_out/r10_c4x.log
