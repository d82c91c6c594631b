mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_scenes.py -m gpu -q -x > gpurun_out/r22.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/r22.log
bash tools/gpu/variants.sh "m4:" "m1:-DHS_SMOOTH_MINB=1" 2>&1 | grep -v fft
for v in m4 m1; do echo "== $v nogroup"; HS_GROUP_LAYERS=0 HS_LIB=/tmp/var_$v/libhybridsea_b200.so timeout 300 python tools/bench_kernels.py --stages compose,smooth 2>&1 | tail -2; done
