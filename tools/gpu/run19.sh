mkdir -p gpurun_out
bash tools/gpu/variants.sh "m4:" "m3:-DHS_SMOOTH_MINB=3" 2>&1
echo "== nogroup m4"; HS_GROUP_LAYERS=0 HS_LIB=/tmp/var_m4/libhybridsea_b200.so timeout 300 python tools/bench_kernels.py --stages compose,smooth 2>&1 | tail -2
