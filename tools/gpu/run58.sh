bash tools/gpu/variants.sh "u24:" "u12:-DHS_SMOOTH_UNROLL_MAX=12" "u10:-DHS_SMOOTH_UNROLL_MAX=10" "u8:-DHS_SMOOTH_UNROLL_MAX=8" "u6:-DHS_SMOOTH_UNROLL_MAX=6" > /dev/null 2>&1
for rep in 1 2 3; do for v in u24 u12 u10 u8 u6; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
for v in u24 u12 u8; do echo "== smooth $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so timeout 300 python tools/bench_kernels.py --stages smooth 2>&1 | tail -1; done
