bash tools/gpu/variants.sh "u8:" "u6:-DHS_SMOOTH_UNROLL_MAX=6" "u5:-DHS_SMOOTH_UNROLL_MAX=5" "u4:-DHS_SMOOTH_UNROLL_MAX=4" > /dev/null 2>&1
for c in C3 PR1; do for rep in 1 2; do for v in u8 u6 u5 u4; do echo "== $c $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py $c 2>&1 | tail -1; done; done; done
