bash tools/gpu/variants.sh "u24:" "u8:-DHS_SMOOTH_UNROLL_MAX=8" > /dev/null 2>&1
for c in C4 PR1 C2; do for rep in 1 2; do for v in u24 u8; do echo "== $c $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py $c 2>&1 | tail -1; done; done; done
