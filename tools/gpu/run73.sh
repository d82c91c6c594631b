bash tools/gpu/variants.sh "m4:" "m5:-DHS_SMOOTH_MINB=5" "m6:-DHS_SMOOTH_MINB=6" > /dev/null 2>&1
for rep in 1 2; do for v in m4 m5 m6; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
for v in m4 m5; do for c in PR1; do echo "== $c $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py $c 2>&1 | tail -1; done; done
