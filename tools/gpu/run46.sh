bash tools/gpu/variants.sh "u24:" "u16:-DHS_SMOOTH_UNROLL_MAX=16" "u8:-DHS_SMOOTH_UNROLL_MAX=8" "u6:-DHS_SMOOTH_UNROLL_MAX=6" 2>&1 | grep -v "fft\|compose"
for rep in 1 2; do for v in u24 u16 u8 u6; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
