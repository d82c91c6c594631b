bash tools/gpu/variants.sh "ct4:" "ct2:-DHS_FFT_COLS_CT=2" "ct1:-DHS_FFT_COLS_CT=1" 2>&1 | grep -v "compose\|smooth"
for rep in 1 2; do for v in ct4 ct2 ct1; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
