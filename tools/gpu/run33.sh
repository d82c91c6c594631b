bash tools/gpu/variants.sh "ct4:" "ct8:-DHS_FFT_COLS_MIN_CT=8" 2>&1 | grep -v "compose\|smooth"
for v in ct4 ct8; do echo "== frame $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -2; done
