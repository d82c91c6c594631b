bash tools/gpu/variants.sh "base:" "r4:-DHS_FFT_ROWS_MINB=4" "r5:-DHS_FFT_ROWS_MINB=5" "c3:-DHS_FFT_COLS_MINB=3" "c4:-DHS_FFT_COLS_MINB=4" 2>&1 | grep fft
for rep in 1 2; do for v in base r4 r5 c3 c4; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
