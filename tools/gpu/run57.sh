bash tools/gpu/variants.sh "base:" "u16:-DHS_SMOOTH_UNROLL_MAX=16" "u12:-DHS_SMOOTH_UNROLL_MAX=12" "res4:-DHS_RES_MINB=4" "cm8:-DHS_COMPOSE_MINB=8" "sm3:-DHS_SMOOTH_MINB=3" > /dev/null 2>&1
for rep in 1 2; do for v in base u16 u12 res4 cm8 sm3; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
