bash tools/gpu/variants.sh "base:" "nl:-DHS_COMPOSE_NO_LIGHT" > /dev/null 2>&1
for rep in 1 2 3; do for v in base nl; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
