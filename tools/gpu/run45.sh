bash tools/gpu/variants.sh "cur:" "wide:-DHS_SMOOTH_WIDE_TILES" > /dev/null 2>&1
for rep in 1 2; do
for v in cur wide; do echo "== $v narrow0"; HS_SMOOTH_NARROW=0 HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done
done
