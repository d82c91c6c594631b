bash tools/gpu/variants.sh "cur:" "nosplat:-DHS_EXP_NOSPLAT" > /dev/null 2>&1
for v in cur nosplat; do for sf in 0 1; do echo "== $v stream=$sf"; HS_ADVECT_STREAM=$sf HS_LIB=/tmp/var_$v/libhybridsea_b200.so timeout 300 python tools/bench_kernels.py --stages advect 2>&1 | tail -1; done; done
