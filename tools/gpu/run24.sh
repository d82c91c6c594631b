bash tools/gpu/variants.sh "cur:" "nosplat:-DHS_EXP_NOSPLAT" 2>&1 | grep -v "fft\|compose\|smooth"
for v in cur nosplat; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so timeout 300 python tools/bench_kernels.py --stages advect 2>&1 | tail -1; done
