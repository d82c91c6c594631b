# build library variants (-D flags) and time the frame's kernels with each
# usage: bash tools/gpu/variants.sh "NAME1:-DFLAG=1 -DX" "NAME2:" ...
mkdir -p gpurun_out
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  python - "$name" $flags <<'PY'
import sys
from paper_2511_02852_b200 import build_lib
name, flags = sys.argv[1], tuple(sys.argv[2:])
build_lib.build(out=f"/tmp/var_{name}/libhybridsea_b200.so", extra=flags, verbose=False)
PY
done
for spec in "$@"; do
  name="${spec%%:*}"
  echo "== $name"
  HS_LIB=/tmp/var_${name}/libhybridsea_b200.so timeout 300 python tools/bench_kernels.py --stages compose,smooth,fft 2>&1 | tail -4
done
