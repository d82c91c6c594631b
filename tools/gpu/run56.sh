# A/B of the last compose change by library variant: HEAD vs HEAD~1 compose.cu
mkdir -p /tmp/abc && git_show() { :; }
python - <<'PY'
import subprocess, os
from paper_2511_02852_b200 import build_lib
build_lib.build(out='/tmp/var_new/libhybridsea_b200.so', verbose=False)
PY
cp paper_2511_02852_b200/csrc/compose.cu /tmp/compose_new.cu
cp tools/gpu/compose_prev.cu paper_2511_02852_b200/csrc/compose.cu
python -c "from paper_2511_02852_b200 import build_lib; build_lib.build(out='/tmp/var_old/libhybridsea_b200.so', verbose=False)"
cp /tmp/compose_new.cu paper_2511_02852_b200/csrc/compose.cu
for rep in 1 2 3; do for v in old new; do echo "== $v"; HS_LIB=/tmp/var_$v/libhybridsea_b200.so SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
