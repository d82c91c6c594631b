python -c "
from paper_2511_02852_b200 import build_lib
build_lib.build(out='/tmp/itrace/libhybridsea_b200.so', extra=('-DHS_INJECT_TRACE',), verbose=False)"
HS_LIB=/tmp/itrace/libhybridsea_b200.so timeout 600 python tools/inject_trace.py ${1:-C3} 2>&1 | tail -8
