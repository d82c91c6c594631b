python -c "
from paper_2511_02852_b200 import build_lib
build_lib.build(out='/tmp/skip/libhybridsea_b200.so', extra=('-DHS_EXP_SKIP',), verbose=False)"
SKIP_SETS="|clear|composite|clear,composite|" HS_LIB=/tmp/skip/libhybridsea_b200.so timeout 600 python tools/skip_frame.py C3 2>&1 | tail -5
