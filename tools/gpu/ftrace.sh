python -c "
from paper_2511_02852_b200 import build_lib
build_lib.build(out='/tmp/ftrace/libhybridsea_b200.so', extra=('-DHS_FFT_TRACE',), verbose=False)"
HS_LIB=/tmp/ftrace/libhybridsea_b200.so timeout 600 python tools/fft_trace.py 2>&1 | tail -20
