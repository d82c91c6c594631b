for v in "new:" "old:-DHS_INJECT_SEPARATE_SINCOS"; do n=${v%%:*}; f=${v#*:}; python -c "
import sys
from paper_2511_02852_b200 import build_lib
build_lib.build(out='/tmp/it_$n/libhybridsea_b200.so', extra=tuple(['-DHS_INJECT_TRACE'] + sys.argv[1:]), verbose=False)" $f; done
for rep in 1 2; do for n in old new; do echo "== $n"; HS_LIB=/tmp/it_$n/libhybridsea_b200.so timeout 300 python tools/inject_trace.py C3 2>&1 | tail -1; done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "inject or parity or scene" > gpurun_out/r62.log 2>&1; echo "gpu rc=$?"; tail -1 gpurun_out/r62.log
