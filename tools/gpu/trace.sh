mkdir -p gpurun_out
python -c "
from paper_2511_02852_b200 import build_lib
build_lib.build(out='/tmp/trace/libhybridsea_b200.so', extra=('-DHS_COMPOSE_TRACE',), verbose=False)"
HS_LIB=/tmp/trace/libhybridsea_b200.so timeout 300 python tools/compose_trace.py > gpurun_out/trace.log 2>&1; echo rc=$?
head -14 gpurun_out/trace.log
bash tools/ncu_launches.sh gpurun_out/t_launches.csv 4; python tools/launch_table.py gpurun_out/t_launches.csv 4 | tail -7
