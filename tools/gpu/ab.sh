mkdir -p gpurun_out
timeout 600 python tools/ab_sched.py ${@} > gpurun_out/ab_sched.log 2>&1; echo rc=$?; tail -8 gpurun_out/ab_sched.log
