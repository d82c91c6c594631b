for rep in 1 2; do for o in group_h coarse_first fine_first natural; do echo "== $o"; HS_SMOOTH_ORDER=$o SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
