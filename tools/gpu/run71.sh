for rep in 1 2; do for o in 0 2 1; do echo "== occ=$o"; HS_RES_OCC=$o SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
