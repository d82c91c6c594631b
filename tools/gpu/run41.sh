for rep in 1 2; do for v in 0 1; do echo "== pool=$v"; HS_POOL_STREAMS=$v SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1; done; done
