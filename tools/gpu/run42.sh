echo "== default"; SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
echo "== no configure"; HS_NO_CONFIGURE=1 SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
echo "== global"; HS_CAPTURE_MODE=global SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
echo "== wide smooth tiles"; HS_SMOOTH_NARROW=0 HS_NO_CONFIGURE=1 HS_CAPTURE_MODE=global HS_POOL_STREAMS=1 SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
