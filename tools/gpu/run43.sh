cd _oldtree && python -c "from paper_2511_02852_b200 import build_lib; build_lib.build(verbose=False)" && timeout 600 python tools/skip_frame.py C3 2>&1 | grep "(none)" | head -1; cd ..
echo "== new"; SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
