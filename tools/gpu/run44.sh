for d in _t_92699cb _t_28bde86; do
  (cd $d && python -c "from paper_2511_02852_b200 import build_lib; build_lib.build(verbose=False)" > /dev/null 2>&1 && echo "== $d" && timeout 600 python tools/skip_frame.py C3 2>&1 | grep "(none)" | head -1)
done
echo "== HEAD"; SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
