(cd _headtree && python -c "from paper_2511_02852_b200 import build_lib; build_lib.build(verbose=False)" > /dev/null 2>&1)
for rep in 1 2 3; do
  echo "== head"; (cd _headtree && SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1)
  echo "== tma"; SKIP_SETS="|" timeout 600 python tools/skip_frame.py C3 2>&1 | tail -1
done
