(cd _headtree && python -c "from paper_2511_02852_b200 import build_lib; build_lib.build(verbose=False)" > /dev/null 2>&1)
for rep in 1 2; do
  echo "== head"; (cd _headtree && timeout 300 python tools/bench_kernels.py --stages compose,smooth,fft,advect 2>&1 | tail -4)
  echo "== tma"; timeout 300 python tools/bench_kernels.py --stages compose,smooth,fft,advect 2>&1 | tail -4
done
