# full round-end check on one GPU: tests, smoke, bench (ours + reference arm), launch list
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu.log 2>&1; echo "gpu rc=$?"; tail -2 gpurun_out/${TAG}_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?"
tail -c 400 gpurun_out/${TAG}_bench_ref.json
bash tools/ncu_launches.sh gpurun_out/${TAG}_launches.csv 4; echo "launches rc=$?"
python tools/launch_table.py gpurun_out/${TAG}_launches.csv 4 | tail -9
