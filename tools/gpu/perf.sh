# bench + launch list + full ncu capture of the top kernels (one GPU)
mkdir -p gpurun_out
TAG=${1:-p}
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/${TAG}_bench.log
bash tools/ncu_launches.sh gpurun_out/${TAG}_launches.csv 4; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"^(compose|advect_resident|fft_rows|fft_cols)" -c 4 \
    -o gpurun_out/${TAG}_full -f python tools/prof_frame.py --frames 2 > gpurun_out/${TAG}_full.log 2>&1
echo "full rc=$?"
