# full ncu captures of the C3 frame's kernels + launch list (one GPU)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"^(compose|advect_resident|smooth|fft_rows|fft_cols|inject)" -c 6 \
    -o gpurun_out/prof_full -f python tools/prof_frame.py --frames 2 > gpurun_out/prof_full.log 2>&1
echo "full rc=$?"
bash tools/ncu_launches.sh gpurun_out/prof_launches.csv 4
echo "launches rc=$?"
