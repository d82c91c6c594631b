mkdir -p gpurun_out
TAG=${1:-pc}
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"^(compose|smooth)" -c 2 \
    -o gpurun_out/${TAG}_full -f python tools/prof_frame.py --frames 1 > gpurun_out/${TAG}_full.log 2>&1
echo "full rc=$?"
