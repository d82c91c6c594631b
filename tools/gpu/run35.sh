bash tools/gpu/variants.sh "nosplat:-DHS_EXP_NOSPLAT" > /dev/null 2>&1
HS_LIB=/tmp/var_nosplat/libhybridsea_b200.so ncu --set full --clock-control none --profile-from-start off \
    -k regex:"^advect_resident" -c 1 -o gpurun_out/adv_nosplat -f python tools/prof_frame.py --frames 1 > gpurun_out/adv_nosplat.log 2>&1
echo "rc=$?"
