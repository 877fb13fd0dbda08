mkdir -p gpurun_out/s2
python tools/one_call.py C3 sort 2 > gpurun_out/s2/one.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_split_pass" -s 2 -c 2 -o gpurun_out/s2/split python tools/one_call.py C3 sort 2 > gpurun_out/s2/ncu.log 2>&1
