set -x
OUT=${1:-gpurun_out/r02n}
mkdir -p $OUT
python tools/one_call.py C3 sort 2 > $OUT/one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${2:-k_tree_merge}" -s 1 -c 1 -o $OUT/full python tools/one_call.py C3 sort 2 > $OUT/ncu.log 2>&1
ls -la $OUT
