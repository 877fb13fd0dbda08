OUT=gpurun_out/r02full6b; mkdir -p $OUT
python tools/one_call.py C3 sort 2 > $OUT/one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile_hist|k_scatter|k_split_count|k_split_scatter|k_tile_sort|k_merge_level|k_merge_partition" -s 35 -c 9 -o $OUT/full python tools/one_call.py C3 sort 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
