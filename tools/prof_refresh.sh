# Round profile refresh: bench line, launch list, ncu full capture (second call of one_call.py)
set -x
OUT=gpurun_out/p6
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.log || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
python tools/one_call.py C3 sort 2 > $OUT/one.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_tile_hist|k_scatter|k_split_count|k_split_scatter|k_tile_sort|k_merge_level|k_merge_partition" -s 33 -c 7 -o $OUT/full python tools/one_call.py C3 sort 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
